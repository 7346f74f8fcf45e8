set -u
timeout 300 python tools/dev/pipe_rate3.py 2>&1
timeout 600 python tools/ablate.py 16384 128 0 2>&1 | cut -c1-120
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -3
