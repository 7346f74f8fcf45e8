set -u
timeout 300 python tools/phase_trace.py 16384 128 0 2>&1 | grep -i "effective\|^ffn \|^dispatch"
timeout 300 python tools/phase_trace.py 16384 128 1 2>&1 | grep -i "effective\|^ffn \|^dispatch"
timeout 2000 python -m pytest tests -m gpu -x -q --timeout 400 > gpurun_out/g9_pytest.log 2>&1; echo pytest rc $?
tail -3 gpurun_out/g9_pytest.log
