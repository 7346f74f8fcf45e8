set -u
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_baseline.py -x -q --timeout 400 2>&1 | tail -3
timeout 600 python bench.py --no-cpu-baseline --no-bulksync --e2e-steps 2 > gpurun_out/g15_bench.json 2> gpurun_out/g15_bench.err; echo bench rc $?
python -c "import json; d=json.load(open('gpurun_out/g15_bench.json')); print(d['ms_per_step'], d['roofline']['frac'], d['clocks']['in_kernel'])"
timeout 1200 python tools/dev/parity_wide.py 2>&1 | grep -v Warn
