set -u
timeout 300 python tools/dev/chunklog_conv.py 2>&1 | tail -2
timeout 600 python bench.py --no-cpu-baseline --no-bulksync --e2e-steps 2 > gpurun_out/g14_bench.json 2> gpurun_out/g14_bench.err; echo bench rc $?
python -c "import json; d=json.load(open('gpurun_out/g14_bench.json')); print(d['ms_per_step'], d['roofline']['frac'], d['clocks']['in_kernel'])"
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_baseline.py -q --timeout 400 2>&1 | tail -2
