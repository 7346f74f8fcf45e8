set -u
timeout 300 python tools/run_layer.py 4096 16 0 3 2>&1 | tail -1
timeout 600 python bench.py --no-cpu-baseline --no-bulksync --e2e-steps 2 > gpurun_out/g8_bench.json 2> gpurun_out/g8_bench.err; echo bench rc $?
python -c "import json; [print(f, json.load(open(f))['ms_per_step']) for f in ('gpurun_out/g8_bench.json',)]"
timeout 300 python tools/phase_trace.py 16384 128 0 > gpurun_out/g8_trace_fp32.txt 2>&1; head -8 gpurun_out/g8_trace_fp32.txt; tail -9 gpurun_out/g8_trace_fp32.txt
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_baseline.py tests/test_gpu_schedule.py -x -q --timeout 300 2>&1 | tail -3
