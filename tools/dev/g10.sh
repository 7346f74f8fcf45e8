set -u
timeout 300 python tools/phase_trace.py 16384 128 0 > gpurun_out/g10_trace_fp32.txt 2>&1; head -25 gpurun_out/g10_trace_fp32.txt
timeout 600 python bench.py --no-cpu-baseline --no-bulksync --e2e-steps 2 > gpurun_out/g10_bench.json 2> gpurun_out/g10_bench.err; echo bench rc $?
timeout 600 python bench.py --precision bf16 --no-cpu-baseline --no-bulksync --e2e-steps 2 > gpurun_out/g10_bench_bf16.json 2>> gpurun_out/g10_bench.err
python -c "import json; [print(f, json.load(open(f))['ms_per_step']) for f in ('gpurun_out/g10_bench.json','gpurun_out/g10_bench_bf16.json')]"
timeout 2000 python -m pytest tests -m gpu -x -q --timeout 400 > gpurun_out/g10_pytest.log 2>&1; echo pytest rc $?
tail -3 gpurun_out/g10_pytest.log
