set -u
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/g1_pytest.log 2>&1; echo pytest rc $?
tail -5 gpurun_out/g1_pytest.log
timeout 600 python bench.py > gpurun_out/g1_bench.json 2> gpurun_out/g1_bench.err; echo bench rc $?
timeout 600 python bench.py --precision bf16 --no-cpu-baseline --no-bulksync > gpurun_out/g1_bench_bf16.json 2>> gpurun_out/g1_bench.err
timeout 300 python tools/phase_trace.py 16384 128 0 > gpurun_out/g1_trace_fp32.txt 2>&1
timeout 300 python tools/phase_trace.py 16384 128 1 > gpurun_out/g1_trace_bf16.txt 2>&1
timeout 600 python tools/configs.py > gpurun_out/g1_configs.jsonl 2>&1
cat gpurun_out/g1_bench.json; cat gpurun_out/g1_bench_bf16.json
