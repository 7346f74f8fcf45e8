set -u
timeout 900 python bench.py --no-cpu-baseline --no-bulksync > gpurun_out/g5_bench.json 2> gpurun_out/g5_bench.err; echo bench rc $?
timeout 600 python bench.py --precision bf16 --no-cpu-baseline --no-bulksync > gpurun_out/g5_bench_bf16.json 2>> gpurun_out/g5_bench.err
python -c "import json; [print(f, json.load(open(f))['ms_per_step']) for f in ('gpurun_out/g5_bench.json','gpurun_out/g5_bench_bf16.json')]"
timeout 300 python tools/phase_trace.py 16384 128 0 > gpurun_out/g5_trace_fp32.txt 2>&1
timeout 300 python tools/phase_trace.py 16384 128 1 > gpurun_out/g5_trace_bf16.txt 2>&1
head -12 gpurun_out/g5_trace_fp32.txt
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/g5_pytest.log 2>&1; echo pytest rc $?
tail -5 gpurun_out/g5_pytest.log
timeout 600 python tools/configs.py > gpurun_out/g5_configs.jsonl 2>&1; cat gpurun_out/g5_configs.jsonl
