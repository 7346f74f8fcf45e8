set -u
timeout 300 python tools/dev/chunklog_fp32.py 2>&1 | grep -v "periods\|  issue\|  wait"
timeout 600 python bench.py --no-cpu-baseline --no-bulksync --e2e-steps 2 > gpurun_out/g7_bench.json 2> gpurun_out/g7_bench.err; echo bench rc $?
timeout 600 python bench.py --precision bf16 --no-cpu-baseline --no-bulksync --e2e-steps 2 > gpurun_out/g7_bench_bf16.json 2>> gpurun_out/g7_bench.err
python -c "import json; [print(f, json.load(open(f))['ms_per_step']) for f in ('gpurun_out/g7_bench.json','gpurun_out/g7_bench_bf16.json')]"

