set -u
timeout 2000 python -m pytest tests -m gpu -q --timeout 600 > gpurun_out/g16_pytest.log 2>&1; echo pytest rc $?
tail -3 gpurun_out/g16_pytest.log
grep "_wide" gpurun_out/numerics.jsonl | python -c "import sys,json; [print(json.loads(l)['case'], json.loads(l)['rank'], round(json.loads(l)['max_err_over_bound'],3)) for l in sys.stdin]"
timeout 900 python bench.py --no-bulksync > gpurun_out/g16_bench.json 2> gpurun_out/g16_bench.err; echo bench rc $?
python -c "import json; d=json.load(open('gpurun_out/g16_bench.json')); print(d['ms_per_step'], d['roofline']['frac'], d['clocks']['in_kernel'], d['e2e']['value'])"
