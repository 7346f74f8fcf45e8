#!/bin/bash
# On the GPU box: bench line, ncu launch list of the bench command, one `--set full` capture of the
# layer kernel (c4 shape). Outputs under gpurun_out/ (summarised into profiles/ by tools/ncu_summary.py).
set -u
TAG=${1:-r01}
make -C oracle >/dev/null 2>&1
timeout 900 python bench.py > gpurun_out/bench_${TAG}.json 2> gpurun_out/bench_${TAG}.err
timeout 600 python bench.py --precision bf16 --no-cpu-baseline > gpurun_out/bench_${TAG}_bf16.json 2>> gpurun_out/bench_${TAG}.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file gpurun_out/launches_${TAG}.csv python bench.py --steps 3 --warmup 3 --e2e-steps 1 --no-cpu-baseline \
    > gpurun_out/ncu_launch_${TAG}.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:fdmoe_layer --launch-skip 2 -c 1 \
    -o gpurun_out/prof_${TAG}_full python tools/run_layer.py 16384 128 0 3 > gpurun_out/ncu_full_${TAG}.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:fdmoe_layer --launch-skip 2 -c 1 \
    -o gpurun_out/prof_${TAG}_full_bf16 python tools/run_layer.py 16384 128 1 3 > gpurun_out/ncu_full_${TAG}_bf16.log 2>&1
tail -c 600 gpurun_out/bench_${TAG}.json; echo; tail -c 300 gpurun_out/bench_${TAG}_bf16.json; echo
tail -2 gpurun_out/ncu_full_${TAG}.log
timeout 300 python tools/phase_trace.py 16384 128 0 > gpurun_out/phase_${TAG}_fp32.txt 2>&1
timeout 300 python tools/phase_trace.py 16384 128 1 > gpurun_out/phase_${TAG}_bf16.txt 2>&1
timeout 600 python tools/configs.py > gpurun_out/configs_${TAG}.jsonl 2>&1
