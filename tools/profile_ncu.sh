#!/bin/bash
# On the GPU box: ncu launch list of the bench command, `--set full` captures of one warm layer launch (FP32, bf16)
# and the phase traces -- profile_round.sh without the bench lines and configs. Outputs under gpurun_out/.
set -u
TAG=${1:-r02e}
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file gpurun_out/launches_${TAG}.csv python bench.py --steps 3 --warmup 3 --e2e-steps 1 --no-cpu-baseline \
    > gpurun_out/ncu_launch_${TAG}.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:fdmoe_layer --launch-skip 2 -c 1 \
    -o gpurun_out/prof_${TAG}_full python tools/run_layer.py 16384 128 0 3 > gpurun_out/ncu_full_${TAG}.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:fdmoe_layer --launch-skip 2 -c 1 \
    -o gpurun_out/prof_${TAG}_full_bf16 python tools/run_layer.py 16384 128 1 3 > gpurun_out/ncu_full_${TAG}_bf16.log 2>&1
timeout 300 python tools/phase_trace.py 16384 128 0 > gpurun_out/phase_${TAG}_fp32.txt 2>&1
timeout 300 python tools/phase_trace.py 16384 128 1 > gpurun_out/phase_${TAG}_bf16.txt 2>&1
tail -2 gpurun_out/ncu_full_${TAG}.log
