set -u
timeout 300 python tools/phase_trace.py 16384 128 0 2>&1 | grep "^gate \|^barrier\|gate-route\|gate-exp\|gate-pairs\|gate-full\|kernel\|^ffn "
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_baseline.py -x -q --timeout 600 2>&1 | tail -2
for l in paper_2506_04667_b200/lib/libfdmoe.so ab_libs/libfdmoe_no_pickw.so; do python tools/ab.py $l 0; done
