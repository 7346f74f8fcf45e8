set -u
timeout 1500 python -m pytest tests/test_gpu_faults.py -x -q -v > gpurun_out/g3_pytest.log 2>&1; echo pytest rc $?
tail -25 gpurun_out/g3_pytest.log
timeout 300 python tools/ab_debug.py 0 16384 128 0,4096 > gpurun_out/g3_ab.txt 2>&1
timeout 300 python tools/ab_debug.py 1 16384 128 0,4096 >> gpurun_out/g3_ab.txt 2>&1
timeout 600 python tools/ablate.py 16384 128 0 > gpurun_out/g3_ablate_fp32.txt 2>&1
cat gpurun_out/g3_ab.txt gpurun_out/g3_ablate_fp32.txt
