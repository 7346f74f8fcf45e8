set -u
timeout 300 python tools/dev/pipe_rate.py > gpurun_out/g4_pipe.txt 2>&1; cat gpurun_out/g4_pipe.txt
timeout 1500 python -m pytest tests/test_gpu_faults.py -x -q > gpurun_out/g4_pytest.log 2>&1; echo pytest rc $?
tail -25 gpurun_out/g4_pytest.log
