timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/r02dq_pytest_gpu.log 2>&1; echo pytest=$?; tail -3 gpurun_out/r02dq_pytest_gpu.log
RSB_XFER=0 timeout 600 python -m pytest tests/test_gpu_halo.py tests/test_gpu_acceptance.py tests/test_gpu_live.py -x -q 2>&1 | tail -1
