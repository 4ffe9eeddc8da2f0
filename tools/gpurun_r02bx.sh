timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/r02bx_pytest_gpu.log 2>&1; echo pytest=$?; tail -4 gpurun_out/r02bx_pytest_gpu.log
