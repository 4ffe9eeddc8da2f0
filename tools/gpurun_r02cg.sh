timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/r02cg_pytest_gpu.log 2>&1; echo pytest=$?; tail -3 gpurun_out/r02cg_pytest_gpu.log
