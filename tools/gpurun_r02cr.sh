timeout 900 python -m pytest tests/test_gpu_halo.py -q -x -k "several or beside or fp32 or live_commands" > gpurun_out/r02cr_pytest.log 2>&1; echo pytest=$?; tail -25 gpurun_out/r02cr_pytest.log
