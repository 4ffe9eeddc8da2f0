timeout 900 python -m pytest tests/test_gpu_halo.py tests/test_gpu_parity.py -q -x -k "grab or halo or Grab" > gpurun_out/r02br_pytest.log 2>&1; echo pytest=$?; tail -15 gpurun_out/r02br_pytest.log
