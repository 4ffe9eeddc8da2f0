timeout 900 python -m pytest tests/test_gpu_halo.py -q -x > gpurun_out/r02cs_pytest.log 2>&1; echo pytest=$?; tail -15 gpurun_out/r02cs_pytest.log
