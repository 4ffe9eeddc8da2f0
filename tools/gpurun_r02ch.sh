timeout 900 python -m pytest tests/test_gpu_halo.py -q -x -k "past_one_cluster" > gpurun_out/r02ch_pytest.log 2>&1; echo pytest=$?; tail -20 gpurun_out/r02ch_pytest.log
