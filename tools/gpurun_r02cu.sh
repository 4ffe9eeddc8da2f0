timeout 900 python -m pytest tests/test_gpu_halo.py tests/test_gpu_parity.py -q -x -k "cfg1 or halo or cantilever or one_cta" > gpurun_out/r02cu_pytest.log 2>&1; echo pytest=$?; tail -2 gpurun_out/r02cu_pytest.log
python tools/k1_host_probe.py
