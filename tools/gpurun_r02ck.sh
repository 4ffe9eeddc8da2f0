for r in 1 2; do for l in base new; do python tools/ab_probe.py build/ab/$l.so; done; done
timeout 900 python -m pytest tests/test_gpu_halo.py tests/test_gpu_parity.py -q -x -k "pair or bind or halo or column" > gpurun_out/r02ck_pytest.log 2>&1; echo pytest=$?; tail -2 gpurun_out/r02ck_pytest.log
