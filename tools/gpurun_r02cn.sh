for r in 1 2; do for l in base new; do python tools/ab_probe.py build/ab/$l.so; done; done
timeout 1500 python -m pytest tests/test_gpu_halo.py tests/test_gpu_parity.py tests/test_gpu_mesh.py tests/test_gpu_live.py tests/test_gpu_scenarios.py tests/test_gpu_acceptance.py -q -x > gpurun_out/r02cn_pytest.log 2>&1; echo pytest=$?; tail -3 gpurun_out/r02cn_pytest.log
