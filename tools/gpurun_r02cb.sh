for r in 1 2; do for l in 8a31e56 current xf; do python tools/ab_probe.py build/ab/$l.so; done; done
timeout 900 python -m pytest tests/test_gpu_halo.py tests/test_gpu_live.py -q -x > gpurun_out/r02cb_pytest.log 2>&1; echo pytest=$?; tail -3 gpurun_out/r02cb_pytest.log
