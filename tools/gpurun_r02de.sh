timeout 300 python tools/k1_launch_probe.py
timeout 1200 python -m pytest tests/test_gpu_halo.py tests/test_gpu_parity.py tests/test_gpu_acceptance.py -x -q 2>&1 | tail -2
