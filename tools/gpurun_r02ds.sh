for r in 1 2 3; do for v in A B; do timeout 300 python tools/frame_probe.py scratch/lib_$v.so 2>&1 | head -1; done; done
timeout 1500 python -m pytest tests/test_gpu_live.py tests/test_gpu_acceptance.py tests/test_gpu_service.py tests/test_gpu_scenarios.py tests/test_gpu_refcore.py tests/test_gpu_halo.py -x -q 2>&1 | tail -2
