for r in 1 2 3; do for v in A B; do timeout 300 python tools/haptic_ab.py scratch/lib_$v.so 2>&1 | tail -1; done; done
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_halo.py tests/test_gpu_acceptance.py tests/test_gpu_live.py -x -q 2>&1 | tail -1
