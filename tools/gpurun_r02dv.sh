for r in 1 2; do for v in A B; do timeout 120 python tools/grid_ab.py scratch/lib_$v.so; done; done
timeout 900 python -m pytest tests/test_gpu_halo.py tests/test_gpu_parity.py -x -q 2>&1 | tail -2
