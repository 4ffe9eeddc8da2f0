for r in 1 2; do for v in A B; do timeout 300 python tools/k1_launch_probe.py scratch/lib_$v.so; done; done
timeout 1500 python -m pytest tests/test_gpu_parity.py -x -q -k "lazy or speculative or one_warp or warp or cfg4 or sweep" 2>&1 | tail -2
