# A/B: halo kernel waits for the previous grid only after its static loads
for r in 1 2; do for v in A B; do
  timeout 300 python tools/k1_launch_probe.py scratch/lib_$v.so
  timeout 300 python tools/ab_probe.py scratch/lib_$v.so
done; done
timeout 1200 python -m pytest tests/test_gpu_halo.py tests/test_gpu_parity.py tests/test_gpu_live.py tests/test_gpu_mesh.py -x -q 2>&1 | tail -3
