for r in 1 2; do for v in A B; do timeout 300 python tools/k1_launch_probe.py scratch/lib_$v.so; done; done
