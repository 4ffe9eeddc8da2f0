for r in 1 2; do for l in 8a31e56 98c8d9e c64883e current; do python tools/ab_probe.py build/ab/$l.so; done; done
