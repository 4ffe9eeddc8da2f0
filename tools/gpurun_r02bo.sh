RSB_DEBUG=4 timeout 900 python tools/halo_fail_probe.py pair 2>&1 | grep -v "^$" | tail -5
