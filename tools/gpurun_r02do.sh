timeout 300 python tools/env_probe.py extensible 10 RSB_HALO_CTAS 1,2,4,8
timeout 300 python tools/env_probe.py extensible 100 RSB_HALO_CTAS 1,2,4,8
timeout 300 python tools/env_probe.py sweep128 100 RSB_HALO_CTAS 1,2,4
timeout 300 python tools/env_probe.py pair 10 RSB_HALO_CTAS 8,12
