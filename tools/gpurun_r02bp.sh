RSB_DEBUG=4 timeout 900 python tools/halo_fail_probe.py pair s1024 2>&1 | grep -E "launches|mask" | tail -6
timeout 900 python -m pytest tests/test_gpu_halo.py -q -x > gpurun_out/r02bp_pytest_halo.log 2>&1; echo pytest_halo=$?; tail -15 gpurun_out/r02bp_pytest_halo.log
python - <<'PY'
import os, sys
sys.path.insert(0, '.')
from paper_2509_04277_b200 import workloads as wl
from paper_2509_04277_b200.engine import Engine
def us(make, k, launches):
    with Engine(make()) as eng:
        dev = eng.device_world
        dev.run(k); dev.synchronize()
        dev.timer_start()
        for _ in range(launches): dev.run(k)
        dev.timer_stop()
        ms = dev.timer_ms()
        redo = dev.last_redo_count()
        return round(ms * 1e3 / (k * launches), 2), redo
for name, mk in (("pair", wl.pair), ("s256", lambda: wl.sweep(256)), ("s1024", lambda: wl.sweep(1024)), ("s16384", lambda: wl.sweep(16384))):
    print(name, {k: us(mk, k, max(2, min(200, 2000 // k))) for k in (1, 10, 100)}, flush=True)
PY
