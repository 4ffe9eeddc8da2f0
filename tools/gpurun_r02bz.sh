python - <<'PY'
import sys
sys.path.insert(0, '.')
from paper_2509_04277_b200 import workloads as wl
from paper_2509_04277_b200.engine import Engine
def us(make, k, launches, **kw):
    with Engine(make(), **kw) as eng:
        dev = eng.device_world
        dev.run(k); dev.synchronize()
        dev.timer_start()
        for _ in range(launches): dev.run(k)
        dev.timer_stop()
        ms = dev.timer_ms()
        return round(ms * 1e3 / (k * launches), 2), dev.last_redo_count()
for name, mk in (("pair", wl.pair), ("s256", lambda: wl.sweep(256)), ("s1024", lambda: wl.sweep(1024)), ("s4096", lambda: wl.sweep(4096)), ("s16384", lambda: wl.sweep(16384))):
    print(name, {k: us(mk, k, max(2, min(200, 2000 // k))) for k in (1, 10, 100)}, flush=True)
PY
