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
        g = eng.plan()["groups"][0]
        return round(dev.timer_ms() * 1e3 / (k * launches), 2), bool(g.get("halo")), g.get("one_warp_rod")
for env in ({}, {"RSB_HALO_CTA": "1"}):
    os.environ.update(env)
    for name, mk in (("n16", lambda: wl.sweep(16)), ("n48", lambda: wl.sweep(48)), ("cfg1", wl.cantilever), ("n96", lambda: wl.sweep(96))):
        print(env, name, {k: us(mk, k, max(2, min(200, 2000 // k))) for k in (1, 10, 100)}, flush=True)
    for k in env: os.environ.pop(k)
PY
