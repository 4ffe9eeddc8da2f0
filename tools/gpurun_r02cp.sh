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
        h = eng.plan()["groups"][0].get("halo")
        return round(dev.timer_ms() * 1e3 / (k * launches), 2), h and h["ctas"]
for env in ({}, {"RSB_HALO_CTA": "1", "RSB_HALO_CTAS": "1"}, {"RSB_HALO_CTA": "1", "RSB_HALO_CTAS": "2"}, {"RSB_HALO_CTA": "1"}):
    os.environ.update(env)
    print(env, {n: {k: us(lambda: wl.sweep(n), k, max(2, min(200, 2000 // k))) for k in (10, 100)} for n in (32, 64, 96, 128)}, flush=True)
    for k in env: os.environ.pop(k)
PY
