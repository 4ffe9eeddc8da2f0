python - <<'PY'
import sys
sys.path.insert(0, '.')
from paper_2509_04277_b200 import workloads as wl, state as st
from paper_2509_04277_b200.engine import Engine
def unbound_pair():
    w = wl._world()
    for y in (1.5e-3, -1.5e-3):
        w.add_rod(st.init_rod(513, 1.0, axis=(0.0, 0.0, 1.0), origin=(0.0, y, -1.0)), st.RodParams(**wl.MATERIAL))
    w.finalize()
    for r in (0, 1):
        w.set_driver(r)
        w.driver_velocity[r] = (0.0, 0.0, 0.05)
    return w
def us(make, k, launches):
    with Engine(make()) as eng:
        dev = eng.device_world
        dev.run(k); dev.synchronize()
        dev.timer_start()
        for _ in range(launches): dev.run(k)
        dev.timer_stop()
        return round(dev.timer_ms() * 1e3 / (k * launches), 2), eng.plan()["groups"][0]["halo"]
print("bound pair", us(wl.pair, 100, 20))
print("unbound pair", us(unbound_pair, 100, 20))
print("single 512", us(lambda: wl.sweep(512, 1.0 / 512), 100, 20))
PY
