#!/usr/bin/env python
"""us/step of one workload under several values of one planner switch, and
whether every final state is bit-identical to the default's:
  python tools/env_probe.py extensible 10 RSB_HALO_CTAS 1,2,4,8,16"""
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2509_04277_b200 import workloads as wl  # noqa: E402
from paper_2509_04277_b200.engine import Engine  # noqa: E402

name, k, var, vals = sys.argv[1], int(sys.argv[2]), sys.argv[3], sys.argv[4].split(",")
make = getattr(wl, name) if not name.startswith("sweep") else (lambda: wl.sweep(int(name[5:])))
launches = max(20, 2000 // k)


def run(val):
    if val is None:
        os.environ.pop(var, None)
    else:
        os.environ[var] = val
    w = make()
    with Engine(w) as eng:
        dev = eng.device_world
        g = eng.plan()["groups"][0]
        dev.run(k)
        dev.synchronize()
        dev.timer_start()
        for _ in range(launches):
            dev.run(k)
        dev.timer_stop()
        us = dev.timer_ms() * 1e3 / (k * launches)
        dev.download()
    return w, round(us, 3), g.get("halo")


ref, us0, h0 = run(None)
print(json.dumps({"workload": name, "k": k, "default_us": us0, "halo": h0}), flush=True)
for v in vals:
    w, us, h = run(v)
    same = all(np.array_equal(getattr(w, f).view(np.int64), getattr(ref, f).view(np.int64))
               for f in ("positions", "velocities", "frames", "angular_velocities"))
    print(json.dumps({var: v, "us": us, "bitwise_equal": same, "halo": h}), flush=True)
