#!/usr/bin/env python
"""Short one-CTA rods: default plan vs one env switch (argv: VAR VALUE sizes
ks; default RSB_HALO_SHORT=2, the wide-halo kernel as one CTA for every
size); us/step and whether the two final states are bit-identical."""
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2509_04277_b200 import workloads as wl  # noqa: E402
from paper_2509_04277_b200.engine import Engine  # noqa: E402


VAR = sys.argv[1] if len(sys.argv) > 1 else "RSB_HALO_SHORT"
VAL = sys.argv[2] if len(sys.argv) > 2 else "2"
SIZES = tuple(int(x) for x in sys.argv[3].split(",")) if len(sys.argv) > 3 else (2, 4, 8, 12, 16, 20, 24, 32, 38)
KS = tuple(int(x) for x in sys.argv[4].split(",")) if len(sys.argv) > 4 else (1, 10)


def run(n, k, launches, env):
    old = os.environ.get(VAR)
    if env is None:
        os.environ.pop(VAR, None)
    else:
        os.environ[VAR] = env
    try:
        w = wl.sweep(n)
        with Engine(w) as eng:
            dev = eng.device_world
            halo = eng.plan()["groups"][0].get("halo") is not None
            dev.run(k)
            dev.synchronize()
            dev.timer_start()
            for _ in range(launches):
                dev.run(k)
            dev.timer_stop()
            us = dev.timer_ms() * 1e3 / (k * launches)
            dev.download()
        return w, round(us, 3), halo
    finally:
        if old is None:
            os.environ.pop(VAR, None)
        else:
            os.environ[VAR] = old


for n in SIZES:
    for k in KS:
        launches = 2000 // k
        a, ua, ha = run(n, k, launches, None)
        b, ub, hb = run(n, k, launches, VAL)
        same = all(np.array_equal(getattr(a, f).view(np.int64), getattr(b, f).view(np.int64))
                   for f in ("positions", "velocities", "frames", "angular_velocities"))
        print(json.dumps({"n": n, "k": k, "default_us": ua, "default_halo": ha, VAR + "=" + VAL: ub,
                          "halo_planned": hb, "bitwise_equal": same}), flush=True)
