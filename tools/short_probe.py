#!/usr/bin/env python
"""Short one-CTA rods at K = 1 / 10: the general CTA kernel vs the wide-halo
kernel as one CTA (RSB_HALO_CTA=1); us/step and whether the two final
states are bit-identical."""
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2509_04277_b200 import workloads as wl  # noqa: E402
from paper_2509_04277_b200.engine import Engine  # noqa: E402


def run(n, k, launches, env):
    old = os.environ.get("RSB_HALO_CTA")
    if env is None:
        os.environ.pop("RSB_HALO_CTA", None)
    else:
        os.environ["RSB_HALO_CTA"] = env
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
            os.environ.pop("RSB_HALO_CTA", None)
        else:
            os.environ["RSB_HALO_CTA"] = old


for n in (8, 16, 24, 32, 38, 48, 63):
    for k in (1, 10):
        launches = 2000 // k
        a, ua, ha = run(n, k, launches, None)
        b, ub, hb = run(n, k, launches, "1")
        same = all(np.array_equal(getattr(a, f).view(np.int64), getattr(b, f).view(np.int64))
                   for f in ("positions", "velocities", "frames", "angular_velocities"))
        print(json.dumps({"n": n, "k": k, "default_us": ua, "default_halo": ha, "halo_us": ub,
                          "halo_planned": hb, "bitwise_equal": same}), flush=True)
