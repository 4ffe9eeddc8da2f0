#!/usr/bin/env python
"""Extensible single rods (no distance projection: 3 phases per step): one
CTA vs a cluster, per size -- the planner's tier choice for such rods."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2509_04277_b200 import workloads as wl  # noqa: E402
from paper_2509_04277_b200.engine import Engine  # noqa: E402


def us(make, k=10, launches=50, **kw):
    with Engine(make(), **kw) as eng:
        dev = eng.device_world
        dev.run(k)
        dev.synchronize()
        dev.timer_start()
        for _ in range(launches):
            dev.run(k)
        dev.timer_stop()
        g = eng.plan()["groups"][0]
        return dev.timer_ms() * 1e3 / (k * launches), g["tier"], g["ctas"]


for n in (64, 128, 256, 384, 512):
    make = lambda n=n: wl.extensible(n, n / 512.0)  # noqa: E731
    row = [us(make)]
    for c in (2, 4, 8):
        try:
            row.append(us(make, force_tier=1, force_ctas=c))
        except Exception as exc:  # size not splittable that way
            row.append(str(exc)[:40])
    print(n, row, flush=True)
