#!/usr/bin/env python
"""One-warp single-rod kernel (rod_warp.cuh) vs the CTA kernel (RSB_RW=0):
bitwise state and device us/step for small sweep rods and cfg1."""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2509_04277_b200 import _lib  # noqa: E402
from paper_2509_04277_b200 import workloads as wl  # noqa: E402
from paper_2509_04277_b200.engine import Engine  # noqa: E402

STATE = ("positions", "velocities", "frames", "angular_velocities")


def run(make, k, launches, rw):
    os.environ["RSB_RW"] = rw
    w = make()
    with Engine(w) as eng:
        dev = eng.device_world
        plan = eng.plan()["groups"][0]
        dev.run(k)
        dev.synchronize()
        dev.timer_start()
        for _ in range(launches):
            dev.run(k)
        dev.timer_stop()
        us = dev.timer_ms() * 1e3 / (k * launches)
        redo = dev.last_redo_count()
        dev.download(_lib.RS_STATE)
    return w, us, plan, redo


def main():
    cases = {"cfg1": wl.cantilever}
    for n in (16, 15, 1, 2, 31, 33, 63, 64):
        cases[f"sweep{n}"] = (lambda n=n: wl.sweep(n))
    out = {}
    for name, make in cases.items():
        for k in (100,):
            a, us_a, plan_a, redo = run(make, k, 10, "1")
            os.environ["RSB_RW1"] = "0"
            c, us_c, _, _ = run(make, k, 10, "1")
            os.environ["RSB_RW1"] = "1"
            b, us_b, plan_b, _ = run(make, k, 10, "0")
            for s_ in STATE:
                assert np.array_equal(getattr(c, s_).view(np.int64), getattr(b, s_).view(np.int64)), (name, s_)
            diff = {s: int(np.count_nonzero(getattr(a, s).view(np.int64) != getattr(b, s).view(np.int64)))
                    for s in STATE}
            out[f"{name}_k{k}"] = {"warp_us": round(us_a, 3), "two_per_lane_us": round(us_c, 3),
                                   "cta_us": round(us_b, 3), "diff": diff,
                                   "one_warp": plan_a.get("one_warp_rod"), "rw1": os.environ.get("RSB_RW1"), "redo": redo}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
