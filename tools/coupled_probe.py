#!/usr/bin/env python
"""Coupled tier (one rod per CTA, mirrored bindings) vs the cluster tier
(RSB_COUPLED=0) on the cfg3 pair: bitwise state and device us/step."""
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


def run(on, k, launches, live=False):
    os.environ["RSB_COUPLED"] = on
    w = wl.pair()
    with Engine(w, live=live) as eng:
        dev = eng.device_world
        plan = eng.plan()["groups"][0]
        dev.run(k)
        dev.synchronize()
        dev.timer_start()
        for _ in range(launches):
            dev.run(k)
        dev.timer_stop()
        us = dev.timer_ms() * 1e3 / (k * launches)
        dev.download(_lib.RS_STATE)
    return w, us, plan


def main():
    out = {}
    for k in (10, 100):
        a, ua, pa = run("1", k, 20)
        b, ub, pb = run("0", k, 20)
        diff = {s: int(np.count_nonzero(getattr(a, s).view(np.int64) != getattr(b, s).view(np.int64))) for s in STATE}
        out[f"k{k}"] = {"coupled_us": round(ua, 3), "cluster_us": round(ub, 3), "diff": diff,
                        "tier": pa["tier"], "ctas": pa["ctas"]}
    a, ua, pa = run("1", 10, 20, live=True)
    out["live_k10"] = {"coupled_us": round(ua, 3), "tier": pa["tier"]}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
