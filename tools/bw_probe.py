#!/usr/bin/env python
"""Warp-per-rod batched kernel vs the general stream kernel (RSB_BW=0):
bitwise state after N launches, device time per launch, redo counts.

  python tools/bw_probe.py --rods 65536 --launches 20 --k 1
"""
import argparse
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


def run(rods, k, launches, precision, env):
    old = {kk: os.environ.get(kk) for kk in env}
    os.environ.update(env)
    try:
        w = wl.hair(rods)
        with Engine(w, precision=precision) as eng:
            dev = eng.device_world
            plan = eng.plan()["groups"][0]
            dev.run(k)
            dev.synchronize()
            dev.timer_start()
            redo = []
            for _ in range(launches):
                dev.run(k)
            dev.timer_stop()
            ms = dev.timer_ms()
            redo.append(dev.last_redo_count())
            dev.download(_lib.RS_STATE)
        return w, ms / launches, plan, redo
    finally:
        for kk, v in old.items():
            if v is None:
                os.environ.pop(kk, None)
            else:
                os.environ[kk] = v


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--rods", type=int, default=65536)
    ap.add_argument("--k", type=int, default=1)
    ap.add_argument("--launches", type=int, default=20)
    ap.add_argument("--precision", default="f64")
    ap.add_argument("--shapes", default="3")
    ap.add_argument("--lib", default=None, help="library build to load (A/B of builds)")
    a = ap.parse_args()
    if a.lib:
        _lib._LIB = _lib.load_library(a.lib)
    ref, ms_ref, plan_ref, _ = run(a.rods, a.k, a.launches, a.precision, {"RSB_BW": "0"})
    out = {"rods": a.rods, "k": a.k, "launches": a.launches, "precision": a.precision,
           "general_ms_per_launch": ms_ref}
    for sh in a.shapes.split(","):
        w, ms, plan, redo = run(a.rods, a.k, a.launches, a.precision, {"RSB_BW": "1", "RSB_BW_SHAPE": sh})
        diff = {}
        for s in STATE:
            x, y = getattr(w, s), getattr(ref, s)
            if a.precision == "f64":
                nbad = int(np.count_nonzero(x.view(np.int64) != y.view(np.int64)))
                diff[s] = nbad
            else:
                diff[s] = float(np.max(np.abs(x - y)))
        out[f"shape{sh}"] = {"ms_per_launch": ms, "diff": diff, "redo_last": redo,
                             "speedup": ms_ref / ms}
    if a.lib:
        out["lib"] = os.path.basename(a.lib)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
