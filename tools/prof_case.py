#!/usr/bin/env python
"""Run one workload for a few launches (for ncu captures and quick timing).

  python tools/prof_case.py hair --rods 65536 --k 1 --launches 5
  python tools/prof_case.py pair --k 10 --launches 5
  python tools/prof_case.py sweep --n 1024 --k 100
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2509_04277_b200 import workloads as wl  # noqa: E402
from paper_2509_04277_b200.engine import Engine  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("case", choices=["hair", "pair", "sweep", "cantilever", "extensible",
                                     "insertion", "floor_drop"])
    ap.add_argument("--rods", type=int, default=65536)
    ap.add_argument("--n", type=int, default=1024)
    ap.add_argument("--k", type=int, default=1)
    ap.add_argument("--launches", type=int, default=5)
    ap.add_argument("--precision", default="f64")
    ap.add_argument("--force-variant", type=int, default=-1)
    ap.add_argument("--force-tier", type=int, default=-1)
    ap.add_argument("--force-ctas", type=int, default=0)
    ap.add_argument("--live", action="store_true")
    a = ap.parse_args()
    if a.case == "hair":
        w = wl.hair(a.rods)
    elif a.case == "sweep":
        w = wl.sweep(a.n)
    else:
        w = getattr(wl, a.case)()
    kw = dict(precision=a.precision, force_variant=a.force_variant, live=a.live)
    if a.force_tier >= 0:
        kw["force_tier"] = a.force_tier
    if a.force_ctas:
        kw["force_ctas"] = a.force_ctas
    with Engine(w, **kw) as eng:
        dev = eng.device_world
        dev.run(a.k)
        dev.synchronize()
        dev.timer_start()
        for _ in range(a.launches):
            dev.run(a.k)
        dev.timer_stop()
        ms = dev.timer_ms()
        print({"case": a.case, "k": a.k, "us_per_step": ms * 1e3 / (a.k * a.launches),
               "plan": eng.plan()["groups"][0]})


if __name__ == "__main__":
    main()
