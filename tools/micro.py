#!/usr/bin/env python
"""Latency microbenchmarks (rs_micro) -> JSON on stdout: the per-op and
per-barrier constants of the single-rod latency roofline."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2509_04277_b200 import _lib  # noqa: E402


def main():
    out = {}
    for k in ("dadd", "dmul", "dfma", "div", "sqrt_add", "div_rn", "rcp", "lds", "dsmem"):
        c, ns = _lib.micro(k)
        out[k] = {"cycles": round(c, 2), "ns": round(ns, 2)}
    for t in (32, 64, 128, 256, 512, 1024):
        c, ns = _lib.micro("bar_sync", t)
        out[f"bar_sync_{t}"] = {"cycles": round(c, 2), "ns": round(ns, 2)}
    for c_ in (2, 4, 8, 16):
        c, ns = _lib.micro("cluster_barrier", c_)
        out[f"cluster_barrier_{c_}"] = {"cycles": round(c, 2), "ns": round(ns, 2)}
        c, ns = _lib.micro("neighbour_sync", c_)
        out[f"neighbour_sync_{c_}"] = {"cycles": round(c, 2), "ns": round(ns, 2)}
    peaks = {n: _lib.pipe_peak(i) for i, n in enumerate(("dfma", "dadd", "dmul", "ffma"))}
    out["pipe_peak_ops_per_s"] = peaks
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
