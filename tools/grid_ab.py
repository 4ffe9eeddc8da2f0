#!/usr/bin/env python
"""A/B of library builds on the grid-exchange halo rods: us/step at K = 1 /
10 / 100 for cfg4 N = 4096 and 16384 (python tools/grid_ab.py LIB.so)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2509_04277_b200 import _lib  # noqa: E402

_lib._LIB = _lib.load_library(sys.argv[1])
from paper_2509_04277_b200 import workloads as wl  # noqa: E402
from paper_2509_04277_b200.engine import Engine  # noqa: E402

out = {}
for n in (4096, 16384):
    with Engine(wl.sweep(n)) as eng:
        dev = eng.device_world
        assert eng.plan()["groups"][0]["halo"]["exchange"] == "grid"
        for k in (1, 10, 100):
            launches = max(20, 1000 // k)
            dev.run(k)
            dev.synchronize()
            dev.timer_start()
            for _ in range(launches):
                dev.run(k)
            dev.timer_stop()
            out[f"n{n}_k{k}"] = round(dev.timer_ms() * 1e3 / (k * launches), 2)
        dev.synchronize()
        out[f"n{n}_redo"] = dev.last_redo_count()
print(os.path.basename(sys.argv[1]), out, flush=True)
