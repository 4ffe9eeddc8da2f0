#!/usr/bin/env python
"""How often does a wide-halo launch fail its vote (lazy exact replay)?
Steps each case in device-resident launches of K steps, checking after each
launch; run with RSB_DEBUG=4 for the failed-check mask (printed at exit)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2509_04277_b200 import workloads as wl  # noqa: E402
from paper_2509_04277_b200.engine import Engine  # noqa: E402

CASES = {"pair": wl.pair, "s1024": lambda: wl.sweep(1024), "s16384": lambda: wl.sweep(16384),
         "ext": wl.extensible, "s256": lambda: wl.sweep(256)}
for name in sys.argv[1:] or list(CASES):
    k, launches = 10, 300
    fails = []
    with Engine(CASES[name]()) as eng:
        dev = eng.device_world
        for n in range(launches):
            dev.run(k)
            if dev.last_redo_count():
                fails.append(n * k)
    print(name, "launches", launches, "K", k, "failed at steps", fails[:20], "count", len(fails), flush=True)
