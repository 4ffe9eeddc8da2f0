#!/usr/bin/env python
"""A/B timing of library builds on one box: python tools/ab_probe.py LIB.so
(us/step at K = 100 for the wide-halo cases; same ABI required)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2509_04277_b200 import _lib  # noqa: E402

_lib._LIB = _lib.load_library(sys.argv[1])
from paper_2509_04277_b200 import workloads as wl  # noqa: E402
from paper_2509_04277_b200.engine import Engine  # noqa: E402


def us(make, k, launches):
    with Engine(make()) as eng:
        dev = eng.device_world
        dev.run(k)
        dev.synchronize()
        dev.timer_start()
        for _ in range(launches):
            dev.run(k)
        dev.timer_stop()
        return round(dev.timer_ms() * 1e3 / (k * launches), 2)


out = {}
for name, mk in (("pair", wl.pair), ("s256", lambda: wl.sweep(256)), ("s1024", lambda: wl.sweep(1024)),
                 ("s16384", lambda: wl.sweep(16384))):
    out[name] = us(mk, 100, 20)
print(os.path.basename(sys.argv[1]), out, flush=True)
