#!/usr/bin/env python
"""K = 1 launch cost without the Python call in the loop: one run(n) call whose
launches are capped at one step each (RSB_MAX_K=1) vs n Python run(1) calls,
plus the bare ctypes round trip (rs_step_counter)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2509_04277_b200 import _lib  # noqa: E402
from paper_2509_04277_b200 import workloads as wl  # noqa: E402
from paper_2509_04277_b200.engine import Engine  # noqa: E402

if len(sys.argv) > 1:   # A/B of library builds (same ABI)
    _lib._LIB = _lib.load_library(sys.argv[1])
    print(os.path.basename(sys.argv[1]), flush=True)
n = 2000
for name, mk in (("n16", lambda: wl.sweep(16)), ("n48", lambda: wl.sweep(48)), ("cfg1", wl.cantilever), ("n1024", lambda: wl.sweep(1024)),
                 ("pair", wl.pair)):
    row = {}
    for mode in ("py", "c"):
        os.environ["RSB_MAX_K"] = "1" if mode == "c" else "65536"
        with Engine(mk()) as eng:
            dev = eng.device_world
            for _ in range(50):
                dev.run(1)
            dev.synchronize()
            dev.timer_start()
            t0 = time.perf_counter()
            if mode == "py":
                for _ in range(n):
                    dev.run(1)
            else:
                dev.run(n)
            t1 = time.perf_counter()
            dev.timer_stop()
            row[mode + "_host_us"] = round((t1 - t0) * 1e6 / n, 2)
            row[mode + "_dev_us"] = round(dev.timer_ms() * 1e3 / n, 2)
            if mode == "py":
                t0 = time.perf_counter()
                for _ in range(n):
                    dev.step_counter()
                row["ctypes_us"] = round((time.perf_counter() - t0) * 1e6 / n, 2)
    print(name, row, flush=True)
