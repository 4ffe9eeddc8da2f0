#!/usr/bin/env python
"""Haptic frame breakdown for the cfg3 pair: Engine.run_epoch(10) wall time
vs the device time of its launch, and the Python-side pieces."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from paper_2509_04277_b200 import _lib  # noqa: E402
from paper_2509_04277_b200 import workloads as wl  # noqa: E402

if len(sys.argv) > 1:   # A/B of library builds (same ABI)
    _lib._LIB = _lib.load_library(sys.argv[1])
    print(os.path.basename(sys.argv[1]), end=" ")
from paper_2509_04277_b200.engine import Engine  # noqa: E402

w = wl.pair()
with Engine(w) as eng:
    for _ in range(20):
        eng.run_epoch(10)
    dev = eng._dev
    n = 300
    t0 = time.perf_counter()
    for _ in range(n):
        eng.run_epoch(10)
    frame = (time.perf_counter() - t0) / n
    t0 = time.perf_counter()
    for _ in range(n):
        eng._push(state=False)
    push = (time.perf_counter() - t0) / n
    t0 = time.perf_counter()
    for _ in range(n):
        dev.run_host(10)
    run_host = (time.perf_counter() - t0) / n
    dev.timer_start()
    for _ in range(n):
        dev.run(10)
    dev.timer_stop()
    kern = dev.timer_ms() / n / 1e3
    print({"frame_us": frame * 1e6, "push_us": push * 1e6, "run_host_us": run_host * 1e6,
           "device_us": kern * 1e6})

    # pieces of run_epoch on the host side
    import cProfile
    import pstats
    pr = cProfile.Profile()
    pr.enable()
    for i in range(300):
        eng.post_command("insert_velocity", rod=0, value=0.05, axis=(0.0, 0.0, 1.0))
        eng.run_epoch(10)
    pr.disable()
    pstats.Stats(pr).sort_stats("tottime").print_stats(14)
