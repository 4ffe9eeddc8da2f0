#!/usr/bin/env python
"""K = 1 launches of a small rod: host wall time per rs_run_epoch call vs
the device time of the same calls (CUDA events) -- which side bounds it."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2509_04277_b200 import workloads as wl  # noqa: E402
from paper_2509_04277_b200.engine import Engine  # noqa: E402

for n in (16, 1024):
    with Engine(wl.sweep(n)) as eng:
        dev = eng.device_world
        for _ in range(100):
            dev.run(1)
        dev.synchronize()
        N = 2000
        dev.timer_start()
        t0 = time.perf_counter()
        for _ in range(N):
            dev.run(1)
        t1 = time.perf_counter()
        dev.timer_stop()
        ms = dev.timer_ms()
        dev.synchronize()
        t2 = time.perf_counter()
        print({"n": n, "host_us_per_call": (t1 - t0) / N * 1e6, "device_us_per_launch": ms * 1e3 / N,
               "wall_us_per_launch": (t2 - t0) / N * 1e6})
