#!/usr/bin/env python
"""K = 1 launches: host wall time per DeviceWorld.run(1) call vs the device
time per step (are one-step epochs host- or device-bound?)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2509_04277_b200 import workloads as wl  # noqa: E402
from paper_2509_04277_b200.engine import Engine  # noqa: E402

for name, mk in (("n16", lambda: wl.sweep(16)), ("cfg1", wl.cantilever), ("n1024", lambda: wl.sweep(1024)),
                 ("pair", wl.pair)):
    with Engine(mk()) as eng:
        dev = eng.device_world
        for _ in range(50):
            dev.run(1)
        dev.synchronize()
        n = 2000
        dev.timer_start()
        t0 = time.perf_counter()
        for _ in range(n):
            dev.run(1)
        t1 = time.perf_counter()
        dev.timer_stop()
        dev_us = dev.timer_ms() * 1e3 / n
        print(name, "host us/call", round((t1 - t0) * 1e6 / n, 2), "device us/step", round(dev_us, 2), flush=True)
