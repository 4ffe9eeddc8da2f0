#!/usr/bin/env python
"""Where an e2e (Engine.run_epoch, host arrays) epoch's time goes for the
cfg5 batch: the pipelined rs_run_epoch_host call vs the Python around it."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2509_04277_b200 import workloads as wl  # noqa: E402
from paper_2509_04277_b200.engine import Engine  # noqa: E402

w = wl.hair(65536)
with Engine(w) as eng:
    for _ in range(2):
        eng.run_epoch(1)
    dev = eng._dev
    t = {"run_epoch": 0.0, "run_host": 0.0}
    n = 5
    for _ in range(n):
        t0 = time.perf_counter()
        eng.run_epoch(1)
        t["run_epoch"] += time.perf_counter() - t0
    for _ in range(n):
        t0 = time.perf_counter()
        dev.run_host(1)
        t["run_host"] += time.perf_counter() - t0
    print({k: round(v / n * 1e3, 2) for k, v in t.items()}, "ms per epoch")
