#!/usr/bin/env python
"""The bench's haptic frame loop (command in, run_epoch(10), tip out) on a
given library build: median / p99 us per frame."""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2509_04277_b200 import _lib  # noqa: E402

if len(sys.argv) > 1:
    _lib._LIB = _lib.load_library(sys.argv[1])
from paper_2509_04277_b200 import workloads as wl  # noqa: E402
from paper_2509_04277_b200.engine import Engine  # noqa: E402

w = wl.pair()
frames = []
with Engine(w) as eng:
    for i in range(1100):
        t0 = time.perf_counter()
        eng.post_command("insert_velocity", rod=0, value=0.05 + 1e-4 * (i % 7), axis=(0.0, 0.0, 1.0))
        eng.run_epoch(10)
        tip = w.positions[w.rod_infos[0].point_offset + w.rod_infos[0].num_points - 1]
        frames.append(time.perf_counter() - t0)
        _ = float(tip[2])
f = np.array(frames[100:]) * 1e6
print(os.path.basename(sys.argv[1]) if len(sys.argv) > 1 else "default",
      {"median_us": round(float(np.median(f)), 1), "p99_us": round(float(np.percentile(f, 99)), 1)}, flush=True)
