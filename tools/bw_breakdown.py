#!/usr/bin/env python
"""Time breakdown of the batched step: device ms per launch for K in {1, 10}
and constraint iterations in {10, 0} (iterations 10 vs 1: nine colour sweeps), per kernel
path (RSB_BW=1 warp-per-rod, RSB_BW=0 general)."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2509_04277_b200 import workloads as wl  # noqa: E402
from paper_2509_04277_b200.engine import Engine  # noqa: E402


def main():
    rods = int(sys.argv[1]) if len(sys.argv) > 1 else 65536
    out = {}
    for bw in ("1", "0"):
        os.environ["RSB_BW"] = bw
        w = wl.hair(rods)
        with Engine(w) as eng:
            dev = eng.device_world
            for k in (1, 10):
                for iters in (10, 1):
                    dev.update_params(1e-4, iters)
                    dev.run(k)
                    dev.synchronize()
                    n = 20 if k == 1 else 3
                    dev.timer_start()
                    for _ in range(n):
                        dev.run(k)
                    dev.timer_stop()
                    out[f"bw{bw}_k{k}_it{iters}"] = round(dev.timer_ms() / (n * k), 4)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
