#!/usr/bin/env python
"""Wide-halo cluster kernel (rod_halo.cuh): bitwise parity against the oracle
and us/step against the general cluster kernel (RSB_HALO=0), per config and
cluster size (RSB_HALO_CTAS).  Prints one JSON line per case."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from oracle.oracle import OracleStepper  # noqa: E402
from paper_2509_04277_b200 import workloads as wl  # noqa: E402
from paper_2509_04277_b200.engine import Engine  # noqa: E402

STATE = ("positions", "velocities", "frames", "angular_velocities")


def timed(make, k, launches, env):
    old = {key: os.environ.get(key) for key in env}
    os.environ.update({key: str(v) for key, v in env.items()})
    try:
        with Engine(make()) as eng:
            dev = eng.device_world
            dev.run(k)
            dev.synchronize()
            dev.timer_start()
            for _ in range(launches):
                dev.run(k)
            dev.timer_stop()
            g = eng.plan()["groups"][0]
            return dev.timer_ms() * 1e3 / (k * launches), g.get("halo"), eng.device_world.last_redo_count()
    finally:
        for key, v in old.items():
            if v is None:
                os.environ.pop(key, None)
            else:
                os.environ[key] = v


def parity(make, steps, k, env):
    old = {key: os.environ.get(key) for key in env}
    os.environ.update({key: str(v) for key, v in env.items()})
    try:
        g, r = make(), make()
        with Engine(g) as eng:
            done = 0
            while done < steps:
                n = min(k, steps - done)
                eng.run_epoch(n)
                done += n
        OracleStepper(r).run(steps)
        return all(np.array_equal(getattr(g, key).view(np.int64), getattr(r, key).view(np.int64)) for key in STATE)
    finally:
        for key, v in old.items():
            if v is None:
                os.environ.pop(key, None)
            else:
                os.environ[key] = v


CASES = {
    "pair": (wl.pair, 10),
    "ext512": (wl.extensible, 10),
    "cfg1": (wl.cantilever, 100),
    "sweep128": (lambda: wl.sweep(128), 100),
    "sweep256": (lambda: wl.sweep(256), 100),
    "sweep512": (lambda: wl.sweep(512), 100),
    "sweep1024": (lambda: wl.sweep(1024), 100),
    "sweep2048": (lambda: wl.sweep(2048), 100),
    "sweep4096": (lambda: wl.sweep(4096), 100),
    "sweep8192": (lambda: wl.sweep(8192), 100),
    "sweep16384": (lambda: wl.sweep(16384), 100),
}
VARIANTS = [{}, {"RSB_HALO_GRID": 0}, {"RSB_HALO_GRID": 1, "RSB_HALO_STEPS": 1},
            {"RSB_HALO_GRID": 1, "RSB_HALO_STEPS": 2}, {"RSB_HALO_GRID": 1, "RSB_HALO_STEPS": 3},
            {"RSB_HALO_GRID": 1, "RSB_HALO_STEPS": 2, "RSB_HALO_W": 192},
            {"RSB_HALO_GRID": 1, "RSB_HALO_STEPS": 2, "RSB_HALO_W": 256},
            {"RSB_HALO_GRID": 0, "RSB_HALO_STEPS": 2}]

if __name__ == "__main__":
    which = sys.argv[1:] or list(CASES)
    for name in which:
        make, k = CASES[name]
        out = {"case": name}
        out["parity_halo"] = parity(make, 200, k, {"RSB_HALO": 1})
        out["parity_halo_grid"] = parity(make, 200, k, {"RSB_HALO": 1, "RSB_HALO_GRID": 1})
        out["parity_halo_s3"] = parity(make, 200, 7, {"RSB_HALO": 1, "RSB_HALO_STEPS": 3})
        out["general"] = timed(make, k, 50, {"RSB_HALO": 0})[0]
        for env in VARIANTS:
            key = "halo" + "".join(f"_{a[9:].lower()}{b}" for a, b in env.items())
            try:
                us, h, redo = timed(make, k, 50, dict({"RSB_HALO": 1}, **env))
                out[key] = {"us": round(us, 3),
                            "plan": h and {x: h[x] for x in ("ctas", "threads", "exchange", "steps_per_exchange")},
                            "redo": redo}
            except Exception as exc:  # noqa: BLE001
                out[key] = str(exc)[:120]
        print(json.dumps(out), flush=True)
