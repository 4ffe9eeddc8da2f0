"""Benchmark cases on the GPU engine, the reference's caller API
(rodsim/bench.py): amortized per-step cost across rod sizes, epoch sizes
(`batch` = steps per epoch = steps per launch) and backends, as plot-ready
rows.  The reference's "python" core (its numpy fallback) has no
counterpart here -- the GPU step is the only core -- so those rows are
skipped by `bench_suite` and refused by `bench_case`.
"""

import csv
import json
import time

from . import HAVE_COMPILED_CORE
from . import state as st
from .engine import Engine
from .world import World

BENCH_HEADER = ["n", "batch", "backend", "core", "blocks", "epochs", "steps", "wall_ns",
                "per_step_ns", "barrier_wait_ns"]


def _bench_world(n):
    """Gravity-free rod near rest (bench.py:21-30): every per-step kernel
    runs, and the dynamics stay stable at any discretization density."""
    params = st.RodParams(radius=1e-3, stretch_modulus=1e7, bend_modulus=1e3, shear_modulus=1e3,
                          linear_density=0.05, damping_translational=1e-4)
    w = World(dt=1e-4, gravity=(0.0, 0.0, 0.0))
    w.add_rod(st.init_rod(n, 0.4, axis=(1.0, 0.0, 0.0)), params)
    w.finalize()
    w.clamp_point(0, 0)
    return w


def bench_case(n, batch, backend, core="compiled", epochs=3, warmup=1, block_cap=512):
    """Time one configuration (wall clock around `epochs` epochs of `batch`
    steps through Engine.run_epoch); returns a BENCH_HEADER row dict."""
    if core != "compiled":
        raise ValueError("only the compiled (GPU) core exists in this build")
    if not HAVE_COMPILED_CORE:
        raise RuntimeError("compiled core unavailable")
    world = _bench_world(n)
    with Engine(world, backend=backend, block_cap=block_cap) as engine:
        for _ in range(warmup):
            engine.run_epoch(batch)
        barrier = 0
        t0 = time.perf_counter_ns()
        for _ in range(epochs):
            barrier += engine.run_epoch(batch)["barrier_wait_ns"]
        wall = time.perf_counter_ns() - t0
        blocks = engine.partition.block_count
    steps = epochs * batch
    return {"n": n, "batch": batch, "backend": backend, "core": core, "blocks": blocks,
            "epochs": epochs, "steps": steps, "wall_ns": wall, "per_step_ns": wall // steps,
            "barrier_wait_ns": barrier}


def bench_suite(matrix):
    """Rows for the cross product of a matrix dict: lists `n`, `batch`,
    `backend`, `core`; scalars `epochs`, `warmup`, `block_cap`."""
    rows = []
    for core in matrix.get("core", ["compiled"]):
        if core != "compiled" or not HAVE_COMPILED_CORE:
            continue
        for backend in matrix.get("backend", ["serial"]):
            for n in matrix["n"]:
                for batch in matrix.get("batch", [10]):
                    rows.append(bench_case(n, batch, backend, core=core,
                                           epochs=matrix.get("epochs", 3),
                                           warmup=matrix.get("warmup", 1),
                                           block_cap=matrix.get("block_cap", 512)))
    return rows


def load_matrix(path):
    with open(path) as fh:
        matrix = json.load(fh)
    if not matrix.get("n"):
        raise ValueError(f"{path}: matrix needs a non-empty 'n' list")
    return matrix


def export_rows(rows, path):
    with open(path, "w", newline="") as fh:
        out = csv.DictWriter(fh, fieldnames=BENCH_HEADER)
        out.writeheader()
        out.writerows(rows)
    return path
