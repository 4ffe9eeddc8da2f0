"""The committed golden fixtures (tests/golden/*.npz, written by the reference
package itself through tests/golden/make_golden.py) and how to replay them:
the builder of each fixture's World, and the epoch schedule the reference ran,
including the `set_params` calls between epochs (engine.py:335-355 ->
_core.update_params, _core.pyx:1083-1089)."""

import os

import numpy as np

from paper_2509_04277_b200 import workloads as wl

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
STATE = ("positions", "velocities", "frames", "angular_velocities")

# name -> (World builder, epoch size the reference used)
BUILDERS = {
    "cfg1_cantilever64": (wl.cantilever, 1000),
    "cfg2_extensible512": (wl.extensible, 10),
    "cfg3_pair2x512": (wl.pair, 10),
    "cfg4_sweep256": (lambda: wl.sweep(256), 100),
    "cfg4_sweep2048": (lambda: wl.sweep(2048), 10),
    "cfg5_hair8": (lambda: wl.hair(8), 100),
    "cfg1_set_params": (wl.cantilever, 50),
    "cfg3_set_params": (wl.pair, 10),
}


def load(name):
    return np.load(os.path.join(GOLDEN, f"{name}.npz"))


def script(g):
    """{step: {"dt": .., "iterations": ..}} -- the parameter changes the
    reference applied at those step boundaries."""
    out = {}
    for key in g.files:
        if key.startswith("set_params_"):
            dt, iters = (float(x) for x in g[key])
            kw = {}
            if not np.isnan(dt):
                kw["dt"] = dt
            if iters >= 1:
                kw["iterations"] = int(iters)
            out[int(key[len("set_params_"):])] = kw
    return out


def replay(g, epoch, run, set_params, on_checkpoint):
    """Drive `run(k)` through the fixture's checkpoints in epochs of at most
    `epoch` steps, calling `set_params(**kw)` where the reference did and
    `on_checkpoint(c)` at every checkpoint."""
    sched = script(g)
    done = 0
    for c in (int(x) for x in g["checkpoints"]):
        while done < c:
            if done in sched:
                set_params(**sched[done])
            k = min(epoch, c - done)
            nxt = [s for s in sched if done < s < done + k]
            if nxt:
                k = min(nxt) - done
            run(k)
            done += k
        on_checkpoint(c)
