"""fp32-mode error on the full cfg5 batch, decomposed (GPU only).

    python tools/fp32_tolerance.py [rods] [steps]

A = fp64 mirror (bitwise the oracle: tests/test_gpu_batch_scale.py),
B = fp32 mode, C = fp64 mirror on the World with every input rounded to
fp32 first (the problem fp32 mode is handed, solved in fp64).  |B - A| is
the fp32 error; |C - A| the part the rounding of the inputs alone explains
(the conditioning of each rod); |B - C| the arithmetic part.  Prints the
max / 99.9 % / 99 % / median of each, for positions (over L = rod length)
and frames, per point / element, as JSON.
"""

import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2509_04277_b200 import workloads as wl  # noqa: E402
from paper_2509_04277_b200.engine import Engine  # noqa: E402

ROUND = ("positions", "velocities", "frames", "angular_velocities", "rest_lengths",
         "intrinsic_strains", "masses", "inv_masses", "inertias", "stretch_k", "penalty_k",
         "gamma_t", "gamma_r", "bend_k")


def run(w, steps, precision, k=100):
    with Engine(w, precision=precision) as eng:
        dev = eng.device_world
        done = 0
        while done < steps:
            dev.run(min(k, steps - done))
            done += min(k, steps - done)
        from paper_2509_04277_b200._lib import RS_STATE
        dev.download(RS_STATE)
    return w


def stats(x):
    x = np.asarray(x).ravel()
    return {"max": float(x.max()), "q999": float(np.quantile(x, 0.999)),
            "q99": float(np.quantile(x, 0.99)), "median": float(np.median(x))}


def main():
    rods = int(sys.argv[1]) if len(sys.argv) > 1 else 65536
    steps = int(sys.argv[2]) if len(sys.argv) > 2 else 1000
    A = run(wl.hair(rods), steps, "f64")
    B = run(wl.hair(rods), steps, "f32")
    c = wl.hair(rods)
    for a in ROUND:
        arr = getattr(c, a)
        arr[...] = arr.astype(np.float32).astype(np.float64)
    c.static_version += 1
    C = run(c, steps, "f64")
    L = 0.4
    out = {"rods": rods, "steps": steps, "L": L}
    for name, (x, y) in {"fp32_err": (B, A), "input_rounding": (C, A), "arith": (B, C)}.items():
        dr = np.linalg.norm(x.positions - y.positions, axis=1) / L
        dq = np.abs(x.frames - y.frames).max(axis=1)
        out[name] = {"dr_over_L": stats(dr), "dq": stats(dq)}
    # per rod: fp32 error against the input-rounding sensitivity
    P = 129
    e32 = (np.linalg.norm(B.positions - A.positions, axis=1) / L).reshape(rods, P).max(axis=1)
    sens = (np.linalg.norm(C.positions - A.positions, axis=1) / L).reshape(rods, P).max(axis=1)
    ratio = e32 / np.maximum(sens, 1e-12)
    out["per_rod_ratio_fp32_over_sensitivity"] = stats(ratio)
    worst = np.argsort(e32)[-5:][::-1]
    out["worst_rods"] = [{"rod": int(r), "err": float(e32[r]), "sens": float(sens[r]),
                          "axis": [float(v) for v in wl.hair_axes(1, int(r))[0]]} for r in worst]
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
