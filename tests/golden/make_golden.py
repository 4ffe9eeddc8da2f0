"""Generate the golden fixtures from the reference package itself.

Runs in the build container only (it needs /root/reference and the
reference's compiled core, built into oracle/_ref by oracle/build_ref.sh).
For each BASELINE configuration (SURVEY.md Appendix B recipes) it builds the
World with the *reference's* API (rodsim.state / rodsim.world), steps it with
the reference Engine(backend="serial") -- i.e. `_core.step_serial` -- and
stores the initial arrays plus state checkpoints.  The committed .npz files
are what tests/test_oracle.py checks our World construction and the oracle
restatement against; nothing on the GPU box reads /root/reference.

    python tests/golden/make_golden.py
"""

import hashlib
import importlib.util
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
REF_SRC = "/root/reference/pkg/src"

STATE = ("positions", "velocities", "frames", "angular_velocities")
STATIC = ("rest_lengths", "intrinsic_strains", "masses", "inv_masses",
          "inertias", "stretch_k", "penalty_k", "gamma_t", "gamma_r",
          "extensible", "bend_k", "point_locked", "frame_locked",
          "elem_point", "elem_parity", "junction_valid", "bind_a", "bind_b",
          "bind_mode", "driven_point", "driven_frame", "driver_velocity")


def import_reference():
    sys.path.insert(0, ROOT)
    from oracle.oracle import load_reference_core
    core = load_reference_core()
    if core is None:
        raise SystemExit("build oracle/_ref first (oracle/build_ref.sh)")
    sys.modules["rodsim._core"] = core
    spec = importlib.util.spec_from_file_location(
        "rodsim", os.path.join(REF_SRC, "rodsim", "__init__.py"),
        submodule_search_locations=[os.path.join(REF_SRC, "rodsim")])
    mod = importlib.util.module_from_spec(spec)
    sys.modules["rodsim"] = mod
    spec.loader.exec_module(mod)
    assert mod.HAVE_COMPILED_CORE
    return mod


MAT = dict(radius=1e-3, stretch_modulus=1e7, bend_modulus=1e6,
           shear_modulus=1e6, linear_density=0.05, penalty_stiffness=1.0,
           damping_translational=2e-4, damping_rotational=1e-8)


def recipes(rs):
    st = rs.state
    from rodsim.constraints import SolverConfig
    from rodsim.world import BIND_BIDIRECTIONAL, World

    def world():
        return World(dt=1e-4, gravity=(0.0, -9.81, 0.0),
                     solver=SolverConfig(iterations=10))

    def cantilever(n=64, length=0.4, **extra):
        w = world()
        w.add_rod(st.init_rod(n + 1, length, axis=(1.0, 0.0, 0.0)),
                  st.RodParams(**dict(MAT, **extra)))
        w.finalize()
        w.clamp_point(0, 0)
        w.clamp_frame(0, 0)
        return w

    def pair(n=512, length=1.0):
        w = world()
        for y in (1.5e-3, -1.5e-3):
            w.add_rod(st.init_rod(n + 1, length, axis=(0.0, 0.0, 1.0),
                                  origin=(0.0, y, -length)), st.RodParams(**MAT))
        w.finalize()
        w.add_bindings(0, 1, BIND_BIDIRECTIONAL, stride=1)
        for r in (0, 1):
            w.set_driver(r)
            w.driver_velocity[r] = (0.0, 0.0, 0.05)
        return w

    def hair(rods=8, n=128):
        w = world()
        for r in range(rods):
            a = np.random.default_rng(r).normal(size=3)
            w.add_rod(st.init_rod(n + 1, 0.4, axis=a / np.linalg.norm(a),
                                  origin=(0.01 * (r % 256), 0.01 * (r // 256), 0.0)),
                      st.RodParams(**MAT))
        w.finalize()
        for r in range(rods):
            w.clamp_point(r, 0)
        return w

    # name -> (builder, checkpoints, epoch size[, {step: set_params kwargs}])
    # The set_params scripts change dt / iterations between epochs through
    # the reference Engine (engine.py:335-355 -> _core.update_params,
    # _core.pyx:1083-1089) at the given step boundaries.
    return {
        "cfg1_cantilever64": (lambda: cantilever(), (1, 10, 100, 1000), 1000),
        "cfg2_extensible512": (lambda: cantilever(512, 1.0, stretch_modulus=1e6,
                                                  extensible=True), (10, 100, 300, 1000), 10),
        "cfg3_pair2x512": (pair, (10, 100, 300, 1000), 10),
        "cfg4_sweep256": (lambda: cantilever(256, 0.512), (100,), 100),
        "cfg4_sweep2048": (lambda: cantilever(2048, 4.096), (20,), 10),
        "cfg5_hair8": (hair, (100, 1000), 100),
        "cfg1_set_params": (lambda: cantilever(), (100, 200, 300), 50,
                            {100: dict(dt=5e-5, iterations=6), 200: dict(dt=1.5e-4, iterations=14)}),
        "cfg3_set_params": (pair, (100, 200, 300), 10,
                            {100: dict(iterations=4), 200: dict(dt=5e-5, iterations=12)}),
    }


def digest(arrays):
    h = hashlib.sha256()
    for a in arrays:
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


def main(only=None):
    rs = import_reference()
    from rodsim.engine import Engine
    for name, recipe in recipes(rs).items():
        if only and name not in only:
            continue
        build, checkpoints, epoch = recipe[:3]
        script = recipe[3] if len(recipe) > 3 else {}
        w = build()
        out = {f"init_{k}": np.array(getattr(w, k)) for k in STATE + STATIC}
        done = 0
        with Engine(w, backend="serial") as eng:
            for c in checkpoints:
                while done < c:
                    if done in script:
                        eng.set_params(**script[done])
                    k = min(epoch, c - done)
                    eng.run_epoch(k)
                    done += k
                for k in STATE:
                    out[f"step{c}_{k}"] = np.array(getattr(w, k))
                out[f"step{c}_sha256"] = np.array(digest(getattr(w, k) for k in STATE))
        out["checkpoints"] = np.array(checkpoints)
        for s_, kw in script.items():
            out[f"set_params_{s_}"] = np.array([kw.get("dt", np.nan), kw.get("iterations", -1)], dtype=np.float64)
        path = os.path.join(HERE, f"{name}.npz")
        np.savez_compressed(path, **out)
        print(f"{name}: P={w.num_points} checkpoints={checkpoints} "
              f"{os.path.getsize(path) / 1e3:.0f} kB")


def copy_knot_assets():
    """The reference's own knot-replay golden data (scenarios.py:86-101,
    test_acceptance.py:455-490): the recorded command session and the
    position checksum after 16000 steps, copied verbatim as fixtures."""
    import json
    import shutil
    src = os.path.join(REF_SRC, "rodsim", "assets")
    shutil.copyfile(os.path.join(src, "knot_session.ndjson"),
                    os.path.join(HERE, "knot_session.ndjson"))
    with open(os.path.join(src, "knot_checksum.json")) as fh:
        rec = json.load(fh)
    with open(os.path.join(HERE, "knot_checksum.json"), "w") as fh:
        json.dump(rec, fh, indent=2)
        fh.write("\n")
    print("knot assets:", rec)


def copy_scenario_assets():
    """Data files the bundled scenarios load (scenarios.py:45-101): the
    curved-tube mesh of the insertion scenes and the knot session log,
    copied verbatim into the package's assets directory."""
    import shutil
    src = os.path.join(REF_SRC, "rodsim", "assets")
    dst = os.path.join(ROOT, "paper_2509_04277_b200", "assets")
    os.makedirs(dst, exist_ok=True)
    for name in ("curved_tube.obj", "knot_session.ndjson"):
        shutil.copyfile(os.path.join(src, name), os.path.join(dst, name))
    print("scenario assets ->", dst)


if __name__ == "__main__":
    if "--knot" in sys.argv:
        copy_knot_assets()
    elif "--assets" in sys.argv:
        copy_scenario_assets()
    elif len(sys.argv) > 1:
        main(set(sys.argv[1:]))   # regenerate the named fixtures only
    else:
        main()
        copy_knot_assets()
        copy_scenario_assets()
