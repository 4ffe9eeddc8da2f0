"""The drop-in boundary exercised from the reference side.

The UNMODIFIED reference package (installed into baseline/_ref, DESIGN.md
§8) is imported with `paper_2509_04277_b200.refcore` registered as its
compiled core `rodsim._core` (/root/reference/pkg/src/rodsim/__init__.py:6-11,
engine.py:22-28).  The reference's own `rodsim.engine.Engine` -- its serial
loop of `step_serial` calls (engine.py:286-292) and its block-parallel worker
pool with `begin_epoch` / `run_epoch_worker` / `epoch_results`
(engine.py:370-418) -- then steps on the GPU, and the results are compared
with the golden checkpoints the reference wrote with its own compiled core
(tests/golden/make_golden.py), bit for bit.  Also checked: `set_params` ->
`update_params` between epochs, command tickets through the staging ring,
the snapshot buffer, and the contact count `epoch_results` reports against
the reference scenario runner's metrics.
"""

import os
import sys

import numpy as np
import pytest

from golden_fixtures import STATE, load, replay
from paper_2509_04277_b200 import refcore

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = os.path.join(ROOT, "baseline", "_ref")

pytestmark = [
    pytest.mark.gpu,
    pytest.mark.skipif(not os.path.isfile(os.path.join(REF, "rodsim", "engine.py")),
                       reason="reference package not installed in baseline/_ref"),
]


@pytest.fixture(scope="module")
def rs():
    saved = {k: v for k, v in sys.modules.items() if k == "rodsim" or k.startswith("rodsim.")}
    for k in saved:
        del sys.modules[k]
    sys.path.insert(0, REF)
    try:
        refcore.install("rodsim")
        import rodsim
        import rodsim.constraints
        import rodsim.engine
        import rodsim.scenarios
        import rodsim.state
        import rodsim.world
        assert rodsim._core is refcore and rodsim.HAVE_COMPILED_CORE
        assert rodsim.engine._core is refcore
        assert os.path.dirname(rodsim.__file__).startswith(REF)
        yield rodsim
    finally:
        sys.path.remove(REF)
        for k in [k for k in sys.modules if k == "rodsim" or k.startswith("rodsim.")]:
            del sys.modules[k]
        sys.modules.update(saved)


def _recipes(rs):
    sys.path.insert(0, os.path.join(ROOT, "tests", "golden"))
    try:
        import make_golden
    finally:
        sys.path.pop(0)
    return make_golden.recipes(rs)


def _bits(a):
    return np.ascontiguousarray(a).view(np.int64)


def _run_fixture(rs, name, backend, upto=None, epoch=None):
    build, _, ref_epoch = _recipes(rs)[name][:3]
    g = load(name)
    w = build()
    for k in STATE:
        assert np.array_equal(_bits(getattr(w, k)), _bits(g[f"init_{k}"])), k
    bad = []
    with rs.engine.Engine(w, backend=backend) as eng:
        def check(c):
            if upto is not None and c > upto:
                return
            for k in STATE:
                if not np.array_equal(_bits(getattr(w, k)), _bits(g[f"step{c}_{k}"])):
                    bad.append((c, k))
            snap = eng.read_snapshot()
            assert snap.step_index == c and np.array_equal(snap.positions, w.positions)

        def run(k):
            if upto is None or w.step_index < upto:
                eng.run_epoch(k)

        replay(g, epoch or ref_epoch, run, eng.set_params, check)
        assert isinstance(eng._ctx, refcore.CoreContext)
    assert not bad, bad
    return w


@pytest.mark.parametrize("backend", ["serial", "parallel"])
def test_reference_engine_cfg1_golden(rs, backend):
    _run_fixture(rs, "cfg1_cantilever64", backend)


@pytest.mark.parametrize("backend", ["serial", "parallel"])
def test_reference_engine_cfg1_set_params_golden(rs, backend):
    _run_fixture(rs, "cfg1_set_params", backend)


def test_reference_engine_cfg3_serial_golden(rs):
    # one step_serial call per step: 300 steps of the 2 x 513-point pair
    _run_fixture(rs, "cfg3_pair2x512", "serial", upto=300)


def test_reference_engine_cfg3_parallel_golden(rs):
    # the parallel backend: one K = 10 launch per epoch, 100 epochs
    _run_fixture(rs, "cfg3_pair2x512", "parallel")


def test_reference_engine_cfg3_set_params_parallel(rs):
    _run_fixture(rs, "cfg3_set_params", "parallel")


def test_reference_engine_commands_serial_equals_parallel(rs):
    # a driver-velocity command through the reference mailbox: the serial
    # path applies it to the World at the step boundary (engine.py:254-260),
    # the parallel path stages it on the ring (engine.py:187-198, drained
    # in the kernel); both report the same apply step and the same state
    build = _recipes(rs)["cfg3_pair2x512"][0]
    out = {}
    for backend in ("serial", "parallel"):
        w = build()
        with rs.engine.Engine(w, backend=backend) as eng:
            eng.run_epoch(20)
            t = eng.post_command("insert_velocity", rod=1, value=0.08)
            eng.run_epoch(20)
            assert t.wait(timeout=5.0) == 20
            log = [(s, c.name) for s, c in eng.command_log]
        assert log == [(20, "insert_velocity")], (backend, log)
        out[backend] = w
    for k in STATE:
        assert np.array_equal(_bits(getattr(out["serial"], k)), _bits(getattr(out["parallel"], k))), k


def test_reference_engine_error_surfaces(rs):
    # a NaN velocity: the kernel stamps the step, the reference engine
    # raises FloatingPointError after the epoch (engine.py:328-333)
    build = _recipes(rs)["cfg1_cantilever64"][0]
    w = build()
    with rs.engine.Engine(w, backend="parallel") as eng:
        eng.run_epoch(5)
        w.velocities[10, 1] = np.nan
        with pytest.raises(FloatingPointError):
            eng.run_epoch(5)


@pytest.mark.parametrize("backend", ["serial", "parallel"])
def test_reference_engine_contacts_floor_drop(rs, backend):
    # mesh contacts through the reference engine: a rod dropped on a floor
    # mesh (the recipe of workloads.floor_drop with the reference's own
    # World, bvh and meshes modules); run_epoch's "contacts" (step_serial's
    # return / epoch_results) and the state equal this package's Engine on
    # the same scene, epoch by epoch
    import rodsim.bvh as rbvh
    import rodsim.meshes as rmesh
    from paper_2509_04277_b200 import workloads as wl
    from paper_2509_04277_b200.engine import Engine as OurEngine
    w = rs.world.World(dt=1e-4, gravity=(0.0, -9.81, 0.0),
                       solver=rs.constraints.SolverConfig(iterations=10, restitution=0.2, mu=0.3))
    w.add_rod(rs.state.init_rod(33, 0.2, axis=(1.0, 0.0, 0.2), origin=(-0.1, 0.02, 0.0)),
              rs.state.RodParams(**wl.MATERIAL), contact_radius=0.01)
    w.finalize()
    w.set_mesh(rbvh.build_aabb_tree(*rmesh.floor_mesh(size=0.3, cells=6)))
    w.velocities[:] = (0.05, -0.5, 0.0)
    mine = wl.floor_drop(restitution=0.2, mu=0.3)
    theirs_c, ours_c = [], []
    with rs.engine.Engine(w, backend=backend) as a, OurEngine(mine, backend=backend) as b:
        for _ in range(60):
            theirs_c.append(a.run_epoch(5)["contacts"])
            ours_c.append(b.run_epoch(5)["contacts"])
    assert theirs_c == ours_c and max(theirs_c) > 0, (theirs_c, ours_c)
    for k in STATE:
        assert np.array_equal(_bits(getattr(w, k)), _bits(getattr(mine, k))), k
