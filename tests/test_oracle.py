"""Pin the CPU oracle (oracle/rod_oracle.c) and the host-side World
construction to the reference, bit for bit.

* tests/golden/*.npz were produced by the reference package itself
  (tests/golden/make_golden.py: reference World + Engine(backend="serial"),
  i.e. the compiled `_core.step_serial`).
* Our builders (paper_2509_04277_b200.workloads) must reproduce the
  reference's initial arrays exactly, and the oracle must reproduce every
  checkpoint exactly.
* When oracle/_ref (the reference core built from /root/reference) is
  present, randomized scenes with drivers, grabs, bindings and mixed
  extensibility are cross-checked oracle vs reference core.
"""

import glob
import hashlib
import os

import numpy as np
import pytest

from oracle.oracle import OracleStepper, ReferenceStepper, load_reference_core
from paper_2509_04277_b200 import state as st
from paper_2509_04277_b200 import workloads as wl
from paper_2509_04277_b200.constraints import SolverConfig
from paper_2509_04277_b200.world import BIND_BIDIRECTIONAL, BIND_ONE_WAY, World

import golden_fixtures as gf

GOLDEN = gf.GOLDEN
STATE = gf.STATE
BUILDERS = {name: make for name, (make, _) in gf.BUILDERS.items()}
golden = gf.load


def test_every_fixture_has_a_builder():
    names = {os.path.basename(p)[:-4] for p in glob.glob(os.path.join(GOLDEN, "*.npz"))}
    assert names == set(BUILDERS)


@pytest.mark.parametrize("name", sorted(BUILDERS))
def test_world_construction_matches_reference(name):
    g = golden(name)
    w = BUILDERS[name]()
    for key in g.files:
        if not key.startswith("init_"):
            continue
        attr = key[5:]
        ours = np.asarray(getattr(w, attr))
        ref = g[key]
        assert ours.shape == ref.shape, attr
        if ref.dtype == bool or ours.dtype == bool:
            assert np.array_equal(ours.astype(bool), ref.astype(bool)), attr
        else:
            assert ours.dtype == ref.dtype, attr
            assert np.array_equal(ours, ref), attr
            assert np.array_equal(np.signbit(ours), np.signbit(ref)), attr


@pytest.mark.parametrize("name", sorted(BUILDERS))
def test_oracle_reproduces_reference_checkpoints(name):
    g = golden(name)
    w = BUILDERS[name]()
    stepper = OracleStepper(w)

    def check(c):
        for k in STATE:
            assert np.array_equal(getattr(w, k), g[f"step{c}_{k}"]), (c, k)
        h = hashlib.sha256()
        for k in STATE:
            h.update(np.ascontiguousarray(getattr(w, k)).tobytes())
        assert h.hexdigest() == str(g[f"step{c}_sha256"])

    # the oracle steps one epoch of any length bitwise like K single steps
    gf.replay(g, 10 ** 9, stepper.run, stepper.set_params, check)
    assert stepper.error_step == -1
    if gf.script(g):   # the parameter changes really changed the trajectory
        assert w.dt == g["set_params_200"][0]


# -- oracle vs the reference's compiled core on randomized scenes -------------

needs_ref = pytest.mark.skipif(load_reference_core() is None,
                               reason="oracle/_ref (reference core) not built")


def random_scene(seed):
    rng = np.random.default_rng(seed)
    w = World(dt=1e-4, gravity=tuple(rng.normal(size=3) * 5.0),
              solver=SolverConfig(iterations=int(rng.integers(1, 12)),
                                  position_bias=float(rng.uniform(0.0, 1.0))))
    nrod = int(rng.integers(1, 5))
    for r in range(nrod):
        n = int(rng.integers(2, 60))
        p = st.RodParams(radius=float(rng.uniform(5e-4, 2e-3)),
                         stretch_modulus=float(rng.uniform(1e5, 1e6)),
                         bend_modulus=float(rng.uniform(1e4, 1e6)),
                         shear_modulus=float(rng.uniform(1e4, 1e6)),
                         penalty_stiffness=float(rng.uniform(0.5, 3.0)),
                         damping_translational=float(rng.uniform(0, 3e-4)),
                         damping_rotational=float(rng.uniform(0, 1e-7)),
                         extensible=bool(rng.integers(0, 2)))
        w.add_rod(st.init_rod(n, 0.003 * n, axis=rng.normal(size=3),
                              origin=rng.normal(size=3) * 0.01), p)
    w.finalize()
    w.velocities[:] = rng.normal(size=w.velocities.shape) * 1e-3
    w.angular_velocities[:] = rng.normal(size=w.angular_velocities.shape) * 1e-2
    for r in range(nrod):
        if rng.random() < 0.5:
            w.clamp_point(r, 0)
        if rng.random() < 0.3:
            w.set_driver(r)
            w.driver_velocity[r] = rng.normal(size=3) * 1e-2
            w.driver_rotation[r] = rng.normal()
    if nrod >= 2 and rng.random() < 0.7:
        w.add_bindings(0, 1, int(rng.integers(0, 2)), stride=int(rng.integers(1, 4)))
        if rng.random() < 0.5:
            w.add_bindings(0, 1, BIND_ONE_WAY, stride=3)
    for _ in range(int(rng.integers(0, 4))):
        r = int(rng.integers(0, nrod))
        i = int(rng.integers(0, w.rod_infos[r].num_points))
        w.grab(r, i, rng.normal(size=3) * 0.01)
    return w


@needs_ref
@pytest.mark.parametrize("seed", range(12))
def test_oracle_matches_reference_core_random_scenes(seed):
    a, b = random_scene(seed), random_scene(seed)
    OracleStepper(a).run(60)
    ReferenceStepper(b, block_cap=7).run(60)
    for k in STATE:
        assert np.array_equal(getattr(a, k), getattr(b, k)), k


@needs_ref
def test_error_step_semantics_match_reference():
    a, b = wl.cantilever(), wl.cantilever()
    a.positions[5] = np.nan
    b.positions[5] = np.nan
    sa, sb = OracleStepper(a), ReferenceStepper(b)
    sa.run(3)
    sb.run(3)
    assert sa.error_step == sb.error_step == 2   # last erroring step
