"""The reference's release criteria (tests/test_acceptance.py) that concern
the step, run on the GPU engine.  Bitwise parity with the oracle already
implies the physics; these check the criteria directly, as the reference
states them, so a user of the reference sees the same guarantees:

  04 pendulum inextensible (< 1 % strain) at every one of 5000 steps
  05 twist relaxes to 2 pi / L (< 5 %); twisted clamped rod loops out of plane
  06 serial and parallel backends agree (here: bit for bit) on every scenario
  07 epochs of 10 steps are cheaper per step than single-step epochs
  08 per-step cost grows far slower than the rod (GPU restatement of the
     reference's CPU scaling criteria)
  10 floor contact: penetration < 1e-3 radius, friction cone every step,
     sliding vs sticking displacement >= 10x
  11 coupling cost: no coupling < one-way ~ mutual
  13 crossing threads never interpenetrate during the knot replay, and the
     replay reproduces the reference's recorded checksum

Criteria 01-03, 09 are host-side (test_host_api.py, test_mesh.py), 12
(cost vs insertion depth) measures the reference's serial per-point contact
loop and has no GPU counterpart (detection runs per thread), 14 is
test_gpu_service.py::test_live_session_replays_bitwise.
"""

import json
import os

import numpy as np
import pytest

from paper_2509_04277_b200 import bvh, meshes, quat, scenarios
from paper_2509_04277_b200 import state as st
from paper_2509_04277_b200.constraints import SolverConfig
from paper_2509_04277_b200.engine import Engine
from paper_2509_04277_b200.scene import build_world, parse_scene
from paper_2509_04277_b200.world import World
from paper_2509_04277_b200 import workloads as wl

pytestmark = pytest.mark.gpu
GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def test_04_pendulum_inextensible_every_step():
    cfg = scenarios.default_config("free_space")
    assert cfg.dt == 1e-4 and cfg.solver.iterations == 10
    w = build_world(cfg)
    worst = 0.0
    with Engine(w, backend="serial") as eng:
        for _ in range(5000):
            eng.run_epoch(1)
            worst = max(worst, w.max_strain())
    assert worst < 0.01, worst


def _locked_rod(n, length, damping_rotational, damping_translational=0.0, iterations=1):
    params = st.RodParams(radius=1e-3, stretch_modulus=1e7, bend_modulus=1e6, shear_modulus=1e6,
                          linear_density=0.05, damping_translational=damping_translational,
                          damping_rotational=damping_rotational)
    w = World(dt=1e-4, gravity=(0.0, 0.0, 0.0), solver=SolverConfig(iterations=iterations))
    w.add_rod(st.init_rod(n, length, axis=(0.0, 0.0, 1.0)), params)
    w.finalize()
    return w


def _twisted(n, phases):
    q = np.zeros((n - 1, 4))
    q[:, 0] = np.cos(0.5 * phases)
    q[:, 3] = np.sin(0.5 * phases)
    return q


def test_05_twist_relaxes_and_drives_looping():
    n, length = 64, 0.4
    s = np.linspace(0.0, length, n)
    mid = 0.5 * (s[:-1] + s[1:])
    # (a) a cubic end-loaded twist relaxes to the uniform density 2 pi / L
    w = _locked_rod(n, length, damping_rotational=1e-7)
    w.point_locked[:] = True
    w.frames[:] = _twisted(n, 2.0 * np.pi * (mid / length) ** 3)
    w.frame_locked[0] = True
    w.frame_locked[n - 2] = True
    with Engine(w) as eng:
        eng.run_epoch(100000)
    q = w.frames
    sign = np.where(np.sum(q[:-1] * q[1:], axis=1) < 0.0, -1.0, 1.0)
    qp = (sign[:, None] * q[1:] - q[:-1]) / w.rest_lengths[:-1, None]
    u3 = 2.0 * quat.multiply(quat.conjugate(q[:-1]), qp)[:, 3]
    target = 2.0 * np.pi / length
    assert np.max(np.abs(u3 - target)) / target < 0.05

    # (b) a slack clamped rod stays planar untwisted, buckles when twisted
    def out_of_plane(turns):
        w = _locked_rod(n, length, 1e-7, damping_translational=1e-4, iterations=10)
        w.positions[:, 2] *= 0.9
        w.positions[:, 1] = 1e-4 * np.sin(np.pi * w.positions[:, 2] / (0.9 * length))
        w.frames[:] = _twisted(n, 2.0 * np.pi * turns * mid / length)
        w.clamp_point(0, 0)
        w.clamp_point(0, n - 1)
        w.frame_locked[0] = True
        w.frame_locked[n - 2] = True
        with Engine(w) as eng:
            eng.run_epoch(40000)
        return float(np.max(np.abs(w.positions[:, 0])))

    assert out_of_plane(0) == 0.0
    assert out_of_plane(4) > 1e-3


@pytest.mark.parametrize("name", scenarios.SCENARIO_NAMES)
def test_06_parallel_backend_matches_serial_bitwise(name):
    ref = build_world(scenarios.default_config(name))
    scenarios.run_scenario(name, scenarios.default_config(name), backend="serial",
                           steps=1000, world=ref)
    for blocks in (2, 4, 8):
        par = build_world(scenarios.default_config(name))
        scenarios.run_scenario(name, scenarios.default_config(name), backend="parallel",
                               blocks=blocks, steps=1000, world=par)
        for a in ("positions", "frames", "velocities", "angular_velocities"):
            assert np.array_equal(getattr(par, a).view(np.int64),
                                  getattr(ref, a).view(np.int64)), (name, blocks, a)


def _per_step_ns(world, k, epochs=20, warmup=3):
    with Engine(world) as eng:
        for _ in range(warmup):
            eng.run_epoch(k)
        return min(eng.run_epoch(k)["wall_ns"] for _ in range(epochs)) / k


def test_07_batched_epochs_cheaper_per_step():
    r1 = _per_step_ns(wl.sweep(3072), 1)
    r10 = _per_step_ns(wl.sweep(3072), 10)
    assert r10 / r1 <= 0.8, (r1, r10)


def test_08_cost_grows_far_slower_than_the_rod():
    # the reference: serial cost linear in N, parallel N=2048/N=512 <= 1.6;
    # on the GPU the elements of a step run side by side
    small = _per_step_ns(wl.sweep(1024), 100, epochs=5)
    large = _per_step_ns(wl.sweep(16384), 100, epochs=5)
    assert large / small <= 4.0, (small, large)   # 16x the elements


def _drop_on_floor(mu, v0=0.0, steps=6000, n=32):
    params = st.RodParams(radius=1e-3, stretch_modulus=1e7, bend_modulus=1e6, shear_modulus=1e6,
                          linear_density=0.05, damping_translational=2e-4)
    w = World(solver=SolverConfig(iterations=10, mu=mu))
    w.add_rod(st.init_rod(n, 0.2, axis=(1.0, 0.0, 0.0), origin=(-0.1, 2e-3, 0.0)), params)
    w.finalize()
    w.set_mesh(bvh.build_aabb_tree(*meshes.floor_mesh(size=0.5, y=0.0, cells=6)))
    w.velocities[:, 0] = v0
    cone_ok = True
    with Engine(w) as eng:
        for _ in range(steps):
            eng.run_epoch(1)
            act = w.contact_active.astype(bool)
            if act.any() and np.any(w.contact_acc_t[act] > mu * w.contact_acc_n[act] + 1e-9):
                cone_ok = False
    return float(np.max(1e-3 - w.positions[:, 1])), cone_ok, float(np.mean(w.positions[:, 0]))


def test_10_floor_contact_settles_within_cone():
    penetration, cone, _ = _drop_on_floor(0.3)
    _, cone0, slide = _drop_on_floor(0.0, v0=0.5, steps=4000)
    _, cone1, stick = _drop_on_floor(1.0, v0=0.5, steps=4000)
    assert penetration < 1e-6 and cone and cone0 and cone1
    assert abs(slide) / max(abs(stick), 1e-12) >= 10.0


def _coupled_pair(mode):
    rod = dict(num_points=512, length=0.25, radius=1e-3, stretch_modulus=1e7, bend_modulus=1e6,
               shear_modulus=1e6, linear_density=0.05, damping_translational=2e-4)
    return build_world(parse_scene({
        "rods": [dict(rod, origin=[0.0, 1.5e-3, -0.25], axis=[0, 0, 1.0]),
                 dict(rod, origin=[0.0, -1.5e-3, -0.25], axis=[0, 0, 1.0])],
        "solver": {"iterations": 30},
        "couplings": [{"rod_a": 0, "rod_b": 1, "mode": mode, "stride": 1}],
    }, base_dir=scenarios.ASSET_DIR))


def test_11_coupling_cost_ordering():
    # device time of a 100-step epoch, best of 5 interleaved repeats.  The
    # one-way and mutual couplings run the same kernel (they differ in one
    # weight), so they are held to within 5 % of each other; no coupling
    # has no binding phase and is strictly cheaper.
    best = {m: float("inf") for m in ("v0", "v1", "v2")}
    for _ in range(5):
        for m in best:
            with Engine(_coupled_pair(m), backend="parallel", block_cap=256, max_blocks=2) as eng:
                dev = eng.device_world
                eng.run_epoch(10)
                dev.enable_timing(True)
                eng.run_epoch(100)
                best[m] = min(best[m], dev.last_kernel_ms())
    assert best["v0"] < min(best["v1"], best["v2"]), best
    assert best["v2"] >= 0.95 * best["v1"], best


def test_13_knot_threads_never_interpenetrate():
    with open(os.path.join(GOLDEN, "knot_checksum.json")) as fh:
        recorded = json.load(fh)
    cfg = scenarios.default_config("knot_replay")
    schedule = scenarios.command_schedule("knot_replay", cfg)
    w = build_world(cfg)
    ia, ib = w.rod_infos
    a = slice(ia.point_offset, ia.point_offset + ia.num_points)
    b = slice(ib.point_offset, ib.point_offset + ib.num_points)
    floor = 0.95 * 2.0 * ia.params.radius
    min_sep, nxt = float("inf"), 0
    with Engine(w) as eng:
        while w.step_index < recorded["steps"]:
            while nxt < len(schedule) and schedule[nxt][0] <= w.step_index:
                _, name, args = schedule[nxt]
                eng.post_command(name, **args)
                nxt += 1
            eng.run_epoch(1)
            d = np.linalg.norm(w.positions[a][:, None, :] - w.positions[b][None, :, :], axis=2)
            min_sep = min(min_sep, float(d.min()))
    assert min_sep >= floor, (min_sep, floor)
    assert abs(float(np.sum(np.abs(w.positions))) - recorded["checksum"]) <= recorded["tolerance"]
