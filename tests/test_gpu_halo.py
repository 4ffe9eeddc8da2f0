"""Wide-halo kernel (csrc/rod_halo.cuh): rods spread over a cluster (or a
co-resident grid) with one inter-CTA exchange per step, bitwise against the
oracle (oracle/rod_oracle.c, pinned to the reference core).

Covers the cluster sizes and the grid exchange, one-way and bidirectional
column bindings, drivers changed between epochs, extensible rods with
external forces, one-CTA rods spread over a cluster, the exact redo when the
speculative launch fails (tiny dividends), error stamps, iteration counts the
ghost width no longer covers, grabs (general kernel), K = 1 launches and the
tolerance modes.
"""

import numpy as np
import pytest

from paper_2509_04277_b200 import state as st
from paper_2509_04277_b200 import workloads as wl
from paper_2509_04277_b200.engine import Engine
from paper_2509_04277_b200.world import BIND_BIDIRECTIONAL, BIND_ONE_WAY

from oracle.oracle import OracleStepper
from test_gpu_parity import _tiny_world, assert_bitwise

pytestmark = pytest.mark.gpu


def halo_run(make, steps, k, env=None, monkeypatch=None, **kw):
    """Step on the GPU and with the oracle; returns (gpu world, plan)."""
    for key, v in (env or {}).items():
        monkeypatch.setenv(key, str(v))
    g, r = make(), make()
    with Engine(g, **kw) as eng:
        done = 0
        while done < steps:
            n = min(k, steps - done)
            eng.run_epoch(n)
            done += n
        plan = eng.plan()
        redo = eng.device_world.last_redo_count()
    OracleStepper(r).run(steps)
    assert_bitwise(g, r)
    return g, plan["groups"][0], redo


@pytest.mark.parametrize("ctas", [4, 7, 12, 16])
def test_pair_cluster_sizes_bitwise(ctas, monkeypatch):
    _, grp, redo = halo_run(wl.pair, 300, 10, {"RSB_HALO_CTAS": ctas}, monkeypatch)
    assert grp["halo"]["ctas"] == ctas and grp["halo"]["bindings"] and grp["halo"]["rods"] == 2
    assert grp["halo"]["exchange"] == "cluster"
    assert redo == 0


@pytest.mark.parametrize("make,k", [(wl.pair, 10), (lambda: wl.sweep(2048), 25),
                                    (lambda: wl.extensible(512, 1.0), 10)])
def test_grid_exchange_bitwise(make, k, monkeypatch):
    _, grp, redo = halo_run(make, 200, k, {"RSB_HALO_GRID": 1}, monkeypatch)
    assert grp["halo"]["exchange"] == "grid" and grp["halo"]["ctas"] > 1
    assert redo == 0


@pytest.mark.parametrize("steps", [1, 2, 3, 4])
@pytest.mark.parametrize("grid", [0, 1])
def test_exchange_periods_bitwise(steps, grid, monkeypatch):
    # S steps per ghost exchange (ghost width S (2I+1)); K = 7 epochs end
    # inside a period
    _, grp, redo = halo_run(lambda: wl.sweep(1500), 70, 7,
                            {"RSB_HALO_STEPS": steps, "RSB_HALO_GRID": grid}, monkeypatch)
    assert grp["halo"]["steps_per_exchange"] == steps
    assert grp["halo"]["exchange"] == ("grid" if grid else "cluster")
    assert redo == 0


def test_long_rod_grid_exchange_default_bitwise():
    # beyond a 16-CTA cluster the planner takes the grid exchange
    _, grp, redo = halo_run(lambda: wl.sweep(16384), 30, 10)
    assert grp["halo"]["exchange"] == "grid" and grp["halo"]["ctas"] > 16
    assert redo == 0


def _pair_custom(mode, stride):
    def make():
        w = wl._world()
        for y in (1.5e-3, -1.5e-3):
            w.add_rod(st.init_rod(201, 0.4, axis=(0.0, 0.0, 1.0), origin=(0.0, y, -0.4)),
                      st.RodParams(**wl.MATERIAL))
        w.finalize()
        w.add_bindings(0, 1, mode, stride=stride)
        w.set_driver(0)
        w.driver_velocity[0] = (0.0, 0.01, 0.05)
        return w
    return make


@pytest.mark.parametrize("mode,stride", [(BIND_ONE_WAY, 3), (BIND_BIDIRECTIONAL, 7), (BIND_ONE_WAY, 1)])
def test_column_bindings_bitwise(mode, stride):
    _, grp, _ = halo_run(_pair_custom(mode, stride), 200, 20)
    assert grp["halo"] and grp["halo"]["bindings"]


def test_overlapping_couplings_keep_the_general_kernel():
    def make():
        w = _pair_custom(BIND_BIDIRECTIONAL, 1)()
        w.add_bindings(0, 1, BIND_ONE_WAY, stride=5)   # not a matching: sequential order
        return w
    _, grp, _ = halo_run(make, 60, 20)
    assert grp["halo"] is None


def test_driver_commands_between_epochs_bitwise():
    def script(world, run):
        run(30)
        world.driver_velocity[0] = (0.01, 0.0, 0.08)
        world.driver_velocity[1] = (0.0, -0.02, 0.0)
        run(30)
        world.driver_rotation[1] = 2.0
        run(20)

    g, r = wl.pair(), wl.pair()
    with Engine(g) as eng:
        assert eng.plan()["groups"][0]["halo"]
        script(g, eng.run_epoch)
    script(r, OracleStepper(r).run)
    assert_bitwise(g, r)


def test_extensible_with_external_forces_bitwise():
    def make():
        w = wl.extensible(700, 1.2)
        w.external_forces[::7] = (1e-4, -2e-4, 5e-5)
        return w
    _, grp, redo = halo_run(make, 100, 10)
    assert grp["halo"] and redo == 0


@pytest.mark.parametrize("n", [128, 300, 512])
def test_one_cta_rods_spread_over_a_cluster_bitwise(n):
    _, grp, redo = halo_run(lambda: wl.sweep(n), 200, 50)
    assert grp["tier"] == "cta" and grp["halo"] and grp["halo"]["ctas"] > 1
    assert redo == 0


def test_k1_launches_bitwise():
    halo_run(wl.pair, 40, 1)
    halo_run(lambda: wl.sweep(4096), 12, 1)


def test_tiny_dividends_replay_the_sweeps_in_the_cta():
    # velocities ~1e-200 on exactly representable geometry: colour-phase
    # dividends below the fast path's window -- the CTA replays its sweeps
    # with IEEE divisions for those lanes, no launch fails its vote
    g, grp, redo = halo_run(lambda: _tiny_world(1, 700), 30, 10)
    assert grp["halo"] and redo == 0
    assert np.max(np.abs(g.velocities)) < 1e-150


def _degenerate_sweep():
    w = wl.sweep(1024)
    w.positions[501] = w.positions[500]   # a zero-length segment at step 0
    return w


def test_failed_vote_replays_the_skipped_launches():
    # a degenerate segment (the reference stamps its error step): the first
    # device-resident launch fails its vote, the later ones return at once,
    # and the download replays all 26 steps on the exact kernel
    from paper_2509_04277_b200 import _lib
    g, r = _degenerate_sweep(), _degenerate_sweep()
    with Engine(g) as eng:
        dev = eng.device_world
        for _ in range(3):
            dev.run(7)
        assert dev.last_redo_count() == 1
        dev.run(5)
        dev.download(_lib.RS_STATE)
        assert dev.error_step() == 0
    OracleStepper(r).run(26)
    assert_bitwise(g, r)


def test_planar_noise_takes_the_inline_fallback_not_the_redo():
    # a planar cantilever's out-of-plane components decay through the
    # subnormal range: those quotients go to the IEEE division in-kernel
    g, _, redo = halo_run(lambda: wl.sweep(1024), 400, 100)
    assert redo == 0


def test_error_step_surfaces():
    w = wl.sweep(1024)
    with Engine(w) as eng:
        assert eng.plan()["groups"][0]["halo"]
        eng.run_epoch(5)
        w.positions[300] = np.nan
        with pytest.raises(FloatingPointError, match="non-finite"):
            eng.run_epoch(5)


def test_more_iterations_than_the_ghost_width_bitwise():
    # the ghost width covers the planned iteration count; more iterations
    # plan the halo again (wider ghosts), fewer keep the plan
    g, r = wl.pair(), wl.pair()
    ref = OracleStepper(r)
    with Engine(g) as eng:
        for it, steps in ((10, 30), (14, 30), (6, 30)):
            eng.set_params(iterations=it)
            ref.set_params(iterations=it)
            eng.run_epoch(steps)
            ref.run(steps)
            assert eng.plan()["groups"][0]["halo"]["ghost"] >= 2 * it + 1
    assert_bitwise(g, r)


def test_more_iterations_on_coupled_rods_past_one_cluster_bitwise():
    g, r = wl.pair(9500, 19.0), wl.pair(9500, 19.0)
    ref = OracleStepper(r)
    with Engine(g) as eng:
        eng.run_epoch(3)
        ref.run(3)
        eng.set_params(iterations=14)
        ref.set_params(iterations=14)
        eng.run_epoch(3)
        ref.run(3)
    assert_bitwise(g, r)


def test_grabs_bitwise():
    # grab anchors on the wide-halo kernel: two slots on one point (slot
    # order), one on an owned boundary point, a release mid-run
    def script(world, run):
        s1 = world.grab(0, 700, (1.5, 0.05, 0.0))
        # a second slot on the same point (the world's arrays directly)
        world.grab_point[5] = world.grab_point[s1]
        world.grab_target[5] = (1.4, 0.02, 0.01)
        world.grab_active[5] = 1
        world.grab(0, 64, (0.1, 0.03, 0.0))   # CTA 0's last owned point, CTA 1's ghost
        run(40)
        world.release(0, 700)
        run(30)

    g, r = wl.sweep(1024), wl.sweep(1024)
    with Engine(g) as eng:
        assert eng.plan()["groups"][0]["halo"]
        script(g, eng.run_epoch)
        assert eng.device_world.last_redo_count() == 0
    script(r, OracleStepper(r).run)
    assert_bitwise(g, r)


def test_tolerance_modes():
    # fp32 / fast fp64 through the halo kernel: within the stated bounds
    for prec, tol_r in (("f32", 1e-5), ("f64_fast", 1e-9)):
        g, r = wl.sweep(1024), wl.sweep(1024)
        with Engine(g, precision=prec) as eng:
            assert eng.plan()["groups"][0]["halo"]
            eng.run_epoch(1000)
        OracleStepper(r).run(1000)
        L = 2e-3 * 1024
        assert np.max(np.abs(g.positions - r.positions)) <= tol_r * L
        assert np.max(np.abs(g.frames - r.frames)) <= (1e-4 if prec == "f32" else 1e-9)


def test_coupled_pair_past_one_cluster_bitwise():
    # 2 x 9500 bound points exceed a 16-CTA cluster: the general planner
    # rejected such sets; the wide-halo grid exchange steps them
    make = lambda: wl.pair(9500, 19.0)   # noqa: E731
    _, grp, redo = halo_run(make, 9, 3)
    assert grp["tier"] == "grid" and grp["halo"]["exchange"] == "grid" and grp["halo"]["rods"] == 2
    assert redo == 0


def test_coupled_pair_past_one_cluster_has_no_exact_fallback():
    # a degenerate segment fails the vote; no general kernel can replay such
    # a set, so the download reports it instead of returning unstepped state
    w = wl.pair(9500, 19.0)
    w.positions[101] = w.positions[100]
    with Engine(w) as eng:
        with pytest.raises(NotImplementedError, match="no exact fallback"):
            eng.run_epoch(3)


def _two_long_rods():
    w = wl._world()
    for z in (0.0, 0.05):
        w.add_rod(st.init_rod(1025, 2.048, axis=(1.0, 0.0, 0.0), origin=(0.0, 0.0, z)), st.RodParams(**wl.MATERIAL))
    w.finalize()
    for r in (0, 1):
        w.clamp_point(r, 0)
        w.clamp_frame(r, 0)
    return w


def test_several_halo_groups_bitwise():
    # two unbound long rods: two cluster groups, two wide-halo launches per epoch
    g, r = _two_long_rods(), _two_long_rods()
    with Engine(g) as eng:
        plan = eng.plan()["groups"]
        assert len(plan) == 2 and all(x["halo"] for x in plan)
        for _ in range(6):
            eng.run_epoch(7)
    OracleStepper(r).run(42)
    assert_bitwise(g, r)


def test_halo_group_beside_a_batch_of_short_rods_bitwise():
    # a long rod and 40 short ones: a CTA-tier group (general / one-warp
    # kernels) and a wide-halo cluster group in one world
    def make():
        w = wl._world()
        w.add_rod(st.init_rod(700, 1.4, axis=(1.0, 0.0, 0.0)), st.RodParams(**wl.MATERIAL))
        for k in range(40):
            w.add_rod(st.init_rod(17, 0.032, axis=(0.0, 0.0, 1.0), origin=(0.01 * k, 0.1, 0.0)),
                      st.RodParams(**wl.MATERIAL))
        w.finalize()
        for rr in range(41):
            w.clamp_point(rr, 0)
        return w
    g, r = make(), make()
    with Engine(g) as eng:
        plan = eng.plan()["groups"]
        assert any(x["halo"] for x in plan) and any(not x["halo"] for x in plan)
        for _ in range(4):
            eng.run_epoch(10)
    OracleStepper(r).run(40)
    assert_bitwise(g, r)


def test_mesh_contacts_fp32_within_tolerance():
    # the insertion scene on the halo kernel in fp32: positions near the
    # fp64 oracle's after 400 steps (contacts switch on and off along the way)
    g, r = wl.insertion(), wl.insertion()
    with Engine(g, precision="f32") as eng:
        assert eng.plan()["groups"][0]["halo"]
        eng.run_epoch(400)
    OracleStepper(r).run(400)
    # the rod sits ~0.3 m from the origin: fp32 rounding of its driven base
    # (ulp ~3e-8 m) accumulates over the 400 steps to ~3e-6 m
    assert np.max(np.abs(g.positions - r.positions)) <= 2e-5
    assert np.max(np.abs(g.frames - r.frames)) <= 1e-4


def test_live_commands_with_mesh_contacts_bitwise():
    # live launches of the insertion scene (scene-feature path of the halo
    # kernel): a driver command posted mid-epoch lands at a step boundary
    import threading
    import time
    steps = 4000
    g = wl.insertion()
    with Engine(g, live=True) as eng:
        assert eng.plan()["live"] and eng.plan()["groups"][0]["halo"]
        eng.run_epoch(1)
        box = {}
        th = threading.Thread(target=lambda: box.setdefault("m", eng.run_epoch(steps)))
        th.start()
        time.sleep(0.01)
        t = eng.post_command("insert_velocity", rod=0, value=0.08, axis=(0.0, 0.0, 1.0))
        th.join()
        s_apply = t.wait(5.0)
    assert 1 < s_apply < 1 + steps
    r = wl.insertion()
    o = OracleStepper(r)
    o.run(s_apply)
    r.driver_velocity[0] = (0.0, 0.0, 0.08)
    o.run(1 + steps - s_apply)
    assert_bitwise(g, r)
