"""Live commands: with Engine(live=True) (the default
for backend="parallel"), a command posted from another thread while a long
epoch runs on a one-CTA or one-cluster plan is drained
by the kernel at the next step boundary -- its ticket reports that step --
and the state equals, bit for bit, the oracle run with the command applied
at exactly that step (_core.pyx:477-506, engine.py:177-198)."""

import threading
import time

import numpy as np
import pytest

from oracle.oracle import OracleStepper
from paper_2509_04277_b200 import workloads as wl
from paper_2509_04277_b200.engine import Engine

pytestmark = pytest.mark.gpu
STATE = ("positions", "velocities", "frames", "angular_velocities")


def _bits(a):
    return np.ascontiguousarray(a).view(np.int64)


def live_run(make, steps, post):
    """Run one epoch of `steps` in a thread, post commands mid-flight."""
    g = make()
    with Engine(g, live=True) as eng:
        assert eng.plan()["live"]
        eng.run_epoch(1)                      # bind / warm up
        box = {}

        def run():
            try:
                box["m"] = eng.run_epoch(steps)
            except Exception as exc:   # surfaced below
                box["error"] = exc
        th = threading.Thread(target=run)
        th.start()
        tickets = post(eng)
        th.join()
        assert "error" not in box, box.get("error")
        applied = [t.wait(5.0) for t in tickets]
    return g, applied


def test_live_driver_velocity_on_cluster_pair():
    steps = 4000

    def post(eng):
        time.sleep(0.02)
        return [eng.post_command("insert_velocity", rod=0, value=0.2, axis=(0.0, 0.0, 1.0))]
    g, (s_apply,) = live_run(wl.pair, steps, post)
    assert 1 < s_apply < 1 + steps          # applied mid-epoch, not at a boundary
    r = wl.pair()
    o = OracleStepper(r)
    o.run(s_apply)
    r.driver_velocity[0] = (0.0, 0.0, 0.2)
    o.run(1 + steps - s_apply)
    assert np.isfinite(r.positions).all()
    for k in STATE:
        assert np.array_equal(_bits(getattr(g, k)), _bits(getattr(r, k))), k
    assert np.array_equal(g.driver_velocity, r.driver_velocity)


def test_live_grab_and_release_on_cta():
    # the knot threads (one CTA, soft and damped): a grab on the second
    # thread's free end and its release, both posted mid-epoch
    steps = 6000

    def post(eng):
        time.sleep(0.01)
        a = eng.post_command("grab", rod=1, index=47, target=(0.11, 0.005, 0.02))
        time.sleep(0.02)
        b = eng.post_command("release", rod=1, index=47)
        return [a, b]
    g, (s_grab, s_rel) = live_run(wl.knot, steps, post)
    assert 1 < s_grab < s_rel < 1 + steps
    r = wl.knot()
    o = OracleStepper(r)
    o.run(s_grab)
    r.grab(1, 47, np.array([0.11, 0.005, 0.02]))
    o.run(s_rel - s_grab)
    r.release(1, 47)
    o.run(1 + steps - s_rel)
    assert np.isfinite(r.positions).all()
    for k in STATE:
        assert np.array_equal(_bits(getattr(g, k)), _bits(getattr(r, k))), k
    assert not g.grab_active.any()


def test_live_is_opt_in():
    with Engine(wl.cantilever()) as eng:
        assert not eng.plan()["live"]
    with Engine(wl.cantilever(), backend="parallel") as eng:
        assert eng.plan()["live"]


def test_live_snapshots_during_an_epoch_match_the_oracle():
    # per-step snapshots published by the kernel (ph_publish): read while a
    # long epoch runs, each equals the oracle's state at its step, bit for bit
    steps = 3000
    g = wl.pair()
    snaps = []
    with Engine(g, live=True) as eng:
        eng.read_snapshot()                   # a reader: per-step publishing on
        eng.run_epoch(1)
        th = threading.Thread(target=lambda: eng.run_epoch(steps))
        th.start()
        while th.is_alive() and len(snaps) < 40:
            snaps.append(eng.read_snapshot())
            time.sleep(0.001)
        th.join()
        last = eng.read_snapshot()
    assert last.step_index == 1 + steps
    assert np.array_equal(_bits(last.positions), _bits(g.positions))
    mid = [s for s in snaps if 1 < s.step_index < 1 + steps]
    assert len(mid) >= 3
    assert all(a.step_index <= b.step_index for a, b in zip(snaps, snaps[1:]))
    r = wl.pair()
    o = OracleStepper(r)
    for s in sorted({s.step_index: s for s in mid}.values(), key=lambda s: s.step_index):
        o.run(s.step_index - r.step_index)
        assert np.array_equal(_bits(s.positions), _bits(r.positions)), s.step_index
        assert np.array_equal(_bits(s.frames), _bits(r.frames)), s.step_index


def test_live_grab_release_and_driver_on_the_wide_halo_kernel():
    # a 1024-element rod on the wide-halo kernel (one cluster, an exchange
    # barrier per step): a grab near a CTA boundary, a driver, then the
    # release, all posted mid-epoch; each lands at a step boundary in every
    # CTA at once
    steps = 8000

    def make():   # (no gravity: the rod rests, the grab pulls 1 mm)
        w = wl.sweep(1024)
        w.gravity[:] = 0.0
        w.set_driver(0)
        return w

    def post(eng):
        assert eng.plan()["groups"][0]["halo"]
        time.sleep(0.005)
        a = eng.post_command("grab", rod=0, index=700, target=(1.4, 1e-3, 0.0))
        time.sleep(0.004)
        b = eng.post_command("insert_velocity", rod=0, value=0.05, axis=(0.0, 1.0, 0.0))
        time.sleep(0.004)
        c = eng.post_command("release", rod=0, index=700)
        return [a, b, c]
    g, (s_grab, s_drv, s_rel) = live_run(make, steps, post)
    assert 1 < s_grab <= s_drv <= s_rel < 1 + steps
    r = make()
    o = OracleStepper(r)
    o.run(s_grab)
    r.grab(0, 700, np.array([1.4, 1e-3, 0.0]))
    o.run(s_drv - s_grab)
    r.driver_velocity[0] = (0.0, 0.05, 0.0)
    o.run(s_rel - s_drv)
    r.release(0, 700)
    o.run(1 + steps - s_rel)
    assert np.isfinite(r.positions).all()
    for k in STATE:
        assert np.array_equal(_bits(getattr(g, k)), _bits(getattr(r, k))), k
