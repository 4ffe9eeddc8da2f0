"""GPU parity of mesh contacts: detection against the
triangle mesh's AABB tree and the contact impulse phase, fp64 mirror mode,
raw-bit equality with the C oracle (itself pinned to the reference core by
tests/test_mesh.py) on positions, velocities, frames, angular velocities and
every contact slot array, plus the per-epoch active-contact count."""

import numpy as np
import pytest

from oracle.oracle import OracleStepper
from paper_2509_04277_b200 import workloads as wl
from paper_2509_04277_b200.engine import Engine

pytestmark = pytest.mark.gpu

STATE = ("positions", "velocities", "frames", "angular_velocities", "contact_active",
         "contact_normal", "contact_depth", "contact_acc_n", "contact_acc_t")
SMALL_TUBE = {"length": 0.2, "radius": 0.006, "rings": 30, "segments": 12}


def _bits(a):
    a = np.ascontiguousarray(a)
    return a.view(np.uint8) if a.dtype == np.uint8 else a.view(np.int64)


def run_pair(make, steps, k, **kw):
    g, r = make(), make()
    ref = OracleStepper(r)
    gpu_counts, ref_counts = [], []
    with Engine(g, **kw) as eng:
        done = 0
        while done < steps:
            n = min(k, steps - done)
            m = eng.run_epoch(n)
            ref.run(n)
            gpu_counts.append(m["contacts"])
            ref_counts.append(ref.contacts)
            done += n
        plan = eng.plan()
    for key in STATE:
        assert np.array_equal(_bits(getattr(g, key)), _bits(getattr(r, key))), key
    assert gpu_counts == ref_counts
    return g, plan, gpu_counts


def test_floor_drop_bitwise():
    _, _, counts = run_pair(lambda: wl.floor_drop(restitution=0.2, mu=0.3), 300, 5)
    assert max(counts) > 0


def test_floor_resting_friction_bitwise():
    # no bounce: the rod lands and slides to rest under friction
    _, _, counts = run_pair(lambda: wl.floor_drop(height=0.011, restitution=0.0, mu=0.5), 400, 100)
    assert counts[-1] > 0


def test_small_tube_insertion_bitwise():
    _, plan, counts = run_pair(lambda: wl.insertion(points=40, length=0.1, speed=0.5, tube=SMALL_TUBE),
                               400, 10)
    assert max(counts) > 0 and plan["groups"][0]["tier"] == "cta"


def test_insertion_scene_bitwise():
    # the paper's scene: 128-point guidewire, 15360-triangle curved tube
    run_pair(lambda: wl.insertion(), 120, 40)


@pytest.mark.parametrize("ctas", [2, 5])
def test_insertion_cluster_tier_bitwise(ctas):
    _, plan, _ = run_pair(lambda: wl.insertion(points=200, length=0.1, speed=0.5, tube=SMALL_TUBE),
                          200, 50, force_tier=1, force_ctas=ctas)
    assert plan["groups"][0]["tier"] == "cluster"


def test_insertion_grid_tier_bitwise():
    _, plan, _ = run_pair(lambda: wl.insertion(points=200, length=0.1, speed=0.5, tube=SMALL_TUBE),
                          100, 25, force_tier=2, force_ctas=3)
    assert plan["groups"][0]["tier"] == "grid"
