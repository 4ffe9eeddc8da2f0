"""Self-collision: the broad phase's pair list, the C
oracle's pair phase pinned bit-for-bit to the reference core, and the
reference's own knot-replay golden checksum (tests/golden/knot_*.json,
copied from the reference assets by tests/golden/make_golden.py)."""

import json
import os

import numpy as np
import pytest

from oracle.oracle import OracleStepper, ReferenceStepper, load_reference_core
from paper_2509_04277_b200 import workloads as wl
from paper_2509_04277_b200.scenarios import load_replay
from paper_2509_04277_b200.selfcollide import (SelfCollisionConfig, point_groups,
                                               self_collision_pairs, world_groups)

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
STATE = ("positions", "velocities", "frames", "angular_velocities", "pair_a", "pair_b",
         "pair_min_dist", "pair_acc")


def _bits(a):
    return np.ascontiguousarray(a).view(np.int64)


def test_groups_and_pairs():
    assert point_groups(10, 4) == [(0, 4), (4, 8), (8, 10)]
    w = wl.crossing()
    rod, gi, gs, ge = world_groups(w, 4)
    assert rod.tolist() == [0] * 6 + [1] * 6 and gi.tolist() == list(range(6)) * 2
    assert gs[6] == 24 and ge[-1] == 48
    cfg = SelfCollisionConfig(group_size=4, sphere_radius=0.01, point_radius=2e-3)
    pairs = self_collision_pairs(w.positions, None, [0, 24], cfg)
    # the crossing points (rod 0 near x = 0, rod 1 near y = 0) are 1.5 mm apart
    assert pairs and all(i < 24 <= j for i, j, _ in pairs)
    assert all(np.linalg.norm(w.positions[j] - w.positions[i]) < 4e-3 for i, j, _ in pairs)


def knot_schedule():
    return load_replay(os.path.join(GOLDEN, "knot_session.ndjson"))


def step_with_schedule(stepper, world, schedule, steps):
    """Apply grab/release commands at their recorded steps (what the engine's
    command ring does at the epoch boundary) and step one at a time."""
    nxt = 0
    while world.step_index < steps:
        while nxt < len(schedule) and schedule[nxt][0] <= world.step_index:
            _, name, a = schedule[nxt]
            if name == "grab":
                world.grab(a.get("rod", 0), int(a["index"]), np.asarray(a["target"], dtype=float))
            elif name == "release":
                world.release(a.get("rod", 0), int(a["index"]))
            nxt += 1
        stepper.run(1)


@pytest.mark.parametrize("interval", [1, 3])
def test_oracle_crossing_matches_reference_core(interval):
    if load_reference_core() is None:
        pytest.skip("oracle/_ref not built")
    a, b = wl.crossing(interval=interval), wl.crossing(interval=interval)
    oa, rb = OracleStepper(a), ReferenceStepper(b)
    seen = 0
    for _ in range(150):
        oa.run(1)
        rb.run(1)
        seen = max(seen, oa.contacts)
    assert seen > 0
    for k in STATE:
        assert np.array_equal(_bits(getattr(a, k)), _bits(getattr(b, k))), k


def test_oracle_knot_matches_reference_core():
    if load_reference_core() is None:
        pytest.skip("oracle/_ref not built")
    sched = knot_schedule()
    a, b = wl.knot(), wl.knot()
    step_with_schedule(OracleStepper(a), a, sched, 400)
    step_with_schedule(ReferenceStepper(b), b, sched, 400)
    for k in STATE:
        assert np.array_equal(_bits(getattr(a, k)), _bits(getattr(b, k))), k


def test_oracle_knot_replay_golden_checksum():
    # the reference's acceptance test 13 (test_acceptance.py:455-486)
    with open(os.path.join(GOLDEN, "knot_checksum.json")) as fh:
        rec = json.load(fh)
    w = wl.knot()
    step_with_schedule(OracleStepper(w), w, knot_schedule(), rec["steps"])
    assert abs(float(np.sum(np.abs(w.positions))) - rec["checksum"]) <= rec["tolerance"]
