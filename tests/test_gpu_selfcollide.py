"""GPU parity of self-collision: the broad phase's
pair list and the ordered pair impulses in the step kernel, raw-bit equal
to the C oracle (pinned to the reference core by tests/test_selfcollide.py),
and the reference's own knot-replay golden checksum after 16000 steps."""

import json
import os

import numpy as np
import pytest

from oracle.oracle import OracleStepper
from paper_2509_04277_b200 import workloads as wl
from paper_2509_04277_b200.engine import Engine
from paper_2509_04277_b200.scenarios import load_replay, replay
from test_selfcollide import GOLDEN, STATE, step_with_schedule

pytestmark = pytest.mark.gpu


def _bits(a):
    return np.ascontiguousarray(a).view(np.int64)


@pytest.mark.parametrize("interval,k", [(1, 10), (3, 7)])
def test_crossing_bitwise(interval, k):
    g, r = wl.crossing(interval=interval), wl.crossing(interval=interval)
    ref = OracleStepper(r)
    counts = []
    with Engine(g) as eng:
        for _ in range(150 // k):
            counts.append((eng.run_epoch(k)["contacts"], None))
            ref.run(k)
            counts[-1] = (counts[-1][0], ref.contacts)
    assert all(a == b for a, b in counts) and max(a for a, _ in counts) > 0
    for key in STATE:
        assert np.array_equal(_bits(getattr(g, key)), _bits(getattr(r, key))), key


@pytest.mark.parametrize("points", [257, 400])
def test_self_collision_beyond_513_points_bitwise(points):
    # the paper's knot size, 2 x 256 elements = 514 points, and larger: one
    # CTA of the largest variant, the broad phase built by the whole CTA
    # (ordered scan), the pair impulses in list order
    g, r = wl.crossing(points=points, length=0.002 * (points - 1)), \
        wl.crossing(points=points, length=0.002 * (points - 1))
    ref = OracleStepper(r)
    counts = []
    with Engine(g) as eng:
        grp = eng.plan()["groups"][0]
        assert grp["tier"] == "cta" and grp["points"] == 2 * points and grp["self_collision"]
        for _ in range(12):
            counts.append(eng.run_epoch(10)["contacts"])
            ref.run(10)
            assert counts[-1] == ref.contacts
    assert max(counts) > 0
    for key in STATE:
        assert np.array_equal(_bits(getattr(g, key)), _bits(getattr(r, key))), key


def test_knot_replay_bitwise():
    sched = load_replay(os.path.join(GOLDEN, "knot_session.ndjson"))
    g, r = wl.knot(), wl.knot()
    with Engine(g) as eng:
        replay(eng, sched, 600, batch=100)
    step_with_schedule(OracleStepper(r), r, sched, 600)
    for key in STATE:
        assert np.array_equal(_bits(getattr(g, key)), _bits(getattr(r, key))), key


def test_knot_replay_golden_checksum():
    # the reference's acceptance test 13 (test_acceptance.py:455-486) on the GPU
    with open(os.path.join(GOLDEN, "knot_checksum.json")) as fh:
        rec = json.load(fh)
    w = wl.knot()
    ia, ib = w.rod_infos
    a = slice(ia.point_offset, ia.point_offset + ia.num_points)
    b = slice(ib.point_offset, ib.point_offset + ib.num_points)
    seps = []

    def min_sep(world):
        d = np.linalg.norm(world.positions[a][:, None, :] - world.positions[b][None, :, :], axis=2)
        seps.append(float(d.min()))
    with Engine(w) as eng:
        replay(eng, load_replay(os.path.join(GOLDEN, "knot_session.ndjson")), rec["steps"],
               batch=100, on_epoch=min_sep)
    checksum = float(np.sum(np.abs(w.positions)))
    assert abs(checksum - rec["checksum"]) <= rec["tolerance"]
    assert min(seps) >= 0.95 * 2.0 * ia.params.radius
