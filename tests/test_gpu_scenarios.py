"""The bundled scenarios through run_scenario on the GPU (SURVEY.md §8(f)
#4; the reference's backend-parity acceptance test, test_acceptance.py:
210-227): every scenario's World after N steps is raw-bit equal to the C
oracle stepping the same scene with the same command schedule."""

import numpy as np
import pytest

from oracle.oracle import OracleStepper
from paper_2509_04277_b200 import scenarios
from paper_2509_04277_b200.scene import build_world
from test_selfcollide import step_with_schedule

pytestmark = pytest.mark.gpu

STATE = ("positions", "velocities", "frames", "angular_velocities", "contact_active",
         "contact_normal", "contact_depth", "contact_acc_n", "contact_acc_t")


def _bits(a):
    a = np.ascontiguousarray(a)
    return a.view(np.uint8) if a.dtype == np.uint8 else a.view(np.int64)


@pytest.mark.parametrize("name", scenarios.SCENARIO_NAMES)
def test_scenario_bitwise(name):
    steps = 300
    cfg = scenarios.default_config(name)
    table, engine = scenarios.run_scenario(name, cfg, steps=steps, batch=64)
    g = engine.world
    assert g.step_index == steps and len(table.rows) >= steps // 64
    r = build_world(scenarios.default_config(name))
    step_with_schedule(OracleStepper(r), r, scenarios.command_schedule(name, cfg), steps)
    for k in STATE:
        assert np.array_equal(_bits(getattr(g, k)), _bits(getattr(r, k))), k


def test_insertion_driver_advances_base_point():
    # reference test_scenarios.py:38-44: base z = -0.3 + 0.05 * 200 * 1e-4
    cfg = scenarios.default_config("insertion")
    _, engine = scenarios.run_scenario("insertion", cfg, steps=200)
    assert abs(engine.world.positions[0, 2] - (-0.3 + 0.05 * 200 * 1e-4)) <= 1e-9


def test_replay_session_matches_run_scenario():
    cfg = scenarios.default_config("knot_replay")
    w = scenarios.replay_session(cfg, scenarios.resolve_path(cfg, cfg.replay), 500, batch=50)
    _, engine = scenarios.run_scenario("knot_replay", scenarios.default_config("knot_replay"),
                                       steps=500, batch=100)
    assert np.array_equal(_bits(w.positions), _bits(engine.world.positions))


def test_bench_case_rows(tmp_path):
    from paper_2509_04277_b200 import bench as rb
    rows = rb.bench_suite({"n": [33, 600], "batch": [10], "backend": ["serial", "parallel"],
                           "core": ["compiled", "python"], "epochs": 2})
    assert len(rows) == 4 and all(r["per_step_ns"] > 0 for r in rows)
    assert rb.export_rows(rows, str(tmp_path / "b.csv"))
