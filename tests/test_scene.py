"""Scene files and bundled scenarios: the schema,
defaults and error paths of the reference's scene module, and World
construction bit-identical to the reference's build_world for every
bundled scenario."""

import json
import os
import sys

import numpy as np
import pytest

from paper_2509_04277_b200 import scenarios, scene
from paper_2509_04277_b200.metrics import HEADER, MetricsTable

REF_SRC = "/root/reference/pkg/src"
ARRAYS = ("positions", "velocities", "frames", "angular_velocities", "rest_lengths",
          "intrinsic_strains", "masses", "inv_masses", "inertias", "stretch_k", "penalty_k",
          "gamma_t", "gamma_r", "bend_k", "point_locked", "frame_locked", "junction_valid",
          "bind_a", "bind_b", "bind_mode", "driven_point", "driven_frame", "driver_velocity",
          "driver_rotation", "contact_radii", "collide_mesh_mask")


def _reference():
    if not os.path.isdir(REF_SRC):
        pytest.skip("reference package not present")
    sys.path.insert(0, ROOT_REF := REF_SRC)
    try:
        from oracle.oracle import load_reference_core
        core = load_reference_core()
        if core is None:
            pytest.skip("oracle/_ref not built")
        sys.modules["rodsim._core"] = core
        import rodsim.scenarios as rsc
        import rodsim.scene as rsn
    finally:
        sys.path.remove(ROOT_REF)
    return rsc, rsn


@pytest.mark.parametrize("name", scenarios.SCENARIO_NAMES)
def test_bundled_scene_matches_reference(name):
    rsc, rsn = _reference()
    ours, theirs = scenarios.default_config(name), rsc.default_config(name)
    assert ours.echo() == theirs.echo()
    a, b = scene.build_world(ours), rsn.build_world(theirs)
    for k in ARRAYS:
        x, y = np.asarray(getattr(a, k)), np.asarray(getattr(b, k))
        assert x.dtype == y.dtype and np.array_equal(x, y), k
    assert (a.tree is None) == (b.tree is None)
    if a.tree is not None:
        for f in ("vertices", "triangles", "node_min", "node_max", "node_start", "node_count",
                  "tri_order"):
            assert np.array_equal(getattr(a.tree, f), getattr(b.tree, f)), f
    assert a.collision_interval == b.collision_interval
    assert a.collision_margin == b.collision_margin


@pytest.mark.parametrize("bad,path", [
    ({"dt": -1.0}, "dt: must be positive"),
    ({"rods": [{"radius": 0.0}]}, "rods[0].radius: must be positive"),
    ({"rods": [{"clamps": [99]}]}, "rods[0].clamps[0]: point index out of range"),
    ({"rods": [{"bogus": 1}]}, "rods[0]: unknown keys ['bogus']"),
    ({"couplings": [{"mode": "v7"}], "rods": [{}, {}]}, "couplings[0].mode"),
    ({"solver": {"position_bias": 2.0}}, "solver.position_bias: must be in [0, 1]"),
    ({"gravity": [0, 0]}, "gravity: expected a list of 3 numbers"),
])
def test_scene_errors_name_the_field(bad, path):
    with pytest.raises(scene.SceneError) as e:
        scene.parse_scene(bad)
    assert path in str(e.value)


def test_scene_round_trip_and_bundle(tmp_path):
    paths = scenarios.write_bundled_scenes(str(tmp_path))
    for name, p in paths.items():
        cfg = scene.load_scene(p)
        assert cfg.echo() == scenarios.default_config(name).echo()
        again = scene.parse_scene(json.loads(json.dumps(cfg.echo())))
        assert again.echo() == cfg.echo()
    with pytest.raises(scene.SceneError):
        scene.load_scene(str(tmp_path / "missing.json"))


def test_replay_loading_and_schedule(tmp_path):
    log = tmp_path / "s.ndjson"
    log.write_text('{"type": "command", "step": 5, "command": {"type": "release", "rod": 0, '
                   '"index": 1}}\n{"type": "status"}\n\n{"type": "command", "step": 2, '
                   '"command": {"type": "grab", "rod": 0, "index": 3, "target": [0, 0, 0]}}\n')
    ev = scenarios.load_replay(str(log))
    assert [e[0] for e in ev] == [2, 5] and ev[0][1] == "grab"
    log.write_text("{not json\n")
    with pytest.raises(ValueError, match="s.ndjson:1"):
        scenarios.load_replay(str(log))
    cfg = scenarios.default_config("knot_replay")
    sched = scenarios.command_schedule("knot_replay", cfg)
    assert len(sched) > 400 and sched[0][1] == "grab"
    with pytest.raises(ValueError):
        scenarios.default_config("nope")


def test_metrics_table(tmp_path):
    t = MetricsTable()
    t.append(epoch=0, steps=10, contacts=3)
    assert t.column("steps") == [10] and t.column("max_strain") == [""]
    with pytest.raises(KeyError):
        t.append(bogus=1)
    text = open(t.export(str(tmp_path / "m.csv"))).read().splitlines()
    assert text[0].split(",") == HEADER
