"""Mesh contacts: the BVH build, the numpy narrow
phase, and the C oracle's contact detection + impulses pinned bit-for-bit to
the reference's compiled core (oracle/_ref) on contact scenes."""

import os
import sys

import numpy as np
import pytest

from oracle.oracle import OracleStepper, ReferenceStepper, load_reference_core
from paper_2509_04277_b200 import bvh, meshes
from paper_2509_04277_b200 import workloads as wl

REF_SRC = "/root/reference/pkg/src"
STATE = ("positions", "velocities", "frames", "angular_velocities", "contact_active",
         "contact_normal", "contact_depth", "contact_acc_n", "contact_acc_t")


def _bits(a):
    a = np.ascontiguousarray(a)
    return a.view(np.uint8) if a.dtype == np.uint8 else a.view(np.int64)


def _reference_bvh():
    if not os.path.isdir(REF_SRC):
        pytest.skip("reference package not present")
    sys.path.insert(0, REF_SRC)
    try:
        import rodsim.bvh as rb
        import rodsim.meshes as rm
    finally:
        sys.path.remove(REF_SRC)
    return rb, rm


def test_meshes_and_tree_match_reference():
    rb, rm = _reference_bvh()
    for kw in ({}, {"curvature": 0.0, "rings": 20, "segments": 7}):
        v1, t1 = rm.curved_tube(**kw)
        v2, t2 = meshes.curved_tube(**kw)
        assert np.array_equal(_bits(v1), _bits(v2)) and np.array_equal(t1, t2)
    v1, t1 = rm.floor_mesh(size=0.3, cells=6)
    v2, t2 = meshes.floor_mesh(size=0.3, cells=6)
    assert np.array_equal(_bits(v1), _bits(v2)) and np.array_equal(t1, t2)
    rng = np.random.default_rng(3)
    for v, t in (meshes.curved_tube(), (rng.normal(size=(60, 3)), rng.integers(0, 60, (97, 3)))):
        a, b = rb.build_aabb_tree(v, t), bvh.build_aabb_tree(v, t)
        for f in ("node_min", "node_max", "node_start", "node_count", "tri_order"):
            assert np.array_equal(getattr(a, f), getattr(b, f)), f
        assert a.max_depth == b.max_depth
        for _ in range(40):
            c = rng.normal(size=3) * 0.2
            assert rb.broadphase_query(a, c, 0.03)[0] == bvh.broadphase_query(b, c, 0.03)[0]


def test_narrow_phase_kats():
    a, b, c = np.array([0.0, 0, 0]), np.array([1.0, 0, 0]), np.array([0.0, 1, 0])
    # above the face interior: normal +z, depth r - height
    n, d = bvh.sphere_triangle([0.2, 0.2, 0.05], 0.1, a, b, c)
    assert np.allclose(n, [0, 0, 1]) and abs(d - 0.05) < 1e-15
    # below: the normal flips toward the centre
    n, d = bvh.sphere_triangle([0.2, 0.2, -0.05], 0.1, a, b, c)
    assert np.allclose(n, [0, 0, -1])
    assert bvh.sphere_triangle([0.2, 0.2, 0.2], 0.1, a, b, c) is None
    # vertex / edge regions of the closest point
    assert np.array_equal(bvh.closest_point_on_triangle(np.array([-1.0, -1, 0]), a, b, c), a)
    assert np.allclose(bvh.closest_point_on_triangle(np.array([0.5, -1, 0]), a, b, c), [0.5, 0, 0])
    with pytest.raises(bvh.DegenerateTriangleError):
        bvh.sphere_triangle([0, 0, 0], 1.0, a, b, 2 * b)
    # aggregation: weighted normal, max depth; cancelling normals -> deepest
    n, d = bvh.aggregate_response([(np.array([0, 0, 1.0]), 0.1), (np.array([0, 1.0, 0]), 0.1)])
    assert np.allclose(n, [0, 2 ** -0.5, 2 ** -0.5]) and d == 0.1
    n, d = bvh.aggregate_response([(np.array([0, 0, 1.0]), 0.1), (np.array([0, 0, -1.0]), 0.2 - 0.1)])
    assert d == 0.1


def _pin(make, steps):
    if load_reference_core() is None:
        pytest.skip("oracle/_ref not built")
    a, b = make(), make()
    oa = OracleStepper(a)
    rb = ReferenceStepper(b)
    contacts = []
    for _ in range(steps):
        oa.run(1)
        rb.run(1)
        contacts.append(oa.contacts)
    for k in STATE:
        assert np.array_equal(_bits(getattr(a, k)), _bits(getattr(b, k))), k
    assert oa.error_step == rb.error_step
    return a, contacts


def test_oracle_floor_drop_matches_reference_core():
    w, contacts = _pin(lambda: wl.floor_drop(restitution=0.2, mu=0.3), 300)
    assert max(contacts) > 0          # the rod hit the floor and bounced


def test_oracle_insertion_matches_reference_core():
    tube = {"length": 0.2, "radius": 0.006, "rings": 30, "segments": 12}
    w, contacts = _pin(lambda: wl.insertion(points=40, length=0.1, speed=0.5, tube=tube), 400)
    assert max(contacts) > 0
