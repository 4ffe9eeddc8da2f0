"""Host-side API parity with the reference package (CPU only).

Known-answer and property tests for the modules a reference user touches
before stepping: state (RodParams, init_rod, lumping), quat, forces (the
energy/gradient statement the kernel implements), constraints (impulse KATs),
world (flat layout) and partition.  Mirrors pkg/tests/test_rod_core.py,
test_quat.py, test_constraints.py, test_world.py and test_partition.py.
"""

import numpy as np
import pytest

from conftest import random_rod_state, random_unit_quats
from paper_2509_04277_b200 import forces, quat
from paper_2509_04277_b200 import state as st
from paper_2509_04277_b200.constraints import (
    BIDIRECTIONAL, ONE_WAY, Contact, ConstraintSet, SolverConfig,
    binding_impulse, contact_impulse, distance_impulse, iterate_constraints,
    self_pair_impulse)
from paper_2509_04277_b200.partition import (block_ranges, partition_blocks,
                                             partition_world)
from paper_2509_04277_b200.world import (BIND_BIDIRECTIONAL, BIND_ONE_WAY,
                                         GRAB_CAPACITY, World)

DT, BETA = 1e-4, 0.2


def _params(**kw):
    base = dict(radius=2e-3, stretch_modulus=1e6, bend_modulus=1e5,
                shear_modulus=5e4, linear_density=0.05, penalty_stiffness=2.0,
                extensible=True)
    base.update(kw)
    return st.RodParams(**base)


def _energy(s, p):
    e = forces.elastic_energies(s, p)
    return e["stretch"] + e["bend"] + e["penalty"]


# -- quaternions ---------------------------------------------------------------

def test_hamilton_product_composes_rotations(rng):
    for qa, qb in zip(random_unit_quats(rng, 20), random_unit_quats(rng, 20)):
        assert np.allclose(quat.to_matrix(quat.multiply(qa, qb)),
                           quat.to_matrix(qa) @ quat.to_matrix(qb), atol=1e-12)


def test_director3_is_third_column_and_jacobian_matches_fd(rng):
    q = random_unit_quats(rng, 30)
    for qi in q:
        assert np.allclose(quat.director3(qi), quat.to_matrix(qi)[:, 2], atol=1e-12)
    jac = quat.director3_jacobian(q)
    h = 1e-7
    for i in range(5):
        for c in range(4):
            dq = np.zeros(4)
            dq[c] = h
            fd = (quat.director3(q[i] + dq) - quat.director3(q[i] - dq)) / (2 * h)
            assert np.allclose(jac[i, :, c], fd, atol=1e-6)


def test_b_forms_are_skew_and_match_conjugate_product(rng):
    for b in quat.B_MATRICES:
        assert np.array_equal(b, -b.T)
    q = random_unit_quats(rng, 500)
    qp = rng.normal(size=(500, 4))
    assert np.max(np.abs(forces.darboux_strains(q, qp)
                         - forces.darboux_strains_bmatrix(q, qp))) < 1e-12


def test_rotate_and_axis_angle():
    q = quat.from_axis_angle((0.0, 0.0, 1.0), np.pi / 2)
    assert np.allclose(quat.rotate(q, np.array([1.0, 0.0, 0.0])), [0, 1, 0], atol=1e-12)


# -- rod state and parameters -----------------------------------------------

def test_stiffness_exponents_and_validation():
    p4, p2 = _params(), _params(cross_section_exponent="r2")
    r = p4.radius
    assert p4.bend_stiffness[0] == pytest.approx(p4.bend_modulus * np.pi * r**4 / 4)
    assert p2.bend_stiffness[0] == pytest.approx(p2.bend_modulus * np.pi * r**2 / 4)
    assert p4.bend_stiffness[2] == pytest.approx(p4.shear_modulus * np.pi * r**4 / 2)
    assert p4.stretch_stiffness == pytest.approx(p4.stretch_modulus * np.pi * r**2)
    for bad in (dict(radius=0.0), dict(cross_section_exponent="r3"),
                dict(damping_translational=-1.0)):
        with pytest.raises(ValueError):
            _params(**bad)


def test_lumped_mass_and_inertia_kats():
    assert np.allclose(st.point_masses(np.array([0.1, 0.3, 0.2]), 2.0), [0.1, 0.4, 0.5, 0.2])
    ms = 0.05 * 0.2
    assert np.allclose(st.frame_inertias(np.array([0.2]), 0.05, 1e-3)[0],
                       [0.25 * ms * 1e-6, 0.25 * ms * 1e-6, 0.5 * ms * 1e-6])


def test_init_rod_straight_and_validated():
    s = st.init_rod(8, 1.0, axis=(0.0, 1.0, 0.0), origin=(1.0, 2.0, 3.0))
    assert s.num_points == 8 and s.num_elements == 7
    assert np.allclose(s.rest_lengths, 1.0 / 7)
    assert np.allclose(quat.director3(s.frames), [0.0, 1.0, 0.0], atol=1e-12)
    for sample in forces.strain_samples(s):
        assert sample.v3 == pytest.approx(1.0) and np.allclose(sample.u, 0.0, atol=1e-12)
    with pytest.raises(ValueError):
        st.init_rod(1, 1.0)
    with pytest.raises(ValueError):
        s2 = s.copy()
        s2.frames[0] *= 2.0
        s2.validate()
    with pytest.raises(st.DegenerateSegmentError):
        st.segment_tangent([0, 0, 0], [0, 0, 0])


# -- forces: the physics statement the kernel restates -----------------------

@pytest.mark.parametrize("term", ["stretch", "bend", "penalty", "all"])
def test_analytic_gradients_match_finite_differences(rng, term):
    tiny = 1e-30
    params = {"stretch": _params(penalty_stiffness=tiny, bend_modulus=tiny, shear_modulus=tiny),
              "bend": _params(stretch_modulus=tiny, penalty_stiffness=tiny),
              "penalty": _params(stretch_modulus=tiny, bend_modulus=tiny, shear_modulus=tiny),
              "all": _params()}[term]
    s = random_rod_state(rng, num_points=8)
    buf = forces.elastic_forces_torques(s, params)
    h = 1e-7
    fd_f = np.zeros_like(s.positions)
    for i in range(s.num_points):
        for k in range(3):
            s2 = s.copy()
            s2.positions[i, k] += h
            ep = _energy(s2, params)
            s2.positions[i, k] -= 2 * h
            fd_f[i, k] = -(ep - _energy(s2, params)) / (2 * h)
    fd_q = np.zeros_like(s.frames)
    for j in range(s.num_elements):
        for k in range(4):
            s2 = s.copy()
            s2.frames[j, k] += h
            ep = _energy(s2, params)
            s2.frames[j, k] -= 2 * h
            fd_q[j, k] = -(ep - _energy(s2, params)) / (2 * h)
    fd_q -= np.sum(fd_q * s.frames, axis=1)[:, None] * s.frames
    assert np.max(np.abs(buf.forces - fd_f)) / max(1.0, np.max(np.abs(fd_f))) < 1e-4
    assert np.max(np.abs(buf.frame_forces - fd_q)) / max(1.0, np.max(np.abs(fd_q))) < 1e-4


def test_rest_rod_is_force_free_and_energy_frame_indifferent(rng):
    buf = forces.elastic_forces_torques(st.init_rod(17, 1.0, axis=(0, 1, 0)), _params())
    assert np.max(np.abs(buf.forces)) <= 1e-12 and np.max(np.abs(buf.body_torques)) <= 1e-12
    s = random_rod_state(rng, num_points=10)
    e0 = _energy(s, _params())
    rot = quat.from_axis_angle(rng.normal(size=3), 1.2345)
    m = s.copy()
    m.positions = quat.rotate(rot, m.positions) + np.array([0.3, -0.2, 0.7])
    m.frames = quat.normalize(quat.multiply(rot, m.frames))
    assert abs(_energy(m, _params()) - e0) <= 1e-10 * max(1.0, abs(e0))


def test_damping_signs():
    s = st.init_rod(4, 0.3)
    s.velocities[2] = (1.0, 0.0, 0.0)
    s.angular_velocities[1] = (0.0, 0.0, 2.0)
    buf = forces.add_damping(s, _params(damping_translational=0.5, damping_rotational=0.1),
                             forces.ForceTorqueBuffer.zeros(4))
    assert buf.forces[2, 0] < 0 < buf.forces[1, 0] and buf.forces[3, 0] > 0
    assert buf.body_torques[1, 2] < 0 < buf.body_torques[0, 2]


# -- constraint impulse KATs ----------------------------------------------------

def test_distance_impulse_kats(rng):
    ja, jb = distance_impulse(np.zeros(3), [1, 0, 0], [1, 0, 0], [-1, 0, 0], 1, 1, 1.0, DT, BETA)
    assert np.allclose(ja, [-1, 0, 0]) and np.allclose(jb, [1, 0, 0])
    ja, jb = distance_impulse(np.zeros(3), [1.01, 0, 0], np.zeros(3), np.zeros(3), 1, 1, 1.0, DT, BETA)
    assert (jb - ja)[0] == pytest.approx(-BETA * 0.01 / DT)
    ja, jb = distance_impulse(np.zeros(3), np.zeros(3), np.zeros(3), np.zeros(3), 1, 1, 1.0, DT, BETA)
    assert not ja.any() and not jb.any()
    for _ in range(20):
        ja, jb = distance_impulse(rng.normal(size=3), rng.normal(size=3), rng.normal(size=3),
                                  rng.normal(size=3), 0.5, 2.0, 0.7, DT, BETA)
        assert np.allclose(ja + jb, 0.0, atol=1e-12)


def test_binding_one_way_leaves_dominant_point():
    pos = np.array([[0.0, 0.0, 0.0], [0.0, 1e-3, 0.0]])
    vel = np.array([[1.0, 0.0, 0.0], [0.0, 0.0, 0.0]])
    out = iterate_constraints(pos, vel.copy(), np.ones(2),
                              ConstraintSet(bindings=[(0, 1, ONE_WAY)]),
                              SolverConfig(iterations=4), DT)
    assert np.array_equal(out[0], vel[0]) and out[1, 1] < 0.0
    ja, jb = binding_impulse(np.zeros(3), [0, 2e-3, 0], np.zeros(3), np.zeros(3), 1, 1, DT, BETA,
                             BIDIRECTIONAL)
    assert np.allclose(ja + jb, 0.0)


def test_contact_and_self_pair_kats():
    c = Contact(0, np.array([0.0, 1.0, 0.0]), 0.0, mu=0.5)
    v, an, at = contact_impulse(np.array([1.0, -1.0, 0.0]), 1.0, c, DT, beta=BETA)
    assert np.allclose(v, [0.5, 0.0, 0.0]) and an == pytest.approx(1.0) and at == pytest.approx(0.5)
    ja, jb, acc = self_pair_impulse(np.zeros(3), [0.01, 0, 0], np.zeros(3), np.zeros(3), 1, 1,
                                    0.004, DT, BETA)
    assert not ja.any() and acc == 0.0


def test_chain_strain_reduced_by_iterations():
    rest = 0.1
    viol = []
    for iters in (1, 5, 10, 20):
        pos = np.outer(np.arange(16), [1.05 * rest, 0.0, 0.0])
        cs = ConstraintSet(distance=[(i, i + 1, rest) for i in range(15)])
        v = iterate_constraints(pos, np.zeros((16, 3)), np.ones(16), cs,
                                SolverConfig(iterations=iters), DT)
        new = pos + DT * v
        viol.append(max(abs(np.linalg.norm(new[i + 1] - new[i]) - rest) for i in range(15)))
    assert all(b <= a + 1e-15 for a, b in zip(viol, viol[1:]))
    with pytest.raises(ValueError):
        SolverConfig(iterations=0)


# -- world layout ----------------------------------------------------------------

def _world(points=(8, 5)):
    w = World()
    for n in points:
        w.add_rod(st.init_rod(n, 0.1 * (n - 1)), st.RodParams())
    return w.finalize()


def test_flat_layout_maps_and_junctions():
    w = _world((8, 5))
    assert (w.num_points, w.num_elements) == (13, 11)
    assert [i.point_offset for i in w.rod_infos] == [0, 8]
    assert [i.elem_offset for i in w.rod_infos] == [0, 7]
    assert list(w.junction_valid) == [True] * 6 + [False] + [True] * 3 + [False]
    w2 = _world((4, 3))
    assert list(w2.elem_point) == [0, 1, 2, 4, 5]
    assert list(w2.elem_parity) == [0, 1, 0, 0, 1]
    assert list(w2.rod_of_point) == [0, 0, 0, 0, 1, 1, 1]


def test_clamps_drivers_bindings_grabs():
    w = _world((8, 5))
    w.clamp_point(1, 2, velocity=(0.1, 0.0, 0.0))
    assert w.point_locked[10] and w.inv_masses[10] == 0.0
    w.set_driver(1)
    assert (w.driven_point[1], w.driven_frame[1]) == (8, 7)
    w6 = _world((6, 6))
    w6.add_bindings(0, 1, BIND_ONE_WAY, stride=2)
    w6.add_bindings(0, 1, BIND_BIDIRECTIONAL, stride=3)
    assert list(w6.bind_a) == [0, 2, 4, 0, 3] and list(w6.bind_b) == [6, 8, 10, 6, 9]
    g = _world((GRAB_CAPACITY + 4,))
    s1 = g.grab(0, 3, (0, 0.1, 0))
    assert g.grab(0, 3, (0, 0.2, 0)) == s1 and np.allclose(g.grab_target[s1], [0, 0.2, 0])
    for i in range(GRAB_CAPACITY - 1):
        g.grab(0, 4 + i, (0, 0, 0))
    with pytest.raises(RuntimeError):
        g.grab(0, GRAB_CAPACITY + 3, (0, 0, 0))
    g.release(0, 3)
    assert not g.grab_active[s1]
    g.release_all_grabs()
    assert not g.grab_active.any()


def test_world_views_diagnostics_and_validation():
    w = _world((8, 5))
    v = w.rod_state(1)
    v.positions[0, 1] = 0.123
    assert w.positions[8, 1] == 0.123
    w4 = _world((4,))
    assert w4.max_strain() == pytest.approx(0.0, abs=1e-12)
    w4.positions[3, 2] += 0.02 * w4.rest_lengths[2]
    assert w4.max_strain() == pytest.approx(0.02, abs=1e-9)
    assert set(w.energies()) == {"stretch", "bend", "penalty"}
    with pytest.raises(ValueError):
        World(dt=0.0)
    with pytest.raises(ValueError):
        World().finalize()
    with pytest.raises(RuntimeError):
        w4.add_rod(st.init_rod(4, 0.3), st.RodParams())


# -- partition ---------------------------------------------------------------

def test_partition_kats_and_properties():
    assert partition_blocks(3072, 512) == [512] * 6
    assert partition_blocks(1030, 512) == [344, 343, 343]
    assert partition_blocks(5, 512) == [5]
    rng = np.random.default_rng(7)
    for _ in range(100):
        n, cap = int(rng.integers(1, 5000)), int(rng.integers(2, 700))
        s = partition_blocks(n, cap)
        assert sum(s) == n and max(s) <= cap and max(s) - min(s) <= 1
    with pytest.raises(ValueError):
        partition_blocks(0)
    w = World()
    for n in (100, 50):
        w.add_rod(st.init_rod(n, 0.1 * n), st.RodParams())
    w.finalize()
    part = partition_world(w, cap=40)
    assert [(b.rod, b.size) for b in part.blocks] == [(0, 34), (0, 33), (0, 33), (1, 25), (1, 25)]
    assert partition_world(w, cap=10, max_blocks=3).block_count == 6   # 3 per rod
    starts, ends = block_ranges(part)
    assert starts.dtype == np.int64 and list(starts) == [0, 34, 67, 100, 125]


# -- numpy twin of the step: forces.* + integrate_* (forces.py:134-236) -------

def test_numpy_twin_integrators_track_the_oracle():
    # An all-extensible free rod has no distance projection, so one step is
    # elastic forces + damping + gravity -> integrate_velocities ->
    # integrate_positions; the numpy twin agrees with the compiled step to
    # rounding (the reference's own check: test_engine.py:175-182, 1e-12).
    from oracle.oracle import OracleStepper
    from paper_2509_04277_b200 import workloads as wl
    p = st.RodParams(**dict(wl.MATERIAL, extensible=True, stretch_modulus=1e6))

    def make():
        w = World(dt=1e-4, gravity=(0.0, -9.81, 0.0), solver=SolverConfig(iterations=3))
        w.add_rod(st.init_rod(20, 0.2, axis=(1.0, 0.3, 0.1)), p)
        w.finalize()
        r = np.random.default_rng(1)
        w.velocities[:] = r.normal(size=w.velocities.shape) * 1e-2
        w.angular_velocities[:] = r.normal(size=w.angular_velocities.shape) * 1e-1
        return w

    a, b = make(), make()
    OracleStepper(a).run(50)
    s = b.rod_state(0)
    for _ in range(50):
        buf = forces.elastic_forces_torques(s, p)
        forces.add_damping(s, p, buf)
        buf.forces += b.masses[:, None] * np.asarray(b.gravity)
        forces.integrate_velocities(s, buf, b.masses, b.inertias, b.dt)
        forces.integrate_positions(s, b.dt)
    assert np.max(np.abs(s.positions - a.positions)) <= 1e-12
    assert np.max(np.abs(s.frames - a.frames)) <= 1e-12
    assert np.max(np.abs(s.velocities - a.velocities)) <= 1e-12
    assert np.max(np.abs(s.angular_velocities - a.angular_velocities)) <= \
        1e-9 * np.max(np.abs(a.angular_velocities))


def test_integrators_locks_and_arguments():
    s = st.init_rod(5, 0.4)
    buf = forces.ForceTorqueBuffer.zeros(5)
    buf.forces[:] = 1.0
    buf.body_torques[:] = 2.0
    m, inert = np.full(5, 0.5), np.full((4, 3), 0.25)
    plock, flock = np.zeros(5, bool), np.zeros(4, bool)
    plock[0] = flock[1] = True
    forces.integrate_velocities(s, buf, m, inert, 0.1, plock, flock)
    assert np.all(s.velocities[0] == 0.0) and np.allclose(s.velocities[1:], 0.2)
    assert np.all(s.angular_velocities[1] == 0.0) and np.allclose(s.angular_velocities[0], 0.8)
    p0 = s.positions.copy()
    forces.integrate_positions(s, 0.1)
    assert np.allclose(s.positions, p0 + 0.1 * s.velocities)
    assert np.allclose(np.linalg.norm(s.frames, axis=1), 1.0)
    with pytest.raises(ValueError):
        forces.integrate_positions(s, 0.0)
    with pytest.raises(ValueError):
        forces.integrate_velocities(s, buf, m, inert, -1.0)
