"""The BASELINE.json configurations as World builders.

cfg1 `cantilever`  inextensible 64-element cantilever under gravity
cfg2 `extensible`  extensible CoRdE rod, 512 elements (E_s = 1e6, L = 1 m)
cfg3 `pair`        catheter/guidewire pair 2 x 512, bidirectional bindings,
                   both bases driven at 5 cm/s, I = 10
cfg4 `sweep`       single inextensible rod of N elements, l = 2 mm
cfg5 `hair`        R rods x 128 elements, roots clamped, random directions
`insertion`        guidewire pushed into a curved tube mesh (mesh contacts)
`floor_drop`       rod dropped onto a floor mesh (contacts + friction)
`knot`             two threads knotted by a recorded grab session (self-collision)
`crossing`         two rods pushed across each other (self-collision pairs)

All use the scenario material defaults (scenarios.py:30-32): r = 1 mm,
E_s = 1e7, E_b = G = 1e6, rho = 0.05 kg/m, K_p = 1, gamma_t = 2e-4,
gamma_r = 1e-8, r^4 stiffness; dt = 1e-4, I = 10, beta = 0.2, gravity
(0, -9.81, 0).
"""

import numpy as np

from . import state as st
from .constraints import SolverConfig
from .world import BIND_BIDIRECTIONAL, World

MATERIAL = dict(radius=1e-3, stretch_modulus=1e7, bend_modulus=1e6,
                shear_modulus=1e6, linear_density=0.05, penalty_stiffness=1.0,
                damping_translational=2e-4, damping_rotational=1e-8)


def _world(iterations=10):
    return World(dt=1e-4, gravity=(0.0, -9.81, 0.0),
                 solver=SolverConfig(iterations=iterations))


def cantilever(elements=64, length=0.4):
    """cfg1: clamped root point and frame, horizontal along x."""
    w = _world()
    w.add_rod(st.init_rod(elements + 1, length, axis=(1.0, 0.0, 0.0)),
              st.RodParams(**MATERIAL))
    w.finalize()
    w.clamp_point(0, 0)
    w.clamp_frame(0, 0)
    return w


def extensible(elements=512, length=1.0):
    """cfg2: extensible rod, E_s = 1e6 (stable at dt = 1e-4, L = 1 m)."""
    w = _world()
    w.add_rod(st.init_rod(elements + 1, length, axis=(1.0, 0.0, 0.0)),
              st.RodParams(**dict(MATERIAL, stretch_modulus=1e6, extensible=True)))
    w.finalize()
    w.clamp_point(0, 0)
    w.clamp_frame(0, 0)
    return w


def pair(elements=512, length=1.0, speed=0.05):
    """cfg3: two rods 3 mm apart along z, coupled point-to-point (v2)."""
    w = _world()
    for y in (1.5e-3, -1.5e-3):
        w.add_rod(st.init_rod(elements + 1, length, axis=(0.0, 0.0, 1.0),
                              origin=(0.0, y, -length)), st.RodParams(**MATERIAL))
    w.finalize()
    w.add_bindings(0, 1, BIND_BIDIRECTIONAL, stride=1)
    for r in (0, 1):
        w.set_driver(r)
        w.driver_velocity[r] = (0.0, 0.0, speed)
    return w


def sweep(elements, seg=2e-3):
    """cfg4: single inextensible cantilever with 2 mm segments."""
    return cantilever(elements, seg * elements)


def hair_axes(rods, first=0):
    """Unit root directions: axis_r ~ N(0, I) with seed r."""
    out = np.empty((rods, 3))
    for r in range(rods):
        a = np.random.default_rng(first + r).normal(size=3)
        out[r] = a / np.linalg.norm(a)
    return out


def hair(rods, elements=128, length=0.4, first=0):
    """cfg5: `rods` independent rods, root points clamped (frames free).

    Rod r (global index first + r) sits at (0.01 (r mod 256), 0.01 (r div
    256), 0) -- shards of a 65536-rod batch use `first` so every rank
    builds exactly its slice of the same global scene.
    """
    w = _world()
    params = st.RodParams(**MATERIAL)
    axes = hair_axes(rods, first)
    for r in range(rods):
        g = first + r
        w.add_rod(st.init_rod(elements + 1, length, axis=axes[r],
                              origin=(0.01 * (g % 256), 0.01 * (g // 256), 0.0)),
                  params)
    w.finalize()
    offs = np.array([i.point_offset for i in w.rod_infos])
    w.point_locked[offs] = True
    w.inv_masses[offs] = 0.0
    w.velocities[offs] = 0.0
    w.static_version += 1
    return w


def shard(total_rods, world_size, rank):
    """(first rod, rod count) of `rank`'s slice of a batch: rods are
    independent, so ranks step disjoint slices with no per-step exchange."""
    if total_rods % world_size:
        raise ValueError("rods must divide evenly across ranks")
    per = total_rods // world_size
    return rank * per, per


def insertion(points=128, length=0.3, speed=0.05, tube=None):
    """Paper insertion scene (scenarios.py:45-53): a guidewire pushed at its
    base into a curved tube (meshes.curved_tube), mesh contacts detected
    every 4th step with a 0.5 mm margin.  `tube` overrides the tube mesh
    parameters (smaller tubes for quick tests)."""
    from . import bvh, meshes
    w = _world()
    w.add_rod(st.init_rod(points, length, axis=(0.0, 0.0, 1.0), origin=(0.0, 0.0, -length)),
              st.RodParams(**MATERIAL))
    w.finalize()
    w.set_mesh(bvh.build_aabb_tree(*meshes.curved_tube(**(tube or {}))))
    w.collision_interval = 4
    w.collision_margin = 5e-4
    w.set_driver(0)
    w.driver_velocity[0] = (0.0, 0.0, speed)
    return w


def floor_drop(points=33, length=0.2, height=0.02, restitution=0.0, mu=0.3):
    """A horizontal rod dropped onto a floor grid (meshes.floor_mesh) with a
    1 cm contact radius: contact detection, normal impulses and friction."""
    from . import bvh, meshes
    w = World(dt=1e-4, gravity=(0.0, -9.81, 0.0),
              solver=SolverConfig(iterations=10, restitution=restitution, mu=mu))
    w.add_rod(st.init_rod(points, length, axis=(1.0, 0.0, 0.2), origin=(-0.1, height, 0.0)),
              st.RodParams(**MATERIAL), contact_radius=0.01)
    w.finalize()
    w.set_mesh(bvh.build_aabb_tree(*meshes.floor_mesh(size=0.3, cells=6)))
    w.velocities[:] = (0.05, -0.5, 0.0)
    return w


THREAD = dict(MATERIAL, bend_modulus=5e3, shear_modulus=5e3,
              damping_translational=2e-3, damping_rotational=1e-7)


def knot():
    """The reference's knot_replay scene (scenarios.py:79-101 through
    scene.build_world, scene.py:262-319): two soft 48-point threads 2 cm
    apart, roots clamped, no gravity, I = 15, beta = 0.5, self-collision
    (groups of 4, 2 cm spheres, 2-group exclusion, 1 mm points).  Driven by
    the recorded grab session tests/golden/knot_session.ndjson."""
    from .selfcollide import SelfCollisionConfig
    w = World(dt=1e-4, gravity=(0.0, 0.0, 0.0),
              solver=SolverConfig(iterations=15, position_bias=0.5),
              self_collision=SelfCollisionConfig(group_size=4, sphere_radius=0.02,
                                                 neighbor_exclusion=2, point_radius=1e-3))
    for z in (0.0, 0.02):
        w.add_rod(st.init_rod(48, 0.24, axis=(1.0, 0.0, 0.0), origin=(-0.12, 0.0, z)),
                  st.RodParams(**THREAD))
    w.finalize()
    w.collision_interval = 1
    w.collision_margin = 0.0
    for r in (0, 1):
        w.clamp_point(r, 0)
    return w


def crossing(points=24, interval=1, length=0.05):
    """Two rods crossing 1.5 mm apart and pushed together: self-collision
    pairs between rods (quick fixture for the pair phase; points=257,
    length=0.5 is the paper's 2 x 256-element size)."""
    from .selfcollide import SelfCollisionConfig
    w = World(dt=1e-4, gravity=(0.0, 0.0, 0.0), solver=SolverConfig(iterations=10),
              self_collision=SelfCollisionConfig(group_size=4, sphere_radius=0.01,
                                                 neighbor_exclusion=2, point_radius=1e-3))
    w.add_rod(st.init_rod(points, length, axis=(1.0, 0.0, 0.0), origin=(-length / 2, 0.0, 0.0)),
              st.RodParams(**THREAD))
    w.add_rod(st.init_rod(points, length, axis=(0.0, 1.0, 0.0), origin=(0.0, -length / 2, 0.0015)),
              st.RodParams(**THREAD))
    w.finalize()
    w.collision_interval = interval
    o = w.rod_infos[1].point_offset
    w.velocities[o:o + points] = (0.0, 0.0, -0.2)
    return w


BUILDERS = {"cantilever": cantilever, "extensible": extensible, "pair": pair,
            "sweep": sweep, "hair": hair, "insertion": insertion, "floor_drop": floor_drop,
            "knot": knot, "crossing": crossing}
