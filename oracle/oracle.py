"""TEST INFRASTRUCTURE ONLY -- CPU oracles for the CoRdE step.

Two checkers, both usable on any World-like object that has the reference
World's flat arrays (world.py:77-182):

* `OracleStepper` -- ctypes wrapper of oracle/rod_oracle.c, the C
  restatement of the reference compiled step (port).  Pinned bit-for-bit to
  the reference by tests/test_oracle.py (golden fixtures + oracle/_ref).
* `load_reference_core()` / `ReferenceStepper` -- the reference's own
  compiled core `rodsim._core`, built from /root/reference by
  oracle/build_ref.sh into oracle/_ref/ (present wherever that build ran;
  the .so travels with the repo snapshot, the reference sources do not).

Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline legs may use
this module, and only as the checker or the timed CPU baseline.
"""

import ctypes
import glob
import importlib.machinery
import importlib.util
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_LIB = os.path.join(HERE, "liboracle.so")
REF_DIR = os.path.join(HERE, "_ref")

_p = ctypes.c_void_p
_i64 = ctypes.c_int64
_f64 = ctypes.c_double


class RoWorld(ctypes.Structure):
    _fields_ = [
        ("P", _i64), ("E", _i64), ("R", _i64), ("iters", _i64),
        ("dt", _f64), ("beta", _f64), ("gx", _f64), ("gy", _f64), ("gz", _f64),
        ("pos", _p), ("vel", _p), ("q", _p), ("w", _p),
        ("rest", _p), ("ustar", _p), ("inert", _p), ("ks", _p), ("kp", _p),
        ("gt", _p), ("gr", _p), ("ext", _p), ("kb", _p),
        ("mass", _p), ("invm", _p), ("fext", _p),
        ("plock", _p), ("flock", _p), ("elem_point", _p), ("elem_parity", _p),
        ("jvalid", _p),
        ("drv_v", _p), ("drv_rot", _p), ("drv_pt", _p), ("drv_fr", _p),
        ("nbind", _i64), ("bind_a", _p), ("bind_b", _p), ("bind_mode", _p),
        ("ngrab", _i64), ("g_act", _p), ("g_pt", _p), ("g_tgt", _p),
        ("ef", _p), ("ff_own", _p), ("ff_next", _p), ("jtau", _p),
        ("pt_elo", _p), ("pt_ehi", _p),
        ("step", _i64), ("err_step", _i64),
        ("has_mesh", _i64), ("n_nodes", _i64),
        ("nmin", _p), ("nmax", _p), ("verts", _p),
        ("nstart", _p), ("ncount", _p), ("torder", _p), ("tris", _p),
        ("cradii", _p), ("cmask", _p), ("cact", _p), ("cnorm", _p), ("cdepth", _p),
        ("cacc_n", _p), ("cacc_t", _p),
        ("coll_interval", _i64), ("coll_margin", _f64), ("restitution", _f64), ("mu", _f64),
        ("contacts", _i64),
        ("has_self", _i64), ("n_groups", _i64), ("excl", _i64), ("pair_cap", _i64),
        ("grp_rod", _p), ("grp_gi", _p), ("grp_s", _p), ("grp_e", _p), ("grp_c", _p),
        ("touch", _f64), ("broad", _f64),
        ("pair_a", _p), ("pair_b", _p), ("pair_md", _p), ("pair_acc", _p),
        ("pairs", _i64),
    ]


_LIB = None


def load_oracle():
    global _LIB
    if _LIB is None:
        if not os.path.exists(ORACLE_LIB):
            raise ImportError(f"{ORACLE_LIB} missing: run `make oracle/liboracle.so`")
        lib = ctypes.CDLL(ORACLE_LIB)
        for name in ("ro_prepare", "ro_scatter", "ro_gather", "ro_central",
                     "ro_contacts", "ro_integrate"):
            getattr(lib, name).argtypes = [ctypes.POINTER(RoWorld)]
            getattr(lib, name).restype = None
        lib.ro_run.argtypes = [ctypes.POINTER(RoWorld), _i64]
        lib.ro_run.restype = None
        lib.ro_distance.argtypes = [ctypes.POINTER(RoWorld), _i64]
        lib.ro_distance.restype = None
        _LIB = lib
    return _LIB


class OracleStepper:
    """Steps a World's arrays in place with the C restatement."""

    def __init__(self, world):
        self.lib = load_oracle()
        self.world = w = world
        c = np.ascontiguousarray
        E, P = w.num_elements, w.num_points
        self.keep = {
            "pos": w.positions, "vel": w.velocities, "q": w.frames,
            "w": w.angular_velocities,
            "rest": c(w.rest_lengths), "ustar": c(w.intrinsic_strains),
            "inert": c(w.inertias), "ks": c(w.stretch_k), "kp": c(w.penalty_k),
            "gt": c(w.gamma_t), "gr": c(w.gamma_r), "ext": c(w.extensible),
            "kb": c(w.bend_k), "mass": c(w.masses), "invm": c(w.inv_masses),
            "fext": c(w.external_forces),
            "plock": c(w.point_locked).view(np.uint8),
            "flock": c(w.frame_locked).view(np.uint8),
            "elem_point": c(w.elem_point, dtype=np.int64),
            "elem_parity": c(w.elem_parity, dtype=np.int64),
            "jvalid": c(w.junction_valid).view(np.uint8),
            "drv_v": c(w.driver_velocity), "drv_rot": c(w.driver_rotation),
            "drv_pt": c(w.driven_point, dtype=np.int64),
            "drv_fr": c(w.driven_frame, dtype=np.int64),
            "bind_a": c(w.bind_a, dtype=np.int64),
            "bind_b": c(w.bind_b, dtype=np.int64),
            "bind_mode": c(w.bind_mode, dtype=np.int64),
            "g_act": c(w.grab_active), "g_pt": c(w.grab_point, dtype=np.int64),
            "g_tgt": c(w.grab_target),
            "ef": np.zeros((E, 3)), "ff_own": np.zeros((E, 4)),
            "ff_next": np.zeros((E, 4)), "jtau": np.zeros((E, 3)),
            "pt_elo": np.zeros(P, dtype=np.int64),
            "pt_ehi": np.zeros(P, dtype=np.int64),
            # contact slots are World state, stepped in place
            "cradii": c(w.contact_radii), "cmask": c(w.collide_mesh_mask).view(np.uint8),
            "cact": w.contact_active, "cnorm": w.contact_normal, "cdepth": w.contact_depth,
            "cacc_n": w.contact_acc_n, "cacc_t": w.contact_acc_t,
        }
        cfg = w.self_collision if getattr(w, "self_collision_enabled", False) else None
        if cfg is not None:
            from paper_2509_04277_b200.selfcollide import world_groups
            g_rod, g_gi, g_s, g_e = world_groups(w, cfg.group_size)
            self.keep.update({"grp_rod": g_rod, "grp_gi": g_gi, "grp_s": g_s, "grp_e": g_e,
                              "grp_c": np.zeros((g_rod.shape[0], 3)),
                              "pair_a": w.pair_a, "pair_b": w.pair_b,
                              "pair_md": w.pair_min_dist, "pair_acc": w.pair_acc})
        tree = getattr(w, "tree", None)
        if tree is not None:
            if tree.max_depth + 1 > 32:
                raise RuntimeError("tree deeper than the traversal stack capacity")
            self.keep.update({
                "nmin": c(tree.node_min), "nmax": c(tree.node_max), "verts": c(tree.vertices),
                "nstart": c(tree.node_start, dtype=np.int64),
                "ncount": c(tree.node_count, dtype=np.int64),
                "torder": c(tree.tri_order, dtype=np.int64),
                "tris": c(tree.triangles, dtype=np.int64)})
        s = RoWorld()
        s.P, s.E, s.R = P, E, len(w.rod_infos)
        s.iters = w.solver.iterations
        s.dt = w.dt
        s.beta = w.solver.position_bias
        s.gx, s.gy, s.gz = (float(x) for x in w.gravity)
        for k, a in self.keep.items():
            setattr(s, k, a.ctypes.data)
        s.nbind = self.keep["bind_a"].shape[0]
        s.ngrab = self.keep["g_act"].shape[0]
        s.step = w.step_index
        s.err_step = -1
        s.has_mesh = int(tree is not None)
        s.n_nodes = tree.node_min.shape[0] if tree is not None else 0
        s.coll_interval = int(w.collision_interval)
        s.coll_margin = float(w.collision_margin)
        s.restitution = float(w.solver.restitution)
        s.mu = float(w.solver.mu)
        if cfg is not None:
            s.has_self = 1
            s.n_groups = self.keep["grp_rod"].shape[0]
            s.excl = int(cfg.neighbor_exclusion)
            s.touch = 2.0 * cfg.point_radius
            s.broad = 2.0 * cfg.sphere_radius
            s.pair_cap = w.pair_a.shape[0]
        self.s = s
        self.lib.ro_prepare(ctypes.byref(s))

    def run(self, steps):
        self.lib.ro_run(ctypes.byref(self.s), int(steps))
        self.world.step_index += int(steps)

    def set_params(self, dt=None, iterations=None):
        """Engine.set_params between epochs (engine.py:335-355): the World's
        dt / solver.iterations and the context's copies
        (_core.update_params, _core.pyx:1083-1089)."""
        if dt is not None:
            self.world.dt = float(dt)
        if iterations is not None:
            self.world.solver.iterations = int(iterations)
        self.s.dt = self.world.dt
        self.s.iters = self.world.solver.iterations

    @property
    def error_step(self):
        return int(self.s.err_step)

    @property
    def contacts(self):
        """Active mesh contacts + self-collision pairs after the last step
        (step_serial's return, _core.pyx:1080)."""
        return int(self.s.contacts) + int(self.s.pairs)


# ---- the reference's own compiled core ---------------------------------------

def reference_core_path():
    hits = sorted(glob.glob(os.path.join(REF_DIR, "_core*.so")))
    return hits[0] if hits else None


_REF = None


def load_reference_core():
    """Import oracle/_ref/_core*.so (the unmodified reference core) or None."""
    global _REF
    if _REF is None:
        path = reference_core_path()
        if path is None:
            return None
        spec = importlib.util.spec_from_file_location(
            "rodsim._core", path,
            loader=importlib.machinery.ExtensionFileLoader("rodsim._core", path))
        mod = importlib.util.module_from_spec(spec)
        spec.loader.exec_module(mod)
        _REF = mod
    return _REF


class ReferenceStepper:
    """The reference's serial path (`step_serial` per step, engine.py:286-293)
    on a World-like object, partitioned like the reference engine."""

    def __init__(self, world, block_cap=512):
        core = load_reference_core()
        if core is None:
            raise ImportError("oracle/_ref not built (oracle/build_ref.sh)")
        from paper_2509_04277_b200.partition import block_ranges, partition_world
        self.core = core
        self.world = world
        starts, ends = block_ranges(partition_world(world, block_cap))
        self.snap = (np.zeros_like(world.positions), np.zeros_like(world.frames),
                     np.zeros(1, dtype=np.int64), np.zeros(1, dtype=np.int64))
        self.ctx = core.make_context(world, starts, ends, *self.snap)

    def run(self, steps):
        for _ in range(int(steps)):
            self.core.step_serial(self.ctx)
            self.world.step_index += 1

    def set_params(self, dt=None, iterations=None):
        if dt is not None:
            self.world.dt = float(dt)
        if iterations is not None:
            self.world.solver.iterations = int(iterations)
        self.core.update_params(self.ctx, self.world.dt, self.world.solver.iterations)

    @property
    def error_step(self):
        return int(self.core.error_step(self.ctx))
