"""ctypes binding of the C ABI in include/rodsim_b200.h.

`librodsim_b200.so` is built in-tree (`make`, or `__graft_entry__.build()`)
and holds the sm_100a kernels.  There is no fallback: importing the engine
without the library, or running it without a CUDA device, raises.
"""

import ctypes
import json
import os

import numpy as np

LIB_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)),
                        "librodsim_b200.so")

RS_ABI_VERSION = 2
RS_OK = 0
RS_E_INVALID = -1
RS_E_CUDA = -2
RS_E_UNSUPPORTED = -3
RS_E_RING_FULL = -4
RS_E_RUNTIME = -5

RS_F64_MIRROR = 0
RS_F32 = 1
RS_F64_FAST = 2
PRECISIONS = {"f64": RS_F64_MIRROR, "f32": RS_F32, "f64_fast": RS_F64_FAST}

RS_STATE = 0x1
RS_STATIC = 0x2
RS_CONTROL = 0x4
RS_STATIC_IF_CHANGED = 0x8

_p = ctypes.c_void_p
_i32 = ctypes.c_int32
_i64 = ctypes.c_int64
_f64 = ctypes.c_double


class WorldDesc(ctypes.Structure):
    """Mirror of `rs_world_desc`."""

    _fields_ = [
        ("abi_version", _i32), ("precision", _i32), ("device", _i32),
        ("force_tier", _i32), ("force_ctas", _i32), ("force_variant", _i32),
        ("P", _i64), ("E", _i64), ("R", _i64), ("iters", _i64),
        ("step_index", _i64),
        ("dt", _f64), ("beta", _f64), ("gx", _f64), ("gy", _f64), ("gz", _f64),
        ("rod_offsets", _p),
        ("pos", _p), ("vel", _p), ("q", _p), ("w", _p),
        ("rest", _p), ("ustar", _p), ("mass", _p), ("invm", _p),
        ("inert", _p), ("fext", _p),
        ("ks", _p), ("kp", _p), ("gt", _p), ("gr", _p), ("ext", _p),
        ("kb", _p),
        ("plock", _p), ("flock", _p), ("jvalid", _p),
        ("elem_point", _p), ("elem_parity", _p),
        ("drv_pt", _p), ("drv_fr", _p),
        ("nbind", _i64), ("bind_a", _p), ("bind_b", _p), ("bind_mode", _p),
        ("drv_v", _p), ("drv_rot", _p),
        ("ngrab", _i64), ("g_act", _p), ("g_pt", _p), ("g_tgt", _p),
        ("has_mesh", _i64), ("n_nodes", _i64), ("mesh_depth", _i64),
        ("n_tris", _i64), ("n_verts", _i64),
        ("nmin", _p), ("nmax", _p), ("nstart", _p), ("ncount", _p),
        ("torder", _p), ("tris", _p), ("verts", _p),
        ("cradii", _p), ("cmask", _p), ("cact", _p), ("cnorm", _p), ("cdepth", _p),
        ("cacc_n", _p), ("cacc_t", _p),
        ("coll_interval", _i64), ("coll_margin", _f64), ("restitution", _f64), ("mu", _f64),
        ("has_self", _i64), ("n_groups", _i64), ("excl", _i64), ("pair_cap", _i64),
        ("grp_rod", _p), ("grp_gi", _p), ("grp_s", _p), ("grp_e", _p),
        ("touch", _f64), ("broad", _f64),
        ("pair_a", _p), ("pair_b", _p), ("pair_md", _p), ("pair_acc", _p),
        ("live", _i64),
    ]


# (symbol, restype, argtypes) of every entry point declared in the header
SIGNATURES = [
    ("rs_create", _i32, [ctypes.POINTER(WorldDesc), ctypes.POINTER(_p)]),
    ("rs_upload", _i32, [_p, ctypes.c_uint32]),
    ("rs_run_epoch", _i32, [_p, _i64, ctypes.POINTER(_i64), ctypes.POINTER(_i64)]),
    ("rs_download", _i32, [_p, ctypes.c_uint32]),
    ("rs_run_epoch_host", _i32, [_p, _i64, ctypes.POINTER(_i64), ctypes.POINTER(_i64)]),
    ("rs_synchronize", _i32, [_p]),
    ("rs_error_step", _i64, [_p]),
    ("rs_step_counter", _i64, [_p]),
    ("rs_update_params", _i32, [_p, _f64, _i64]),
    ("rs_stage_commands", _i32, [_p, _p, _i64, _p]),
    ("rs_applied_step_for", _i64, [_p, _i64]),
    ("rs_read_snapshot", _i32, [_p, _p, _p, ctypes.POINTER(_i64), ctypes.POINTER(_i64)]),
    ("rs_destroy", None, [_p]),
    ("rs_last_error", ctypes.c_char_p, []),
    ("rs_enable_timing", _i32, [_p, _i32]),
    ("rs_last_kernel_ms", _f64, [_p]),
    ("rs_launch_count", _i64, [_p]),
    ("rs_last_redo_count", _i64, [_p]),
    ("rs_plan_json", _i32, [_p, ctypes.c_char_p, _i64]),
    ("rs_device_ptr", _i32, [_p, _i32, ctypes.POINTER(_p)]),
    ("rs_selftest_div", _i32, [_p, _p, _i64, _p, _p]),
    ("rs_selftest_fn", _i32, [_i32, _p, _i64, _p, _p]),
    ("rs_timer_start", _i32, [_p]),
    ("rs_timer_stop", _i32, [_p]),
    ("rs_timer_ms", _f64, [_p]),
    ("rs_pipe_peak", _i32, [_i32, ctypes.POINTER(_f64)]),
    ("rs_plan_dry", _i32, [ctypes.POINTER(WorldDesc), _i32, ctypes.c_char_p, _i64]),
    ("rs_micro", _i32, [_i32, _i32, ctypes.POINTER(_f64)]),
    ("rs_live_snapshots", _i32, [_p, _i32]),
    ("rs_barrier_timing", _i32, [_p, _i32]),
]

MICRO_KINDS = {"dadd": 0, "dmul": 1, "dfma": 2, "div": 3, "sqrt_add": 4, "div_rn": 5,
               "rcp": 6, "lds": 7, "bar_sync": 8, "cluster_barrier": 9, "dsmem": 10,
               "neighbour_sync": 11, "grid_flags": 12}


def micro(kind, param=0):
    """(cycles, ns) per operation of a latency microbenchmark (rs_micro)."""
    lib = load_library()
    out = (_f64 * 2)()
    check(lib.rs_micro(MICRO_KINDS.get(kind, kind), int(param), out), lib)
    return out[0], out[1]


def pipe_peak(kind):
    """Measured ops/s of one pipe: 0 DFMA, 1 DADD, 2 DMUL, 3 FFMA."""
    lib = load_library()
    out = _f64(0.0)
    check(lib.rs_pipe_peak(int(kind), ctypes.byref(out)), lib)
    return out.value

_LIB = None


def load_library(path=None):
    """Load (once) and type the shared library; raises if it is missing."""
    global _LIB
    if _LIB is not None and path is None:
        return _LIB
    path = path or LIB_PATH
    if not os.path.exists(path):
        raise ImportError(
            f"{path} not found: build the CUDA library first "
            "(`make` or `python -c 'import __graft_entry__ as g; g.build()'`)")
    lib = ctypes.CDLL(path)
    for name, res, args in SIGNATURES:
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    if path == LIB_PATH:
        _LIB = lib
    return lib


class RodsimError(RuntimeError):
    pass


def check(code, lib=None):
    if code == RS_OK:
        return
    lib = lib or load_library()
    msg = lib.rs_last_error().decode(errors="replace")
    if code == RS_E_INVALID:
        raise ValueError(msg)
    if code == RS_E_UNSUPPORTED:
        raise NotImplementedError(msg)
    raise RodsimError(msg)


def _ptr(a):
    return None if a is None else a.ctypes.data


def build_desc(world, precision="f64", device=0, force_tier=-1, force_ctas=0,
               force_variant=-1, live=False):
    """`rs_world_desc` over the World's arrays (bound by pointer, like
    make_context, _core.pyx:219-403) plus the dict keeping them alive."""
    w = world
    c = np.ascontiguousarray
    offs = np.array([i.point_offset for i in w.rod_infos] + [w.num_points],
                    dtype=np.int64)
    arrays = {
        "rod_offsets": offs,
        "pos": w.positions, "vel": w.velocities, "q": w.frames,
        "w": w.angular_velocities,
        "rest": c(w.rest_lengths), "ustar": c(w.intrinsic_strains),
        "mass": c(w.masses), "invm": c(w.inv_masses),
        "inert": c(w.inertias), "fext": c(w.external_forces),
        "ks": c(w.stretch_k), "kp": c(w.penalty_k), "gt": c(w.gamma_t),
        "gr": c(w.gamma_r), "ext": c(w.extensible), "kb": c(w.bend_k),
        "plock": c(w.point_locked).view(np.uint8),
        "flock": c(w.frame_locked).view(np.uint8),
        "jvalid": c(w.junction_valid).view(np.uint8),
        "elem_point": c(w.elem_point, dtype=np.int64),
        "elem_parity": c(w.elem_parity, dtype=np.int64),
        "drv_pt": c(w.driven_point, dtype=np.int64),
        "drv_fr": c(w.driven_frame, dtype=np.int64),
        "bind_a": c(w.bind_a, dtype=np.int64),
        "bind_b": c(w.bind_b, dtype=np.int64),
        "bind_mode": c(w.bind_mode, dtype=np.int64),
        "drv_v": w.driver_velocity, "drv_rot": w.driver_rotation,
        "g_act": w.grab_active, "g_pt": w.grab_point, "g_tgt": w.grab_target,
        # contact slots are state (mutated in place, like the reference's)
        "cradii": c(w.contact_radii), "cmask": c(w.collide_mesh_mask).view(np.uint8),
        "cact": w.contact_active, "cnorm": w.contact_normal, "cdepth": w.contact_depth,
        "cacc_n": w.contact_acc_n, "cacc_t": w.contact_acc_t,
    }
    cfg = w.self_collision if getattr(w, "self_collision_enabled", False) else None
    if cfg is not None:
        from .selfcollide import world_groups
        g_rod, g_gi, g_s, g_e = world_groups(w, cfg.group_size)
        arrays.update({"grp_rod": g_rod, "grp_gi": g_gi, "grp_s": g_s, "grp_e": g_e,
                       "pair_a": w.pair_a, "pair_b": w.pair_b, "pair_md": w.pair_min_dist,
                       "pair_acc": w.pair_acc})
    tree = getattr(w, "tree", None)
    if tree is not None:
        arrays.update({
            "nmin": c(tree.node_min, dtype=float), "nmax": c(tree.node_max, dtype=float),
            "nstart": c(tree.node_start, dtype=np.int64),
            "ncount": c(tree.node_count, dtype=np.int64),
            "torder": c(tree.tri_order, dtype=np.int64),
            "tris": c(tree.triangles, dtype=np.int64), "verts": c(tree.vertices, dtype=float)})
    for k in ("pos", "vel", "q", "w", "drv_v", "drv_rot", "g_act", "g_pt", "g_tgt",
              "cact", "cnorm", "cdepth", "cacc_n", "cacc_t"):
        a = arrays[k]
        if not (a.flags.c_contiguous and a.flags.writeable):
            raise ValueError(f"world array {k} must be C-contiguous and writeable")
    d = WorldDesc()
    d.abi_version = RS_ABI_VERSION
    d.precision = PRECISIONS[precision]
    d.device = device
    d.force_tier = force_tier
    d.force_ctas = force_ctas
    d.force_variant = force_variant
    d.P, d.E, d.R = w.num_points, w.num_elements, len(w.rod_infos)
    d.iters = w.solver.iterations
    d.step_index = w.step_index
    d.dt = w.dt
    d.beta = w.solver.position_bias
    d.gx, d.gy, d.gz = (float(x) for x in w.gravity)
    for name, arr in arrays.items():
        setattr(d, name, _ptr(arr))
    d.nbind = arrays["bind_a"].shape[0]
    d.ngrab = arrays["g_act"].shape[0]
    if tree is not None:
        d.has_mesh = 1
        d.n_nodes = arrays["nmin"].shape[0]
        d.mesh_depth = int(tree.max_depth)
        d.n_tris = arrays["tris"].shape[0]
        d.n_verts = arrays["verts"].shape[0]
    d.coll_interval = int(w.collision_interval)
    d.coll_margin = float(w.collision_margin)
    d.restitution = float(w.solver.restitution)
    d.mu = float(w.solver.mu)
    d.live = int(bool(live))
    if cfg is not None:
        d.has_self = 1
        d.n_groups = arrays["grp_rod"].shape[0]
        d.excl = int(cfg.neighbor_exclusion)
        d.pair_cap = arrays["pair_a"].shape[0]
        d.touch = 2.0 * cfg.point_radius
        d.broad = 2.0 * cfg.sphere_radius
    return d, arrays


def plan_dry(world, num_sms=148, precision="f64", **force):
    """Launch plan for `world` without a device (rs_plan_dry)."""
    lib = load_library()
    d, keep = build_desc(world, precision, 0, force.get("force_tier", -1),
                         force.get("force_ctas", 0), force.get("force_variant", -1))
    buf = ctypes.create_string_buffer(1 << 16)
    check(lib.rs_plan_dry(ctypes.byref(d), int(num_sms), buf, len(buf)), lib)
    del keep
    return json.loads(buf.value.decode())


# rs_run_epoch with plain integer arguments (handle and out-parameter
# addresses): the cheapest ctypes conversion for one-step launches
_RUN_PROTO = ctypes.CFUNCTYPE(ctypes.c_int32, _p, _i64, _p, _p)


class DeviceWorld:
    """One device mirror of a World (a C handle) plus the arrays it binds.

    `arrays` keeps every bound numpy array alive, like the reference
    context's `refs` (_core.pyx:180, 402).
    """

    def __init__(self, world, precision="f64", device=0, force_tier=-1,
                 force_ctas=0, force_variant=-1, live=False):
        self.lib = load_library()
        self.world = world
        self.precision = precision
        self.desc, self.arrays = build_desc(world, precision, device, force_tier,
                                            force_ctas, force_variant, live)
        d = self.desc
        h = _p()
        check(self.lib.rs_create(ctypes.byref(d), ctypes.byref(h)), self.lib)
        self.handle = h
        # run()'s out-parameters and entry point, made once: a one-step
        # launch is a few microseconds, and the per-call ctypes objects were
        # a third of its host time
        self._contacts, self._bns = _i64(0), _i64(0)
        self._out = (ctypes.addressof(self._contacts), ctypes.addressof(self._bns))
        self._hval = h.value
        self._run_epoch = _RUN_PROTO(("rs_run_epoch", self.lib))

    def state_pointers(self):
        return tuple(self.arrays[k].ctypes.data for k in ("pos", "vel", "q", "w"))

    def upload(self, mask):
        check(self.lib.rs_upload(self.handle, mask), self.lib)

    def run(self, steps):
        rc = self._run_epoch(self._hval, int(steps), *self._out)
        if rc != RS_OK:
            check(rc, self.lib)
        return self._contacts.value, self._bns.value

    def run_host(self, steps):
        """Upload the state, run `steps` steps, download the state (one
        call, copies pipelined with the launches where the plan allows)."""
        contacts, bns = _i64(0), _i64(0)
        check(self.lib.rs_run_epoch_host(self.handle, int(steps), ctypes.byref(contacts),
                                         ctypes.byref(bns)), self.lib)
        return contacts.value, bns.value

    def download(self, mask=RS_STATE):
        check(self.lib.rs_download(self.handle, mask), self.lib)

    def synchronize(self):
        check(self.lib.rs_synchronize(self.handle), self.lib)

    def error_step(self):
        return int(self.lib.rs_error_step(self.handle))

    def step_counter(self):
        return int(self.lib.rs_step_counter(self.handle))

    def update_params(self, dt, iters):
        check(self.lib.rs_update_params(self.handle, float(dt), int(iters)), self.lib)

    def barrier_timing(self, on=True):
        """Account barrier waits in run()'s barrier_ns (rs_barrier_timing)."""
        check(self.lib.rs_barrier_timing(self.handle, int(bool(on))), self.lib)

    def stage_commands(self, ops):
        ops = np.ascontiguousarray(ops, dtype=np.float64)
        if ops.ndim != 2 or ops.shape[1] != 6:
            raise ValueError("ops must have shape (n, 6)")
        slots = np.zeros(ops.shape[0], dtype=np.int64)
        code = self.lib.rs_stage_commands(self.handle, ops.ctypes.data, ops.shape[0],
                                          slots.ctypes.data)
        if code == RS_E_RING_FULL:
            raise RuntimeError(self.lib.rs_last_error().decode())
        check(code, self.lib)
        return [int(s) for s in slots]

    def applied_step_for(self, slot):
        return int(self.lib.rs_applied_step_for(self.handle, int(slot)))

    def live_snapshots(self, on=True):
        check(self.lib.rs_live_snapshots(self.handle, 1 if on else 0), self.lib)

    def read_snapshot(self):
        w = self.world
        pos = np.empty((w.num_points, 3))
        q = np.empty((w.num_elements, 4))
        seq, step = _i64(0), _i64(0)
        check(self.lib.rs_read_snapshot(self.handle, pos.ctypes.data, q.ctypes.data,
                                        ctypes.byref(seq), ctypes.byref(step)), self.lib)
        return seq.value, step.value, pos, q

    def enable_timing(self, on=True):
        check(self.lib.rs_enable_timing(self.handle, 1 if on else 0), self.lib)

    def last_kernel_ms(self):
        return float(self.lib.rs_last_kernel_ms(self.handle))

    def launch_count(self):
        return int(self.lib.rs_launch_count(self.handle))

    def last_redo_count(self):
        """Rods the last speculative batched launch left to the exact kernel."""
        return int(self.lib.rs_last_redo_count(self.handle))

    def timer_start(self):
        check(self.lib.rs_timer_start(self.handle), self.lib)

    def timer_stop(self):
        check(self.lib.rs_timer_stop(self.handle), self.lib)

    def timer_ms(self):
        return float(self.lib.rs_timer_ms(self.handle))

    def plan(self):
        buf = ctypes.create_string_buffer(1 << 16)
        check(self.lib.rs_plan_json(self.handle, buf, len(buf)), self.lib)
        return json.loads(buf.value.decode())

    def device_ptr(self, which):
        out = _p()
        check(self.lib.rs_device_ptr(self.handle, int(which), ctypes.byref(out)), self.lib)
        return out.value

    def close(self):
        if getattr(self, "handle", None):
            self.lib.rs_destroy(self.handle)
            self.handle = None
            self._hval = None   # run() after close: a null handle (RS_E_INVALID)

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
