"""Epoch engine: steps a World on the B200 through the C ABI.

Drop-in for the reference Engine (rodsim/engine.py:144-367): same
constructor, `run_epoch` metrics dict, command tickets, command log,
snapshot buffer and error surfacing.  Both reference backends ("serial",
"parallel") map to the one GPU path -- a persistent sm_100a kernel that
advances K = `steps` time steps per launch.  There is no CPU fallback: if
the CUDA library or device is missing, constructing an Engine raises.

Per epoch (the reference's epoch, _core.pyx:1091-1139):
  1. queued commands are applied at the epoch's first step boundary and
     logged with that step (the serial path's semantics, engine.py:265-270);
  2. host arrays -> HBM (state every epoch; constants when they changed);
  3. one launch per tier runs all K steps on-chip;
  4. HBM -> host arrays; a recorded non-finite / degenerate step raises
     FloatingPointError like the reference (engine.py:328-333).
"""

import queue
import threading
import time
from dataclasses import dataclass

import numpy as np

from . import _lib
from .partition import partition_world

OP_DRIVER_VELOCITY = 0
OP_DRIVER_ROTATION = 1
OP_GRAB = 2
OP_RELEASE = 3

# worlds at most this large re-check their constant arrays every epoch
# (cheap); larger ones re-upload them when World.static_version changes
SMALL_WORLD_POINTS = 1 << 14

_STATIC_ATTRS = ("rest_lengths", "intrinsic_strains", "masses", "inv_masses",
                 "inertias", "external_forces", "stretch_k", "penalty_k",
                 "gamma_t", "gamma_r", "extensible", "bend_k", "point_locked",
                 "frame_locked", "junction_valid", "elem_point", "elem_parity",
                 "driven_point", "driven_frame", "bind_a", "bind_b",
                 "bind_mode", "contact_radii", "collide_mesh_mask")
_BOUND_ATTRS = _STATIC_ATTRS + ("positions", "velocities", "frames",
                                "angular_velocities", "driver_velocity",
                                "driver_rotation", "grab_active",
                                "grab_point", "grab_target", "contact_active",
                                "contact_normal", "contact_depth", "contact_acc_n",
                                "contact_acc_t", "pair_a", "pair_b", "pair_min_dist",
                                "pair_acc")


@dataclass
class Command:
    name: str
    args: dict
    id: int = -1


class Ticket:
    """Resolved with the step index at which the command took effect."""

    def __init__(self, command):
        self.command = command
        self._event = threading.Event()
        self.apply_step = None

    def resolve(self, step):
        self.apply_step = step
        self._event.set()

    def wait(self, timeout=None):
        if not self._event.wait(timeout):
            raise TimeoutError("command not applied in time")
        return self.apply_step


class Mailbox:
    """Multi-producer queue of steering commands."""

    def __init__(self):
        self._queue = queue.Queue()
        self._next_id = 0
        self._lock = threading.Lock()

    def post(self, name, **args):
        with self._lock:
            cmd = Command(name, args, self._next_id)
            self._next_id += 1
        ticket = Ticket(cmd)
        self._queue.put((cmd, ticket))
        return ticket

    def drain(self):
        out = []
        while True:
            try:
                out.append(self._queue.get_nowait())
            except queue.Empty:
                return out


@dataclass
class Snapshot:
    sequence: int
    step_index: int
    positions: np.ndarray
    frames: np.ndarray = None


class SnapshotBuffer:
    """Single-writer seqlock (odd sequence while a publish is in flight)."""

    def __init__(self, world):
        self.positions = np.zeros_like(world.positions)
        self.frames = np.zeros_like(world.frames)
        self.seq = np.zeros(1, dtype=np.int64)
        self.step = np.zeros(1, dtype=np.int64)

    def publish(self, world):
        self.seq[0] += 1
        self.positions[:] = world.positions
        self.frames[:] = world.frames
        self.step[0] = world.step_index
        self.seq[0] += 1

    def read(self, max_retries=100000):
        for _ in range(max_retries):
            s1 = int(self.seq[0])
            if s1 % 2:
                continue
            pos, frames = self.positions.copy(), self.frames.copy()
            step = int(self.step[0])
            if int(self.seq[0]) == s1:
                return Snapshot(s1, step, pos, frames)
        raise RuntimeError("snapshot read kept tearing")


class HaloTracker:
    """Barrier-generation counters per block (stale-halo detection API,
    engine.py:126-141).  On the device the barriers are bar.sync /
    barrier.cluster / release-acquire flags; this host object is kept for
    callers and tests of the reference API."""

    def __init__(self, num_blocks):
        self.generation = np.zeros(num_blocks, dtype=np.int64)

    def barrier(self):
        self.generation += 1

    def check(self, block, neighbor):
        if self.generation[block] != self.generation[neighbor]:
            raise RuntimeError(
                f"stale halo read: block {block} at generation "
                f"{self.generation[block]}, neighbor {neighbor} at "
                f"{self.generation[neighbor]}")
        return True


class Engine:
    """Steps a World on the GPU (reference backends map to the same path)."""

    def __init__(self, world, backend="serial", block_cap=512,
                 use_compiled=None, max_blocks=None, precision="f64",
                 device=0, force_tier=-1, force_ctas=0, force_variant=-1, live=None):
        if backend not in ("serial", "parallel"):
            raise ValueError("backend must be 'serial' or 'parallel'")
        self.world = world
        self.backend = backend
        self.precision = precision
        self.device = device
        self.partition = partition_world(world, block_cap, max_blocks=max_blocks)
        self.mailbox = Mailbox()
        self.snapshot_buffer = SnapshotBuffer(world)
        self.halo = HaloTracker(self.partition.block_count)
        self.command_log = []
        self.last_contacts = 0
        self.compiled = True       # the CUDA core is the only backend
        self._pending = []
        self._force = (force_tier, force_ctas, force_variant)
        # live launches apply commands posted mid-epoch at the next step (the
        # reference's parallel backend); default: on for backend="parallel"
        self._want_live = (backend == "parallel") if live is None else bool(live)
        self._lock = threading.Lock()
        self._stage_lock = threading.Lock()
        self._running = False      # an epoch's launch is in flight
        self._live = False
        self._live_snaps = False   # per-step snapshots requested
        self._snapshot_readers = False
        self._snapshot_stale = False
        self._dev = None
        self._bind()
        self.snapshot_buffer.publish(world)

    # -- device handle -----------------------------------------------------

    def _bind(self):
        if self._dev is not None:
            self._dev.close()
        ft, fc, fv = self._force
        self._dev = _lib.DeviceWorld(self.world, self.precision, self.device,
                                     force_tier=ft, force_ctas=fc,
                                     force_variant=fv, live=self._want_live)
        self._live = bool(self._dev.plan().get("live", False))
        # the parallel backend reports barrier waits (engine.py:300-313: the
        # serial backend's barrier_wait_ns is 0, it has no barriers)
        if self.backend == "parallel":
            self._dev.barrier_timing(True)
        self._live_snaps = False
        self._bound = {a: getattr(self.world, a) for a in _BOUND_ATTRS}
        # the mesh and the collision scalars are bound too (make_context)
        self._bound_scene = self._scene_key()
        self._static_version = self.world.static_version
        self._small = self.world.num_points <= SMALL_WORLD_POINTS

    def _scene_key(self):
        w = self.world
        return (id(w.tree), id(w.self_collision), w.collision_interval,
                w.collision_margin, w.solver.restitution, w.solver.mu)

    def _push(self, state=True):
        """Host -> device before an epoch.  Returns False when the World had
        to be re-bound (everything, state included, is then uploaded);
        state=False leaves the state to rs_run_epoch_host."""
        w = self.world
        if (any(getattr(w, a) is not arr for a, arr in self._bound.items())
                or self._scene_key() != self._bound_scene):
            # an array attribute was replaced: re-bind (re-plans and uploads)
            self._bind()
            return False
        mask = (_lib.RS_STATE if state else 0) | _lib.RS_CONTROL
        if w.static_version != self._static_version:
            mask |= _lib.RS_STATIC
            self._static_version = w.static_version
        elif self._small:
            # the reference reads the static arrays live: catch in-place
            # edits (a memcmp against the last upload, in the library)
            mask |= _lib.RS_STATIC_IF_CHANGED
        self._dev.upload(mask)
        return True

    # -- commands ----------------------------------------------------------

    def post_command(self, name, **args):
        """Queue a command.  Between epochs it applies at the next epoch's
        first step boundary; while an epoch runs on a live plan (one CTA or
        one cluster) it is staged on the device ring right away and the
        kernel applies it at the next step boundary, like the reference's
        parallel backend (engine.py:177-198)."""
        ticket = self.mailbox.post(name, **args)
        if self._running and self._live:
            self._stage_pending()
        return ticket

    def _stage_pending(self):
        """Encode queued commands onto the device ring (_core.stage_commands);
        their tickets resolve once the kernel reports the apply step."""
        with self._stage_lock:
            for cmd, ticket in self.mailbox.drain():
                ops = self._encode(cmd)
                if not ops:
                    ticket.resolve(self.world.step_index)
                    continue
                slots = self._dev.stage_commands(np.array(ops, dtype=np.float64))
                self._pending.append((cmd, ticket, slots[-1]))

    def _encode(self, cmd):
        """Command -> [op, i0, i1, f0, f1, f2] rows (engine.py:200-226)."""
        w, a = self.world, cmd.args
        if cmd.name == "insert_velocity":
            rod = a.get("rod", 0)
            vel = float(a["value"]) * np.asarray(a.get("axis", self._driver_axis(rod)))
            return [[OP_DRIVER_VELOCITY, rod, 0, vel[0], vel[1], vel[2]]]
        if cmd.name == "rotate_velocity":
            return [[OP_DRIVER_ROTATION, a.get("rod", 0), 0, float(a["value"]), 0.0, 0.0]]
        if cmd.name == "grab":
            rod = a.get("rod", 0)
            point = w.rod_infos[rod].point_offset + int(a["index"])
            t = np.asarray(a["target"], dtype=float)
            return [[OP_GRAB, self._grab_slot(point), point, t[0], t[1], t[2]]]
        if cmd.name == "release":
            point = w.rod_infos[a.get("rod", 0)].point_offset + int(a["index"])
            return [[OP_RELEASE, s, 0, 0.0, 0.0, 0.0]
                    for s in range(w.grab_active.shape[0]) if w.grab_point[s] == point]
        raise ValueError(f"unknown command {cmd.name!r}")

    def _grab_slot(self, point):
        w = self.world
        for slot in range(w.grab_active.shape[0]):
            if w.grab_point[slot] == point:
                return slot
        for slot in range(w.grab_active.shape[0]):
            if not w.grab_active[slot] and w.grab_point[slot] == -1:
                w.grab_point[slot] = point
                return slot
        raise RuntimeError("no free grab slot")

    def _driver_axis(self, rod):
        v = self.world.driver_velocity[rod]
        n = np.linalg.norm(v)
        return v / n if n > 0.0 else np.array([0.0, 0.0, 1.0])

    def _apply_command(self, cmd):
        w, a = self.world, cmd.args
        if cmd.name == "insert_velocity":
            rod = a.get("rod", 0)
            w.driver_velocity[rod] = float(a["value"]) * np.asarray(
                a.get("axis", self._driver_axis(rod)))
        elif cmd.name == "rotate_velocity":
            w.driver_rotation[a.get("rod", 0)] = float(a["value"])
        elif cmd.name == "grab":
            w.grab(a.get("rod", 0), int(a["index"]),
                   np.asarray(a["target"], dtype=float))
        elif cmd.name == "release":
            w.release(a.get("rod", 0), int(a["index"]))
        else:
            raise ValueError(f"unknown command {cmd.name!r}")

    def _drain_at_boundary(self):
        for cmd, ticket in self.mailbox.drain():
            self._apply_command(cmd)
            self.command_log.append((self.world.step_index, cmd))
            ticket.resolve(self.world.step_index)

    def stage_commands(self, ops):
        """Stage encoded ops on the device handle's ring; they apply at the
        next epoch's first step boundary (rs_stage_commands)."""
        return self._dev.stage_commands(ops)

    def _resolve_applied(self):
        # _stage_pending may append from a posting thread meanwhile
        with self._stage_lock:
            still = []
            for cmd, ticket, slot in self._pending:
                step = self._dev.applied_step_for(slot)
                if step >= 0:
                    self.command_log.append((step, cmd))
                    ticket.resolve(step)
                else:
                    still.append((cmd, ticket, slot))
            self._pending = still

    # -- stepping ----------------------------------------------------------

    def run_epoch(self, steps):
        """Execute `steps` time steps (one persistent launch); metrics dict."""
        if steps < 1:
            raise ValueError("steps must be >= 1")
        with self._lock:
            t0 = time.perf_counter_ns()
            with self._stage_lock:
                self._drain_at_boundary()
            pushed = self._push(state=False)
            self._running = True
            try:
                if self._live:   # posted just before the launch: the kernel drains them
                    self._stage_pending()
                if pushed:
                    contacts, barrier_ns = self._dev.run_host(steps)
                else:   # re-bound: the state was just uploaded
                    contacts, barrier_ns = self._dev.run(steps)
                    self._dev.download(_lib.RS_STATE)
            finally:
                self._running = False
            self.world.step_index += steps
            self._resolve_applied()
            self.last_contacts = contacts
            if self._small or self._snapshot_readers:
                self.snapshot_buffer.publish(self.world)
                self._snapshot_stale = False
            else:   # large batches: publish on first read (saves a full copy)
                self._snapshot_stale = True
            self._check_core_error()
            wall = time.perf_counter_ns() - t0
        return {"wall_ns": wall, "steps": steps,
                "barrier_wait_ns": barrier_ns, "contacts": contacts}

    def _check_core_error(self):
        step = self._dev.error_step()
        if step >= 0:
            raise FloatingPointError(
                f"non-finite force/torque or degenerate geometry at step {step}")

    def set_params(self, dt=None, iterations=None):
        if dt is not None:
            if dt <= 0.0:
                raise ValueError("dt must be positive")
            self.world.dt = float(dt)
        if iterations is not None:
            if iterations < 1:
                raise ValueError("iterations must be >= 1")
            self.world.solver.iterations = int(iterations)
        self._dev.update_params(self.world.dt, self.world.solver.iterations)

    def read_snapshot(self):
        """The latest published (positions, frames).  Live engines read the
        kernel's per-step snapshot, so a reader sees progress inside a
        running epoch (ph_publish, _core.pyx:1045-1052); otherwise the
        snapshot is published at epoch boundaries."""
        if self._live:
            if not self._live_snaps:   # from the next launch on, one per step
                with self._lock:
                    self._dev.live_snapshots(True)
                    self._live_snaps = True
            seq, step, pos, frames = self._dev.read_snapshot()
            return Snapshot(seq, step, pos, frames)
        with self._lock:
            self._snapshot_readers = True
            if self._snapshot_stale:
                self.snapshot_buffer.publish(self.world)
                self._snapshot_stale = False
        return self.snapshot_buffer.read()

    # -- introspection -----------------------------------------------------

    @property
    def device_world(self):
        return self._dev

    def plan(self):
        return self._dev.plan()

    def close(self):
        if self._dev is not None:
            self._dev.close()
            self._dev = None

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()
