"""`rodsim._core` on the B200 step: the reference engine's core interface
over the C ABI (include/rodsim_b200.h).

The reference package binds its compiled core as `rodsim._core`
(/root/reference/pkg/src/rodsim/__init__.py:6-11, engine.py:22-28) and
calls exactly these functions:

  make_context(world, starts, ends, snap_pos, snap_frames, snap_seq,
               snap_step)                           engine.py:165-170
  step_serial(ctx) -> contacts                      engine.py:290
  begin_epoch(ctx)                                  engine.py:402
  run_epoch_worker(ctx, block, steps)               engine.py:395
  epoch_results(ctx) -> (contacts, barrier_ns)      engine.py:412
  stage_commands(ctx, ops (n,6) f64) -> [slots]     engine.py:196-197
  applied_step_for(ctx, slot) -> int                engine.py:320
  error_step(ctx) -> int                            engine.py:329
  update_params(ctx, dt, iters)                     engine.py:352-353

(_core.pyx:1058-1184).  `install()` registers this module as
`sys.modules["rodsim._core"]` before the reference package is imported, so
the reference's own `rodsim.engine.Engine` -- both backends, its command
mailbox, ring staging, ticket resolution and error surfacing -- steps on the
GPU.  tests/test_gpu_refcore.py runs it against the reference's golden
checkpoints.

Ownership follows the reference: the World's numpy arrays are the state.
The context binds them by pointer (rs_create); before a launch the control
arrays are uploaded (the library skips unchanged ones) and the state only
when the host copy moved since the last download (a caller edited the World
between epochs); after the launch the state comes back into the World's
arrays and the snapshot buffer is published like ph_publish
(_core.pyx:1045-1052).  The serial path therefore costs one launch and one
state read-back per step, the parallel path one launch of K steps and one
read-back per epoch.

The parallel backend stages commands while an epoch runs
(engine.py:177-198); the context is created live on the parallel path (the
kernel drains the ring at step boundaries, one-CTA / one-cluster plans) so a
mid-epoch command takes effect at a step inside the launch, as in the
reference.  The device mirror is created at first use: `begin_epoch` /
`stage_commands` first -> live, `step_serial` first -> plain.
"""

import sys

import numpy as np

from . import _lib

# the reference core's ring capacity (_core.pyx RING_CAP), mirrored by
# rod_common.h RING_CAP
RING_CAP = 64

_STATE_ATTRS = ("positions", "velocities", "frames", "angular_velocities",
                "contact_active", "contact_normal", "contact_depth", "contact_acc_n",
                "contact_acc_t", "pair_a", "pair_b", "pair_min_dist", "pair_acc")


class CoreContext:
    """The context `make_context` returns (the reference's `CoreContext`,
    _core.pyx:72-182): the World, its device mirror and the snapshot
    buffer it publishes into."""

    def __init__(self, world, starts, ends, snap_pos, snap_frames, snap_seq, snap_step):
        self.world = world
        self.starts = np.asarray(starts, dtype=np.int64)
        self.ends = np.asarray(ends, dtype=np.int64)
        self.snap = (snap_pos, snap_frames, snap_seq, snap_step)
        self.dev = None
        self.shadow = None       # host state at the last download
        self.contacts = 0
        self.barrier_ns = 0

    def device(self, live):
        if self.dev is None:
            self.dev = _lib.DeviceWorld(self.world, live=live)
        return self.dev

    def _state(self):
        w = self.world
        return [getattr(w, a) for a in _STATE_ATTRS if getattr(w, a, None) is not None]

    def sync_in(self):
        dev = self.dev
        dev.upload(_lib.RS_CONTROL)
        cur = self._state()
        if self.shadow is None or any(not np.array_equal(a.view(np.uint8), b.view(np.uint8))
                                      for a, b in zip(cur, self.shadow)):
            dev.upload(_lib.RS_STATE)

    def sync_out(self):
        self.dev.download(_lib.RS_STATE)
        self.shadow = [a.copy() for a in self._state()]
        # ph_publish: seqlock odd while the copy is in flight
        pos, q, seq, step = self.snap
        seq[0] += 1
        pos[:] = self.world.positions
        q[:] = self.world.frames
        step[0] = self.dev.step_counter()
        seq[0] += 1


def core_available():
    return True


def make_context(world, starts, ends, snap_pos, snap_frames, snap_seq, snap_step):
    """_core.pyx:219-403: bind the World (the device mirror is created at
    first use, see the module docstring)."""
    return CoreContext(world, starts, ends, snap_pos, snap_frames, snap_seq, snap_step)


def step_serial(ctx):
    """_core.pyx:1058-1080: one step of every block; returns the contact
    count of the step."""
    dev = ctx.device(live=False)
    ctx.sync_in()
    contacts, _ = dev.run(1)
    ctx.sync_out()
    return int(contacts)


def begin_epoch(ctx):
    """_core.pyx:1092-1099: epoch bookkeeping before the workers start."""
    ctx.device(live=True)
    ctx.sync_in()
    ctx.contacts = 0
    ctx.barrier_ns = 0


def run_epoch_worker(ctx, block, steps):
    """_core.pyx:1101-1130: the reference runs one thread per block; here
    block 0 launches the whole K-step epoch (every block's share) and the
    others have nothing left to do."""
    if int(block) != 0:
        return
    ctx.contacts, ctx.barrier_ns = ctx.dev.run(int(steps))
    ctx.sync_out()


def epoch_results(ctx):
    """_core.pyx:1133-1139: (contacts + pairs after the last step, summed
    barrier wait ns)."""
    return int(ctx.contacts), int(ctx.barrier_ns)


def stage_commands(ctx, ops):
    """_core.pyx:1151-1175: append rows to the ring; their global slots."""
    ops = np.asarray(ops, dtype=np.float64)
    if ops.ndim != 2 or ops.shape[1] != 6:
        raise ValueError("ops must have shape (n, 6)")
    return ctx.device(live=True).stage_commands(ops)


def applied_step_for(ctx, slot):
    """_core.pyx:1178-1184: the core step a staged row was applied at, or -1."""
    return -1 if ctx.dev is None else ctx.dev.applied_step_for(int(slot))


def error_step(ctx):
    """_core.pyx:1142-1144: the last erroring step, or -1."""
    return -1 if ctx.dev is None else ctx.dev.error_step()


def step_counter(ctx):
    """_core.pyx:1146-1148."""
    return int(ctx.world.step_index) if ctx.dev is None else ctx.dev.step_counter()


def update_params(ctx, dt, iters):
    """_core.pyx:1083-1089: dt / iterations between epochs."""
    if dt <= 0.0 or iters < 1:
        raise ValueError("dt must be positive and iters >= 1")
    ctx.world.dt = float(dt)
    if ctx.dev is not None:
        ctx.dev.update_params(float(dt), int(iters))


def install(package="rodsim"):
    """Register this module as `<package>._core` (before the reference
    package is imported) and return it."""
    mod = sys.modules[__name__]
    sys.modules[f"{package}._core"] = mod
    return mod
