"""`step(world)`: one full time step of a World (reference pystep.py:226-237).

The reference's numpy twin of the step is its readable specification and
its engine's fallback backend; this package has no CPU path, so the same
call runs one step of the CUDA kernel.  The World's host arrays stay
authoritative between calls: each call uploads what changed, steps once on
the device and downloads the state, so callers may edit the arrays between
steps exactly as with the reference.  The step is bit-identical to the
reference's compiled core (the numpy twin agrees with that core to 1e-12,
test_engine.py:175-182 of the reference).
"""

from .engine import Engine


def _engine(world):
    eng = getattr(world, "_pystep_engine", None)
    if eng is None or eng.device_world is None:
        eng = Engine(world, backend="serial")
        world._pystep_engine = eng
    return eng


def step(world):
    """One full time-step; returns the number of active contacts (mesh
    contacts plus self-collision pairs).  Raises FloatingPointError on a
    non-finite force or torque, like the reference."""
    eng = _engine(world)
    eng.run_epoch(1)
    return eng.last_contacts


def release(world):
    """Free the device copy `step` keeps for this World."""
    eng = getattr(world, "_pystep_engine", None)
    if eng is not None:
        eng.close()
        world._pystep_engine = None
