"""`pystep.step(world)` (reference pystep.py:226-237) on the GPU: single
steps with host-side edits between them equal the oracle bit for bit, the
contact count is returned, and a non-finite force raises like the
reference."""

import numpy as np
import pytest

from oracle.oracle import OracleStepper
from paper_2509_04277_b200 import pystep
from paper_2509_04277_b200 import workloads as wl

pytestmark = pytest.mark.gpu
STATE = ("positions", "velocities", "frames", "angular_velocities")


def _bits_equal(a, b):
    return all(np.array_equal(getattr(a, k).view(np.int64), getattr(b, k).view(np.int64))
               for k in STATE)


def test_single_steps_with_host_edits_bitwise():
    g, r = wl.cantilever(), wl.cantilever()
    ref = OracleStepper(r)
    for i in range(30):
        if i == 10:   # the host arrays stay authoritative between steps
            for w in (g, r):
                w.velocities[20] += (0.0, 0.5, 0.0)
                w.driver_velocity[0] = (0.0, 0.0, 0.01)
        assert pystep.step(g) == 0
        ref.run(1)
    assert g.step_index == r.step_index == 30
    assert _bits_equal(g, r)
    pystep.release(g)


def test_contacts_returned():
    g = wl.floor_drop()
    counts = [pystep.step(g) for _ in range(400)]
    assert max(counts) > 0
    pystep.release(g)


def test_non_finite_raises():
    g = wl.cantilever()
    pystep.step(g)
    g.positions[5] = np.nan
    with pytest.raises(FloatingPointError, match="non-finite"):
        pystep.step(g)
    pystep.release(g)
