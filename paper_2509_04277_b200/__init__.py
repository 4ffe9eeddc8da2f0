"""B200-native CoRdE Cosserat-rod time step (arXiv 2509.04277).

Drop-in for the reference `rodsim` package's rod-construction and
step/simulate API on its hot path: `state.RodParams`, `state.init_rod`,
`world.World`, `engine.Engine.run_epoch`.  The step itself runs as
hand-written sm_100a CUDA behind the C ABI in include/rodsim_b200.h
(`librodsim_b200.so`, built in-tree).  Host-side modules (state, quat,
forces, constraints, world, partition) import without a GPU; the engine
refuses to run without the CUDA library and a device -- there is no CPU
fallback.
"""

import os as _os

__version__ = "0.1.0"

from ._lib import LIB_PATH as _LIB_PATH

# the reference's probe (rodsim/__init__.py:6-11), here: is the CUDA core built
HAVE_COMPILED_CORE = _os.path.exists(_LIB_PATH)
