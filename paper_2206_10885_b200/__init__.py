"""paper_2206_10885_b200 -- B200-native (sm_100a) KiloNeuS render hot path.

A drop-in for the render / sphere-trace / batched multi-network forward path of the reference
``kilofield`` package (grid.py, cameras.py, surface.py, pathtrace.py), running on hand-written
CUDA kernels behind the C-ABI in ``include/knf_b200.h``.  No CPU fallback.
"""

from . import _native  # noqa: F401
from . import cameras, grid, hooks, modelio, nn, surface  # noqa: F401
from . import pathtrace  # noqa: F401

__version__ = "0.1.0"
