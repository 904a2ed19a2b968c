"""B200-native expert-parallel MoE layer (hot path of arxiv 2605.05049, "Piper").

The product is ``libmoe.so`` (C ABI in ``include/moe.h``, sm_100a kernels in
``csrc/``).  ``_lib`` is the ctypes binding (same names as the C entry points);
``layer.MoELayer`` composes one layer's forward and backward from those calls.
Importing this package loads libmoe.so and fails loudly if it is missing.
"""
from . import _lib  # noqa: F401  (loads libmoe.so)
from ._lib import *  # noqa: F401,F403
from .layer import LayerDims, MoELayer  # noqa: F401
