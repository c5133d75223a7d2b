"""B200-native hot path of hierarchical multicontinuum homogenization (arXiv 2503.01276).

The compute path is the C-ABI library ``lib/libmch.so`` (hand-written sm_100a CUDA kernels,
see ``csrc/``); this package is argument marshalling over it.  It never imports ``oracle``
and has no CPU fallback: importing it without the built library raises.
"""
from .api import Homogenizer, mch_create, mch_destroy, mch_effective_coeffs, mch_solve_level

__all__ = ["Homogenizer", "mch_create", "mch_solve_level", "mch_effective_coeffs", "mch_destroy"]
