"""B200-native KV-Runahead parallel prompt phase (arXiv 2405.05329).

The product is ``_lib/libkvp_b200.so`` (sm_100a kernels + C++ host runtime, C-ABI in
``include/kvp_b200.h``); :mod:`paper_2405_05329_b200.kvprefill` mirrors the reference's
``kvprefill`` API on top of it.
"""
from . import kvprefill  # noqa: F401
from .kvprefill import *  # noqa: F401,F403

__all__ = [n for n in dir(kvprefill) if not n.startswith("_")]
