"""paper_2411_10958_b200 -- B200-native (sm_100a) SageAttention2 (arXiv 2411.10958) forward pass.

The product is libsage2.so (csrc/, C ABI in include/sage2.h); ``sage2`` is its thin ctypes
binding and ``synth`` the seeded input generators.  There is no CPU fallback.
"""
from . import synth  # noqa: F401
from .sage2 import Sage2Error, attn, attn_host  # noqa: F401
