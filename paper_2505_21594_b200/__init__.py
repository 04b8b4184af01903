"""B200-native verify step of arXiv 2505.21594 (speculative edge-cloud decoding
with early exits): hand-written sm_100a kernels behind the C ABI in
include/sv.h (libsv.so), with a thin ctypes binding in `sv`.

The product path never imports `oracle/` and has no CPU fallback.
"""
from . import sv  # noqa: F401

__all__ = ["sv"]
