"""paper_2412_20796_b200 — B200-native FastCHGNet training step (arXiv 2412.20796).

The hot path lives in libchg.so (CUDA C++ for sm_100a behind the C ABI of
include/chg.h); `chg` is its thin ctypes binding.  There is no CPU fallback.
"""
from . import chg  # noqa: F401
