"""B200-native anisotropic product quantization hot path (arXiv 1908.10396).

The product is the C ABI library `libanisoq_b200.so` (hand-written sm_100a
kernels, csrc/) behind the reference's own API: `anisoq` (Python mirror of
/root/reference/proj/include/anisoq) and include/anisoq/*.hpp (C++ drop-in).
"""
from . import build  # noqa: F401

__all__ = ["anisoq", "build"]
