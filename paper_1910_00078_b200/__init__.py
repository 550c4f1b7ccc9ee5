"""primkit-b200: B200-native convolution hot path of MIOpen (arXiv 1910.00078).

The product is ``lib/libprimkit.so`` (C++ host layer + sm_100a CUDA kernels
behind the primkit C ABI, ``include/primkit/primkit.h``). This package holds
its sources (``csrc/``) and a ctypes binding (``primkit``) that mirrors the
reference C API for Python callers and tests.
"""
from . import abi  # noqa: F401

__all__ = ["abi", "primkit"]
