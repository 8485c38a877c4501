"""B200-native inflight-refactor KV transition (FlexPipe hot path).

The product is the CUDA library ``_lib/libkvx.so`` behind the C-ABI of
``include/kvx.h``; ``kvx`` is its ctypes face.  Import ``kvx`` lazily so that
building (``build``) and the pure-input helpers (``workload``) work without it.
"""
__all__ = ["build", "kvx", "workload"]
