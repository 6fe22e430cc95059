"""paper_2605_17821_b200 — TierCheck's differential checkpoint codec, B200-native.

The hot path (BASELINE.json north_star) lives in libtc.so (csrc/, C ABI in include/tc.h);
``tc`` is its thin ctypes binding and ``checkpoint`` the save/retrieve/reclaim lifecycle
helper built on it.  Importing ``tc`` fails loudly when libtc.so is missing: there is no
CPU fallback anywhere in this package.
"""
__all__ = ["tc"]
