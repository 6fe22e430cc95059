"""ORACLE for the TierCheck differential checkpoint codec — TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may import this package.  The product package
``paper_2605_17821_b200`` never imports it, and the two share no code: this module
wraps ``oracle/tco.c`` (plain scalar C, see its header for the passages it follows)
through ctypes, marshalling numpy arrays only.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
SRC = os.path.join(HERE, "tco.c")
LIB = os.path.join(HERE, "libtco.so")

OK, ERR_INVALID, ERR_CORRUPT, ERR_PROTOCOL, ERR_CAPACITY = 0, 1, 5, 6, 8

_lib = None


def build(force: bool = False) -> str:
    """Compile tco.c into oracle/libtco.so (plain -O2, no vector intrinsics)."""
    if force or not os.path.exists(LIB) or os.path.getmtime(LIB) < max(
        os.path.getmtime(SRC), os.path.getmtime(os.path.join(HERE, "tco.h"))
    ):
        subprocess.check_call(
            ["gcc", "-O2", "-std=c11", "-Wall", "-Wextra", "-shared", "-fPIC", "-o", LIB, SRC]
        )
    return LIB


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(LIB)
        u64, u32, vp = ctypes.c_uint64, ctypes.c_uint32, ctypes.c_void_p
        L.tco_record_bytes.restype = u64
        L.tco_record_bytes.argtypes = [u64, u32, u32, u64]
        L.tco_record_bytes_index.restype = u64
        L.tco_record_bytes_index.argtypes = [u64, u32, u32, u64]
        L.tco_encode.restype = ctypes.c_int
        L.tco_encode.argtypes = [
            vp, vp, vp, vp, ctypes.c_int, u32, u64, ctypes.c_int, ctypes.c_int, u64, u64, vp, u64,
            ctypes.POINTER(u64),
        ]
        L.tco_apply.restype = ctypes.c_int
        L.tco_apply.argtypes = [vp, vp, vp, ctypes.c_int, ctypes.POINTER(u64), vp, u64]
        L.tco_fold.restype = ctypes.c_int
        L.tco_fold.argtypes = [vp, vp, vp, ctypes.c_int, ctypes.POINTER(u64), vp, vp, ctypes.c_int]
        _lib = L
    return _lib


def _ptr(a: np.ndarray) -> int:
    return a.ctypes.data


def _seg_arrays(segs):
    for a in segs:
        assert a.flags.c_contiguous and a.dtype in (np.uint16, np.uint32), a.dtype
    n = np.array([a.size for a in segs], dtype=np.uint64)
    w = np.array([a.itemsize for a in segs], dtype=np.uint32)
    return n, w


def record_bytes(m: int, tile_words: int, word_bytes: int, count: int, index_mode: bool = False) -> int:
    f = lib().tco_record_bytes_index if index_mode else lib().tco_record_bytes
    return int(f(m, tile_words, word_bytes, count))


def worst_case_bytes(sizes, word_bytes, tile_words: int, chunk_words: int, index_mode: bool = False) -> int:
    tot = 0
    for n, w in zip(sizes, word_bytes):
        off = 0
        while True:
            m = min(n - off, chunk_words)
            tot += record_bytes(m, tile_words, w, m, index_mode)
            off += m
            if off >= n:
                break
    return tot


def encode(ref, cur, tile_words=4096, chunk_words=1 << 28, advance_ref=True, version=1,
           ref_version=0, cap=None, index_mode=False):
    """Encode lists of per-segment numpy arrays (uint16 / uint32).  Returns (rc, bytes).

    ``ref`` arrays are modified in place when ``advance_ref`` is true."""
    n, w = _seg_arrays(ref)
    n2, w2 = _seg_arrays(cur)
    assert (n == n2).all() and (w == w2).all()
    if cap is None:
        cap = worst_case_bytes([int(x) for x in n], [int(x) for x in w], tile_words, chunk_words, index_mode)
    out = np.zeros(max(cap, 1), dtype=np.uint8)
    rp = (ctypes.c_void_p * len(ref))(*[_ptr(a) for a in ref])
    cp = (ctypes.c_void_p * len(cur))(*[_ptr(a) for a in cur])
    ob = ctypes.c_uint64(0)
    rc = lib().tco_encode(rp, cp, _ptr(n), _ptr(w), len(ref), tile_words, chunk_words,
                          1 if advance_ref else 0, 1 if index_mode else 0, version, ref_version, _ptr(out), cap,
                          ctypes.byref(ob))
    return rc, out[: ob.value].copy()


def apply(state, state_version: int, diff: np.ndarray):
    """Apply one shard diff in place.  Returns (rc, new_state_version)."""
    n, w = _seg_arrays(state)
    sp = (ctypes.c_void_p * len(state))(*[_ptr(a) for a in state])
    sv = ctypes.c_uint64(state_version)
    d = np.ascontiguousarray(diff, dtype=np.uint8)
    rc = lib().tco_apply(sp, _ptr(n), _ptr(w), len(state), ctypes.byref(sv),
                         _ptr(d) if d.size else None, d.size)
    return rc, sv.value


def fold(state, state_version: int, diffs):
    """Apply diffs oldest -> newest.  Returns (rc, new_state_version)."""
    n, w = _seg_arrays(state)
    sp = (ctypes.c_void_p * len(state))(*[_ptr(a) for a in state])
    ds = [np.ascontiguousarray(d, dtype=np.uint8) for d in diffs]
    dp = (ctypes.c_void_p * len(ds))(*[_ptr(d) for d in ds])
    db = np.array([d.size for d in ds], dtype=np.uint64)
    sv = ctypes.c_uint64(state_version)
    rc = lib().tco_fold(sp, _ptr(n), _ptr(w), len(state), ctypes.byref(sv), dp, _ptr(db), len(ds))
    return rc, sv.value
