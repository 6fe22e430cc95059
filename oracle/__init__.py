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
SRC_GRAD = os.path.join(HERE, "tco_grad.c")
LIB = os.path.join(HERE, "libtco.so")

OK, ERR_INVALID, ERR_CORRUPT, ERR_PROTOCOL, ERR_CAPACITY = 0, 1, 5, 6, 8

_lib = None


def build(force: bool = False) -> str:
    """Compile tco.c into oracle/libtco.so (plain -O2, no vector intrinsics)."""
    deps = [SRC, SRC_GRAD, os.path.join(HERE, "tco.h"), os.path.join(HERE, "tco_grad.h")]
    if force or not os.path.exists(LIB) or os.path.getmtime(LIB) < max(os.path.getmtime(d) for d in deps):
        # -ffp-contract=off: every fp32 product and sum rounded as written (tco_grad.h)
        subprocess.check_call(
            ["gcc", "-O2", "-std=c11", "-Wall", "-Wextra", "-ffp-contract=off", "-shared", "-fPIC", "-o", LIB,
             SRC, SRC_GRAD, "-lm"]
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
        L.tco_record_bytes_full.restype = u64
        L.tco_record_bytes_full.argtypes = [u64, u32]
        L.tco_encode.restype = ctypes.c_int
        L.tco_encode.argtypes = [
            vp, vp, vp, vp, ctypes.c_int, u32, u64, ctypes.c_int, ctypes.c_int, u64, u64, vp, u64,
            ctypes.POINTER(u64),
        ]
        L.tco_apply.restype = ctypes.c_int
        L.tco_apply.argtypes = [vp, vp, vp, ctypes.c_int, ctypes.POINTER(u64), vp, u64]
        L.tco_fold.restype = ctypes.c_int
        L.tco_fold.argtypes = [vp, vp, vp, ctypes.c_int, ctypes.POINTER(u64), vp, vp, ctypes.c_int]
        f32 = ctypes.c_float
        L.tco_grad_bound.restype = u64
        L.tco_grad_bound.argtypes = [u64, u64, u64]
        L.tco_grad_compress.restype = ctypes.c_int
        L.tco_grad_compress.argtypes = [vp, u64, u64, u32, u32, u64, u64, vp, u64, ctypes.POINTER(u64)]
        L.tco_grad_decompress.restype = ctypes.c_int
        L.tco_grad_decompress.argtypes = [vp, u64, vp, u64]
        L.tco_f32_to_f16.restype = ctypes.c_uint16
        L.tco_f32_to_f16.argtypes = [f32]
        L.tco_f16_to_f32.restype = f32
        L.tco_f16_to_f32.argtypes = [ctypes.c_uint16]
        L.tco_f32_to_bf16.restype = ctypes.c_uint16
        L.tco_f32_to_bf16.argtypes = [f32]
        L.tco_adam_step.restype = None
        L.tco_adam_step.argtypes = [vp, vp, vp, vp, u64, vp, f32, f32, f32, f32, f32]
        L.tco_adam_replay.restype = ctypes.c_int
        L.tco_adam_replay.argtypes = [vp, vp, vp, vp, u64, vp, vp, ctypes.c_int, f32, f32, f32, vp, vp, vp]
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


def record_bytes(m: int, tile_words: int, word_bytes: int, count: int, index_mode: bool = False,
                 full: bool = False) -> int:
    if full:
        return int(lib().tco_record_bytes_full(m, word_bytes))
    f = lib().tco_record_bytes_index if index_mode else lib().tco_record_bytes
    return int(f(m, tile_words, word_bytes, count))


def worst_case_bytes(sizes, word_bytes, tile_words: int, chunk_words: int, index_mode: bool = False,
                     full: bool = False) -> int:
    tot = 0
    for n, w in zip(sizes, word_bytes):
        off = 0
        while True:
            m = min(n - off, chunk_words)
            tot += record_bytes(m, tile_words, w, m, index_mode, full)
            off += m
            if off >= n:
                break
    return tot


def encode(ref, cur, tile_words=4096, chunk_words=1 << 28, advance_ref=True, version=1,
           ref_version=0, cap=None, index_mode=False, full=False):
    """Encode lists of per-segment numpy arrays (uint16 / uint32).  Returns (rc, bytes).
    Record format: mask (default), index (``index_mode``) or full (``full``: every word).

    ``ref`` arrays are modified in place when ``advance_ref`` is true."""
    n, w = _seg_arrays(ref)
    n2, w2 = _seg_arrays(cur)
    assert (n == n2).all() and (w == w2).all()
    if cap is None:
        cap = worst_case_bytes([int(x) for x in n], [int(x) for x in w], tile_words, chunk_words, index_mode, full)
    out = np.zeros(max(cap, 1), dtype=np.uint8)
    rp = (ctypes.c_void_p * len(ref))(*[_ptr(a) for a in ref])
    cp = (ctypes.c_void_p * len(cur))(*[_ptr(a) for a in cur])
    ob = ctypes.c_uint64(0)
    rc = lib().tco_encode(rp, cp, _ptr(n), _ptr(w), len(ref), tile_words, chunk_words,
                          1 if advance_ref else 0, 2 if full else (1 if index_mode else 0), version, ref_version,
                          _ptr(out), cap,
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


# ---------------------------------------------------------------------------------------------
# The paper's own (lossy) differential: adaptive gradient codec + Adam replay (oracle/tco_grad.h)
SMALL_THRESHOLD = 100_000   # P:395 "100K-element INT8 threshold"
K_DEFAULT = 0.01            # P:395 "k = 0.01"
SAMPLE_SIZE = 4096          # SPEC.md:146 sample of 4096 entries
CHUNK_LIMIT = (1 << 31) - 4096  # the largest multiple of 4096 below 2^31 (INT32 local indices)


def sample_rank(k: float, sample_size: int) -> int:
    """ceil((1-k) * S), clamped to [1, S]: the 1-based rank of the threshold in the sorted sample."""
    import math

    return max(1, min(sample_size, math.ceil((1.0 - k) * sample_size)))


def grad_bound(n: int, small_threshold: int = SMALL_THRESHOLD, chunk_elems: int = CHUNK_LIMIT) -> int:
    return int(lib().tco_grad_bound(n, small_threshold, chunk_elems))


def grad_compress(x: np.ndarray, seed: int, k: float = K_DEFAULT, small_threshold: int = SMALL_THRESHOLD,
                  sample_size: int = SAMPLE_SIZE, chunk_elems: int = CHUNK_LIMIT):
    """Compress an fp32 gradient shard.  Returns (rc, payload bytes)."""
    x = np.ascontiguousarray(x, dtype=np.float32)
    cap = grad_bound(x.size, small_threshold, chunk_elems)
    out = np.zeros(cap, dtype=np.uint8)
    ob = ctypes.c_uint64(0)
    rc = lib().tco_grad_compress(_ptr(x) if x.size else None, x.size, small_threshold, sample_size,
                                 sample_rank(k, sample_size), chunk_elems, seed, _ptr(out), cap, ctypes.byref(ob))
    return rc, out[: ob.value].copy()


def grad_decompress(payload: np.ndarray, n: int):
    """Returns (rc, fp32 array of n)."""
    p = np.ascontiguousarray(payload, dtype=np.uint8)
    out = np.zeros(max(n, 1), dtype=np.float32)
    rc = lib().tco_grad_decompress(_ptr(p), p.size, _ptr(out), n)
    return rc, out[:n]


def f32_to_f16_bits(f: float) -> int:
    return int(lib().tco_f32_to_f16(float(f)))


def f16_bits_to_f32(h: int) -> float:
    return float(lib().tco_f16_to_f32(int(h)))


def f32_to_bf16_bits(f: float) -> int:
    return int(lib().tco_f32_to_bf16(float(f)))


def adam_consts(step: int, lr: float, b1: float, b2: float):
    """step_size = lr / (1 - b1^t), inv_c2s = 1 / sqrt(1 - b2^t) for 1-based step t, in double,
    rounded to fp32 (tco_grad.h)."""
    import math

    return np.float32(lr / (1.0 - b1 ** step)), np.float32(1.0 / math.sqrt(1.0 - b2 ** step))


def adam_step(master, m, v, w16, g, step: int, lr=1e-3, b1=0.9, b2=0.999, eps=1e-8):
    """In place on float32 master/m/v and uint16 (bf16 bits) w16; ``step`` 1-based."""
    ss, ic = adam_consts(step, lr, b1, b2)
    g = np.ascontiguousarray(g, dtype=np.float32)
    lib().tco_adam_step(_ptr(master), _ptr(m), _ptr(v), _ptr(w16), master.size, _ptr(g), b1, b2, eps,
                        float(ss), float(ic))


def adam_replay(master, m, v, w16, payloads, first_step: int, lr=1e-3, b1=0.9, b2=0.999, eps=1e-8) -> int:
    """Sequential replay: payload j is the gradient of step first_step + j.  In place; returns rc."""
    ps = [np.ascontiguousarray(p, dtype=np.uint8) for p in payloads]
    pp = (ctypes.c_void_p * len(ps))(*[_ptr(p) for p in ps])
    pb = np.array([p.size for p in ps], dtype=np.uint64)
    cs = [adam_consts(first_step + j, lr, b1, b2) for j in range(len(ps))]
    ss = np.array([c[0] for c in cs], dtype=np.float32)
    ic = np.array([c[1] for c in cs], dtype=np.float32)
    scratch = np.zeros(max(master.size, 1), dtype=np.float32)
    return int(lib().tco_adam_replay(_ptr(master), _ptr(m), _ptr(v), _ptr(w16), master.size, pp, _ptr(pb), len(ps),
                                     b1, b2, eps, _ptr(ss), _ptr(ic), _ptr(scratch)))
