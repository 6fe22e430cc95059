"""Seeded synthetic training-state generator (numpy side).

This module holds NONE of the codec's arithmetic: it only produces input words.  It is
the one module both sides may share (tests feed its arrays to the oracle and to the
CUDA path).  The CUDA side implements the *same* counter-based generator as a kernel
(``tc_synth_base`` / ``tc_synth_step`` in include/tc_synth.h) so that full-size bench
inputs can be made on the device; tests/test_gpu_synth.py checks the two agree bit
for bit.  Recipe (after SURVEY.md §8(d)):

    h(x)         = splitmix64(x): z = x + 0x9E3779B97F4A7C15;
                   z = (z ^ z>>30) * 0xBF58476D1CE4E5B9; z = (z ^ z>>27) * 0x94D049BB133111EB;
                   return z ^ z>>31                                      (mod 2^64)
    K(seed,s,t)  = h(seed ^ (s << 56) ^ (t << 32))
    base_s[i]    = low w*8 bits of h(K(seed,s,0) + i)
    changed_t[i] = (h((K(seed,s,t) ^ 0xC0FFEE) + j) >> 11) < p53,  j = i (S1) or i >> 12 (S2),
                   p53 = round(f * 2^53)
    new word     = old ^ ((h((K(seed,s,t) ^ 0xBEEF) + i) & lowmask_w) | 1),
                   lowmask = 0xFFFF (4-byte words) / 0xF (2-byte words)   -> always != old

Per-rank seed = 0x7C0DEC + rank.  State at version t = base with steps 1..t applied.
"""
from __future__ import annotations

import numpy as np

M64 = (1 << 64) - 1
GAMMA = 0x9E3779B97F4A7C15
SEED0 = 0x7C0DEC

S1_IID = 0
S2_RUNS = 1


def _h_scalar(x: int) -> int:
    z = (x + GAMMA) & M64
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & M64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & M64
    return z ^ (z >> 31)


def _h_vec(x: np.ndarray) -> np.ndarray:
    with np.errstate(over="ignore"):
        z = x + np.uint64(GAMMA)
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        return z ^ (z >> np.uint64(31))


def key(seed: int, seg: int, t: int) -> int:
    return _h_scalar((seed ^ (seg << 56) ^ (t << 32)) & M64)


def p53_of(f: float) -> int:
    """Integer change threshold shared by both generators (f in [0, 1])."""
    f = min(max(float(f), 0.0), 1.0)
    return int(round(f * (1 << 53)))


def _dtype(word_bytes: int):
    return np.uint16 if word_bytes == 2 else np.uint32


def base(n: int, word_bytes: int, seed: int, seg: int, start: int = 0) -> np.ndarray:
    """Words [start, start+n) of segment ``seg`` at version 0."""
    k = key(seed, seg, 0)
    with np.errstate(over="ignore"):
        i = np.arange(start, start + n, dtype=np.uint64) + np.uint64(k)
    return _h_vec(i).astype(_dtype(word_bytes))


def change_mask(n: int, word_bytes: int, seed: int, seg: int, t: int, f: float,
                structure: int = S1_IID, start: int = 0) -> np.ndarray:
    k = key(seed, seg, t) ^ 0xC0FFEE
    i = np.arange(start, start + n, dtype=np.uint64)
    j = i if structure == S1_IID else (i >> np.uint64(12))
    with np.errstate(over="ignore"):
        u = _h_vec(j + np.uint64(k))
    return (u >> np.uint64(11)) < np.uint64(p53_of(f))


def step(words: np.ndarray, seed: int, seg: int, t: int, f: float, structure: int = S1_IID,
         start: int = 0) -> np.ndarray:
    """Return version-t words from version-(t-1) ``words`` (which cover [start, start+n))."""
    wb = words.itemsize
    n = words.size
    ch = change_mask(n, wb, seed, seg, t, f, structure, start)
    k = key(seed, seg, t) ^ 0xBEEF
    with np.errstate(over="ignore"):
        r = _h_vec(np.arange(start, start + n, dtype=np.uint64) + np.uint64(k))
    low = np.uint64(0xFFFF if wb == 4 else 0xF)
    delta = ((r & low) | np.uint64(1)).astype(words.dtype)
    out = words.copy()
    out[ch] ^= delta[ch]
    return out


def state(sizes, word_bytes, seed: int, version: int, f: float, structure: int = S1_IID,
          start: int = 0):
    """Per-segment arrays of the state at ``version`` (words [start, start+n) of each)."""
    segs = []
    for s, (n, wb) in enumerate(zip(sizes, word_bytes)):
        a = base(n, wb, seed, s, start)
        for t in range(1, version + 1):
            a = step(a, seed, s, t, f, structure, start)
        segs.append(a)
    return segs


# ---- model shapes (GPT-2 parameter formula) -------------
def gpt_params(h: int, L: int, V: int = 50257, P: int = 1024, inter: int | None = None) -> int:
    """Phi = V*h + P*h + L*(12 h^2 + 13 h) + 2h for inter = 4h.  With a
    different MLP width the per-layer count is 4h^2 + 2*h*inter + 9h + inter."""
    if inter is None or inter == 4 * h:
        return V * h + P * h + L * (12 * h * h + 13 * h) + 2 * h
    return V * h + P * h + L * (4 * h * h + 2 * h * inter + 9 * h + inter) + 2 * h


CONFIGS = {
    # name: (Phi, D, has_bf16_segment)
    "cfg1": (1 << 20, 1, False),
    "cfg2": (gpt_params(1600, 48), 1, True),
    "cfg3": (gpt_params(4096, 32), 8, True),
    "cfg4": (gpt_params(5120, 40), 8, True),
    "cfg5": (gpt_params(5120, 128, inter=20480), 8, True),
}


def shard_layout(cfg: str, rank: int = 0):
    """(sizes, word_bytes) of one rank's shard: bf16 weights + fp32 master/m/v, each
    the rank's contiguous 1/D partition [r*n, (r+1)*n) with the last one short
    (PAPER.md:89 14-Phi accounting)."""
    phi, D, bf16 = CONFIGS[cfg]
    n = -(-phi // D)
    lo = min(rank * n, phi)
    hi = min((rank + 1) * n, phi)
    m = hi - lo
    if bf16:
        return [m, m, m, m], [2, 4, 4, 4]
    return [m, m, m], [4, 4, 4]


def segment_versions(n: int, word_bytes: int, seed: int, seg: int, versions, f: float,
                     structure: int = S1_IID, start: int = 0, block: int = 1 << 23, threads: int | None = None):
    """Words [start, start+n) of segment ``seg`` at each version in ``versions`` (ascending), made
    block by block on a thread pool (numpy releases the GIL): the same words as ``state``, for
    full-size (2^28-word) chunks where one thread would take minutes.  Returns {version: array}."""
    import os
    from concurrent.futures import ThreadPoolExecutor

    versions = sorted(set(int(v) for v in versions))
    out = {v: np.empty(n, dtype=_dtype(word_bytes)) for v in versions}

    def one(b0):
        m = min(block, n - b0)
        a = base(m, word_bytes, seed, seg, start + b0)
        t = 0
        for v in versions:
            while t < v:
                t += 1
                a = step(a, seed, seg, t, f, structure, start + b0)
            out[v][b0:b0 + m] = a

    with ThreadPoolExecutor(threads or os.cpu_count() or 1) as ex:
        list(ex.map(one, range(0, n, block)))
    return out
