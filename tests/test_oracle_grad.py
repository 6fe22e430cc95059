"""Pins of the gradient-codec / Adam-replay oracle (oracle/tco_grad.c, NEXT row 3) against what
the paper, SPEC.md and the mathematics fix: library conversions (numpy float16, torch bfloat16),
the SPEC.md:119-135 examples, the quantization error bound, the exact keeping predicate, chunk
rebasing, closed-form sizes, and an fp64 Adam reference."""
import math

import numpy as np
import pytest

import oracle

RNG = np.random.default_rng(11)


def hdr(p):
    return {"variant": int(p[4]), "chunks": int(np.frombuffer(p[8:12].tobytes(), np.uint32)[0]),
            "s": float(np.frombuffer(p[12:16].tobytes(), np.float32)[0]),
            "n": int(np.frombuffer(p[16:24].tobytes(), np.uint64)[0]),
            "kept": int(np.frombuffer(p[24:32].tobytes(), np.uint64)[0]),
            "total": int(np.frombuffer(p[48:56].tobytes(), np.uint64)[0])}


def pad16(x):
    return (x + 15) // 16 * 16


# ---------------------------------------------------------------- conversions ----------
def test_f16_matches_numpy():
    vals = np.concatenate([
        RNG.standard_normal(3000).astype(np.float32) * 10.0 ** RNG.integers(-9, 6, 3000),
        np.array([0.0, -0.0, 65504.0, 65519.0, 65520.0, 1e6, -1e6, 2 ** -24, 2 ** -25, 2 ** -25 * 1.0001,
                  2 ** -14, 2 ** -14 * (1 - 2 ** -11), 1.0 + 2 ** -11, 1.0 + 3 * 2 ** -11, np.inf, -np.inf],
                 dtype=np.float32)])
    for v in vals:
        with np.errstate(over="ignore"):  # overflow to infinity is the expected conversion
            want = int(np.array([v], np.float32).astype(np.float16).view(np.uint16)[0])
        assert oracle.f32_to_f16_bits(v) == want, v
        assert oracle.f16_bits_to_f32(want) == float(np.array([want], np.uint16).view(np.float16).astype(np.float32)[0])


def test_bf16_matches_torch():
    torch = pytest.importorskip("torch")
    vals = (RNG.standard_normal(5000) * 10.0 ** RNG.integers(-30, 30, 5000)).astype(np.float32)
    vals[:4] = [0.0, -0.0, 1.0 + 2 ** -8, 1.0 + 3 * 2 ** -8]  # halfway cases: to even
    want = torch.from_numpy(vals).to(torch.bfloat16).view(torch.int16).numpy().view(np.uint16)
    got = np.array([oracle.f32_to_bf16_bits(v) for v in vals], np.uint16)
    assert np.array_equal(got, want)


# ------------------------------------------------------------------- INT8 dense ----------
def test_int8_constant_tensor_spec_example():
    """length 10 constant c > 0 -> q all 127, scale = c/127."""
    rc, p = oracle.grad_compress(np.full(10, 2.5, np.float32), seed=1)
    h = hdr(p)
    assert rc == 0 and h["variant"] == 1 and h["total"] == p.size == 64 + 16
    assert (p[64:74].view(np.int8) == 127).all()
    assert h["s"] == np.float32(2.5) / np.float32(127)


def test_int8_all_zero_and_error_bound():
    rc, p = oracle.grad_compress(np.zeros(100, np.float32), seed=1)
    assert rc == 0 and hdr(p)["s"] == 1.0 and not p[64:164].any()
    x = (RNG.standard_normal(50_000) * 3).astype(np.float32)
    rc, p = oracle.grad_compress(x, seed=2)
    s = hdr(p)["s"]
    assert s == np.float32(np.abs(x).max()) / np.float32(127)
    rc, y = oracle.grad_decompress(p, x.size)
    assert rc == 0 and np.all(np.abs(y.astype(np.float64) - x) <= s / 2 * (1 + 1e-6))  # SPEC.md:106 bound
    q = p[64:64 + x.size].view(np.int8)
    assert np.array_equal(y, np.float32(s) * q.astype(np.float32))


# -------------------------------------------------------------------- sparse ----------
def test_sparse_all_zero_keeps_nothing():
    rc, p = oracle.grad_compress(np.zeros(200_000, np.float32), seed=3)
    h = hdr(p)
    assert rc == 0 and h["variant"] == 2 and h["kept"] == 0
    rc, y = oracle.grad_decompress(p, 200_000)
    assert rc == 0 and not y.any()


def test_sparse_normal_band_and_exact_keeping():
    """10^6 normal, k = 0.01: kept in [0.5kn, 2kn]; the kept set is exactly the
    entries at or above the threshold (so every kept magnitude >= every discarded one)."""
    n = 1_000_000
    x = RNG.standard_normal(n).astype(np.float32)
    rc, p = oracle.grad_compress(x, seed=7)
    h = hdr(p)
    assert rc == 0 and 0.5 * 0.01 * n <= h["kept"] <= 2 * 0.01 * n
    thr = np.float32(h["s"])
    keep = (x != 0) & (np.abs(x) >= thr)
    assert keep.sum() == h["kept"]
    assert np.abs(x[keep]).min() >= np.abs(x[~keep]).max()
    # the threshold is the (1-k)-quantile estimate: within a few sampling sigmas of the true one
    true_q = np.quantile(np.abs(x), 0.99)
    assert abs(thr - true_q) < 0.1
    rc, y = oracle.grad_decompress(p, n)
    assert rc == 0
    assert np.array_equal(np.nonzero(y)[0], np.nonzero(keep)[0])
    assert np.array_equal(y[keep], x[keep].astype(np.float16).astype(np.float32))
    # closed-form size; <= 2 % of the dense fp32 bytes
    assert p.size == 64 + 16 + pad16(2 * h["kept"]) + pad16(4 * h["kept"]) and p.size <= 0.02 * 4 * n


def test_sparse_ties_kept_and_monotone_in_k():
    x = RNG.integers(-3, 4, 300_000).astype(np.float32)  # few distinct magnitudes: many ties
    counts = []
    for k in (0.001, 0.01, 0.1, 0.5):
        rc, p = oracle.grad_compress(x, seed=5, k=k)
        h = hdr(p)
        keep = (x != 0) & (np.abs(x) >= np.float32(h["s"]))
        assert rc == 0 and keep.sum() == h["kept"]  # ties at the threshold are kept
        counts.append(h["kept"])
    assert counts == sorted(counts)  # SPEC.md:141 monotone threshold


def test_chunk_rebasing_equals_single_chunk():
    """chunked payloads decompress to the single-chunk result."""
    x = (RNG.standard_normal(6 * 4096 * 5 + 77) * 2).astype(np.float32)
    rc1, p1 = oracle.grad_compress(x, seed=9, k=0.05)
    rc2, p2 = oracle.grad_compress(x, seed=9, k=0.05, chunk_elems=4096 * 5)
    assert rc1 == rc2 == 0 and hdr(p2)["chunks"] == 7 and p1.size != p2.size
    r1, y1 = oracle.grad_decompress(p1, x.size)
    r2, y2 = oracle.grad_decompress(p2, x.size)
    assert r1 == r2 == 0 and np.array_equal(y1, y2)


def test_deterministic_and_tamper():
    x = RNG.standard_normal(150_000).astype(np.float32)
    _, a = oracle.grad_compress(x, seed=4)
    _, b = oracle.grad_compress(x, seed=4)
    assert np.array_equal(a, b)
    h = hdr(a)
    ioff = 64 + 16 + pad16(2 * h["kept"])
    bad = a.copy()
    bad[ioff: ioff + 4] = np.frombuffer(np.int32(150_000).tobytes(), np.uint8)  # index past the chunk
    assert oracle.grad_decompress(bad, x.size)[0] == oracle.ERR_CORRUPT
    bad = a.copy()
    bad[ioff: ioff + 8] = bad[[ioff + 4, ioff + 5, ioff + 6, ioff + 7, ioff, ioff + 1, ioff + 2, ioff + 3]]
    assert oracle.grad_decompress(bad, x.size)[0] == oracle.ERR_CORRUPT  # not increasing
    assert oracle.grad_decompress(a[:-16], x.size)[0] == oracle.ERR_CORRUPT


# ---------------------------------------------------------------------- Adam ----------
def adam_f64(master, m, v, g, t, lr=1e-3, b1=0.9, b2=0.999, eps=1e-8):
    m = b1 * m + (1 - b1) * g
    v = b2 * v + (1 - b2) * g * g
    mh, vh = m / (1 - b1 ** t), v / (1 - b2 ** t)
    return master - lr * mh / (np.sqrt(vh) + eps), m, v


def test_adam_hand_example():
    """w = 1, g = 0.1, lr = 0.1: the first bias-corrected step moves w by ~lr."""
    w = np.ones(1, np.float32)
    m, v, w16 = np.zeros(1, np.float32), np.zeros(1, np.float32), np.zeros(1, np.uint16)
    oracle.adam_step(w, m, v, w16, np.array([0.1], np.float32), 1, lr=0.1)
    assert abs(w[0] - 0.9) < 1e-5 and m[0] == np.float32(0.1) * np.float32(1 - np.float32(0.9))
    w = np.ones(4, np.float32)
    z = np.zeros(4, np.float32)
    oracle.adam_step(w, z.copy(), z.copy(), np.zeros(4, np.uint16), z, 1)
    assert (w == 1).all()  # zero gradient, zero moments: weights unchanged


def test_adam_matches_fp64_reference_over_steps():
    n = 4096
    master = RNG.standard_normal(n).astype(np.float32)
    m = (RNG.standard_normal(n) * 1e-2).astype(np.float32)
    v = (np.abs(RNG.standard_normal(n)) * 1e-4).astype(np.float32)
    w16 = np.zeros(n, np.uint16)
    M, Mm, Mv = master.astype(np.float64), m.astype(np.float64), v.astype(np.float64)
    for t in range(1, 6):
        g = (RNG.standard_normal(n) * 1e-2).astype(np.float32)
        oracle.adam_step(master, m, v, w16, g, t)
        M, Mm, Mv = adam_f64(M, Mm, Mv, g.astype(np.float64), t)
    # fp32 rounding of (1 - beta) and of every product: absolute error far below any formula slip
    assert np.allclose(m, Mm, rtol=1e-5, atol=2e-8) and np.allclose(v, Mv, rtol=1e-4, atol=2e-10)
    assert np.allclose(master, M, rtol=1e-6, atol=1e-6)
    torch = pytest.importorskip("torch")
    assert np.array_equal(w16, torch.from_numpy(master).to(torch.bfloat16).view(torch.int16).numpy().view(np.uint16))


def test_replay_is_the_sequential_application():
    n = 50_000  # INT8 payloads
    st0 = [RNG.standard_normal(n).astype(np.float32), np.zeros(n, np.float32), np.zeros(n, np.float32)]
    grads = [(RNG.standard_normal(n) * 1e-2).astype(np.float32) for _ in range(5)]
    pays = [oracle.grad_compress(g, seed=j)[1] for j, g in enumerate(grads)]
    a = [x.copy() for x in st0] + [np.zeros(n, np.uint16)]
    assert oracle.adam_replay(a[0], a[1], a[2], a[3], pays, first_step=3) == 0
    b = [x.copy() for x in st0] + [np.zeros(n, np.uint16)]
    for j, p in enumerate(pays):
        rc, g = oracle.grad_decompress(p, n)
        oracle.adam_step(b[0], b[1], b[2], b[3], g, 3 + j)
    assert all(np.array_equal(x, y) for x, y in zip(a, b))
    M = st0[0].astype(np.float64)
    Mm = np.zeros(n)
    Mv = np.zeros(n)
    for j, p in enumerate(pays):  # fp64 Adam on the decoded gradients: the same trajectory
        g = oracle.grad_decompress(p, n)[1].astype(np.float64)
        M, Mm, Mv = adam_f64(M, Mm, Mv, g, 3 + j)
    assert np.allclose(a[0], M, rtol=1e-6, atol=1e-6)
    assert math.isfinite(float(a[0].sum()))


def test_adam_eps_placement_pinned():
    """Where ε sits (DESIGN G8: denom = √v̂ + ε, ε added after the bias correction, outside the
    square root).  With v = 0 and m ≠ 0 the step is exactly lr·m̂/ε; with √v̂ comparable to ε the
    two terms are summed.  ε inside the root (√(v̂+ε)) or ahead of the correction ((√v + ε)/√(1−β2ᵗ))
    changes these steps by orders of magnitude."""
    lr, b1, b2, eps = 1e-3, 0.9, 0.999, 1e-8
    m0 = np.array([1e-9, -3e-9, 2e-10, 5e-9, 1e-9, -1e-9], np.float32)
    # v0 = 0 (pure ε), then v̂ = ε², 4ε², ε²/4 at step t (√v̂ = ε, 2ε, ε/2)
    for t in (1, 2, 7):
        c2 = 1 - b2 ** t
        vh_target = np.array([0, 0, 0, eps ** 2, 4 * eps ** 2, 0.25 * eps ** 2])
        v0 = (vh_target * c2 / b2).astype(np.float32)  # g = 0: v = β2·v0
        master = np.zeros(6, np.float32)  # the update itself, at full fp32 relative precision
        m, v = m0.copy(), v0.copy()
        oracle.adam_step(master, m, v, np.zeros(6, np.uint16), np.zeros(6, np.float32), t, lr=lr, b1=b1, b2=b2,
                         eps=eps)
        mh = b1 * m0.astype(np.float64) / (1 - b1 ** t)
        vh = b2 * v0.astype(np.float64) / c2
        expect = -lr * mh / (np.sqrt(vh) + eps)
        assert np.allclose(master, expect, rtol=1e-5, atol=0), (t, master, expect)
        wrong_in_root = -lr * mh / np.sqrt(vh + eps)
        wrong_before_corr = -lr * mh / ((np.sqrt(b2 * v0.astype(np.float64)) + eps) / np.sqrt(c2))
        assert not np.allclose(master, wrong_in_root, rtol=1e-2)
        assert not np.allclose(master, wrong_before_corr, rtol=1e-2)
