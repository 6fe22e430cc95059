"""GPU parity of the paper's lossy differential (NEXT row 3, include/tc_grad.h) against the
oracle (oracle/tco_grad.c): compressed payload bytes, decompressed values, the Adam step and the
fused multi-step replay — all bit-exact — plus the capacity and corruption paths."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a GPU", allow_module_level=True)

import oracle  # noqa: E402
from paper_2605_17821_b200 import tc  # noqa: E402

RNG = np.random.default_rng(23)


@pytest.fixture(scope="module")
def tco_lossless():
    return oracle


@pytest.fixture(scope="module")
def ctx():
    c = tc.Ctx(0)
    yield c
    c.close()


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def gpu_compress(ctx, x, seed, **opts):
    cap = tc.grad_bound(x.size, **opts)
    out = torch.full((cap + 64,), 0xAB, dtype=torch.uint8, device="cuda")
    ob = torch.zeros(1, dtype=torch.int64, device="cuda")
    tc.grad_compress(ctx, dev(x), seed, out[:cap], ob, **opts)
    ctx.check()
    n = int(ob.item())
    return out[:n].cpu().numpy(), out


def grad_of(kind, n):
    if kind == "normal":
        return (RNG.standard_normal(n) * 1e-2).astype(np.float32)
    if kind == "zeros_mixed":
        x = RNG.standard_normal(n).astype(np.float32)
        x[RNG.random(n) < 0.5] = 0.0
        return x
    if kind == "ties":
        return RNG.integers(-3, 4, n).astype(np.float32)
    if kind == "zero":
        return np.zeros(n, np.float32)
    if kind == "wide":
        return (RNG.standard_normal(n) * 10.0 ** RNG.integers(-20, 20, n)).astype(np.float32)
    raise ValueError(kind)


CASES = [
    (10, "normal", {}), (4097, "wide", {}), (99_999, "normal", {}),        # INT8 dense
    (100_000, "normal", {}), (100_001, "ties", {}), (1_000_003, "normal", {}),
    (300_000, "zeros_mixed", {"k": 0.1}), (250_000, "zero", {}), (200_000, "wide", {"k": 0.3}),
    (123_457, "normal", {"chunk_elems": 4096 * 3}),                       # chunk rebasing
    (70_000, "normal", {"small_threshold": 1000, "k": 0.6}),              # dense blocks (spill overflow)
]


@pytest.mark.parametrize("n,kind,opts", CASES)
def test_compress_decompress_match_oracle(ctx, n, kind, opts):
    x = grad_of(kind, n)
    rc, exp = oracle.grad_compress(x, seed=n, **opts)
    assert rc == 0
    got, full = gpu_compress(ctx, x, n, **opts)
    assert got.size == exp.size and np.array_equal(got, exp), "payload bytes differ from the oracle"
    rc, y = oracle.grad_decompress(exp, n)
    out = torch.full((n,), float("nan"), dtype=torch.float32, device="cuda")
    tc.grad_decompress(ctx, full, got.size, out)
    ctx.check()
    assert np.array_equal(out.cpu().numpy().view(np.uint32), y.view(np.uint32))


def test_compress_capacity_on_device(ctx):
    x = grad_of("normal", 400_000)
    rc, exp = oracle.grad_compress(x, seed=1)
    out = torch.full((exp.size,), 0xAB, dtype=torch.uint8, device="cuda")
    ob = torch.zeros(1, dtype=torch.int64, device="cuda")
    small = exp.size - 32
    tc.grad_compress(ctx, dev(x), 1, out[:small], ob)
    assert ctx.check_status() == tc.ERR_CAPACITY and int(ob.item()) == exp.size
    assert (out[small:].cpu().numpy() == 0xAB).all()


def test_decompress_tamper_corrupt(ctx):
    x = grad_of("normal", 150_000)
    rc, p = oracle.grad_compress(x, seed=4)
    kept = int(np.frombuffer(p[24:32].tobytes(), np.uint64)[0])
    ioff = 64 + 16 + (2 * kept + 15) // 16 * 16
    out = torch.zeros(150_000, dtype=torch.float32, device="cuda")
    for how in ("range", "order", "truncate", "magic"):
        bad = p.copy()
        if how == "range":
            bad[ioff: ioff + 4] = np.frombuffer(np.int32(150_000).tobytes(), np.uint8)
        elif how == "order":
            bad[ioff: ioff + 8] = bad[[ioff + 4, ioff + 5, ioff + 6, ioff + 7, ioff, ioff + 1, ioff + 2, ioff + 3]]
        elif how == "truncate":
            bad = bad[:-16]
        else:
            bad[0] = ord("X")
        assert oracle.grad_decompress(bad, 150_000)[0] == oracle.ERR_CORRUPT
        tc.grad_decompress(ctx, dev(np.concatenate([bad, np.zeros(16, np.uint8)])), bad.size, out)
        assert ctx.check_status() == tc.ERR_CORRUPT, how


def state(n, seed):
    r = np.random.default_rng(seed)
    return [r.standard_normal(n).astype(np.float32), (r.standard_normal(n) * 1e-3).astype(np.float32),
            (np.abs(r.standard_normal(n)) * 1e-6).astype(np.float32), np.zeros(n, np.uint16)]


def to_gpu_state(st):
    return [dev(st[0]), dev(st[1]), dev(st[2]), dev(st[3].view(np.int16))]


def same_state(g, o):
    return all(np.array_equal(a.cpu().numpy().view(np.uint32 if a.dtype == torch.float32 else np.uint16),
                              b.view(np.uint32 if b.dtype == np.float32 else np.uint16)) for a, b in zip(g, o))


@pytest.mark.parametrize("hp", [{}, {"lr": 0.1}, {"lr": 3e-4, "beta1": 0.8, "beta2": 0.99, "eps": 1e-6}])
def test_adam_step_matches_oracle(ctx, hp):
    n = 70_001
    st = state(n, 5)
    g = grad_of("wide", n)
    g[:100] = 0.0
    gs = to_gpu_state(st)
    for t in (1, 2, 1000):
        tc.adam_step(ctx, *gs, dev(g), t, **hp)
        oracle.adam_step(st[0], st[1], st[2], st[3], g, t, **{"lr": 1e-3, "b1": 0.9, "b2": 0.999, "eps": 1e-8,
                                                               **{{"beta1": "b1", "beta2": "b2"}.get(k, k): v
                                                                  for k, v in hp.items()}})
    ctx.check()
    assert same_state(gs, st)


@pytest.mark.parametrize("N", [1, 2, 5, 10])
@pytest.mark.parametrize("n,kind,opts", [(50_000, "normal", {}), (300_001, "normal", {}),
                                          (200_000, "zeros_mixed", {"k": 0.05, "chunk_elems": 4096 * 7}),
                                          # ~1230 entries per 4096-element tile and step: past the
                                          # replay's shared stage (2048 per tile) from N = 3 on
                                          (150_001, "normal", {"k": 0.3, "small_threshold": 1000})])
def test_fused_replay_matches_sequential_oracle(ctx, N, n, kind, opts):
    """fused replay of N payloads == sequential decompress + adam_step, bit-exact."""
    st = state(n, N)
    pays = [oracle.grad_compress(grad_of(kind, n), seed=100 + j, **opts)[1] for j in range(N)]
    gs = to_gpu_state(st)
    assert oracle.adam_replay(st[0], st[1], st[2], st[3], pays, first_step=7) == 0
    dp = [dev(np.concatenate([p, np.zeros(16, np.uint8)])) for p in pays]
    scratch = torch.empty(n, dtype=torch.float32, device="cuda")
    tc.adam_replay(ctx, *gs, dp, [p.size for p in pays], 7, scratch)
    ctx.check()
    assert same_state(gs, st)


def test_replay_corrupt_payload(ctx):
    n = 120_000
    st = state(n, 1)
    pays = [oracle.grad_compress(grad_of("normal", n), seed=j)[1] for j in range(3)]
    bad = pays[1].copy()
    bad[0] = ord("X")
    gs = to_gpu_state(st)
    dp = [dev(np.concatenate([p, np.zeros(16, np.uint8)])) for p in (pays[0], bad, pays[2])]
    tc.adam_replay(ctx, *gs, dp, [pays[0].size, bad.size, pays[2].size], 1, torch.empty(n, device="cuda"))
    assert ctx.check_status() == tc.ERR_CORRUPT


@pytest.mark.parametrize("index_mode", [False, True, "full"])
@pytest.mark.parametrize("n,T,C,zero_frac", [(0, 4096, 1 << 28, 0.0), (1, 4096, 1 << 28, 0.0), (1000, 4096, 1 << 28, 0.5),
                                             (70_001, 256, 8192, 0.9), (300_000, 4096, 1 << 28, 0.99),
                                             # ~20 % changed in the moment segments' second half: sparse
                                             # blocks with many changes per lane (the word-by-word gather)
                                             (200_000, 4096, 1 << 28, 0.8),
                                             # chunks of 96 words: a chunk's mask words start at any
                                             # 4-byte offset (no 16-byte mask loads there)
                                             (50_003, 32, 96, 0.9),
                                             # many chunks: record starts chained across the warps
                                             (3_000_000, 4096, 1 << 20, 0.99)])
def test_adam_step_encode_matches_oracle(ctx, tco_lossless, n, T, C, zero_frac, index_mode):
    """NEXT row 2: the fused Adam step + lossless diff == oracle adam_step, then oracle encode of
    (state before -> state after), byte for byte; the state equals the oracle's."""
    r = np.random.default_rng(n)
    st = [r.standard_normal(n).astype(np.float32), np.zeros(n, np.float32), np.zeros(n, np.float32),
          np.zeros(n, np.uint16)]
    st[1][: n // 2] = (r.standard_normal(n // 2) * 1e-3).astype(np.float32)
    st[2][: n // 2] = (np.abs(r.standard_normal(n // 2)) * 1e-6).astype(np.float32)
    g = (r.standard_normal(n) * 1e-2).astype(np.float32)
    g[r.random(n) < zero_frac] = 0.0
    before = [a.copy() for a in st]
    oracle.adam_step(st[0], st[1], st[2], st[3], g, 5)
    ref = [before[3], before[0].view(np.uint32), before[1].view(np.uint32), before[2].view(np.uint32)]
    cur = [st[3], st[0].view(np.uint32), st[1].view(np.uint32), st[2].view(np.uint32)]
    full = index_mode == "full"  # full records: written by the Adam pass itself (adam_full_kernel)
    index_mode = index_mode is True
    rc, exp = tco_lossless.encode([a.copy() for a in ref], cur, tile_words=T, chunk_words=C, advance_ref=False,
                                  version=5, ref_version=4, index_mode=index_mode, full=full)
    assert rc == 0
    gs = to_gpu_state(before)
    cap = tc.diff_bound([n] * 4, [2, 4, 4, 4], T, C, index_mode, full=full)
    out = torch.full((cap,), 0xAB, dtype=torch.uint8, device="cuda")
    ob = torch.zeros(1, dtype=torch.int64, device="cuda")
    tc.adam_step_encode(ctx, *gs, dev(g), 5, out, ob, T, C, index_mode, full=full)
    ctx.check()
    nb = int(ob.item())
    assert nb == exp.size and np.array_equal(out[:nb].cpu().numpy(), exp)
    assert same_state(gs, st)


def _idx_offset(p):
    """Byte offset of the INT32 index array of a sparse payload (oracle/tco_grad.h layout)."""
    h = p[:64]
    chunks = int(h[8:12].view("<u4")[0])
    kept = int(h[24:32].view("<u8")[0])
    return 64 + 16 * chunks + (2 * kept + 15) // 16 * 16, kept


@pytest.mark.parametrize("k,N", [(0.01, 3), (0.3, 4)])
@pytest.mark.parametrize("tamper", ["order", "range"])
def test_replay_corrupt_indices(ctx, k, N, tamper):
    """An index out of order within a tile, or pointing past the tile's chunk span, is CORRUPT in
    the fused replay (both the staged path and, at k = 0.3, the path past the stage)."""
    n = 150_001
    st = state(n, N)
    opts = {"k": k, "small_threshold": 1000}
    pays = [oracle.grad_compress(grad_of("normal", n), seed=40 + j, **opts)[1] for j in range(N)]
    bad = pays[0].copy()
    off, kept = _idx_offset(bad)
    idx = bad[off: off + 4 * kept].view("<i4")
    j = kept // 2
    if tamper == "order":
        idx[j], idx[j + 1] = idx[j + 1], idx[j]
    else:
        idx[j] = idx[j] + 5 * 4096
    gs = to_gpu_state(st)
    dp = [dev(np.concatenate([p, np.zeros(16, np.uint8)])) for p in [bad] + pays[1:]]
    tc.adam_replay(ctx, *gs, dp, [p.size for p in [bad] + pays[1:]], 1, torch.empty(n, device="cuda"))
    assert ctx.check_status() == tc.ERR_CORRUPT


def _wide_floats(r, n, lo_exp, hi_exp, zeros=0.05, denormals=0.05, signed=True):
    """fp32 values with exponents uniform in [lo_exp, hi_exp], plus exact zeros and denormals."""
    assert -126 <= lo_exp <= hi_exp <= 127  # normal exponents (no inf / NaN)
    mant = r.integers(0, 1 << 23, n, dtype=np.uint32)
    ex = r.integers(lo_exp + 127, hi_exp + 128, n).astype(np.uint32)
    bits = (ex << 23) | mant
    u = r.random(n)
    bits[u < zeros] = 0
    den = (u >= zeros) & (u < zeros + denormals)
    bits[den] = mant[den] | 1
    if signed:
        bits |= (r.random(n) < 0.5).astype(np.uint32) << 31
    return bits.view(np.float32)


@pytest.mark.parametrize("variant", ["int8", "sparse"])
def test_fused_replay_wide_state(ctx, variant):
    """The replay's branch-free Adam update (fast sqrt / quotient sequences, ranges checked per
    element, the rest redone with the intrinsics) against the oracle over m, v spanning the whole
    fp32 range — tiny, huge, denormal and zero moments — bit for bit."""
    n = 60_000 if variant == "int8" else 300_001
    r = np.random.default_rng(77)
    st = [r.standard_normal(n).astype(np.float32) * 10,
          _wide_floats(r, n, -126, 60),
          _wide_floats(r, n, -126, 120, signed=False),
          np.zeros(n, np.uint16)]
    N = 4
    # FP16-representable gradients (a "wide" one would hold infinities, and NaN payload bits are
    # not comparable across the two implementations)
    pays = [oracle.grad_compress(grad_of("normal", n) * np.float32(10.0 ** (j - 2)), seed=200 + j)[1]
            for j in range(N)]
    gs = to_gpu_state(st)
    for hp in ({}, {"eps": 1e-30, "beta2": 0.99999}):
        o = {"lr": 1e-3, "b1": 0.9, "b2": 0.999, "eps": 1e-8, **{"b2" if k == "beta2" else k: v for k, v in hp.items()}}
        assert oracle.adam_replay(st[0], st[1], st[2], st[3], pays, first_step=3, **o) == 0
        dp = [dev(np.concatenate([p, np.zeros(16, np.uint8)])) for p in pays]
        tc.adam_replay(ctx, *gs, dp, [p.size for p in pays], 3, torch.empty(n, device="cuda"), **hp)
        ctx.check()
        assert same_state(gs, st)
