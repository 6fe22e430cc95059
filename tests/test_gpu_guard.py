"""Out-of-bounds write checks without compute-sanitizer (closed on this GPU pool:
profiles/rd3j_compute_sanitizer_closed.txt).  Every device buffer a call touches — segments,
reference, record, length word, Tier-2 slot and mailbox, fold state, Adam state, payloads,
scratch — is carved out of one arena with a random guard band directly before its first and
directly after its last byte (no padding to a vector or sector size), the call runs, and the
whole arena outside the buffers must equal the pattern byte for byte.  Results are compared with
the oracle as in the parity suites, at ragged sizes where the kernels' tails and vector paths
meet the buffer ends."""
import numpy as np
import pytest

import synth

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a GPU", allow_module_level=True)

import oracle  # noqa: E402
from paper_2605_17821_b200 import tc  # noqa: E402

GUARD = 4096  # bytes of pattern on each side of a buffer
_DT = {2: torch.int16, 4: torch.int32}


class Arena:
    """One device allocation: buffers at 256-byte aligned starts, ends exact, guards between."""

    def __init__(self, nbytes: int, seed: int = 0):
        g = torch.Generator().manual_seed(seed)
        self.pat = torch.randint(0, 256, (nbytes,), dtype=torch.uint8, generator=g).cuda()
        self.buf = self.pat.clone()
        self.off = GUARD
        self.spans = []

    def take(self, nbytes: int) -> torch.Tensor:
        start = (self.off + 255) // 256 * 256
        end = start + nbytes
        self.off = end + GUARD
        assert self.off <= self.buf.numel(), "arena too small for the case"
        self.spans.append((start, end))
        return self.buf[start:end]

    def zeros(self, nbytes: int) -> torch.Tensor:
        t = self.take(nbytes)
        t.zero_()
        return t

    def words(self, a: np.ndarray) -> torch.Tensor:
        t = self.take(a.nbytes)
        if a.nbytes:
            t.copy_(torch.from_numpy(np.ascontiguousarray(a).view(np.uint8)))
        return t.view(_DT[a.itemsize]) if a.itemsize in _DT else t

    def f32(self, a: np.ndarray) -> torch.Tensor:
        t = self.take(a.nbytes)
        if a.nbytes:
            t.copy_(torch.from_numpy(np.ascontiguousarray(a, dtype=np.float32).view(np.uint8)))
        return t.view(torch.float32)

    def u8(self, a: np.ndarray) -> torch.Tensor:
        t = self.take(a.nbytes)
        if a.nbytes:
            t.copy_(torch.from_numpy(np.ascontiguousarray(a)))
        return t

    def check(self):
        torch.cuda.synchronize()
        outside = torch.ones(self.buf.numel(), dtype=torch.bool, device=self.buf.device)
        for s, e in self.spans:
            outside[s:e] = False
        bad = (self.buf != self.pat) & outside
        n = int(bad.sum().item())
        if n:
            first = int(torch.nonzero(bad)[0].item())
            owner = min(self.spans, key=lambda se: min(abs(first - se[0]), abs(first - se[1])))
            raise AssertionError(f"{n} guard bytes overwritten, first at arena byte {first} "
                                 f"(nearest buffer [{owner[0]}, {owner[1]}))")


def host(t: torch.Tensor, dtype) -> np.ndarray:
    return t.cpu().numpy().view(dtype)


def np_of(t: torch.Tensor) -> np.ndarray:
    return t.cpu().numpy().view(np.uint16 if t.dtype == torch.int16 else np.uint32)


@pytest.fixture(scope="module")
def ctx():
    c = tc.Ctx(0)
    yield c
    c.close()


FORMATS = {"mask": {}, "index": {"index_mode": True}, "full": {"full": True}}

ENC_CASES = [
    # sizes, widths, f, T, C
    ([5], [2], 0.7, 4096, 1 << 28),
    ([4099], [4], 0.3, 4096, 1 << 28),          # one word past a block, ragged 16-byte vector
    ([8195], [2], 0.3, 4096, 1 << 28),
    ([100003, 77], [4, 2], 0.01, 4096, 1 << 28),
    ([50001], [2], 1.0, 4096, 1 << 28),
    ([20003], [4], 0.2, 32, 32),
    ([30001, 1, 12345], [4, 2, 4], 0.05, 128, 4096 * 3),
    ([70001], [2], 0.1, 65536, 65536),
]


# index records need tile_words <= 8192 (include/tc.h tc_encode_opts): no index case at T = 65536
@pytest.mark.parametrize("advance", [True, False])
@pytest.mark.parametrize("sizes,wb,f,T,C,fmt", [c + (fmt,) for c in ENC_CASES for fmt in FORMATS
                                                if not (fmt == "index" and c[3] > 8192)])
def test_encode_writes_stay_in_bounds(ctx, tco, sizes, wb, f, T, C, advance, fmt):
    states = [synth.state(sizes, wb, 41, v, f) for v in (0, 1)]
    ref_o = [a.copy() for a in states[0]]
    rc, exp = tco.encode(ref_o, states[1], tile_words=T, chunk_words=C, advance_ref=advance, version=3,
                         ref_version=2, **FORMATS[fmt])
    assert rc == 0
    A = Arena(sum(a.nbytes for a in states[0]) * 2 + exp.size + 64 * GUARD, seed=len(sizes))
    ref = [A.words(a) for a in states[0]]
    cur = [A.words(a) for a in states[1]]
    out = A.zeros(exp.size)            # exactly the record: no slack behind it
    ob = A.zeros(8).view(torch.int64)
    tc.diff_encode(ctx, ref, cur, out, ob, 3, 2, T, C, advance, **FORMATS[fmt])
    ctx.check()
    assert int(ob.item()) == exp.size
    assert np.array_equal(out.cpu().numpy(), exp)
    assert all(np.array_equal(np_of(a), b) for a, b in zip(ref, ref_o))
    assert all(np.array_equal(np_of(a), b) for a, b in zip(cur, states[1]))
    A.check()


@pytest.mark.parametrize("fmt", list(FORMATS))
def test_refused_encode_writes_stay_in_bounds(ctx, tco, fmt):
    sizes, wb, T, C = [70001, 3001], [4, 2], 256, 8192
    states = [synth.state(sizes, wb, 43, v, 0.3) for v in (0, 1)]
    rc, exp = tco.encode([a.copy() for a in states[0]], states[1], tile_words=T, chunk_words=C, advance_ref=False,
                         version=1, ref_version=0, **FORMATS[fmt])
    assert rc == 0
    for cap in (exp.size - 16, exp.size // 3, 64):
        A = Arena(sum(a.nbytes for a in states[0]) * 2 + exp.size + 16 * GUARD, seed=cap)
        ref = [A.words(a) for a in states[0]]
        cur = [A.words(a) for a in states[1]]
        out = A.zeros(cap)
        ob = A.zeros(8).view(torch.int64)
        tc.diff_encode(ctx, ref, cur, out, ob, 1, 0, T, C, False, **FORMATS[fmt])
        assert ctx.check_status() == tc.ERR_CAPACITY
        assert int(ob.item()) == exp.size
        A.check()


@pytest.mark.parametrize("fmt", list(FORMATS))
def test_range_encode_writes_stay_in_bounds(ctx, tco, fmt):
    n, w, T, C = 50001, 4, 1024, 8192
    states = [synth.state([n], [w], 47, v, 0.2)[0] for v in (0, 1)]
    rc, whole = tco.encode([states[0].copy()], [states[1]], tile_words=T, chunk_words=C, advance_ref=True,
                           version=1, ref_version=0, **FORMATS[fmt])
    assert rc == 0
    A = Arena(4 * states[0].nbytes + 2 * whole.size + 32 * GUARD, seed=5)
    ref, cur = A.words(states[0]), A.words(states[1])
    n_chunks = (n + C - 1) // C
    pieces = []
    for first, cnt in ((0, 2), (2, n_chunks - 2)):
        cap = tc.diff_bound_range(n, w, first, cnt, T, C, index_mode=fmt == "index", full=fmt == "full")
        out, ob = A.zeros(cap), A.zeros(8).view(torch.int64)
        tc.diff_encode_range(ctx, ref, cur, 0, first, cnt, out, ob, 1, 0, T, C, True, **FORMATS[fmt])
        ctx.check()
        pieces.append(out[: int(ob.item())].cpu().numpy())
    A.check()
    # the ranges are that part of the whole record (header once, in the first range's output)
    assert sum(p.size for p in pieces) == whole.size
    assert np.array_equal(np.concatenate(pieces), whole)


def _chain(tco, sizes, wb, fmts, f, T, C, seed):
    states = [synth.state(sizes, wb, seed, v, f) for v in range(len(fmts) + 1)]
    ref = [a.copy() for a in states[0]]
    diffs = []
    for v, fmt in enumerate(fmts, start=1):
        rc, d = tco.encode(ref, states[v], tile_words=T, chunk_words=C, version=v, ref_version=v - 1,
                           **FORMATS[fmt])
        assert rc == 0
        diffs.append(d)
    return states, diffs


FOLD_CASES = [
    (["mask"], 0.05), (["index"], 0.001), (["index"], 0.02), (["full"], 1.0),
    (["index"] * 6, 0.002),                      # sparse chain: the entry pass
    (["index"] * 5, 0.05),                       # the list (streaming) pass
    (["mask", "index", "full", "index", "mask"], 0.05),
]


@pytest.mark.parametrize("permille", [None, 0, 0xFFFFFFFF])
@pytest.mark.parametrize("fmts,f", FOLD_CASES)
def test_fold_writes_stay_in_bounds(tco, fmts, f, permille):
    sizes, wb, T, C = [40009, 3, 20011, 8193], [4, 2, 2, 4], 4096, 1 << 16
    states, diffs = _chain(tco, sizes, wb, fmts, f, T, C, seed=53)
    c = tc.Ctx(0)
    try:
        if permille is not None:
            c.set_fold_dense_permille(permille)
        A = Arena(sum(a.nbytes for a in states[0]) + sum(d.size for d in diffs) + 32 * GUARD, seed=7)
        st = [A.words(a) for a in states[0]]
        recs = [A.u8(d) for d in diffs]
        tc.diff_apply(c, st, 0, recs, [d.size for d in diffs])
        c.check()
        assert all(np.array_equal(np_of(a), b) for a, b in zip(st, states[-1]))
        A.check()
    finally:
        c.close()


def _adam_state(r, n):
    st = [r.standard_normal(n).astype(np.float32), np.zeros(n, np.float32), np.zeros(n, np.float32),
          np.zeros(n, np.uint16)]
    st[1][: n // 2] = (r.standard_normal(n // 2) * 1e-3).astype(np.float32)
    st[2][: n // 2] = (np.abs(r.standard_normal(n // 2)) * 1e-6).astype(np.float32)
    return st


@pytest.mark.parametrize("n,kind", [(10, "dense"), (99_999, "dense"), (100_001, "topk"), (250_003, "topk")])
def test_grad_codec_writes_stay_in_bounds(ctx, n, kind):
    r = np.random.default_rng(n)
    g = (r.standard_normal(n) * 1e-2).astype(np.float32)
    rc, exp = oracle.grad_compress(g, seed=n)
    assert rc == 0
    A = Arena(8 * n + 2 * exp.size + 16 * GUARD, seed=n)
    gd = A.f32(g)
    out, ob = A.zeros(exp.size), A.zeros(8).view(torch.int64)
    tc.grad_compress(ctx, gd, n, out, ob)
    ctx.check()
    assert int(ob.item()) == exp.size and np.array_equal(out.cpu().numpy(), exp)
    y = A.zeros(4 * n).view(torch.float32)
    tc.grad_decompress(ctx, out, exp.size, y)
    ctx.check()
    rc, y_o = oracle.grad_decompress(exp, n)
    assert rc == 0 and np.array_equal(host(y, np.uint32), y_o.view(np.uint32))
    A.check()


@pytest.mark.parametrize("N,n", [(1, 50_001), (3, 300_001)])
def test_adam_replay_writes_stay_in_bounds(ctx, N, n):
    r = np.random.default_rng(N * n)
    st = _adam_state(r, n)
    pays = [oracle.grad_compress((r.standard_normal(n) * 1e-2).astype(np.float32), seed=j)[1] for j in range(N)]
    A = Arena(18 * n + sum(p.size for p in pays) + 32 * GUARD, seed=N)
    gs = [A.f32(st[0]), A.f32(st[1]), A.f32(st[2]), A.words(st[3])]
    dp = [A.u8(p) for p in pays]
    scratch = A.zeros(4 * n).view(torch.float32)
    assert oracle.adam_replay(st[0], st[1], st[2], st[3], pays, first_step=4) == 0
    tc.adam_replay(ctx, *gs, dp, [p.size for p in pays], 4, scratch)
    ctx.check()
    for a, b in zip(gs, st):
        assert np.array_equal(a.cpu().numpy().view(b.dtype), b)
    A.check()


@pytest.mark.parametrize("fmt", list(FORMATS))
@pytest.mark.parametrize("n,T,C", [(1, 4096, 1 << 28), (70_001, 256, 8192), (300_003, 4096, 1 << 28)])
def test_adam_step_encode_writes_stay_in_bounds(ctx, tco, n, T, C, fmt):
    r = np.random.default_rng(n + 1)
    st = _adam_state(r, n)
    g = (r.standard_normal(n) * 1e-2).astype(np.float32)
    g[r.random(n) < 0.9] = 0.0
    before = [a.copy() for a in st]
    oracle.adam_step(st[0], st[1], st[2], st[3], g, 5)
    ref = [before[3], before[0].view(np.uint32), before[1].view(np.uint32), before[2].view(np.uint32)]
    cur = [st[3], st[0].view(np.uint32), st[1].view(np.uint32), st[2].view(np.uint32)]
    rc, exp = tco.encode([a.copy() for a in ref], cur, tile_words=T, chunk_words=C, advance_ref=False, version=5,
                         ref_version=4, **FORMATS[fmt])
    assert rc == 0
    A = Arena(20 * n + exp.size + 32 * GUARD, seed=n)
    gs = [A.f32(before[0]), A.f32(before[1]), A.f32(before[2]), A.words(before[3])]
    gd = A.f32(g)
    out, ob = A.zeros(exp.size), A.zeros(8).view(torch.int64)
    tc.adam_step_encode(ctx, *gs, gd, 5, out, ob, T, C, index_mode=fmt == "index", full=fmt == "full")
    ctx.check()
    assert int(ob.item()) == exp.size and np.array_equal(out.cpu().numpy(), exp)
    for a, b in zip(gs, st):
        assert np.array_equal(a.cpu().numpy().view(b.dtype), b)
    A.check()


@pytest.mark.parametrize("fmt", list(FORMATS))
def test_fused_push_writes_stay_in_bounds(ctx, tco, fmt):
    """Fused Tier-2 emit into a slot of exactly the record's size, mailbox of 16 bytes."""
    sizes, wb = [30001, 12345, 7], [2, 4, 4]
    states = [synth.state(sizes, wb, 59, v, 0.03) for v in (0, 1)]
    rc, exp = tco.encode([a.copy() for a in states[0]], states[1], version=1, ref_version=0, **FORMATS[fmt])
    assert rc == 0
    A = Arena(4 * sum(a.nbytes for a in states[0]) + 2 * exp.size + 32 * GUARD, seed=9)
    ref = [A.words(a) for a in states[0]]
    cur = [A.words(a) for a in states[1]]
    out, ob = A.zeros(exp.size), A.zeros(8).view(torch.int64)
    slot, mail = A.zeros(exp.size), A.zeros(16)
    got = A.zeros(8).view(torch.int64)
    tc.diff_encode_push(ctx, ref, cur, out, ob, 1, 0, slot, exp.size, mail, index_mode=fmt == "index",
                        full=fmt == "full")
    tc.peer_wait(ctx, mail, 1, got)
    ctx.check()
    assert int(got.item()) == exp.size
    assert np.array_equal(slot.cpu().numpy(), exp) and np.array_equal(out.cpu().numpy(), exp)
    A.check()


@pytest.mark.parametrize("nbytes", [1, 17, 4095, (1 << 20) + 7])
def test_push_copy_writes_stay_in_bounds(ctx, nbytes):
    r = np.random.default_rng(nbytes)
    src_np = r.integers(0, 256, nbytes, dtype=np.uint8)
    A = Arena(3 * nbytes + 16 * GUARD, seed=nbytes)
    src = A.u8(src_np)
    sb = A.zeros(8).view(torch.int64)
    sb.fill_(nbytes)
    slot, mail = A.zeros(nbytes), A.zeros(16)
    tc.push_peer(ctx, src, sb, slot, nbytes, mail, 4)
    tc.peer_wait(ctx, mail, 4)
    ctx.check()
    assert np.array_equal(slot.cpu().numpy(), src_np)
    A.check()
