"""GPU parity: libtc's CUDA encoder / fold vs the oracle, element by element (byte-exact
records, bit-exact states), on seeded inputs that span several scan blocks, ragged tails,
chunk boundaries inside and across blocks, and the edge cases of the format."""
import numpy as np
import pytest

import synth

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a GPU", allow_module_level=True)

from paper_2605_17821_b200 import tc  # noqa: E402
from tests.gpu_util import gpu_encode, gpu_fold, to_dev, to_np  # noqa: E402

RNG = np.random.default_rng(7)


@pytest.fixture(scope="module")
def ctx():
    c = tc.Ctx(0)
    yield c
    c.close()


# restore strategies (include/tc.h tc_ctx_set_fold_dense_permille): the default threshold, every
# chunk streamed through shared memory (fold_dense_kernel), every chunk scattered (fold_kernel)
FOLD_STRATEGIES = {"auto": None, "stream": 0, "scatter": 0xFFFFFFFF}


@pytest.fixture(scope="module", params=list(FOLD_STRATEGIES))
def fctx(request):
    c = tc.Ctx(0)
    if FOLD_STRATEGIES[request.param] is not None:
        c.set_fold_dense_permille(FOLD_STRATEGIES[request.param])
    yield c
    c.close()


def rand_pair(n, w, f, rng=RNG):
    dt = np.uint16 if w == 2 else np.uint32
    ref = rng.integers(0, 1 << (8 * w), size=n, dtype=np.uint64).astype(dt)
    ch = rng.random(n) < f
    cur = ref.copy()
    cur[ch] ^= rng.integers(1, 1 << (8 * w), size=int(ch.sum()), dtype=np.uint64).astype(dt)
    return ref, cur


CASES = [
    # sizes, widths, f, T, C
    ([6], [4], 0.5, 4096, 1 << 28),
    ([3], [2], 0.7, 4096, 1 << 28),
    ([0], [4], 0.0, 4096, 1 << 28),
    ([1], [2], 1.0, 32, 32),
    ([7], [2], 1.0, 32, 64),
    ([4097], [4], 0.3, 4096, 1 << 28),
    ([8193], [2], 0.3, 4096, 1 << 28),
    ([100003], [4], 0.01, 4096, 1 << 28),
    ([100003], [2], 0.01, 4096, 1 << 28),
    ([50000], [4], 1.0, 4096, 1 << 28),
    ([50000], [2], 1.0, 4096, 1 << 28),
    ([50000], [4], 0.0, 4096, 1 << 28),
    ([20000], [4], 0.2, 32, 32),          # one block per 32-word chunk
    ([20000], [2], 0.2, 64, 192),         # chunks of 3 tiles, not a block multiple
    ([70000], [4], 0.1, 8192, 16384),     # T > block words (4096)
    ([70000], [2], 0.1, 65536, 65536),    # T = max
    ([30001], [4], 0.05, 128, 4096 * 3),  # chunk = 3 blocks, ragged tail chunk
    ([777, 1000, 0, 2049], [2, 4, 4, 4], 0.3, 32, 512),
    ([123457, 123457, 123457, 123457], [2, 4, 4, 4], 0.01, 4096, 1 << 16),
]


@pytest.mark.parametrize("sizes,wb,f,T,C", CASES)
@pytest.mark.parametrize("advance", [True, False])
def test_encode_matches_oracle_bytes(ctx, tco, sizes, wb, f, T, C, advance):
    pairs = [rand_pair(n, w, f) for n, w in zip(sizes, wb)]
    ref = [p[0] for p in pairs]
    cur = [p[1] for p in pairs]
    ref_o = [r.copy() for r in ref]
    rc, exp = tco.encode(ref_o, cur, tile_words=T, chunk_words=C, advance_ref=advance, version=9, ref_version=8)
    assert rc == 0
    got, ref_after, nbytes = gpu_encode(ctx, ref, cur, T, C, advance, 9, 8)
    assert nbytes == exp.size
    assert np.array_equal(got, exp), "record bytes differ from the oracle"
    for a, b in zip(ref_after, ref_o):
        assert np.array_equal(a, b)


@pytest.mark.parametrize("f", [0.0, 0.001, 0.01, 0.1, 0.5, 1.0])
def test_encode_synth_cfg1_shape(ctx, tco, f):
    """cfg1 (BASELINE.json configs[0]): 1M fp32 params + Adam m/v, one base and one step."""
    sizes, wb = [1 << 20] * 3, [4, 4, 4]
    base = synth.state(sizes, wb, synth.SEED0, 0, f)
    cur = synth.state(sizes, wb, synth.SEED0, 1, f)
    ref_o = [a.copy() for a in base]
    rc, exp = tco.encode(ref_o, cur)
    got, ref_after, _ = gpu_encode(ctx, base, cur)
    assert np.array_equal(got, exp)
    assert all(np.array_equal(a, b) for a, b in zip(ref_after, cur))


def test_encode_is_deterministic(ctx):
    ref, cur = rand_pair(300000, 4, 0.2)
    a, _, _ = gpu_encode(ctx, [ref], [cur], 256, 4096 * 8)
    b, _, _ = gpu_encode(ctx, [ref], [cur], 256, 4096 * 8)
    assert np.array_equal(a, b)


@pytest.mark.parametrize("index_mode", [False, True])
@pytest.mark.parametrize("sizes,wb,f,T,C", [
    ([30000, 20001], [4, 2], 0.05, 4096, 1 << 28),
    ([70001], [4], 0.3, 256, 8192),   # several chunks: the overflow lands in a later record
])
def test_encode_capacity_checked_on_device(ctx, tco, sizes, wb, f, T, C, index_mode):
    """out_cap below the worst-case bound: a diff that fits is byte-exact; one that does not is
    refused on the device (sticky CAPACITY), writes nothing at or past out_cap, and reports the
    length it needs (include/tc.h tc_diff_encode)."""
    ref_np = [synth.base(n, w, 3, i) for i, (n, w) in enumerate(zip(sizes, wb))]
    cur_np = synth.state(sizes, wb, 3, 1, f)
    rc, exp = tco.encode([a.copy() for a in ref_np], cur_np, tile_words=T, chunk_words=C, advance_ref=False,
                         version=1, ref_version=0, index_mode=index_mode)
    assert rc == 0
    n = exp.size
    ref = [to_dev(a) for a in ref_np]
    cur = [to_dev(a) for a in cur_np]
    for cap in (n, n - 16, n // 2, 100):
        buf = torch.full((n + 4096,), 0xAB, dtype=torch.uint8, device="cuda")
        ob = torch.zeros(1, dtype=torch.int64, device="cuda")
        tc.diff_encode(ctx, ref, cur, buf[:cap], ob, 1, 0, T, C, advance_ref=False, index_mode=index_mode)
        rc = ctx.check_status()
        got = buf.cpu().numpy()
        assert int(ob.item()) == n
        if cap == n:
            assert rc == tc.OK and np.array_equal(got[:n], exp)
        else:
            assert rc == tc.ERR_CAPACITY
            assert (got[cap:] == 0xAB).all(), "bytes written past out_cap"


def test_range_encode_capacity_checked_on_device(ctx, tco):
    n_words, T, C = 50000, 1024, 8192
    ref_np = synth.base(n_words, 4, 9, 0)
    cur_np = synth.state([n_words], [4], 9, 1, 0.2)[0]
    ref, cur = to_dev(ref_np), to_dev(cur_np)
    cap_full = tc.diff_bound_range(n_words, 4, 1, 3, T, C)
    buf = torch.full((cap_full,), 0xAB, dtype=torch.uint8, device="cuda")
    ob = torch.zeros(1, dtype=torch.int64, device="cuda")
    tc.diff_encode_range(ctx, ref, cur, 0, 1, 3, buf, ob, 1, 0, T, C, advance_ref=False)
    ctx.check()
    need = int(ob.item())
    small = need - 32
    buf.fill_(0xAB)
    tc.diff_encode_range(ctx, ref, cur, 0, 1, 3, buf[:small], ob, 1, 0, T, C, advance_ref=False)
    assert ctx.check_status() == tc.ERR_CAPACITY and int(ob.item()) == need
    assert (buf[small:].cpu().numpy() == 0xAB).all()


# ------------------------------------------------------------------ fold -------------
def make_chain(tco, sizes, wb, N, f, T, C, seed=5, structure=synth.S1_IID):
    states = [synth.state(sizes, wb, seed, v, f, structure) for v in range(N + 1)]
    ref = [a.copy() for a in states[0]]
    diffs = []
    for v in range(1, N + 1):
        rc, d = tco.encode(ref, states[v], tile_words=T, chunk_words=C, version=v, ref_version=v - 1)
        assert rc == 0
        diffs.append(d)
    return states, diffs


@pytest.mark.parametrize("N", [1, 2, 5, 8, 10])
@pytest.mark.parametrize("layout", [
    ([30011, 30011, 30011, 30011], [2, 4, 4, 4], 4096, 1 << 28),
    ([20000, 9000], [4, 2], 64, 1024),
    ([40000], [4], 16384, 32768),
])
def test_fold_matches_oracle(fctx, tco, N, layout):
    sizes, wb, T, C = layout
    states, diffs = make_chain(tco, sizes, wb, N, 0.05, T, C)
    st_o = [a.copy() for a in states[0]]
    rc, ver = tco.fold(st_o, 0, diffs)
    assert rc == 0 and ver == N
    rc, st_g = gpu_fold(fctx, states[0], 0, diffs)
    assert rc == tc.OK
    for a, b, c in zip(st_g, st_o, states[N]):
        assert np.array_equal(a, b) and np.array_equal(a, c)


def test_fold_max_chain(fctx, tco):
    """TC_MAX_FOLD records: 8 batches of kDBatch records in the streaming fold."""
    N = tc.MAX_FOLD
    states, diffs = make_chain(tco, [9000, 7001], [4, 2], N, 0.01, 1024, 1 << 28, seed=21)
    rc, st_g = gpu_fold(fctx, states[0], 0, diffs)
    assert rc == tc.OK
    assert all(np.array_equal(a, b) for a, b in zip(st_g, states[N]))


@pytest.mark.parametrize("sizes,wb,T,C,f", [
    ([1027, 3], [4, 4], 32, 64, 0.6),        # T < 1024 (sub-unit of many tiles), ragged words
    ([5000, 5001], [2, 2], 2048, 4096, 0.9),  # index windows longer than 32 entries
    ([33000], [4], 8192, 8192, 0.3),          # T > 1024: carried positions across sub-units
])
def test_index_fold_strategies(fctx, tco, sizes, wb, T, C, f):
    N = 4
    states = [synth.state(sizes, wb, 17, v, f) for v in range(N + 1)]
    ref = [a.copy() for a in states[0]]
    diffs = []
    for v in range(1, N + 1):
        rc, d = tco.encode(ref, states[v], tile_words=T, chunk_words=C, version=v, ref_version=v - 1,
                           index_mode=True)
        assert rc == 0
        diffs.append(d)
    rc, st_g = gpu_fold(fctx, states[0], 0, diffs)
    assert rc == tc.OK
    assert all(np.array_equal(a, b) for a, b in zip(st_g, states[N]))


@pytest.mark.parametrize("f", [0.0, 0.01, 1.0])
def test_fold_dense_and_empty(fctx, tco, f):
    states, diffs = make_chain(tco, [50000, 50000], [2, 4], 3, f, 4096, 1 << 28, seed=9)
    rc, st_g = gpu_fold(fctx, states[0], 0, diffs)
    assert rc == tc.OK
    assert all(np.array_equal(a, b) for a, b in zip(st_g, states[3]))


def test_fold_s2_runs(fctx, tco):
    states, diffs = make_chain(tco, [100000, 100000], [2, 4], 5, 0.2, 4096, 1 << 28, seed=2,
                               structure=synth.S2_RUNS)
    rc, st_g = gpu_fold(fctx, states[0], 0, diffs)
    assert rc == tc.OK
    assert all(np.array_equal(a, b) for a, b in zip(st_g, states[5]))


def test_fold_of_gpu_encoded_chain(fctx, tco):
    """GPU encode (incremental, fused ref advance) -> GPU fold reproduces the final state."""
    sizes, wb = [60000, 60000, 60000, 60000], [2, 4, 4, 4]
    N = 8
    states = [synth.state(sizes, wb, 77, v, 0.02) for v in range(N + 1)]
    ref = [a.copy() for a in states[0]]
    diffs = []
    for v in range(1, N + 1):
        d, ref, _ = gpu_encode(fctx, ref, states[v], version=v, ref_version=v - 1)
        diffs.append(d)
    rc, st_g = gpu_fold(fctx, states[0], 0, diffs)
    assert rc == tc.OK
    assert all(np.array_equal(a, b) for a, b in zip(st_g, states[N]))


# ------------------------------------------------------------- tampering -------------
def _chain1(tco, n=20000, w=4, T=256):
    states, diffs = make_chain(tco, [n], [w], 1, 0.2, T, 1 << 28, seed=3)
    return states, diffs[0]


def test_tamper_mask_bit_corrupt(fctx, tco):
    states, d = _chain1(tco)
    bad = d.copy()
    bad[64 + 4 * 17] ^= 0x10
    rc, _ = gpu_fold(fctx, states[0], 0, [bad])
    assert rc == tc.ERR_CORRUPT == tco.fold([a.copy() for a in states[0]], 0, [bad])[0]


def test_tamper_tile_off_corrupt(fctx, tco):
    states, d = _chain1(tco)
    bad = d.copy()
    m = 20000
    toff = 64 + ((4 * -(-m // 32) + 15) // 16) * 16
    bad[toff + 4 * 5] ^= 1
    rc, _ = gpu_fold(fctx, states[0], 0, [bad])
    assert rc == tc.ERR_CORRUPT == tco.fold([a.copy() for a in states[0]], 0, [bad])[0]


@pytest.mark.parametrize("byte,val", [(0, ord("X")), (4, 2), (6, 8), (7, 3), (8, 33), (12, 1)])
def test_tamper_header_corrupt_state_untouched(fctx, tco, byte, val):
    states, d = _chain1(tco)
    bad = d.copy()
    bad[byte] = val
    rc, st = gpu_fold(fctx, states[0], 0, [bad])
    assert rc == tc.ERR_CORRUPT
    assert np.array_equal(st[0], states[0][0])


def test_truncated_corrupt(fctx, tco):
    states, d = _chain1(tco)
    rc, st = gpu_fold(fctx, states[0], 0, [d[:-16]])
    assert rc == tc.ERR_CORRUPT and np.array_equal(st[0], states[0][0])


def test_chain_gap_protocol(fctx, tco):
    states, diffs = make_chain(tco, [5000], [4], 3, 0.1, 64, 1 << 28)
    rc, st = gpu_fold(fctx, states[0], 0, [diffs[0], diffs[2]])
    assert rc == tc.ERR_PROTOCOL and np.array_equal(st[0], states[0][0])
    rc, st = gpu_fold(fctx, states[0], 1, [diffs[0]])
    assert rc == tc.ERR_PROTOCOL
    # the context is clean again after check
    rc, st = gpu_fold(fctx, states[0], 0, diffs)
    assert rc == tc.OK and np.array_equal(st[0], states[3][0])


def test_layout_mismatch_invalid(fctx, tco):
    sizes, wb = [5000], [4]
    s = [synth.state(sizes, wb, 1, v, 0.1) for v in range(3)]
    ref = [a.copy() for a in s[0]]
    _, d1 = tco.encode(ref, s[1], tile_words=64, version=1, ref_version=0)
    _, d2 = tco.encode(ref, s[2], tile_words=128, version=2, ref_version=1)
    rc, _ = gpu_fold(fctx, s[0], 0, [d1, d2])
    assert rc == tc.ERR_INVALID
    # applied one at a time they restore
    rc, st = gpu_fold(fctx, s[0], 0, [d1])
    assert rc == tc.OK
    rc, st = gpu_fold(fctx, st, 1, [d2])
    assert rc == tc.OK and np.array_equal(st[0], s[2][0])


def test_launch_counter(ctx):
    before = ctx.launches
    ref = torch.zeros(5000, dtype=torch.int32, device="cuda")
    out = torch.zeros(tc.diff_bound([5000], [4]), dtype=torch.uint8, device="cuda")
    ob = torch.zeros(1, dtype=torch.int64, device="cuda")
    tc.diff_encode(ctx, [ref], [ref.clone()], out, ob, 1, 0)
    tc.diff_apply(ctx, [ref], 0, [out], [int(ob.item())])
    ctx.check()
    assert ctx.launches == before + 10  # encode (mask, prefix, emit) + fold (walker, scatter, stream, list, mask-list x2, entries)


@pytest.mark.parametrize("advance", [True, False])
def test_range_encode_concatenates_to_full(ctx, tco, advance):
    """tc_diff_encode_range over consecutive chunk runs of every segment == tc_diff_encode."""
    sizes, wb, T, C = [40001, 70003, 0, 33000], [2, 4, 4, 4], 256, 8192
    pairs = [rand_pair(n, w, 0.05) for n, w in zip(sizes, wb)]
    full, ref_full, n_full = gpu_encode(ctx, [p[0] for p in pairs], [p[1] for p in pairs], T, C, advance, 3, 2)
    parts = []
    refs = [to_dev(p[0]) for p in pairs]
    curs = [to_dev(p[1]) for p in pairs]
    for s, (n, w) in enumerate(zip(sizes, wb)):
        nch = max(1, -(-n // C))
        for c0 in range(0, nch, 2):
            cap = tc.diff_bound_range(n, w, c0, 2, T, C)
            out = torch.full((cap,), 0xCD, dtype=torch.uint8, device="cuda")
            ob = torch.zeros(1, dtype=torch.int64, device="cuda")
            tc.diff_encode_range(ctx, refs[s], curs[s], s, c0, 2, out, ob, 3, 2, T, C, advance)
            ctx.check()
            parts.append(out[: int(ob.item())].cpu().numpy())
    got = np.concatenate(parts)
    assert got.size == n_full and np.array_equal(got, full)
    for a, b in zip(refs, ref_full):
        assert np.array_equal(to_np(a), b)


# ------------------------------------------------------------ index mode -------------
IDX_CASES = [c for c in CASES if c[3] <= 8192]


@pytest.mark.parametrize("sizes,wb,f,T,C", IDX_CASES)
def test_index_mode_encode_matches_oracle_bytes(ctx, tco, sizes, wb, f, T, C):
    pairs = [rand_pair(n, w, f) for n, w in zip(sizes, wb)]
    ref = [p[0] for p in pairs]
    cur = [p[1] for p in pairs]
    ref_o = [r.copy() for r in ref]
    rc, exp = tco.encode(ref_o, cur, tile_words=T, chunk_words=C, version=9, ref_version=8, index_mode=True)
    assert rc == 0
    got, ref_after, nbytes = gpu_encode(ctx, ref, cur, T, C, True, 9, 8, index_mode=True)
    assert nbytes == exp.size and np.array_equal(got, exp), "index-mode record bytes differ from the oracle"
    assert all(np.array_equal(a, b) for a, b in zip(ref_after, ref_o))


@pytest.mark.parametrize("N", [1, 3, 8, 10])
@pytest.mark.parametrize("layout", [
    ([30011, 30011, 30011, 30011], [2, 4, 4, 4], 4096, 1 << 28),
    ([20000, 9000], [4, 2], 64, 1024),
    ([40000], [4], 8192, 16384),
])
def test_index_and_mixed_mode_fold_matches_oracle(fctx, tco, N, layout):
    sizes, wb, T, C = layout
    states = [synth.state(sizes, wb, 13, v, 0.03) for v in range(N + 1)]
    ref = [a.copy() for a in states[0]]
    diffs = []
    for v in range(1, N + 1):
        rc, d = tco.encode(ref, states[v], tile_words=T, chunk_words=C, version=v, ref_version=v - 1,
                           index_mode=(v % 3 != 0))
        assert rc == 0
        diffs.append(d)
    st_o = [a.copy() for a in states[0]]
    rc, ver = tco.fold(st_o, 0, diffs)
    assert rc == 0
    rc, st_g = gpu_fold(fctx, states[0], 0, diffs)
    assert rc == tc.OK
    for a, b, c in zip(st_g, st_o, states[N]):
        assert np.array_equal(a, b) and np.array_equal(a, c)


def test_index_mode_gpu_chain_dense_and_sparse(fctx, tco):
    """GPU index-mode encode over sparse and dense blocks, folded on the GPU."""
    sizes, wb = [50000, 50000], [2, 4]
    for f in (0.005, 0.7):
        states = [synth.state(sizes, wb, 31, v, f) for v in range(4)]
        ref = [a.copy() for a in states[0]]
        diffs = []
        for v in range(1, 4):
            d, ref, _ = gpu_encode(fctx, ref, states[v], version=v, ref_version=v - 1, index_mode=True)
            diffs.append(d)
        rc, st_g = gpu_fold(fctx, states[0], 0, diffs)
        assert rc == tc.OK and all(np.array_equal(a, b) for a, b in zip(st_g, states[3]))


def test_index_tamper_gpu(fctx, tco):
    ref, cur = rand_pair(20000, 4, 0.1)
    rc, rec = tco.encode([ref.copy()], [cur], tile_words=256, version=1, ref_version=0, index_mode=True)
    nt = -(-20000 // 256)
    p = 64 + ((4 * (nt + 1) + 15) // 16) * 16
    bad = rec.copy()
    bad[p: p + 2] = np.frombuffer(np.uint16(300).tobytes(), np.uint8)  # outside a 256-word tile
    rc, _ = gpu_fold(fctx, [ref], 0, [bad])
    assert rc == tc.ERR_CORRUPT == tco.fold([ref.copy()], 0, [bad])[0]
    bad = rec.copy()
    bad[7] = 2
    rc, st = gpu_fold(fctx, [ref], 0, [bad])
    assert rc == tc.ERR_CORRUPT and np.array_equal(st[0], ref)


@pytest.mark.parametrize("f", [0.01, 0.3])
def test_index_list_fold_t4096(fctx, tco, f):
    """All-index chains at T = 4096 (the streaming fold's list path): ragged chunk ends, records
    larger than the stage (f = 0.3), chunk boundaries inside a segment."""
    sizes, wb, T, C = [70001, 9000, 4096], [4, 2, 4], 4096, 4096 * 5
    N = 6
    states = [synth.state(sizes, wb, 41, v, f) for v in range(N + 1)]
    ref = [a.copy() for a in states[0]]
    diffs = []
    for v in range(1, N + 1):
        rc, d = tco.encode(ref, states[v], tile_words=T, chunk_words=C, version=v, ref_version=v - 1,
                           index_mode=True)
        assert rc == 0
        diffs.append(d)
    rc, st_g = gpu_fold(fctx, states[0], 0, diffs)
    assert rc == tc.OK
    assert all(np.array_equal(a, b) for a, b in zip(st_g, states[N]))


def test_index_list_tamper(fctx, tco):
    ref, cur = rand_pair(9000, 4, 0.05)
    rc, rec = tco.encode([ref.copy()], [cur], tile_words=4096, version=1, ref_version=0, index_mode=True)
    nt = -(-9000 // 4096)
    p = 64 + ((4 * (nt + 1) + 15) // 16) * 16
    bad = rec.copy()
    bad[p: p + 4] = bad[[p + 2, p + 3, p, p + 1]]  # two positions out of order
    assert tco.fold([ref.copy()], 0, [bad])[0] == tc.ERR_CORRUPT
    rc, _ = gpu_fold(fctx, [ref], 0, [bad])
    assert rc == tc.ERR_CORRUPT
    bad = rec.copy()
    toff1 = 64 + 4
    v = int(np.frombuffer(bad[toff1:toff1 + 4].tobytes(), np.uint32)[0])
    bad[toff1:toff1 + 4] = np.frombuffer(np.uint32(v + 1).tobytes(), np.uint8)  # tile 0 claims one more entry
    assert tco.fold([ref.copy()], 0, [bad])[0] == tc.ERR_CORRUPT
    rc, _ = gpu_fold(fctx, [ref], 0, [bad])
    assert rc == tc.ERR_CORRUPT


def test_index_mode_range_encode(ctx, tco):
    sizes, wb, T, C = [40001, 70003], [2, 4], 256, 8192
    pairs = [rand_pair(n, w, 0.02) for n, w in zip(sizes, wb)]
    full, _, n_full = gpu_encode(ctx, [p[0] for p in pairs], [p[1] for p in pairs], T, C, False, 3, 2, index_mode=True)
    parts = []
    for s, (n, w) in enumerate(zip(sizes, wb)):
        ref_d, cur_d = to_dev(pairs[s][0]), to_dev(pairs[s][1])
        for c0 in range(0, -(-n // C), 3):
            cap = tc.diff_bound_range(n, w, c0, 3, T, C, index_mode=True)
            out = torch.empty(cap, dtype=torch.uint8, device="cuda")
            ob = torch.zeros(1, dtype=torch.int64, device="cuda")
            tc.diff_encode_range(ctx, ref_d, cur_d, s, c0, 3, out, ob, 3, 2, T, C, False, index_mode=True)
            ctx.check()
            parts.append(out[: int(ob.item())].cpu().numpy())
    assert np.array_equal(np.concatenate(parts), full)


@pytest.mark.parametrize("N", [32, 33])
def test_index_list_fold_chain_length_limit(fctx, tco, N):
    """All-index T = 4096 chains at the list kernel's record-table limit (kListMaxRec = 32) and one
    past it (such chunks go to the other fold paths): both restore the chain head."""
    sizes, wb, T = [20000, 9001], [4, 2], 4096
    states = [synth.state(sizes, wb, 43, v, 0.02) for v in range(N + 1)]
    ref = [a.copy() for a in states[0]]
    diffs = []
    for v in range(1, N + 1):
        rc, d = tco.encode(ref, states[v], tile_words=T, version=v, ref_version=v - 1, index_mode=True)
        assert rc == 0
        diffs.append(d)
    rc, st_g = gpu_fold(fctx, states[0], 0, diffs)
    assert rc == tc.OK
    assert all(np.array_equal(a, b) for a, b in zip(st_g, states[N]))


# ------------------------------------------------------- ADVICE r1 regressions -------------
@pytest.mark.parametrize("n,w", [(4099, 4), (4097, 4), (8195, 2), (8193, 2), (13, 2), (3, 4)])
def test_advance_ref_view_keeps_bytes_past_the_segment(ctx, tco, n, w):
    """The fused ref advance writes nothing past n_words: the ref is a view into a larger buffer
    whose trailing bytes are sentinels (include/tc.h tc_segment: only the first n_words words are
    the caller's segment).  The last vector straddles the segment end and its tail word changed."""
    dt = torch.int16 if w == 2 else torch.int32
    ref_np, cur_np = rand_pair(n, w, 0.0)
    cur_np[-1] ^= 1  # the straddling vector holds a change
    cur_np[0] ^= 1
    buf = torch.full((n + 64,), -0x5A5A if w == 2 else -0x5A5A5A5A, dtype=dt, device="cuda")
    buf[:n] = to_dev(ref_np)
    ref = buf[:n]
    cur = to_dev(cur_np)
    cap = tc.diff_bound([n], [w])
    out = torch.empty(cap, dtype=torch.uint8, device="cuda")
    ob = torch.zeros(1, dtype=torch.int64, device="cuda")
    tc.diff_encode(ctx, [ref], [cur], out, ob, 1, 0, advance_ref=True)
    ctx.check()
    rc, exp = tco.encode([ref_np.copy()], [cur_np], version=1, ref_version=0)
    assert rc == 0 and np.array_equal(out[: int(ob.item())].cpu().numpy(), exp)
    assert np.array_equal(to_np(buf[:n]), cur_np)
    tail = buf[n:].cpu()
    assert bool((tail == (-0x5A5A if w == 2 else -0x5A5A5A5A)).all()), "bytes past the segment were written"


def test_index_tamper_t8192_chain(fctx, tco):
    """Index mode at T = 8192 (tiles span two 4096-word fold units), N = 2: a non-increasing
    position list in the second record must surface as CORRUPT, never as out-of-range shared
    memory writes (tc_apply.cu build_mask_from_index)."""
    n, T = 40000, 8192
    states = [synth.state([n], [4], 77, v, 0.05) for v in range(3)]
    ref = [states[0][0].copy()]
    recs = []
    for v in (1, 2):
        rc, d = tco.encode(ref, [states[v][0]], tile_words=T, version=v, ref_version=v - 1, index_mode=True)
        assert rc == 0
        recs.append(d)
    nt = -(-n // T)
    p = 64 + ((4 * (nt + 1) + 15) // 16) * 16
    toff = np.frombuffer(recs[1][64: 64 + 4 * (nt + 1)].tobytes(), np.uint32)
    k0, k1 = int(toff[0]), int(toff[1])
    assert k1 - k0 > 4
    for lo, hi in ((k0, k1 - 1), (k0 + 1, k1 - 2)):  # swap entries: the list is no longer increasing
        bad = recs[1].copy()
        a = bad[p + 2 * lo: p + 2 * lo + 2].copy()
        bad[p + 2 * lo: p + 2 * lo + 2] = bad[p + 2 * hi: p + 2 * hi + 2]
        bad[p + 2 * hi: p + 2 * hi + 2] = a
        assert tco.fold([states[0][0].copy()], 0, [recs[0], bad])[0] == tc.ERR_CORRUPT
        rc, _ = gpu_fold(fctx, states[0], 0, [recs[0], bad])
        assert rc == tc.ERR_CORRUPT
    rc, st = gpu_fold(fctx, states[0], 0, recs)
    assert rc == tc.OK and np.array_equal(st[0], states[2][0])


# ------------------------------------------------------------ full records (R21) ------------
@pytest.mark.parametrize("sizes,wb,f,T,C", CASES)
@pytest.mark.parametrize("advance", [True, False])
def test_full_encode_matches_oracle_bytes(ctx, tco, sizes, wb, f, T, C, advance):
    """Full-format records (every word, kernel F): byte-exact vs the oracle, ref advanced."""
    pairs = [rand_pair(n, w, f) for n, w in zip(sizes, wb)]
    ref = [p[0] for p in pairs]
    cur = [p[1] for p in pairs]
    ref_o = [r.copy() for r in ref]
    rc, exp = tco.encode(ref_o, cur, tile_words=T, chunk_words=C, advance_ref=advance, version=9, ref_version=8,
                         full=True)
    assert rc == 0
    refd = [to_dev(a) for a in ref]
    curd = [to_dev(a) for a in cur]
    cap = tc.diff_bound([a.size for a in ref], [a.itemsize for a in ref], T, C, full=True)
    assert cap == exp.size
    out = torch.full((cap + 64,), 0xAB, dtype=torch.uint8, device="cuda")
    ob = torch.zeros(1, dtype=torch.int64, device="cuda")
    tc.diff_encode(ctx, refd, curd, out, ob, 9, 8, T, C, advance, full=True)
    ctx.check()
    assert int(ob.item()) == exp.size
    got = out.cpu().numpy()
    assert np.array_equal(got[: exp.size], exp) and (got[exp.size:] == 0xAB).all()
    assert all(np.array_equal(to_np(a), b) for a, b in zip(refd, ref_o))


@pytest.mark.parametrize("N", [1, 3, 6])
def test_full_mask_index_chain_fold_matches_oracle(fctx, tco, N):
    """Chains mixing full, mask and index records fold bit-exactly under every restore strategy."""
    sizes, wb, T, C = [70001, 9000, 33333], [4, 2, 4], 4096, 4096 * 5
    fs = [0.02, 1.0, 0.3, 0.001, 0.99, 0.05]
    states = [synth.state(sizes, wb, 61, 0, 0.0)]
    for v in range(1, N + 1):
        states.append([synth.step(a, 61, s, v, fs[v - 1]) for s, a in enumerate(states[-1])])
    ref = [a.copy() for a in states[0]]
    diffs = []
    for v in range(1, N + 1):
        rc, d = tco.encode(ref, states[v], tile_words=T, chunk_words=C, version=v, ref_version=v - 1,
                           index_mode=v % 3 == 1, full=v % 3 == 2)
        assert rc == 0
        diffs.append(d)
    rc, st_g = gpu_fold(fctx, states[0], 0, diffs)
    assert rc == tc.OK
    assert all(np.array_equal(a, b) for a, b in zip(st_g, states[N]))


def test_full_range_encode_and_tamper(ctx, tco):
    """Range encodes of full records concatenate to the full encode; a full record whose count is
    not m, or whose flags say FULL|INDEX, is CORRUPT with the state untouched."""
    sizes, wb, T, C = [40001, 70003], [2, 4], 256, 8192
    ref_np, cur_np = zip(*[rand_pair(n, w, 0.9) for n, w in zip(sizes, wb)])
    rc, exp = tco.encode([a.copy() for a in ref_np], list(cur_np), tile_words=T, chunk_words=C, advance_ref=False,
                         version=2, ref_version=1, full=True)
    parts = []
    for i, (n, w) in enumerate(zip(sizes, wb)):
        nch = -(-n // C)
        for c0 in range(0, nch, 3):
            k = min(3, nch - c0)
            cap = tc.diff_bound_range(n, w, c0, k, T, C, full=True)
            out = torch.zeros(cap, dtype=torch.uint8, device="cuda")
            ob = torch.zeros(1, dtype=torch.int64, device="cuda")
            tc.diff_encode_range(ctx, to_dev(ref_np[i]), to_dev(cur_np[i]), i, c0, k, out, ob, 2, 1, T, C, False,
                                 full=True)
            ctx.check()
            parts.append(out[: int(ob.item())].cpu().numpy())
    assert np.array_equal(np.concatenate(parts), exp)
    for byte, val in ((32, 1), (7, 7)):
        bad = exp.copy()
        bad[byte] = (int(bad[byte]) + val) & 0xFF if byte == 32 else val
        rc, st = gpu_fold(ctx, list(ref_np), 1, [bad])
        assert rc == tc.ERR_CORRUPT and all(np.array_equal(a, b) for a, b in zip(st, ref_np))
    rc, st = gpu_fold(ctx, list(ref_np), 1, [exp])
    assert rc == tc.OK and all(np.array_equal(a, b) for a, b in zip(st, cur_np))


@pytest.mark.parametrize("N", [1, 2, 5, 9])
@pytest.mark.parametrize("T", [4096, 256])
def test_sparse_index_chain_entry_passes(fctx, tco, N, T):
    """Sparse all-index chains (<= 0.25 % per record on average: walker strategy 3, one entry pass
    per record oldest first) fold bit-exactly; a non-increasing position list in a middle record is
    CORRUPT (the fold may have started: the state is then unspecified)."""
    sizes, wb, C = [300_001, 70_001, 200_003], [4, 2, 4], 4096 * 16
    states = [synth.state(sizes, wb, 71, v, 0.002) for v in range(N + 1)]
    ref = [a.copy() for a in states[0]]
    diffs = []
    for v in range(1, N + 1):
        rc, d = tco.encode(ref, states[v], tile_words=T, chunk_words=C, version=v, ref_version=v - 1,
                           index_mode=True)
        assert rc == 0
        diffs.append(d)
    rc, st_g = gpu_fold(fctx, states[0], 0, diffs)
    assert rc == tc.OK
    assert all(np.array_equal(a, b) for a, b in zip(st_g, states[N]))
    # tamper record (N+1)//2: swap the first two positions of the first tile holding >= 2 entries
    j = (N + 1) // 2 - 1
    bad = diffs[j].copy()
    nt = -(-min(sizes[0], C) // T)
    toff = bad[64: 64 + 4 * (nt + 1)].view("<u4")
    t = int(np.nonzero(np.diff(toff.astype(np.int64)) >= 2)[0][0])
    p = 64 + ((4 * (nt + 1) + 15) // 16) * 16 + 2 * int(toff[t])
    bad[p: p + 4] = bad[[p + 2, p + 3, p, p + 1]]
    chain = diffs[:j] + [bad] + diffs[j + 1:]
    assert tco.fold([a.copy() for a in states[0]], 0, chain)[0] == tc.ERR_CORRUPT
    rc, _ = gpu_fold(fctx, states[0], 0, chain)
    assert rc == tc.ERR_CORRUPT


def test_fold_max_records_hint(tco):
    """tc_ctx_set_fold_max_records: the exact records-per-diff bound folds exactly (descriptor
    scratch sized by it); a bound below the diff's record count is refused (CAPACITY), state kept."""
    sizes, wb, T, C = [20000, 9000, 0], [4, 2, 4], 256, 4096
    states, diffs = make_chain(tco, sizes, wb, 3, 0.1, T, C, seed=41)
    per_diff = sum(max(1, -(-n // C)) for n in sizes)  # 5 + 3 + 1 (an empty segment is one record)
    c = tc.Ctx(0)
    try:
        c.set_fold_max_records(per_diff)
        rc, st_g = gpu_fold(c, states[0], 0, diffs)
        assert rc == tc.OK and all(np.array_equal(a, b) for a, b in zip(st_g, states[3]))
        c.set_fold_max_records(per_diff - 1)
        rc, st_g = gpu_fold(c, states[0], 0, diffs)
        assert rc == tc.ERR_CAPACITY
        assert all(np.array_equal(a, b) for a, b in zip(st_g, states[0]))
        c.set_fold_max_records(0)
        rc, st_g = gpu_fold(c, states[0], 0, diffs)
        assert rc == tc.OK and all(np.array_equal(a, b) for a, b in zip(st_g, states[3]))
    finally:
        c.close()
