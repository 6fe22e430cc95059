"""GPU parity of the mask-list fold (fold_mlist_kernel, walker strategy 4): chains
of mask-mode records at T = 4096 streamed through shared-memory tiles, newest record winning per
word (§3.3).  Bit-exact against the oracle's fold on chains that
the walker sends to it (long or dense, or every chain with the streaming fixture), ragged last
tiles, chunks of a few tiles, bf16 and fp32 segments, up to the 32-record limit (and past it, where
other kernels take the chain), mixed mask / index chains, and tampered records (CORRUPT)."""
import numpy as np
import pytest

import synth

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a GPU", allow_module_level=True)

from paper_2605_17821_b200 import tc  # noqa: E402
from tests.gpu_util import gpu_fold  # noqa: E402

STRATEGIES = {"auto": None, "stream": 0, "scatter": 0xFFFFFFFF}


@pytest.fixture(scope="module", params=list(STRATEGIES))
def fctx(request):
    c = tc.Ctx(0)
    if STRATEGIES[request.param] is not None:
        c.set_fold_dense_permille(STRATEGIES[request.param])
    yield c
    c.close()


def chain(tco, sizes, wb, N, f, C, seed, index_of=lambda v: False, structure=synth.S1_IID, T=4096):
    states = [synth.state(sizes, wb, seed, v, f, structure) for v in range(N + 1)]
    ref = [a.copy() for a in states[0]]
    diffs = []
    for v in range(1, N + 1):
        rc, d = tco.encode(ref, states[v], tile_words=T, chunk_words=C, version=v, ref_version=v - 1,
                           index_mode=index_of(v))
        assert rc == 0
        diffs.append(d)
    return states, diffs


def check(fctx, tco, states, diffs):
    N = len(diffs)
    st_o = [a.copy() for a in states[0]]
    rc, ver = tco.fold(st_o, 0, diffs)
    assert rc == 0 and ver == N
    rc, st_g = gpu_fold(fctx, states[0], 0, diffs)
    assert rc == tc.OK
    for a, b, c in zip(st_g, st_o, states[N]):
        assert np.array_equal(a, b) and np.array_equal(a, c)


LAYOUTS = [
    ([4096 * 5 + 777, 4096 * 3 + 1, 4096 * 4, 33], [2, 4, 4, 4], 1 << 28),  # ragged last tiles, a tiny segment
    ([4096 * 7 + 100, 4096 * 6 + 5], [4, 2], 4096 * 3),                       # chunks of 3 tiles, ragged tails
]


@pytest.mark.parametrize("N", [1, 2, 8])
@pytest.mark.parametrize("f", [0.01, 0.1, 0.6, 1.0])
@pytest.mark.parametrize("layout", LAYOUTS)
def test_mask_chain_fold_matches_oracle(fctx, tco, N, f, layout):
    sizes, wb, C = layout
    states, diffs = chain(tco, sizes, wb, N, f, C, seed=31 + N)
    check(fctx, tco, states, diffs)


@pytest.mark.parametrize("N", [32, 33])
def test_mask_chain_record_limit(fctx, tco, N):
    """32 records: the mask-list kernel (rounds of 8 records, several rounds per tile); 33: the
    other fold paths take the chain."""
    states, diffs = chain(tco, [4096 * 3 + 9, 4096 * 2], [4, 2], N, 0.05, 1 << 28, seed=5)
    check(fctx, tco, states, diffs)


def test_mask_chain_runs_larger_than_a_round(fctx, tco):
    """Dense records whose value runs fill the stage alone (one record per round)."""
    states, diffs = chain(tco, [4096 * 4 + 3, 8192 * 2 + 1], [4, 2], 6, 0.95, 1 << 28, seed=8)
    check(fctx, tco, states, diffs)


def test_mask_chain_s2_runs(fctx, tco):
    states, diffs = chain(tco, [4096 * 9 + 17, 4096 * 9 + 17], [2, 4], 5, 0.2, 4096 * 4, seed=2,
                          structure=synth.S2_RUNS)
    check(fctx, tco, states, diffs)


def test_mixed_mask_and_index_chain(fctx, tco):
    """Mask and index records alternate (the adaptive format crossing its threshold): exact."""
    states, diffs = chain(tco, [4096 * 5 + 1, 4096 * 5 + 1], [2, 4], 6, 0.04, 1 << 28, seed=6,
                          index_of=lambda v: v % 2 == 0)
    check(fctx, tco, states, diffs)


def _tamper_chain(tco):
    return chain(tco, [4096 * 6 + 50], [4], 4, 0.1, 1 << 28, seed=13)


def test_mlist_tamper_mask_bit(fctx, tco):
    states, diffs = _tamper_chain(tco)
    bad = [d.copy() for d in diffs]
    bad[2][64 + 4 * 200] ^= 0x40  # a mask bit of record 3 (tile 1): the popcount no longer matches tile_off
    rc_o = tco.fold([a.copy() for a in states[0]], 0, bad)[0]
    rc, _ = gpu_fold(fctx, states[0], 0, bad)
    assert rc == tc.ERR_CORRUPT == rc_o


def test_mlist_tamper_tile_off(fctx, tco):
    states, diffs = _tamper_chain(tco)
    m = 4096 * 6 + 50
    toff = 64 + ((4 * -(-m // 32) + 15) // 16) * 16
    bad = [d.copy() for d in diffs]
    bad[1][toff + 4 * 3] ^= 2  # tile_off[3] of record 2
    rc_o = tco.fold([a.copy() for a in states[0]], 0, bad)[0]
    rc, _ = gpu_fold(fctx, states[0], 0, bad)
    assert rc == tc.ERR_CORRUPT == rc_o


def test_mlist_tamper_padding_bit(fctx, tco):
    """A mask bit past the chunk's last word (in the last, partial tile)."""
    states, diffs = _tamper_chain(tco)
    m = 4096 * 6 + 50
    bad = [d.copy() for d in diffs]
    last = 64 + 4 * (m // 32)  # the mask word holding words m-18 .. m+13
    bad[3][last + 3] |= 0x80   # bit 31 of it: word 32 * (m // 32) + 31 >= m
    rc_o = tco.fold([a.copy() for a in states[0]], 0, bad)[0]
    rc, _ = gpu_fold(fctx, states[0], 0, bad)
    assert rc == tc.ERR_CORRUPT == rc_o


@pytest.mark.parametrize("T,C", [(32, 1 << 28), (256, 4096 * 3), (1024, 1024 * 5), (2048, 1 << 28)])
@pytest.mark.parametrize("f", [0.05, 0.5])
def test_mask_chain_small_tiles(fctx, tco, T, C, f):
    """T < 4096: a fold unit of 4096 words holds several tiles; their inner tile_off entries are
    checked against the running count; chunks need not be a multiple of 4096 words."""
    states, diffs = chain(tco, [4096 * 3 + 777, 9000 + 31], [4, 2], 4, f, C, seed=19, T=T)
    check(fctx, tco, states, diffs)


@pytest.mark.parametrize("T", [256, 1024])
def test_mlist_tamper_inner_tile_off(fctx, tco, T):
    """A tile_off entry inside a 4096-word unit (T < 4096) that disagrees with the mask: CORRUPT."""
    m = 4096 * 3 + 50
    states, diffs = chain(tco, [m], [4], 4, 0.2, 1 << 28, seed=23, T=T)
    toff = 64 + ((4 * -(-m // 32) + 15) // 16) * 16
    bad = [d.copy() for d in diffs]
    bad[2][toff + 4 * 5] ^= 4  # tile_off[5]: inside unit 0 (T = 256) / unit 1 (T = 1024)
    rc_o = tco.fold([a.copy() for a in states[0]], 0, bad)[0]
    rc, _ = gpu_fold(fctx, states[0], 0, bad)
    assert rc == tc.ERR_CORRUPT == rc_o
