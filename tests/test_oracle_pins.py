"""Pins for the ORACLE (oracle/tco.c) against things other than itself:
hand examples, numpy library special cases, closed forms,
invariants named by BASELINE.json's north_star, brute force on tiny inputs, and tamper
cases for the error classes.  CPU only."""
import itertools
import os

import numpy as np
import pytest

import synth
from tests import recfmt

GOLD = os.path.join(os.path.dirname(__file__), "golden")
RNG = np.random.default_rng(20261018)


def gold(name):
    with open(os.path.join(GOLD, name), "rb") as fh:
        return np.frombuffer(fh.read(), dtype=np.uint8)


# ------------------------------------------------------------ hand examples ----
def test_hand_example_fp32(tco):
    """SURVEY.md Appendix A, hand example 1: +0 -> -0 is a change, a NaN whose payload
    changed is a change, a bit-identical NaN is not (reading R5)."""
    ref = np.array([0x3F800000, 0, 0x80000000, 0x7FC00000, 0x12345678, 0x7FC00000], np.uint32)
    cur = np.array([0x3F800000, 0x80000000, 0x80000000, 0x7FC00001, 0x12345678, 0x7FC00000],
                   np.uint32)
    rc, rec = tco.encode([ref], [cur], tile_words=4096, advance_ref=False, version=7,
                         ref_version=6)
    assert rc == 0
    assert rec.size == 112
    r = recfmt.parse(rec)
    assert r["magic"] == b"TCD1" and r["fmt"] == 1 and r["w"] == 4 and r["flags"] == 1
    assert r["T"] == 4096 and r["seg"] == 0 and r["off"] == 0 and r["m"] == 6
    assert r["version"] == 7 and r["ref_version"] == 6 and r["total"] == 112
    assert list(r["mask"]) == [0x0000000A]
    assert r["count"] == 2
    assert list(r["toff"]) == [0, 2]
    assert list(r["values"]) == [0x80000000, 0x7FC00001]
    assert np.array_equal(rec, gold("hand1_fp32.bin"))
    # a float compare would give a different mask on this input (the pin bites)
    fmask = ref.view(np.float32) != cur.view(np.float32)
    assert list(np.nonzero(fmask)[0]) != [1, 3]


def test_hand_example_bf16(tco):
    ref = np.array([0x3F80, 0x3F80, 0xFFFF], np.uint16)
    cur = np.array([0x3F81, 0x3F80, 0xFFFF], np.uint16)
    rc, rec = tco.encode([ref], [cur], tile_words=4096, advance_ref=False)
    assert rc == 0 and rec.size == 112
    r = recfmt.parse(rec)
    assert r["w"] == 2 and list(r["mask"]) == [1] and r["count"] == 1
    assert list(r["values"]) == [0x3F81] and list(r["toff"]) == [0, 1]
    assert np.array_equal(rec, gold("hand2_bf16.bin"))


def test_empty_segment_is_80_bytes(tco):
    e = np.zeros(0, np.uint32)
    rc, rec = tco.encode([e], [e.copy()])
    assert rc == 0 and rec.size == 80
    r = recfmt.parse(rec)
    assert r["m"] == 0 and r["count"] == 0 and list(r["toff"]) == [0]
    assert np.array_equal(rec, gold("empty_m0.bin"))
    # and it applies cleanly to an empty state
    rc, v = tco.apply([np.zeros(0, np.uint32)], 0, rec)
    assert rc == 0 and v == 1


# ------------------------------------------------- library special cases -------
def _rand_pair(n, w, f):
    dt = np.uint16 if w == 2 else np.uint32
    ref = RNG.integers(0, 1 << (8 * w), size=n, dtype=np.uint64).astype(dt)
    ch = RNG.random(n) < f
    cur = ref.copy()
    cur[ch] ^= RNG.integers(1, 1 << (8 * w), size=int(ch.sum()), dtype=np.uint64).astype(dt)
    return ref, cur


def _np_mask_words(changed):
    """Library special case: np.packbits little-endian, padded, viewed as <u4."""
    nb = -(-changed.size // 32) * 4
    b = np.packbits(changed.astype(np.uint8), bitorder="little")
    b = np.concatenate([b, np.zeros(nb - b.size, np.uint8)])
    return b.view("<u4")


@pytest.mark.parametrize("n,w,f,T,C", [
    (1, 4, 1.0, 32, 32), (31, 2, 0.5, 32, 64), (1000, 4, 0.01, 64, 256),
    (4097, 4, 0.3, 4096, 4096), (10000, 2, 0.1, 128, 1024), (12345, 4, 1.0, 32, 4096),
    (70000, 2, 0.003, 4096, 8192), (5000, 4, 0.0, 64, 64),
])
def test_records_equal_library_special_cases(tco, n, w, f, T, C):
    ref, cur = _rand_pair(n, w, f)
    ref0 = ref.copy()
    rc, rec = tco.encode([ref], [cur], tile_words=T, chunk_words=C, advance_ref=True)
    assert rc == 0
    changed = ref0 != cur  # unsigned integer compare of the word bits
    recs = recfmt.records(rec)
    assert len(recs) == -(-n // C)
    pos = 0
    for k, r in enumerate(recs):
        m = r["m"]
        sl = slice(r["off"], r["off"] + m)
        assert r["off"] == k * C and m == min(C, n - k * C)
        ch = changed[sl]
        assert np.array_equal(r["mask"], _np_mask_words(ch))
        assert np.array_equal(r["values"], cur[sl][ch])
        per_tile = np.add.reduceat(ch.astype(np.int64), np.arange(0, m, T)) if m else []
        assert np.array_equal(r["toff"], np.concatenate([[0], np.cumsum(per_tile)]))
        assert r["count"] == int(np.count_nonzero(ch)) == int(
            sum(bin(int(x)).count("1") for x in r["mask"])) == r["toff"][-1] == r["values"].size
        # closed form (SURVEY.md §8(c) "record size")
        p16 = recfmt.pad16
        assert r["total"] == 64 + p16(4 * -(-m // 32)) + p16(4 * (-(-m // T) + 1)) + p16(w * r["count"])
        # pad bytes are zero
        a = rec[r["pos"]: r["pos"] + r["total"]]
        used = np.zeros(r["total"], bool)
        used[:64] = True
        o = 64
        used[o: o + 4 * -(-m // 32)] = True
        o += p16(4 * -(-m // 32))
        used[o: o + 4 * (-(-m // T) + 1)] = True
        o += p16(4 * (-(-m // T) + 1))
        used[o: o + w * r["count"]] = True
        assert not a[~used].any()
        pos += r["total"]
    assert pos == rec.size
    # fused ref advance: ref now equals cur
    assert np.array_equal(ref, cur)


def test_identical_states_give_empty_diff(tco):
    a = RNG.integers(0, 1 << 32, size=9999, dtype=np.uint64).astype(np.uint32)
    rc, rec = tco.encode([a.copy()], [a], tile_words=64, chunk_words=4096)
    assert rc == 0
    for r in recfmt.records(rec):
        assert r["count"] == 0 and not r["mask"].any() and not r["toff"].any()
    assert rec.size == sum(tco.record_bytes(m, 64, 4, 0) for m in (4096, 4096, 1807))


# ------------------------------------------------------------- invariants -------
@pytest.mark.parametrize("w", [2, 4])
@pytest.mark.parametrize("f", [0.0, 0.001, 0.1, 1.0])
def test_round_trip_bitwise(tco, w, f):
    ref, cur = _rand_pair(20000, w, f)
    base = ref.copy()
    rc, rec = tco.encode([ref], [cur], tile_words=256, chunk_words=4096)
    assert rc == 0
    st = base.copy()
    rc, v = tco.apply([st], 0, rec)
    assert rc == 0 and v == 1
    assert np.array_equal(st, cur)


def _newest_first_hit(base_segs, diffs):
    """Independent restatement of the fold with numpy: each word takes its value from
    the newest diff whose mask bit is set; untouched words keep the base value."""
    out = [b.copy() for b in base_segs]
    done = [np.zeros(b.size, bool) for b in base_segs]
    for d in reversed(diffs):
        for r in recfmt.records(d):
            ch = np.unpackbits(r["mask"].view(np.uint8), bitorder="little")[: r["m"]].astype(bool)
            idx = np.nonzero(ch)[0]
            seg, off = r["seg"], r["off"]
            take = ~done[seg][off + idx]
            out[seg][off + idx[take]] = r["values"][take]
            done[seg][off + idx] = True
    return out


@pytest.mark.parametrize("N", [1, 2, 5, 8, 10])
def test_chain_fold_equals_final_state(tco, N):
    sizes, wb = [3001, 7000, 7000, 7000], [2, 4, 4, 4]
    f = 0.05
    states = [synth.state(sizes, wb, synth.SEED0 + 3, v, f) for v in range(N + 1)]
    ref = [a.copy() for a in states[0]]
    diffs = []
    for v in range(1, N + 1):
        rc, d = tco.encode(ref, states[v], tile_words=64, chunk_words=2048, version=v,
                           ref_version=v - 1)
        assert rc == 0
        diffs.append(d)
    st = [a.copy() for a in states[0]]
    rc, ver = tco.fold(st, 0, diffs)
    assert rc == 0 and ver == N
    for a, b in zip(st, states[N]):
        assert np.array_equal(a, b)
    # fold == N sequential applies == newest-first-hit restatement
    st2 = [a.copy() for a in states[0]]
    ver = 0
    for d in diffs:
        rc, ver = tco.apply(st2, ver, d)
        assert rc == 0
    nf = _newest_first_hit(states[0], diffs)
    for a, b, c in zip(st, st2, nf):
        assert np.array_equal(a, b) and np.array_equal(a, c)


def test_cumulative_mode_restores_from_latest_only(tco):
    """Reading R2: with advance_ref = 0 every record is against the base, so restore uses
    only the newest record; folding cumulative records would be wrong when a word
    reverts to its base value."""
    base = np.arange(100, dtype=np.uint32)
    s1 = base.copy(); s1[5] = 999
    s2 = base.copy()  # word 5 reverts
    s2[7] = 1234
    r = base.copy()
    _, d1 = tco.encode([r], [s1], tile_words=32, advance_ref=False, version=1, ref_version=0)
    _, d2 = tco.encode([r], [s2], tile_words=32, advance_ref=False, version=2, ref_version=0)
    assert np.array_equal(r, base)  # no advance
    st = base.copy()
    rc, v = tco.apply([st], 0, d2)
    assert rc == 0 and v == 2 and np.array_equal(st, s2)


# ------------------------------------------------------------ brute force -------
@pytest.mark.parametrize("w", [2, 4])
def test_all_change_masks_m12(tco, w):
    dt = np.uint16 if w == 2 else np.uint32
    base = RNG.integers(0, 1 << (8 * w), size=12, dtype=np.uint64).astype(dt)
    for bits in range(1 << 12):
        ch = np.array([(bits >> i) & 1 for i in range(12)], bool)
        cur = base.copy()
        cur[ch] ^= dt(0x5A5A & ((1 << (8 * w)) - 1) | 1)
        ref = base.copy()
        rc, rec = tco.encode([ref], [cur], tile_words=32, chunk_words=32)
        assert rc == 0
        r = recfmt.parse(rec)
        assert int(r["mask"][0]) == bits
        assert r["count"] == bin(bits).count("1")
        st = base.copy()
        rc, _ = tco.apply([st], 0, rec)
        assert rc == 0 and np.array_equal(st, cur)


def test_chunked_equals_unchunked_small(tco):
    """S:140 analog: for every m in [0, 70], T in {32, 64} and chunk_words in
    {T, 2T, 4096}, the chunk records rebased by chunk_word_offset reproduce the
    single-chunk record's mask and values, and restore identically."""
    for m in range(0, 71):
        for w in (2, 4):
            ref, cur = _rand_pair(m, w, 0.4)
            for T in (32, 64):
                rc, whole = tco.encode([ref.copy()], [cur], tile_words=T, chunk_words=4096)
                assert rc == 0
                W = recfmt.parse(whole)
                for C in (T, 2 * T, 4096):
                    rc, ch = tco.encode([ref.copy()], [cur], tile_words=T, chunk_words=C)
                    assert rc == 0
                    recs = recfmt.records(ch)
                    bits = np.concatenate([np.unpackbits(r["mask"].view(np.uint8),
                                                         bitorder="little")[: r["m"]]
                                           for r in recs]) if m else np.zeros(0, np.uint8)
                    wbits = np.unpackbits(W["mask"].view(np.uint8), bitorder="little")[:m]
                    assert np.array_equal(bits, wbits)
                    vals = np.concatenate([r["values"] for r in recs])
                    assert np.array_equal(vals, W["values"])
                    st = ref.copy()
                    rc, _ = tco.apply([st], 0, ch)
                    assert rc == 0 and np.array_equal(st, cur)


# --------------------------------------------------------------- tampering ------
def _one_record(tco, n=300, w=4, f=0.2, T=64):
    ref, cur = _rand_pair(n, w, f)
    base = ref.copy()
    rc, rec = tco.encode([ref], [cur], tile_words=T, chunk_words=4096, version=5, ref_version=4)
    assert rc == 0
    return base, cur, rec


def _expect(tco, base, rec, code, sv=4):
    st = base.copy()
    rc, v = tco.apply([st], sv, rec)
    assert rc == code
    assert v == sv and np.array_equal(st, base)  # untouched on error


def test_tamper_mask_bit_is_corrupt(tco):
    base, cur, rec = _one_record(tco)
    bad = rec.copy()
    bad[64] ^= 0x40  # flip one mask bit
    _expect(tco, base, bad, tco.ERR_CORRUPT)


def test_tamper_tail_bit_is_corrupt(tco):
    base, cur, rec = _one_record(tco, n=300)  # 300 % 32 = 12 -> bits 12..31 of word 9 unused
    bad = rec.copy()
    bad[64 + 4 * 9 + 3] |= 0x80
    _expect(tco, base, bad, tco.ERR_CORRUPT)


def test_tamper_tile_off_is_corrupt(tco):
    base, cur, rec = _one_record(tco)
    r = recfmt.parse(rec)
    bad = rec.copy()
    toff_pos = 64 + recfmt.pad16(4 * -(-r["m"] // 32))
    bad[toff_pos + 4] ^= 1
    _expect(tco, base, bad, tco.ERR_CORRUPT)


@pytest.mark.parametrize("byte,val", [(0, ord("X")), (4, 2), (6, 8), (7, 3), (8, 33), (12, 1)])
def test_tamper_header_is_corrupt(tco, byte, val):
    base, cur, rec = _one_record(tco)
    bad = rec.copy()
    bad[byte] = val
    _expect(tco, base, bad, tco.ERR_CORRUPT)


def test_truncated_is_corrupt(tco):
    base, cur, rec = _one_record(tco)
    _expect(tco, base, rec[:-16], tco.ERR_CORRUPT)
    _expect(tco, base, rec[:40], tco.ERR_CORRUPT)


def test_version_gap_is_protocol(tco):
    base, cur, rec = _one_record(tco)
    _expect(tco, base, rec, tco.ERR_PROTOCOL, sv=3)  # state at 3, record links 4 -> 5
    bad = rec.copy()
    bad[40:48] = np.frombuffer(np.uint64(4).tobytes(), np.uint8)  # version == ref_version
    _expect(tco, base, bad, tco.ERR_PROTOCOL)


def test_chain_skip_is_protocol(tco):
    sizes, wb = [500], [4]
    s = [synth.state(sizes, wb, 11, v, 0.1) for v in range(4)]
    ref = [a.copy() for a in s[0]]
    ds = []
    for v in (1, 2, 3):
        rc, d = tco.encode(ref, s[v], tile_words=32, version=v, ref_version=v - 1)
        ds.append(d)
    st = [a.copy() for a in s[0]]
    rc, _ = tco.fold(st, 0, [ds[0], ds[2]])  # skip v2
    assert rc == tco.ERR_PROTOCOL


def test_invalid_parameters(tco):
    a = np.zeros(10, np.uint32)
    assert tco.encode([a], [a.copy()], tile_words=48)[0] == tco.ERR_INVALID
    assert tco.encode([a], [a.copy()], tile_words=16)[0] == tco.ERR_INVALID
    assert tco.encode([a], [a.copy()], tile_words=64, chunk_words=96)[0] == tco.ERR_INVALID
    assert tco.encode([a], [a.copy()], tile_words=64, chunk_words=1 << 31)[0] == tco.ERR_INVALID


# ------------------------------------------------------------ determinism -------
def test_golden_chain_is_reproduced(tco):
    sizes, wb = [3000, 3000, 3000], [4, 4, 4]
    s = [synth.state(sizes, wb, synth.SEED0, v, 0.01) for v in range(3)]
    ref = [a.copy() for a in s[0]]
    rc, r1 = tco.encode(ref, s[1], tile_words=64, chunk_words=1024, version=1, ref_version=0)
    rc, r2 = tco.encode(ref, s[2], tile_words=64, chunk_words=1024, version=2, ref_version=1)
    assert np.array_equal(r1, gold("cfg1_small_v1.bin"))
    assert np.array_equal(r2, gold("cfg1_small_v2.bin"))
    st = [a.copy() for a in s[0]]
    rc, v = tco.fold(st, 0, [r1, r2])
    assert rc == 0 and v == 2 and all(np.array_equal(a, b) for a, b in zip(st, s[2]))


def test_multi_segment_order_and_mixed_widths(tco):
    segs_w = [2, 4, 4, 4]
    sizes = [777, 1000, 0, 2049]
    pairs = [_rand_pair(n, w, 0.3) for n, w in zip(sizes, segs_w)]
    ref = [p[0].copy() for p in pairs]
    cur = [p[1] for p in pairs]
    rc, rec = tco.encode(ref, cur, tile_words=32, chunk_words=512)
    assert rc == 0
    recs = recfmt.records(rec)
    key = [(r["seg"], r["off"], r["m"]) for r in recs]
    exp = []
    for s, n in enumerate(sizes):
        if n == 0:
            exp.append((s, 0, 0))
        for off in range(0, n, 512):
            exp.append((s, off, min(512, n - off)))
    assert key == exp
    st = [p[0].copy() for p in pairs]
    rc, _ = tco.apply(st, 0, rec)
    assert rc == 0 and all(np.array_equal(a, b) for a, b in zip(st, cur))


# ------------------------------------------------------- index-mode records ------
def _parse_index(rec, pos=0):
    """Independent parse of an index-mode record: header | tile_off | idx | values."""
    import struct
    (magic, fmt, w, flags, T, seg, off, m, count, version, ref_version, total) = recfmt.HDR.unpack(
        bytes(rec[pos: pos + 64]))
    n_tiles = -(-m // T)
    p = pos + 64
    toff = rec[p: p + 4 * (n_tiles + 1)].view("<u4")
    p += recfmt.pad16(4 * (n_tiles + 1))
    idx = rec[p: p + 2 * count].view("<u2")
    p += recfmt.pad16(2 * count)
    vals = rec[p: p + w * count].view("<u2" if w == 2 else "<u4")
    return dict(flags=flags, T=T, m=m, count=count, total=total, toff=toff, idx=idx, values=vals, off=off, seg=seg)


def test_hand_example_fp32_index_mode(tco):
    ref = np.array([0x3F800000, 0, 0x80000000, 0x7FC00000, 0x12345678, 0x7FC00000], np.uint32)
    cur = np.array([0x3F800000, 0x80000000, 0x80000000, 0x7FC00001, 0x12345678, 0x7FC00000], np.uint32)
    rc, rec = tco.encode([ref], [cur], tile_words=4096, advance_ref=False, version=7, ref_version=6,
                         index_mode=True)
    assert rc == 0 and rec.size == 64 + 16 + 16 + 16
    r = _parse_index(rec)
    assert r["flags"] == 3 and list(r["idx"]) == [1, 3] and list(r["toff"]) == [0, 2]
    assert list(r["values"]) == [0x80000000, 0x7FC00001]
    assert np.array_equal(rec, gold("hand1_fp32_index.bin"))
    st = ref.copy()
    rc, v = tco.apply([st], 6, rec)
    assert rc == 0 and v == 7 and np.array_equal(st, cur)


@pytest.mark.parametrize("n,w,f,T,C", [(1000, 4, 0.01, 64, 256), (70000, 2, 0.003, 4096, 8192),
                                       (12345, 4, 1.0, 32, 4096), (5000, 2, 0.0, 64, 64),
                                       (40000, 4, 0.2, 65536, 65536)])
def test_index_records_equal_library_special_cases(tco, n, w, f, T, C):
    ref, cur = _rand_pair(n, w, f)
    changed = ref != cur
    rc, rec = tco.encode([ref.copy()], [cur], tile_words=T, chunk_words=C, index_mode=True)
    assert rc == 0
    pos = 0
    for k in range(-(-n // C)):
        r = _parse_index(rec, pos)
        m = r["m"]
        ch = changed[r["off"]: r["off"] + m]
        where = np.nonzero(ch)[0]
        assert np.array_equal(r["idx"], (where % T).astype(np.uint16))  # in-tile positions
        assert np.array_equal(r["values"], cur[r["off"]: r["off"] + m][ch])
        per_tile = np.add.reduceat(ch.astype(np.int64), np.arange(0, m, T)) if m else []
        assert np.array_equal(r["toff"], np.concatenate([[0], np.cumsum(per_tile)]))
        assert r["total"] == tco.record_bytes(m, T, w, r["count"], index_mode=True) == (
            64 + recfmt.pad16(4 * (-(-m // T) + 1)) + recfmt.pad16(2 * r["count"]) + recfmt.pad16(w * r["count"]))
        pos += r["total"]
    assert pos == rec.size
    st = ref.copy()
    rc, _ = tco.apply([st], 0, rec)
    assert rc == 0 and np.array_equal(st, cur)


@pytest.mark.parametrize("w", [2, 4])
def test_index_mode_all_change_masks_m12(tco, w):
    dt = np.uint16 if w == 2 else np.uint32
    base = RNG.integers(0, 1 << (8 * w), size=12, dtype=np.uint64).astype(dt)
    for bits in range(0, 1 << 12, 7):
        ch = np.array([(bits >> i) & 1 for i in range(12)], bool)
        cur = base.copy()
        cur[ch] ^= dt(0x3C)
        rc, rec = tco.encode([base.copy()], [cur], tile_words=32, chunk_words=32, index_mode=True)
        assert rc == 0
        assert list(_parse_index(rec)["idx"]) == [i for i in range(12) if ch[i]]
        st = base.copy()
        rc, _ = tco.apply([st], 0, rec)
        assert rc == 0 and np.array_equal(st, cur)


def test_mixed_mode_chain_fold(tco):
    sizes, wb = [3000, 5000], [2, 4]
    s = [synth.state(sizes, wb, 21, v, 0.05) for v in range(5)]
    ref = [a.copy() for a in s[0]]
    ds = []
    for v in range(1, 5):
        rc, d = tco.encode(ref, s[v], tile_words=64, chunk_words=1024, version=v, ref_version=v - 1,
                           index_mode=(v % 2 == 1))
        assert rc == 0
        ds.append(d)
    st = [a.copy() for a in s[0]]
    rc, ver = tco.fold(st, 0, ds)
    assert rc == 0 and ver == 4 and all(np.array_equal(a, b) for a, b in zip(st, s[4]))


def _index_rec(tco):
    ref, cur = _rand_pair(300, 4, 0.2)
    rc, rec = tco.encode([ref.copy()], [cur], tile_words=64, version=5, ref_version=4, index_mode=True)
    return ref, rec


def test_index_tamper_out_of_tile_is_corrupt(tco):
    base, rec = _index_rec(tco)
    r = _parse_index(rec)
    bad = rec.copy()
    p = 64 + recfmt.pad16(4 * (-(-300 // 64) + 1))
    bad[p: p + 2] = np.frombuffer(np.uint16(64).tobytes(), np.uint8)  # position 64 is outside a 64-word tile
    _expect(tco, base, bad, tco.ERR_CORRUPT)
    assert r["count"] > 1


def test_index_tamper_not_increasing_is_corrupt(tco):
    base, rec = _index_rec(tco)
    r = _parse_index(rec)
    bad = rec.copy()
    p = 64 + recfmt.pad16(4 * (-(-300 // 64) + 1))
    first = int(r["idx"][0])
    bad[p + 2: p + 4] = np.frombuffer(np.uint16(first).tobytes(), np.uint8)  # duplicate of idx[0]
    if int(r["toff"][1]) >= 2:
        _expect(tco, base, bad, tco.ERR_CORRUPT)


def test_index_tamper_flags_is_corrupt(tco):
    base, rec = _index_rec(tco)
    bad = rec.copy()
    bad[7] = 2  # INDEX without REPLACE
    _expect(tco, base, bad, tco.ERR_CORRUPT)


# --------------------------------------------------------------- full records (R21) -------
def _parse_full(rec, pos=0):
    """Full-format record sections from the layout table: header | values (w*m)."""
    h = rec[pos: pos + 64]
    w, flags = int(h[6]), int(h[7])
    m, count, total = (int(h[a: a + 8].view("<u8")[0]) for a in (24, 32, 56))
    vals = rec[pos + 64: pos + 64 + w * m].view("<u2" if w == 2 else "<u4")
    return dict(w=w, flags=flags, m=m, count=count, total=total, values=vals,
                pad=rec[pos + 64 + w * m: pos + total])


@pytest.mark.parametrize("n,w,f,C", [(0, 4, 0.0, 4096), (1, 2, 1.0, 4096), (7, 2, 0.5, 4096), (300, 4, 0.97, 4096),
                                     (5000, 4, 1.0, 1024), (9001, 2, 0.2, 2048)])
def test_full_records_equal_cur(tco, n, w, f, C):
    """A full record is the chunk of `cur` itself (identity special case): flags 5, count = m, values =
    cur[chunk], size 64 + pad16(w m) with zero padding; chunks rebased like the other formats; the
    reference advances to cur; apply(ref, full) == cur."""
    ref, cur = _rand_pair(n, w, f)
    r0 = ref.copy()
    rc, rec = tco.encode([ref], [cur], tile_words=64, chunk_words=C, version=3, ref_version=2, full=True)
    assert rc == 0
    assert np.array_equal(ref, cur), "advance_ref: ref != cur"
    pos, off = 0, 0
    while True:
        r = _parse_full(rec, pos)
        m = min(n - off, C)
        assert r["flags"] == 5 and r["m"] == m and r["count"] == m and r["w"] == w
        assert r["total"] == 64 + recfmt.pad16(w * m) == tco.record_bytes(m, 64, w, m, full=True)
        assert int(rec[pos + 16: pos + 24].view("<u8")[0]) == off
        assert np.array_equal(r["values"], cur[off: off + m]) and not r["pad"].any()
        pos += r["total"]
        off += m
        if off >= n:
            break
    assert pos == rec.size
    st = r0.copy()
    rc, v = tco.apply([st], 2, rec)
    assert rc == 0 and v == 3 and np.array_equal(st, cur)


def test_full_mask_index_chain_fold(tco):
    """A chain mixing the three formats folds to the final state == sequential applies; a full
    record hides every older change of its chunk (newest wins)."""
    sizes, wb = [3000, 5000], [2, 4]
    s = [synth.state(sizes, wb, 23, v, 0.3) for v in range(7)]
    ref = [a.copy() for a in s[0]]
    ds = []
    for v in range(1, 7):
        rc, d = tco.encode(ref, s[v], tile_words=64, chunk_words=1024, version=v, ref_version=v - 1,
                           index_mode=v % 3 == 1, full=v % 3 == 2)
        assert rc == 0
        ds.append(d)
    st = [a.copy() for a in s[0]]
    rc, ver = tco.fold(st, 0, ds)
    assert rc == 0 and ver == 6 and all(np.array_equal(a, b) for a, b in zip(st, s[6]))
    # from the base, a single full record of version 5 followed by record 6 gives the same state
    ref5 = [a.copy() for a in s[0]]
    rc, d5 = tco.encode(ref5, s[5], tile_words=64, chunk_words=1024, version=5, ref_version=0, full=True)
    st = [a.copy() for a in s[0]]
    assert tco.fold(st, 0, [d5, ds[5]])[0] == 0 and all(np.array_equal(a, b) for a, b in zip(st, s[6]))


@pytest.mark.parametrize("byte,val", [(7, 7), (32, 1), (56, 3)])
def test_full_tamper_is_corrupt(tco, byte, val):
    """flags FULL|INDEX, count != m, total != 64 + pad16(w m) -> CORRUPT, state untouched."""
    ref, cur = _rand_pair(300, 4, 0.9)
    base = ref.copy()
    rc, rec = tco.encode([ref], [cur], tile_words=64, version=5, ref_version=4, full=True)
    bad = rec.copy()
    bad[byte] = (int(bad[byte]) + val) & 0xFF if byte != 7 else val
    _expect(tco, base, bad, tco.ERR_CORRUPT)
    _expect(tco, base, rec[:-16], tco.ERR_CORRUPT)
