"""GPU: the save / retrieve lifecycle (cfg4 scenario, scaled down): a chain of 8 incremental
records, a simulated GPU failure that wipes the live state and the reference, restore from
Tier-1 (H2D of the staged records) with one fold of the chain — bit-exact against the state the
seeded generator defines; plus the full-size (cfg2) parity of the bench launch configuration on
sampled chunks and a full-size round trip."""
import gc

import numpy as np
import pytest

import synth

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a GPU", allow_module_level=True)

from paper_2605_17821_b200 import tc  # noqa: E402
from paper_2605_17821_b200.checkpoint import Checkpointer  # noqa: E402
from tests.gpu_util import to_dev, to_np  # noqa: E402


def _dev_state(sizes, wb, seed, version, f):
    segs = []
    for s, (n, w) in enumerate(zip(sizes, wb)):
        t = torch.empty(n, dtype=torch.int16 if w == 2 else torch.int32, device="cuda")
        tc.synth_base(t, seed, s)
        for v in range(1, version + 1):
            tc.synth_step(t, seed, s, v, synth.p53_of(f))
        segs.append(t)
    return segs


@pytest.mark.parametrize("source", ["t1", "t2", None])
def test_chain_of_8_restore_after_failure(source):
    sizes, wb, seed, f = [70001, 70001, 70001, 70001], [2, 4, 4, 4], synth.SEED0 + 4, 0.01
    live = _dev_state(sizes, wb, seed, 0, f)
    base_host = [to_np(s) for s in live]  # the base checkpoint (version 0)
    ck = Checkpointer(live, tile_words=4096, chunk_words=1 << 14, tier2="push", expected_f=f)
    for v in range(1, 9):
        for s, t in enumerate(live):  # one training step changes a fraction f of the words
            tc.synth_step(t, seed, s, v, synth.p53_of(f))
        ck.save_step(v)
    ck.flush()
    torch.cuda.synchronize()
    expect = synth.state(sizes, wb, seed, 8, f)
    assert all(np.array_equal(to_np(a), b) for a, b in zip(live, expect))
    restored = [to_dev(b) for b in base_host]  # base fetched back (Tier-1/2/3)
    ver = ck.restore(restored, source=source, batch=8)
    assert ver == 8
    for a, b in zip(restored, expect):
        assert np.array_equal(to_np(a), b)
    # restore to an intermediate version with batches of 5 (N = 5)
    mid = [to_dev(b) for b in base_host]
    assert ck.restore(mid, upto=6, batch=5) == 6
    exp6 = synth.state(sizes, wb, seed, 6, f)
    assert all(np.array_equal(to_np(a), b) for a, b in zip(mid, exp6))
    ck.reclaim(6)
    assert ck.chain.base_version == 6 and [e.version for e in ck.chain.entries] == [7, 8]
    ck.close()


@pytest.mark.parametrize("lose_t1", [False, True])
def test_recover_after_gpu_failure_ring_of_one(lose_t1):
    """The lifecycle end to end on one GPU (the ring of one is this GPU): base staged to Tier-1 and
    streamed to the (local) Tier-2 neighbour, 7 saves through the one-step-ahead pipeline with the
    adaptive record format and a hot standby replica, then a GPU failure (state + reference
    wiped) — and optionally a node failure (Tier-1 lost too) — and recover(): consensus, the
    cascade Tier-1 -> Tier-2 for the base and every record, one fold per batch
    of 5.  The recovered state, the reference and the standby equal the seeded chain head."""
    sizes, wb, seed = [90001, 90001, 90001, 90001], [2, 4, 4, 4], synth.SEED0 + 9
    fs = [0.002, 0.3, 0.01, 0.0, 1.0, 0.02, 0.05]  # mixes index / mask records
    live = _dev_state(sizes, wb, seed, 0, 0.0)
    standby = [t.clone() for t in live]
    ck = Checkpointer(live, tier2="push", expected_f=1.0, standby=standby, t2_slots=8, chunk_words=1 << 15)
    expect = [to_np(t) for t in live]
    for v, f in enumerate(fs, start=1):
        for s, t in enumerate(live):
            tc.synth_step(t, seed, s, v, synth.p53_of(f))
        ck.save_step(v)
        expect = [synth.step(e, seed, s, v, f) for s, e in enumerate(expect)]
    ck.base_rep.flush(100)  # the paced base stream completes (sync flush)
    ck.flush()
    ck.base_rep.s.synchronize()
    torch.cuda.synchronize()
    assert all(np.array_equal(to_np(a), b) for a, b in zip(standby, expect))
    formats = {ck.where[e.version]["fmt"] for e in ck.chain.entries}
    assert formats == {"mask", "index", "full"}, f"the adaptive format should use all three: {formats}"
    ck.drop_tier("hbm")
    if lose_t1:
        ck.drop_tier("t1")
    assert ck.recover(batch=5) == len(fs)
    for t in (live, ck.ref):
        assert all(np.array_equal(to_np(a), b) for a, b in zip(t, expect))
    # the chain continues after the recovery
    for s, t in enumerate(live):
        tc.synth_step(t, seed, s, 8, synth.p53_of(0.01))
    ck.save_step(8)
    ck.flush()
    torch.cuda.synchronize()
    assert all(torch.equal(a, b) for a, b in zip(standby, live))
    ck.close()


def test_checkpointer_cfg2_saves_without_reallocation():
    """BASELINE configs[1] (cfg2, 21.8 GB) through the product path: 12 saves with every buffer
    allocated once (record slots sized to the expected change fraction, mapped-pinned lengths,
    one Tier-1 arena), no host synchronization on the encode it just issued, a hot standby folded
    behind every record; device memory does not grow after the first save."""
    sizes, wb = synth.shard_layout("cfg2")
    seed, f = synth.SEED0, 0.01
    W = sum(n * w for n, w in zip(sizes, wb))
    gc.collect()
    torch.cuda.empty_cache()  # blocks cached by earlier tests count as used
    if torch.cuda.mem_get_info()[0] < 3.4 * W:
        pytest.skip("not enough device memory for the full-size case")
    live = _dev_state(sizes, wb, seed, 0, f)
    standby = [t.clone() for t in live]
    ck = Checkpointer(live, expected_f=f, standby=standby, stage_base=False, t1_bytes=16 * (1 << 30))
    torch.cuda.synchronize()
    mem0 = None
    for v in range(1, 13):
        for s, t in enumerate(live):
            tc.synth_step(t, seed, s, v, synth.p53_of(f))
        ck.save_step(v)
        if v == 2:
            torch.cuda.synchronize()
            mem0 = torch.cuda.memory_allocated()
    ck.flush()
    torch.cuda.synchronize()
    assert torch.cuda.memory_allocated() == mem0
    assert [e.version for e in ck.chain.entries] == list(range(1, 13))
    assert all("t1" in e.tiers for e in ck.chain.entries)
    assert all(torch.equal(a, b) for a, b in zip(standby, live))
    assert all(torch.equal(a, b) for a, b in zip(ck.ref, live))
    ck.close()


def test_fullsize_cfg2_sampled_parity_and_round_trip(tco):
    """BASELINE configs[1] (cfg2, 21.8 GB) in the launch configuration bench.py times
    (T = 4096, C = 2^28): GPU record bytes == oracle bytes on sampled chunks, and the fold of the
    full record reproduces the current state exactly."""
    sizes, wb = synth.shard_layout("cfg2")
    seed, f = synth.SEED0, 0.01
    gc.collect()
    torch.cuda.empty_cache()  # blocks cached by earlier tests count as used
    free = torch.cuda.mem_get_info()[0]
    W = sum(n * w for n, w in zip(sizes, wb))
    if free < 4.5 * W:
        pytest.skip("not enough device memory for the full-size case")
    X = _dev_state(sizes, wb, seed, 0, f)
    Y = [x.clone() for x in X]
    for s, t in enumerate(Y):
        tc.synth_step(t, seed, s, 1, synth.p53_of(f))
    ctx = tc.Ctx(0)
    cap = tc.diff_bound(sizes, wb)
    out = torch.empty(cap, dtype=torch.uint8, device="cuda")
    ob = torch.zeros(1, dtype=torch.int64, device="cuda")
    tc.diff_encode(ctx, X, Y, out, ob, 1, 0, advance_ref=False)
    ctx.check()
    n = int(ob.item())
    # locate records on the device copy: walk headers (64 B reads)
    hdrs = []
    pos = 0
    while pos < n:
        h = out[pos: pos + 64].cpu().numpy()
        seg = int(h[12:16].view("<u4")[0])
        off = int(h[16:24].view("<u8")[0])
        m = int(h[24:32].view("<u8")[0])
        total = int(h[56:64].view("<u8")[0])
        hdrs.append((seg, off, m, pos, total))
        pos += total
    assert pos == n
    C = 1 << 28
    picks = [hdrs[0], [h for h in hdrs if h[0] == 3][-1]]  # seg 0 chunk 0 (bf16), seg 3 last chunk
    for seg, off, m, pos, total in picks:
        gpu_rec = out[pos: pos + total].cpu().numpy()
        w = wb[seg]
        ref_np = synth.base(m, w, seed, seg, start=off)
        cur_np = synth.step(ref_np, seed, seg, 1, f, start=off)
        rc, exp = tco.encode([ref_np], [cur_np], tile_words=4096, chunk_words=C, advance_ref=False,
                             version=1, ref_version=0)
        assert rc == 0 and exp.size == total
        # the oracle encoded a one-segment shard: patch segment id and chunk offset, then compare
        exp = exp.copy()
        exp[12:16] = np.frombuffer(np.uint32(seg).tobytes(), np.uint8)
        exp[16:24] = np.frombuffer(np.uint64(off).tobytes(), np.uint8)
        assert np.array_equal(gpu_rec, exp), f"segment {seg} chunk at {off} differs"
    # full-size round trip
    tc.diff_apply(ctx, X, 0, [out], [n])
    ctx.check()
    assert all(torch.equal(a, b) for a, b in zip(X, Y))
    ctx.close()


def _idx_record(buf, pos):
    """Sections of one index-mode record (header | tile_off u32[nt+1] | idx u16[count] |
    values), parsed from the layout table, not from either implementation."""
    h = buf[pos: pos + 64]
    w, flags = int(h[6]), int(h[7])
    T = int(h[8:12].view("<u4")[0])
    seg = int(h[12:16].view("<u4")[0])
    off, m, count = (int(h[a:a + 8].view("<u8")[0]) for a in (16, 24, 32))
    total = int(h[56:64].view("<u8")[0])
    nt = -(-m // T)
    p = pos + 64
    toff = buf[p: p + 4 * (nt + 1)].view("<u4")
    p += -(-4 * (nt + 1) // 16) * 16
    idx = buf[p: p + 2 * count].view("<u2")
    p += -(-2 * count // 16) * 16
    vals = buf[p: p + w * count].view("<u2" if w == 2 else "<u4")
    return dict(w=w, flags=flags, T=T, seg=seg, off=off, m=m, count=count, total=total, toff=toff, idx=idx,
                vals=vals, pos=pos)


@pytest.mark.parametrize("workload,shard", [("cfg2", 0), ("cfg3", 7)])
def test_fullsize_bench_config_chain_parity(tco, workload, shard):
    """BASELINE configs[1] (cfg2, 21.8 GB; and the last cfg3 shard of 8, 11.6 GB, as a rank of the
    N > 1 bench lines holds it, seed SEED0 + shard) in exactly the configuration bench.py times: index-mode
    records, advance_ref = 1, T = 4096, C = 2^28, two chained versions (v0 -> v1 -> v2, the second
    encoded against the advanced reference).  Per segment, the first and the last chunk record are
    byte-compared whole with oracle.encode of that chunk; every other chunk is compared on 8
    random 256-tile windows (tile_off differences, positions and values of the window == the
    oracle's record of the window) — SURVEY §8(d) sampled-chunk rule; the oracle's inputs come from
    synth (numpy), never from the device.  Then the chain folds onto the base bit-exactly."""
    from concurrent.futures import ThreadPoolExecutor

    sizes, wb = synth.shard_layout(workload, shard)
    seed, f, T, C = synth.SEED0 + shard, 0.01, 4096, 1 << 28
    W = sum(n * w for n, w in zip(sizes, wb))
    gc.collect()
    torch.cuda.empty_cache()  # blocks cached by earlier tests count as used
    if torch.cuda.mem_get_info()[0] < 3.3 * W:
        pytest.skip("not enough device memory for the full-size case")
    ref = _dev_state(sizes, wb, seed, 0, f)
    cur = [r.clone() for r in ref]
    ctx = tc.Ctx(0)
    recs = []
    for v in (1, 2):
        for s, t in enumerate(cur):
            tc.synth_step(t, seed, s, v, synth.p53_of(f))
        cap = tc.diff_bound(sizes, wb, T, C, index_mode=True)
        out = torch.empty(cap, dtype=torch.uint8, device="cuda")
        ob = torch.zeros(1, dtype=torch.int64, device="cuda")
        tc.diff_encode(ctx, ref, cur, out, ob, v, v - 1, T, C, True, index_mode=True)
        ctx.check()
        assert all(torch.equal(a, b) for a, b in zip(ref, cur)), "advance_ref: ref != cur after the encode"
        n = int(ob.item())
        recs.append((out, n))
    host = [o[:n].cpu().numpy() for o, n in recs]
    per = []  # (version, record dict)
    for v, buf in zip((1, 2), host):
        pos = 0
        while pos < buf.size:
            r = _idx_record(buf, pos)
            assert r["flags"] == 3 and r["T"] == T
            per.append((v, r))
            pos += r["total"]
        assert pos == buf.size
    rng = np.random.default_rng(2026)
    full_jobs, win_jobs = [], []
    for s in range(4):
        chunks = sorted({r["off"] for v, r in per if r["seg"] == s})
        assert chunks == list(range(0, sizes[s], C))
        for c0 in chunks:
            if c0 in (chunks[0], chunks[-1]):
                full_jobs.append((s, c0))
            else:
                m = min(C, sizes[s] - c0)
                nt = -(-m // T)
                for t0 in rng.choice(nt - 256, size=8, replace=False):
                    win_jobs.append((s, c0, int(t0)))

    def rec_of(v, s, c0):
        return next(r for vv, r in per if vv == v and r["seg"] == s and r["off"] == c0)

    def check_full(job):
        s, c0 = job
        m = min(C, sizes[s] - c0)
        st = synth.segment_versions(m, wb[s], seed, s, [0, 1, 2], f, start=c0, threads=4)
        bad = []
        for v in (1, 2):
            rc, exp = tco.encode([st[v - 1].copy()], [st[v]], tile_words=T, chunk_words=C, advance_ref=True,
                                 version=v, ref_version=v - 1, index_mode=True)
            exp = exp.copy()
            exp[12:16] = np.frombuffer(np.uint32(s).tobytes(), np.uint8)  # the one-segment oracle run
            exp[16:24] = np.frombuffer(np.uint64(c0).tobytes(), np.uint8)  # names segment 0, offset 0
            r = rec_of(v, s, c0)
            buf = host[v - 1]
            if rc != 0 or not np.array_equal(buf[r["pos"]: r["pos"] + r["total"]], exp):
                bad.append((v, s, c0))
        return bad

    def check_window(job):
        s, c0, t0 = job
        a = c0 + t0 * T
        st = synth.segment_versions(256 * T, wb[s], seed, s, [0, 1, 2], f, start=a, threads=1)
        bad = []
        for v in (1, 2):
            rc, exp = tco.encode([st[v - 1].copy()], [st[v]], tile_words=T, chunk_words=C, advance_ref=True,
                                 version=v, ref_version=v - 1, index_mode=True)
            e = _idx_record(exp, 0)
            r = rec_of(v, s, c0)
            k0, k1 = int(r["toff"][t0]), int(r["toff"][t0 + 256])
            ok = rc == 0 and np.array_equal(r["toff"][t0: t0 + 257] - np.uint32(k0), e["toff"]) \
                and np.array_equal(r["idx"][k0:k1], e["idx"]) and np.array_equal(r["vals"][k0:k1], e["vals"])
            if not ok:
                bad.append((v, s, c0, t0))
        return bad

    with ThreadPoolExecutor(4) as ex:
        bad = sum(ex.map(check_full, full_jobs), []) + sum(ex.map(check_window, win_jobs), [])
    assert not bad, f"records differ from the oracle: {bad[:8]}"
    assert len(full_jobs) == 8 and len(win_jobs) == 8 * (sum(-(-n // C) for n in sizes) - 8)
    # the chain folds onto the base bit-exactly (index-mode chain, default strategy)
    for s, t in enumerate(ref):
        tc.synth_base(t, seed, s)
    tc.diff_apply(ctx, ref, 0, [o for o, _ in recs], [n for _, n in recs])
    ctx.check()
    assert all(torch.equal(a, b) for a, b in zip(ref, cur))
    ctx.close()


def test_record_overflow_forces_a_base_and_the_chain_recovers():
    """R20: record slots sized for a sparse job; a dense step's record does not fit — refused on the
    device, so the next save is a base (§3.1 base stream): the reference becomes the
    live state, Tier-1 holds the new base, the neighbour (ring of one) receives it in paced chunks.
    The chain continues from it and recover() after a GPU failure lands on the chain head."""
    sizes, wb, seed = [60001, 60001, 60001, 60001], [2, 4, 4, 4], synth.SEED0 + 13
    live = _dev_state(sizes, wb, seed, 0, 0.0)
    ck = Checkpointer(live, tier2="push", rec_cap=64 << 10, t2_slots=4, chunk_words=1 << 15, base_interval=4)
    small = ck.rec_cap
    expect = [to_np(t) for t in live]
    fs = {1: 0.001, 2: 0.9, 3: 0.001, 4: 0.002, 5: 0.001}
    for v in range(1, 6):
        for s, t in enumerate(live):
            tc.synth_step(t, seed, s, v, synth.p53_of(fs[v]))
        expect = [synth.step(e, seed, s, v, fs[v]) for s, e in enumerate(expect)]
        ck.save_step(v)
    ck.flush()
    ck.base_rep.flush(99)
    torch.cuda.synchronize()
    assert small < sum(n * w for n, w in zip(sizes, wb)) * 0.9  # the dense record cannot fit
    # v2 overflowed (found when save 3 finished it; v3, linked to v2, is dropped), so save 4 is a
    # base: the chain restarts at 4
    assert ck.chain.base_version == 4 and [e.version for e in ck.chain.entries] == [5]
    assert ck.base_rep.committed_version() == 4
    ck.drop_tier("hbm")
    assert ck.recover(batch=5) == 5
    assert all(np.array_equal(to_np(a), b) for a, b in zip(live, expect))
    ck.close()
