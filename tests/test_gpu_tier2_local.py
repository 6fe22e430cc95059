"""GPU, one device: the Tier-2 paths exercised where the
round-end GPU run can see them — the ring of one.

- tc_push_peer / tc_diff_encode_push + tc_peer_wait into a slot and mailbox allocated with
  tc_ipc_alloc on the same GPU (the receiver's side of the NVLink push, §3.1 ring
  mapping, §3.2: the size travels in the mailbox): content, alternating slots / versions,
  capacity refusal (nothing written, receiver sees TC_ERR_CAPACITY), lengths that are not a
  multiple of 16 bytes;
- tc_replicate_peer over a one-rank NCCL communicator (P = 1: the replica is the local record);
- BaseReplicator with world = 1: paced chunks, all-or-nothing commit, the committed base intact
  while the next one streams into the other slot, sync flush on spillover.
The multi-GPU versions of these checks are tests/test_gpu_multi.py (>= 2 GPUs)."""
import numpy as np
import pytest

import synth

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a GPU", allow_module_level=True)

from paper_2605_17821_b200 import tc  # noqa: E402
from paper_2605_17821_b200.checkpoint import BaseReplicator  # noqa: E402
from tests.gpu_util import to_dev, to_np  # noqa: E402

SIZES, WB = [70001, 50000, 33333], [2, 4, 4]


@pytest.fixture(scope="module")
def ctx():
    c = tc.Ctx(0)
    yield c
    c.close()


def _shard(v, f, seed=synth.SEED0 + 11):
    return synth.state(SIZES, WB, seed, v, f)


@pytest.mark.parametrize("ctas", [0, 1, 16, 148])
def test_encode_push_into_local_slot(ctx, tco, ctas):
    ctx.set_push_ctas(ctas)
    slot_cap = tc.diff_bound(SIZES, WB)
    slots = [tc.IpcBuffer(slot_cap) for _ in range(2)]
    mail = [tc.IpcBuffer(16) for _ in range(2)]
    s = torch.cuda.Stream()
    states = [_shard(v, f) for v, f in ((0, 0.0), (1, 0.01), (2, 0.5), (3, 1.0))]
    ref = [to_dev(a) for a in states[0]]
    base = [to_dev(a) for a in states[0]]
    ref_o = [a.copy() for a in states[0]]
    for v in (1, 2, 3):
        k = v % 2
        index_mode = v == 1
        cur = [to_dev(a) for a in states[v]]
        out = torch.zeros(slot_cap, dtype=torch.uint8, device="cuda")
        ob = torch.zeros(1, dtype=torch.int64, device="cuda")
        got = torch.zeros(1, dtype=torch.int64, device="cuda")
        tc.diff_encode_push(ctx, ref, cur, out, ob, v, v - 1, slots[k], slot_cap, mail[k], stream=s,
                            index_mode=index_mode)
        tc.peer_wait(ctx, mail[k], v, got, stream=s)
        ctx.check(s)
        n = int(got.item())
        rc, exp = tco.encode(ref_o, states[v], version=v, ref_version=v - 1, index_mode=index_mode)
        assert rc == 0 and n == int(ob.item()) == exp.size
        assert np.array_equal(slots[k].tensor[:n].cpu().numpy(), exp), "pushed record != oracle record"
        mw = mail[k].tensor.view(torch.int64).cpu().tolist()
        assert mw == [n, v]
        # the receiver folds its replica onto the sender's state of v - 1 (Tier-2 restore)
        tc.diff_apply(ctx, base, v - 1, [slots[k].tensor], [n], stream=s)
        ctx.check(s)
        assert all(np.array_equal(to_np(a), b) for a, b in zip(base, states[v]))
    ctx.set_push_ctas(0)
    for b in slots + mail:
        b.free()


@pytest.mark.parametrize("nbytes", [0, 1, 15, 16, 17, 4095, 1 << 20, (1 << 20) + 7, 3 * (1 << 22) + 13])
def test_push_any_length(ctx, nbytes):
    """Every byte of the payload arrives, nothing after it is written (tail handling)."""
    src = torch.randint(0, 256, (max(16, nbytes + 32),), dtype=torch.uint8, device="cuda")
    slot = tc.IpcBuffer(nbytes + 64)
    slot.tensor.fill_(0xEE)
    mail = tc.IpcBuffer(16)
    nb = torch.tensor([nbytes], dtype=torch.int64, device="cuda")
    s = torch.cuda.Stream()
    tc.push_peer(ctx, src, nb, slot, nbytes + 64, mail, 5, stream=s)
    got = torch.zeros(1, dtype=torch.int64, device="cuda")
    tc.peer_wait(ctx, mail, 5, got, stream=s)
    ctx.check(s)
    assert int(got.item()) == nbytes
    assert torch.equal(slot.tensor[:nbytes], src[:nbytes])
    assert bool((slot.tensor[nbytes:] == 0xEE).all())
    slot.free()
    mail.free()


def test_push_capacity_refused(ctx):
    """A record larger than the slot is not copied; the receiver's wait reports CAPACITY, and a
    later push that fits works on the same mailbox."""
    src = torch.randint(0, 256, (4096,), dtype=torch.uint8, device="cuda")
    slot = tc.IpcBuffer(1024)
    slot.tensor.fill_(0x11)
    mail = tc.IpcBuffer(16)
    s = torch.cuda.Stream()
    nb = torch.tensor([4096], dtype=torch.int64, device="cuda")
    tc.push_peer(ctx, src, nb, slot, 1024, mail, 1, stream=s)
    got = torch.full((1,), -5, dtype=torch.int64, device="cuda")
    tc.peer_wait(ctx, mail, 1, got, stream=s)
    assert ctx.check_status(s) == tc.ERR_CAPACITY
    assert int(got.item()) == 0
    assert bool((slot.tensor == 0x11).all()), "a refused push wrote into the slot"
    nb.fill_(1000)
    tc.push_peer(ctx, src, nb, slot, 1024, mail, 2, stream=s)
    tc.peer_wait(ctx, mail, 2, got, stream=s)
    ctx.check(s)
    assert int(got.item()) == 1000 and torch.equal(slot.tensor[:1000], src[:1000])
    slot.free()
    mail.free()


def test_push_argument_errors(ctx):
    src = torch.zeros(64, dtype=torch.uint8, device="cuda")
    nb = torch.zeros(1, dtype=torch.int64, device="cuda")
    mail = tc.IpcBuffer(16)
    with pytest.raises(tc.TcError):
        tc.push_peer(ctx, src[1:], nb, mail, 16, mail, 1)      # misaligned source
    with pytest.raises(tc.TcError):
        tc.push_peer(ctx, src, nb, mail, 16, mail, 0)          # version 0
    with pytest.raises(tc.TcError):
        tc.peer_wait(ctx, mail, 0)
    mail.free()


def test_replicate_peer_ring_of_one(ctx, tco):
    """tc_replicate_peer with P = 1: size read on the comm stream, the local record copied into
    recv, recv_bytes = its length; a recv buffer that is too small -> CAPACITY, nothing copied."""
    comm = tc.Comm(0, 1, 0)
    states = [_shard(0, 0.0), _shard(1, 0.02)]
    ref = [to_dev(a) for a in states[0]]
    cur = [to_dev(a) for a in states[1]]
    cap = tc.diff_bound(SIZES, WB)
    out = torch.zeros(cap, dtype=torch.uint8, device="cuda")
    ob = torch.zeros(1, dtype=torch.int64, device="cuda")
    s = torch.cuda.Stream()
    tc.diff_encode(ctx, ref, cur, out, ob, 1, 0, stream=s)
    recv = torch.zeros(cap, dtype=torch.uint8, device="cuda")
    n = comm.replicate_peer(out, ob, recv, tc.TO_NEXT, stream=s)
    ctx.check(s)
    rc, exp = tco.encode([a.copy() for a in states[0]], states[1], version=1, ref_version=0)
    assert n == exp.size and np.array_equal(recv[:n].cpu().numpy(), exp)
    small = torch.full((n // 2,), 7, dtype=torch.uint8, device="cuda")
    with pytest.raises(tc.TcError) as e:
        comm.replicate_peer(out, ob, small, tc.TO_PREV, stream=s)
    assert e.value.status == tc.ERR_CAPACITY
    s.synchronize()
    assert bool((small == 7).all())
    comm.close()


def test_base_replicator_ring_of_one():
    """Paced base replication (§3.2; SPEC.md:291 all-or-nothing) with world = 1."""
    dev = torch.device("cuda", 0)
    g = torch.Generator().manual_seed(3)

    def shard(seed):
        g.manual_seed(seed)
        return [torch.randint(-32768, 32767, (300_001,), dtype=torch.int16, generator=g).to(dev),
                torch.randint(-2**31, 2**31 - 1, (250_003,), dtype=torch.int32, generator=g).to(dev)]

    def flat(segs):
        return torch.cat([t.view(torch.uint8).reshape(-1) for t in segs])

    b1, b2, b3 = shard(1), shard(2), shard(3)
    n = flat(b1).numel()
    rep = BaseReplicator(n, 0, 1, 0)
    assert rep.committed_version() == -1 and rep.received().numel() == 0
    plan = rep.intercept(b1, version=10, interval=10, margin=2, cap=1 << 30)
    assert not plan.spillover and plan.iters == 8
    for it in range(1, 11):
        rep.pump(it)
        rep.s.synchronize()
        assert rep.committed_version() == (10 if it >= plan.iters else -1), it
    assert torch.equal(rep.received(), flat(b1))
    assert torch.equal(rep.host.tensor[:n], flat(b1).cpu())
    # base 2 spills over (small chunk cap): while it streams, base 1 stays committed and intact
    plan = rep.intercept(b2, version=20, interval=10, margin=2, cap=64 << 10)
    assert plan.spillover
    for it in range(11, 19):
        rep.pump(it)
        rep.s.synchronize()
        assert rep.committed_version() == 10
        assert torch.equal(rep.received(), flat(b1)), "committed base torn by the next one"
    rep.intercept(b3, version=30, interval=10, margin=2, cap=1 << 30)  # flushes base 2 first
    rep.s.synchronize()
    assert any(k == "sync_flush" for _, k, _ in rep.log)
    assert rep.committed_version() == 20 and torch.equal(rep.received(), flat(b2))
    for it in range(21, 31):
        rep.pump(it)
    rep.s.synchronize()
    assert rep.committed_version() == 30 and torch.equal(rep.received(), flat(b3))
    with pytest.raises(ValueError):
        rep.intercept(b1[:1], version=40, interval=10)
    rep.ctx.check(rep.s)
    rep.close()


@pytest.mark.parametrize("index_mode", [False, True])
def test_fused_encode_push_capacity_and_ranges(ctx, tco, index_mode):
    """tc_diff_encode_push (the encoder writes the record into the peer slot itself): a slot too
    small for the record -> the mailbox reports refusal (tc_peer_wait: CAPACITY) while the local
    record is still exact; several chunks and tile sizes land byte-exact in a slot that fits."""
    sizes, wb = [70001, 9000, 40000], [4, 2, 4]
    states = [synth.state(sizes, wb, 91, v, 0.2) for v in range(3)]
    for T, C, ok in ((4096, 1 << 28, False), (256, 8192, True), (1024, 4096 * 3, True)):
        ref = [to_dev(a) for a in states[0]]
        cur = [to_dev(a) for a in states[1]]
        rc, exp = tco.encode([a.copy() for a in states[0]], states[1], tile_words=T, chunk_words=C, version=1,
                             ref_version=0, index_mode=index_mode)
        cap = tc.diff_bound(sizes, wb, T, C, index_mode)
        slot_cap = exp.size if ok else exp.size // 2
        slot = tc.IpcBuffer(max(16, slot_cap))
        mail = tc.IpcBuffer(16)
        out = torch.zeros(cap, dtype=torch.uint8, device="cuda")
        ob = torch.zeros(1, dtype=torch.int64, device="cuda")
        got = torch.zeros(1, dtype=torch.int64, device="cuda")
        s = torch.cuda.Stream()
        tc.diff_encode_push(ctx, ref, cur, out, ob, 1, 0, slot, slot_cap, mail, T, C, True, stream=s,
                            index_mode=index_mode)
        tc.peer_wait(ctx, mail, 1, got, stream=s)
        rc = ctx.check_status(s)
        n = int(ob.item())
        assert n == exp.size and np.array_equal(out[:n].cpu().numpy(), exp)
        if ok:
            assert rc == tc.OK and int(got.item()) == n
            assert np.array_equal(slot.tensor[:n].cpu().numpy(), exp)
        else:
            assert rc == tc.ERR_CAPACITY and int(got.item()) == 0
        slot.free()
        mail.free()


def test_fused_encode_push_full_records(ctx, tco):
    """The fused Tier-2 emit of full records (kernel F writes both copies, publishes the mailbox)."""
    states = [_shard(0, 0.0), _shard(1, 1.0)]
    ref = [to_dev(a) for a in states[0]]
    cur = [to_dev(a) for a in states[1]]
    rc, exp = tco.encode([a.copy() for a in states[0]], states[1], version=1, ref_version=0, full=True)
    cap = tc.diff_bound(SIZES, WB, full=True)
    slot, mail = tc.IpcBuffer(cap), tc.IpcBuffer(16)
    out = torch.zeros(cap, dtype=torch.uint8, device="cuda")
    ob = torch.zeros(1, dtype=torch.int64, device="cuda")
    got = torch.zeros(1, dtype=torch.int64, device="cuda")
    s = torch.cuda.Stream()
    tc.diff_encode_push(ctx, ref, cur, out, ob, 1, 0, slot, cap, mail, stream=s, full=True)
    tc.peer_wait(ctx, mail, 1, got, stream=s)
    ctx.check(s)
    n = int(got.item())
    assert n == exp.size == int(ob.item())
    assert np.array_equal(out[:n].cpu().numpy(), exp) and np.array_equal(slot.tensor[:n].cpu().numpy(), exp)
    slot.free()
    mail.free()


@pytest.mark.parametrize("fmt", ["mask", "index", "full"])
def test_fused_encode_emit_into_mapped_host_memory(ctx, tco, fmt):
    """The fused emit with a page-locked mapped host buffer as the destination (the Tier-1 emit
    option, tools/t1_emit_bench.py): host bytes == oracle record, host mailbox == {n, version}."""
    kw = {"index_mode": fmt == "index", "full": fmt == "full"}
    states = [_shard(0, 0.0), _shard(1, 0.02)]
    ref = [to_dev(a) for a in states[0]]
    cur = [to_dev(a) for a in states[1]]
    rc, exp = tco.encode([a.copy() for a in states[0]], states[1], version=1, ref_version=0, **kw)
    assert rc == 0
    cap = tc.diff_bound(SIZES, WB, **kw)
    host, mail = tc.HostBuffer(cap), tc.HostBuffer(16)
    mail.tensor.zero_()
    out = torch.zeros(cap, dtype=torch.uint8, device="cuda")
    ob = torch.zeros(1, dtype=torch.int64, device="cuda")
    s = torch.cuda.Stream()
    tc.diff_encode_push(ctx, ref, cur, out, ob, 1, 0, host, cap, mail, stream=s, **kw)
    ctx.check(s)
    n = exp.size
    assert int(ob.item()) == n
    assert mail.tensor.view(torch.int64).tolist() == [n, 1]
    assert np.array_equal(host.tensor[:n].numpy(), exp)
    host.free()
    mail.free()
