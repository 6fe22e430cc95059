"""Host-side logic of the multi-rank path on CPU: world-size-2 gloo process group (consensus MIN,
ring mapping, unique-id broadcast shape) and the version-chain bookkeeping."""
import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2605_17821_b200.checkpoint import DiffChain, consensus, ring_peers


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        # every rank can recover a different newest base / chain end: consensus takes the MIN
        base = [100, 150][rank]
        end = [137, 149][rank]
        got = consensus(base, end)
        nxt, prv = ring_peers(rank, world)
        # the ring is a permutation: my next's prev is me
        peers = [None] * world
        dist.all_gather_object(peers, (nxt, prv))
        ring_ok = all(peers[peers[r][0]][1] == r for r in range(world))
        # the 128-byte NCCL unique id travels over the process group as uint8 (Comm.__init__)
        uid = torch.arange(128, dtype=torch.uint8) if rank == 0 else torch.zeros(128, dtype=torch.uint8)
        dist.broadcast(uid, src=0)
        q.put((rank, got, ring_ok, bool((uid == torch.arange(128, dtype=torch.uint8)).all())))
    finally:
        dist.destroy_process_group()


def test_consensus_and_ring_world2():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, got, ring_ok, uid_ok in res:
        assert got == (100, 137)
        assert ring_ok and uid_ok


def test_ring_peers():
    assert ring_peers(0, 1) == (0, 0)
    assert ring_peers(0, 2) == (1, 1)
    assert ring_peers(3, 4) == (0, 2)
    with pytest.raises(ValueError):
        ring_peers(4, 4)


def test_consensus_single_process():
    assert consensus(7, 9) == (7, 9)


def test_diff_chain_links_batches_reclaim():
    c = DiffChain(base_version=50)
    for v in range(51, 64):
        c.append(v, v - 1, 1000 + v, tiers=("t1", "t2") if v < 60 else ("t1",))
    with pytest.raises(ValueError):
        c.append(70, 68, 1)  # gap
    with pytest.raises(ValueError):
        c.append(63, 63, 1)  # version must advance
    assert c.head == 63
    assert c.replay_end() == 63 and c.replay_end("t2") == 59
    b = c.batches(5)
    assert [len(x) for x in b] == [5, 5, 3] and b[0][0].version == 51 and b[-1][-1].version == 63
    assert [len(x) for x in c.batches(5, upto=57)] == [5, 2]
    gone = c.reclaim(55)
    assert [e.version for e in gone] == [51, 52, 53, 54, 55]
    assert c.base_version == 55 and c.entries[0].version == 56
    with pytest.raises(ValueError):
        c.reclaim(40)


# ------------------------------------------------------ NEXT row 4: paced base replication ----
def test_plan_chunks_spec_examples():
    """1 GiB, I = 50, s = 5, C = 256 MiB -> ceil(1 GiB / 45) per iteration over 45
    iterations, no spillover; 0 bytes -> no chunks; 20 GiB, I = 10, s = 2 -> capped at 256 MiB,
    80 iterations, spillover."""
    from paper_2605_17821_b200.checkpoint import MiB, plan_chunks

    p = plan_chunks(1 << 30, 50, 5, 256 * MiB)
    assert p.chunk_bytes == -(-(1 << 30) // 45) and p.iters == 45 and not p.spillover
    assert round(p.chunk_bytes / MiB) == 23
    p = plan_chunks(0, 50, 5)
    assert p.chunk_bytes == 0 and p.iters == 0 and not p.spillover
    p = plan_chunks(20 << 30, 10, 2, 256 * MiB)
    assert p.chunk_bytes == 256 * MiB and p.iters == 80 and p.spillover
    assert plan_chunks(1 << 20, 50).margin == 5  # default s = ceil(0.1 I)


def test_plan_chunks_invariants():
    import random

    from paper_2605_17821_b200.checkpoint import plan_chunks

    rng = random.Random(3)
    for _ in range(2000):
        total, interval = rng.randrange(0, 1 << 40), rng.randrange(1, 500)
        margin, cap = rng.randrange(0, interval + 3), rng.randrange(1, 1 << 30)
        p = plan_chunks(total, interval, margin, cap)
        if total == 0:
            assert p.iters == 0
            continue
        avail = max(1, interval - margin)
        assert p.chunk_bytes == min(cap, -(-total // avail))
        assert p.iters == -(-total // p.chunk_bytes) and p.chunk_bytes * p.iters >= total
        assert p.spillover == (p.iters > avail)


def test_plan_loading_cascade():
    from paper_2605_17821_b200.checkpoint import plan_loading

    assert plan_loading(True, True) == "t1" and plan_loading(True, False) == "t1"
    assert plan_loading(False, True) == "t2" and plan_loading(False, False) == "t3"


class _FakeBuf:
    def __init__(self, n):
        self.nbytes = n


def test_host_arena_ring_allocation():
    """The Tier-1 arena (checkpoint.HostArena) is a FIFO ring: entries are 16-byte padded, placed
    after the newest, wrap to offset 0 when the tail is full, never overlap a live entry, and the
    space of reclaimed (oldest) entries is reused."""
    from paper_2605_17821_b200.checkpoint import HostArena

    a = HostArena(1000, buffer=_FakeBuf(1000))
    assert a.alloc("r1", 300) == 0
    assert a.alloc("r2", 301) == 304          # padded to 16
    assert a.alloc("r3", 400) is None         # 304 + 304 + 400 > 1000 and no room at the front
    a.release(lambda k: k != "r1")            # reclaim r1: [0, 304) is free
    assert a.alloc("r3", 200) == 608          # still fits after r2
    assert a.alloc("r4", 250) == 0            # wraps into the reclaimed front
    assert a.alloc("r5", 100) is None         # [256, 304) is too small; r2 and r3 are live
    a.release(lambda k: k not in ("r2", "r3"))
    assert a.alloc("r5", 100) == 256          # after r4, in the freed middle
    live = sorted((o, o + n) for _, o, n in a.q)
    assert all(b0 <= a1 for (a0, b0), (a1, b1) in zip(live, live[1:])), live
    a.clear()
    assert a.alloc("x", 992) == 0 and a.alloc("y", 1) is None  # 1000 bytes hold 992 padded
