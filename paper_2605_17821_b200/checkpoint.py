"""Save / retrieve / reclaim lifecycle around libtc (§1; §3.1).

Host-side bookkeeping only — every byte of state is encoded, staged, replicated and folded by
libtc (tc.py); nothing here computes on the data.

    ring_peers        the Tier-2 ring mapping r -> (r+1) mod P (§3.1)
    consensus         global MIN of (latest base version, replay end) (§3.3)
    DiffChain         the version chain of one rank: links, N-record batches, watermark reclaim
                      (PAPER.md:226 version = iteration; P:207 batching N; P:306-310 watermark)
    Checkpointer      per-rank save_step (encode -> Tier-1 D2H -> Tier-2 ring) and restore
                      (fetch from Tier-1 / Tier-2, then one fold of the chain) on libtc
    plan_chunks       paced base replication plan (§3.2)
    BaseReplicator    a base checkpoint intercepted once in memory, staged to Tier-1, replicated
                      to the ring neighbour in paced chunks over NVLink stores, committed
                      all-or-nothing; sync flush on spillover
    plan_loading      the retrieval cascade Tier-1 -> Tier-2 peer (§3.3)
"""
from __future__ import annotations

from dataclasses import dataclass, field

import torch


# --------------------------------------------------------------------- ring + consensus ----
def bind_local_numa(device: int) -> str:
    """Bind this process to the CPUs of GPU `device`'s NUMA node, so the pinned Tier-1 staging
    buffers allocated afterwards (first touch) live in host memory local to the GPU's PCIe root
    ("local volatile memory", §1).  Reads the PCI bus id from torch and the node's
    CPU list from sysfs; a no-op (with the reason returned) where either is unavailable."""
    import os

    try:
        p = torch.cuda.get_device_properties(device)
        bus = f"{p.pci_domain_id:04x}:{p.pci_bus_id:02x}:{p.pci_device_id:02x}.0"
        base = f"/sys/bus/pci/devices/{bus}"
        node = int(open(f"{base}/numa_node").read().strip())
        cpus_txt = open(f"{base}/local_cpulist").read().strip()
    except (OSError, ValueError, AttributeError, RuntimeError) as e:
        return f"no binding ({type(e).__name__})"
    cpus = set()
    for part in cpus_txt.split(","):
        a, _, b = part.partition("-")
        cpus.update(range(int(a), int(b or a) + 1))
    cpus &= os.sched_getaffinity(0) if hasattr(os, "sched_getaffinity") else cpus
    if not cpus:
        return f"no binding (GPU {bus} on node {node}: no allowed CPU in {cpus_txt})"
    os.sched_setaffinity(0, cpus)
    return f"GPU {bus} NUMA node {node}: bound to CPUs {cpus_txt}"


def ring_peers(rank: int, world: int) -> tuple[int, int]:
    """(next, prev): rank r replicates to (r+1) mod P and holds the replica of (r-1) mod P."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank / world")
    return (rank + 1) % world, (rank - 1 + world) % world


def consensus(base_version: int, replay_end: int, group=None) -> tuple[int, int]:
    """Global consensus on the latest checkpoint (§3.3): every rank offers
    the highest base version it can recover and the end of its recoverable diff chain; the job
    resumes from the MIN of each (one tiny all_reduce, off the bandwidth path)."""
    import torch.distributed as dist

    t = torch.tensor([base_version, replay_end], dtype=torch.int64)
    if dist.is_available() and dist.is_initialized():
        if dist.get_backend(group) == "nccl":
            t = t.cuda()
        dist.all_reduce(t, op=dist.ReduceOp.MIN, group=group)
    return int(t[0].item()), int(t[1].item())


# ----------------------------------------------------------------------------- chain ------
@dataclass
class DiffEntry:
    version: int
    ref_version: int
    nbytes: int
    tiers: set = field(default_factory=set)  # {"t1", "t2"}


class DiffChain:
    """One rank's differential chain on top of a base version.

    - `append` enforces the link rule of the record headers (ref_version == previous version,
      version > ref_version; "gap in batch chain -> protocol error");
    - `batches(n)` groups the chain into runs of N consecutive records (N = 5
      default) — one `tc_diff_apply` call per batch;
    - `reclaim(watermark)` drops every record whose version <= watermark and advances the base
      (§3.4: volatile histories are reclaimed once a newer base is safe)."""

    def __init__(self, base_version: int):
        self.base_version = base_version
        self.entries: list[DiffEntry] = []

    @property
    def head(self) -> int:
        return self.entries[-1].version if self.entries else self.base_version

    def append(self, version: int, ref_version: int, nbytes: int, tiers=("t1",)) -> DiffEntry:
        if ref_version != self.head or version <= ref_version:
            raise ValueError(f"chain gap: record {ref_version}->{version} after head {self.head}")
        e = DiffEntry(version, ref_version, nbytes, set(tiers))
        self.entries.append(e)
        return e

    def replay_end(self, tier: str | None = None) -> int:
        """Latest version reachable from the base through records available (on `tier`)."""
        v = self.base_version
        for e in self.entries:
            if tier is not None and tier not in e.tiers:
                break
            v = e.version
        return v

    def batches(self, n: int, upto: int | None = None):
        sel = [e for e in self.entries if upto is None or e.version <= upto]
        return [sel[i: i + n] for i in range(0, len(sel), n)]

    def reclaim(self, watermark: int) -> list[DiffEntry]:
        if watermark < self.base_version:
            raise ValueError("watermark must be monotone")
        gone = [e for e in self.entries if e.version <= watermark]
        self.entries = [e for e in self.entries if e.version > watermark]
        self.base_version = watermark
        return gone


# ----------------------------------------------------------------------- checkpointer -----
class Checkpointer:
    """Per-rank save / restore of a shard through libtc (GPU only).

    segments: list of CUDA tensors (the live training state: 16-bit weights, fp32 master/m/v).
    The reference copy (`ref`) is owned here and advanced by every encode (reading R2)."""

    def __init__(self, segments, rank: int = 0, world: int = 1, comm=None, ring_slots: int = 8,
                 tile_words: int = 4096, chunk_words: int = 1 << 28):
        from . import tc

        self.tc = tc
        self.rank, self.world, self.comm = rank, world, comm
        self.segments = segments
        self.device = segments[0].device
        self.ctx = tc.Ctx(self.device.index)
        self.T, self.C = tile_words, chunk_words
        self.ref = [s.clone() for s in segments]  # the base / reference (version 0)
        self.cap = tc.diff_bound([s.numel() for s in segments], [s.element_size() for s in segments],
                                 tile_words, chunk_words)
        self.chain = DiffChain(0)
        self.s_copy = torch.cuda.Stream(self.device)
        self.s_comm = torch.cuda.Stream(self.device)
        self.out_len = tc.HostBuffer(8 * ring_slots)
        self.t1: dict[int, object] = {}   # version -> HostBuffer (Tier-1, local host memory)
        self.t2: dict[int, tuple] = {}    # version -> (device tensor, nbytes) replica of prev rank
        self.dev_rec: dict[int, torch.Tensor] = {}

    def save_step(self, version: int, stream=None) -> int:
        """Encode the current state as the differential of `version` against the chain head,
        stage it to Tier-1 and replicate it to the ring neighbour (Tier-2)."""
        tc = self.tc
        s = stream or torch.cuda.current_stream(self.device)
        ref_version = self.chain.head
        out = torch.empty(self.cap, dtype=torch.uint8, device=self.device)
        ob = self.out_len.view(torch.int64)[version % (self.out_len.nbytes // 8):][:1]
        tc.diff_encode(self.ctx, self.ref, self.segments, out, ob, version, ref_version, self.T, self.C,
                       True, stream=s)
        done = torch.cuda.Event()
        done.record(s)
        done.synchronize()
        self.ctx.check(s)
        n = int(ob.item())
        host = tc.HostBuffer(n)
        self.s_copy.wait_event(done)
        tc.stage_host(host, out, n, tc.D2H, stream=self.s_copy)
        tiers = {"t1"}
        if self.comm is not None and self.world > 1:
            self.s_comm.wait_event(done)
            recv = torch.empty(self.cap, dtype=torch.uint8, device=self.device)
            got = self.comm.replicate_peer(out, ob, recv, tc.TO_NEXT, stream=self.s_comm)
            self.t2[version] = (recv, got)
            tiers.add("t2")
        self.t1[version] = host
        self.dev_rec[version] = out
        self.chain.append(version, ref_version, n, tiers)
        return n

    def restore(self, base, upto: int | None = None, source: str = "t1", batch: int = 8, stream=None):
        """Rebuild the state at `upto` (default: chain head) onto `base` (list of CUDA tensors
        holding the base version): fetch the records from Tier-1 (H2D) and fold them in batches
        of `batch` records, oldest first (PAPER.md:283 fused multi-step replay)."""
        tc = self.tc
        s = stream or torch.cuda.current_stream(self.device)
        ver = self.chain.base_version
        for b in self.chain.batches(batch, upto):
            recs, lens = [], []
            for e in b:
                if source == "t1":
                    d = torch.empty(max(e.nbytes, 16), dtype=torch.uint8, device=self.device)
                    tc.stage_host(d, self.t1[e.version], e.nbytes, tc.H2D, stream=s)
                else:
                    d = self.dev_rec[e.version]
                recs.append(d)
                lens.append(e.nbytes)
            tc.diff_apply(self.ctx, base, ver, recs, lens, stream=s)
            ver = b[-1].version
        self.ctx.check(s)
        return ver

    def reclaim(self, watermark: int):
        for e in self.chain.reclaim(watermark):
            self.t1.pop(e.version, None)
            self.t2.pop(e.version, None)
            self.dev_rec.pop(e.version, None)


# ------------------------------------------------------- NEXT row 4: paced base replication ----
MiB = 1 << 20


@dataclass
class ChunkPlan:
    """Paced replication of one base checkpoint (SPEC.md:233 ChunkPlan; §3.2 "evenly
    divides this volume across the available training iterations ... reserving a brief safety
    margin ... caps the maximum chunk size")."""
    total_bytes: int
    interval: int        # I: iterations between bases
    margin: int          # s: safety margin (iterations)
    cap: int             # C: chunk cap (bytes)
    chunk_bytes: int
    iters: int           # iterations the transfer is scheduled over
    spillover: bool      # more iterations than I - s: the rest is flushed synchronously


def plan_chunks(total_bytes: int, interval: int, margin: int | None = None, cap: int = 256 * MiB) -> ChunkPlan:
    """chunk = min(C, ceil(total / max(1, I - s))); iterations = ceil(total / chunk); spillover iff
    iterations > I - s.  s defaults to ceil(0.1 I)."""
    if interval < 1 or cap < 1 or total_bytes < 0:
        raise ValueError("interval >= 1, cap >= 1, total >= 0")
    if margin is None:
        margin = -(-interval // 10)
    avail = max(1, interval - margin)
    if total_bytes == 0:
        return ChunkPlan(0, interval, margin, cap, 0, 0, False)
    chunk = min(cap, -(-total_bytes // avail))
    iters = -(-total_bytes // chunk)
    return ChunkPlan(total_bytes, interval, margin, cap, chunk, iters, iters > avail)


class BaseReplicator:
    """One rank's base stream.  `intercept` serializes the shard once
    into a flat device payload (§3.2 "in-memory byte payloads", no write-then-read)
    and stages it to Tier-1 (pinned host); `pump` (once per training iteration) pushes the next
    paced chunk into the ring neighbour's staging buffer with NVLink stores (tc_push_peer); the
    replica becomes visible only when every byte has arrived — all-or-nothing;
    `flush` sends the remainder at once (the sync flush on spillover).

    The receiver keeps TWO staging slots, sized by the previous rank's shard (the rank it receives
    from).  Successive bases alternate slots, and the commit mailbox names the slot:
    {bytes, 2·version + slot}.  While base k+1 streams into one slot, the commit still points at
    base k in the other, so a recovering rank never reads a torn replica.  The sender checks on
    the host that its payload fits the neighbour's slot before it pushes anything.
    Collective at construction (IPC handle exchange over torch.distributed); one per rank.  With
    world == 1 the ring of one is this GPU itself: no handle exchange, local slots."""

    def __init__(self, shard_bytes: int, rank: int, world: int, device: int, stream=None):
        from . import tc

        self.tc = tc
        self.n = int(shard_bytes)
        self.rank, self.world = rank, world
        self.dev = torch.device("cuda", device)
        self.s = stream or torch.cuda.Stream(self.dev)
        self.ctx = tc.Ctx(device)
        self.ctx.set_push_ctas(16)
        self.payload = torch.empty(_pad16(self.n), dtype=torch.uint8, device=self.dev)
        self.host = tc.HostBuffer(max(1, self.n))
        if world > 1:
            import torch.distributed as dist

            sizes = [None] * world
            dist.all_gather_object(sizes, self.n)
        else:
            sizes = [self.n]
        nxt, prv = ring_peers(rank, world)
        self.prev_n, self.peer_n = int(sizes[prv]), int(sizes[nxt])
        # this GPU receives the previous rank's bases here (two slots), plus the mailboxes
        self.stage = [tc.IpcBuffer(_pad16(self.prev_n)) for _ in range(2)]
        self.progress = tc.IpcBuffer(16)
        self.commit = tc.IpcBuffer(16)
        if world > 1:
            hs = [None] * world
            dist.all_gather_object(hs, [b.handle for b in self.stage] + [self.progress.handle, self.commit.handle])
            nx = hs[nxt]
            self._maps = [tc.PeerMapping(nx[0], _pad16(self.peer_n)), tc.PeerMapping(nx[1], _pad16(self.peer_n)),
                          tc.PeerMapping(nx[2], 16), tc.PeerMapping(nx[3], 16)]
            self.peer_stage, self.peer_progress, self.peer_commit = self._maps[:2], self._maps[2], self._maps[3]
        else:  # the ring of one: the neighbour is this GPU
            self._maps = []
            self.peer_stage, self.peer_progress, self.peer_commit = self.stage, self.progress, self.commit
        self.len_dev = torch.zeros(1, dtype=torch.int64, device=self.dev)
        self.zero_dev = torch.zeros(1, dtype=torch.int64, device=self.dev)
        self.plan = None
        self.sent = 0
        self.version = 0
        self.slot = 1      # the slot of the base in flight (the first base goes to slot 0)
        self.seq = 0
        self.log = []   # (iteration, kind, bytes): chunk | sync_flush | commit

    def intercept(self, segments, version: int, interval: int, margin: int | None = None, cap: int = 256 * MiB):
        """Serialize the shard (device segments, in order) once, stage it to Tier-1, plan the pacing."""
        if self.plan is not None and self.sent < self.plan.total_bytes:
            self.flush(version)  # the previous base must be complete before the next one starts
        if int(version) < 1:
            raise ValueError("base versions are >= 1")
        o = sum(t.numel() * t.element_size() for t in segments)
        if o != self.n:
            raise ValueError(f"shard is {o} bytes, replicator built for {self.n}")
        if self.n > self.peer_n:  # the neighbour sized its slots for the shard it expects from us
            raise ValueError(f"shard of {self.n} bytes does not fit the neighbour's {self.peer_n}-byte slot")
        with torch.cuda.stream(self.s):
            o = 0
            for t in segments:
                b = t.contiguous().view(torch.uint8).reshape(-1)
                self.payload[o:o + b.numel()].copy_(b)
                o += b.numel()
        self.tc.stage_host(self.host, self.payload, self.n, self.tc.D2H, stream=self.s)
        self.plan = plan_chunks(self.n, interval, margin, cap)
        self.sent, self.version = 0, int(version)
        self.slot ^= 1  # the other slot: the committed base stays intact until this one commits
        return self.plan

    def _push(self, nbytes: int):
        # 16-byte aligned cover of [sent, sent + nbytes) (payload and slots are padded to 16 bytes;
        # an overlap re-sends bytes the peer already holds, with the same values)
        a0 = self.sent & ~15
        end = min(_pad16(self.n), (self.sent + nbytes + 15) // 16 * 16)
        self.len_dev.fill_(end - a0)
        self.seq += 1
        self.tc.push_peer(self.ctx, self.payload[a0:], self.len_dev, _Offset(self.peer_stage[self.slot], a0),
                          _pad16(self.peer_n) - a0, self.peer_progress, self.seq, stream=self.s)
        self.sent += nbytes

    def _commit(self, it: int):
        # stream-ordered after every chunk push of this base (same stream, each push fences at
        # system scope before its CTAs count out): {0, 2·version + slot} with a release store
        self.tc.push_peer(self.ctx, self.payload, self.zero_dev, self.peer_stage[self.slot], 0, self.peer_commit,
                          2 * self.version + self.slot, stream=self.s)
        self.log.append((it, "commit", 0))

    def pump(self, it: int):
        """This iteration's paced chunk (no-op once the base is out)."""
        if self.plan is None or self.sent >= self.plan.total_bytes:
            return
        with torch.cuda.stream(self.s):
            nb = min(self.plan.chunk_bytes, self.plan.total_bytes - self.sent)
            self._push(nb)
            self.log.append((it, "chunk", nb))
            if self.sent >= self.plan.total_bytes:
                self._commit(it)

    def flush(self, it: int):
        """Synchronous flush of the remaining bytes (spillover at the next base boundary)."""
        if self.plan is None or self.sent >= self.plan.total_bytes:
            return
        with torch.cuda.stream(self.s):
            rest = self.plan.total_bytes - self.sent
            self._push(rest)
            self.log.append((it, "sync_flush", rest))
            self._commit(it)
        self.s.synchronize()

    def _commit_word(self) -> int:
        return int(self.commit.tensor[8:16].view(torch.int64).item())

    def committed_version(self) -> int:
        """Version of the previous rank's base held complete in this GPU's staging slots (0: none)."""
        return self._commit_word() >> 1

    def received(self) -> torch.Tensor:
        """The previous rank's committed base (its slot; empty if none is committed)."""
        w = self._commit_word()
        if w == 0:
            return self.stage[0].tensor[:0]
        return self.stage[w & 1].tensor[: self.prev_n]

    def close(self):
        for p_ in self._maps:
            p_.close()
        torch.cuda.synchronize(self.dev)


def _pad16(n: int) -> int:
    return max(16, (int(n) + 15) // 16 * 16)


class _Offset:
    """A PeerMapping shifted by a byte offset (tc_push_peer writes at data_ptr())."""

    def __init__(self, mapping, off: int):
        self.p = mapping.data_ptr() + off

    def data_ptr(self):
        return self.p


def plan_loading(have_t1: bool, have_t2: bool) -> str:
    """The retrieval cascade ordered by cost (§3.3): Tier-1 (local
    host) if the rank's copy survived, else the ring peer's Tier-2 replica, else Tier-3 (out of
    scope here: reported as unavailable)."""
    if have_t1:
        return "t1"
    if have_t2:
        return "t2"
    return "t3"
