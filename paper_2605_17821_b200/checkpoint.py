"""Save / retrieve / reclaim lifecycle around libtc (§1; §3.1).

Host-side bookkeeping only — every byte of state is encoded, staged, replicated and folded by
libtc (tc.py); nothing here computes on the data.

    ring_peers        the Tier-2 ring mapping r -> (r+1) mod P (§3.1)
    consensus         global MIN of (latest base version, replay end) (§3.3)
    DiffChain         the version chain of one rank: links, N-record batches, watermark reclaim
                      (PAPER.md:226 version = iteration; P:207 batching N; P:306-310 watermark)
    Checkpointer      per-rank save_step (encode -> Tier-1 D2H -> Tier-2 ring) and restore
                      (fetch from Tier-1 / Tier-2, then one fold of the chain) on libtc
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
