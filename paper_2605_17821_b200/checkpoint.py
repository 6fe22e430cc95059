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

from collections import deque
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
class HostArena:
    """Tier-1 store ("local volatile memory", §1; §4 "pinned host memory
    buffers"): ONE page-locked buffer allocated up front, used as a FIFO ring of variable-size
    entries (records oldest -> newest, reclaimed from the oldest).  `alloc` returns a byte offset,
    or None when the entry does not fit (the caller then keeps that entry off Tier-1)."""

    def __init__(self, nbytes: int, buffer=None):
        if buffer is None:
            from . import tc

            buffer = tc.HostBuffer(max(16, int(nbytes)))
        self.buf = buffer  # tc.HostBuffer (anything with .nbytes / .tensor / .data_ptr())
        self.cap = self.buf.nbytes
        self.q = deque()  # (key, off, nbytes16)

    def alloc(self, key, nbytes: int):
        n = max(16, (int(nbytes) + 15) // 16 * 16)
        if not self.q:
            off = 0 if n <= self.cap else None
        else:
            head = self.q[0][1]
            tail = self.q[-1][1] + self.q[-1][2]
            if tail > head:
                off = tail if tail + n <= self.cap else (0 if n <= head else None)
            else:  # wrapped: free space is [tail, head)
                off = tail if tail + n <= head else None
        if off is not None:
            self.q.append((key, off, n))
        return off

    def release(self, keep):
        """Drop entries from the oldest while keep(key) is False (FIFO reclaim)."""
        while self.q and not keep(self.q[0][0]):
            self.q.popleft()

    def clear(self):
        self.q.clear()

    def view(self, off: int, nbytes: int):
        return self.buf.tensor[off: off + nbytes]

    def ptr(self, off: int):
        return _Offset(self.buf, off)


class Checkpointer:
    """Per-rank save / retrieve / reclaim of one ZeRO shard through libtc — the product path
    (§1 lifecycle; §3.1-3.4).  Every byte is encoded, staged, replicated and folded
    by libtc kernels; this class only orders the calls, owns the buffers and keeps the version chain.

    Allocated once, at construction (nothing per save):
      - the reference `ref` (the base, advanced by every encode: reading R2);
      - `dev_slots` device record slots of `rec_cap` bytes, sized to the expected change fraction
        (a record that outgrows its slot is refused on the device — R20 — and the next save is
        forced to be a base);
      - the record lengths in mapped pinned memory (the encoder writes them; no D2H copy);
      - the Tier-1 HostArena (the base + the records since it);
      - Tier-2 (`tier2="push"`): `t2_slots` slots + mailboxes on this GPU for the previous rank's
        records, the next rank's mapped here (CUDA IPC, one exchange) — NVLink stores, no NCCL;
        the paced base stream to the same neighbour (BaseReplicator).  world == 1 is the ring of one.
    save_step(v): encode v on the caller's stream (fused ref advance; with Tier-2 the encoder also
      writes the record into the neighbour's slot over NVLink and publishes its mailbox — the
      fused emit, NEXT row 1) and, one step behind (the host never waits for the encode it just
      issued), finish v-1: read its length, stage it to Tier-1 on the copy stream, fold it onto
      the optional hot `standby` replica, append it to the chain, pick the next format (R19).
    recover(): consensus on (base, replay end) over the group, the cascade
      Tier-1 -> Tier-2 per item (plan_loading), the base fetched into the live state
      and the chain folded onto it in batches of N; the reference follows.
    reclaim(w): drop records <= w."""

    def __init__(self, segments, rank: int = 0, world: int = 1, *, group=None, tier2: str | None = None,
                 expected_f: float = 0.05, record_format: str = "adaptive", dev_slots: int = 2,
                 t1_bytes: int | None = None, t2_slots: int = 8, standby=None, tile_words: int = 4096,
                 chunk_words: int = 1 << 28, ahead: bool = True, stage_base: bool = True, ref=None,
                 stream=None, base_version: int = 0, push_ctas: int = 16, timing: bool = False,
                 base_interval: int = 50, fused_t2: bool = True, rec_cap: int | None = None,
                 overlap_standby: bool = False):
        from . import tc

        self.tc = tc
        self.rank, self.world, self.group = rank, world, group
        self.seg = list(segments)
        self.device = self.seg[0].device
        dev = self.device.index
        self.ctx = tc.Ctx(dev)
        self.T, self.C = tile_words, chunk_words
        self.sizes = [s.numel() for s in self.seg]
        self.wb = [s.element_size() for s in self.seg]
        self.W = sum(n * w for n, w in zip(self.sizes, self.wb))
        self.words = sum(self.sizes)
        self.ref = list(ref) if ref is not None else [s.clone() for s in self.seg]
        self.cap_mask = tc.diff_bound(self.sizes, self.wb, tile_words, chunk_words)
        self.cap_idx = tc.diff_bound(self.sizes, self.wb, tile_words, chunk_words, index_mode=True) \
            if tile_words <= 8192 else 0
        self.cap_full = tc.diff_bound(self.sizes, self.wb, tile_words, chunk_words, full=True)
        worst = max(self.cap_mask, self.cap_idx, self.cap_full)
        self.rec_cap = int(rec_cap) if rec_cap is not None else \
            int(min(worst, (expected_f * 1.1 + 0.05) * self.W + (64 << 20)))
        if record_format not in ("adaptive", "mask", "index", "full"):
            raise ValueError("record_format: adaptive | mask | index | full")
        self.format = record_format
        self.next_fmt = record_format if record_format != "adaptive" else "mask"
        self.full_run = 0  # consecutive full records (adaptive: every 8th is a mask probe of the density)
        self.dev = [torch.empty(self.rec_cap, dtype=torch.uint8, device=self.device) for _ in range(dev_slots)]
        self.lens = tc.HostBuffer(8 * dev_slots)
        self.lens_v = self.lens.view(torch.int64)
        self.slot_busy: list[list] = [[] for _ in range(dev_slots)]  # events to wait before reuse
        self.s_comp = stream or torch.cuda.current_stream(self.device)
        self.s_copy = torch.cuda.Stream(self.device, priority=0)
        self.s_comm = torch.cuda.Stream(self.device, priority=-1)
        self.standby = list(standby) if standby is not None else None
        # the standby fold of record k-1 on a stream (and context) of its own, beside the encode of
        # record k — or behind it on the compute stream
        self.s_stby, self.sctx = self.s_comp, self.ctx
        if overlap_standby and self.standby is not None:
            self.s_stby = torch.cuda.Stream(self.device, priority=-1)
            self.sctx = tc.Ctx(dev)
        # every diff of this layout holds sum_s max(1, ceil(n_s / C)) records: the folds' descriptor
        # scratch is sized for that, not for the worst case the record bytes allow
        self.records_per_diff = sum(max(1, -(-n // chunk_words)) for n in self.sizes)
        for c in {id(self.ctx): self.ctx, id(self.sctx): self.sctx}.values():
            c.set_fold_max_records(self.records_per_diff)
        self.ahead = ahead
        self.timing = timing
        self.times = {"encode": [], "stage": [], "push": [], "fold": []}
        self.chain = DiffChain(base_version)
        self.where: dict[int, dict] = {}  # version -> {"t1": offset, "t2": slot, "n": bytes, "d2h": Event}
        self.pending = deque()
        self.needs_base = False
        self.dropped = set()  # tiers this rank lost (failure simulation / detection)
        if t1_bytes is None:
            t1_bytes = 8 * self.rec_cap
        self.t1 = HostArena(t1_bytes)                 # the records since the base
        self.t1_base_buf = tc.HostBuffer(self.W) if stage_base else None  # the base
        self.t1_base = None  # (version, Event) of the base on Tier-1
        # Tier-2
        self.tier2 = tier2
        self.t2_slots = t2_slots
        self.base_rep = None
        if tier2 == "push":
            self._init_push(t2_slots, push_ctas)
            if stage_base:
                self.base_rep = BaseReplicator(self.W, rank, world, dev)
        elif tier2 is not None:
            raise ValueError("tier2 must be None or 'push'")
        self.stage_base = stage_base
        self.base_interval = base_interval
        self.fused_t2 = fused_t2  # Tier-2 written by the encoder itself (else a push kernel after it)
        if stage_base:
            self._stage_base_t1(base_version)
            if self.base_rep is not None:
                self.base_rep.s.wait_stream(self.s_comp)
                self.base_rep.intercept(self.ref, base_version, interval=base_interval)

    # ------------------------------------------------------------------ setup helpers --
    def _init_push(self, slots: int, push_ctas: int):
        tc = self.tc
        caps = [self.rec_cap]
        if self.world > 1:
            import torch.distributed as dist

            caps = [None] * self.world
            dist.all_gather_object(caps, self.rec_cap, group=self.group)
        nxt, prv = ring_peers(self.rank, self.world)
        # my slots receive the previous rank's records; the next rank sized its slots for mine
        self.prev_cap, self.next_cap = int(caps[prv]), self.rec_cap
        self.rx = [tc.IpcBuffer(self.prev_cap) for _ in range(slots)]    # previous rank's records land here
        self.rx_mail = [tc.IpcBuffer(16) for _ in range(slots)]
        self.pctx = tc.Ctx(self.device.index)
        self.pctx.set_push_ctas(push_ctas)
        if self.world > 1:
            import torch.distributed as dist

            hs = [None] * self.world
            dist.all_gather_object(hs, [b.handle for b in self.rx] + [m.handle for m in self.rx_mail],
                                   group=self.group)
            self._maps = [tc.PeerMapping(h, self.next_cap) for h in hs[nxt][:slots]]
            self._maps += [tc.PeerMapping(h, 16) for h in hs[nxt][slots:]]
            self.tx, self.tx_mail = self._maps[:slots], self._maps[slots:]
        else:
            self._maps = []
            self.tx, self.tx_mail = self.rx, self.rx_mail

    def _stage_base_t1(self, version: int):
        """The base on Tier-1: the reference flattened into its pinned buffer (D2H per segment);
        the record arena restarts (the records of the previous base are reclaimed)."""
        tc = self.tc
        self.t1.clear()
        if "t1" in self.dropped:
            self.t1_base = None
            return
        o = 0
        for r in self.ref:
            nb = r.numel() * r.element_size()
            if nb:
                tc.stage_host(_Offset(self.t1_base_buf, o), r, nb, tc.D2H, stream=self.s_copy)
            o += nb
        self.t1_base = (version, torch.cuda.Event())
        self.t1_base[1].record(self.s_copy)

    def _ev(self, stream):
        e = torch.cuda.Event(enable_timing=self.timing)
        e.record(stream)
        return e

    # ----------------------------------------------------------------------- SAVE ------
    def save_step(self, version: int, segments=None) -> int | None:
        """Checkpoint the live state as version `version` (> chain head).  Returns the byte length
        of the record finished by this call (version - 1 when running one step ahead), or None."""
        tc = self.tc
        if segments is not None:
            self.seg = list(segments)
        if self.needs_base:
            self.flush()
            self.save_base(version)
            return None
        slot = version % len(self.dev)
        for e in self.slot_busy[slot]:
            self.s_comp.wait_event(e)
        self.slot_busy[slot] = []
        ref_version = self.pending[-1]["v"] if self.pending else self.chain.head
        e0 = self._ev(self.s_comp) if self.timing else None
        fmt = self.next_fmt if (self.next_fmt != "index" or self.cap_idx > 0) else "mask"
        index_mode, full = fmt == "index", fmt == "full"
        if self.tier2 == "push" and self.fused_t2:
            # Tier-2 fused into the encode: the record is written locally and, over NVLink, into
            # the neighbour's slot version % t2_slots; the encoder publishes its mailbox
            t2 = version % self.t2_slots
            tc.diff_encode_push(self.ctx, self.ref, self.seg, self.dev[slot], self.lens_v[slot: slot + 1], version,
                                ref_version, self.tx[t2], self.next_cap, self.tx_mail[t2], self.T, self.C, True,
                                stream=self.s_comp, index_mode=index_mode, full=full)
        else:
            tc.diff_encode(self.ctx, self.ref, self.seg, self.dev[slot], self.lens_v[slot: slot + 1], version,
                           ref_version, self.T, self.C, True, stream=self.s_comp, index_mode=index_mode, full=full)
        e1 = self._ev(self.s_comp)
        self.pending.append({"v": version, "ref_v": ref_version, "slot": slot, "e0": e0, "e1": e1,
                             "index": index_mode, "fmt": fmt})
        out = None
        while self.pending and (not self.ahead or len(self.pending) > 1):
            out = self._finish(self.pending.popleft())
        if self.base_rep is not None:
            self.base_rep.pump(version)
        return out

    def flush(self) -> int | None:
        out = None
        while self.pending:
            out = self._finish(self.pending.popleft())
        return out

    def _finish(self, p) -> int:
        tc = self.tc
        v, slot, e1 = p["v"], p["slot"], p["e1"]
        e1.synchronize()
        n = int(self.lens_v[slot].item())
        if self.timing and p["e0"] is not None:
            self.times["encode"].append((p["e0"], e1))
        if n > self.rec_cap:
            # the record outgrew its slot (R20): the reference has advanced, so this version can only
            # be recovered from a base — the next save takes one (§3.1 base stream).
            # Records issued after it are useless (they link to it) and dropped; the device's sticky
            # TC_ERR_CAPACITY of the refused record is consumed here.
            self.needs_base = True
            self.pending.clear()
            self.ctx.check_status(self.s_comp)
            return n
        count = self._count_of(n, p["fmt"])
        if self.format == "adaptive":
            self.next_fmt = self._choose(count, p["fmt"])
        tiers = set()
        busy = []
        # Tier-1: D2H into the arena on the copy stream
        off = self.t1.alloc(("rec", v), n) if "t1" not in self.dropped else None
        d2h = None
        if off is not None:
            self.s_copy.wait_event(e1)
            c0 = self._ev(self.s_copy) if self.timing else None
            tc.stage_host(self.t1.ptr(off), self.dev[slot], n, tc.D2H, stream=self.s_copy)
            d2h = self._ev(self.s_copy)
            busy.append(d2h)
            tiers.add("t1")
            if self.timing:
                self.times["stage"].append((c0, d2h))
        # Tier-2: the encode already wrote the record into the neighbour's slot v % t2_slots and
        # published its mailbox {bytes, v} (fused emit) — or, unfused, a push kernel copies it now
        t2 = None
        if self.tier2 == "push" and n <= self.next_cap:
            t2 = v % self.t2_slots
            if not self.fused_t2:
                self.s_comm.wait_event(e1)
                r0 = self._ev(self.s_comm) if self.timing else None
                tc.push_peer(self.pctx, self.dev[slot], self.lens_v[slot: slot + 1], self.tx[t2], self.next_cap,
                             self.tx_mail[t2], v, stream=self.s_comm)
                r1 = self._ev(self.s_comm)
                busy.append(r1)
                if self.timing:
                    self.times["push"].append((r0, r1))
            tiers.add("t2")
            # the record that used this neighbour slot before is no longer on Tier-2
            for e in self.chain.entries:
                if e.version != v and self.where.get(e.version, {}).get("t2") == t2:
                    e.tiers.discard("t2")
                    self.where[e.version]["t2"] = None
        # hot standby: fold the record onto the replica right behind the encode
        if self.standby is not None:
            if self.s_stby is not self.s_comp:
                self.s_stby.wait_event(e1)
            f0 = self._ev(self.s_stby) if self.timing else None
            tc.diff_apply(self.sctx, self.standby, p["ref_v"], [self.dev[slot]], [n], stream=self.s_stby)
            f1 = self._ev(self.s_stby)
            busy.append(f1)
            if self.timing:
                self.times["fold"].append((f0, f1))
        self.slot_busy[slot] = busy
        self.chain.append(v, p["ref_v"], n, tiers)
        self.where[v] = {"t1": off, "t2": t2, "n": n, "d2h": d2h, "count": count, "index": p["index"],
                         "fmt": p["fmt"]}
        return n

    def _count_of(self, n: int, fmt: str):
        """Changed words of a record of n bytes (None for a full record: it holds every word)."""
        w_avg = self.W / max(1, self.words)
        if fmt == "full":
            return None
        if fmt == "index":
            return max(0.0, n - (self.cap_idx - (2 + w_avg) * self.words)) / (2 + w_avg)
        return max(0.0, n - (self.cap_mask - self.W)) / w_avg

    def _choose(self, count, fmt: str) -> str:
        """Adaptive record format (R19; the paper adapts its payload format per tensor):
        the smallest record for the last density — index below 1/16 changed, full when a mask
        record would be within 2 % of it (full records encode in one streaming pass).  After a
        full record the density is unknown: stay full, with a mask record every 8th as a probe."""
        if count is None:
            self.full_run += 1
            return "mask" if self.full_run % 8 == 0 else "full"
        self.full_run = 0
        w_avg = self.W / max(1, self.words)
        if self.cap_idx > 0 and count * 16 < self.words:
            return "index"
        mask_bytes = (self.cap_mask - self.W) + count * w_avg
        return "full" if self.cap_full <= 1.02 * mask_bytes else "mask"

    def save_base(self, version: int):
        """A new base at `version` (§3.1 base stream; P:209 paced): the live state
        becomes the reference, Tier-1 keeps it (the arena restarts: older records are reclaimed),
        and the ring neighbour receives it in paced chunks (BaseReplicator)."""
        self.flush()
        for e in self.slot_busy:
            for ev in e:
                self.s_comp.wait_event(ev)
        with torch.cuda.stream(self.s_comp):
            for r, s_ in zip(self.ref, self.seg):
                r.copy_(s_)
        self.s_copy.wait_stream(self.s_comp)
        self.chain = DiffChain(version)
        self.where.clear()
        self.needs_base = False
        if self.stage_base:
            self._stage_base_t1(version)
            if self.base_rep is not None:
                self.base_rep.s.wait_stream(self.s_comp)
                self.base_rep.intercept(self.ref, version, interval=self.base_interval)

    # ------------------------------------------------------------------- RETRIEVE ------
    def available(self, tier: str) -> bool:
        return tier not in self.dropped

    def drop_tier(self, tier: str):
        """Failure simulation: this rank lost `tier` ("t1": its host memory, a node failure;
        "hbm": its device state — the live segments and the reference are zeroed)."""
        if tier == "hbm":
            torch.cuda.synchronize(self.device)
            for t in self.seg + self.ref:
                t.zero_()
            self.pending.clear()
            return
        self.dropped.add(tier)
        if tier == "t1":
            self.t1_base = None
            for e in self.chain.entries:
                e.tiers.discard("t1")

    def recover(self, upto: int | None = None, batch: int = 5, source: str | None = None) -> int:
        """Rebuild the live state (and the reference) at the consensus version (PAPER.md:226-263
        §3.3): every rank offers its latest base and the end of its recoverable chain, the job takes
        the MIN of each; the base and each record come from the cheapest tier that holds them
        (plan_loading: Tier-1, else the ring neighbour's Tier-2), and the chain is folded onto the
        base in batches of `batch` records (P:283 fused multi-step replay, N = 5 P:395)."""
        tc = self.tc
        self.flush()
        end = self.chain.head if upto is None else upto
        reach = self.chain.base_version
        for e in self.chain.entries:
            if e.version > end or not (e.tiers & {"t1", "t2"}):
                break
            reach = e.version
        base_v, end = consensus(self.chain.base_version, reach, self.group)
        if base_v != self.chain.base_version:
            raise RuntimeError(f"rank {self.rank}: consensus base {base_v} is not this rank's base "
                               f"{self.chain.base_version} (older bases are reclaimed)")
        s = self.s_comp
        # the base: Tier-1 host copy, else the neighbour's committed replica (NVLink read)
        src = source or plan_loading(self.t1_base is not None and self.available("t1"),
                                     self.base_rep is not None and self._t2_base_version() == base_v)
        if src == "t1":
            s.wait_event(self.t1_base[1])
            o = 0
            for t in self.seg:
                nb = t.numel() * t.element_size()
                if nb:
                    tc.stage_host(t, _Offset(self.t1_base_buf, o), nb, tc.H2D, stream=s)
                o += nb
        elif src == "t2":
            flat = self._t2_base_tensor()
            o = 0
            with torch.cuda.stream(s):
                for t in self.seg:
                    nb = t.numel() * t.element_size()
                    t.view(-1).view(torch.uint8).copy_(flat[o: o + nb])
                    o += nb
        else:
            raise RuntimeError(f"rank {self.rank}: base {base_v} is on no volatile tier (Tier-3 is out of scope)")
        # the chain: batches of records, each from Tier-1 (H2D into a slot) or Tier-2 (fold straight
        # from the neighbour's HBM over NVLink)
        sel = [e for e in self.chain.entries if e.version <= end]
        ver = base_v
        stage = None
        for i in range(0, len(sel), batch):
            b = sel[i: i + batch]
            recs, lens = [], []
            need_stage = sum(max(16, (e.nbytes + 15) // 16 * 16) for e in b
                             if plan_loading("t1" in e.tiers, "t2" in e.tiers) == "t1")
            if need_stage and (stage is None or stage.numel() < need_stage):
                stage = torch.empty(need_stage, dtype=torch.uint8, device=self.device)
            o = 0
            for e in b:
                w = self.where[e.version]
                how = plan_loading("t1" in e.tiers, "t2" in e.tiers)
                if how == "t1":
                    if w["d2h"] is not None:
                        s.wait_event(w["d2h"])
                    d = stage[o:]
                    tc.stage_host(d, self.t1.ptr(w["t1"]), e.nbytes, tc.H2D, stream=s)
                    o += max(16, (e.nbytes + 15) // 16 * 16)
                elif how == "t2":
                    self._check_t2_mail(w["t2"], e.version)
                    d = self.tx[w["t2"]]
                else:
                    raise RuntimeError(f"record {e.version} is on no volatile tier")
                recs.append(d)
                lens.append(e.nbytes)
            tc.diff_apply(self.ctx, self.seg, ver, recs, lens, stream=s)
            ver = b[-1].version
        self.ctx.check(s)
        with torch.cuda.stream(s):
            for r, t in zip(self.ref, self.seg):
                r.copy_(t)
        if self.standby is not None:
            s.wait_stream(self.s_stby)  # a standby fold still in flight finishes before the copy
            if self.sctx is not self.ctx:
                self.sctx.check(self.s_stby)
            with torch.cuda.stream(s):
                for r, t in zip(self.standby, self.seg):
                    r.copy_(t)
        # records past the recovered version are gone from the chain (the job resumes at `ver`)
        for e in [e for e in self.chain.entries if e.version > ver]:
            self.where.pop(e.version, None)
        self.chain.entries = [e for e in self.chain.entries if e.version <= ver]
        s.synchronize()
        return ver

    def restore(self, target, upto: int | None = None, source: str | None = None, batch: int = 8,
                stream=None) -> int:
        """Fold this rank's records onto `target` (CUDA tensors holding the base), each record from
        `source` ("t1" / "t2" / "device"; None = the cascade per record).  Lower-level than
        recover(): no consensus, the live state untouched."""
        tc = self.tc
        self.flush()
        s = stream or self.s_comp
        ver = self.chain.base_version
        for b in self.chain.batches(batch, upto):
            recs, lens = [], []
            for e in b:
                w = self.where[e.version]
                how = source or plan_loading("t1" in e.tiers, "t2" in e.tiers)
                if how == "t1":
                    if w["d2h"] is not None:
                        s.wait_event(w["d2h"])
                    d = torch.empty(max(e.nbytes, 16), dtype=torch.uint8, device=self.device)
                    tc.stage_host(d, self.t1.ptr(w["t1"]), e.nbytes, tc.H2D, stream=s)
                elif how == "t2":
                    self._check_t2_mail(w["t2"], e.version)
                    d = self.tx[w["t2"]]
                else:
                    raise ValueError(f"record {e.version}: source {how} unavailable")
                recs.append(d)
                lens.append(e.nbytes)
            tc.diff_apply(self.ctx, target, ver, recs, lens, stream=s)
            ver = b[-1].version
        self.ctx.check(s)
        return ver

    def _check_t2_mail(self, slot, version: int):
        """The neighbour's mailbox of `slot` must carry {bytes, version} (the record is there)."""
        if slot is None:
            raise RuntimeError(f"record {version} is not on Tier-2")
        self.s_comm.synchronize()
        m = torch.empty(2, dtype=torch.int64, device=self.device)
        _copy_from(m.view(torch.uint8), self.tx_mail[slot], 16)
        got = m.tolist()
        if got[1] != version:
            raise RuntimeError(f"Tier-2 slot {slot} holds version {got[1]}, not {version}")

    def _t2_base_version(self) -> int:
        if self.base_rep is None:
            return -1
        m = torch.empty(2, dtype=torch.int64, device=self.device)
        _copy_from(m.view(torch.uint8), self.base_rep.peer_commit, 16)
        return (int(m[1].item()) >> 1) - 1

    def _t2_base_tensor(self):
        m = torch.empty(2, dtype=torch.int64, device=self.device)
        _copy_from(m.view(torch.uint8), self.base_rep.peer_commit, 16)
        slot = int(m[1].item()) & 1
        flat = torch.empty(self.W, dtype=torch.uint8, device=self.device)
        _copy_from(flat, self.base_rep.peer_stage[slot], self.W)
        return flat

    # -------------------------------------------------------------------- RECLAIM ------
    def reclaim(self, watermark: int):
        """Drop every record with version <= watermark (§3.4: volatile histories
        are reclaimed once a newer base is safe).  The caller has folded them into its new base."""
        gone = {e.version for e in self.chain.reclaim(watermark)}
        for v in gone:
            self.where.pop(v, None)
        self.t1.release(lambda k: not (k[0] == "rec" and k[1] in gone))

    def close(self):
        torch.cuda.synchronize(self.device)
        for m in getattr(self, "_maps", []):
            m.close()
        if self.base_rep is not None:
            self.base_rep.close()


def _copy_from(dst: torch.Tensor, src, nbytes: int):
    """Device copy of `nbytes` from a raw device pointer (a peer mapping) into `dst`."""
    t = _RawView(src.data_ptr(), nbytes, dst.device)
    dst[:nbytes].copy_(t.tensor)
    torch.cuda.synchronize(dst.device)


class _RawView:
    """A uint8 CUDA tensor view of raw device memory (e.g. a peer IPC mapping)."""

    def __init__(self, ptr: int, nbytes: int, device):
        self.__cuda_array_interface__ = {"shape": (int(nbytes),), "typestr": "|u1", "data": (int(ptr), False),
                                         "version": 2, "strides": None}
        self.tensor = torch.as_tensor(self, device=device)


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
    {bytes, 2·(version + 1) + slot} (0 = nothing committed yet).  While base k+1 streams into one slot, the commit still points at
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
        # my slots hold the previous rank's base; the next rank sized its slots for mine
        self.prev_n, self.peer_n = int(sizes[prv]), self.n
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
        if int(version) < 0:
            raise ValueError("base versions are >= 0")
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
        # system scope before its CTAs count out): {0, 2·(version + 1) + slot} with a release store
        self.tc.push_peer(self.ctx, self.payload, self.zero_dev, self.peer_stage[self.slot], 0, self.peer_commit,
                          2 * (self.version + 1) + self.slot, stream=self.s)
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
        """Version of the previous rank's base held complete in this GPU's staging slots (-1: none)."""
        return (self._commit_word() >> 1) - 1

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
