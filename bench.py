#!/usr/bin/env python
"""bench.py — TierCheck differential-checkpoint hot path on B200 (BASELINE.json metric:
"diff encode & restore GB/s per GPU vs HBM peak; peer-replicate GB/s vs NVLink").

One STEP = one pass of the whole hot path for one checkpoint version
of each rank's shard:
    a2-a4  tc_diff_encode   ref(version k) vs cur(version k+1), fused ref advance -> record
    a5     tc_stage_host    record -> pinned host ring (Tier-1, copy stream)
    a6     tc_replicate_peer record -> ring neighbour over NCCL (Tier-2, comm stream; N > 1)
    a7     tc_diff_apply    fold the record onto the restore replica (version k -> k+1)
    a8     versions chained k -> k+1; every record links to the previous one.
The current state alternates between two synthetic versions X (v0) and Y (v1 = X + f changes),
so every step encodes a genuine incremental diff of change fraction f (X->Y->X->...).

value = state bytes of all ranks / step time (GB/s of state), inputs resident in HBM.
e2e   = the same through the C ABI with HOST buffers: every step copies the new state version
        from pinned host memory (H2D) and reads the record back (D2H), inside the timed region.

Usage: python bench.py [--gpus N] [--steps K] [--warmup W] [--workload cfg2] [--f 0.01]
       python bench.py --impl reference ...   (the oracle on host cores, bounded sample)
Multi-GPU: python -m torch.distributed.run --nproc-per-node N ... bench.py --gpus N
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)
# independent hardware work queues for the compute / copy / comm streams (the default of 8
# connections can alias two streams onto one queue and serialize them)
os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")
# stdout carries only the JSON line: anything a library writes to fd 1 (NCCL's version banner)
# goes to stderr, and the JSON is written through a private duplicate of the original stdout
_JSON_OUT = sys.stdout


def _private_stdout():
    global _JSON_OUT
    sys.stdout.flush()
    _JSON_OUT = os.fdopen(os.dup(1), "w")
    os.dup2(2, 1)


def emit(res):
    _JSON_OUT.write(json.dumps(res) + "\n")
    _JSON_OUT.flush()

import numpy as np  # noqa: E402

import synth  # noqa: E402

METRIC = "diff encode & restore GB/s per GPU vs HBM peak; peer-replicate GB/s vs NVLink"
WORKLOADS = {
    "cfg1": "cfg1: 1M fp32 params + Adam m/v (3 fp32 segments of 2^20 words), one step",
    "cfg2": "cfg2: GPT-2 1.5B-shaped (h1600 L48) bf16 weights + fp32 master/m/v, 1 GPU",
    "cfg3": "cfg3: GPT 7B-shaped (h4096 L32) ZeRO shard r of 8 per rank + Tier-2 ring replication",
    "cfg4": "cfg4: GPT 13B-shaped (h5120 L40) ZeRO shard r of 8 per rank",
}
NVLINK_GBS = 900.0          # nominal per direction per GPU
NVLINK_MEASURED_GBS = 770.0  # B200_PROFILING.md measured peer copy per direction


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as fh:
            d = json.load(fh)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md)"


# ------------------------------------------------------------------ helpers -------------
def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def record_counts(host_u8: np.ndarray, nbytes: int):
    """Parse the record headers of a staged diff (host copy) -> per-record (seg, m, w, T, count)."""
    out = []
    pos = 0
    while pos < nbytes:
        h = host_u8[pos: pos + 64]
        w = int(h[6])
        flags = int(h[7])
        T = int(h[8:12].view("<u4")[0])
        seg = int(h[12:16].view("<u4")[0])
        m = int(h[24:32].view("<u8")[0])
        count = int(h[32:40].view("<u8")[0])
        total = int(h[56:64].view("<u8")[0])
        out.append((seg, m, w, T, count, total, flags))
        pos += total
    return out


def algorithmic_bytes(recs, sector=False):
    """encode reads ref+cur (2W), writes mask + tile_off + header + values, and
    (advance_ref) the changed ref words.  Fold (N=1): reads mask + tile_off + header + values,
    writes the changed state words.  Word-granular unless sector=True (32-byte sectors)."""
    enc = fold = 0
    for seg, m, w, T, count, total, flags in recs:
        W = m * w
        if flags == 5:  # full record: read cur, write every word (+ ref <- cur); fold: read + write all
            enc += 64 + 3 * W
            fold += 64 + 2 * W
            continue
        if flags & 2:  # index mode: tile_off + u16 position per changed word instead of the mask
            meta = 64 + 4 * (-(-m // T) + 1) + 2 * count
        else:
            meta = 64 + 4 * -(-m // 32) + 4 * (-(-m // T) + 1)
        vals = w * count
        if sector and m:
            f = count / m
            scat = W * (1 - (1 - f) ** (32 // w))
        else:
            scat = vals
        enc += 2 * W + meta + vals + scat
        fold += meta + vals + scat
    return enc, fold


class Clocks:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.p = None
        self.path = os.path.join("/tmp", f"tc_clocks_{os.getpid()}.csv")

    def start(self):
        try:
            self.fh = open(self.path, "w")
            self.p = subprocess.Popen(["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.FIELDS}",
                                       "--format=csv,noheader,nounits", "-lms", "100"],
                                      stdout=self.fh, stderr=subprocess.DEVNULL)
        except Exception:
            self.p = None

    def stop(self):
        if self.p is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.p.terminate()
        try:
            self.p.wait(timeout=5)
        except Exception:
            self.p.kill()
        self.fh.close()
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        with open(self.path) as fh:
            for line in fh:
                parts = [x.strip() for x in line.split(",")]
                if len(parts) < 9:
                    continue
                try:
                    sm.append(float(parts[1]))
                    mx.append(float(parts[2]))
                except ValueError:
                    continue
                for nm, v in zip(names, parts[5:9]):
                    if v.lower() == "active":
                        reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(sm)}


# ------------------------------------------------------------- the GPU arm --------------
S3_ADAM = 2  # --structure 2: the state before / after one real Adam step


def adam_pair(X, Y, seed, s):
    """S3 "Adam-realistic" inputs (input preparation only — torch ops, untimed): X =
    a mid-training state (bf16 weights = RNE of the fp32 master ~ N(0, 0.02²), moments ~ 1e-3
    scale), Y = X after ONE bias-corrected Adam step (lr 1e-4, betas 0.9 / 0.999, eps 1e-8, step
    100) with a random gradient ~ N(0, 1e-3²).  Every fp32 word of master / m / v changes; the bf16
    words change where the update moves the master across a bf16 rounding boundary (~half)."""
    import torch

    g = torch.Generator(device=X[1].device).manual_seed(int(seed))
    lr, b1, b2, eps, t = 1e-4, 0.9, 0.999, 1e-8, 100
    n = X[1].numel()
    step = 1 << 26
    with torch.cuda.stream(s):
        for a in range(0, n, step):
            b = min(n, a + step)
            master = X[1].view(torch.float32)[a:b]
            m = X[2].view(torch.float32)[a:b]
            v = X[3].view(torch.float32)[a:b]
            master.normal_(0.0, 0.02, generator=g)
            m.normal_(0.0, 1e-3, generator=g)
            v.normal_(0.0, 1e-3, generator=g)
            v.mul_(v)
            X[0][a:b].copy_(master.to(torch.bfloat16).view(torch.int16))
            grad = torch.empty_like(master).normal_(0.0, 1e-3, generator=g)
            m2 = m * b1 + grad * (1 - b1)
            v2 = v * b2 + grad * grad * (1 - b2)
            upd = (m2 / (1 - b1 ** t)) / ((v2 / (1 - b2 ** t)).sqrt() + eps)
            master2 = master - lr * upd
            Y[1].view(torch.float32)[a:b].copy_(master2)
            Y[2].view(torch.float32)[a:b].copy_(m2)
            Y[3].view(torch.float32)[a:b].copy_(v2)
            Y[0][a:b].copy_(master2.to(torch.bfloat16).view(torch.int16))
    s.synchronize()
def run_ours(args):
    import torch
    import torch.distributed as dist

    from paper_2605_17821_b200 import tc

    rank, world, local = dist_env()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    numa = None
    if world > 1 and args.numa_bind:
        # every rank stages into host memory at once: pin each rank (and so its pinned Tier-1
        # buffers, first touch) to its GPU's NUMA node (N = 1 keeps every core for the oracle arm)
        from paper_2605_17821_b200.checkpoint import bind_local_numa

        numa = bind_local_numa(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    workload = args.workload or ("cfg2" if world == 1 else "cfg3")
    if workload == "cfg5":
        return run_streaming(args, rank, world, local, dev)
    shard = rank % 8 if workload in ("cfg3", "cfg4", "cfg5") else 0
    sizes, wb = synth.shard_layout(workload, shard)
    W = sum(n * w for n, w in zip(sizes, wb))
    seed = synth.SEED0 + shard
    p53 = synth.p53_of(args.f)
    T, C = args.tile_words, args.chunk_words

    def alloc(n, w):
        return torch.empty(n, dtype=torch.int16 if w == 2 else torch.int32, device=dev)

    s_comp = torch.cuda.Stream(device=dev)
    s_copy = torch.cuda.Stream(device=dev, priority=0)
    s_comm = torch.cuda.Stream(device=dev, priority=-1)  # NCCL CTAs get SM slots ahead of the encode
    # --overlap-fold: the latency-bound fold of record k-1 on its own high-priority stream, beside
    # the HBM-bound encode of record k (N = 1, one step ahead only)
    s_fold = torch.cuda.Stream(device=dev, priority=-1) if args.overlap_fold else s_comp
    ctx = tc.Ctx(local)
    ctx_f = tc.Ctx(local) if s_fold is not s_comp else ctx  # a tc_ctx serves one stream at a time
    if args.fold_dense_permille is not None:
        ctx.set_fold_dense_permille(args.fold_dense_permille)
        ctx_f.set_fold_dense_permille(args.fold_dense_permille)
    comm = tc.Comm(rank, world, local) if world > 1 else None
    rep_pool = None
    if comm is not None:
        from concurrent.futures import ThreadPoolExecutor

        rep_pool = ThreadPoolExecutor(1, initializer=lambda: torch.cuda.set_device(local))

    # inputs: X = version 0, Y = version 1 (device synth; input preparation, untimed)
    X = [alloc(n, w) for n, w in zip(sizes, wb)]
    Y = [alloc(n, w) for n, w in zip(sizes, wb)]
    A = [alloc(n, w) for n, w in zip(sizes, wb)]  # the advancing reference (chain state)
    R = [alloc(n, w) for n, w in zip(sizes, wb)]  # the restore replica (fold target)
    if args.structure == S3_ADAM:
        if wb != [2, 4, 4, 4]:
            raise SystemExit("--structure 2 needs the bf16 + fp32 master/m/v layout")
        adam_pair(X, Y, seed, s_comp)
        with torch.cuda.stream(s_comp):
            for s in range(len(sizes)):
                A[s].copy_(X[s])
                R[s].copy_(X[s])
    else:
        with torch.cuda.stream(s_comp):
            for s in range(len(sizes)):
                tc.synth_base(X[s], seed, s, stream=s_comp)
                Y[s].copy_(X[s])
                tc.synth_step(Y[s], seed, s, 1, p53, args.structure, stream=s_comp)
                A[s].copy_(X[s])
                R[s].copy_(X[s])
    s_comp.synchronize()
    cap = tc.diff_bound(sizes, wb, T, C)
    cap_idx = tc.diff_bound(sizes, wb, T, C, index_mode=True)
    allow_index = args.format in ("index", "adaptive") and T <= 8192
    if allow_index:
        cap = max(cap, cap_idx)
    fixed_mask = tc.diff_bound(sizes, [w for w in wb], T, C) - sum(n * w for n, w in zip(sizes, wb))
    # records: the bound at f is ~ (f + 0.036) W; allocate the bound only when it fits
    free = torch.cuda.mem_get_info(dev)[0]
    f_exp = 1.0 if args.structure == S3_ADAM else args.f  # S3: every fp32 word changes
    est = int(min(max(cap, tc.diff_bound(sizes, wb, T, C, full=True)), (f_exp * 1.1 + 0.05) * W + (64 << 20)))
    spill_need = (sum(sizes) // 4096 + 1) * (8192 + 1024)  # encode scratch (index mode: 8 KB spill + mask stage)
    # the step runs through the product lifecycle (paper_2605_17821_b200.checkpoint.Checkpointer) —
    # encode, Tier-1 staging, Tier-2 NVLink push, hot-standby fold, the version chain — except
    # with --tier2 nccl (kept as the NCCL baseline, driven here)
    use_ck = comm is None or args.tier2 == "push"
    ck = None
    if use_ck:
        from paper_2605_17821_b200.checkpoint import Checkpointer

        ck = Checkpointer(Y, rank, world, tier2="push" if world > 1 else None,
                          expected_f=1.0 if args.structure == S3_ADAM else args.f,
                          record_format=args.format if allow_index else "mask", dev_slots=args.dev_slots,
                          t1_bytes=(args.dev_slots + 1) * est,
                          t2_slots=2, standby=R, tile_words=T, chunk_words=C,
                          ahead=True if args.ahead is None else bool(args.ahead),
                          stage_base=False, ref=A, stream=s_comp, push_ctas=args.push_ctas, timing=True,
                          fused_t2=bool(args.t2_fused), overlap_standby=bool(args.overlap_standby))
        rec_cap = ck.rec_cap
        recs = ck.dev
        s_copy, s_comm = ck.s_copy, ck.s_comm  # the step's side streams are the lifecycle's
    else:
        rec_cap = cap if 2 * cap + est + spill_need + (8 << 30) < free else est
        recs = [torch.empty(rec_cap, dtype=torch.uint8, device=dev) for _ in range(2)]
    # the Tier-2 receive buffer: the neighbour's record (its capacity is exchanged by
    # tc_replicate_peer, so it need not be the worst-case bound)
    recv = torch.empty(est, dtype=torch.uint8, device=dev) if comm else None
    # NCCL-free Tier-2 (--tier2 push): two IPC slots + mailboxes on this GPU receive the previous
    # rank's records; the next rank's are mapped here and written with NVLink stores
    push = None
    if ck is not None and world > 1:
        push = {"mine": {"slots": ck.rx, "mail": ck.rx_mail}, "cap": ck.next_cap, "ctx": ck.pctx,
                "ctas": args.push_ctas, "peer_slots": ck.tx, "peer_mail": ck.tx_mail}
    elif comm is not None and args.tier2 == "push":
        import torch.distributed as dist

        mine = {"slots": [tc.IpcBuffer(est) for _ in range(2)], "mail": [tc.IpcBuffer(16) for _ in range(2)]}
        hs = [None] * world
        dist.all_gather_object(hs, [b.handle for b in mine["slots"]] + [m.handle for m in mine["mail"]])
        nxt_h = hs[(rank + 1) % world]
        pctx = tc.Ctx(local)
        pctx.set_push_ctas(args.push_ctas)
        push = {"mine": mine, "cap": est, "ctx": pctx, "ctas": args.push_ctas,
                "peer_slots": [tc.PeerMapping(h, est) for h in nxt_h[:2]],
                "peer_mail": [tc.PeerMapping(h, 16) for h in nxt_h[2:]]}
    # the encode kernel writes each record's length straight into mapped pinned memory, so the
    # host learns it without a copy-engine round trip
    ob_host = tc.HostBuffer(64)
    ob_view = ob_host.view(torch.int64) if ck is None else ck.lens_v
    obytes = [ob_view[i: i + 1] for i in range(2)]
    host_cap = est  # Tier-1 ring slots sized to the expected record, not the state
    host_ring = [tc.HostBuffer(host_cap) for _ in range(2)]  # libtc-pinned Tier-1 ring

    ev = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731
    state = {"ref_version": 0, "rest_version": 0, "content": "X",  # content of A and R
             "index": args.format == "index" and allow_index, "modes": []}
    total_words = sum(sizes)
    w_avg = W / total_words

    def next_mode(nbytes, was_index):
        """Adaptive record format (the paper adapts its payload format per tensor; here per
        checkpoint from the last record's density): index mode iff 2 B per changed word beats
        the 4 B per 32 words of the mask, i.e. fewer than 1/16 of the words changed."""
        if args.format != "adaptive" or not allow_index:
            return state["index"]
        if was_index:
            count = max(0.0, nbytes - (cap_idx - (2 + w_avg) * total_words)) / (2 + w_avg)
        else:
            count = max(0.0, nbytes - fixed_mask) / w_avg
        return count * 16 < total_words
    done_ev = [None, None]  # (copy_done, comm_done) for each record slot
    n_ops = {"encode": [], "fold": [], "stage": [], "replicate": []}
    host_t = {"stage": [], "fold": []}

    # At N = 1 the host runs one step ahead of the device: step k issues encode(k), then finishes step
    # k-1 (reads its record length — encode(k-1) is done by then or about to be —, stages it,
    # folds it, replicates it).  The device queue never waits for the host's length round trip;
    # the format choice for encode(k) therefore comes from record k-2 (one step of lag).
    def issue(k, timed):
        slot = k % 2
        cur = Y if state["content"] == "X" else X
        v = state["ref_version"] + 1
        if done_ev[slot] is not None:
            evs, fut_prev, timed_prev = done_ev[slot]
            for e in evs:
                s_comp.wait_event(e)
            if fut_prev is not None:
                r0p, r1p, nbp = fut_prev.result()
                s_comp.wait_event(r1p)
                if timed_prev:
                    n_ops["replicate"].append((r0p, r1p, nbp))
        e0, e1 = ev(), ev()
        e0.record(s_comp)
        use_index = state["index"]
        tc.diff_encode(ctx, A, cur, recs[slot], obytes[slot], v, v - 1, T, C, True, stream=s_comp,
                       index_mode=use_index)
        e1.record(s_comp)
        state["ref_version"] = v
        state["content"] = "Y" if state["content"] == "X" else "X"
        return {"slot": slot, "v": v, "e0": e0, "e1": e1, "use_index": use_index, "timed": timed}

    def finish(p):
        slot, v, e0, e1, timed = p["slot"], p["v"], p["e0"], p["e1"], p["timed"]
        e1.synchronize()
        nbytes = int(ob_view[slot].item())
        if nbytes > min(rec_cap, host_cap):
            raise RuntimeError("record exceeds the staging buffers")
        state["index"] = next_mode(nbytes, p["use_index"])
        if timed:
            state["modes"].append("index" if p["use_index"] else "mask")
        # Tier-1: D2H into the pinned ring on the copy stream
        s_copy.wait_event(e1)
        c0, c1 = ev(), ev()
        c0.record(s_copy)
        th0 = time.perf_counter()
        tc.stage_host(host_ring[slot], recs[slot], nbytes, tc.D2H, stream=s_copy)
        host_t["stage"].append(time.perf_counter() - th0)
        c1.record(s_copy)
        # Tier-2: ring-neighbour replication, issued from a background thread (the size exchange
        # blocks its caller until both neighbours are ready; the training-side thread must not)
        fut = None
        if comm is not None and push is None:
            def _replicate(slot=slot, e1=e1, nb=nbytes):
                s_comm.wait_event(e1)
                r0, r1 = ev(), ev()
                r0.record(s_comm)
                comm.replicate_peer(recs[slot], obytes[slot], recv, tc.TO_NEXT, stream=s_comm)
                r1.record(s_comm)
                return r0, r1, nb
            fut = rep_pool.submit(_replicate)
        # restore: fold the record onto the replica
        f0, f1 = ev(), ev()
        th0 = time.perf_counter()
        if s_fold is not s_comp:
            s_fold.wait_event(e1)
        f0.record(s_fold)
        tc.diff_apply(ctx_f, R, state["rest_version"], [recs[slot]], [nbytes], stream=s_fold)
        f1.record(s_fold)
        host_t["fold"].append(time.perf_counter() - th0)
        if push is not None:
            # Tier-2 push: kernels only (no host synchronization, no helper thread), started after
            # the fold so its NVLink stores overlap the next encode rather than the latency-bound fold
            s_comm.wait_event(f1)
            r0, r1 = ev(), ev()
            r0.record(s_comm)
            tc.push_peer(push["ctx"], recs[slot], obytes[slot], push["peer_slots"][slot], push["cap"],
                         push["peer_mail"][slot], v, stream=s_comm)
            tc.peer_wait(push["ctx"], push["mine"]["mail"][slot], v, None, stream=s_comm)
            r1.record(s_comm)
            fut = _Done((r0, r1, nbytes))
        state["rest_version"] = v
        done_ev[slot] = ([c1, f1] if s_fold is not s_comp else [c1], fut, timed)
        if timed:
            n_ops["encode"].append((e0, e1))
            n_ops["fold"].append((f0, f1))
            n_ops["stage"].append((c0, c1))
        return nbytes

    pending = [None]
    # With a ring neighbour the record slot written by encode(k) is the one Tier-2 still reads for
    # record k-2; running one step ahead would make encode(k) wait for that push (measured at N = 2:
    # 5.65 -> 6.14 ms per step), so at N > 1 each step finishes before the next is issued.
    ahead = world == 1

    def step(k, timed):
        """Issue step k and finish step k-1 (N = 1) or k itself (N > 1); returns the finished
        step's record bytes (None when nothing finished)."""
        p = issue(k, timed)
        if not ahead:
            return finish(p)
        out = finish(pending[0]) if pending[0] is not None else None
        pending[0] = p
        return out

    def flush():
        out = finish(pending[0]) if pending[0] is not None else None
        pending[0] = None
        return out

    def sync_all():
        for s in (s_comp, s_copy, s_comm, s_fold) + ((ck.s_stby,) if ck is not None else ()):
            s.synchronize()

    def drain():
        for sl in range(2):  # outstanding replications of the last two steps
            if done_ev[sl] is not None and done_ev[sl][1] is not None:
                r0p, r1p, nbp = done_ev[sl][1].result()
                if done_ev[sl][2]:
                    n_ops["replicate"].append((r0p, r1p, nbp))
                done_ev[sl] = (done_ev[sl][0], None, False)

    if ck is not None:
        # the product path: one save_step per version (the Checkpointer runs one step ahead at
        # N = 1 and finishes each step before the next at N > 1, as above); the records older
        # than the last one are reclaimed every step, so the Tier-1 arena
        # is a ring, as a deployment that takes a base every I iterations would keep it
        ck_done = []  # (version, bytes, index mode) of every finished save

        def ck_finished(nb):
            if nb is not None and ck.needs_base:
                raise RuntimeError(f"a {nb}-byte record outgrew the {ck.rec_cap}-byte record slot (R20)")
            if nb is not None:
                ck_done.append((ck.chain.head, nb, ck.where[ck.chain.head]["fmt"]))
                ck.reclaim(max(ck.chain.base_version, ck.chain.head - 1))
            return nb

        def step(k, timed):  # noqa: F811
            cur = Y if state["content"] == "X" else X
            v = state["ref_version"] + 1
            nb = ck.save_step(v, segments=cur)
            state["ref_version"] = v
            state["content"] = "Y" if state["content"] == "X" else "X"
            return ck_finished(nb)

        def flush():  # noqa: F811
            return ck_finished(ck.flush())

        def drain():  # noqa: F811
            pass

    for k in range(args.warmup):
        step(k, False)
    flush()
    drain()
    sync_all()
    if ck is not None:
        for v_ in ck.times.values():
            v_.clear()
        v_timed0 = state["ref_version"] + 1
    ctx.check(s_comp)
    ctx_f.check(s_fold)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    clocks = Clocks(local)
    clocks.start()
    time.sleep(0.3)
    def n_launch():
        if ck is not None:
            return ck.ctx.launches + (ck.pctx.launches if world > 1 else 0) + \
                (ck.sctx.launches if ck.sctx is not ck.ctx else 0)
        return ctx.launches + (push["ctx"].launches if push else 0) + (ctx_f.launches if ctx_f is not ctx else 0)

    launches0 = n_launch()
    t_start, t_end = ev(), ev()
    t_start.record(s_comp)
    sizes_seen = []
    for k in range(args.warmup, args.warmup + args.steps):
        nb = step(k, True)
        if nb is not None:
            sizes_seen.append(nb)
    nb = flush()
    if nb is not None:
        sizes_seen.append(nb)
    drain()
    for s in (s_copy, s_comm, s_fold) + ((ck.s_stby,) if ck is not None else ()):
        e = torch.cuda.Event()
        e.record(s)
        s_comp.wait_event(e)
    t_end.record(s_comp)
    sync_all()
    torch.cuda.synchronize()
    launches = n_launch() - launches0
    if world > 1:
        dist.barrier()
    clk = clocks.stop()
    ctx.check(s_comp)
    ctx_f.check(s_fold)
    if push:
        push["ctx"].check(s_comm)
    if ck is not None:
        ck.ctx.check(s_comp)
        if ck.sctx is not ck.ctx:
            ck.sctx.check(ck.s_stby)
        n_ops["encode"] = ck.times["encode"]
        n_ops["fold"] = ck.times["fold"]
        n_ops["stage"] = ck.times["stage"]
        state["rest_version"] = ck.chain.head  # the standby replica (R) and the reference (A)
        state["index"] = ck.next_fmt == "index"  # the format the next record would take
        state["fmt"] = ck.next_fmt
        timed_done = [d for d in ck_done if d[0] >= v_timed0]
        n_ops["replicate"] = [(a, b, d[1]) for (a, b), d in zip(ck.times["push"], timed_done)]
        state["modes"] = [d[2] for d in timed_done]
    ms = t_start.elapsed_time(t_end)
    t = torch.tensor([ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_max = float(t.item())
    ms_step = ms_max / args.steps

    def avg(pairs):
        return sum(a.elapsed_time(b) for a, b, *_ in pairs) / max(1, len(pairs))

    enc_ms, fold_ms, stage_ms = avg(n_ops["encode"]), avg(n_ops["fold"]), avg(n_ops["stage"])
    per_rank = None
    if world > 1:  # the slowest rank sets the step: every rank's encode / fold / Tier-1 time
        tt = torch.tensor([enc_ms, fold_ms, stage_ms], dtype=torch.float64, device=dev)
        allr = [torch.zeros_like(tt) for _ in range(world)]
        dist.all_gather(allr, tt)
        per_rank = {k: [round(float(x[i]), 3) for x in allr] for i, k in enumerate(("encode_ms", "fold_ms", "stage_ms"))}
    if args.timeline and rank == 0:
        print("host call ms:", {k: [round(x * 1e3, 3) for x in v] for k, v in host_t.items()}, file=sys.stderr)
        for name, pairs in n_ops.items():
            for pr in pairs:
                print(f"timeline {name:9s} start {t_start.elapsed_time(pr[0]):9.3f} end {t_start.elapsed_time(pr[1]):9.3f}",
                      file=sys.stderr)
    rep_ms = avg(n_ops["replicate"]) if n_ops["replicate"] else None
    # verify the chain: the restore replica equals the reference (both at the last version)
    ok = all(torch.equal(a, r) for a, r in zip(A, R))
    last_cur = Y if state["content"] == "Y" else X
    ok = ok and all(torch.equal(a, c) for a, c in zip(A, last_cur))
    if ck is not None:
        w_last = ck.where[ck.chain.head]
        host_last = ck.t1.view(w_last["t1"], w_last["n"]).numpy()
    else:
        host_last = host_ring[(args.warmup + args.steps - 1) % 2].numpy()
    recs_info = record_counts(host_last, sizes_seen[-1])
    enc_b, fold_b = algorithmic_bytes(recs_info)
    enc_bs, fold_bs = algorithmic_bytes(recs_info, sector=True)
    peak, peak_src = peaks()
    rec_bytes = sizes_seen[-1]
    changed = sum(r[4] for r in recs_info)
    # Tier-1 denominator, measured live after the timed region: a plain cudaMemcpyAsync (torch) of
    # the same record into the same pinned ring slot, all ranks at once as in the step; best of 3
    pcie = None
    if rec_bytes:
        hv = host_ring[0].view(torch.uint8)[:rec_bytes]
        best = None
        for _ in range(3):
            p0, p1 = ev(), ev()
            p0.record(s_copy)
            with torch.cuda.stream(s_copy):
                hv.copy_(recs[0][:rec_bytes], non_blocking=True)
            p1.record(s_copy)
            s_copy.synchronize()
            t_ = p0.elapsed_time(p1)
            best = t_ if best is None else min(best, t_)
        pcie = rec_bytes / best / 1e6

    scatter_ref = None
    # (sparse steps only: at high f the position lists alone outgrow the memory the step leaves)
    if world == 1 and args.f <= 0.05 and args.structure != S3_ADAM:  # writes Y's values at the X/Y differences into R, then puts R back
        scatter_ref = scatter_reference(X, Y, R, s_comp)
        if state["content"] == "X":
            with torch.cuda.stream(s_comp):
                for r_, x in zip(R, X):
                    r_.copy_(x)
            s_comp.synchronize()
    restore = None
    if args.restore_chain > 0:
        try:
            restore = restore_bench(tc, ctx, X, Y, A, R, recs[0], sizes, wb, seed, p53, T, C, s_comp,
                                    args.restore_chain, args.structure if args.structure != S3_ADAM else 0, peak,
                                    dev, state["index"], comm=comm,
                                    spare=recs[1] if len(recs) > 1 else None,
                                    recovery=args.recovery if args.recovery is not None else workload == "cfg4",
                                    full=state.get("fmt") == "full")
        except (torch.OutOfMemoryError, tc.TcError) as ex:  # an untimed probe must not lose the step's line
            restore = {"unavailable": f"{type(ex).__name__}: {ex}"[:300]}
            s_comp.synchronize()
            torch.cuda.empty_cache()
        # put the step buffers back to the X / Y pair (X intact; Y, A, R were reused)
        if args.structure == S3_ADAM:
            adam_pair(X, Y, seed, s_comp)
        with torch.cuda.stream(s_comp):
            for i in range(len(sizes)):
                if args.structure != S3_ADAM:
                    Y[i].copy_(X[i])
                    tc.synth_step(Y[i], seed, i, 1, p53, args.structure, stream=s_comp)
                A[i].copy_(X[i])
                R[i].copy_(X[i])
        s_comp.synchronize()
        state["content"] = "X"
    rep_probe = None
    if comm is not None:
        rep_probe = replicate_probe(tc, comm, recs[0], obytes, recv, rec_bytes, dev, s_comm, push)
    e2e = None
    if not args.no_e2e:
        try:
            e2e = run_e2e(args, tc, ctx, dev, sizes, wb, X, Y, A, R, recs, obytes, host_ring, rec_cap, T, C,
                          state, world, s_comp, s_copy)
        except (tc.TcError, RuntimeError) as ex:  # e.g. pinned host memory for 2 state versions per rank
            e2e = {"unavailable": f"{type(ex).__name__}: {ex}"[:300]}
    lossy = None
    if args.lossy and world == 1:
        lossy = lossy_probe(tc, ctx, X, Y, A, R, recs[0], s_comp, dev, peak)
    traffic = load_traffic(workload, args.f)

    if rank == 0:
        res = {
            "metric": METRIC,
            "value": round(world * W / (ms_step * 1e-3) / 1e9, 2),
            "unit": "GB/s",
            "n_gpus": world,
            "steps": args.steps,
            "warmup": args.warmup,
            "ms_per_step": round(ms_step, 4),
            "higher_is_better": True,
            "scaling": "weak",
            "vs_baseline": None,
            "dtype": "u16+u32 (bitwise)",
            "data": "synthetic (seeded splitmix64 state shards, DESIGN.md §6)",
            "config": {
                "workload": WORKLOADS.get(workload, workload),
                "shard_of_8": shard if workload != "cfg2" else None,
                "phi": synth.CONFIGS[workload][0],
                "segments": [[n, w] for n, w in zip(sizes, wb)],
                "state_bytes_per_rank": W,
                "f": args.f,
                "structure": {0: "S1 iid", 1: "S2 runs", S3_ADAM: "S3 Adam step (torch, lr 1e-4)"}[args.structure],
                "tile_words": T,
                "chunk_words": C,
                "fold_records_per_step": 1,
                "record_format": args.format,
                "record_modes_timed": sorted(set(state["modes"])),
                "l2": f"no flush: every step streams {W / 1e9:.1f} GB of state per rank (> 126 MB L2)",
                "step": ("Checkpointer.save_step: " if ck is not None else "") + (
                    "encode(advance_ref) writing the record over NVLink into the ring neighbour's IPC slot "
                    "(fused Tier-2 emit) + D2H stage + fold onto restore replica"
                    if (ck is not None and world > 1 and args.t2_fused)
                    else "encode(advance_ref) + D2H stage + " + (
                        ("NVLink push to the ring neighbour's IPC slot + " if push else "NCCL ring replicate + ")
                        if world > 1 else "") + "fold onto restore replica"),
                "parallelism": f"dp{world} (independent ZeRO shards; Tier-2 ring r->r+1)" if world > 1 else "1 GPU",
                "numa": numa,
            },
            "roofline": {
                "kernel": "tc_diff_encode = encode_mask_kernel + encode_prefix_kernel + encode_emit_kernel",
                "bound": "hbm",
                "achieved": round(enc_bs / (enc_ms * 1e-3) / 1e9, 1),
                "peak": peak,
                "unit": "GB/s",
                "frac": round(enc_bs / (enc_ms * 1e-3) / 1e9 / peak, 4),
                "traffic": traffic.get("encode"),
                "traffic_source": (f"stored ncu capture {traffic.get('source')} ({traffic.get('round', 'r6')}), "
                                   "same kernels and workload; not measured in this run") if traffic else None,
                "algorithmic_bytes": int(enc_bs),
                "bytes_basis": "sector-granular (SURVEY §8(d): a scattered 4-byte ref-advance write moves its "
                               "32-byte sector); word-granular below",
                "algorithmic_bytes_word": enc_b,
                "achieved_word": round(enc_b / (enc_ms * 1e-3) / 1e9, 1),
                "frac_word": round(enc_b / (enc_ms * 1e-3) / 1e9 / peak, 4),
                "peak_source": peak_src,
                "per_launch_ms": round(enc_ms, 4),
            },
            "breakdown": {
                "encode": {"ms": round(enc_ms, 4), "state_gbs": round(W / enc_ms / 1e6, 1),
                           "hbm_gbs": round(enc_b / enc_ms / 1e6, 1), "frac_hbm": round(enc_b / enc_ms / 1e6 / peak, 4)},
                "fold": {"ms": round(fold_ms, 4), "state_gbs": round(W / fold_ms / 1e6, 1),
                         "hbm_gbs_word": round(fold_b / fold_ms / 1e6, 1),
                         "hbm_gbs_sector": round(fold_bs / fold_ms / 1e6, 1),
                         "frac_hbm_sector": round(fold_bs / fold_ms / 1e6 / peak, 4),
                         "traffic": traffic.get("fold"),
                         "dram_gbs": round(traffic["fold"] / fold_ms / 1e6, 1) if traffic.get("fold") else None,
                         "scatter_reference": scatter_ref,
                         "scatter_roofline": scatter_roofline(changed, fold_ms, args.f)},
                "stage_d2h": {"ms": round(stage_ms, 4), "gbs": round(rec_bytes / stage_ms / 1e6, 2),
                              "pcie_copy_gbs": round(pcie, 2) if pcie else None,
                              "frac_pcie": round(rec_bytes / stage_ms / 1e6 / pcie, 4) if pcie else None,
                              "pcie_note": "denominator: a plain D2H cudaMemcpyAsync of the same record into "
                                           "the same pinned slot, measured after the timed region"},
                "replicate_in_step": ({"fused": "Tier-2 written by the encode kernels into the neighbour's "
                                                "IPC slot over NVLink (tc_diff_encode_push): no separate copy in "
                                                "the step; see 'replicate' for the isolated push"}
                                      if (ck is not None and world > 1 and args.t2_fused) else None)
                if rep_ms is None else {
                    "ms": round(rep_ms, 4), "gbs_per_direction": round(rec_bytes / rep_ms / 1e6, 1),
                    "note": "inside the pipelined step: shares HBM with encode/fold, PCIe with the "
                            "Tier-1 D2H, and waits for the slower neighbour's encode"},
                "replicate": rep_probe,
                "lossy_differential": lossy,
                "restore_chain": restore,
                "per_rank": per_rank,
                "record_bytes": rec_bytes,
                "changed_words": changed,
                "restore_equals_state": bool(ok),
            },
            "gpu_launches": launches,
            "clocks": clk,
            "e2e": e2e,
        }
        if args.cpu_baseline and world == 1:
            res["cpu_baseline"] = cpu_baseline(workload, args)
        emit(res)
    if comm is not None:
        comm.close()
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    if not ok:
        sys.exit(1)


def run_streaming(args, rank, world, local, dev):
    """cfg5 (the paper's 40B: h 5120, inter 20480, L 128; shard r of 8 = 70.9 GB per rank),
    checkpointing EVERY step (BASELINE configs[4]): the state evolves by one synthetic training
    step per version (untimed), and each version is checkpointed against the advancing reference
    (advance_ref = 1: state + reference = 141.9 GB of HBM).  The record bound (73.5 GB) does not fit
    beside them, so the checkpoint is encoded in runs of whole chunks (tc_diff_encode_range)
    through a 2-slot device ring, each run staged to the rank's pinned Tier-1 arena — and at N > 1
    pushed into the ring neighbour's slot over NVLink (Tier-2) — while the next run is encoded.
    ms_per_step = the end-to-end per-rank checkpoint of one version (the north star's "well under
    10 s").  After the timed steps the whole chain is verified: the reference equals the state, the
    base is regenerated and every version's diff is folded back from Tier-1 (bit-exact against the
    live state), and one 256-tile window per segment of the last version is byte-compared with the
    oracle on inputs from synth."""
    import torch
    import torch.distributed as dist

    from paper_2605_17821_b200 import tc

    shard = rank % 8
    sizes, wb = synth.shard_layout("cfg5", shard)
    W = sum(n * w for n, w in zip(sizes, wb))
    seed = synth.SEED0 + shard
    p53 = synth.p53_of(args.f)
    T, C, K = args.tile_words, args.chunk_words, args.stream_chunks
    s_comp = torch.cuda.Stream(device=dev)
    s_copy = torch.cuda.Stream(device=dev)
    s_comm = torch.cuda.Stream(device=dev, priority=-1)
    ctx = tc.Ctx(local)
    if args.fold_dense_permille is not None:
        ctx.set_fold_dense_permille(args.fold_dense_permille)
    S = [torch.empty(n, dtype=torch.int16 if w == 2 else torch.int32, device=dev) for n, w in zip(sizes, wb)]
    R = [torch.empty(n, dtype=torch.int16 if w == 2 else torch.int32, device=dev) for n, w in zip(sizes, wb)]
    with torch.cuda.stream(s_comp):
        for i in range(len(sizes)):
            tc.synth_base(S[i], seed, i, stream=s_comp)
            R[i].copy_(S[i])
    s_comp.synchronize()
    runs = []
    for i, n in enumerate(sizes):
        nch = max(1, -(-n // C))
        for c0 in range(0, nch, K):
            runs.append((i, c0, min(K, nch - c0)))
    # the checkpoint's last run is one chunk: its Tier-1 copy is the only one nothing overlaps
    if runs and runs[-1][2] > 1:
        i, c0, k = runs.pop()
        runs += [(i, c0, k - 1), (i, c0 + k - 1, 1)]
    allow_index = args.format in ("index", "adaptive") and T <= 8192
    slot_cap = max(max(tc.diff_bound_range(sizes[i], wb[i], c0, k, T, C),
                       tc.diff_bound_range(sizes[i], wb[i], c0, k, T, C, index_mode=True) if allow_index else 0)
                   for i, c0, k in runs)
    total_words = sum(sizes)
    w_avg = W / total_words
    fixed_mask = tc.diff_bound(sizes, wb, T, C) - W
    fixed_idx = tc.diff_bound(sizes, wb, T, C, index_mode=True) - (2 + w_avg) * total_words
    mode = {"index": args.format == "index" and allow_index}
    slots = [torch.empty(slot_cap, dtype=torch.uint8, device=dev) for _ in range(2)]
    push = None
    if world > 1:  # Tier-2: two IPC slots + mailboxes on this GPU for the previous rank's runs
        mine = {"slots": [tc.IpcBuffer(slot_cap) for _ in range(2)], "mail": [tc.IpcBuffer(16) for _ in range(2)]}
        hs = [None] * world
        dist.all_gather_object(hs, [b_.handle for b_ in mine["slots"]] + [m.handle for m in mine["mail"]])
        nx = hs[(rank + 1) % world]
        pctx = tc.Ctx(local)
        pctx.set_push_ctas(args.push_ctas)
        push = {"mine": mine, "ctx": pctx, "slots": [tc.PeerMapping(h, slot_cap) for h in nx[:2]],
                "mail": [tc.PeerMapping(h, 16) for h in nx[2:]]}
    lens_h = tc.HostBuffer(8 * max(2, len(runs)))
    lens = lens_h.view(torch.int64)
    n_versions = args.warmup + args.steps
    # Tier-1 keeps every version's diff (for the round trip): the first is a mask-mode record, the
    # adaptive format then takes index mode below 1/16 changed
    mask_est = int(fixed_mask + 1.1 * args.f * W) + (64 << 20)
    idx_est = int(fixed_idx + 1.1 * args.f * (2 + w_avg) * total_words) + (64 << 20)
    later = idx_est if (allow_index and args.f < 1 / 16) else mask_est
    host = tc.HostBuffer((mask_est if args.format != "index" else idx_est) + (n_versions - 1) * later)
    ev = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731
    diffs = []  # (version, host offset, bytes)
    seq = [0]

    def checkpoint(v, times, pos0):
        """One version: the runs' encodes issued one run ahead of the host, which learns each run's
        length (mapped pinned memory) only after issuing the next encode — the device never idles
        for the host's round trip — then stages it to Tier-1 and pushes it to the neighbour."""
        pos = [pos0]
        done = [None, None]

        def issue(r_i):
            i, c0, k = runs[r_i]
            sl = r_i % 2
            for e in done[sl] or []:
                s_comp.wait_event(e)
            e0, e1 = ev(), ev()
            e0.record(s_comp)
            tc.diff_encode_range(ctx, R[i], S[i], i, c0, k, slots[sl], lens[r_i: r_i + 1], v, v - 1, T, C, True,
                                 stream=s_comp, index_mode=mode["index"])
            e1.record(s_comp)
            return e0, e1

        def finish(r_i, e0, e1):
            sl = r_i % 2
            e1.synchronize()
            n = int(lens[r_i].item())
            if pos[0] + n > host.nbytes:
                raise RuntimeError("host Tier-1 buffer too small")
            s_copy.wait_event(e1)
            tc.stage_host(host.tensor[pos[0]:], slots[sl], n, tc.D2H, stream=s_copy)
            c1 = torch.cuda.Event()
            c1.record(s_copy)
            done[sl] = [c1]
            if push is not None:
                s_comm.wait_event(e1)
                seq[0] += 1
                tc.push_peer(push["ctx"], slots[sl], lens[r_i: r_i + 1], push["slots"][sl], slot_cap,
                             push["mail"][sl], seq[0], stream=s_comm)
                r1 = torch.cuda.Event()
                r1.record(s_comm)
                done[sl].append(r1)
            pos[0] += n
            if times is not None:
                times.append((e0, e1))

        pend = None
        for r_i in range(len(runs)):
            # the slot of run r_i was last used by run r_i - 2, finished (its copy enqueued) by now
            cur = (r_i,) + issue(r_i)
            if pend is not None:
                finish(*pend)
            pend = cur
        finish(*pend)
        if args.format == "adaptive" and allow_index:  # density of this checkpoint picks the next format
            nb = pos[0] - pos0
            if mode["index"]:
                count = max(0.0, nb - fixed_idx) / (2 + w_avg)
            else:
                count = max(0.0, nb - fixed_mask) / w_avg
            mode["index"] = count * 16 < total_words
        return pos[0]

    def train_step(v):  # the synthetic optimizer step producing version v (untimed)
        with torch.cuda.stream(s_comp):
            for i in range(len(sizes)):
                tc.synth_step(S[i], seed, i, v, p53, args.structure, stream=s_comp)

    pos = 0
    for v in range(1, args.warmup + 1):
        train_step(v)
        p1 = checkpoint(v, None, pos)
        diffs.append((v, pos, p1 - pos))
        pos = p1
    for st in (s_comp, s_copy, s_comm):
        st.synchronize()
    ctx.check(s_comp)
    if world > 1:
        dist.barrier()
    clocks = Clocks(local)
    clocks.start()
    time.sleep(0.3)
    launches0 = ctx.launches + (push["ctx"].launches if push else 0)
    enc_times, step_ms, modes = [], [], []
    for v in range(args.warmup + 1, n_versions + 1):
        train_step(v)
        t0, t1 = ev(), ev()
        t0.record(s_comp)
        modes.append("index" if mode["index"] else "mask")
        p1 = checkpoint(v, enc_times, pos)
        for st in (s_copy, s_comm):
            e = torch.cuda.Event()
            e.record(st)
            s_comp.wait_event(e)
        t1.record(s_comp)
        diffs.append((v, pos, p1 - pos))
        pos = p1
        step_ms.append((t0, t1))
    for st in (s_comp, s_copy, s_comm):
        st.synchronize()
    launches = ctx.launches + (push["ctx"].launches if push else 0) - launches0
    clk = clocks.stop()
    ctx.check(s_comp)
    if push is not None:
        push["ctx"].check(s_comm)
    ms_sum = sum(a.elapsed_time(b) for a, b in step_ms)
    tt = torch.tensor([ms_sum], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
    ms_step = float(tt.item()) / args.steps
    enc_ms = sum(a.elapsed_time(b) for a, b in enc_times) / args.steps
    last_v, last_pos, last_n = diffs[-1]
    recs_info = record_counts(host.numpy()[last_pos:], last_n)
    enc_b, _ = algorithmic_bytes(recs_info)
    enc_bs, _ = algorithmic_bytes(recs_info, sector=True)
    peak, peak_src = peaks()
    # ---- verification (untimed): advance, full round trip from Tier-1, oracle windows ----
    ok_adv = all(torch.equal(r, s_) for r, s_ in zip(R, S))
    with torch.cuda.stream(s_comp):
        for i in range(len(sizes)):
            tc.synth_base(R[i], seed, i, stream=s_comp)
    del slots
    big = max(max(16, n) for _, _, n in diffs)
    torch.cuda.empty_cache()  # (the timed run's ring slots went above)
    fit = int(torch.cuda.mem_get_info(dev)[0] * 0.8) // big  # batches of up to N = 5 that fit
    stage = [torch.empty(big, dtype=torch.uint8, device=dev) for _ in range(max(1, min(5, len(diffs), fit)))]
    tr0, tr1 = ev(), ev()
    tr0.record(s_comp)
    for j in range(0, len(diffs), len(stage)):
        batch = diffs[j: j + len(stage)]
        for (v, off, n), buf in zip(batch, stage):
            tc.stage_host(buf, host.tensor[off:], n, tc.H2D, stream=s_comp)
        tc.diff_apply(ctx, R, batch[0][0] - 1, stage[:len(batch)], [n for _, _, n in batch], stream=s_comp)
    tr1.record(s_comp)
    ctx.check(s_comp)
    ok_rt = all(torch.equal(r, s_) for r, s_ in zip(R, S))
    restore_ms = tr0.elapsed_time(tr1)
    del stage
    ok_or = _cfg5_oracle_windows(host.numpy(), last_pos, last_n, sizes, wb, seed, args.f, last_v, T, C)
    ok = ok_adv and ok_rt and ok_or
    if rank == 0:
        res = {
            "metric": METRIC, "value": round(world * W / (ms_step * 1e-3) / 1e9, 2), "unit": "GB/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms_step, 3),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u16+u32 (bitwise)",
            "data": "synthetic (seeded splitmix64 state shards, DESIGN.md §6)",
            "config": {"workload": "cfg5: paper's 40B (h5120 inter20480 L128) ZeRO shard r of 8 per rank, "
                                   "checkpoint every step of an evolving state, streamed encode + async host staging",
                       "phi": synth.CONFIGS["cfg5"][0], "segments": [[n, w] for n, w in zip(sizes, wb)],
                       "state_bytes_per_rank": W, "f": args.f, "tile_words": T, "chunk_words": C,
                       "chunks_per_run": K, "runs": len(runs), "advance_ref": 1, "versions": n_versions,
                       "record_format": args.format, "record_modes_timed": sorted(set(modes)),
                       "tier2": "NVLink push into the ring neighbour's IPC slot" if push else None,
                       "l2": f"no flush: {W / 1e9:.1f} GB of state per rank per step",
                       "parallelism": f"dp{world} shards of the 8-way split" if world > 1 else "1 GPU (shard 0 of 8)"},
            "end_to_end_checkpoint_s": round(ms_step / 1e3, 4),
            "paper_context": "TierCheck reports < 10 s end-to-end checkpointing for up to 40B on 16x A800 (P:16)",
            "roofline": {"kernel": "tc_diff_encode_range x runs (encode_mask + prefix + emit)", "bound": "hbm",
                         "achieved": round(enc_bs / (enc_ms * 1e-3) / 1e9, 1), "peak": peak, "unit": "GB/s",
                         "frac": round(enc_bs / (enc_ms * 1e-3) / 1e9 / peak, 4), "traffic": None,
                         "algorithmic_bytes": int(enc_bs), "bytes_basis": "sector-granular (SURVEY §8(d))",
                         "frac_word": round(enc_b / (enc_ms * 1e-3) / 1e9 / peak, 4),
                         "peak_source": peak_src, "encode_ms_per_step": round(enc_ms, 3)},
            "breakdown": {"record_bytes_last": last_n, "changed_words_last": sum(r[4] for r in recs_info),
                          "tier1_gbs": round(last_n / ms_step / 1e6, 2),
                          "verify": {"reference_equals_state": bool(ok_adv),
                                     "chain_round_trip_from_tier1": bool(ok_rt),
                                     "restore_ms_all_versions": round(restore_ms, 2),
                                     "oracle_windows_last_version": bool(ok_or)}},
            "gpu_launches": launches, "clocks": clk,
            "e2e": None, "e2e_note": "not measured for cfg5: a per-step H2D of the 70.9 GB state would only "
                                     "measure PCIe (see the cfg2 line for the e2e contract)",
        }
        emit(res)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    if not ok:
        sys.exit(1)


def _cfg5_oracle_windows(buf, pos0, nbytes, sizes, wb, seed, f, v, T, C):
    """One 256-tile window per segment (chunk 0, tiles 1000..1255) of version v's diff, byte-
    compared with the oracle's record of that window — inputs from synth (numpy), never the GPU."""
    import oracle

    pos, ok = pos0, True
    seen = set()
    while pos < pos0 + nbytes:
        h = buf[pos: pos + 64]
        w, flags = int(h[6]), int(h[7])
        seg = int(h[12:16].view("<u4")[0])
        off, m, count = (int(h[a: a + 8].view("<u8")[0]) for a in (16, 24, 32))
        total = int(h[56:64].view("<u8")[0])
        if off == 0 and seg not in seen and m >= 1300 * T:
            seen.add(seg)
            t0 = 1000
            st = synth.segment_versions(256 * T, w, seed, seg, [v - 1, v], f, start=t0 * T, threads=4)
            rc, exp = oracle.encode([st[v - 1].copy()], [st[v]], tile_words=T, chunk_words=C, advance_ref=True,
                                    version=v, ref_version=v - 1, index_mode=bool(flags & 2))
            nt = -(-m // T)
            p = pos + 64
            if flags & 2:
                toff = buf[p: p + 4 * (nt + 1)].view("<u4")
                pi = p + (-(-4 * (nt + 1) // 16) * 16)
                idx = buf[pi: pi + 2 * count].view("<u2")
                pv = pi + (-(-2 * count // 16) * 16)
            else:
                pm = p
                p = pm + (-(-4 * (-(-m // 32)) // 16) * 16)
                toff = buf[p: p + 4 * (nt + 1)].view("<u4")
                pv = p + (-(-4 * (nt + 1) // 16) * 16)
            vals = buf[pv: pv + w * count].view("<u2" if w == 2 else "<u4")
            k0, k1 = int(toff[t0]), int(toff[t0 + 256])
            e = exp
            eh_m = 256 * T
            ep = 64
            if flags & 2:
                et = e[ep: ep + 4 * 257].view("<u4")
                ei = ep + (-(-4 * 257 // 16) * 16)
                ecount = int(e[32:40].view("<u8")[0])
                eidx = e[ei: ei + 2 * ecount].view("<u2")
                ev_ = e[ei + (-(-2 * ecount // 16) * 16):].view("<u2" if w == 2 else "<u4")[:ecount]
                ok = ok and rc == 0 and np.array_equal(toff[t0: t0 + 257] - np.uint32(k0), et) and \
                    np.array_equal(idx[k0:k1], eidx) and np.array_equal(vals[k0:k1], ev_)
            else:
                emask = e[ep: ep + 4 * (eh_m // 32)].view("<u4")
                ok = ok and rc == 0 and np.array_equal(buf[pm + 4 * (t0 * T // 32): pm + 4 * ((t0 + 256) * T // 32)].view("<u4"), emask)
                ecount = int(e[32:40].view("<u8")[0])
                et0 = ep + (-(-4 * (eh_m // 32) // 16) * 16)
                et = e[et0: et0 + 4 * 257].view("<u4")
                ev_ = e[et0 + (-(-4 * 257 // 16) * 16):].view("<u2" if w == 2 else "<u4")[:ecount]
                ok = ok and np.array_equal(toff[t0: t0 + 257] - np.uint32(k0), et) and np.array_equal(vals[k0:k1], ev_)
        pos += total
    return ok and len(seen) == len(sizes)


def scatter_reference(X, Y, R, s):
    """The practical ceiling of the fold's access pattern, measured live: torch's index_put_ writing
    the same changed words (the positions where the two step versions differ) into the replica — a
    library scatter with no record parsing at all.  Not on the product path: a reference only."""
    import torch

    pos, vals = [], []
    with torch.cuda.stream(s):
        for x, y in zip(X, Y):
            for a in range(0, x.numel(), 1 << 27):
                d = (x[a: a + (1 << 27)] != y[a: a + (1 << 27)]).nonzero().squeeze(1) + a
                pos.append(d)
                vals.append(y[d])
    s.synchronize()
    ev = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731
    out = []
    for _ in range(3):
        a, b = ev(), ev()
        a.record(s)
        with torch.cuda.stream(s):
            k = 0
            for r_, x in zip(R, X):
                for o in range(0, x.numel(), 1 << 27):
                    r_.index_put_((pos[k],), vals[k])
                    k += 1
        b.record(s)
        s.synchronize()
        out.append(a.elapsed_time(b))
    n = sum(p.numel() for p in pos)
    del pos, vals
    ms = statistics.median(out)
    return {"ms": round(ms, 4), "words": n,
            "note": "torch index_put_ of the step's changed words into the replica (library scatter, same "
                    "positions, no record parsing): the measured ceiling of this access pattern"}


class _Done:
    """An already-completed future (the push path enqueues kernels and returns at once)."""

    def __init__(self, value):
        self.value = value

    def result(self):
        return self.value


def recovery_bench(tc, ctx, comm, X, Z, R, recs, lens, hosts, spare, s, dev):
    """Config 4's "chained restore from base + differentials after a simulated GPU failure"
    (BASELINE.json configs[3]; the paper's T_rollback + T_rerun).  The rank's state R
    is overwritten (its HBM contents are lost), then rebuilt and checked against the chain head Z:
    Tier-1: H2D of the base shard and the records from pinned host memory + one fold;
    Tier-2 (N > 1): every rank pulls its base and records back from the ring neighbour that holds
    them (tc_replicate_peer TO_PREV over NVLink) + one fold.  CUDA events, max over ranks."""
    import torch
    import torch.distributed as dist

    ev = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731
    world = dist.get_world_size() if dist.is_initialized() else 1

    def mx(v):
        if world == 1:
            return v
        t = torch.tensor([v], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    out = {"records": len(recs), "base_bytes": sum(x.numel() * x.element_size() for x in X),
           "record_bytes_total": sum(lens)}
    # Tier-1 copy of the base (the last base checkpoint, staged once)
    hb = [tc.HostBuffer(x.numel() * x.element_size()) for x in X]
    for h, x in zip(hb, X):
        tc.stage_host(h, x, x.numel() * x.element_size(), tc.D2H, stream=s)
    s.synchronize()

    def fail():
        with torch.cuda.stream(s):
            for r_ in R:
                r_.fill_(0x5A)  # the failed GPU's state is gone
        s.synchronize()

    fail()
    staged = [torch.empty(max(n, 16), dtype=torch.uint8, device=dev) for n in lens]
    e = [ev() for _ in range(4)]
    e[0].record(s)
    for r_, h in zip(R, hb):
        tc.stage_host(r_, h, r_.numel() * r_.element_size(), tc.H2D, stream=s)
    e[1].record(s)
    for d, h, n in zip(staged, hosts, lens):
        tc.stage_host(d, h, n, tc.H2D, stream=s)
    e[2].record(s)
    tc.diff_apply(ctx, R, 0, staged, lens, stream=s)
    e[3].record(s)
    s.synchronize()
    ctx.check(s)
    ok1 = all(torch.equal(r_, z) for r_, z in zip(R, Z))
    out["tier1"] = {"base_h2d_ms": round(mx(e[0].elapsed_time(e[1])), 3),
                    "records_h2d_ms": round(mx(e[1].elapsed_time(e[2])), 3),
                    "fold_ms": round(mx(e[2].elapsed_time(e[3])), 3),
                    "total_ms": round(mx(e[0].elapsed_time(e[3])), 3),
                    "restored_equals_head": bool(ok1)}
    for h in hb:
        h.free()
    if comm is not None:
        # save side (untimed): base segments and records -> the next rank's holding buffer, laid
        # out by the previous rank's sizes (shards and records differ in size between ranks)
        mine = [x.numel() * x.element_size() for x in X] + list(lens)
        every = [None] * world
        dist.all_gather_object(every, mine)
        prev_sizes = every[(dist.get_rank() - 1) % world]
        offs, o = [], 0
        for n in prev_sizes:
            offs.append(o)
            o += (n + 15) // 16 * 16
        holder = spare if spare is not None and spare.numel() >= o else None
        if holder is None:
            free = torch.cuda.mem_get_info(dev)[0]
            if free > o + (4 << 30):
                holder = torch.empty(o, dtype=torch.uint8, device=dev)
        if holder is None:
            out["tier2"] = {"skipped": "no room for the neighbour's base + records on this GPU"}
            return out
        srcs = [x.view(torch.uint8) for x in X] + [r[:n] for r, n in zip(recs, lens)]
        for src, off, pn in zip(srcs, offs, prev_sizes):
            nb = torch.tensor([src.numel()], dtype=torch.int64, device=dev)
            comm.replicate_peer(src, nb, holder[off: off + pn], tc.TO_NEXT, stream=s)
        s.synchronize()
        fail()
        dist.barrier()
        dsts = [r_.view(torch.uint8) for r_ in R] + [d[:n] for d, n in zip(staged, lens)]
        nbs = [torch.tensor([pn], dtype=torch.int64, device=dev) for pn in prev_sizes]
        e = [ev() for _ in range(4)]
        e[0].record(s)
        for i, (d, off, nb, pn) in enumerate(zip(dsts, offs, nbs, prev_sizes)):
            if i == len(X):
                e[1].record(s)
            comm.replicate_peer(holder[off: off + pn], nb, d, tc.TO_PREV, stream=s)
        e[2].record(s)
        tc.diff_apply(ctx, R, 0, staged, lens, stream=s)
        e[3].record(s)
        s.synchronize()
        ctx.check(s)
        ok2 = all(torch.equal(r_, z) for r_, z in zip(R, Z))
        out["tier2"] = {"base_pull_ms": round(mx(e[0].elapsed_time(e[1])), 3),
                        "records_pull_ms": round(mx(e[1].elapsed_time(e[2])), 3),
                        "fold_ms": round(mx(e[2].elapsed_time(e[3])), 3),
                        "total_ms": round(mx(e[0].elapsed_time(e[3])), 3),
                        "base_pull_gbs": round(out["base_bytes"] / mx(e[0].elapsed_time(e[1])) / 1e6, 1),
                        "restored_equals_head": bool(ok2)}
        del holder
    del staged
    return out


def restore_bench(tc, ctx, X, Z, ref, R, tmp, sizes, wb, seed, p53, T, C, s, nrec, structure, peak, dev,
                  index_mode=False, comm=None, spare=None, recovery=False, full=False):
    """a7 at N = nrec (SURVEY §8(a), config 4's "chained restore of 8 differentials"): build a real
    chain of `nrec` incremental records (versions 1..nrec, each a fresh f-change set), then
    (1) fold all of them onto a base copy in one tc_diff_apply call (records resident in HBM), and
    (2) restore from Tier-1: H2D of the records from pinned host memory + the same fold.
    CUDA events on the stream; the restored state is checked against the chain head."""
    import torch

    with torch.cuda.stream(s):  # Z (chain head) and ref start at the base X
        for z, r_, x in zip(Z, ref, X):
            z.copy_(x)
            r_.copy_(x)
    ob = torch.zeros(1, dtype=torch.int64, device=dev)
    recs, lens, counts = [], [], []
    with torch.cuda.stream(s):
        for v in range(1, nrec + 1):
            # dense chains outgrow the HBM the step leaves (f = 30 %: 7 GB per record at cfg2): the
            # chain stops at the records that fit (reported) instead of failing the run
            if lens and torch.cuda.mem_get_info(dev)[0] < lens[-1] * 1.05 + (2 << 30):
                break
            for i, z in enumerate(Z):
                tc.synth_step(z, seed, i, 1000 + v, p53, structure, stream=s)
            cnt = 0
            for r_, z in zip(ref, Z):
                for a in range(0, z.numel(), 1 << 27):
                    cnt += int((r_[a: a + (1 << 27)] != z[a: a + (1 << 27)]).sum().item())
            counts.append(cnt)
            tc.diff_encode(ctx, ref, Z, tmp, ob, v, v - 1, T, C, True, stream=s, index_mode=index_mode, full=full)
            s.synchronize()
            n = int(ob.item())
            if not recs and torch.cuda.mem_get_info(dev)[0] < n + (1 << 30):
                return {"unavailable": f"one {n / 1e9:.1f} GB record does not fit beside the step's buffers"}
            recs.append(tmp[:n].clone())
            lens.append(n)
    cut = len(recs) < nrec
    nrec = len(recs)
    union, line_bytes = 0, 0
    with torch.cuda.stream(s):
        for x, z, w_ in zip(X, Z, wb):
            for a in range(0, x.numel(), 1 << 27):  # slices: no full-size temporaries
                d = x[a: a + (1 << 27)] != z[a: a + (1 << 27)]
                union += int(d.sum().item())
                k = d.numel() // 32 * 32  # 32-word lines touched by the chain (the streaming fold writes them)
                line_bytes += (int(d[:k].view(-1, 32).any(dim=1).sum().item()) * 32 +
                               int(d[k:].any().item()) * (d.numel() - k)) * w_
                del d
    hosts = [tc.HostBuffer(n) for n in lens]
    for h, r, n in zip(hosts, recs, lens):
        tc.stage_host(h, r, n, tc.D2H, stream=s)
    s.synchronize()
    ev = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731
    fold_ms, t1_ms = [], []
    for rep in range(3):
        with torch.cuda.stream(s):
            for r_, x in zip(R, X):
                r_.copy_(x)
        a, b = ev(), ev()
        a.record(s)
        tc.diff_apply(ctx, R, 0, recs, lens, stream=s)
        b.record(s)
        s.synchronize()
        fold_ms.append(a.elapsed_time(b))
        with torch.cuda.stream(s):
            for r_, x in zip(R, X):
                r_.copy_(x)
        staged = recs  # the H2D lands in the device records themselves (same bytes; no 2nd copy of the chain)
        a, b = ev(), ev()
        a.record(s)
        for d, h, n in zip(staged, hosts, lens):
            tc.stage_host(d, h, n, tc.H2D, stream=s)
        tc.diff_apply(ctx, R, 0, staged, lens, stream=s)
        b.record(s)
        s.synchronize()
        t1_ms.append(a.elapsed_time(b))
        del staged
    ctx.check(s)
    ok = all(torch.equal(r_, z) for r_, z in zip(R, Z))
    rec_out = recovery_bench(tc, ctx, comm, X, Z, R, recs, lens, hosts, spare, s, dev) if recovery else None
    # algorithmic bytes of the fold: every record's mask + tile_off + header, the winning values
    # read and the state words written (word-granular), SURVEY §8(d)
    meta = 0
    for n_, w_ in zip(sizes, wb):
        chunks = max(1, -(-n_ // C))
        meta += nrec * (64 * chunks if full else
                        (0 if index_mode else 4 * -(-n_ // 32)) + 4 * (-(-n_ // T) + chunks) + 64 * chunks)
    if index_mode:  # every record's u16 positions: 2 bytes per changed word of each record
        meta += 2 * sum(counts)
    wmean = sum(n_ * w_ for n_, w_ in zip(sizes, wb)) / sum(sizes)
    fold_b = meta + 2 * union * wmean
    fm = statistics.median(fold_ms)
    for h in hosts:
        h.free()
    W = sum(n_ * w_ for n_, w_ in zip(sizes, wb))
    # the streaming fold (chunks whose records change > 3 % of the words) reads the
    # whole state and the records and writes back every touched 32-word line
    # the default strategy of tc_diff_apply (include/tc.h): index-mode chains at T = 4096 stream
    # when long (N >= 4, >= 0.5 % in total) or dense (> 6 %)
    tot, words = sum(counts), sum(sizes)
    # (mask chains at T = 4096: the mask-list kernel when > 6 % in total)
    if full:
        dense = False
    elif index_mode:
        dense = T == 4096 and ((nrec >= 4 and tot * 1000 >= words * 5) or tot * 1000 > words * 60)
    else:
        dense = T == 4096 and nrec <= 32 and tot * 1000 > words * 60
    stream_b = W + line_bytes + sum(lens)
    # SURVEY §8(d) sector-granular: the records' metadata, the winning values, every 32-byte sector
    # holding a word of the union written
    fu = union / max(1, words)
    fold_bs = meta + union * wmean + sum(n_ * w_ * (1 - (1 - fu) ** (32 // w_)) for n_, w_ in zip(sizes, wb))
    return {"records": nrec, **({"chain_cut": "HBM left after the step holds this many records"} if cut else {}),
            "record_format": "full" if full else "index" if index_mode else "mask",
            "strategy": ("stream (mask-list)" if not index_mode else "stream (list)") if dense else "scatter",
            "record_bytes_total": sum(lens), "union_changed_words": union,
            "fold_ms": round(fm, 4), "state_gbs": round(W / fm / 1e6, 1),
            "hbm_gbs_word": round(fold_b / fm / 1e6, 1), "frac_hbm_word": round(fold_b / fm / 1e6 / peak, 4),
            "hbm_gbs_sector": round(fold_bs / fm / 1e6, 1), "frac_hbm_sector": round(fold_bs / fm / 1e6 / peak, 4),
            "streaming_model": {"bytes": stream_b, "gbs": round(stream_b / fm / 1e6, 1),
                                "note": "NOT SURVEY §8(d) bytes: the whole state read + touched lines written + "
                                        "records (what the streaming fold moves)"},
            "touched_sector_floor": touched_floor(fu, W, fm),
            "tier1_restore_ms": round(statistics.median(t1_ms), 3),
            "restored_equals_head": bool(ok),
            "failure_recovery": rec_out}


def replicate_probe(tc, comm, rec, obytes, recv, rec_bytes, dev, s_comm, push=None):
    """Tier-2 in isolation: ring shifts of this step's record and of a fixed 1 GiB payload through
    tc_replicate_peer (NCCL: size exchange + send/recv) and, with --tier2 push, through
    tc_push_peer + tc_peer_wait (NVLink stores into the neighbour's IPC slot).  CUDA events on
    the comm stream, max over ranks."""
    import torch
    import torch.distributed as dist

    def timed(fn, reps=5):
        for i in range(2):
            fn(i)
        s_comm.synchronize()
        dist.barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s_comm)
        for i in range(reps):
            fn(2 + i)
        e1.record(s_comm)
        s_comm.synchronize()
        t = torch.tensor([e0.elapsed_time(e1) / reps], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    def frac(g):
        return {"gbs_per_direction": round(g, 1), "frac_nvlink_nominal": round(g / NVLINK_GBS, 4),
                "frac_nvlink_measured": round(g / NVLINK_MEASURED_GBS, 4)}

    G = 1 << 30
    nb_dev = torch.tensor([rec_bytes], dtype=torch.int64, device=dev)
    big = torch.empty(G, dtype=torch.uint8, device=dev)
    big_r = torch.empty(G, dtype=torch.uint8, device=dev)
    gb_dev = torch.tensor([G], dtype=torch.int64, device=dev)
    ms_rec = timed(lambda i: comm.replicate_peer(rec, nb_dev, recv, tc.TO_NEXT, stream=s_comm))
    ms_1g = timed(lambda i: comm.replicate_peer(big, gb_dev, big_r, tc.TO_NEXT, stream=s_comm))
    del big_r
    out = {"record_bytes": rec_bytes, "ms": round(ms_rec, 4), **frac(rec_bytes / ms_rec / 1e6),
           "ring_shift_1GiB": {"ms": round(ms_1g, 4), **frac(G / ms_1g / 1e6)},
           "note": "isolated tc_replicate_peer ring shift (size exchange + NCCL send/recv), max over ranks; "
                   "nominal 900 GB/s, measured peer copy 770 GB/s (B200_PROFILING.md)"}
    if push is not None:
        pc = push["ctx"]
        base = 1 << 40  # mailbox versions of the probe, above any step's version

        def push_rec(i):
            tc.push_peer(pc, rec, nb_dev, push["peer_slots"][0], push["cap"], push["peer_mail"][0], base + i,
                         stream=s_comm)
            tc.peer_wait(pc, push["mine"]["mail"][0], base + i, None, stream=s_comm)

        ms_prec = timed(push_rec)
        # the record-size push by CTA count (the step uses few CTAs so as not to slow the encode
        # beside it; alone, more stores in flight reach more of the link)
        by_ctas = {}
        for ctas in (16, 64, 148, 296, 592):
            pc.set_push_ctas(ctas)
            by_ctas[ctas] = timed(push_rec)
        pc.set_push_ctas(push["ctas"])
        best_ctas = min(by_ctas, key=by_ctas.get)
        land, lmail = tc.IpcBuffer(G), tc.IpcBuffer(16)
        hs = [None] * dist.get_world_size()
        dist.all_gather_object(hs, [land.handle, lmail.handle])
        nx = hs[(dist.get_rank() + 1) % len(hs)]
        pl, pm = tc.PeerMapping(nx[0], G), tc.PeerMapping(nx[1], 16)

        def push_1g(i):
            tc.push_peer(pc, big, gb_dev, pl, G, pm, base + i, stream=s_comm)
            tc.peer_wait(pc, lmail, base + i, None, stream=s_comm)

        ms_p1g = timed(push_1g)
        pc.set_push_ctas(2 * torch.cuda.get_device_properties(dev).multi_processor_count)
        ms_p1g_max = timed(push_1g)
        pc.set_push_ctas(push["ctas"])
        pc.check(s_comm)
        dist.barrier()
        pl.close()
        pm.close()
        land.free()
        lmail.free()
        out["push"] = {"ms": round(ms_prec, 4), **frac(rec_bytes / ms_prec / 1e6),
                       "ctas": push["ctas"],
                       "record_by_ctas": {str(c): {"ms": round(t_, 4), **frac(rec_bytes / t_ / 1e6)}
                                          for c, t_ in by_ctas.items()},
                       "record_best": {"ctas": best_ctas, "ms": round(by_ctas[best_ctas], 4),
                                       **frac(rec_bytes / by_ctas[best_ctas] / 1e6)},
                       "ring_shift_1GiB": {"ms": round(ms_p1g, 4), **frac(G / ms_p1g / 1e6)},
                       "ring_shift_1GiB_all_sms": {"ms": round(ms_p1g_max, 4), **frac(G / ms_p1g_max / 1e6)},
                       "note": "tc_push_peer (NVLink stores from every SM into the neighbour's IPC-mapped slot, "
                               "mailbox publish) + tc_peer_wait on the receiver; no NCCL, no host sync"}
    del big
    return out


def lossy_probe(tc, ctx, X, Y, A, R, rec, s, dev, peak, N=5, k=0.01, reps=3):
    """NEXT row 3: the paper's lossy differential on this rank's shard size — compress
    one fp32 gradient of the shard (sparse form), decompress it, and replay N payloads through Adam
    fused vs sequentially.  Runs after the step measurements in the step's own buffers (viewed as
    fp32 gradient / master / m / v / scratch; the bf16 weight segment as the 16-bit copy)."""
    import torch

    n = X[1].numel()
    g = Y[1].view(torch.float32)
    master, m, v, w16 = X[1].view(torch.float32), X[2].view(torch.float32), X[3].view(torch.float32), X[0]
    if w16.numel() != n or any(t.numel() != n for t in (Y[1], X[2], X[3], A[0], A[1], A[2], A[3], R[1])):
        return {"skipped": "needs four equal-length segments"}
    dense = R[1].view(torch.float32)
    slot = (rec.numel() // N) & ~15
    cap = tc.grad_bound(n, k=k)
    need = (min(cap, int(6.5 * k * 3 * n)) + 15) & ~15
    if slot < need:  # the step's record slots are sized for its records: payload slots of their own
        if torch.cuda.mem_get_info(dev)[0] < N * need + (2 << 30):
            return {"skipped": "no device memory for the payload slots"}
        rec = torch.empty(N * need, dtype=torch.uint8, device=dev)
        slot = need
    pays = [rec[j * slot:(j + 1) * slot] for j in range(N)]
    ob = torch.zeros(N, dtype=torch.int64, device=dev)
    ev = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731

    def timed(fn):
        out = []
        for _ in range(reps):
            a, b = ev(), ev()
            a.record(s)
            fn()
            b.record(s)
            s.synchronize()
            out.append(a.elapsed_time(b))
        return statistics.median(out)

    with torch.cuda.stream(s):
        for j in range(N):
            torch.randn(n, out=g, generator=torch.Generator(device=dev).manual_seed(j))
            g.mul_(1e-2)
            tc.grad_compress(ctx, g, j, pays[j], ob[j:j + 1], stream=s, k=k)
        torch.randn(n, out=master, generator=torch.Generator(device=dev).manual_seed(99))
        m.zero_()
        v.zero_()
        w16.zero_()
        snap = [A[1].view(torch.float32), A[2].view(torch.float32), A[3].view(torch.float32), A[0]]
        for dst, src in zip(snap, (master, m, v, w16)):
            dst.copy_(src)
    s.synchronize()
    ctx.check(s)
    nb = [int(x) for x in ob.tolist()]
    tmp_ob = torch.zeros(1, dtype=torch.int64, device=dev)
    ms_c = timed(lambda: tc.grad_compress(ctx, g, N - 1, pays[N - 1], tmp_ob, stream=s, k=k))
    ms_d = timed(lambda: tc.grad_decompress(ctx, pays[0], nb[0], dense, stream=s))

    def reset():
        with torch.cuda.stream(s):
            for dst, src in zip((master, m, v, w16), snap):
                dst.copy_(src)

    f_ms, s_ms = [], []
    same = True
    for _ in range(reps):
        reset()
        a, b = ev(), ev()
        a.record(s)
        tc.adam_replay(ctx, master, m, v, w16, pays, nb, 1, dense, stream=s)
        b.record(s)
        s.synchronize()
        f_ms.append(a.elapsed_time(b))
        fused = [Y[1].view(torch.float32), Y[2].view(torch.float32), Y[3].view(torch.float32)]
        with torch.cuda.stream(s):  # the gradient buffer is free by now: keep the fused result there
            for dst, src in zip(fused, (master, m, v)):
                dst.copy_(src)
        reset()
        a, b = ev(), ev()
        a.record(s)
        for j in range(N):
            tc.grad_decompress(ctx, pays[j], nb[j], dense, stream=s)
            tc.adam_step(ctx, master, m, v, w16, dense, 1 + j, stream=s)
        b.record(s)
        s.synchronize()
        s_ms.append(a.elapsed_time(b))
        with torch.cuda.stream(s):
            for x, y in zip((master, m, v), fused):
                for o in range(0, n, 1 << 27):  # slices: no full-size temporaries
                    same = same and torch.equal(x[o:o + (1 << 27)], y[o:o + (1 << 27)])
    ctx.check(s)
    kept = (nb[-1] - 80) // 6
    c_b, d_b = 4 * n + nb[-1] + 6 * kept, 4 * n + nb[0]
    fm, sm = statistics.median(f_ms), statistics.median(s_ms)
    f_b = 24 * n + sum(nb[:-1]) + (4 * n + nb[-1]) + (4 * n + 24 * n + 2 * n)
    return {"n": n, "N": N, "k": k, "payload_bytes": nb[0], "kept": kept,
            "compress": {"ms": round(ms_c, 3), "gbs": round(c_b / ms_c / 1e6, 1),
                         "frac_hbm": round(c_b / ms_c / 1e6 / peak, 4)},
            "decompress": {"ms": round(ms_d, 3), "gbs": round(d_b / ms_d / 1e6, 1),
                           "frac_hbm": round(d_b / ms_d / 1e6 / peak, 4)},
            "replay_fused_ms": round(fm, 3), "replay_fused_gbs": round(f_b / fm / 1e6, 1),
            "replay_sequential_ms": round(sm, 3), "speedup_fused_vs_sequential": round(sm / fm, 3),
            "fused_equals_sequential": bool(same),
            "note": "NEXT row 3 (DESIGN.md §12): sampled-threshold top-k (k = 0.01) FP16+INT32 payloads of an fp32 "
                    "gradient the size of one shard segment; fused = N-1 Adam steps in one pass + the native step; "
                    "paper context: 16.6 s fused vs 26.0 s sequential (A800, 20B, 100 steps, P:586)"}


def run_e2e(args, tc, ctx, dev, sizes, wb, X, Y, A, R, recs, obytes, host_ring, rec_cap, T, C, state, world,
            s_comp, s_copy):
    """e2e through the C ABI with host buffers: per step H2D of the new state version from pinned
    host memory, encode, D2H of the record (the result), fold onto the replica."""
    import torch
    import torch.distributed as dist

    steps = min(args.steps, args.e2e_steps)
    # pinned host copies of both state versions; every rank must get them before any collective
    try:
        bX = [tc.HostBuffer(x.numel() * x.element_size()) for x in X]
        bY = [tc.HostBuffer(y.numel() * y.element_size()) for y in Y]
        got = 1
    except tc.TcError:
        bX = bY = []
        got = 0
    if world > 1:
        t = torch.tensor([got], dtype=torch.int32, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MIN)
        got = int(t.item())
    if not got:
        for b in bX + bY:
            b.free()
        raise RuntimeError("pinned host memory for two state versions per rank is not available")
    hX = [b.view(x.dtype) for b, x in zip(bX, X)]
    hY = [b.view(y.dtype) for b, y in zip(bY, Y)]
    for h, d in zip(hX + hY, X + Y):
        h.copy_(d)
    torch.cuda.synchronize()
    if min(h.numel() for h in host_ring) < 1:
        return None
    # Two landing buffers: the H2D of step k+1 (copy stream) runs while step k encodes, stages its
    # record and folds (compute stream), so the step costs max(H2D, device work) instead of their
    # sum.  The landing buffers are Y (for the steps whose new version is Y's content) and X (for
    # X's): every step still moves its whole state version over PCIe and the encode waits for it,
    # and no HBM beyond the step's own buffers is needed (cfg2 leaves < 22 GB free here).
    bufs = [Y, X]
    nb = 2
    landed = [torch.cuda.Event() for _ in range(nb)]   # H2D into bufs[i] complete
    freed = [None] * nb                                 # encode done reading bufs[i]
    ev = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731
    h2d = d2h = 0

    def src_of(content):
        return hY if content == "X" else hX

    def issue_h2d(i, src, stream):
        nonlocal h2d
        if freed[i] is not None:
            stream.wait_event(freed[i])
        for hs, ds in zip(src, bufs[i]):
            tc.stage_host(ds, hs, hs.numel() * hs.element_size(), tc.H2D, stream=stream)
            h2d += hs.numel() * hs.element_size()
        landed[i].record(stream)

    def buf_of(content):  # the step whose current content is `content` lands in bufs[i]
        return 0 if content == "X" else 1

    def one(k, last):
        nonlocal d2h
        i = buf_of(state["content"])
        if not last:  # prefetch the next step's state version (the content flips every step)
            nxt = "Y" if state["content"] == "X" else "X"
            issue_h2d(buf_of(nxt), src_of(nxt), s_copy)
        s_comp.wait_event(landed[i])
        dst = bufs[i]
        v = state["ref_version"] + 1
        tc.diff_encode(ctx, A, dst, recs[0], obytes[0], v, v - 1, T, C, True, stream=s_comp,
                       index_mode=state["index"])
        e = torch.cuda.Event()
        e.record(s_comp)
        freed[i] = e
        e.synchronize()
        n = int(obytes[0].item())
        if n > host_ring[0].nbytes:
            raise RuntimeError("record exceeds the host ring slot")
        tc.stage_host(host_ring[0], recs[0], n, tc.D2H, stream=s_comp)
        d2h += n + 8
        tc.diff_apply(ctx, R, state["rest_version"], [recs[0]], [n], stream=s_comp)
        state["ref_version"] = v
        state["rest_version"] = v
        state["content"] = "Y" if state["content"] == "X" else "X"

    # warm (the first H2D of each pinned buffer, into every landing buffer)
    issue_h2d(buf_of(state["content"]), src_of(state["content"]), s_comp)
    one(0, True)
    issue_h2d(buf_of(state["content"]), src_of(state["content"]), s_comp)
    s_comp.synchronize()
    s_copy.synchronize()
    if world > 1:
        dist.barrier()
    h2d = d2h = 0
    t0, t1 = ev(), ev()
    t0.record(s_comp)
    s_copy.wait_event(t0)  # prologue: step 1's H2D, ordered after t0
    issue_h2d(buf_of(state["content"]), src_of(state["content"]), s_copy)
    for k in range(1, steps + 1):
        one(k, k == steps)
    t1.record(s_comp)
    s_comp.synchronize()
    ctx.check(s_comp)
    ms = t0.elapsed_time(t1)
    t = torch.tensor([ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms = float(t.item()) / steps
    W = sum(n * w for n, w in zip(sizes, wb))
    # the ceiling of this e2e: a plain H2D of one state version alone (same pinned buffers, same call)
    c0, c1 = ev(), ev()
    c0.record(s_copy)
    for hs, ds in zip(src_of(state["content"]), bufs[buf_of(state["content"])]):
        tc.stage_host(ds, hs, hs.numel() * hs.element_size(), tc.H2D, stream=s_copy)
    c1.record(s_copy)
    s_copy.synchronize()
    h2d_gbs = W / (c0.elapsed_time(c1) * 1e-3) / 1e9
    del hX, hY
    for b in bX + bY:
        b.free()
    return {"value": round(world * W / (ms * 1e-3) / 1e9, 2), "unit": "GB/s", "steps": steps,
            "ms_per_step": round(ms, 3), "h2d_bytes_per_step": h2d // steps, "d2h_bytes_per_step": d2h // steps,
            "landing_buffers": nb, "plain_h2d_gbs": round(h2d_gbs, 2),
            "frac_h2d": round(W / (ms * 1e-3) / 1e9 / h2d_gbs, 3),
            "note": "H2D of the new state version from pinned host (copy stream, one step ahead, two landing "
                    "buffers) + encode + D2H record + fold (compute stream)"}


# the measured floor of a scattered fold: the pure scatter of sorted (position, value) entries into a
# 16 GB fp32 state (tools/fold_probe.cu, profiles/rd4e_fold_probe_scatter.txt), G entries/s by density
SCATTER_FLOOR = {0.001: 20.43, 0.01: 23.61, 0.03: 33.80}


# the measured floor of a chained fold: read-modify-write of ONLY the touched 32-byte sectors of a
# 16 GB fp32 state (tools/fold_probe.cu rmw16, profiles/rd4e_fold_probe_scatter.txt), ms per GB of
# state by union density
RMW_FLOOR_MS_PER_GB = {0.0773: 6.272 / 16.0}


def touched_floor(union_frac, state_bytes, fold_ms):
    """The chain fold against the best valid touched-sector pattern measured at its density."""
    for p, msgb in RMW_FLOOR_MS_PER_GB.items():
        if abs(union_frac - p) < 0.005:
            floor = msgb * state_bytes / 1e9
            return {"floor_ms": round(floor, 3), "frac_of_floor": round(floor / fold_ms, 3),
                    "source": "tools/fold_probe.cu rmw16 at p = %.4f (profiles/rd4e_fold_probe_scatter.txt, "
                              "profiles/rd2_fold_floor_probe.md): at this density the touched sectors span 92 %% "
                              "of the 128-byte lines, so DRAM reads ~0.96 of the state" % p}
    return None


def scatter_roofline(changed, fold_ms, f):
    """The step's N = 1 fold against the random-store roofline, where measured."""
    peak = SCATTER_FLOOR.get(f)
    if not changed or not fold_ms or peak is None:
        return None
    got = changed / fold_ms / 1e6
    return {"unit": "G entries/s", "achieved": round(got, 2), "peak": peak, "frac": round(got / peak, 3),
            "peak_source": "pure scatter of sorted u32 positions + values, one 4-byte store each, at this "
                           "density (tools/fold_probe.cu, profiles/rd4e_fold_probe_scatter.txt)"}


def load_traffic(workload, f):
    p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if not os.path.exists(p):
        return {}
    with open(p) as fh:
        d = json.load(fh)
    key = f"{workload}_f{f}"
    return d.get(key, {})


# ------------------------------------------------------------- the oracle arm -----------
def oracle_sample(workload, f, sample_words):
    """A bounded sample of the workload: words [0, sample_words) of every segment of shard 0."""
    sizes, wb = synth.shard_layout(workload, 0)
    sizes = [min(n, sample_words) for n in sizes]
    seed = synth.SEED0
    X = synth.state(sizes, wb, seed, 0, f)
    Y = synth.state(sizes, wb, seed, 1, f)
    return sizes, wb, X, Y


def time_oracle(workload, f, sample_words, steps):
    import oracle

    sizes, wb, X, Y = oracle_sample(workload, f, sample_words)
    W = sum(n * w for n, w in zip(sizes, wb))
    ref = [a.copy() for a in X]
    rest = [a.copy() for a in X]
    times = []
    ver = 0
    for k in range(steps):
        cur = Y if k % 2 == 0 else X
        t0 = time.perf_counter()
        rc, rec = oracle.encode(ref, cur, version=ver + 1, ref_version=ver)
        rc2, _ = oracle.apply(rest, ver, rec)
        times.append(time.perf_counter() - t0)
        assert rc == 0 and rc2 == 0
        ver += 1
    return W, times, sizes


def time_oracle_parallel(workload, f, sample_words, steps, threads):
    """The same oracle calls on all host cores: the sample's segments are cut into `threads` slices
    per segment (whole 4096-word tiles), and each thread encodes + restores its slices as their own
    one-segment shards (the oracle as it stands; ctypes releases the GIL around each C call)."""
    from concurrent.futures import ThreadPoolExecutor

    import oracle

    sizes, wb, X, Y = oracle_sample(workload, f, sample_words)
    W = sum(n * w for n, w in zip(sizes, wb))
    jobs = []
    for s, n in enumerate(sizes):
        step_ = -(-n // threads + 4095) // 4096 * 4096
        for a in range(0, n, step_):
            b = min(n, a + step_)
            jobs.append({"X": X[s][a:b], "Y": Y[s][a:b], "ref": X[s][a:b].copy(), "rest": X[s][a:b].copy()})

    def one(j, k):
        cur = j["Y"] if k % 2 == 0 else j["X"]
        rc, rec = oracle.encode([j["ref"]], [cur], version=k + 1, ref_version=k)
        rc2, _ = oracle.apply([j["rest"]], k, rec)
        assert rc == 0 and rc2 == 0

    times = []
    with ThreadPoolExecutor(threads) as ex:
        for k in range(steps):
            t0 = time.perf_counter()
            list(ex.map(lambda j: one(j, k), jobs))
            times.append(time.perf_counter() - t0)
    return W, times, sizes, len(jobs)


def cpu_baseline(workload, args):
    W, times, sizes = time_oracle(workload, args.f, args.sample_words, args.oracle_steps)
    t = statistics.median(times)
    ncpu = len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else (os.cpu_count() or 1)
    Wp, times_p, _, njobs = time_oracle_parallel(workload, args.f, args.sample_words, args.oracle_steps + 1, ncpu)
    tp = statistics.median(times_p[1:])
    return {"value": round(W / t / 1e9, 4), "unit": "GB/s", "cores": 1, "kind": "oracle",
            "sample": f"words [0, {sizes[0]}) of each of {len(sizes)} segments of the {workload} shard "
                      f"({W / 1e6:.0f} MB of state); encode + restore per step; median of {len(times)}",
            "all_cores": {"value": round(Wp / tp / 1e9, 4), "unit": "GB/s", "cores": ncpu, "kind": "oracle",
                          "sample": f"the same sample cut into {njobs} slices (whole tiles), one thread per core; "
                                    f"median of {len(times_p) - 1} after one warm-up"},
            "host": host_desc()}


def host_desc():
    try:
        with open("/proc/cpuinfo") as fh:
            model = next((ln.split(":", 1)[1].strip() for ln in fh if ln.startswith("model name")), "?")
    except Exception:
        model = "?"
    return {"nproc": os.cpu_count(), "cpu": model}


def run_reference(args):
    rank, world, local = dist_env()
    if rank != 0:
        return
    workload = args.workload or ("cfg2" if world == 1 else "cfg3")
    # the oracle on all of the box's host cores (slices of the sample, one thread per core)
    ncpu = len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else (os.cpu_count() or 1)
    W, times, sizes, njobs = time_oracle_parallel(workload, args.f, args.sample_words, args.warmup + args.steps, ncpu)
    times = times[args.warmup:]
    ms = 1e3 * sum(times) / len(times)
    v = round(W / (ms * 1e-3) / 1e9, 4)
    res = {
        "impl": "reference", "metric": METRIC, "value": v, "unit": "GB/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms, 3), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "u16+u32 (bitwise)", "data": "synthetic",
        "config": {"workload": WORKLOADS.get(workload, workload), "f": args.f,
                   "sample": f"words [0, {sizes[0]}) of each segment ({W / 1e6:.0f} MB of state) per step"},
        "cpu_baseline": {"value": v, "unit": "GB/s", "cores": ncpu, "kind": "oracle",
                         "sample": f"words [0, {sizes[0]}) of each of {len(sizes)} segments, cut into {njobs} "
                                   f"slices over {ncpu} threads; encode + restore",
                         "host": host_desc()},
        "e2e": {"value": v, "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    emit(res)


def main():
    _private_stdout()
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default=None, choices=[None, "cfg1", "cfg2", "cfg3", "cfg4", "cfg5"])
    ap.add_argument("--stream-chunks", type=int, default=4, help="cfg5: chunks per streamed encode run")
    ap.add_argument("--f", type=float, default=0.01)
    ap.add_argument("--structure", type=int, default=0)
    ap.add_argument("--tile-words", type=int, default=4096)
    ap.add_argument("--chunk-words", type=int, default=1 << 28)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--overlap-standby", type=int, default=0,
                    help="Checkpointer: the standby fold of record k-1 on its own stream beside encode k")
    ap.add_argument("--overlap-fold", type=int, default=0,
                    help="N = 1: fold record k-1 on a high-priority stream beside encode k")
    ap.add_argument("--timeline", action="store_true")
    ap.add_argument("--format", default="adaptive", choices=["mask", "index", "full", "adaptive"],
                    help="record format: mask, index (u16 positions), or adaptive per step from density")
    ap.add_argument("--restore-chain", type=int, default=8, help="records in the chained-restore probe (0: off)")
    ap.add_argument("--e2e-steps", type=int, default=6)
    ap.add_argument("--lossy", type=int, default=1,
                    help="N=1: also measure the paper's lossy differential (NEXT row 3) in the step's buffers")
    ap.add_argument("--push-ctas", type=int, default=16,
                    help="CTAs of the Tier-2 NVLink push inside the step (fewer = less interference)")
    ap.add_argument("--dev-slots", type=int, default=3,
                    help="device record slots of the Checkpointer (a slot is reused once its Tier-1 copy is done)")
    ap.add_argument("--t2-fused", type=int, default=0,
                    help="push mode: 1 = the encoder writes the record into the neighbour's slot (fused), "
                         "0 = a separate push kernel on the Tier-2 stream, beside the fold and the next encode "
                         "(default: with the host one step ahead it is the faster step, N = 2: 5.92 vs 6.18 ms, "
                         "profiles/rd7a_t2_fused_ab.txt)")
    ap.add_argument("--tier2", default="push", choices=["push", "nccl"],
                    help="Tier-2 replication: NVLink stores into the neighbour's IPC slot, or NCCL send/recv")
    ap.add_argument("--recovery", type=int, default=None,
                    help="simulated-failure recovery probe (Tier-1 and, N > 1, Tier-2); default: on for cfg4")
    ap.add_argument("--fold-dense-permille", type=int, default=None,
                    help="restore strategy threshold (tc_ctx_set_fold_dense_permille); default: libtc's")
    ap.add_argument("--ahead", type=int, default=None,
                    help="Checkpointer runs the host one step ahead of the device (default on; N = 2: 6.08 vs "
                         "6.27 ms per step with the fused emit, 5.92 vs 6.19 with the push kernel, profiles/rd5u_*, "
                         "rd7a_*)")
    ap.add_argument("--cpu-baseline", type=int, default=1)
    ap.add_argument("--numa-bind", type=int, default=1,
                    help="N > 1: bind each rank to its GPU's NUMA node before the pinned buffers are allocated")
    ap.add_argument("--sample-words", type=int, default=1 << 25)
    ap.add_argument("--oracle-steps", type=int, default=3)
    args = ap.parse_args()
    if args.warmup < 3 and args.impl == "ours":
        print("warning: --warmup < 3 violates the timing rules", file=sys.stderr)
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
