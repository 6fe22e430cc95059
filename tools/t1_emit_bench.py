"""Tier-1 emit options on one GPU: how a record
reaches page-locked host memory.

  copy   tc_diff_encode into HBM, then the copy engine (tc_stage_host, cudaMemcpyAsync D2H)
  push   tc_diff_encode into HBM, then tc_push_peer with the host buffer as destination (SM
         stores over PCIe, the record re-read from HBM)
  fused  tc_diff_encode_push with the host buffer (and a host mailbox) as the peer: the encode
         kernels store every record byte into mapped pinned memory as they write it to HBM

For each: the latency of one checkpoint (encode start -> record in host memory, one stream) and
the per-step time when steps are pipelined (copy of record k beside the encode of k+1 on a
second stream, as the Checkpointer runs it).  Every variant's host bytes are compared with the
device record.  cfg2 state (21.8 GB), S1 changes, advance_ref on.

    python tools/t1_emit_bench.py --f 0.001 0.01 0.05 --steps 8
"""
import argparse
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import synth  # noqa: E402
from paper_2605_17821_b200 import tc  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="cfg2")
    ap.add_argument("--f", type=float, nargs="+", default=[0.001, 0.01, 0.05])
    ap.add_argument("--steps", type=int, default=8)
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--format", default="index", choices=["index", "mask"])
    a = ap.parse_args()
    sizes, wb = synth.shard_layout(a.workload, 0)
    dev = torch.device("cuda", 0)
    T, C = 4096, 1 << 28
    index = a.format == "index"

    def alloc(n, w):
        return torch.empty(n, dtype=torch.int16 if w == 2 else torch.int32, device=dev)

    X = [alloc(n, w) for n, w in zip(sizes, wb)]
    Y = [alloc(n, w) for n, w in zip(sizes, wb)]
    R = [alloc(n, w) for n, w in zip(sizes, wb)]
    ctx = tc.Ctx(0)
    s_enc = torch.cuda.Stream(dev)
    s_cp = torch.cuda.Stream(dev)
    d2h_gbs = None
    for f in a.f:
        for s in range(len(sizes)):
            tc.synth_base(X[s], synth.SEED0, s)
            Y[s].copy_(X[s])
            tc.synth_step(Y[s], synth.SEED0, s, 1, synth.p53_of(f), synth.S1_IID)
        torch.cuda.synchronize()
        # the record size of this f (deterministic: X -> Y)
        probe = torch.empty(tc.diff_bound(sizes, wb, T, C, index), dtype=torch.uint8, device=dev)
        ob = torch.zeros(1, dtype=torch.int64, device=dev)
        for x, r in zip(X, R):
            r.copy_(x)
        tc.diff_encode(ctx, R, Y, probe, ob, 1, 0, T, C, True, index_mode=index)
        ctx.check()
        n = int(ob.item())
        slot = (n + 4095) // 4096 * 4096 + 4096
        outs = [probe[:slot]] + [torch.empty(slot, dtype=torch.uint8, device=dev) for _ in range(1)]
        obs = [torch.zeros(1, dtype=torch.int64, device=dev) for _ in range(2)]
        hosts = [tc.HostBuffer(slot) for _ in range(2)]
        mails = [tc.HostBuffer(16) for _ in range(2)]
        ref_bytes = probe[:n].cpu()
        res = {"f": f, "format": a.format, "record_bytes": n}

        def reset_ref():
            for x, r in zip(X, R):
                r.copy_(x)

        def enc(k, variant, stream):
            if variant == "fused":
                tc.diff_encode_push(ctx, R, Y, outs[k], obs[k], 1, 0, hosts[k], slot, mails[k], T, C, True,
                                    stream=stream, index_mode=index)
            else:
                tc.diff_encode(ctx, R, Y, outs[k], obs[k], 1, 0, T, C, True, stream=stream, index_mode=index)

        def move(k, variant, stream):
            if variant == "copy":
                tc.stage_host(hosts[k].tensor, outs[k], n, 0, stream=stream)
            elif variant == "push":
                tc.push_peer(ctx, outs[k], obs[k], hosts[k], slot, mails[k], 1, stream=stream)

        for variant in ("copy", "push", "fused"):
            lat, pipe = [], []
            for rep in range(a.reps + 1):
                # latency: one checkpoint, encode -> host, one stream (ref reset outside the timing:
                # X -> Y again, so every encode has the same record)
                reset_ref()
                torch.cuda.synchronize()
                mails[0].tensor.zero_()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                with torch.cuda.stream(s_enc):
                    e0.record(s_enc)
                    enc(0, variant, s_enc)
                    move(0, variant, s_enc)
                    e1.record(s_enc)
                s_enc.synchronize()
                ctx.check(s_enc)
                if rep:
                    lat.append(e0.elapsed_time(e1))
                # host bytes == the device record; the mailbox (push, fused) carries {n, version}
                assert torch.equal(hosts[0].tensor[:n], ref_bytes), f"{variant}: host bytes != record"
                if variant != "copy":
                    assert mails[0].tensor.view(torch.int64).tolist() == [n, 1], f"{variant}: mailbox"
                # pipelined steps: encode k+1 beside the move of record k (two slots); advance_ref
                # off here (every step re-encodes X -> Y: same record, same work)
                torch.cuda.synchronize()
                done = [torch.cuda.Event() for _ in range(2)]
                moved = [torch.cuda.Event() for _ in range(2)]
                p0, p1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                p0.record(s_enc)
                for k in range(a.steps):
                    j = k % 2
                    if k >= 2:
                        s_enc.wait_event(moved[j])
                    if variant == "fused":
                        tc.diff_encode_push(ctx, X, Y, outs[j], obs[j], 1, 0, hosts[j], slot, mails[j], T, C,
                                            False, stream=s_enc, index_mode=index)
                        moved[j].record(s_enc)
                    else:
                        tc.diff_encode(ctx, X, Y, outs[j], obs[j], 1, 0, T, C, False, stream=s_enc,
                                       index_mode=index)
                        done[j].record(s_enc)
                        s_cp.wait_event(done[j])
                        move(j, variant, s_cp)
                        moved[j].record(s_cp)
                s_enc.wait_stream(s_cp)
                p1.record(s_enc)
                torch.cuda.synchronize()
                ctx.check(s_enc)
                if rep:
                    pipe.append(p0.elapsed_time(p1) / a.steps)
            res[variant] = {"latency_ms": round(statistics.median(lat), 3),
                            "step_ms_pipelined": round(statistics.median(pipe), 3),
                            "t1_gbs_latency": round(n / statistics.median(lat) / 1e6, 1)}
        # the plain D2H copy of the record alone (the PCIe ceiling of the copy variant)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ts = []
        for _ in range(3):
            e0.record()
            tc.stage_host(hosts[0].tensor, outs[0], n, 0)
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        d2h_gbs = n / min(ts) / 1e6
        res["d2h_alone_ms"] = round(min(ts), 3)
        res["d2h_gbs"] = round(d2h_gbs, 1)
        print(json.dumps(res), flush=True)
        for h in hosts + mails:
            h.free()
        del probe, outs
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
