"""Probe: does running kernel B (emit) of one part of the state beside kernel A (compare) of the
next part pay?  cfg2 state, one tc_diff_encode_range per segment:

  whole    tc_diff_encode of the state (one A, P, B sequence)
  serial   the 4 segment ranges one after another on one stream / context
  overlap  segments alternate between 2 streams with their own contexts (scratch), so the next
           segment's kernel A can run beside this segment's kernels P and B

    python tools/overlap_probe.py --f 0.01 0.1 0.3
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
    ap.add_argument("--f", type=float, nargs="+", default=[0.01, 0.1, 0.3])
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--index", action="store_true")
    a = ap.parse_args()
    sizes, wb = synth.shard_layout("cfg2", 0)
    dev = torch.device("cuda", 0)
    T, C = 4096, 1 << 28

    def alloc(n, w):
        return torch.empty(n, dtype=torch.int16 if w == 2 else torch.int32, device=dev)

    X = [alloc(n, w) for n, w in zip(sizes, wb)]
    Y = [alloc(n, w) for n, w in zip(sizes, wb)]
    R = [alloc(n, w) for n, w in zip(sizes, wb)]
    caps = [tc.diff_bound_range(n, w, 0, -(-n // C), T, C, a.index) for n, w in zip(sizes, wb)]
    outs = [torch.empty(c, dtype=torch.uint8, device=dev) for c in caps]
    obs = [torch.zeros(1, dtype=torch.int64, device=dev) for _ in sizes]
    whole = torch.empty(tc.diff_bound(sizes, wb, T, C, a.index), dtype=torch.uint8, device=dev) \
        if sum(caps) < 40e9 else None
    ob = torch.zeros(1, dtype=torch.int64, device=dev)
    ctxs = [tc.Ctx(0), tc.Ctx(0)]
    streams = [torch.cuda.Stream(dev), torch.cuda.Stream(dev)]
    for f in a.f:
        for s in range(len(sizes)):
            tc.synth_base(X[s], synth.SEED0, s)
            Y[s].copy_(X[s])
            tc.synth_step(Y[s], synth.SEED0, s, 1, synth.p53_of(f), synth.S1_IID)
        torch.cuda.synchronize()
        res = {"f": f, "index": a.index}
        for mode in ("whole", "serial", "overlap", "whole"):
            if mode == "whole" and whole is None:
                continue
            ts = []
            for rep in range(a.reps + 1):
                for x, r in zip(X, R):
                    r.copy_(x)
                torch.cuda.synchronize()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(streams[0])
                if mode == "whole":
                    tc.diff_encode(ctxs[0], R, Y, whole, ob, 1, 0, T, C, True, stream=streams[0], index_mode=a.index)
                else:
                    streams[1].wait_event(e0)
                    for s in range(len(sizes)):
                        k = s % 2 if mode == "overlap" else 0
                        tc.diff_encode_range(ctxs[k], R[s], Y[s], s, 0, -(-sizes[s] // C), outs[s], obs[s], 1, 0,
                                             T, C, True, stream=streams[k], index_mode=a.index)
                    streams[0].wait_stream(streams[1])
                e1.record(streams[0])
                torch.cuda.synchronize()
                for c in ctxs:
                    c.check()
                if rep:
                    ts.append(e0.elapsed_time(e1))
            res[mode] = round(statistics.median(ts), 3)
            if mode != "whole":
                res[mode + "_bytes"] = sum(int(o.item()) for o in obs)
            else:
                res["whole_bytes"] = int(ob.item())
        print(json.dumps(res), flush=True)


if __name__ == "__main__":
    main()
