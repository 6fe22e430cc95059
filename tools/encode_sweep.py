"""Encoder sweep on one GPU: for each change fraction f, time tc_diff_encode of the workload's state
(X -> Y, S1 structure) under each library build (TC_LIB_PATH=exp/libtc_*.so for A/B runs of
experiment builds; --libs lists labels only, the caller sets the path per run), and print the
SURVEY §8(d) sector-granular HBM fraction.

    python tools/encode_sweep.py --workload cfg2 --f 0.01 0.1 0.3 1.0 --advance 1
Prints one JSON line per (f, variant) on stdout.
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


def headers(out, n):
    pos, recs = 0, []
    while pos < n:
        h = out[pos: pos + 64].cpu().numpy()
        w, flags = int(h[6]), int(h[7])
        T = int(h[8:12].view("<u4")[0])
        m, count, total = (int(h[a:a + 8].view("<u8")[0]) for a in (24, 32, 56))
        recs.append((m, w, T, count, flags))
        pos += total
    return recs


def enc_bytes(recs, advance):
    b = 0
    for m, w, T, count, flags in recs:
        W = m * w
        if flags == 5:  # full record: read cur, write the values (+ ref <- cur): no compare
            b += 64 + 2 * W + (W if advance else 0)
            continue
        meta = 64 + 4 * (-(-m // T) + 1) + (2 * count if flags & 2 else 4 * -(-m // 32))
        b += 2 * W + meta + w * count
        if advance and m:
            b += W * (1 - (1 - count / m) ** (32 // w))
    return b


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="cfg2")
    ap.add_argument("--f", type=float, nargs="+", default=[0.01, 0.1, 0.3, 1.0])
    ap.add_argument("--defer", type=int, nargs="+", default=[0], help="(kept for the log format)")
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--advance", type=int, default=1)
    ap.add_argument("--index", action="store_true")
    ap.add_argument("--full", action="store_true", help="full records (every word, kernel F)")
    ap.add_argument("--structure", type=int, default=synth.S1_IID)
    a = ap.parse_args()
    peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"]
    sizes, wb = synth.shard_layout(a.workload, 0)
    dev = torch.device("cuda", 0)
    T, C = 4096, 1 << 28

    def alloc(n, w):
        return torch.empty(n, dtype=torch.int16 if w == 2 else torch.int32, device=dev)

    X = [alloc(n, w) for n, w in zip(sizes, wb)]
    Y = [alloc(n, w) for n, w in zip(sizes, wb)]
    R = [alloc(n, w) for n, w in zip(sizes, wb)] if a.advance else X
    cap = tc.diff_bound(sizes, wb, T, C, a.index, full=a.full)
    out = torch.empty(cap, dtype=torch.uint8, device=dev)
    first = torch.empty(cap, dtype=torch.uint8, device=dev)
    ob = torch.zeros(1, dtype=torch.int64, device=dev)
    W = sum(n * w for n, w in zip(sizes, wb))
    ctx = tc.Ctx(0)
    for f in a.f:
        for s in range(len(sizes)):
            tc.synth_base(X[s], synth.SEED0, s)
            Y[s].copy_(X[s])
            tc.synth_step(Y[s], synth.SEED0, s, 1, synth.p53_of(f), a.structure)
        torch.cuda.synchronize()
        n0 = None
        for d in a.defer:
            ms = []
            for r in range(a.reps + 1):
                if a.advance:
                    for x, r_ in zip(X, R):
                        r_.copy_(x)
                torch.cuda.synchronize()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                tc.diff_encode(ctx, R, Y, out, ob, 1, 0, T, C, bool(a.advance), index_mode=a.index, full=a.full)
                e1.record()
                ctx.check()
                if r:
                    ms.append(e0.elapsed_time(e1))
            n = int(ob.item())
            same = None
            if n0 is None:
                n0 = n
                first[:n].copy_(out[:n])
                recs = headers(out, n)
            else:
                same = n == n0 and torch.equal(out[:n], first[:n])
            if a.advance:
                same_ref = all(torch.equal(r_, y) for r_, y in zip(R, Y))
                same = same_ref if same is None else (same and same_ref)
            t = statistics.median(ms)
            b = enc_bytes(recs, a.advance)
            print(json.dumps({"f": f, "defer": d, "index": a.index, "full": a.full, "advance": a.advance, "ms": round(t, 3),
                              "ms_all": [round(x, 3) for x in ms], "record_bytes": n,
                              "alg_bytes": int(b), "gbs": round(b / t / 1e6, 1), "frac": round(b / t / 1e6 / peak, 3),
                              "state_gbs": round(W / t / 1e6, 1), "identical_to_first": same}), flush=True)


if __name__ == "__main__":
    main()
