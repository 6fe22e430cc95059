"""Minimal driver for ncu / compute-sanitizer: build one workload's state on the device, then run
`--reps` encodes (advance_ref=0 so every rep does identical work) and `--reps` folds of the
produced record.  Prints per-launch CUDA-event times.

    python tools/prof_kernels.py --workload cfg2 --f 0.01 --reps 3
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import synth  # noqa: E402
from paper_2605_17821_b200 import tc  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="cfg2")
    ap.add_argument("--f", type=float, default=0.01)
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--fold-n", type=int, default=1)
    ap.add_argument("--tile-words", type=int, default=4096)
    ap.add_argument("--scale", type=float, default=1.0, help="shrink every segment (sanitizer runs)")
    ap.add_argument("--no-fold", action="store_true")
    ap.add_argument("--index", action="store_true", help="index-mode records")
    ap.add_argument("--dense-permille", type=int, default=None, help="tc_ctx_set_fold_dense_permille")
    a = ap.parse_args()
    sizes, wb = synth.shard_layout(a.workload, 0)
    sizes = [max(1, int(n * a.scale)) for n in sizes]
    dev = torch.device("cuda", 0)
    p53 = synth.p53_of(a.f)

    def alloc(n, w):
        return torch.empty(n, dtype=torch.int16 if w == 2 else torch.int32, device=dev)

    X = [alloc(n, w) for n, w in zip(sizes, wb)]
    Y = [alloc(n, w) for n, w in zip(sizes, wb)]
    for s in range(len(sizes)):
        tc.synth_base(X[s], synth.SEED0, s)
        Y[s].copy_(X[s])
        tc.synth_step(Y[s], synth.SEED0, s, 1, p53)
    torch.cuda.synchronize()
    ctx = tc.Ctx(0)
    if a.dense_permille is not None:
        ctx.set_fold_dense_permille(a.dense_permille)
    cap = tc.diff_bound(sizes, wb, a.tile_words, 1 << 28, a.index)
    out = torch.empty(cap, dtype=torch.uint8, device=dev)
    ob = torch.zeros(1, dtype=torch.int64, device=dev)
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2 * a.reps)]
    for r in range(a.reps):
        ev[2 * r].record()
        tc.diff_encode(ctx, X, Y, out, ob, 1, 0, a.tile_words, 1 << 28, advance_ref=False, index_mode=a.index)
        ev[2 * r + 1].record()
    ctx.check()
    n = int(ob.item())
    W = sum(n_ * w for n_, w in zip(sizes, wb))
    print("encode ms:", [round(ev[2 * r].elapsed_time(ev[2 * r + 1]), 3) for r in range(a.reps)],
          "record bytes", n, "state GB", W / 1e9)
    if a.no_fold:
        return
    # chain of fold_n records: record t = encode(state t-1 -> state t), ref advancing
    recs, lens = [out[:n].clone()], [n]
    if a.fold_n > 1:
        ref = [y.clone() for y in Y]
        for t in range(2, a.fold_n + 1):
            for s_ in range(len(sizes)):
                tc.synth_step(Y[s_], synth.SEED0, s_, t, p53)
            tc.diff_encode(ctx, ref, Y, out, ob, t, t - 1, a.tile_words, 1 << 28, advance_ref=True,
                           index_mode=a.index)
            ctx.check()
            m = int(ob.item())
            recs.append(out[:m].clone())
            lens.append(m)
        del ref
    del out
    R = [x.clone() for x in X]
    ms = []
    for r in range(a.reps):
        for r_, x in zip(R, X):
            r_.copy_(x)
        torch.cuda.synchronize()
        ev[0].record()
        tc.diff_apply(ctx, R, 0, recs, lens)
        ev[1].record()
        ctx.check()
        ms.append(round(ev[0].elapsed_time(ev[1]), 3))
    print("fold N=%d ms:" % a.fold_n, ms, "record bytes", sum(lens))
    assert all(torch.equal(r_, y) for r_, y in zip(R, Y))
    print("ok")


if __name__ == "__main__":
    main()
