"""NEXT row 2 on one B200: the Adam step fused with the lossless differential of its update
(tc_adam_step_encode) against the unfused path (tc_adam_step, then tc_diff_encode of the state
against the advancing reference copy), on a cfg2-sized shard (1.56 G parameters: bf16 weights +
fp32 master / m / v).  Two gradient regimes: dense (every moment changes: the record is ~ the
state) and sparse (1 % nonzero, fresh moments: ~1 % of the words change), the sparse one in both
record modes (mask, index).  CUDA events,
inputs resident; prints one JSON line.

    python tools/adam_encode_bench.py [--n 1557611200] [--reps 3]
"""
import argparse
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2605_17821_b200 import tc  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=1_557_611_200)
    ap.add_argument("--reps", type=int, default=3)
    a = ap.parse_args()
    n = a.n
    dev = torch.device("cuda", 0)
    s = torch.cuda.Stream()
    ctx = tc.Ctx(0)
    peak = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                       "MEASURED_PEAKS.json"))).get("hbm_gbs", 6456.2)
    master = torch.empty(n, dtype=torch.float32, device=dev)
    m = torch.empty_like(master)
    v = torch.empty_like(master)
    w16 = torch.empty(n, dtype=torch.int16, device=dev)
    g = torch.empty_like(master)
    refs = [torch.empty_like(w16), torch.empty_like(master), torch.empty_like(master), torch.empty_like(master)]
    cap = max(max(tc.diff_bound([n] * 4, [2, 4, 4, 4], 4096, 1 << 28, index_mode=im) for im in (False, True)),
              tc.diff_bound([n] * 4, [2, 4, 4, 4], 4096, 1 << 28, full=True))
    out = torch.empty(cap, dtype=torch.uint8, device=dev)
    ob = torch.zeros(1, dtype=torch.int64, device=dev)
    W = 14 * n
    res = {"n": n, "state_bytes": W}
    for regime, imode in (("sparse", False), ("sparse_index", True), ("dense", False), ("dense_full", "full")):
        full = imode == "full"
        imode = imode is True
        gen = torch.Generator(device=dev).manual_seed(1)
        with torch.cuda.stream(s):
            torch.randn(n, out=master, generator=gen)
            torch.randn(n, out=g, generator=gen)
            g.mul_(1e-2)
            if regime.startswith("sparse"):
                g.mul_((torch.rand(n, device=dev, generator=gen) < 0.01).float())
                m.zero_()
                v.zero_()
            else:
                torch.randn(n, out=m, generator=gen)
                m.mul_(1e-3)
                torch.randn(n, out=v, generator=gen)
                v.abs_().mul_(1e-6)
            w16.copy_(master.to(torch.bfloat16).view(torch.int16))
            snap = [t.clone() for t in (master, m, v, w16)]  # on s: after the initialisation above
        s.synchronize()

        def reset():
            with torch.cuda.stream(s):
                for t, x in zip((master, m, v, w16), snap):
                    t.copy_(x)
                for r_, x in zip(refs, (w16, master, m, v)):  # the reference = the state before
                    r_.copy_(x)
            s.synchronize()

        def ev():
            return torch.cuda.Event(enable_timing=True)

        fused, unfused = [], []
        for _ in range(a.reps):
            reset()
            e0, e1 = ev(), ev()
            e0.record(s)
            tc.adam_step_encode(ctx, master, m, v, w16, g, 7, out, ob, stream=s, index_mode=imode, full=full)
            e1.record(s)
            s.synchronize()
            fused.append(e0.elapsed_time(e1))
            nb_f = int(ob.item())
            f_rec = out[:nb_f].clone()  # the fused record, compared with the unfused one below
            reset()
            e0, e1, e2 = ev(), ev(), ev()
            e0.record(s)
            tc.adam_step(ctx, master, m, v, w16, g, 7, stream=s)
            e1.record(s)
            tc.diff_encode(ctx, refs, [w16, master.view(torch.int32), m.view(torch.int32), v.view(torch.int32)],
                           out, ob, 7, 6, stream=s, index_mode=imode, full=full)
            e2.record(s)
            s.synchronize()
            unfused.append((e0.elapsed_time(e1), e1.elapsed_time(e2)))
            same = int(ob.item()) == nb_f and torch.equal(out[:nb_f], f_rec)
            del f_rec
        ctx.check(s)
        fm = statistics.median(fused)
        am = statistics.median(x[0] for x in unfused)
        em = statistics.median(x[1] for x in unfused)
        nb = int(ob.item())
        changed_bytes, off = 0, 0  # the words the step rewrote: Σ count·w over the record headers
        while off < nb:
            h = out[off:off + 64].cpu().numpy().view("<u8")
            changed_bytes += int(h[4]) * ((int(h[0]) >> 48) & 0xFF)
            off += int(h[7])
        res[regime] = {"record_bytes": nb, "record_equal": bool(same),
                       "fused_ms": round(fm, 3), "fused_state_gbs": round(W / fm / 1e6, 1),
                       "unfused_adam_ms": round(am, 3), "unfused_encode_ms": round(em, 3),
                       "unfused_ms": round(am + em, 3), "speedup": round((am + em) / fm, 3),
                       "changed_bytes": changed_bytes,
                       "fused_frac_hbm_min_bytes": round((4 * n + W + changed_bytes + nb) / fm / 1e6 / peak, 4)}
        if full:  # the full path writes every state word and every record word: grad + 2 W + record
            res[regime]["fused_frac_hbm"] = round((4 * n + 2 * W + nb) / fm / 1e6 / peak, 4)
    res["note"] = ("NEXT row 2 (DESIGN.md §13): tc_adam_step_encode vs tc_adam_step + tc_diff_encode(ref copy); "
                   "fused_frac_hbm_min_bytes counts grad + state read + changed words written + record")
    print(json.dumps(res))


if __name__ == "__main__":
    main()
