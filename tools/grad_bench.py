"""Throughput of the paper's lossy differential on one B200 (NEXT row 3): gradient compression
(sparse form, k = 0.01) and decompression of a cfg2-sized fp32 gradient shard, and the fused
multi-step Adam replay of N payloads against N sequential decompress + Adam steps (the paper's
Exp#7 comparison).  CUDA events; inputs resident in HBM; prints one JSON line.

    python tools/grad_bench.py [--n 1557611200] [--N 5] [--reps 3]
"""
import argparse
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2605_17821_b200 import tc  # noqa: E402


def timed(fn, reps, s):
    out = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(s)
        fn()
        b.record(s)
        s.synchronize()
        out.append(a.elapsed_time(b))
    return statistics.median(out)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=1_557_611_200)  # cfg2: GPT-2 1.5B parameters on 1 GPU
    ap.add_argument("--N", type=int, default=5)              # P:395 batch of N = 5 diffs
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--k", type=float, default=0.01)
    ap.add_argument("--state", default="zero", choices=["zero", "mid"],
                    help="Adam moments before the replay: zero (a fresh optimizer) or mid-training "
                         "(m ~ N(0, 1e-3), v ~ |N(0, 1)| 1e-6 everywhere)")
    a = ap.parse_args()
    n, N = a.n, a.N
    dev = torch.device("cuda", 0)
    s = torch.cuda.Stream()
    ctx = tc.Ctx(0)
    peak = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                       "MEASURED_PEAKS.json"))).get("hbm_gbs", 6456.2)
    g = torch.empty(n, dtype=torch.float32, device=dev)
    cap = tc.grad_bound(n, k=a.k)
    est = int(n * a.k * 2.5 * 6) + (1 << 20)  # expected payload at k, with room
    pays = [torch.empty(min(cap, est), dtype=torch.uint8, device=dev) for _ in range(N)]
    ob = torch.zeros(N, dtype=torch.int64, device=dev)
    with torch.cuda.stream(s):
        for j in range(N):
            torch.randn(n, out=g, generator=torch.Generator(device=dev).manual_seed(j))
            g.mul_(1e-2)
            tc.grad_compress(ctx, g, j, pays[j], ob[j:j + 1], stream=s, k=a.k)
    s.synchronize()
    ctx.check(s)
    nbytes = [int(x) for x in ob.tolist()]
    tmp = torch.empty(pays[0].numel(), dtype=torch.uint8, device=dev)
    ob_t = torch.zeros(1, dtype=torch.int64, device=dev)
    ms_c = timed(lambda: tc.grad_compress(ctx, g, N - 1, tmp, ob_t, stream=s, k=a.k), a.reps, s)
    ctx.check(s)
    assert int(ob_t.item()) == nbytes[-1] and torch.equal(tmp[:nbytes[-1]], pays[-1][:nbytes[-1]])
    del tmp
    kept = (nbytes[-1] - 80) // 6
    c_bytes = 4 * n + nbytes[-1] + 6 * kept  # gradient read once + payload written (+ spill round trip)
    dense = torch.empty(n, dtype=torch.float32, device=dev)
    ms_d = timed(lambda: tc.grad_decompress(ctx, pays[0], nbytes[0], dense, stream=s), a.reps, s)
    d_bytes = 4 * n + nbytes[0]
    del g
    master = torch.randn(n, dtype=torch.float32, device=dev)
    m = torch.zeros(n, dtype=torch.float32, device=dev)
    v = torch.zeros(n, dtype=torch.float32, device=dev)
    if a.state == "mid":
        m.normal_(0.0, 1e-3)
        v.normal_(0.0, 1.0).abs_().mul_(1e-6)
    w16 = torch.zeros(n, dtype=torch.int16, device=dev)
    snap = [x.clone() for x in (master, m, v, w16)]

    def reset():
        for x, y in zip((master, m, v, w16), snap):
            x.copy_(y)

    def fused():
        tc.adam_replay(ctx, master, m, v, w16, pays, nbytes, 1, dense, stream=s)

    def sequential():
        for j in range(N):
            tc.grad_decompress(ctx, pays[j], nbytes[j], dense, stream=s)
            tc.adam_step(ctx, master, m, v, w16, dense, 1 + j, stream=s)

    res_f, res_s = [], []
    for _ in range(a.reps):
        with torch.cuda.stream(s):
            reset()
        s.synchronize()
        res_f.append(timed(fused, 1, s))
        fused_state = [x.clone() for x in (master, m, v, w16)]
        with torch.cuda.stream(s):
            reset()
        s.synchronize()
        res_s.append(timed(sequential, 1, s))
        same = all(torch.equal(x, y) for x, y in zip((master, m, v, w16), fused_state))
        del fused_state
    ctx.check(s)
    ms_f, ms_s = statistics.median(res_f), statistics.median(res_s)
    # algorithmic bytes: fused = (master, m, v) read + written once for N-1 steps + the payloads,
    # then the native step (dense gradient write + read, state read + write, w16 write)
    st = 12 * n
    f_bytes = 2 * st + sum(nbytes[:-1]) + (4 * n + nbytes[-1]) + (4 * n + 2 * st + 2 * n)
    s_bytes = N * ((4 * n + nbytes[0]) + (4 * n + 2 * st + 2 * n))
    out = {"n": n, "N": N, "k": a.k, "state": a.state, "payload_bytes": nbytes[0], "kept": kept,
           "compress": {"ms": round(ms_c, 3), "gbs": round(c_bytes / ms_c / 1e6, 1),
                        "frac_hbm": round(c_bytes / ms_c / 1e6 / peak, 4), "bytes": c_bytes},
           "decompress": {"ms": round(ms_d, 3), "gbs": round(d_bytes / ms_d / 1e6, 1),
                          "frac_hbm": round(d_bytes / ms_d / 1e6 / peak, 4)},
           "replay_fused": {"ms": round(ms_f, 3), "gbs": round(f_bytes / ms_f / 1e6, 1),
                            "frac_hbm": round(f_bytes / ms_f / 1e6 / peak, 4), "bytes": f_bytes},
           "replay_sequential": {"ms": round(ms_s, 3), "gbs": round(s_bytes / ms_s / 1e6, 1), "bytes": s_bytes},
           "speedup_fused_vs_sequential": round(ms_s / ms_f, 3),
           "fused_equals_sequential": bool(same), "peak_hbm_gbs": peak,
           "paper_context": "Exp#7 (A800, GPT2 20B, 100-iteration chain): fused 16.6 s vs sequential 26.0 s (P:586)"}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
