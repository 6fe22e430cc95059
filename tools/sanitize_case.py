"""Small encode -> fold round trip for compute-sanitizer (memcheck / racecheck / synccheck):
mixed widths, ragged tails, several chunks, sparse and dense blocks, N = 3 fold."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import synth  # noqa: E402
from paper_2605_17821_b200 import tc  # noqa: E402

sizes, wb = [20011, 45001, 9000, 0], [2, 4, 4, 4]
ctx = tc.Ctx(0)
for f in (0.02, 0.6):
    X = [torch.empty(n, dtype=torch.int16 if w == 2 else torch.int32, device="cuda") for n, w in zip(sizes, wb)]
    for i, t in enumerate(X):
        tc.synth_base(t, 5, i)
    ref = [x.clone() for x in X]
    cur = [x.clone() for x in X]
    cap = tc.diff_bound(sizes, wb, 256, 8192)
    recs, lens = [], []
    for v in (1, 2, 3):
        for i, t in enumerate(cur):
            tc.synth_step(t, 5, i, v, synth.p53_of(f))
        out = torch.empty(cap, dtype=torch.uint8, device="cuda")
        ob = torch.zeros(1, dtype=torch.int64, device="cuda")
        tc.diff_encode(ctx, ref, cur, out, ob, v, v - 1, 256, 8192)
        ctx.check()
        recs.append(out)
        lens.append(int(ob.item()))
    R = [x.clone() for x in X]
    tc.diff_apply(ctx, R, 0, recs, lens)
    ctx.check()
    assert all(torch.equal(a, b) for a, b in zip(R, cur))
print("sanitize case ok")
