"""Read-only / write-only vs copy stream ceilings on one B200: torch sum / amax over a
cfg2-sized fp32 gradient (6.23 GB, what the lossy counting pass reads), a fill of it (what the
decompression writes) and a copy of it.  CUDA events.

    python tools/read_probe.py
"""
import torch, statistics
x = torch.randn(1_557_611_200, device="cuda")
y = torch.empty_like(x)
def t(fn, reps=10):
    out=[]
    for _ in range(reps):
        a,b=torch.cuda.Event(enable_timing=True),torch.cuda.Event(enable_timing=True)
        a.record(); fn(); b.record(); torch.cuda.synchronize(); out.append(a.elapsed_time(b))
    return min(out), statistics.median(out)
n=x.numel()*4
for name, fn in [("sum (read only)", lambda: x.sum()), ("amax (read only)", lambda: x.abs().amax() if False else torch.amax(x)), ("fill (write only)", lambda: y.fill_(0.5)), ("zero (write only)", lambda: y.zero_()), ("copy (read+write)", lambda: y.copy_(x))]:
    mn, md = t(fn)
    by = n if "only" in name else 2*n
    print(name, "min %.3f ms  %.0f GB/s   median %.3f ms" % (mn, by/mn/1e6, md))
