"""Tier-1 staging probe: host-side call latency and D2H/H2D bandwidth of tc_stage_host into
(a) libtc-pinned memory (tc_host_alloc) and (b) torch pin_memory tensors; 1 GiB copies."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2605_17821_b200 import tc  # noqa: E402

N = 1 << 30
d = torch.empty(N, dtype=torch.uint8, device="cuda")
s = torch.cuda.Stream()
for name, h in (("libtc", tc.HostBuffer(N)), ("torch", torch.empty(N, dtype=torch.uint8, pin_memory=True))):
    for direction, label in ((tc.D2H, "D2H"), (tc.H2D, "H2D")):
        dst, src = (h, d) if direction == tc.D2H else (d, h)
        tc.stage_host(dst, src, N, direction, stream=s)
        s.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        t0 = time.perf_counter()
        tc.stage_host(dst, src, N, direction, stream=s)
        t_call = time.perf_counter() - t0
        e1.record(s)
        s.synchronize()
        ms = e0.elapsed_time(e1)
        print(f"{name:6s} {label}: call returned after {t_call * 1e3:8.3f} ms, copy {ms:8.3f} ms = {N / ms / 1e6:6.1f} GB/s")
