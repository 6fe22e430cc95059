import torch, time
n = 1557611200
x = torch.zeros(n, dtype=torch.int32, device="cuda")
for f in (0.001, 0.01, 0.1):
    g = torch.Generator(device="cuda").manual_seed(1)
    mask = torch.rand(n, device="cuda", generator=g) < f
    idx = mask.nonzero().squeeze(1)
    del mask
    v = torch.arange(idx.numel(), dtype=torch.int32, device="cuda")
    for _ in range(2):
        x[idx] = v
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(3):
        x[idx] = v
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 3
    # pure sorted gather+scatter: read v, idx, write scattered
    print(f"f={f}: {idx.numel()/1e6:.1f}M scattered fp32 writes into 6.2 GB: {ms:.3f} ms", flush=True)
    del idx, v
# streaming copy for reference
y = torch.empty_like(x)
torch.cuda.synchronize()
e0.record(); y.copy_(x); e1.record(); torch.cuda.synchronize()
print(f"copy 6.2 GB: {e0.elapsed_time(e1):.3f} ms")
