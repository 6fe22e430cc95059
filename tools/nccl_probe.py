"""Tier-2 probe (run under torchrun, N ranks): time tc_replicate_peer ring shifts of S bytes,
split into the size exchange and the payload, next to torch.distributed send/recv."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

from paper_2605_17821_b200 import tc  # noqa: E402

rank, world, local = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"]), int(os.environ["LOCAL_RANK"])
torch.cuda.set_device(local)
dev = torch.device("cuda", local)
dist.init_process_group("nccl", device_id=dev)
comm = tc.Comm(rank, world, local)
s = torch.cuda.Stream()
for S in (64 << 20, 256 << 20, 1 << 30, 4 << 30):
    send = torch.empty(S, dtype=torch.uint8, device=dev).fill_(rank + 1)
    recv = torch.empty(S, dtype=torch.uint8, device=dev)
    nb = torch.tensor([S], dtype=torch.int64, device=dev)
    for _ in range(2):
        comm.replicate_peer(send, nb, recv, tc.TO_NEXT, stream=s)
    s.synchronize()
    dist.barrier()
    reps = 5
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    e0.record(s)
    for _ in range(reps):
        got = comm.replicate_peer(send, nb, recv, tc.TO_NEXT, stream=s)
    e1.record(s)
    s.synchronize()
    wall = (time.perf_counter() - t0) / reps
    ms = e0.elapsed_time(e1) / reps
    ok = bool((recv[:16] == ((rank - 1) % world) + 1).all().item()) and got == S
    # torch.distributed reference ring shift
    dist.barrier()
    torch.cuda.synchronize()
    f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    f0.record()
    for _ in range(reps):
        ops = [dist.P2POp(dist.isend, send, (rank + 1) % world), dist.P2POp(dist.irecv, recv, (rank - 1) % world)]
        for w in dist.batch_isend_irecv(ops):
            w.wait()
    f1.record()
    torch.cuda.synchronize()
    tms = f0.elapsed_time(f1) / reps
    if rank == 0:
        print(f"S={S >> 20:5d} MiB  tc_replicate_peer {ms:8.3f} ms ({S / ms / 1e6:7.1f} GB/s per dir, wall {wall * 1e3:7.3f} ms) ok={ok}  "
              f"torch p2p {tms:8.3f} ms ({S / tms / 1e6:7.1f} GB/s)", flush=True)
comm.close()
dist.destroy_process_group()
