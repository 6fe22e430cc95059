"""Tier-1 staging under contention: every rank copies 1 GiB D2H at the same time into pinned host
memory allocated (a) wherever the process happens to run and (b) after binding the process to the
CPUs of its GPU's NUMA node (paper_2605_17821_b200.checkpoint.bind_local_numa).  Run under torchrun:

    python -m torch.distributed.run --nproc-per-node 4 --master-addr 127.0.0.1 tools/numa_probe.py
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

from paper_2605_17821_b200 import tc  # noqa: E402
from paper_2605_17821_b200.checkpoint import bind_local_numa  # noqa: E402

N = 1 << 30


def timed(d, h, s):
    dist.barrier()
    torch.cuda.synchronize()
    dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    tc.stage_host(h, d, N, tc.D2H, stream=s)
    e1.record(s)
    s.synchronize()
    ms = torch.tensor([e0.elapsed_time(e1)], device="cuda")
    dist.all_reduce(ms, op=dist.ReduceOp.MAX)
    return float(ms.item())


def main():
    rank, world, local = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"]), int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    d = torch.empty(N, dtype=torch.uint8, device="cuda")
    s = torch.cuda.Stream()
    h_default = tc.HostBuffer(N)
    info = bind_local_numa(local)
    h_local = tc.HostBuffer(N)
    for name, h in (("default", h_default), ("numa-local", h_local)):
        tc.stage_host(h, d, N, tc.D2H, stream=s)
        s.synchronize()
        ms = sorted(timed(d, h, s) for _ in range(3))[1]
        if rank == 0:
            print(f"{name:10s}: {world} ranks x 1 GiB D2H at once: {ms:8.3f} ms (max over ranks) = "
                  f"{N / ms / 1e6:6.1f} GB/s per GPU, {world * N / ms / 1e6:7.1f} GB/s aggregate", flush=True)
    print(f"rank {rank}: {info}", flush=True)
    h_default.free()
    h_local.free()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
