"""Multi-GPU check of the paced base replication (paper_2605_17821_b200.checkpoint.BaseReplicator,
NEXT row 4; run under torchrun, N >= 2): a base shard intercepted once, staged to Tier-1, pushed to
the ring neighbour in paced chunks over NVLink stores, visible there only when complete; a plan
that spills over is flushed synchronously at the next base boundary.  Exits non-zero on failure."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

from paper_2605_17821_b200.checkpoint import BaseReplicator  # noqa: E402

rank, world, local = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"]), int(os.environ["LOCAL_RANK"])
torch.cuda.set_device(local)
dev = torch.device("cuda", local)
dist.init_process_group("nccl", device_id=dev)
prv = (rank - 1) % world
fails = []
SIZES = [300_001, 300_001, 300_001, 300_001]


def shard(r, version):
    g = torch.Generator(device="cpu").manual_seed(1000 * r + version)
    segs = [torch.randint(-32768, 32767, (SIZES[0],), dtype=torch.int16, generator=g)]
    segs += [torch.randint(-2**31, 2**31 - 1, (n,), dtype=torch.int32, generator=g) for n in SIZES[1:]]
    return [t.to(dev) for t in segs]


def flat(segs):
    return torch.cat([t.view(torch.uint8).reshape(-1) for t in segs])


n = sum(t.numel() * t.element_size() for t in shard(rank, 1))
rep = BaseReplicator(n, rank, world, local)
# base 1: no spillover (I = 10, s = 2: 8 paced chunks)
plan = rep.intercept(shard(rank, 1), version=10, interval=10, margin=2, cap=1 << 30)
if plan.spillover or plan.iters != 8:
    fails.append(f"plan 1: {plan}")
for it in range(1, 11):
    rep.pump(it)
    rep.s.synchronize()
    dist.barrier()
    seen = rep.committed_version()
    if it < plan.iters and seen != -1:
        fails.append(f"replica visible before completion (iteration {it})")
    if it >= plan.iters and seen != 10:
        fails.append(f"replica not committed after {it} iterations: {seen}")
    dist.barrier()  # no rank pushes the next chunk (or the commit) before every rank has looked
if not torch.equal(rep.received(), flat(shard(prv, 1))):
    fails.append("base 1 replica differs from the neighbour's shard")
if not torch.equal(rep.host.tensor[:n], flat(shard(rank, 1)).cpu()):
    fails.append("Tier-1 copy differs")
# base 2: spills over (small cap), flushed at the next base boundary
plan = rep.intercept(shard(rank, 2), version=20, interval=10, margin=2, cap=64 << 10)
if not plan.spillover:
    fails.append(f"plan 2 should spill over: {plan}")
for it in range(11, 19):
    rep.pump(it)
rep.s.synchronize()
dist.barrier()
if rep.committed_version() != 10:
    fails.append("spillover base visible before its flush")
if not torch.equal(rep.received(), flat(shard(prv, 1))):  # base 2 streams into the other slot
    fails.append("committed base 1 torn while base 2 was in flight")
dist.barrier()
rep.intercept(shard(rank, 3), version=30, interval=10, margin=2, cap=1 << 30)  # flushes base 2 first
rep.s.synchronize()
dist.barrier()
if not any(k == "sync_flush" for _, k, _ in rep.log):
    fails.append("no sync_flush logged")
if rep.committed_version() != 20 or not torch.equal(rep.received(), flat(shard(prv, 2))):
    fails.append(f"base 2 not complete after the flush (commit {rep.committed_version()})")
rep.ctx.check(rep.s)
rep.close()
dist.barrier()
print(f"rank {rank}: {'OK' if not fails else 'FAIL ' + '; '.join(fails)}", flush=True)
dist.destroy_process_group()
sys.exit(1 if fails else 0)
