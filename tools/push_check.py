"""Multi-GPU correctness and bandwidth of the NCCL-free Tier-2 path (tc_ipc_* + tc_diff_encode_push
+ tc_peer_wait; run under torchrun, N >= 2 ranks).  Each rank encodes its shard and pushes the
record into its ring neighbour's slot over NVLink; the neighbour waits on its mailbox and
compares the received bytes with the same record replicated through NCCL (tc_replicate_peer),
then folds it onto its copy of our base.  Also: the capacity refusal (receiver sees
TC_ERR_CAPACITY, nobody hangs), alternating slots over several versions, and 1 GiB push vs
NCCL ring-shift bandwidth (max over ranks, printed as JSON).  Exits non-zero on any mismatch."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import synth  # noqa: E402
from paper_2605_17821_b200 import tc  # noqa: E402

rank, world, local = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"]), int(os.environ["LOCAL_RANK"])
torch.cuda.set_device(local)
dev = torch.device("cuda", local)
dist.init_process_group("nccl", device_id=dev)
comm = tc.Comm(rank, world, local)
ctx = tc.Ctx(local)
s = torch.cuda.Stream()
nxt, prv = (rank + 1) % world, (rank - 1) % world
fails = []

SLOT = 64 << 20
slots = [tc.IpcBuffer(SLOT) for _ in range(2)]   # the previous rank's records land here
mail = [tc.IpcBuffer(16) for _ in range(2)]
handles = [None] * world
dist.all_gather_object(handles, [b.handle for b in slots] + [m.handle for m in mail])
peer_slots = [tc.PeerMapping(h, SLOT) for h in handles[nxt][:2]]   # the next rank's slots
peer_mail = [tc.PeerMapping(h, 16) for h in handles[nxt][2:]]

sizes, wb = [70001, 50000, 33333], [2, 4, 4]


def shard(r, v, f):
    return [torch.from_numpy(a.view("int16" if w == 2 else "int32")).to(dev)
            for a, w in zip(synth.state(sizes, wb, synth.SEED0 + r, v, f), wb)]


for v, f, index_mode in ((1, 0.01, True), (2, 0.5, False), (3, 0.02, True), (4, 1.0, False)):
    k = v % 2
    ref, cur = shard(rank, v - 1, f), shard(rank, v, f)
    base_prev = shard(prv, v - 1, f)
    cap = tc.diff_bound(sizes, wb, 4096, 1 << 28, index_mode)
    out = torch.zeros(cap, dtype=torch.uint8, device=dev)
    ob = torch.zeros(1, dtype=torch.int64, device=dev)
    got_b = torch.zeros(1, dtype=torch.int64, device=dev)
    dist.barrier()
    tc.diff_encode_push(ctx, ref, cur, out, ob, v, v - 1, peer_slots[k], SLOT, peer_mail[k], stream=s,
                        index_mode=index_mode)
    tc.peer_wait(ctx, mail[k], v, got_b, stream=s)
    s.synchronize()
    ctx.check(s)
    n_got = int(got_b.item())
    # the same record through NCCL, for comparison
    recv = torch.zeros(SLOT, dtype=torch.uint8, device=dev)
    n_nccl = comm.replicate_peer(out, ob, recv, tc.TO_NEXT, stream=s)
    s.synchronize()
    if n_got != n_nccl or not torch.equal(slots[k].tensor[:n_got], recv[:n_nccl]):
        fails.append(f"v{v}: pushed record differs from the NCCL copy ({n_got} vs {n_nccl} bytes)")
    # the received record restores the previous rank's state on this GPU
    tc.diff_apply(ctx, base_prev, v - 1, [slots[k].tensor], [n_got], stream=s)
    rc = ctx.check_status(s)
    if rc != tc.OK or not all(torch.equal(a, b) for a, b in zip(base_prev, shard(prv, v, f))):
        fails.append(f"v{v}: fold of the pushed record did not restore rank {prv}'s state (rc {rc})")

# capacity refusal: the push to rank 0 claims a 1 KB slot
ref, cur = shard(rank, 0, 0.5), shard(rank, 1, 0.5)
out = torch.zeros(tc.diff_bound(sizes, wb), dtype=torch.uint8, device=dev)
ob = torch.zeros(1, dtype=torch.int64, device=dev)
dist.barrier()
tc.diff_encode_push(ctx, ref, cur, out, ob, 7, 6, peer_slots[1], 1024 if nxt == 0 else SLOT, peer_mail[1], stream=s)
tc.peer_wait(ctx, mail[1], 7, None, stream=s)
rc = ctx.check_status(s)
if rc != (tc.ERR_CAPACITY if rank == 0 else tc.OK):
    fails.append(f"capacity path: rank {rank} got status {rc}")
dist.barrier()

# bandwidth: 1 GiB push vs NCCL ring shift, 5 reps each, max over ranks
G = 1 << 30
big = torch.randint(0, 256, (G,), dtype=torch.uint8, device=dev)
nbig = torch.tensor([G], dtype=torch.int64, device=dev)
land = tc.IpcBuffer(G)
lmail = tc.IpcBuffer(16)
hs = [None] * world
dist.all_gather_object(hs, [land.handle, lmail.handle])
pl, pm = tc.PeerMapping(hs[nxt][0], G), tc.PeerMapping(hs[nxt][1], 16)


def timed(fn, reps=5):
    fn(0)
    s.synchronize()
    dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    for i in range(reps):
        fn(i + 1)
    e1.record(s)
    s.synchronize()
    t = torch.tensor([e0.elapsed_time(e1) / reps], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def push(i):
    tc.push_peer(ctx, big, nbig, pl, G, pm, 100 + i, stream=s)
    tc.peer_wait(ctx, lmail, 100 + i, None, stream=s)


rbuf = torch.empty(G, dtype=torch.uint8, device=dev)
ms_push = timed(push)
ms_nccl = timed(lambda i: comm.replicate_peer(big, nbig, rbuf, tc.TO_NEXT, stream=s))
if not torch.equal(land.tensor[:1 << 20], rbuf[:1 << 20]):
    fails.append("1 GiB push content differs from the NCCL copy")
ctx.check(s)
res = {"world": world, "push_1GiB_ms": round(ms_push, 4), "push_gbs_per_direction": round(G / ms_push / 1e6, 1),
       "nccl_1GiB_ms": round(ms_nccl, 4), "nccl_gbs_per_direction": round(G / ms_nccl / 1e6, 1)}
for p in peer_slots + peer_mail + [pl, pm]:
    p.close()
dist.barrier()
if rank == 0:
    print(json.dumps(res))
print(f"rank {rank}: {'OK' if not fails else 'FAIL ' + '; '.join(fails)}", flush=True)
comm.close()
dist.destroy_process_group()
sys.exit(1 if fails else 0)
