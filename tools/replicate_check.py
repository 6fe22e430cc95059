"""Multi-GPU correctness of tc_replicate_peer (run under torchrun, N >= 2 ranks): ring shift in
both directions with distinct payload sizes per rank, byte-exact content, the capacity refusal
path (no hang: sender and receiver agree to skip), and a GPU-encoded record replicated and folded
on the neighbour.  Exits non-zero on any mismatch."""
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
s = torch.cuda.Stream()
nxt, prv = (rank + 1) % world, (rank - 1) % world
fails = []


def payload(r, n):
    g = torch.Generator(device="cpu").manual_seed(1000 + r)
    return torch.randint(0, 256, (n,), dtype=torch.uint8, generator=g).to(dev)


for direction, src in ((tc.TO_NEXT, prv), (tc.TO_PREV, nxt)):
    n_mine = 1000003 + 4096 * rank
    send = payload(rank, n_mine)
    nb = torch.tensor([n_mine], dtype=torch.int64, device=dev)
    recv = torch.zeros(4 << 20, dtype=torch.uint8, device=dev)
    got = comm.replicate_peer(send, nb, recv, direction, stream=s)
    s.synchronize()
    n_src = 1000003 + 4096 * src
    if got != n_src or not torch.equal(recv[:got], payload(src, n_src)):
        fails.append(f"direction {direction}: got {got}, expected {n_src} from {src}")

# capacity refusal: rank 0's receive buffer is too small; everyone returns, nobody hangs
send = payload(rank, 1 << 20)
nb = torch.tensor([1 << 20], dtype=torch.int64, device=dev)
recv = torch.zeros((1 << 10) if rank == 0 else (2 << 20), dtype=torch.uint8, device=dev)
try:
    comm.replicate_peer(send, nb, recv, tc.TO_NEXT, stream=s)
    if rank == 0:
        fails.append("capacity error not raised")
except tc.TcError as e:
    if rank != 0 or e.status != tc.ERR_CAPACITY:
        fails.append(f"unexpected {e}")
s.synchronize()

# an encoded record travels to the neighbour and restores its copy of our state there
sizes, wb, f = [50000, 50000], [2, 4], 0.05
seed = synth.SEED0 + rank
ctx = tc.Ctx(local)
X = [torch.empty(n, dtype=torch.int16 if w == 2 else torch.int32, device=dev) for n, w in zip(sizes, wb)]
for i, t in enumerate(X):
    tc.synth_base(t, seed, i)
Y = [x.clone() for x in X]
for i, t in enumerate(Y):
    tc.synth_step(t, seed, i, 1, synth.p53_of(f))
cap = tc.diff_bound(sizes, wb)
out = torch.empty(cap, dtype=torch.uint8, device=dev)
ob = torch.zeros(1, dtype=torch.int64, device=dev)
tc.diff_encode(ctx, [x.clone() for x in X], Y, out, ob, 1, 0)
torch.cuda.synchronize()
recv = torch.empty(cap, dtype=torch.uint8, device=dev)
got = comm.replicate_peer(out, ob, recv, tc.TO_NEXT, stream=s)
s.synchronize()
# rebuild the previous rank's state from its base (regenerated) + the replica
pseed = synth.SEED0 + prv
PX = [torch.empty(n, dtype=torch.int16 if w == 2 else torch.int32, device=dev) for n, w in zip(sizes, wb)]
for i, t in enumerate(PX):
    tc.synth_base(t, pseed, i)
PY = [x.clone() for x in PX]
for i, t in enumerate(PY):
    tc.synth_step(t, pseed, i, 1, synth.p53_of(f))
tc.diff_apply(ctx, PX, 0, [recv], [got])
ctx.check()
if not all(torch.equal(a, b) for a, b in zip(PX, PY)):
    fails.append("replica fold mismatch")

res = torch.tensor([len(fails)], device=dev)
dist.all_reduce(res)
if fails:
    print(f"rank {rank}: " + "; ".join(fails), flush=True)
if rank == 0:
    print(f"replicate_check world={world}: {'OK' if res.item() == 0 else 'FAIL'}", flush=True)
comm.close()
dist.destroy_process_group()
sys.exit(1 if res.item() else 0)
