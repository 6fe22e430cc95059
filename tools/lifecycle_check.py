"""Multi-GPU check of the product lifecycle (paper_2605_17821_b200.checkpoint.Checkpointer, run under
torchrun, N >= 2): every rank saves a chain of versions of its shard with Tier-1 staging and Tier-2
NVLink push to its ring neighbour (the base streamed there in paced chunks); then rank 0 suffers a
node failure — its HBM state, its reference AND its Tier-1 host copies are gone — and every rank
calls recover(): consensus on (base, replay end) over the group, and the cascade sends rank 0 to
its neighbour's Tier-2 replicas (base + records read over NVLink) while the others use Tier-1.
Every rank's recovered state must equal its seeded chain head bit for bit; the chain then
continues.  Exits non-zero on failure."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import synth  # noqa: E402
from paper_2605_17821_b200 import tc  # noqa: E402
from paper_2605_17821_b200.checkpoint import Checkpointer  # noqa: E402

rank, world, local = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"]), int(os.environ["LOCAL_RANK"])
torch.cuda.set_device(local)
dev = torch.device("cuda", local)
dist.init_process_group("nccl", device_id=dev)
fails = []
sizes, wb = [120001 + 64 * rank, 120001, 120001, 120001], [2, 4, 4, 4]  # ranks differ in size
seed = synth.SEED0 + rank
fs = [0.01, 0.2, 0.003, 1.0, 0.05, 0.01]


def dev_state(version_fs):
    segs = []
    for s, (n, w) in enumerate(zip(sizes, wb)):
        t = torch.empty(n, dtype=torch.int16 if w == 2 else torch.int32, device=dev)
        tc.synth_base(t, seed, s)
        for v, f in enumerate(version_fs, start=1):
            tc.synth_step(t, seed, s, v, synth.p53_of(f))
        segs.append(t)
    return segs


live = dev_state([])
ck = Checkpointer(live, rank, world, tier2="push", expected_f=1.0, t2_slots=8, chunk_words=1 << 15,
                  base_interval=4)
for v, f in enumerate(fs, start=1):
    for s, t in enumerate(live):
        tc.synth_step(t, seed, s, v, synth.p53_of(f))
    ck.save_step(v)
ck.flush()
for it in range(3):
    ck.base_rep.pump(100 + it)  # base_interval 4: the paced plan is 3 chunks
ck.base_rep.flush(200)
ck.base_rep.s.synchronize()
torch.cuda.synchronize()
dist.barrier()
expect = dev_state(fs)
if not all(torch.equal(a, b) for a, b in zip(live, expect)):
    fails.append("live state != seeded chain head before the failure")
if rank == 0:  # node failure: HBM and host memory of rank 0 are lost
    ck.drop_tier("hbm")
    ck.drop_tier("t1")
dist.barrier()
ver = ck.recover(batch=5)
if ver != len(fs):
    fails.append(f"recovered version {ver} != {len(fs)}")
if not all(torch.equal(a, b) for a, b in zip(live, expect)):
    fails.append("recovered state != chain head")
if not all(torch.equal(a, b) for a, b in zip(ck.ref, expect)):
    fails.append("reference != chain head after recovery")
# the chain continues on every rank
for s, t in enumerate(live):
    tc.synth_step(t, seed, s, len(fs) + 1, synth.p53_of(0.02))
ck.save_step(len(fs) + 1)
ck.flush()
torch.cuda.synchronize()
if ck.chain.head != len(fs) + 1:
    fails.append(f"chain head {ck.chain.head} after the post-recovery save")
dist.barrier()
ck.close()
dist.barrier()
print(f"rank {rank}: {'OK' if not fails else 'FAIL ' + '; '.join(fails)}", flush=True)
dist.destroy_process_group()
sys.exit(1 if fails else 0)
