"""Helpers for the GPU parity tests: move numpy word arrays to CUDA tensors (bit views) and
call libtc through the binding."""
from __future__ import annotations

import numpy as np
import torch

from paper_2605_17821_b200 import tc

_VIEW = {np.dtype(np.uint16): np.int16, np.dtype(np.uint32): np.int32}
_BACK = {torch.int16: np.uint16, torch.int32: np.uint32}


def to_dev(a: np.ndarray) -> torch.Tensor:
    t = torch.from_numpy(np.ascontiguousarray(a).view(_VIEW[a.dtype]).copy())
    return t.cuda()


def to_np(t: torch.Tensor) -> np.ndarray:
    return t.cpu().numpy().view(_BACK[t.dtype])


def gpu_encode(ctx, ref_np, cur_np, tile_words=4096, chunk_words=1 << 28, advance_ref=True, version=1,
               ref_version=0, index_mode=False):
    """Returns (record bytes as numpy uint8, ref-after numpy list, out_bytes)."""
    ref = [to_dev(a) for a in ref_np]
    cur = [to_dev(a) for a in cur_np]
    cap = tc.diff_bound([a.size for a in ref_np], [a.itemsize for a in ref_np], tile_words, chunk_words, index_mode)
    out = torch.full((cap + 64,), 0xAB, dtype=torch.uint8, device="cuda")  # poison: pads must be written
    ob = torch.zeros(1, dtype=torch.int64, device="cuda")
    tc.diff_encode(ctx, ref, cur, out, ob, version, ref_version, tile_words, chunk_words, advance_ref,
                   index_mode=index_mode)
    ctx.check()
    n = int(ob.item())
    return out[:n].cpu().numpy(), [to_np(r) for r in ref], n


def gpu_fold(ctx, state_np, state_version, diffs_np):
    """Fold numpy record buffers onto a device copy of state_np.  Returns (status, state numpy)."""
    st = [to_dev(a) for a in state_np]
    recs = []
    for d in diffs_np:
        t = torch.zeros(max(d.size, 16), dtype=torch.uint8, device="cuda")
        if d.size:
            t[: d.size] = torch.from_numpy(np.ascontiguousarray(d))
        recs.append(t)
    tc.diff_apply(ctx, st, state_version, recs, [d.size for d in diffs_np])
    rc = ctx.check_status()
    return rc, [to_np(s) for s in st]
