"""Independent numpy parser of the record wire format, used by tests to
pin the oracle (and, in GPU tests, to inspect CUDA-path records).  It re-derives
section offsets from the layout table, not from either implementation."""
from __future__ import annotations

import struct

import numpy as np

HDR = struct.Struct("<4sHBBIIQQQQQQ")  # 64 bytes


def pad16(x: int) -> int:
    return -(-x // 16) * 16


def parse(buf, pos: int = 0):
    b = bytes(np.asarray(buf, dtype=np.uint8)[pos: pos + 64])
    (magic, fmt, w, flags, T, seg, off, m, count, version, ref_version, total) = HDR.unpack(b)
    n_mask = -(-m // 32)
    n_tiles = -(-m // T)
    a = np.asarray(buf, dtype=np.uint8)
    p = pos + 64
    mask = a[p: p + 4 * n_mask].view("<u4")
    p += pad16(4 * n_mask)
    toff = a[p: p + 4 * (n_tiles + 1)].view("<u4")
    p += pad16(4 * (n_tiles + 1))
    vals = a[p: p + w * count].view("<u2" if w == 2 else "<u4")
    return dict(magic=magic, fmt=fmt, w=w, flags=flags, T=T, seg=seg, off=off, m=m,
                count=count, version=version, ref_version=ref_version, total=total,
                mask=mask, toff=toff, values=vals, pos=pos)


def records(buf):
    a = np.asarray(buf, dtype=np.uint8)
    out = []
    pos = 0
    while pos < a.size:
        r = parse(a, pos)
        out.append(r)
        pos += r["total"]
    return out
