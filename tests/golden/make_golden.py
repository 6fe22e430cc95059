"""Writes the golden record files in tests/golden/ by calling ONLY oracle/ (and the seeded
input generator synth/).  Run:  python tests/golden/make_golden.py

Files and what pins them (see README.md in this directory):
  hand1_fp32.bin   SURVEY.md Appendix A hand example 1 (fp32, m=6, T=4096, v7 <- v6)
  hand2_bf16.bin   SURVEY.md Appendix A hand example 2 (bf16, m=3)
  empty_m0.bin     SURVEY.md §8(c) reading c12 (empty segment -> 80-byte record)
  hand1_fp32_index.bin  hand example 1 as an index-mode record (idx = [1, 3])
  cfg1_small_v1.bin / cfg1_small_v2.bin
                   a two-link chain on a cfg1-shaped (3 fp32 segments) 3000-word shard,
                   f = 1 %, T = 64, chunk_words = 1024, seed 0x7C0DEC (determinism pin)
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

import oracle  # noqa: E402
import synth  # noqa: E402

HAND1_REF = [0x3F800000, 0x00000000, 0x80000000, 0x7FC00000, 0x12345678, 0x7FC00000]
HAND1_CUR = [0x3F800000, 0x80000000, 0x80000000, 0x7FC00001, 0x12345678, 0x7FC00000]
HAND2_REF = [0x3F80, 0x3F80, 0xFFFF]
HAND2_CUR = [0x3F81, 0x3F80, 0xFFFF]


def hand1():
    ref = np.array(HAND1_REF, dtype=np.uint32)
    cur = np.array(HAND1_CUR, dtype=np.uint32)
    rc, rec = oracle.encode([ref], [cur], tile_words=4096, advance_ref=False, version=7,
                            ref_version=6)
    assert rc == 0
    return rec


def hand2():
    ref = np.array(HAND2_REF, dtype=np.uint16)
    cur = np.array(HAND2_CUR, dtype=np.uint16)
    rc, rec = oracle.encode([ref], [cur], tile_words=4096, advance_ref=False, version=1,
                            ref_version=0)
    assert rc == 0
    return rec


def hand1_index():
    ref = np.array(HAND1_REF, dtype=np.uint32)
    cur = np.array(HAND1_CUR, dtype=np.uint32)
    rc, rec = oracle.encode([ref], [cur], tile_words=4096, advance_ref=False, version=7,
                            ref_version=6, index_mode=True)
    assert rc == 0
    return rec


def empty():
    e = np.zeros(0, dtype=np.uint32)
    rc, rec = oracle.encode([e], [e.copy()], tile_words=4096, advance_ref=False, version=1,
                            ref_version=0)
    assert rc == 0
    return rec


def cfg1_small():
    sizes, wb = [3000, 3000, 3000], [4, 4, 4]
    s0 = synth.state(sizes, wb, synth.SEED0, 0, 0.01)
    s1 = synth.state(sizes, wb, synth.SEED0, 1, 0.01)
    s2 = synth.state(sizes, wb, synth.SEED0, 2, 0.01)
    ref = [a.copy() for a in s0]
    rc, r1 = oracle.encode(ref, s1, tile_words=64, chunk_words=1024, version=1, ref_version=0)
    assert rc == 0
    rc, r2 = oracle.encode(ref, s2, tile_words=64, chunk_words=1024, version=2, ref_version=1)
    assert rc == 0
    return r1, r2


def main():
    out = {
        "hand1_fp32.bin": hand1(),
        "hand2_bf16.bin": hand2(),
        "empty_m0.bin": empty(),
        "hand1_fp32_index.bin": hand1_index(),
    }
    r1, r2 = cfg1_small()
    out["cfg1_small_v1.bin"] = r1
    out["cfg1_small_v2.bin"] = r2
    for name, data in out.items():
        with open(os.path.join(HERE, name), "wb") as fh:
            fh.write(bytes(data))
        print(name, len(data))


if __name__ == "__main__":
    main()
