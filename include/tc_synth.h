/*
 * tc_synth.h — seeded synthetic training-state generator on the device (bench / test INPUT
 * preparation only; not part of the codec and never called inside a timed region).
 *
 * It is the CUDA twin of synth/__init__.py (same counter-based splitmix64 recipe, DESIGN.md
 * §6, after SURVEY.md §8(d)); tests/test_gpu_synth.py checks the two agree bit for bit.
 *   base_s[i]    = low bits of h(K(seed,s,0) + i)
 *   changed_t[i] = (h((K(seed,s,t) ^ 0xC0FFEE) + j) >> 11) < p53, j = i (S1) | i >> 12 (S2)
 *   new word     = old ^ ((h((K(seed,s,t) ^ 0xBEEF) + i) & lowmask) | 1)
 * with K(seed,s,t) = h(seed ^ (s << 56) ^ (t << 32)).  `start` offsets the word counter so a
 * window [start, start+n) of a segment can be generated.
 */
#ifndef TC_SYNTH_H
#define TC_SYNTH_H
#include <stdint.h>

#include "tc.h"

#ifdef __cplusplus
extern "C" {
#endif

/* dst: device, n words of word_bytes (2|4) bytes; version-0 words of segment `seg`. */
tc_status tc_synth_base(void* dst, uint64_t n, uint32_t word_bytes, uint64_t seed, uint32_t seg,
                        uint64_t start, tc_stream stream);
/* words: device, in place: version t-1 -> version t.  p53 = round(f * 2^53);
 * structure 0 = S1 i.i.d. per word, 1 = S2 runs of 4096 words. */
tc_status tc_synth_step(void* words, uint64_t n, uint32_t word_bytes, uint64_t seed, uint32_t seg,
                        uint64_t t, uint64_t p53, int structure, uint64_t start, tc_stream stream);

#ifdef __cplusplus
}
#endif
#endif
