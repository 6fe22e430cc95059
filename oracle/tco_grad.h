/*
 * tco_grad.h — ORACLE for the paper's own (lossy) differential: the adaptive gradient codec and
 * the Adam replay.  Plain scalar C, host only.
 *
 * TEST INFRASTRUCTURE ONLY (same rules as tco.h): only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs load it; it shares nothing with the CUDA path.
 *
 * What it computes (§3.2; §3.3):
 *   - compress: a gradient shard of n fp32 values becomes
 *       n < small_threshold (100K) -> INT8 symmetric: scale = max|x|/127 (1 if all
 *         zero), q[i] = clamp(rint(x[i]/scale), -127, 127)                 ("dense INT8 quantization")
 *       else -> sparse: the magnitude threshold is the ceil((1-k)*S)-th smallest of |x| over S
 *         sampled entries (S = 4096, uniform, seeded: index_j = splitmix64(seed + j) mod n;
 *         "estimates a magnitude threshold via sampling"), then one pass keeps every entry with
 *         |x| >= threshold and x != 0 as an FP16 value (round to nearest even) + INT32 index local
 *         to its chunk of chunk_elems entries ("FP16 values and INT32 indices ... chunked before
 *         compression and safely rebased").
 *   - decompress: INT8 -> scale * q; sparse -> zeros with the FP16 values widened at
 *     base_offset + index (§4 "sparse payloads are fused into dense tensors and INT8
 *     payloads are dequantized from their stored scales").
 *   - adam_step (standard bias-corrected Adam, in the efficient ordering of the
 *     Adam paper's Algorithm 1 note / PyTorch's implementation): m = b1 m + (1-b1) g;
 *     v = b2 v + (1-b2) g^2; denom = sqrt(v) * inv_c2s + eps; master -= step_size * (m / denom),
 *     with step_size = lr / (1 - b1^t) and inv_c2s = 1 / sqrt(1 - b2^t) evaluated by the caller in
 *     double and rounded to fp32; weights = bf16 round-to-nearest-even of master.  Operation order
 *     is fixed as written (every product, sum and quotient rounded to fp32; -ffp-contract=off).
 *   - replay: payloads applied in temporal order, one adam_step each (the sequential definition
 *     the fused replay must reproduce bit-exactly).
 * Readings: DESIGN.md §12.
 *
 * Payload layout (little-endian, sections padded to 16 bytes):
 *   off size field
 *     0    4 magic "TCG1"
 *     4    1 variant: 1 = INT8 dense, 2 = sparse
 *     5    3 zero
 *     8    4 chunk_count (sparse; dense: 0)
 *    12    4 scale (dense) / threshold (sparse), f32
 *    16    8 n (original length)
 *    24    8 kept (sparse: entries; dense: n)
 *    32    8 chunk_elems
 *    40    8 seed
 *    48    8 total_bytes
 *    56    8 zero
 *    64      dense: i8 q[n]
 *    64      sparse: chunk table {u64 base_offset, u64 entry_count}[chunk_count] | f16 values[kept]
 *            | i32 indices[kept]   (chunk c's entries are the c-th run of values / indices)
 */
#ifndef TCO_GRAD_H
#define TCO_GRAD_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

uint64_t tco_grad_bound(uint64_t n, uint64_t small_threshold, uint64_t chunk_elems);
/* rank = ceil((1-k)*sample_size) in [1, sample_size], computed by the caller in double */
int tco_grad_compress(const float* x, uint64_t n, uint64_t small_threshold, uint32_t sample_size,
                      uint32_t rank, uint64_t chunk_elems, uint64_t seed, uint8_t* out, uint64_t cap,
                      uint64_t* out_bytes);
int tco_grad_decompress(const uint8_t* p, uint64_t bytes, float* out, uint64_t n);
uint16_t tco_f32_to_f16(float f);
float tco_f16_to_f32(uint16_t h);
uint16_t tco_f32_to_bf16(float f);
void tco_adam_step(float* master, float* m, float* v, uint16_t* w16, uint64_t n, const float* g, float b1, float b2,
                   float eps, float step_size, float inv_c2s);
/* payloads[j] at step first_step + j uses step_size[j], inv_c2s[j]; scratch: n floats */
int tco_adam_replay(float* master, float* m, float* v, uint16_t* w16, uint64_t n, const uint8_t* const* payloads,
                    const uint64_t* bytes, int n_payloads, float b1, float b2, float eps, const float* step_size,
                    const float* inv_c2s, float* scratch);

#ifdef __cplusplus
}
#endif
#endif
