/* include/tc_grad.h — the paper's own (lossy) differential: adaptive gradient compression and
 * fused multi-step Adam replay, on the GPU.
 *
 * PAPER.md:203 §3.2 — "gradients ... under 100K elements are compressed with dense INT8
 * quantization; otherwise ... estimates a magnitude threshold via sampling ... and selects
 * values in a single fused pass ... stored as FP16 values and INT32 indices; oversized tensors
 * are chunked before compression and safely rebased".  PAPER.md:283 §3.3 / P:322 §4 — the fused
 * replay "reads the model weights, first moments, and second moments exactly once, applies the
 * corresponding N-1 incremental gradients in temporal order ... and writes the final results
 * back", the final step going through the native optimizer path.  Readings (threshold sampler,
 * rounding, chunk size, Adam operation order) are DESIGN.md §12; the payload layout is the one
 * oracle/tco_grad.h documents (64-byte header "TCG1", INT8 codes or chunk table | FP16 values |
 * INT32 indices, sections padded to 16 bytes).
 *
 * Conventions as in tc.h (tc_status, sticky device errors at tc_ctx_check, 16-byte aligned
 * device pointers, stream-ordered, caller-owned buffers). */
#ifndef TC_GRAD_H
#define TC_GRAD_H
#include "tc.h"

#ifdef __cplusplus
extern "C" {
#endif

typedef struct tc_grad_opts {
    uint64_t small_threshold; /* < this many elements: INT8 dense (default 100000) */
    double k;                 /* kept fraction target of the sparse form (default 0.01) */
    uint32_t sample_size;     /* threshold sample (default 4096) */
    uint32_t reserved;
    uint64_t chunk_elems;     /* sparse chunk length, a multiple of 4096, <= 2^31-1 (default 2^31-4096) */
} tc_grad_opts;

typedef struct tc_adam_hp {
    /* defaults 1e-3, 0.9, 0.999, 1e-8.  Per element: m = b1 m + (1-b1) g;
     * v = b2 v + (1-b2) g^2; master -= step_size * (m / (sqrt(v) * inv_c2s + eps)), with
     * step_size = lr / (1 - beta1^t) and inv_c2s = 1 / sqrt(1 - beta2^t) evaluated in double and
     * rounded to fp32; beta1, beta2, eps used as their fp32 roundings (oracle/tco_grad.h) */
    double lr, beta1, beta2, eps;
} tc_adam_hp;

typedef struct tc_adam_state {
    float* master;    /* fp32 master weights, n */
    float* m;         /* fp32 first moments */
    float* v;         /* fp32 second moments */
    uint16_t* w16;    /* bf16 weights (bits), rewritten from master by every native step */
    uint64_t n;
} tc_adam_state;

/* Worst-case payload bytes for n elements (host only). */
tc_status tc_grad_bound(uint64_t n, const tc_grad_opts* opts, uint64_t* max_bytes);
/* Compress the fp32 gradient `grad` (n elements, device) into `out` (device, out_cap bytes;
 * tc_grad_bound always suffices; a smaller buffer -> sticky TC_ERR_CAPACITY, nothing written
 * past out_cap); *out_bytes (device or mapped pinned) = payload length.  `seed` drives the
 * threshold sample (deterministic).  Bytes are identical to oracle/tco_grad.c's. */
tc_status tc_grad_compress(tc_ctx* ctx, const float* grad, uint64_t n, const tc_grad_opts* opts, uint64_t seed,
                           void* out, uint64_t out_cap, uint64_t* out_bytes, tc_stream stream);
/* Decompress a payload of `bytes` bytes into the dense fp32 `out` (n elements).  A malformed
 * payload (header, chunk table, an index out of its chunk or not increasing) -> sticky
 * TC_ERR_CORRUPT; `out` is then unspecified. */
tc_status tc_grad_decompress(tc_ctx* ctx, const void* payload, uint64_t bytes, float* out, uint64_t n,
                             tc_stream stream);
/* One native Adam step (1-based `step`) with the dense fp32 gradient `grad`. */
tc_status tc_adam_step(tc_ctx* ctx, const tc_adam_state* st, const float* grad, const tc_adam_hp* hp,
                       uint64_t step, tc_stream stream);
/* Replay n_payloads compressed gradients of steps first_step, first_step+1, ...: the first
 * n_payloads-1 in ONE fused pass over (master, m, v) (read once, updated in registers, written
 * once), the last through tc_grad_decompress + tc_adam_step into `scratch` (n floats, device).
 * Bit-identical to sequential decompress + tc_adam_step per payload.
 * 1 <= n_payloads <= TC_MAX_FOLD. */
tc_status tc_adam_replay(tc_ctx* ctx, const tc_adam_state* st, const void* const* payloads,
                         const uint64_t* payload_bytes, int n_payloads, const tc_adam_hp* hp,
                         uint64_t first_step, float* scratch, tc_stream stream);

/* The native Adam step fused with the lossless differential of its own update (SURVEY.md §8(f)
 * NEXT row 2: "Adam already holds the old w/m/v and the new values in registers").  One pass
 * reads grad and the state, writes the updated state (only the words that changed) and one
 * change mask per state segment; the records are then built from those masks and the new state
 * (no reference copy, no re-read of ref and cur).  The diff has four segments, in this order:
 * 0 = w16 (2-byte words), 1 = master, 2 = m, 3 = v (4-byte words); version = step, ref_version
 * = step - 1; opts as for tc_diff_encode (advance_ref is ignored: the state itself advances).
 * Bytes equal tc_diff_encode(ref = state before, cur = state after).  out_cap as for
 * tc_diff_encode (device-checked, sticky TC_ERR_CAPACITY). */
tc_status tc_adam_step_encode(tc_ctx* ctx, const tc_adam_state* st, const float* grad, const tc_adam_hp* hp,
                              uint64_t step, const tc_encode_opts* opts, void* out, uint64_t out_cap,
                              uint64_t* out_bytes, tc_stream stream);

#ifdef __cplusplus
}
#endif
#endif
