// tc_internal.h — libtc internals shared by the runtime (.cpp) and the kernels (.cu).
// Product code only; nothing here is shared with oracle/ (DESIGN.md §2 independence).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <string>

#include "../../include/tc.h"

namespace tc {

constexpr uint32_t kHdrBytes = 64;
constexpr uint64_t kMaxChunkWords = 2147483647ull;  // 2^31-1 (PAPER.md:203 chunk + rebase)

// Encode block ("scan unit") sizes: one CTA stages ref+cur of one block in 32 KB of smem.
constexpr int TC_MAX_DEVICES = 64;          // per-device caches (function attributes)
constexpr uint32_t kEncThreads = 256;
constexpr uint32_t kEncBlockWords4 = 4096;  // 4-byte words
constexpr uint32_t kEncBlockWords2 = 8192;  // 2-byte words
// Fold: one warp per unit of max(T, kFoldWords) words.
constexpr uint32_t kFoldThreads = 256;
constexpr uint32_t kFoldWords = 4096;  // minimum fold unit (one warp: 128 mask words)
constexpr uint32_t kListMaxRec = 32;    // longest chain fold_list_kernel takes (its per-record tables)
constexpr uint32_t kListT = 4096;      // tile size of the chains fold_list_kernel takes (one tile = one unit)

__host__ __device__ inline uint64_t pad16(uint64_t x) { return (x + 15) & ~uint64_t(15); }
__host__ __device__ inline uint64_t cdiv(uint64_t a, uint64_t b) { return (a + b - 1) / b; }
__host__ __device__ inline uint64_t record_fixed_bytes(uint64_t m, uint32_t T) {
    return kHdrBytes + pad16(4 * cdiv(m, 32)) + pad16(4 * (cdiv(m, T) + 1));
}
__host__ __device__ inline uint64_t record_bytes(uint64_t m, uint32_t T, uint32_t w, uint64_t count) {
    return record_fixed_bytes(m, T) + pad16(uint64_t(w) * count);
}
// index mode (flags bit1): header | tile_off | idx u16[count] | values
__host__ __device__ inline uint64_t index_toff_off() { return kHdrBytes; }
__host__ __device__ inline uint64_t index_idx_off(uint64_t m, uint32_t T) { return kHdrBytes + pad16(4 * (cdiv(m, T) + 1)); }
__host__ __device__ inline uint64_t index_val_off(uint64_t m, uint32_t T, uint64_t count) {
    return index_idx_off(m, T) + pad16(2 * count);
}
__host__ __device__ inline uint64_t record_bytes_index(uint64_t m, uint32_t T, uint32_t w, uint64_t count) {
    return index_val_off(m, T, count) + pad16(uint64_t(w) * count);
}
constexpr uint32_t kIndexMaxT = 8192;
// full record (flags 5, reading R21): header | values (w * m), every word of the chunk
__host__ __device__ inline uint64_t record_bytes_full(uint64_t m, uint32_t w) { return kHdrBytes + pad16(uint64_t(w) * m); }
constexpr int kFormatFull = 2;  // tc_encode_opts.index_mode value of full records

// ---- per-segment launch description of one encode (kernel parameter, no table) ----
struct EncSeg {
    uint8_t* ref;
    const uint8_t* cur;
    uint64_t n;             // words
    uint64_t first_block;   // global block index of the segment's first block
    uint64_t first_chunk;   // global chunk index of the segment's first chunk
    uint64_t blocks_per_chunk;  // blocks of a full chunk (>= 1)
    uint64_t n_chunks;      // >= 1 (an empty segment is one empty chunk)
    uint32_t w;
    uint32_t block_words;   // B
    uint32_t seg_id;        // segment_id written in the headers
    uint32_t pad_;
    uint64_t word_base;     // added to chunk offsets in the headers (range encodes)
    const uint32_t* mask_in;  // precomputed change mask of the segment (kernel A', encode_maskin_kernel), else nullptr
    uint64_t full_base;       // full records (index_mode 2): byte offset of the segment's first record in out
};

struct EncParams {
    EncSeg seg[TC_MAX_SEGMENTS];
    int nseg;
    uint32_t T;
    uint64_t C;
    uint64_t total_blocks;
    uint64_t total_chunks;
    uint64_t n_groups;           // ceil(total_blocks / kEmitGroup)
    uint64_t version, ref_version;
    uint8_t* out;
    uint64_t out_cap;            // records are written only where they fit (else TC_ERR_CAPACITY)
    uint64_t* out_bytes;
    // scratch (tc_ctx), zeroed per call: ticket | chunk_acc | rstart | group_sum
    unsigned long long* ticket;
    unsigned long long* chunk_acc;    // [total_chunks] {blocks counted : 24 | changed words : 40}
    unsigned long long* rstart;       // [total_chunks + 1] record start | 1 once published
    unsigned long long* group_sum;    // [n_groups] changed words per group of kEmitGroup blocks
    // scratch, fully written each call
    uint32_t* info;                   // [total_blocks] count | kDenseFlag
    unsigned long long* gpre;         // [n_groups] exclusive prefix of group_sum
    unsigned long long* cbase;        // [total_chunks] exclusive prefix of the chunk counts
    uint8_t* spill;                   // [total_blocks] slots of kSpillBytes: packed values
    unsigned int* err;                // sticky error word
    uint32_t* mstage;                 // index mode: [total_blocks][kMaskStageWords] mask words
    int advance_ref;
    int index_mode;
    // fused Tier-2 emit (tc_diff_encode_push): every record byte is also stored at the same offset
    // of the ring neighbour's slot (NVLink), where it fits peer_cap; the last emit CTA publishes
    // {bytes | UINT64_MAX if refused, peer_version} into peer_mail.  peer_out == nullptr: off.
    uint8_t* peer_out;
    uint64_t peer_cap;
    unsigned long long* peer_mail;
    uint64_t peer_version;
    unsigned int* peer_counter;
    uint64_t full_total;         // full records: the diff's length (known up front)
};

constexpr uint32_t kMaskStageWords = 256;  // mask words of one block (8192 16-bit words max)

constexpr uint32_t kEmitGroup = 256;        // blocks per emit CTA / per group sum
constexpr uint32_t kSpillBytes = 4096;      // per-block spill slot (1/4 of a block's words)
// mask mode: spill slot per block.  8 KB = the index mode's slot (2 x kSpillBytes: values and
// positions), so a context that encodes both formats holds one buffer; with kernel B's vector
// copy it beats re-reading cur for blocks of up to 2048 fp32 / 4096 bf16 changed words
// (f = 30 % 16.3 -> 14.2 ms).  Experiment builds override it.
#ifndef TC_SPILL_MASK
#define TC_SPILL_MASK 8192
#endif
constexpr uint32_t kSpillMask = TC_SPILL_MASK;
constexpr uint32_t kDenseFlag = 0x80000000u;
constexpr int kAccDoneShift = 40;  // chunk_acc: blocks counted above bit 40 (a chunk has <= 2^19 blocks)
constexpr unsigned long long kAccCountMask = (1ull << kAccDoneShift) - 1;

// ---- fold descriptors ----
struct FoldRec {           // one record of one diff, as located by the walker
    const uint8_t* mask;   // mask mode (nullptr in index mode)
    const uint8_t* idx;    // index mode: u16 in-tile positions (nullptr in mask mode)
    const uint8_t* toff;
    const uint8_t* values;
    uint64_t chunk_off;
    uint64_t count;
    uint32_t m;
    uint32_t T;
    uint32_t seg;
    uint32_t w;
    uint32_t dense;        // desc[r] of diff 0 only: 0 fold_kernel, 1 fold_dense_kernel, 2 fold_list_kernel
    uint32_t full;         // a full record (every word of the chunk; mask / idx / toff are nullptr)
};

struct FoldParams {
    uint8_t* state[TC_MAX_SEGMENTS];
    uint64_t n[TC_MAX_SEGMENTS];
    uint32_t w[TC_MAX_SEGMENTS];
    const uint8_t* rec[TC_MAX_FOLD];
    uint64_t rec_bytes[TC_MAX_FOLD];
    int nseg;
    int nrec;               // diffs folded
    uint32_t cap;           // descriptor capacity per diff
    uint32_t cap_hinted;    // cap comes from tc_ctx_set_fold_max_records: more records -> TC_ERR_CAPACITY
    uint64_t state_version;
    uint32_t dense_permille;  // chunk r is dense when sum_j count_j * 1000 > m * dense_permille
    FoldRec* desc;          // [nrec][cap]
    uint64_t* unit_first;   // [cap + 1]
    unsigned long long* info;  // [0] records per diff, [1] total units, chunks for [2] fold_dense, [3] fold, [4] fold_list, [5] fold_entries
    unsigned int* err;
};

// launchers (tc_encode.cu / tc_apply.cu / tc_synth.cu); return cudaError_t
cudaError_t launch_encode(const EncParams& p, cudaStream_t s);
cudaError_t launch_fold(const FoldParams& p, cudaStream_t s, int num_sms, uint64_t* launches);

// thread-local detail string
void set_error(const std::string& msg);

// tc_ctx accessors for the other translation units (the struct is private to tc_runtime.cu)
unsigned int* ctx_err(tc_ctx* c);
int ctx_device(tc_ctx* c);
int ctx_num_sms(tc_ctx* c);
void ctx_add_launches(tc_ctx* c, uint64_t n);
uint32_t ctx_push_ctas(tc_ctx* c);
tc_status ctx_grad_scratch(tc_ctx* c, size_t bytes, cudaStream_t s, void** out);
tc_status encode_push(tc_ctx* ctx, const tc_segment* segs, int nseg, const tc_encode_opts* opts, uint64_t version,
                      uint64_t ref_version, void* out, uint64_t out_cap, uint64_t* out_bytes, void* peer_dst,
                      uint64_t peer_cap, void* peer_mailbox, cudaStream_t s);
tc_status encode_from_masks(tc_ctx* ctx, const tc_segment* segs, const uint32_t* const* masks, int nseg,
                            const tc_encode_opts* opts, uint64_t version, uint64_t ref_version, void* out,
                            uint64_t out_cap, uint64_t* out_bytes, cudaStream_t s);

}  // namespace tc

// device-side sticky error: first error wins
#ifdef __CUDACC__
__device__ __forceinline__ void tc_set_err(unsigned int* err, unsigned int code) {
    atomicCAS(err, 0u, code);
}
#endif
