// tc_encode.cu — the differential-checkpoint encoder for sm_100a (tc_diff_encode).
//
// What it computes: for every chunk of every segment,
// the mask of changed words (unsigned bitwise compare, reading R5), the in-chunk exclusive
// counts at every tile start (tile_off), the packed new words (values) and the record header;
// optionally ref[i] <- cur[i] for the changed words.  The paper extracts and compacts the
// surviving entries in "a single fused pass" (§3.2) instead of multi-pass Top-K;
// here the one pass over the 2W bytes of ref+cur is kernel A, and everything else touches only
// the changed words.
//
// Three launches, no look-back chain through HBM latency (DESIGN.md §7.1 explains why the
// decoupled look-back single pass of v1 capped at ~2.5 TB/s):
//   A  encode_mask_kernel   one CTA per scan block of B words (B = 4096 4-byte / 8192 2-byte
//                           words; 16 KB per operand).  A dynamic ticket orders the blocks.
//                           ref+cur are staged by two 1-D TMA bulk copies into shared memory;
//                           each lane compares one 128-bit vector (4 fp32 / 8 bf16 words) and a
//                           shfl_xor OR across the 8 | 4 lanes sharing a mask word assembles it
//                           (LSB-first); __popc + warp scans give counts; ref advance is fused.  A sparse
//                           block (<= 8 KB of changed words in mask records, <= 4 KB in index
//                           records) packs its new words into its spill slot; a dense one leaves
//                           them for kernel B.  The mask and the
//                           block-relative tile_off entries go straight to their final place once
//                           the chunk's record start is known (chunk c waits only for chunk c-1's
//                           counts, i.e. only at chunk boundaries); the block completing a chunk
//                           writes its header and publishes the next record start.
//   A' encode_maskin_kernel the mask-input variant (tc_adam_step_encode: the mask comes from the
//                           Adam pass, no ref): persistent warps, a warp per block, 4 blocks per
//                           ticket; same outputs as A.
//   P  encode_prefix_kernel (1 CTA) exclusive scans of the per-group and per-chunk counts.
//   B  encode_emit_kernel   one CTA per 256 blocks: block-wide scan of the block counts -> each
//                           block's in-chunk prefix (a thread per block, which also adds it to
//                           the block's tile_off entries); each warp then moves its blocks'
//                           spilled words into place (runs of <= 64 words 4 blocks per batch,
//                           longer ones in 16-byte vectors) and packs dense blocks from mask + cur.
#include <cuda_runtime.h>

#include "tc_internal.h"
#include "tc_ptx.cuh"

namespace tc {

namespace {

constexpr uint32_t kSpinLimit = 1u << 26;  // watchdog: a bug must not hang the GPU

__device__ __forceinline__ unsigned long long ld_relaxed(const unsigned long long* p) {
    unsigned long long v;
    asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_relaxed(unsigned long long* p, unsigned long long v) {
    asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
template <int W>
struct Word;
template <>
struct Word<4> {
    using T = uint32_t;
    static constexpr uint32_t kBlock = kEncBlockWords4;
};
template <>
struct Word<2> {
    using T = uint16_t;
    static constexpr uint32_t kBlock = kEncBlockWords2;
};

constexpr uint32_t kWarps = kEncThreads / 32;

// Where block b lives (pure arithmetic on the per-segment launch table).
struct BlockInfo {
    unsigned long long b;          // global block index
    unsigned long long chunk;      // global chunk index
    unsigned long long chunk_off;  // word offset of the chunk in its segment
    uint32_t m;                    // words in the chunk
    uint32_t k;                    // block index within the chunk
    uint32_t nblk;                 // blocks in the chunk
    uint32_t p0;                   // chunk-relative first word of the block
    uint32_t nb;                   // words in this block
    uint32_t seg;
    uint32_t w;
};

__device__ __forceinline__ BlockInfo decode_block(const EncParams& P, unsigned long long b) {
    BlockInfo I;
    I.b = b;
    int s = 0;
    while (s + 1 < P.nseg && b >= P.seg[s + 1].first_block) ++s;
    const EncSeg& S = P.seg[s];
    const uint32_t lb = static_cast<uint32_t>(b - S.first_block);
    const uint32_t bpc = static_cast<uint32_t>(S.blocks_per_chunk);
    const uint32_t cl = lb / bpc;
    I.k = lb - cl * bpc;
    I.seg = s;
    I.w = S.w;
    I.chunk = S.first_chunk + cl;
    I.chunk_off = static_cast<unsigned long long>(cl) * P.C;
    I.m = static_cast<uint32_t>(S.n - I.chunk_off < P.C ? S.n - I.chunk_off : P.C);
    I.nblk = I.m ? (I.m + S.block_words - 1) / S.block_words : 1u;
    I.p0 = I.k * S.block_words;
    I.nb = I.m > I.p0 ? (I.m - I.p0 < S.block_words ? I.m - I.p0 : S.block_words) : 0u;
    return I;
}

// Record start of chunk c (published by the block completing chunk c-1 as value | 1).
__device__ __forceinline__ unsigned long long wait_rstart(const EncParams& P, unsigned long long c) {
    if (c == 0) return 0;
    uint32_t spins = 0;
    unsigned long long v;
    while (((v = ld_relaxed(&P.rstart[c])) & 1ull) == 0) {
        if (++spins > kSpinLimit) {
            tc_set_err(P.err, TC_ERR_INTERNAL);
            return 0;
        }
        __nanosleep(64);
    }
    return v & ~1ull;
}

struct SmemA {
    BlockInfo I;
    uint64_t bar;
    uint32_t warp_cnt[kWarps];
    unsigned long long rs;
};

// ------------------------------------------------------------------ kernel A ------------
__device__ __forceinline__ uint32_t ldg_cur(const uint32_t* p) { return __ldg(p); }
__device__ __forceinline__ uint16_t ldg_cur(const uint16_t* p) {
    return static_cast<uint16_t>(__ldg(reinterpret_cast<const unsigned short*>(p)));
}

// Every record write goes through rec_store: with the fused Tier-2 emit on (P.peer_out), the same
// bytes are also stored at the same offset of the ring neighbour's slot over NVLink — where they fit
// its capacity (§3.2).  The record is never re-read.
template <bool PEER, typename T>
__device__ __forceinline__ void rec_store(const EncParams& P, T* local, T v) {
    *local = v;
    if (PEER) {
        const uint64_t o = static_cast<uint64_t>(reinterpret_cast<const uint8_t*>(local) - P.out);
        if (o + sizeof(T) <= P.peer_cap) *reinterpret_cast<T*>(P.peer_out + o) = v;
    }
}
// Block / chunk bookkeeping (one thread, after its own stores; nobody waits for it): one packed
// atomic {done blocks : 24 | changed words : 40} per chunk tells the block that completes the
// chunk, which writes the header and publishes the next record start.  `nblocks` blocks of chunk
// I.chunk with `total` changed words between them are counted at once (kernel A: one block).
__device__ __forceinline__ void note_block(const EncParams& P, unsigned long long b, uint32_t total, bool sparse) {
    P.info[b] = total | (sparse ? 0u : kDenseFlag);
    atomicAdd(&P.group_sum[b / kEmitGroup], static_cast<unsigned long long>(total));
}

template <int W, bool PEER>
__device__ __forceinline__ void count_blocks(const EncParams& P, const BlockInfo& I, uint32_t nblocks,
                                             unsigned long long total, unsigned long long rs) {
    const bool imode = P.index_mode != 0;
    const unsigned long long old =
        atomicAdd(&P.chunk_acc[I.chunk], (static_cast<unsigned long long>(nblocks) << kAccDoneShift) | total);
    if ((old >> kAccDoneShift) + nblocks == I.nblk) {
        const uint64_t count = (old & kAccCountMask) + total;
        const uint64_t n_mask = cdiv(I.m, 32);
        const uint64_t n_tiles = cdiv(I.m, P.T);
        const uint64_t rec_total = imode ? record_bytes_index(I.m, P.T, W, count) : record_bytes(I.m, P.T, W, count);
        const unsigned long long next = rs + rec_total;
        if (next > P.out_cap) tc_set_err(P.err, TC_ERR_CAPACITY);  // this record is not written
        else {
        uint8_t* rec = P.out + rs;
        uint64_t* h = reinterpret_cast<uint64_t*>(rec);
        rec_store<PEER, uint64_t>(P, h + 0, 0x31444354ull /* "TCD1" */ | (1ull << 32) | (static_cast<uint64_t>(W) << 48) |
                                          ((imode ? 3ull : 1ull) << 56));
        rec_store<PEER, uint64_t>(P, h + 1, static_cast<uint64_t>(P.T) | (static_cast<uint64_t>(P.seg[I.seg].seg_id) << 32));
        rec_store<PEER, uint64_t>(P, h + 2, P.seg[I.seg].word_base + I.chunk_off);
        rec_store<PEER, uint64_t>(P, h + 3, I.m);
        rec_store<PEER, uint64_t>(P, h + 4, count);
        rec_store<PEER, uint64_t>(P, h + 5, P.version);
        rec_store<PEER, uint64_t>(P, h + 6, P.ref_version);
        rec_store<PEER, uint64_t>(P, h + 7, rec_total);
        uint32_t* gtoff;
        uint8_t* gval;
        if (imode) {
            gtoff = reinterpret_cast<uint32_t*>(rec + index_toff_off());
            uint8_t* gidx = rec + index_idx_off(I.m, P.T);
            for (uint64_t x = 2 * count; x < pad16(2 * count); ++x) rec_store<PEER, uint8_t>(P, gidx + x, 0);
            gval = rec + index_val_off(I.m, P.T, count);
        } else {
            uint32_t* gmask = reinterpret_cast<uint32_t*>(rec + kHdrBytes);
            for (uint64_t x = n_mask; x < pad16(4 * n_mask) / 4; ++x) rec_store<PEER, uint32_t>(P, gmask + x, 0u);
            gtoff = reinterpret_cast<uint32_t*>(rec + kHdrBytes + pad16(4 * n_mask));
            gval = rec + record_fixed_bytes(I.m, P.T);
        }
        rec_store<PEER, uint32_t>(P, gtoff + n_tiles, static_cast<uint32_t>(count));
        for (uint64_t x = n_tiles + 1; x < pad16(4 * (n_tiles + 1)) / 4; ++x) rec_store<PEER, uint32_t>(P, gtoff + x, 0u);
        for (uint64_t x = W * count; x < pad16(W * count); ++x) rec_store<PEER, uint8_t>(P, gval + x, 0);
        }
        st_relaxed(&P.rstart[I.chunk + 1], next | 1ull);
        if (I.chunk + 1 == P.total_chunks) *P.out_bytes = next;
    }
}

template <int W, bool PEER>
__device__ __forceinline__ void mask_block(const EncParams& P, SmemA& sm, uint8_t* tile, int tid) {
    using word_t = typename Word<W>::T;
    constexpr uint32_t B = Word<W>::kBlock;
    constexpr uint32_t MPW = B / 32 / kWarps;  // mask words per warp (16 | 32)
    const int lane = tid & 31, wid = tid >> 5;
    const BlockInfo I = sm.I;
    const EncSeg& S = P.seg[I.seg];
    word_t* sref = reinterpret_cast<word_t*>(tile);
    word_t* scur = sref + B;
    word_t* gref = reinterpret_cast<word_t*>(S.ref) + I.chunk_off + I.p0;
    const word_t* gcur = reinterpret_cast<const word_t*>(S.cur) + I.chunk_off + I.p0;

    const bool adv = P.advance_ref != 0;
    const uint32_t mw0 = wid * MPW;
    uint32_t mine = 0;  // lane q keeps mask word mw0 + q
    // words past the bulk copy: the < 16-byte tail, and equal padding up to B so that pass 1
    // needs no bounds test
    if (I.nb < B) {
        const uint32_t bulk = (I.nb * W) & ~15u;
        for (uint32_t i = bulk / W + tid; i < B; i += kEncThreads) {
            const bool in = i < I.nb;
            sref[i] = in ? gref[i] : word_t(0);
            scur[i] = in ? gcur[i] : word_t(0);
        }
    }
    mbar_wait_parity(&sm.bar, 0);
    if (I.nb < B) __syncthreads();

    // ---- pass 1: 128-bit shared loads, per-lane change bits -> mask words; fused ref advance.
    //      Lane l of iteration q compares words [VW*(32q'+l), +VW) (VW = 16 / W): its VW change
    //      bits are OR-shuffled across the VW/... lanes of one 32-word mask word (LSB-first). ----
    {
        constexpr uint32_t VW = 16 / W;          // words per 128-bit vector (4 | 8)
        constexpr uint32_t LPM = 32 / VW;        // lanes per mask word (8 | 4)
        constexpr uint32_t ITER = MPW * 32 / (32 * VW);  // vectors per lane over the warp range (4)
        const uint4* r4 = reinterpret_cast<const uint4*>(sref);
        const uint4* c4 = reinterpret_cast<const uint4*>(scur);
        uint4* g4 = reinterpret_cast<uint4*>(gref);
        uint32_t* s_bal = reinterpret_cast<uint32_t*>(tile) + (2 * B * W) / 4;  // after ref|cur
#pragma unroll
        for (uint32_t q = 0; q < ITER; ++q) {
            const uint32_t vi = (wid * ITER + q) * 32 + lane;  // vector index in the block
            const uint4 a = r4[vi];
            const uint4 v = c4[vi];
            uint32_t bits;
            if (W == 4) {
                bits = (a.x != v.x ? 1u : 0u) | (a.y != v.y ? 2u : 0u) | (a.z != v.z ? 4u : 0u) | (a.w != v.w ? 8u : 0u);
            } else {
                const uint32_t d0 = __vcmpne2(a.x, v.x), d1 = __vcmpne2(a.y, v.y);
                const uint32_t d2 = __vcmpne2(a.z, v.z), d3 = __vcmpne2(a.w, v.w);
                bits = (d0 & 1u) | ((d0 >> 15) & 2u) | ((d1 & 1u) << 2) | ((d1 >> 13) & 8u) |
                       ((d2 & 1u) << 4) | ((d2 >> 11) & 32u) | ((d3 & 1u) << 6) | ((d3 >> 9) & 128u);
            }
            if (adv && bits) {
                if ((vi + 1) * VW <= I.nb) {
                    g4[vi] = v;  // new ref = cur on the whole vector (equal where unchanged)
                } else {
                    // the vector straddling the segment end: only its in-range words (the ref may
                    // be a view into a larger buffer; nothing past n_words is written)
                    const word_t* cv = scur + vi * VW;
                    for (uint32_t k = 0; k < VW; ++k)
                        if ((bits >> k) & 1u) gref[vi * VW + k] = cv[k];
                }
            }
            uint32_t x = bits << (VW * (lane & (LPM - 1)));
#pragma unroll
            for (uint32_t d = 1; d < LPM; d <<= 1) x |= __shfl_xor_sync(0xffffffffu, x, d);
            if ((lane & (LPM - 1)) == 0) s_bal[mw0 + q * (32 / LPM) + lane / LPM] = x;
        }
        __syncwarp();
    }
    if (lane < static_cast<int>(MPW))
        mine = reinterpret_cast<const uint32_t*>(tile)[(2 * B * W) / 4 + mw0 + lane];
    // ---- counts: lane-per-mask-word popcount scan over the warp's range (the barrier below
    //      also publishes thread 0's prefetched record start) ----
    const uint32_t c = __popc(mine);
    uint32_t inc = c;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        const uint32_t t = __shfl_up_sync(0xffffffffu, inc, d);
        if (lane >= d) inc += t;
    }
    const uint32_t pre = inc - c;  // changed words of the warp range before this mask word
    if (lane == 31) sm.warp_cnt[wid] = inc;
    __syncthreads();
    uint32_t woff = 0, total = 0;
#pragma unroll
    for (int k = 0; k < static_cast<int>(kWarps); ++k) {
        const uint32_t v = sm.warp_cnt[k];
        woff += k < wid ? v : 0u;
        total += v;
    }
    const bool imode = P.index_mode != 0;
    const bool sparse = total * W <= (imode ? kSpillBytes : kSpillMask);

    // ---- sparse block: pack the new words into the block's spill slot now (index mode: and
    //      their u16 in-tile positions in the second half of the slot) ----
    const size_t slot_bytes = imode ? 2 * kSpillBytes : kSpillMask;
    if (sparse && total) {
        word_t* slot = reinterpret_cast<word_t*>(P.spill + I.b * slot_bytes) + woff;
        uint16_t* islot = reinterpret_cast<uint16_t*>(P.spill + I.b * slot_bytes + kSpillBytes) + woff;
        const uint32_t tmask = P.T - 1;
#ifndef TC_PACK_SERIAL
#define TC_PACK_SERIAL 96
#endif
        if (__shfl_sync(0xffffffffu, inc, 31) <= TC_PACK_SERIAL) {
            // few changes in this warp's range: each lane packs its own mask word's words
            uint32_t wv = mine;
            uint32_t k = pre;
            const uint32_t q0 = (mw0 + lane) * 32;
            while (wv) {
                const uint32_t b = __ffs(wv) - 1;
                wv &= wv - 1;
                slot[k] = scur[q0 + b];
                if (imode) islot[k] = static_cast<uint16_t>((I.p0 + q0 + b) & tmask);
                ++k;
            }
        } else {
            // many changes in this warp's range (round 2, vectorized): lane l re-derives the change
            // bits of its vector of iteration q from the shared tile, a warp scan of the lanes'
            // popcounts places its words after those of the lanes (and iterations) before
            constexpr uint32_t kVW = 16 / W;
            constexpr uint32_t kIter = MPW * 32 / (32 * kVW);
            const uint4* r4 = reinterpret_cast<const uint4*>(sref);
            const uint4* c4 = reinterpret_cast<const uint4*>(scur);
            uint32_t run = 0;
#pragma unroll
            for (uint32_t q = 0; q < kIter; ++q) {
                const uint32_t vi = (wid * kIter + q) * 32 + lane;
                const uint4 a = r4[vi];
                const uint4 v = c4[vi];
                uint32_t bits;
                if (W == 4) {
                    bits = (a.x != v.x ? 1u : 0u) | (a.y != v.y ? 2u : 0u) | (a.z != v.z ? 4u : 0u) | (a.w != v.w ? 8u : 0u);
                } else {
                    const uint32_t d0 = __vcmpne2(a.x, v.x), d1 = __vcmpne2(a.y, v.y);
                    const uint32_t d2 = __vcmpne2(a.z, v.z), d3 = __vcmpne2(a.w, v.w);
                    bits = (d0 & 1u) | ((d0 >> 15) & 2u) | ((d1 & 1u) << 2) | ((d1 >> 13) & 8u) |
                           ((d2 & 1u) << 4) | ((d2 >> 11) & 32u) | ((d3 & 1u) << 6) | ((d3 >> 9) & 128u);
                }
                const uint32_t c2 = __popc(bits);
                uint32_t inc2 = c2;
#pragma unroll
                for (int d = 1; d < 32; d <<= 1) {
                    const uint32_t t = __shfl_up_sync(0xffffffffu, inc2, d);
                    if (lane >= d) inc2 += t;
                }
                uint32_t o = run + inc2 - c2;
                run += __shfl_sync(0xffffffffu, inc2, 31);
                const word_t* cv = scur + vi * kVW;
#pragma unroll
                for (uint32_t e = 0; e < kVW; ++e)
                    if ((bits >> e) & 1u) {
                        slot[o] = cv[e];
                        if (imode) islot[o] = static_cast<uint16_t>((I.p0 + vi * kVW + e) & tmask);
                        ++o;
                    }
            }
        }
    }
    // index mode, dense block: its mask words go to the staging area (kernel B packs from them)
    if (imode && !sparse && lane < static_cast<int>(MPW))
        P.mstage[I.b * kMaskStageWords + mw0 + lane] = mine;

    // ---- record start of the chunk: prefetched by thread 0 at block start; only the first
    //      blocks of a chunk can find it unpublished and wait (block-uniform branch) ----
    unsigned long long rs = sm.rs;
    if (!(rs & 1ull)) {
        __syncthreads();  // every thread has read sm.rs before thread 0 rewrites it
        if (tid == 0) sm.rs = wait_rstart(P, I.chunk) | 1ull;
        __syncthreads();
        rs = sm.rs;
    }
    rs &= ~1ull;

    // ---- mask words (mask mode) and block-relative tile_off entries, in their final place
    //      (only where the record's fixed sections fit the output buffer) ----
    const uint64_t fixed = imode ? index_idx_off(I.m, P.T) : record_fixed_bytes(I.m, P.T);
    if (rs + fixed > P.out_cap) {
        if (tid == 0) tc_set_err(P.err, TC_ERR_CAPACITY);
    } else {
        uint8_t* rec = P.out + rs;
        const uint64_t n_mask = cdiv(I.m, 32);
        uint32_t* gmask = reinterpret_cast<uint32_t*>(rec + kHdrBytes);
        uint32_t* gtoff = reinterpret_cast<uint32_t*>(rec + (imode ? index_toff_off() : kHdrBytes + pad16(4 * n_mask)));
        const uint32_t p = I.p0 + (mw0 + lane) * 32;
        if (lane < static_cast<int>(MPW) && p < I.m) {
            if (!imode) rec_store<PEER, uint32_t>(P, gmask + (I.p0 >> 5) + mw0 + lane, mine);
            if ((p & (P.T - 1)) == 0) gtoff[p / P.T] = woff + pre;  // kernel B adds the block prefix
        }
    }

    if (tid == 0) {
        note_block(P, I.b, total, sparse);
        count_blocks<W, PEER>(P, I, 1, total, rs);
    }
    // (kernel A's NVLink stores are ordered before kernel B's publish by the kernel boundary and
    // B's system-scope fence; a per-CTA fence here cost 2.5x on the encode: r2 measurement)
}

template <bool PEER>
__global__ void __launch_bounds__(kEncThreads, 6) encode_mask_kernel(const __grid_constant__ EncParams P) {
    extern __shared__ __align__(128) uint8_t tile[];
    __shared__ SmemA sm;
    const int tid = threadIdx.x;
    if (tid == 0) {
        // one thread: ticket, decode, barrier init, TMA issue — the loads start at once
        const BlockInfo I = decode_block(P, atomicAdd(P.ticket, 1ull));
        sm.I = I;
        mbar_init(&sm.bar, 1);
        sm.rs = I.chunk == 0 ? 1ull : 0ull;  // chunk 0 starts at 0; others: prefetched below
        const uint32_t bulk = (I.nb * I.w) & ~15u;
        if (bulk) {
            const EncSeg& S = P.seg[I.seg];
            const uint8_t* gref = S.ref + (I.chunk_off + I.p0) * I.w;
            const uint8_t* gcur = S.cur + (I.chunk_off + I.p0) * I.w;
            mbar_arrive_expect_tx(&sm.bar, 2 * bulk);
            bulk_g2s(tile, gref, bulk, &sm.bar);
            bulk_g2s(tile + 16384, gcur, bulk, &sm.bar);
        } else {
            mbar_arrive(&sm.bar);
        }
    }
    __syncthreads();
    if (tid == 0 && sm.I.chunk != 0) sm.rs = ld_relaxed(&P.rstart[sm.I.chunk]);  // value | 1 once published
    if (sm.I.w == 4)
        mask_block<4, PEER>(P, sm, tile, tid);
    else
        mask_block<2, PEER>(P, sm, tile, tid);
}

// ------------------------------------------------------------------ kernel F -------------
// Full records (tc_encode_opts.index_mode = 2; reading R21): every word of the chunk, no mask —
// the dense-regime format (every fp32 word of a real Adam step changes).  Record
// sizes do not depend on the data, so every block knows its output position up front: one
// streaming pass, cur -> record values (+ ref <- cur with advance_ref), 3 W of HBM traffic and no
// compare, no prefix, no spill.  A CTA per scan block; the chunk's first block writes the header,
// its last the padding; block 0 the diff's length.  With the fused Tier-2 emit (PEER) the same
// bytes also go to the neighbour's slot and the last CTA publishes the mailbox.
template <bool PEER>
__global__ void __launch_bounds__(kEncThreads) encode_full_kernel(const __grid_constant__ EncParams P) {
    const int tid = threadIdx.x;
    const BlockInfo I = decode_block(P, blockIdx.x);
    const EncSeg& S = P.seg[I.seg];
    const unsigned long long cl = I.chunk - S.first_chunk;
    const unsigned long long rs = S.full_base + cl * record_bytes_full(P.C, I.w);  // earlier chunks are full
    const uint64_t total = record_bytes_full(I.m, I.w);
    if (rs + total > P.out_cap) {
        if (tid == 0 && I.k == 0) tc_set_err(P.err, TC_ERR_CAPACITY);  // this record is not written
    } else {
        uint8_t* rec = P.out + rs;
        const uint32_t nbytes = I.nb * I.w;
        const uint4* src = reinterpret_cast<const uint4*>(S.cur + (I.chunk_off + I.p0) * I.w);
        uint4* dst = reinterpret_cast<uint4*>(rec + kHdrBytes + static_cast<uint64_t>(I.p0) * I.w);
        uint4* ref = reinterpret_cast<uint4*>(S.ref + (I.chunk_off + I.p0) * I.w);
        const uint32_t nv = nbytes / 16;
        const bool adv = P.advance_ref != 0;
        constexpr uint32_t kV = 16384 / 16 / kEncThreads;  // 4 vectors per thread per block
        uint4 v[kV];
#pragma unroll
        for (uint32_t q = 0; q < kV; ++q) {
            const uint32_t i = tid + q * kEncThreads;
            if (i < nv) v[q] = __ldg(src + i);
        }
#pragma unroll
        for (uint32_t q = 0; q < kV; ++q) {
            const uint32_t i = tid + q * kEncThreads;
            if (i < nv) {
                rec_store<PEER, uint4>(P, dst + i, v[q]);
                if (adv) ref[i] = v[q];
            }
        }
        // the segment's last block: the words past the last whole 16-byte vector
        for (uint32_t x = nv * 16 + tid * I.w; x < nbytes; x += kEncThreads * I.w) {
            const uint8_t* sb = reinterpret_cast<const uint8_t*>(src) + x;
            uint8_t* db = reinterpret_cast<uint8_t*>(dst) + x;
            uint8_t* rb = reinterpret_cast<uint8_t*>(ref) + x;
            if (I.w == 4) {
                const uint32_t wv = *reinterpret_cast<const uint32_t*>(sb);
                rec_store<PEER, uint32_t>(P, reinterpret_cast<uint32_t*>(db), wv);
                if (adv) *reinterpret_cast<uint32_t*>(rb) = wv;
            } else {
                const uint16_t wv = *reinterpret_cast<const uint16_t*>(sb);
                rec_store<PEER, uint16_t>(P, reinterpret_cast<uint16_t*>(db), wv);
                if (adv) *reinterpret_cast<uint16_t*>(rb) = wv;
            }
        }
        if (tid == 0 && I.k == 0) {
            uint64_t* h = reinterpret_cast<uint64_t*>(rec);
            rec_store<PEER, uint64_t>(P, h + 0, 0x31444354ull /* "TCD1" */ | (1ull << 32) |
                                                    (static_cast<uint64_t>(I.w) << 48) | (5ull << 56));
            rec_store<PEER, uint64_t>(P, h + 1, static_cast<uint64_t>(P.T) | (static_cast<uint64_t>(S.seg_id) << 32));
            rec_store<PEER, uint64_t>(P, h + 2, S.word_base + I.chunk_off);
            rec_store<PEER, uint64_t>(P, h + 3, I.m);
            rec_store<PEER, uint64_t>(P, h + 4, I.m);  // count: every word
            rec_store<PEER, uint64_t>(P, h + 5, P.version);
            rec_store<PEER, uint64_t>(P, h + 6, P.ref_version);
            rec_store<PEER, uint64_t>(P, h + 7, total);
        }
        if (I.k + 1 == I.nblk)
            for (uint64_t x = kHdrBytes + static_cast<uint64_t>(I.w) * I.m + tid; x < total; x += kEncThreads)
                rec_store<PEER, uint8_t>(P, rec + x, 0);
    }
    if (blockIdx.x == 0 && tid == 0) *reinterpret_cast<volatile uint64_t*>(P.out_bytes) = P.full_total;
    if (PEER) {
        __threadfence_system();
        __syncthreads();
        if (tid == 0) {
            const unsigned prev = atomicAdd(P.peer_counter, 1u);
            if (prev == gridDim.x - 1) {
                *P.peer_counter = 0u;
                __threadfence_system();
                const unsigned long long nb = P.full_total;
                const bool ok = nb <= P.peer_cap && *reinterpret_cast<const volatile unsigned int*>(P.err) == 0u;
                asm volatile("st.relaxed.sys.global.u64 [%0], %1;" ::"l"(P.peer_mail), "l"(ok ? nb : ~0ull) : "memory");
                asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(P.peer_mail + 1),
                             "l"(static_cast<unsigned long long>(P.peer_version)) : "memory");
            }
        }
    }
}

// ------------------------------------------------------------------ kernel A' -----------
// Mask-input variant of kernel A (EncSeg::mask_in: the change mask comes precomputed, e.g. from
// the fused Adam step, tc_adam_step_encode; `cur` is the only state: no ref, no compare, no ref
// advance).  Without a tile to stage a block is a few hundred bytes of mask words, so one WARP
// takes a block (persistent warps, each claiming tickets in order): lane l holds mask words
// [l·K, l·K+K) of the block (K = 4 | 8, 16-byte loads), popcounts + one warp scan give the
// offsets, a sparse block gathers its changed words from global cur into its spill slot (lane-
// serial, or mask word by mask word when a lane holds many), and the rest — mask / tile_off
// stores, index-mode staging, bookkeeping — is kernel A's, so kernels P and B are unchanged.
// Returns the block's changed words; *rs_out = the chunk's record start.
template <int W>
__device__ __forceinline__ uint32_t maskin_block(const EncParams& P, const BlockInfo& I, unsigned long long rs,
                                                 int lane, unsigned long long* rs_out) {
    using word_t = typename Word<W>::T;
    constexpr uint32_t B = Word<W>::kBlock;
    constexpr uint32_t K = B / 32 / 32;  // mask words per lane (4 | 8)
    const EncSeg& S = P.seg[I.seg];
    const word_t* gcur = reinterpret_cast<const word_t*>(S.cur) + I.chunk_off + I.p0;
    const uint32_t* gm = S.mask_in + ((I.chunk_off + I.p0) >> 5) + lane * K;
    const uint32_t nmw = (I.nb + 31) / 32;
    uint32_t mw[K];
    // 16-byte loads where the chunk start keeps them aligned (chunk_words need only be a
    // multiple of T >= 32, so a chunk's first mask word can sit at any 4-byte offset)
    if ((lane + 1) * K <= nmw && ((I.chunk_off >> 5) & 3) == 0) {
#pragma unroll
        for (uint32_t v = 0; v < K / 4; ++v) {
            const uint4 x = __ldg(reinterpret_cast<const uint4*>(gm) + v);
            mw[4 * v] = x.x, mw[4 * v + 1] = x.y, mw[4 * v + 2] = x.z, mw[4 * v + 3] = x.w;
        }
    } else {
#pragma unroll
        for (uint32_t j = 0; j < K; ++j) mw[j] = lane * K + j < nmw ? __ldg(gm + j) : 0u;
    }
    uint32_t c = 0;
#pragma unroll
    for (uint32_t j = 0; j < K; ++j) c += __popc(mw[j]);
    uint32_t inc = c;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        const uint32_t t = __shfl_up_sync(0xffffffffu, inc, d);
        if (lane >= d) inc += t;
    }
    const uint32_t lpre = inc - c;  // changed words of the block before this lane's mask words
    const uint32_t total = __shfl_sync(0xffffffffu, inc, 31);
    const bool imode = P.index_mode != 0;
    const bool sparse = total * W <= (imode ? kSpillBytes : kSpillMask);
    const uint32_t tmask = P.T - 1;

    if (sparse && total) {
        const size_t slot_bytes = imode ? 2 * kSpillBytes : kSpillMask;
        word_t* slot = reinterpret_cast<word_t*>(P.spill + I.b * slot_bytes);
        uint16_t* islot = reinterpret_cast<uint16_t*>(P.spill + I.b * slot_bytes + kSpillBytes);
        const uint32_t maxc = __reduce_max_sync(0xffffffffu, c);
        if (maxc <= 16u) {
            // few per lane: each lane packs its own words, 4 gathers in flight before the stores
            uint32_t rem[K];
#pragma unroll
            for (uint32_t j = 0; j < K; ++j) rem[j] = mw[j];
            uint32_t k = lpre;
            for (uint32_t r = 0; r < maxc; r += 4) {
                word_t v[4];
                uint32_t q[4];
#pragma unroll
                for (uint32_t u = 0; u < 4; ++u) {
                    q[u] = 0xffffffffu;
#pragma unroll
                    for (uint32_t j = 0; j < K; ++j)
                        if (q[u] == 0xffffffffu && rem[j]) {
                            q[u] = (lane * K + j) * 32 + __ffs(rem[j]) - 1;
                            rem[j] &= rem[j] - 1;
                        }
                    if (q[u] != 0xffffffffu) v[u] = ldg_cur(gcur + q[u]);
                }
#pragma unroll
                for (uint32_t u = 0; u < 4; ++u)
                    if (q[u] != 0xffffffffu) {
                        slot[k] = v[u];
                        if (imode) islot[k] = static_cast<uint16_t>((I.p0 + q[u]) & tmask);
                        ++k;
                    }
            }
        } else {
            // mask word by mask word: lane l takes word l of it (coalesced gathers); the K mask
            // words of a source lane are gathered with every load in flight before the stores
            const uint32_t lt = (1u << lane) - 1u;
            constexpr uint32_t kSrc = 1;  // source lanes per batch
            for (uint32_t src = 0; src < 32; src += kSrc) {
                word_t v[kSrc * K];
                uint32_t d[kSrc * K];
#pragma unroll
                for (uint32_t h = 0; h < kSrc; ++h) {
                    uint32_t o = __shfl_sync(0xffffffffu, lpre, src + h);
#pragma unroll
                    for (uint32_t j = 0; j < K; ++j) {
                        const uint32_t bb = __shfl_sync(0xffffffffu, mw[j], src + h);
                        d[h * K + j] = 0xffffffffu;
                        if ((bb >> lane) & 1u) {
                            const uint32_t q = ((src + h) * K + j) * 32 + lane;
                            v[h * K + j] = ldg_cur(gcur + q);
                            d[h * K + j] = o + __popc(bb & lt);
                            if (imode) islot[d[h * K + j]] = static_cast<uint16_t>((I.p0 + q) & tmask);
                        }
                        o += __popc(bb);
                    }
                }
#pragma unroll
                for (uint32_t x = 0; x < kSrc * K; ++x)
                    if (d[x] != 0xffffffffu) slot[d[x]] = v[x];
            }
        }
    }
    // index mode, dense block: its mask words go to the staging area (kernel B packs from them)
    if (imode && !sparse) {
        uint4* st = reinterpret_cast<uint4*>(P.mstage + I.b * kMaskStageWords + lane * K);
#pragma unroll
        for (uint32_t v = 0; v < K / 4; ++v) st[v] = make_uint4(mw[4 * v], mw[4 * v + 1], mw[4 * v + 2], mw[4 * v + 3]);
    }
    // record start of the chunk (prefetched by lane 0 at ticket time)
    if (lane == 0 && !(rs & 1ull)) rs = wait_rstart(P, I.chunk) | 1ull;
    rs = __shfl_sync(0xffffffffu, rs, 0) & ~1ull;

    const uint64_t fixed = imode ? index_idx_off(I.m, P.T) : record_fixed_bytes(I.m, P.T);
    if (rs + fixed > P.out_cap) {
        if (lane == 0) tc_set_err(P.err, TC_ERR_CAPACITY);
    } else {
        uint8_t* rec = P.out + rs;
        const uint64_t n_mask = cdiv(I.m, 32);
        uint32_t* gmask = reinterpret_cast<uint32_t*>(rec + kHdrBytes) + (I.p0 >> 5) + lane * K;
        uint32_t* gtoff = reinterpret_cast<uint32_t*>(rec + (imode ? index_toff_off() : kHdrBytes + pad16(4 * n_mask)));
        const bool full = (lane + 1) * K <= nmw;
        if (!imode && full) {
#pragma unroll
            for (uint32_t v = 0; v < K / 4; ++v)
                reinterpret_cast<uint4*>(gmask)[v] = make_uint4(mw[4 * v], mw[4 * v + 1], mw[4 * v + 2], mw[4 * v + 3]);
        }
        uint32_t pre = lpre;
#pragma unroll
        for (uint32_t j = 0; j < K; ++j) {
            const uint32_t p = I.p0 + (lane * K + j) * 32;
            if (p < I.m) {
                if (!imode && !full) rec_store<false, uint32_t>(P, gmask + j, mw[j]);
                if ((p & tmask) == 0) gtoff[p / P.T] = pre;  // kernel B adds the block prefix
            }
            pre += __popc(mw[j]);
        }
    }
    if (lane == 0) note_block(P, I.b, total, sparse);
    *rs_out = rs;
    return total;
}

// A warp claims kMaskinBatch consecutive blocks per ticket and counts each run of them that
// lies in one chunk with one chunk atomic: the ticket and the chunk counter are the two
// same-address atomics every block would otherwise return through (they serialised the kernel).
// Deadlock-free as in kernel A: a run is counted before the warp moves to the next chunk, and a
// block only ever waits for earlier chunks.
constexpr uint32_t kMaskinBatch = 4;

__device__ __noinline__ void count_run(const EncParams& P, const BlockInfo& R, uint32_t n, unsigned long long cnt,
                                       unsigned long long rs) {
    if (R.w == 4)
        count_blocks<4, false>(P, R, n, cnt, rs);
    else
        count_blocks<2, false>(P, R, n, cnt, rs);
}

__global__ void __launch_bounds__(kEncThreads, 3) encode_maskin_kernel(const __grid_constant__ EncParams P) {
    const int lane = threadIdx.x & 31;
    for (;;) {
        unsigned long long t = 0;
        if (lane == 0) t = atomicAdd(P.ticket, 1ull);
        const unsigned long long b0 = __shfl_sync(0xffffffffu, t, 0) * kMaskinBatch;
        if (b0 >= P.total_blocks) return;
        const unsigned long long b1 = b0 + kMaskinBatch < P.total_blocks ? b0 + kMaskinBatch : P.total_blocks;
        BlockInfo R{};  // the pending run: blocks of chunk R.chunk not yet counted
        uint32_t run_n = 0;
        unsigned long long run_cnt = 0, run_rs = 0;
        for (unsigned long long b = b0; b < b1; ++b) {
            const BlockInfo I = decode_block(P, b);
            if (run_n && I.chunk != R.chunk) {
                if (lane == 0) count_run(P, R, run_n, run_cnt, run_rs);
                run_n = 0;
                run_cnt = 0;
            }
            unsigned long long rs = 0;
            if (lane == 0) rs = I.chunk == 0 ? 1ull : ld_relaxed(&P.rstart[I.chunk]);  // value | 1 once published
            const uint32_t total = I.w == 4 ? maskin_block<4>(P, I, rs, lane, &run_rs)
                                            : maskin_block<2>(P, I, rs, lane, &run_rs);
            R = I;
            ++run_n;
            run_cnt += total;
        }
        if (lane == 0) count_run(P, R, run_n, run_cnt, run_rs);
    }
}

// ------------------------------------------------------------------ kernel P ------------
__global__ void __launch_bounds__(1024) encode_prefix_kernel(const __grid_constant__ EncParams P) {
    __shared__ unsigned long long s_carry;
    __shared__ unsigned long long s_warp[32];
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    for (int pass = 0; pass < 2; ++pass) {
        const unsigned long long* in = pass == 0 ? P.group_sum : P.chunk_acc;
        unsigned long long* out = pass == 0 ? P.gpre : P.cbase;
        const uint64_t n = pass == 0 ? P.n_groups : P.total_chunks;
        if (tid == 0) s_carry = 0;
        __syncthreads();
        for (uint64_t base = 0; base < n; base += 1024) {
            const uint64_t i = base + tid;
            const unsigned long long v = i < n ? (pass == 0 ? in[i] : in[i] & kAccCountMask) : 0ull;
            unsigned long long x = v;
#pragma unroll
            for (int d = 1; d < 32; d <<= 1) {
                const unsigned long long y = __shfl_up_sync(0xffffffffu, x, d);
                if (lane >= d) x += y;
            }
            if (lane == 31) s_warp[wid] = x;
            __syncthreads();
            unsigned long long wp = 0, tot = 0;
            for (int k = 0; k < 32; ++k) {
                const unsigned long long t = s_warp[k];
                wp += k < wid ? t : 0ull;
                tot += t;
            }
            const unsigned long long carry = s_carry;
            if (i < n) out[i] = carry + wp + x - v;
            __syncthreads();
            if (tid == 0) s_carry = carry + tot;
            __syncthreads();
        }
    }
}

// ------------------------------------------------------------------ kernel B ------------

__device__ __forceinline__ uint32_t word4(const uint4& o, int i) {  // i: compile-time after unrolling
    return i == 0 ? o.x : i == 1 ? o.y : i == 2 ? o.z : o.w;
}

// Dense block (more changed words than its spill slot holds): re-read its mask words from the
// record and the changed words from cur, pack them in index order (a warp per block).
template <int W, bool PEER>
__device__ __forceinline__ void emit_dense(const EncParams& P, const BlockInfo& I, uint32_t info,
                                           unsigned long long prefix, int lane, uint8_t* ring) {
    using word_t = typename Word<W>::T;
    const bool imode = P.index_mode != 0;
    const unsigned long long rs = ld_relaxed(&P.rstart[I.chunk]) & ~1ull;
    uint8_t* rec = P.out + rs;
    // mask words: from the record (mask mode) or the staging area (index mode, block-relative)
    const uint32_t* gmask = imode ? P.mstage + I.b * kMaskStageWords - (I.p0 >> 5)
                                  : reinterpret_cast<const uint32_t*>(rec + kHdrBytes);
    const uint64_t ccount = P.chunk_acc[I.chunk] & kAccCountMask;
    word_t* gval = reinterpret_cast<word_t*>(rec + (imode ? index_val_off(I.m, P.T, ccount)
                                                          : record_fixed_bytes(I.m, P.T))) + prefix;
    uint16_t* gidx = reinterpret_cast<uint16_t*>(rec + index_idx_off(I.m, P.T)) + prefix;
    const uint32_t tmask = P.T - 1;
    const EncSeg& S = P.seg[I.seg];
    const word_t* gcur = reinterpret_cast<const word_t*>(S.cur) + I.chunk_off + I.p0;
    const uint32_t nmw = (I.nb + 31) / 32;
    (void)info;
    // Vectorized (round 2; r2 ncu: the mask-word-at-a-time loop issued on 75 % of cycles, ~6 300
    // warp instructions per 4096-word block): lane l takes the 16-byte vector l of a group of 32
    // vectors (its VW = 4 | 8 words, VW bits of one mask word), a warp scan of the lanes' popcounts
    // gives each lane its first output slot, and it stores its changed words in order; two groups
    // per iteration keep two vector loads in flight per lane.
    constexpr uint32_t VW = 16 / W;    // words per 16-byte vector
    constexpr uint32_t LPM = 32 / VW;  // lanes per mask word
    constexpr uint32_t MPG = 32 / LPM; // mask words per group of 32 vectors
    const uint4* gcur4 = reinterpret_cast<const uint4*>(gcur);
    uint32_t base = 0;
    if (!imode && ring) {
        // mask records: the packed words go through a 2 KB warp-private ring in shared memory
        // indexed by their DESTINATION address mod 2 KB, and leave it as 16-byte aligned vectors
        // (the run's first and last vectors in 2-byte pieces: their other bytes are the
        // neighbouring blocks').  r2 ncu: the word-per-lane stores made this loop store-issue bound.
        const uintptr_t g0a = reinterpret_cast<uintptr_t>(gval);  // run start (any W alignment)
        uintptr_t done = g0a;                                       // written up to here
        auto flush = [&](uintptr_t upto, bool last) {
            // the vectors [done & ~15, upto) (last: including upto's partial vector)
            const uintptr_t v0 = done & ~uintptr_t(15);
            const uintptr_t v1 = last ? ((upto + 15) & ~uintptr_t(15)) : (upto & ~uintptr_t(15));
            for (uintptr_t va = v0 + 16 * static_cast<uintptr_t>(lane); va < v1; va += 512) {
                const uint4 o = *reinterpret_cast<const uint4*>(ring + (va & 2047));
                uint8_t* dstv = reinterpret_cast<uint8_t*>(va);
                if (va >= done && va + 16 <= upto) {
                    rec_store<PEER, uint4>(P, reinterpret_cast<uint4*>(dstv), o);
                } else {
#pragma unroll
                    for (int e = 0; e < 8; ++e) {
                        const uintptr_t x = va + 2 * e;
                        if (x >= done && x < upto)
                            rec_store<PEER, uint16_t>(P, reinterpret_cast<uint16_t*>(x),
                                                      static_cast<uint16_t>(word4(o, e >> 1) >> (16 * (e & 1))));
                    }
                }
            }
            done = v1 < upto ? v1 : upto;
        };
        for (uint32_t g0 = 0; g0 < nmw; g0 += 2 * MPG) {
            uint32_t bits[2];
            uint4 vec[2];
#pragma unroll
            for (int u = 0; u < 2; ++u) {
                const uint32_t mwi = g0 + u * MPG + lane / LPM;
                const uint32_t mw = mwi < nmw ? gmask[(I.p0 >> 5) + mwi] : 0u;
                bits[u] = (mw >> ((lane % LPM) * VW)) & ((1u << VW) - 1u);
                if (bits[u]) vec[u] = __ldg(gcur4 + (g0 + u * MPG) * LPM + lane);
            }
#pragma unroll
            for (int u = 0; u < 2; ++u) {
                const uint32_t c = __popc(bits[u]);
                uint32_t inc = c;
#pragma unroll
                for (int d = 1; d < 32; d <<= 1) {
                    const uint32_t t = __shfl_up_sync(0xffffffffu, inc, d);
                    if (lane >= d) inc += t;
                }
                uint32_t o = base + inc - c;
                base += __shfl_sync(0xffffffffu, inc, 31);
                if (bits[u]) {
                    const word_t* vw = reinterpret_cast<const word_t*>(&vec[u]);
#pragma unroll
                    for (uint32_t k = 0; k < VW; ++k)
                        if ((bits[u] >> k) & 1u) {
                            *reinterpret_cast<word_t*>(ring + ((g0a + static_cast<uintptr_t>(o) * W) & 2047)) = vw[k];
                            ++o;
                        }
                }
            }
            __syncwarp();
            flush(g0a + static_cast<uintptr_t>(base) * W, false);
            __syncwarp();
        }
        flush(g0a + static_cast<uintptr_t>(base) * W, true);
        __syncwarp();
        return;
    }
    for (uint32_t g0 = 0; g0 < nmw; g0 += 2 * MPG) {
        uint32_t bits[2];
        uint4 vec[2];
#pragma unroll
        for (int u = 0; u < 2; ++u) {
            const uint32_t mwi = g0 + u * MPG + lane / LPM;
            const uint32_t mw = mwi < nmw ? gmask[(I.p0 >> 5) + mwi] : 0u;
            bits[u] = (mw >> ((lane % LPM) * VW)) & ((1u << VW) - 1u);
            // a vector holding a changed word lies inside the block's 16-byte aligned words
            if (bits[u]) vec[u] = __ldg(gcur4 + (g0 + u * MPG) * LPM + lane);
        }
#pragma unroll
        for (int u = 0; u < 2; ++u) {
            const uint32_t c = __popc(bits[u]);
            uint32_t inc = c;
#pragma unroll
            for (int d = 1; d < 32; d <<= 1) {
                const uint32_t t = __shfl_up_sync(0xffffffffu, inc, d);
                if (lane >= d) inc += t;
            }
            uint32_t o = base + inc - c;
            base += __shfl_sync(0xffffffffu, inc, 31);
            if (bits[u]) {
                const word_t* vw = reinterpret_cast<const word_t*>(&vec[u]);
                const uint32_t w0 = (g0 + u * MPG) * 32 + lane * VW;  // block-relative first word
#pragma unroll
                for (uint32_t k = 0; k < VW; ++k)
                    if ((bits[u] >> k) & 1u) {
                        if (imode) rec_store<PEER, uint16_t>(P, gidx + o, static_cast<uint16_t>((I.p0 + w0 + k) & tmask));
                        rec_store<PEER, word_t>(P, gval + o, vw[k]);
                        ++o;
                    }
            }
        }
    }
}

// Bytes [0, nbytes) of a 16-byte aligned spill run -> the record at `dst` (any 2-byte alignment k),
// with 16-byte loads and 16-byte stores: in the 16-byte aligned window starting at dst - k, vector
// u holds source bytes [16u - k, 16u - k + 16) = the tail of source vector u - 1 and the head of
// vector u, joined by funnel shifts (source vector u - 1 comes from the neighbouring lane).  The
// window's first and last vectors are stored in 2-byte pieces (the bytes around the run belong to
// other blocks).  Four vectors per lane in flight.  (Kernel B copied spilled runs with one 2- or
// 4-byte word per lane: 64-128 bytes per warp instruction, long-scoreboard bound at 22 % issue,
// f = 10 %, ncu rd4h.)
__device__ __forceinline__ uint4 funnel16(uint4 p, uint4 c, uint32_t s) {
    const uint32_t r = (s & 3u) * 8u;
    uint32_t w0, w1, w2, w3, w4;
    switch (s >> 2) {
        case 0: w0 = p.x; w1 = p.y; w2 = p.z; w3 = p.w; w4 = c.x; break;
        case 1: w0 = p.y; w1 = p.z; w2 = p.w; w3 = c.x; w4 = c.y; break;
        case 2: w0 = p.z; w1 = p.w; w2 = c.x; w3 = c.y; w4 = c.z; break;
        default: w0 = p.w; w1 = c.x; w2 = c.y; w3 = c.z; w4 = c.w; break;
    }
    return make_uint4(__funnelshift_r(w0, w1, r), __funnelshift_r(w1, w2, r), __funnelshift_r(w2, w3, r),
                      __funnelshift_r(w3, w4, r));
}

// window vector u (bytes [16u, 16u + 16) from D) of a run occupying window bytes [k, k + nbytes)
template <bool PEER>
__device__ __forceinline__ void store_window_vec(const EncParams& P, uint8_t* D, uint32_t u, uint4 o, uint32_t k,
                                                 uint32_t nbytes) {
    const uint32_t lo = 16 * u;
    if (lo >= k && lo + 16 <= k + nbytes) {
        rec_store<PEER, uint4>(P, reinterpret_cast<uint4*>(D) + u, o);
        return;
    }
#pragma unroll
    for (int e = 0; e < 8; ++e) {
        const uint32_t x = lo + 2 * e;
        if (x >= k && x < k + nbytes)
            rec_store<PEER, uint16_t>(P, reinterpret_cast<uint16_t*>(D + x), static_cast<uint16_t>(word4(o, e >> 1) >> (16 * (e & 1))));
    }
}

template <bool PEER>
__device__ __forceinline__ void copy_vec(const EncParams& P, uint8_t* dst, const uint8_t* src, uint32_t nbytes,
                                         int lane) {
    if (nbytes == 0) return;
    const uint32_t k = static_cast<uint32_t>(reinterpret_cast<uintptr_t>(dst) & 15u);
    uint8_t* D = dst - k;
    const uint32_t nd = (k + nbytes + 15) >> 4;  // window vectors
    const uint32_t ns = (nbytes + 15) >> 4;      // source vectors (the slot is 16-byte padded)
    const uint4* S = reinterpret_cast<const uint4*>(src);
    const uint32_t sh = 16 - k;
    const uint4 z = make_uint4(0, 0, 0, 0);
    uint4 carry = z;  // source vector (first vector of this pass) - 1, for lane 0
    for (uint32_t u0 = 0; u0 < nd; u0 += 128) {
        uint4 c[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const uint32_t u = u0 + 32 * q + lane;
            c[q] = u < ns ? __ldg(S + u) : z;
        }
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const uint32_t u = u0 + 32 * q + lane;
            uint4 pv;
            pv.x = __shfl_up_sync(0xffffffffu, c[q].x, 1);
            pv.y = __shfl_up_sync(0xffffffffu, c[q].y, 1);
            pv.z = __shfl_up_sync(0xffffffffu, c[q].z, 1);
            pv.w = __shfl_up_sync(0xffffffffu, c[q].w, 1);
            if (lane == 0) pv = carry;
            carry.x = __shfl_sync(0xffffffffu, c[q].x, 31);
            carry.y = __shfl_sync(0xffffffffu, c[q].y, 31);
            carry.z = __shfl_sync(0xffffffffu, c[q].z, 31);
            carry.w = __shfl_sync(0xffffffffu, c[q].w, 31);
            if (u < nd) store_window_vec<PEER>(P, D, u, k ? funnel16(pv, c[q], sh) : c[q], k, nbytes);
            if (u0 + 32 * q + 32 >= nd) break;  // (warp-uniform) the run ends in this group
        }
    }
}

template <bool PEER>
__global__ void __launch_bounds__(kEncThreads, 4) encode_emit_kernel(const __grid_constant__ EncParams P) {
    __shared__ uint32_t s_warp[kWarps];
    __shared__ __align__(16) uint8_t s_ring[kWarps][2048];  // dense blocks: per-warp output ring
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    const unsigned long long g = blockIdx.x;
    const unsigned long long b = g * kEmitGroup + tid;
    const bool valid = b < P.total_blocks;
    const uint32_t info = valid ? P.info[b] : 0u;
    const uint32_t c = info & ~kDenseFlag;
    uint32_t inc = c;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        const uint32_t t = __shfl_up_sync(0xffffffffu, inc, d);
        if (lane >= d) inc += t;
    }
    if (lane == 31) s_warp[wid] = inc;
    __syncthreads();
    uint32_t wp = 0;
#pragma unroll
    for (int k = 0; k < static_cast<int>(kWarps); ++k) wp += k < wid ? s_warp[k] : 0u;

    // ---- per block (one thread each): in-chunk prefix, tile_off entries, destination ----
    const bool imode = P.index_mode != 0;
    uint8_t* dst = nullptr;
    uint8_t* idst = nullptr;
    const uint8_t* src = nullptr;
    uint32_t w = 4;
    bool dense = false, fits = true;
    if (valid) {
        const BlockInfo I = decode_block(P, b);
        w = I.w;
        const unsigned long long prefix = P.gpre[g] + wp + inc - c - P.cbase[I.chunk];
        const unsigned long long rs = ld_relaxed(&P.rstart[I.chunk]) & ~1ull;
        const uint64_t ccount = P.chunk_acc[I.chunk] & kAccCountMask;
        fits = rs + (imode ? record_bytes_index(I.m, P.T, I.w, ccount) : record_bytes(I.m, P.T, I.w, ccount)) <=
               P.out_cap;  // else kernel A flagged TC_ERR_CAPACITY: nothing of this record is written
        uint8_t* rec = P.out + rs;
        const uint64_t n_mask = cdiv(I.m, 32);
        uint32_t* gtoff = reinterpret_cast<uint32_t*>(rec + (imode ? index_toff_off() : kHdrBytes + pad16(4 * n_mask)));
        const uint32_t pr = static_cast<uint32_t>(prefix);
        const uint32_t B = I.w == 4 ? kEncBlockWords4 : kEncBlockWords2;
        if (I.nb && fits) {  // kernel A wrote the tile_off entries of the block block-relative
            if (P.T >= B) {
                if ((I.p0 & (P.T - 1)) == 0) rec_store<PEER, uint32_t>(P, gtoff + I.p0 / P.T, gtoff[I.p0 / P.T] + pr);
            } else {
                const uint32_t n_t = (I.nb + P.T - 1) / P.T;
                for (uint32_t t = 0; t < n_t; ++t) rec_store<PEER, uint32_t>(P, gtoff + I.p0 / P.T + t, gtoff[I.p0 / P.T + t] + pr);
            }
        }
        if (imode) {
            dst = rec + index_val_off(I.m, P.T, ccount) + prefix * I.w;
            idst = rec + index_idx_off(I.m, P.T) + prefix * 2;
            src = P.spill + b * (2 * kSpillBytes);
        } else {
            dst = rec + record_fixed_bytes(I.m, P.T) + prefix * I.w;
            src = P.spill + b * kSpillMask;
        }
        dense = (info & kDenseFlag) != 0 && c != 0 && fits;
    }

    // ---- sparse blocks of this warp: packed words spill slot -> record.  Runs of <= 64 words: 4
    //      blocks per batch, a word per lane; longer runs: whole, in 16-byte vectors (copy_vec) ----
    uint32_t todo = __ballot_sync(0xffffffffu, valid && fits && !dense && c != 0 && c <= 64);
    uint32_t longr = __ballot_sync(0xffffffffu, valid && fits && !dense && c > 64);
    while (longr) {
        const int sl = __ffs(longr) - 1;
        longr &= longr - 1;
        const uint32_t cn = __shfl_sync(0xffffffffu, c, sl);
        const uint32_t wq = __shfl_sync(0xffffffffu, w, sl);
        uint8_t* dq = reinterpret_cast<uint8_t*>(__shfl_sync(0xffffffffu, reinterpret_cast<unsigned long long>(dst), sl));
        const uint8_t* sq = reinterpret_cast<const uint8_t*>(__shfl_sync(0xffffffffu, reinterpret_cast<unsigned long long>(src), sl));
        copy_vec<PEER>(P, dq, sq, cn * wq, lane);
        if (imode) {
            uint8_t* iq = reinterpret_cast<uint8_t*>(__shfl_sync(0xffffffffu, reinterpret_cast<unsigned long long>(idst), sl));
            copy_vec<PEER>(P, iq, sq + kSpillBytes, cn * 2, lane);
        }
    }
    while (todo) {
        int bl[4];
        uint32_t cn[4], wq[4];
        uint8_t* dq[4];
        const uint8_t* sq[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            bl[q] = todo ? __ffs(todo) - 1 : -1;
            if (todo) todo &= todo - 1;
            const int sl = bl[q] < 0 ? 0 : bl[q];
            cn[q] = bl[q] < 0 ? 0u : __shfl_sync(0xffffffffu, c, sl);
            wq[q] = __shfl_sync(0xffffffffu, w, sl);
            dq[q] = reinterpret_cast<uint8_t*>(__shfl_sync(0xffffffffu, reinterpret_cast<unsigned long long>(dst), sl));
            sq[q] = reinterpret_cast<const uint8_t*>(__shfl_sync(0xffffffffu, reinterpret_cast<unsigned long long>(src), sl));
        }
        uint32_t v[4][2];
#pragma unroll
        for (int q = 0; q < 4; ++q)
#pragma unroll
            for (int k = 0; k < 2; ++k) {
                const uint32_t i = lane + 32 * k;
                v[q][k] = 0;
                if (i < cn[q])
                    v[q][k] = wq[q] == 4 ? __ldg(reinterpret_cast<const uint32_t*>(sq[q]) + i)
                                         : __ldg(reinterpret_cast<const unsigned short*>(sq[q]) + i);
            }
#pragma unroll
        for (int q = 0; q < 4; ++q)
#pragma unroll
            for (int k = 0; k < 2; ++k) {
                const uint32_t i = lane + 32 * k;
                if (i < cn[q]) {
                    if (wq[q] == 4)
                        rec_store<PEER, uint32_t>(P, reinterpret_cast<uint32_t*>(dq[q]) + i, v[q][k]);
                    else
                        rec_store<PEER, uint16_t>(P, reinterpret_cast<uint16_t*>(dq[q]) + i, static_cast<uint16_t>(v[q][k]));
                }
            }
        if (imode) {  // the u16 in-tile positions, same batching
            uint16_t iv[4][2];
            uint8_t* iq[4];
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const int sl = bl[q] < 0 ? 0 : bl[q];
                iq[q] = reinterpret_cast<uint8_t*>(__shfl_sync(0xffffffffu, reinterpret_cast<unsigned long long>(idst), sl));
#pragma unroll
                for (int k = 0; k < 2; ++k) {
                    const uint32_t i = lane + 32 * k;
                    iv[q][k] = i < cn[q] ? static_cast<uint16_t>(__ldg(reinterpret_cast<const unsigned short*>(sq[q] + kSpillBytes) + i)) : 0;
                }
            }
#pragma unroll
            for (int q = 0; q < 4; ++q)
#pragma unroll
                for (int k = 0; k < 2; ++k) {
                    const uint32_t i = lane + 32 * k;
                    if (i < cn[q]) rec_store<PEER, uint16_t>(P, reinterpret_cast<uint16_t*>(iq[q]) + i, iv[q][k]);
                }
        }
    }

    // ---- dense blocks: re-read mask + cur, pack in index order (a warp per block) ----
    uint32_t dn = __ballot_sync(0xffffffffu, dense);
    while (dn) {
        const int t = __ffs(dn) - 1;
        dn &= dn - 1;
        const unsigned long long bb = g * kEmitGroup + wid * 32 + t;
        const BlockInfo I = decode_block(P, bb);
        const unsigned long long prefix =
            P.gpre[g] + __shfl_sync(0xffffffffu, wp + inc - c, t) - P.cbase[I.chunk];
        const uint32_t inf = __shfl_sync(0xffffffffu, info, t);
        if (I.w == 4)
            emit_dense<4, PEER>(P, I, inf, prefix, lane, s_ring[wid]);
        else
            emit_dense<2, PEER>(P, I, inf, prefix, lane, s_ring[wid]);
    }
    // fused Tier-2 emit: every CTA's peer stores are fenced at system scope; the last CTA publishes
    // {bytes, version} into the neighbour's mailbox (a refused record: bytes = UINT64_MAX)
    if (PEER) {
        __threadfence_system();
        __syncthreads();
        if (tid == 0) {
            const unsigned prev = atomicAdd(P.peer_counter, 1u);
            if (prev == gridDim.x - 1) {
                *P.peer_counter = 0u;  // ready for the next push on this ctx (stream-ordered)
                __threadfence_system();
                const unsigned long long nb = *reinterpret_cast<const volatile unsigned long long*>(P.out_bytes);
                const bool ok = nb <= P.peer_cap && *reinterpret_cast<const volatile unsigned int*>(P.err) == 0u;
                asm volatile("st.relaxed.sys.global.u64 [%0], %1;" ::"l"(P.peer_mail), "l"(ok ? nb : ~0ull) : "memory");
                asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(P.peer_mail + 1),
                             "l"(static_cast<unsigned long long>(P.peer_version)) : "memory");
            }
        }
    }
}

}  // namespace

constexpr size_t kEncDynSmem = 2 * 16384 + 1024;  // ref | cur | mask words

cudaError_t launch_encode(const EncParams& p, cudaStream_t s) {
    static bool attr_set[TC_MAX_DEVICES] = {};  // a function attribute is per device
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev < 0 || dev >= TC_MAX_DEVICES || !attr_set[dev]) {
        cudaFuncSetAttribute(encode_mask_kernel<false>, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
        cudaFuncSetAttribute(encode_mask_kernel<true>, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
        if (dev >= 0 && dev < TC_MAX_DEVICES) attr_set[dev] = true;
    }
    if (p.total_blocks == 0) return cudaSuccess;
    if (p.index_mode == kFormatFull) {  // full records: one streaming pass (kernel F)
        if (p.peer_out)
            encode_full_kernel<true><<<static_cast<unsigned>(p.total_blocks), kEncThreads, 0, s>>>(p);
        else
            encode_full_kernel<false><<<static_cast<unsigned>(p.total_blocks), kEncThreads, 0, s>>>(p);
        return cudaGetLastError();
    }
    if (p.seg[0].mask_in) {
        // persistent warps: as many CTAs as fit, never more than one warp per block
        static int per_sm = 0;
        if (!per_sm && cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, encode_maskin_kernel, kEncThreads, 0) !=
                           cudaSuccess)
            return cudaGetLastError();
        int sms = 0;
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        const uint64_t want = (p.total_blocks + kWarps * kMaskinBatch - 1) / (kWarps * kMaskinBatch);
        const uint64_t cap = static_cast<uint64_t>(sms) * (per_sm > 0 ? per_sm : 1);
        encode_maskin_kernel<<<static_cast<unsigned>(want < cap ? want : cap), kEncThreads, 0, s>>>(p);
    } else {
        if (p.peer_out)
            encode_mask_kernel<true><<<static_cast<unsigned>(p.total_blocks), kEncThreads, kEncDynSmem, s>>>(p);
        else
            encode_mask_kernel<false><<<static_cast<unsigned>(p.total_blocks), kEncThreads, kEncDynSmem, s>>>(p);
    }
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    encode_prefix_kernel<<<1, 1024, 0, s>>>(p);
    e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    if (p.peer_out)
        encode_emit_kernel<true><<<static_cast<unsigned>(p.n_groups), kEncThreads, 0, s>>>(p);
    else
        encode_emit_kernel<false><<<static_cast<unsigned>(p.n_groups), kEncThreads, 0, s>>>(p);
    return cudaGetLastError();
}

}  // namespace tc
