// tc_encode.cu — single-pass differential-checkpoint encoder for sm_100a.
//
// What it computes: for every chunk of every segment,
// the mask of changed words (unsigned bitwise compare, reading R5), the in-chunk exclusive
// counts at every tile start (tile_off), the packed new words (values) and the record header;
// optionally ref[i] <- cur[i] for changed words.  The paper's own compaction is "a single
// fused pass to extract and compact surviving entries" (§3.2) — this kernel is
// that single pass for the lossless word diff.
//
// B200 design:
//   * one CTA = one scan block of B words (B = 4096 fp32 / 8192 16-bit words = 16 KB per
//     operand); a CTA takes a dynamic ticket so blocks are processed in stream order, which
//     makes the decoupled look-back deadlock-free;
//   * ref and cur of the block are staged to shared memory with two 1-D TMA bulk copies
//     (cp.async.bulk ... mbarrier::complete_tx) — no register staging, 6 CTAs/SM keep
//     ~190 KB of HBM reads in flight per SM;
//   * lane l of a warp tests word 32*q + l, so __ballot_sync IS the mask word (LSB-first,
//     reading R6) and __popc gives the counts;
//   * in-chunk prefix: decoupled look-back over 64-bit status words {2-bit flag | count}
//     (warp-wide 32-predecessor windows); chunk-level record start: a chain of "record
//     start" words published by each chunk's last block (value | 1);
//   * values are written compacted in index order (consecutive lanes -> consecutive
//     addresses); mask words are written coalesced from shared memory.
#include <cuda_runtime.h>

#include "tc_internal.h"

namespace tc {

namespace {

constexpr unsigned long long kFlagAgg = 1ull << 62;
constexpr unsigned long long kFlagInc = 2ull << 62;
constexpr uint32_t kSpinLimit = 1u << 26;  // watchdog: a bug must not hang the GPU

__device__ __forceinline__ unsigned long long ld_relaxed(const unsigned long long* p) {
    unsigned long long v;
    asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_relaxed(unsigned long long* p, unsigned long long v) {
    asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ uint32_t smem_addr(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(bar)), "r"(count) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_addr(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait_parity(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n"
        ".reg .pred P1;\n"
        "TC_WAIT:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
        "@!P1 bra TC_WAIT;\n"
        "}\n" ::"r"(smem_addr(bar)),
        "r"(parity)
        : "memory");
}
// 1-D TMA bulk copy global -> shared, completion counted on the mbarrier (bytes % 16 == 0).
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_addr(dst)),
        "l"(src), "r"(bytes), "r"(smem_addr(bar))
        : "memory");
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

// Warp-cooperative decoupled look-back within one chunk.  Block b's predecessors in the
// same chunk are b-1 ... first (the chunk's first block, which always publishes INCLUSIVE).
__device__ __forceinline__ uint32_t lookback(const EncParams& P, uint64_t b, uint64_t first, int lane) {
    uint32_t excl = 0;
    int64_t j = static_cast<int64_t>(b) - 1;
    uint32_t spins = 0;
    while (true) {
        const int64_t idx = j - lane;
        const unsigned long long sv = idx >= static_cast<int64_t>(first) ? ld_relaxed(&P.status[idx]) : kFlagInc;
        const uint32_t flag = static_cast<uint32_t>(sv >> 62);
        const uint32_t incl = __ballot_sync(0xffffffffu, flag == 2);
        const uint32_t empty = __ballot_sync(0xffffffffu, flag == 0);
        const uint32_t upto = incl ? (((incl & (0u - incl)) << 1) - 1u) : 0xffffffffu;
        if (empty & upto) {
            if (++spins > kSpinLimit) {
                if (lane == 0) tc_set_err(P.err, TC_ERR_INTERNAL);
                return excl;
            }
            __nanosleep(20);
            continue;
        }
        uint32_t v = ((upto >> lane) & 1u) ? static_cast<uint32_t>(sv) : 0u;
#pragma unroll
        for (int d = 16; d; d >>= 1) v += __shfl_xor_sync(0xffffffffu, v, d);
        excl += v;
        if (incl) return excl;
        j -= 32;
    }
}

__device__ __forceinline__ unsigned long long wait_rstart(const EncParams& P, uint64_t c) {
    if (c == 0) return 0;
    uint32_t spins = 0;
    unsigned long long v;
    while (((v = ld_relaxed(&P.rstart[c])) & 1ull) == 0) {
        if (++spins > kSpinLimit) {
            tc_set_err(P.err, TC_ERR_INTERNAL);
            return 0;
        }
        __nanosleep(32);
    }
    return v & ~1ull;
}

struct BlockInfo {
    uint64_t b;          // global block index (= ticket)
    uint64_t first;      // global index of the chunk's first block
    uint64_t chunk;      // global chunk index
    uint64_t chunk_off;  // word offset of the chunk in its segment
    uint32_t m;          // words in the chunk
    uint32_t k;          // block index within the chunk
    uint32_t p0;         // chunk-relative first word of the block
    uint32_t nb;         // words in this block
    uint32_t seg;
    bool last;           // last block of its chunk
};

template <int W>
__device__ __forceinline__ void encode_block(const EncParams& P, const BlockInfo& I, uint8_t* tile,
                                             uint32_t* s_bal, uint32_t* s_warp, uint64_t* s_bar,
                                             uint32_t* s_excl, unsigned long long* s_rs) {
    using word_t = typename Word<W>::T;
    constexpr uint32_t B = Word<W>::kBlock;
    constexpr uint32_t kWarps = kEncThreads / 32;
    constexpr uint32_t MPW = B / 32 / kWarps;  // mask words per warp (16 | 32)
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    const EncSeg& S = P.seg[I.seg];

    word_t* sref = reinterpret_cast<word_t*>(tile);
    word_t* scur = sref + B;
    word_t* gref = reinterpret_cast<word_t*>(S.ref) + I.chunk_off + I.p0;
    const word_t* gcur = reinterpret_cast<const word_t*>(S.cur) + I.chunk_off + I.p0;

    // ---- stage ref / cur of the block into shared memory (TMA bulk + tail words) ----
    const uint32_t bytes = I.nb * W;
    const uint32_t bulk = bytes & ~15u;
    if (tid == 0) {
        if (bulk) {
            mbar_arrive_expect_tx(s_bar, 2 * bulk);
            bulk_g2s(sref, gref, bulk, s_bar);
            bulk_g2s(scur, gcur, bulk, s_bar);
        } else {
            mbar_arrive(s_bar);
        }
    }
    const uint32_t tail = (bytes - bulk) / W;
    if (static_cast<uint32_t>(tid) < tail) {
        const uint32_t i = bulk / W + tid;
        sref[i] = gref[i];
        scur[i] = gcur[i];
    }
    mbar_wait_parity(s_bar, 0);
    __syncthreads();

    // ---- pass 1: compare, ballot -> mask word, popc; fused ref advance ----
    uint32_t cnt = 0;
    const bool adv = P.advance_ref != 0;
#pragma unroll 4
    for (uint32_t q = 0; q < MPW; ++q) {
        const uint32_t mw = wid * MPW + q;
        const uint32_t i = mw * 32 + lane;
        const word_t a = sref[i];
        const word_t v = scur[i];
        const bool ch = (i < I.nb) && (a != v);
        const uint32_t bal = __ballot_sync(0xffffffffu, ch);
        if (lane == 0) s_bal[mw] = bal;
        if (adv && ch) gref[i] = v;
        cnt += __popc(bal);
    }
    if (lane == 0) s_warp[wid] = cnt;
    __syncthreads();

    // ---- block total, warp offsets, look-back, record start (warp 0) ----
    if (wid == 0) {
        const uint32_t wc = lane < static_cast<int>(kWarps) ? s_warp[lane] : 0u;
        uint32_t inc = wc;
#pragma unroll
        for (int d = 1; d < static_cast<int>(kWarps); d <<= 1) {
            const uint32_t t = __shfl_up_sync(0xffffffffu, inc, d);
            if (lane >= d) inc += t;
        }
        const uint32_t total = __shfl_sync(0xffffffffu, inc, kWarps - 1);
        if (lane < static_cast<int>(kWarps)) s_warp[kWarps + lane] = inc - wc;  // warp exclusive offsets
        uint32_t excl = 0;
        if (I.k == 0) {
            if (lane == 0) st_relaxed(&P.status[I.b], kFlagInc | total);
        } else {
            if (lane == 0) st_relaxed(&P.status[I.b], kFlagAgg | total);
            excl = lookback(P, I.b, I.first, lane);
            if (lane == 0) st_relaxed(&P.status[I.b], kFlagInc | static_cast<unsigned long long>(excl + total));
        }
        if (lane == 0) {
            const unsigned long long rs = wait_rstart(P, I.chunk);
            if (I.last) {
                const uint64_t count = static_cast<uint64_t>(excl) + total;
                const uint64_t n_mask = cdiv(I.m, 32);
                const uint64_t n_tiles = cdiv(I.m, P.T);
                const uint64_t rec_total = record_bytes(I.m, P.T, W, count);
                uint8_t* rec = P.out + rs;
                uint64_t* h = reinterpret_cast<uint64_t*>(rec);
                h[0] = 0x31444354ull /* "TCD1" */ | (1ull << 32) | (static_cast<uint64_t>(W) << 48) | (1ull << 56);
                h[1] = static_cast<uint64_t>(P.T) | (static_cast<uint64_t>(I.seg) << 32);
                h[2] = I.chunk_off;
                h[3] = I.m;
                h[4] = count;
                h[5] = P.version;
                h[6] = P.ref_version;
                h[7] = rec_total;
                uint32_t* gmask = reinterpret_cast<uint32_t*>(rec + kHdrBytes);
                for (uint64_t x = n_mask; x < pad16(4 * n_mask) / 4; ++x) gmask[x] = 0;
                uint32_t* gtoff = reinterpret_cast<uint32_t*>(rec + kHdrBytes + pad16(4 * n_mask));
                gtoff[n_tiles] = static_cast<uint32_t>(count);
                for (uint64_t x = n_tiles + 1; x < pad16(4 * (n_tiles + 1)) / 4; ++x) gtoff[x] = 0;
                word_t* gval = reinterpret_cast<word_t*>(rec + record_fixed_bytes(I.m, P.T));
                for (uint64_t x = count; x < pad16(W * count) / W; ++x) gval[x] = 0;
                const unsigned long long next = rs + rec_total;
                st_relaxed(&P.rstart[I.chunk + 1], next | 1ull);
                if (I.chunk + 1 == P.total_chunks) *P.out_bytes = next;
            }
            *s_excl = excl;
            *s_rs = rs;
        }
    }
    __syncthreads();

    // ---- pass 2: tile_off entries, compacted values, mask words ----
    const unsigned long long rs = *s_rs;
    uint8_t* rec = P.out + rs;
    const uint64_t n_mask = cdiv(I.m, 32);
    uint32_t* gmask = reinterpret_cast<uint32_t*>(rec + kHdrBytes);
    uint32_t* gtoff = reinterpret_cast<uint32_t*>(rec + kHdrBytes + pad16(4 * n_mask));
    word_t* gval = reinterpret_cast<word_t*>(rec + record_fixed_bytes(I.m, P.T));
    uint32_t running = *s_excl + s_warp[kWarps + wid];
    const uint32_t lt = (1u << lane) - 1u;
    for (uint32_t q = 0; q < MPW; ++q) {
        const uint32_t mw = wid * MPW + q;
        const uint32_t p = I.p0 + mw * 32;
        if (p >= I.m) break;
        const uint32_t bal = s_bal[mw];
        if (lane == 0 && (p & (P.T - 1)) == 0) gtoff[p / P.T] = running;
        if (bal) {
            if ((bal >> lane) & 1u) gval[running + __popc(bal & lt)] = scur[mw * 32 + lane];
            running += __popc(bal);
        }
    }
    const uint32_t nmw = static_cast<uint32_t>(cdiv(I.nb, 32));
    for (uint32_t t = tid; t < nmw; t += kEncThreads) gmask[I.p0 / 32 + t] = s_bal[t];
}

__global__ void __launch_bounds__(kEncThreads, 6) encode_kernel(const __grid_constant__ EncParams P) {
    extern __shared__ __align__(128) uint8_t tile[];
    __shared__ uint32_t s_bal[kEncBlockWords2 / 32];
    __shared__ uint32_t s_warp[2 * (kEncThreads / 32)];
    __shared__ __align__(8) uint64_t s_bar;
    __shared__ unsigned long long s_b;
    __shared__ uint32_t s_excl;
    __shared__ unsigned long long s_rs;

    if (threadIdx.x == 0) {
        s_b = atomicAdd(P.ticket, 1ull);
        mbar_init(&s_bar, 1);
    }
    __syncthreads();

    BlockInfo I;
    I.b = s_b;
    int s = 0;
    while (s + 1 < P.nseg && I.b >= P.seg[s + 1].first_block) ++s;
    const EncSeg& S = P.seg[s];
    const uint64_t lb = I.b - S.first_block;
    const uint64_t cl = lb / S.blocks_per_chunk;
    I.k = static_cast<uint32_t>(lb - cl * S.blocks_per_chunk);
    I.seg = s;
    I.chunk = S.first_chunk + cl;
    I.chunk_off = cl * P.C;
    I.m = static_cast<uint32_t>(S.n - I.chunk_off < P.C ? S.n - I.chunk_off : P.C);
    I.first = I.b - I.k;
    const uint32_t nblk = I.m ? static_cast<uint32_t>(cdiv(I.m, S.block_words)) : 1u;
    I.last = (I.k + 1 == nblk);
    I.p0 = I.k * S.block_words;
    I.nb = I.m > I.p0 ? (I.m - I.p0 < S.block_words ? I.m - I.p0 : S.block_words) : 0u;

    if (S.w == 4)
        encode_block<4>(P, I, tile, s_bal, s_warp, &s_bar, &s_excl, &s_rs);
    else
        encode_block<2>(P, I, tile, s_bal, s_warp, &s_bar, &s_excl, &s_rs);
}

}  // namespace

constexpr size_t kEncDynSmem = 2 * 16384;

cudaError_t launch_encode(const EncParams& p, cudaStream_t s) {
    static bool attr_set = false;
    if (!attr_set) {
        cudaFuncSetAttribute(encode_kernel, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
        attr_set = true;
    }
    if (p.total_blocks == 0) return cudaSuccess;
    encode_kernel<<<static_cast<unsigned>(p.total_blocks), kEncThreads, kEncDynSmem, s>>>(p);
    return cudaGetLastError();
}

}  // namespace tc
