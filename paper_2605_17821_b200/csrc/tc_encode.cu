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

// Record start of chunk c (published by the last block of chunk c-1 as value | 1).
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

__device__ __forceinline__ void bar_sync(uint32_t id, uint32_t n) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}
__device__ __forceinline__ void bar_arrive(uint32_t id, uint32_t n) {
    asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(n) : "memory");
}

constexpr uint32_t kComputeWarps = kEncThreads / 32;   // 8 warps compare/compact
constexpr uint32_t kCtaThreads = kEncThreads + 32;     // + 1 scan warp (look-back)
constexpr uint32_t kBarCompute = 1;                    // named barrier: compute warps only
constexpr uint32_t kBarPrefix = 2;                     // scan warp -> compute warps

struct BlockInfo {
    unsigned long long b;          // global block index (= ticket)
    unsigned long long first;      // global index of the chunk's first block
    unsigned long long chunk;      // global chunk index
    unsigned long long chunk_off;  // word offset of the chunk in its segment
    uint32_t m;                    // words in the chunk
    uint32_t k;                    // block index within the chunk
    uint32_t p0;                   // chunk-relative first word of the block
    uint32_t nb;                   // words in this block
    uint32_t seg;
    uint32_t w;
    uint32_t last;                 // last block of its chunk
};

struct EncSmem {
    BlockInfo I;
    uint64_t bar;
    uint32_t bal[kEncBlockWords2 / 32];  // mask words of the block
    uint32_t warp_cnt[kComputeWarps];
    uint32_t warp_off[kComputeWarps];
    uint32_t total;
    uint32_t ready;   // counts published to the scan warp (polled)
    uint32_t excl;    // in-chunk exclusive count of the block
    unsigned long long rs;  // byte offset of the block's record
};

// Scan warp: decoupled look-back over the in-chunk status words.  The exclusive prefix of
// block b does not depend on b's own data, so the look-back starts as soon as the ticket is
// claimed, overlapping the TMA load and pass 1; b's AGGREGATE is published from inside the
// polling loop the moment the compute warps report the block count.
__device__ __forceinline__ void scan_warp(const EncParams& P, EncSmem& sm, int lane) {
    const BlockInfo& I = sm.I;
    volatile uint32_t* ready = &sm.ready;
    uint32_t excl = 0;
    bool published = false;
    uint32_t spins = 0;
    if (I.k != 0) {
        long long j = static_cast<long long>(I.b) - 1;
        while (true) {
            if (!published && __any_sync(0xffffffffu, *ready != 0)) {
                if (lane == 0) st_relaxed(&P.status[I.b], kFlagAgg | sm.total);
                published = true;
            }
            const long long idx = j - lane;
            const unsigned long long sv =
                idx >= static_cast<long long>(I.first) ? ld_relaxed(&P.status[idx]) : kFlagInc;
            const uint32_t flag = static_cast<uint32_t>(sv >> 62);
            const uint32_t incl = __ballot_sync(0xffffffffu, flag == 2);
            const uint32_t empty = __ballot_sync(0xffffffffu, flag == 0);
            const uint32_t upto = incl ? (((incl & (0u - incl)) << 1) - 1u) : 0xffffffffu;
            if (empty & upto) {
                if (++spins > kSpinLimit) {
                    if (lane == 0) tc_set_err(P.err, TC_ERR_INTERNAL);
                    break;
                }
                __nanosleep(32);
                continue;
            }
            uint32_t v = ((upto >> lane) & 1u) ? static_cast<uint32_t>(sv) : 0u;
#pragma unroll
            for (int d = 16; d; d >>= 1) v += __shfl_xor_sync(0xffffffffu, v, d);
            excl += v;
            if (incl) break;
            j -= 32;
        }
    }
    while (!*ready) __nanosleep(20);
    const uint32_t total = sm.total;
    if (lane == 0) {
        st_relaxed(&P.status[I.b], kFlagInc | static_cast<unsigned long long>(excl + total));
        const unsigned long long rs = wait_rstart(P, I.chunk);
        if (I.last) {
            const uint64_t W = I.w;
            const uint64_t count = static_cast<uint64_t>(excl) + total;
            const uint64_t n_mask = cdiv(I.m, 32);
            const uint64_t n_tiles = cdiv(I.m, P.T);
            const uint64_t rec_total = record_bytes(I.m, P.T, I.w, count);
            uint8_t* rec = P.out + rs;
            uint64_t* h = reinterpret_cast<uint64_t*>(rec);
            h[0] = 0x31444354ull /* "TCD1" */ | (1ull << 32) | (W << 48) | (1ull << 56);
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
            uint8_t* gval = rec + record_fixed_bytes(I.m, P.T);
            for (uint64_t x = W * count; x < pad16(W * count); ++x) gval[x] = 0;
            const unsigned long long next = rs + rec_total;
            st_relaxed(&P.rstart[I.chunk + 1], next | 1ull);
            if (I.chunk + 1 == P.total_chunks) *P.out_bytes = next;
        }
        sm.excl = excl;
        sm.rs = rs;
    }
    __syncwarp();
    bar_arrive(kBarPrefix, kCtaThreads);
}

// Compute warps (8): stage wait, pass 1 (compare -> ballot = mask word; fused ref advance),
// counts, then (after the scan warp's prefix) pass 2 (mask words, tile_off, packed values).
template <int W>
__device__ __forceinline__ void compute_warps(const EncParams& P, EncSmem& sm, uint8_t* tile, int tid) {
    using word_t = typename Word<W>::T;
    constexpr uint32_t B = Word<W>::kBlock;
    constexpr uint32_t MPW = B / 32 / kComputeWarps;  // mask words per warp (16 | 32)
    const int lane = tid & 31, wid = tid >> 5;
    const BlockInfo& I = sm.I;
    const EncSeg& S = P.seg[I.seg];
    word_t* sref = reinterpret_cast<word_t*>(tile);
    word_t* scur = sref + B;
    word_t* gref = reinterpret_cast<word_t*>(S.ref) + I.chunk_off + I.p0;
    const word_t* gcur = reinterpret_cast<const word_t*>(S.cur) + I.chunk_off + I.p0;

    // tail words (< 16 bytes) not covered by the bulk copy; pad the rest of a short block with
    // equal words so pass 1 needs no bounds test
    const uint32_t bytes = I.nb * W;
    const uint32_t bulk = bytes & ~15u;
    if (I.nb < B) {
        for (uint32_t i = bulk / W + tid; i < B; i += kEncThreads) {
            const bool in = i < I.nb;
            sref[i] = in ? gref[i] : word_t(0);
            scur[i] = in ? gcur[i] : word_t(0);
        }
    }
    mbar_wait_parity(&sm.bar, 0);
    if (I.nb < B) bar_sync(kBarCompute, kEncThreads);

    // ---- pass 1 ----
    const bool adv = P.advance_ref != 0;
    const uint32_t mw0 = wid * MPW;
#pragma unroll 4
    for (uint32_t q = 0; q < MPW; ++q) {
        const uint32_t i = (mw0 + q) * 32 + lane;
        const word_t v = scur[i];
        const bool ch = sref[i] != v;
        const uint32_t bal = __ballot_sync(0xffffffffu, ch);
        if (lane == 0) sm.bal[mw0 + q] = bal;
        if (adv && bal) {
            if (ch) gref[i] = v;
        }
    }
    __syncwarp();
    // ---- counts: lane-per-mask-word popcount scan over the warp's range ----
    uint32_t bal = 0, pre = 0;
    if (lane < static_cast<int>(MPW)) bal = sm.bal[mw0 + lane];
    const uint32_t c = __popc(bal);
    uint32_t inc = c;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        const uint32_t t = __shfl_up_sync(0xffffffffu, inc, d);
        if (lane >= d) inc += t;
    }
    pre = inc - c;
    if (lane == 31) sm.warp_cnt[wid] = inc;
    bar_sync(kBarCompute, kEncThreads);
    if (wid == 0) {
        const uint32_t wc = lane < static_cast<int>(kComputeWarps) ? sm.warp_cnt[lane] : 0u;
        uint32_t x = wc;
#pragma unroll
        for (int d = 1; d < static_cast<int>(kComputeWarps); d <<= 1) {
            const uint32_t t = __shfl_up_sync(0xffffffffu, x, d);
            if (lane >= d) x += t;
        }
        if (lane < static_cast<int>(kComputeWarps)) sm.warp_off[lane] = x - wc;
        if (lane == kComputeWarps - 1) {
            sm.total = x;
            __threadfence_block();
            *reinterpret_cast<volatile uint32_t*>(&sm.ready) = 1u;
        }
    }
    bar_sync(kBarPrefix, kCtaThreads);  // scan warp has the exclusive prefix + record start

    // ---- pass 2 ----
    uint8_t* rec = P.out + sm.rs;
    const uint64_t n_mask = cdiv(I.m, 32);
    uint32_t* gmask = reinterpret_cast<uint32_t*>(rec + kHdrBytes);
    uint32_t* gtoff = reinterpret_cast<uint32_t*>(rec + kHdrBytes + pad16(4 * n_mask));
    word_t* gval = reinterpret_cast<word_t*>(rec + record_fixed_bytes(I.m, P.T));
    const uint32_t base = sm.excl + sm.warp_off[wid];
    const uint32_t p = I.p0 + (mw0 + lane) * 32;  // chunk-relative first word of this lane's mask word
    const bool mine = lane < static_cast<int>(MPW) && p < I.m;
    if (mine) {
        gmask[(I.p0 >> 5) + mw0 + lane] = bal;
        if ((p & (P.T - 1)) == 0) gtoff[p / P.T] = base + pre;
    }
    uint32_t nz = __ballot_sync(0xffffffffu, bal != 0);
    const uint32_t lt = (1u << lane) - 1u;
    while (nz) {
        const int src = __ffs(nz) - 1;
        nz &= nz - 1;
        const uint32_t b = __shfl_sync(0xffffffffu, bal, src);
        const uint32_t o = __shfl_sync(0xffffffffu, pre, src);
        if ((b >> lane) & 1u) gval[base + o + __popc(b & lt)] = scur[(mw0 + src) * 32 + lane];
    }
}

__global__ void __launch_bounds__(kCtaThreads, 6) encode_kernel(const __grid_constant__ EncParams P) {
    extern __shared__ __align__(128) uint8_t tile[];
    __shared__ EncSmem sm;
    const int tid = threadIdx.x;

    if (tid == kEncThreads) {
        // one thread: ticket, decode, barrier init, TMA issue — loads start as early as possible
        BlockInfo I;
        I.b = atomicAdd(P.ticket, 1ull);
        int s = 0;
        while (s + 1 < P.nseg && I.b >= P.seg[s + 1].first_block) ++s;
        const EncSeg& S = P.seg[s];
        const uint32_t lb = static_cast<uint32_t>(I.b - S.first_block);
        const uint32_t bpc = static_cast<uint32_t>(S.blocks_per_chunk);
        const uint32_t cl = lb / bpc;
        I.k = lb - cl * bpc;
        I.seg = s;
        I.w = S.w;
        I.chunk = S.first_chunk + cl;
        I.chunk_off = static_cast<unsigned long long>(cl) * P.C;
        I.m = static_cast<uint32_t>(S.n - I.chunk_off < P.C ? S.n - I.chunk_off : P.C);
        I.first = I.b - I.k;
        const uint32_t nblk = I.m ? (I.m + S.block_words - 1) / S.block_words : 1u;
        I.last = (I.k + 1 == nblk);
        I.p0 = I.k * S.block_words;
        I.nb = I.m > I.p0 ? (I.m - I.p0 < S.block_words ? I.m - I.p0 : S.block_words) : 0u;
        sm.I = I;
        sm.ready = 0;
        mbar_init(&sm.bar, 1);
        const uint32_t bulk = (I.nb * S.w) & ~15u;
        if (bulk) {
            const uint8_t* gref = S.ref + (I.chunk_off + I.p0) * S.w;
            const uint8_t* gcur = S.cur + (I.chunk_off + I.p0) * S.w;
            mbar_arrive_expect_tx(&sm.bar, 2 * bulk);
            bulk_g2s(tile, gref, bulk, &sm.bar);
            bulk_g2s(tile + 16384, gcur, bulk, &sm.bar);
        } else {
            mbar_arrive(&sm.bar);
        }
    }
    __syncthreads();
    if (tid >= kEncThreads) {
        scan_warp(P, sm, tid & 31);
    } else if (sm.I.w == 4) {
        compute_warps<4>(P, sm, tile, tid);
    } else {
        compute_warps<2>(P, sm, tile, tid);
    }
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
    encode_kernel<<<static_cast<unsigned>(p.total_blocks), kCtaThreads, kEncDynSmem, s>>>(p);
    return cudaGetLastError();
}

}  // namespace tc
