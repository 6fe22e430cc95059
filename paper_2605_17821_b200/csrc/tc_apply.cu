// tc_apply.cu — restore: fold N differential records onto the base in one pass (sm_100a).
//
// What it computes: the state after applying the N
// shard diffs oldest -> newest.  Realised as "newest first hit": each word takes the value of
// the newest record whose mask bit is set, so each state word is written at most once and
// only winning values are read — the lossless analog of the paper's fused multi-step replay
// that "reads the model weights, first moments, and second moments exactly once, applies
// the corresponding N-1 incremental gradients in temporal order ... and writes the final
// results back" (§3.3).
//
// Kernels:
//   fold_walk_kernel  (1 CTA)  walks every record header of every diff, validates structure
//                              (-> CORRUPT), the version chain (-> PROTOCOL) and
//                              the common chunk layout (-> INVALID); builds the descriptor
//                              table and the per-record unit prefix.
//   fold_kernel       (persistent, one warp per unit of max(T, 1024) words; see the fold
//                              section) newest-first winner masks, popcount warp scans for
//                              the value offsets, warp-broadcast scatter of the winning
//                              words; tile_off consistency checked on the way (-> CORRUPT).
#include <cuda_runtime.h>

#include "tc_internal.h"

namespace tc {

namespace {

__device__ __forceinline__ bool is_pow2(uint64_t x) { return x && !(x & (x - 1)); }

__device__ __forceinline__ uint64_t ld_u64(const uint8_t* p) { return *reinterpret_cast<const uint64_t*>(p); }

// ------------------------------------------------------------------ walker ----------
__global__ void __launch_bounds__(TC_MAX_FOLD) fold_walk_kernel(const __grid_constant__ FoldParams P) {
    __shared__ unsigned s_err[TC_MAX_FOLD];
    __shared__ unsigned s_mixed[TC_MAX_FOLD];
    __shared__ unsigned s_nrec[TC_MAX_FOLD];
    __shared__ unsigned long long s_ver[TC_MAX_FOLD];
    __shared__ unsigned long long s_rver[TC_MAX_FOLD];
    __shared__ unsigned s_code;

    const int j = threadIdx.x;
    if (j < P.nrec) {
        const uint8_t* base = P.rec[j];
        const uint64_t bytes = P.rec_bytes[j];
        FoldRec* D = P.desc + static_cast<size_t>(j) * P.cap;
        unsigned err = 0, mixed = 0;
        uint64_t pos = 0, r = 0, ver = 0, rver = 0;
        for (int s = 0; s < P.nseg && !err; ++s) {
            uint64_t off = 0;
            do {
                if (pos + kHdrBytes > bytes) { err = TC_ERR_CORRUPT; break; }
                const uint8_t* h = base + pos;
                const uint64_t h0 = ld_u64(h), h1 = ld_u64(h + 8);
                const uint32_t magic = static_cast<uint32_t>(h0);
                const uint32_t fmt = static_cast<uint32_t>(h0 >> 32) & 0xffffu;
                const uint32_t w = static_cast<uint32_t>(h0 >> 48) & 0xffu;
                const uint32_t flags = static_cast<uint32_t>(h0 >> 56);
                const uint32_t T = static_cast<uint32_t>(h1);
                const uint32_t seg = static_cast<uint32_t>(h1 >> 32);
                const uint64_t coff = ld_u64(h + 16), m = ld_u64(h + 24), count = ld_u64(h + 32);
                const uint64_t version = ld_u64(h + 40), ref_version = ld_u64(h + 48), total = ld_u64(h + 56);
                const bool imode = flags == 3;
                if (magic != 0x31444354u || fmt != 1 || (w != 2 && w != 4) || (flags != 1 && flags != 3) ||
                    !is_pow2(T) || T < 32 || T > 65536 || seg != static_cast<uint32_t>(s) || w != P.w[s] ||
                    coff != off || coff % T != 0 || m > kMaxChunkWords || count > m ||
                    (m == 0 && P.n[s] != 0) || off + m > P.n[s] ||
                    total != (imode ? record_bytes_index(m, T, w, count) : record_bytes(m, T, w, count)) ||
                    total > bytes - pos) {
                    err = TC_ERR_CORRUPT;
                    break;
                }
                if (r >= P.cap) { err = TC_ERR_CAPACITY; break; }
                if (imode && T > kIndexMaxT) { err = TC_ERR_INVALID; break; }  // unsupported here
                FoldRec R;
                if (imode) {
                    R.mask = nullptr;
                    R.toff = h + index_toff_off();
                    R.idx = h + index_idx_off(m, T);
                    R.values = h + index_val_off(m, T, count);
                } else {
                    R.mask = h + kHdrBytes;
                    R.idx = nullptr;
                    R.toff = R.mask + pad16(4 * cdiv(m, 32));
                    R.values = h + record_fixed_bytes(m, T);
                }
                R.chunk_off = coff;
                R.count = count;
                R.m = static_cast<uint32_t>(m);
                R.T = T;
                R.seg = seg;
                R.w = w;
                D[r] = R;
                if (r == 0) {
                    ver = version;
                    rver = ref_version;
                } else if (version != ver || ref_version != rver) {
                    mixed = 1;
                }
                off += m;
                pos += total;
                ++r;
            } while (off < P.n[s]);
        }
        if (!err && pos != bytes) err = TC_ERR_CORRUPT;
        s_err[j] = err;
        s_mixed[j] = mixed;
        s_nrec[j] = static_cast<unsigned>(r);
        s_ver[j] = ver;
        s_rver[j] = rver;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned code = 0;
        for (int k = 0; k < P.nrec && !code; ++k) {
            if (s_err[k]) { code = s_err[k]; break; }
            const unsigned long long expect = k == 0 ? P.state_version : s_ver[k - 1];
            if (s_mixed[k] || s_rver[k] != expect || s_ver[k] <= s_rver[k]) code = TC_ERR_PROTOCOL;
        }
        if (!code)
            for (int k = 1; k < P.nrec; ++k)
                if (s_nrec[k] != s_nrec[0]) code = TC_ERR_INVALID;
        s_code = code;
    }
    __syncthreads();
    if (!s_code) {
        // every diff must share the chunk layout of diff 0 (records of one encode config do)
        const unsigned R = s_nrec[0];
        for (unsigned idx = threadIdx.x; idx < R * static_cast<unsigned>(P.nrec); idx += blockDim.x) {
            const unsigned k = idx / R, r = idx % R;
            if (k == 0) continue;
            const FoldRec& a = P.desc[r];
            const FoldRec& b = P.desc[static_cast<size_t>(k) * P.cap + r];
            if (a.m != b.m || a.T != b.T || a.seg != b.seg || a.chunk_off != b.chunk_off) atomicCAS(&s_code, 0u, TC_ERR_INVALID);
        }
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        if (s_code) {
            tc_set_err(P.err, s_code);
            P.info[0] = 0;
            P.info[1] = 0;
        } else {
            const unsigned R = s_nrec[0];
            uint64_t u = 0;
            for (unsigned r = 0; r < R; ++r) {
                P.unit_first[r] = u;
                const FoldRec& a = P.desc[r];
                const uint64_t U = a.T > kFoldWords ? a.T : kFoldWords;
                u += a.m ? cdiv(a.m, U) : 0;
            }
            P.unit_first[R] = u;
            P.info[0] = R;
            P.info[1] = u;
        }
    }
}

// -------------------------------------------------------------------- fold ----------
// One WARP per unit of U = max(T, kFoldWords) chunk words (units never straddle a tile
// boundary, so each unit starts at a tile_off entry).  A unit is walked in sub-units of up to
// kSub = 4096 words = 4 groups of 32 mask words, lane l holding mask word 32g + l of group g.
// For each record, newest first: load its mask words (4 independent loads per lane), popcount
// warp scans give every mask word's in-chunk value offset, winners = mask & rem (rem = words
// no newer record covers), and the winners are scattered: for each lane whose mask word has
// winners, the warp broadcasts (win, mask, offset) and lane b copies word 32*src+b.  No
// barriers and no shared-memory staging; latency is hidden by 64 resident warps per SM.
constexpr uint32_t kFoldWarps = kFoldThreads / 32;
constexpr uint32_t kSubGroups = 4;
constexpr uint32_t kSub = kSubGroups * 1024;
constexpr int kBatch = 4;  // gathers in flight per lane in the dense scatter
constexpr uint32_t kLaneSerialMax = 96;  // winners per 1024 words below which lanes scatter alone

template <int W>
struct Word;
template <>
struct Word<4> { using T = uint32_t; };
template <>
struct Word<2> { using T = uint16_t; };

__device__ __forceinline__ uint32_t ldg_u32(const uint32_t* p) { return __ldg(p); }
__device__ __forceinline__ uint32_t ldg_word(const uint32_t* p) { return __ldg(p); }
__device__ __forceinline__ uint16_t ldg_word(const uint16_t* p) {
    return static_cast<uint16_t>(__ldg(reinterpret_cast<const unsigned short*>(p)));
}

// Index-mode record: set the bits of the changed words of [sub, send) (chunk-relative) in the
// warp's 128 shared mask words.  Checks each position lies inside its tile and strictly increases
// within the tile (the oracle's index-mode body check); duplicates merge and are caught by the
// unit-end popcount check.
__device__ __forceinline__ void build_mask_from_index(const FoldRec& R, uint32_t sub, uint32_t send, uint32_t* imask,
                                                      int lane, bool& bad) {
#pragma unroll
    for (uint32_t g = 0; g < kSubGroups; ++g) imask[32 * g + lane] = 0;
    __syncwarp();
    const uint32_t T = R.T, m = R.m;
    const uint32_t* toff = reinterpret_cast<const uint32_t*>(R.toff);
    const uint16_t* idx = reinterpret_cast<const uint16_t*>(R.idx);
    for (uint32_t t = sub / T; t * T < send; ++t) {
        const uint32_t ts = t * T;
        const uint32_t tlen = m - ts < T ? m - ts : T;
        const uint32_t a = ldg_u32(toff + t), b = ldg_u32(toff + t + 1);
        if (b < a || b > R.count) {
            bad = true;
            break;
        }
        uint32_t lo = a, hi = b;
        if (ts < sub || ts + T > send) {  // the tile is larger than the sub-unit: find its slice
            const uint32_t want_lo = sub > ts ? sub - ts : 0, want_hi = send - ts;
            uint32_t l = a, h = b;
            while (l < h) {
                const uint32_t mid = (l + h) >> 1;
                if (__ldg(reinterpret_cast<const unsigned short*>(idx) + mid) < want_lo) l = mid + 1; else h = mid;
            }
            lo = l;
            h = b;
            while (l < h) {
                const uint32_t mid = (l + h) >> 1;
                if (__ldg(reinterpret_cast<const unsigned short*>(idx) + mid) < want_hi) l = mid + 1; else h = mid;
            }
            hi = l;
        }
        for (uint32_t k = lo + lane; k < hi; k += 32) {
            const uint32_t x = __ldg(reinterpret_cast<const unsigned short*>(idx) + k);
            if (x >= tlen) {
                bad = true;
                continue;
            }
            if (k > a && __ldg(reinterpret_cast<const unsigned short*>(idx) + k - 1) >= x) bad = true;
            const uint32_t pos = ts + x - sub;
            atomicOr(&imask[pos >> 5], 1u << (pos & 31));
        }
    }
    __syncwarp();
}

template <int W>
__device__ void fold_unit(const FoldParams& P, uint64_t r, uint64_t ku, uint32_t* carry, uint32_t* imask, int lane,
                          bool& bad) {
    using word_t = typename Word<W>::T;
    const int N = P.nrec;
    const FoldRec& L = P.desc[r];  // the chunk layout (shared by every diff)
    const uint32_t m = L.m, T = L.T;
    const uint32_t U = T > kFoldWords ? T : kFoldWords;
    const uint32_t ustart = static_cast<uint32_t>(ku) * U;
    const uint32_t uend = ustart + U < m ? ustart + U : m;
    word_t* state = reinterpret_cast<word_t*>(P.state[L.seg]) + L.chunk_off;
    const uint32_t lt = (1u << lane) - 1u;

    for (uint32_t sub = ustart; sub < uend; sub += kSub) {
        const uint32_t send = sub + kSub < uend ? sub + kSub : uend;
        uint32_t rem[kSubGroups];
#pragma unroll
        for (uint32_t g = 0; g < kSubGroups; ++g) rem[g] = 0xffffffffu;
        for (int j = N - 1; j >= 0; --j) {
            const FoldRec& R = P.desc[static_cast<size_t>(j) * P.cap + r];
            const uint32_t* mask = reinterpret_cast<const uint32_t*>(R.mask);
            const uint32_t* toff = reinterpret_cast<const uint32_t*>(R.toff);
            const word_t* vals = reinterpret_cast<const word_t*>(R.values);
            const uint32_t count = static_cast<uint32_t>(R.count);
            // all mask words of the sub-unit first (independent read-only loads)
            uint32_t mk[kSubGroups];
            if (R.idx) {
                // index-mode record: build this sub-unit's mask words from the in-tile positions
                build_mask_from_index(R, sub, send, imask, lane, bad);
#pragma unroll
                for (uint32_t g = 0; g < kSubGroups; ++g) mk[g] = imask[32 * g + lane];
            } else {
#pragma unroll
                for (uint32_t g = 0; g < kSubGroups; ++g) {
                    const uint32_t p = sub + (32 * g + lane) * 32;
                    mk[g] = p < send ? ldg_u32(mask + (p >> 5)) : 0u;
                }
            }
            uint32_t run = sub == ustart ? ldg_u32(toff + ustart / T) : carry[j];
            if (sub == ustart && ku == 0 && run != 0) bad = true;
#pragma unroll
            for (uint32_t g = 0; g < kSubGroups; ++g) {
                const uint32_t p = sub + (32 * g + lane) * 32;
                if (p + 32 > send && p < send) {  // the chunk's tail word: bits past m must be 0
                    const uint32_t vb = (1u << (send - p)) - 1u;
                    if (mk[g] & ~vb) bad = true;
                    mk[g] &= vb;
                }
                const uint32_t c = __popc(mk[g]);
                uint32_t inc = c;
#pragma unroll
                for (int d = 1; d < 32; d <<= 1) {
                    const uint32_t t = __shfl_up_sync(0xffffffffu, inc, d);
                    if (lane >= d) inc += t;
                }
                const uint32_t pre = run + inc - c;  // in-chunk offset of this mask word's values
                run += __shfl_sync(0xffffffffu, inc, 31);
                if (T < kSub && p < send && p != ustart && (p & (T - 1)) == 0 && ldg_u32(toff + p / T) != pre)
                    bad = true;
                const uint32_t win = mk[g] & rem[g];
                rem[g] &= ~mk[g];
                if (__reduce_add_sync(0xffffffffu, __popc(win)) <= kLaneSerialMax) {
                    // sparse group: each lane walks the winners of its own mask word (at f = 1 %
                    // ~1 bit per lane, so the warp needs a few iterations for all 32 mask words);
                    // two gathers in flight per lane per iteration
                    uint32_t wv = win;
                    const uint32_t base_w = sub + (32 * g + lane) * 32;
                    while (__any_sync(0xffffffffu, wv != 0)) {
                        word_t v0 = 0, v1 = 0;
                        uint32_t d0 = 0xffffffffu, d1 = 0xffffffffu;
                        if (wv) {
                            const uint32_t b = __ffs(wv) - 1;
                            wv &= wv - 1;
                            const uint32_t idx = pre + __popc(mk[g] & ((1u << b) - 1u));
                            if (idx < count) { v0 = ldg_word(vals + idx); d0 = base_w + b; }
                        }
                        if (wv) {
                            const uint32_t b = __ffs(wv) - 1;
                            wv &= wv - 1;
                            const uint32_t idx = pre + __popc(mk[g] & ((1u << b) - 1u));
                            if (idx < count) { v1 = ldg_word(vals + idx); d1 = base_w + b; }
                        }
                        if (d0 != 0xffffffffu) state[d0] = v0;
                        if (d1 != 0xffffffffu) state[d1] = v1;
                    }
                    continue;
                }
                uint32_t nz = __ballot_sync(0xffffffffu, win != 0);
                // batches of kBatch source mask words: the value gathers of a batch are issued
                // before its stores, so kBatch gathers are in flight per lane
                while (nz) {
                    word_t v[kBatch];
                    uint32_t dst[kBatch];
#pragma unroll
                    for (int q = 0; q < kBatch; ++q) {
                        dst[q] = 0xffffffffu;
                        if (nz) {  // warp-uniform
                            const int src = __ffs(nz) - 1;
                            nz &= nz - 1;
                            const uint32_t wb = __shfl_sync(0xffffffffu, win, src);
                            const uint32_t mb = __shfl_sync(0xffffffffu, mk[g], src);
                            const uint32_t o = __shfl_sync(0xffffffffu, pre, src);
                            const uint32_t idx = o + __popc(mb & lt);
                            if (((wb >> lane) & 1u) && idx < count) {  // idx < count keeps a corrupt
                                v[q] = ldg_word(vals + idx);           // record's reads in bounds
                                dst[q] = sub + (32 * g + src) * 32 + lane;
                            }
                        }
                    }
#pragma unroll
                    for (int q = 0; q < kBatch; ++q)
                        if (dst[q] != 0xffffffffu) state[dst[q]] = v[q];
                }
            }
            carry[j] = run;
            if (send == uend) {  // unit end: the next unit's first entry, or the final entry
                const uint32_t want = uend < m ? ldg_u32(toff + uend / T) : ldg_u32(toff + (m + T - 1) / T);
                if (want != run || (uend == m && count != run)) bad = true;
            }
        }
    }
}

__global__ void __launch_bounds__(kFoldThreads, 4) fold_kernel(const __grid_constant__ FoldParams P) {
    __shared__ uint32_t s_carry[kFoldWarps][TC_MAX_FOLD];
    __shared__ uint32_t s_imask[kFoldWarps][kSubGroups * 32];  // index-mode records: built mask words
    if (*reinterpret_cast<volatile unsigned*>(P.err) != 0) return;  // sticky error pending
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const uint64_t R = P.info[0];
    const uint64_t total = P.info[1];
    const uint64_t nwarps = static_cast<uint64_t>(gridDim.x) * kFoldWarps;
    bool bad = false;
    for (uint64_t u = static_cast<uint64_t>(blockIdx.x) * kFoldWarps + wid; u < total; u += nwarps) {
        // record r: unit_first[r] <= u < unit_first[r+1]
        uint64_t lo = 0, hi = R;
        while (hi - lo > 1) {
            const uint64_t mid = (lo + hi) >> 1;
            if (P.unit_first[mid] <= u) lo = mid; else hi = mid;
        }
        const uint64_t ku = u - P.unit_first[lo];
        if (P.desc[lo].w == 4)
            fold_unit<4>(P, lo, ku, s_carry[wid], s_imask[wid], lane, bad);
        else
            fold_unit<2>(P, lo, ku, s_carry[wid], s_imask[wid], lane, bad);
        if (__any_sync(0xffffffffu, bad)) {  // malformed record: state unspecified
            if (lane == 0) tc_set_err(P.err, TC_ERR_CORRUPT);
            return;
        }
    }
}

}  // namespace

cudaError_t launch_fold(const FoldParams& p, cudaStream_t s, int num_sms, uint64_t* launches) {
    fold_walk_kernel<<<1, TC_MAX_FOLD, 0, s>>>(p);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    static int occ = 0;
    if (!occ) {
        if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, fold_kernel, kFoldThreads, 0) != cudaSuccess || occ < 1)
            occ = 1;
    }
    fold_kernel<<<num_sms * occ, kFoldThreads, 0, s>>>(p);
    *launches += 2;
    return cudaGetLastError();
}

}  // namespace tc
