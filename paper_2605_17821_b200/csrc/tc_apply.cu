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
// Kernels (every fold launches all four; each returns at once when no chunk is its kind):
//   fold_walk_kernel  (1 CTA)  walks every record header of every diff, validates structure
//                              (-> CORRUPT), the version chain (-> PROTOCOL) and
//                              the common chunk layout (-> INVALID); builds the descriptor
//                              table and the per-record unit prefix; picks each chunk's strategy.
//   fold_kernel       (persistent, one warp per unit of max(T, 4096) words) scatter: newest-
//                              first winner masks, popcount warp scans for the value offsets,
//                              scatter of the winning words (a sparse single index record
//                              straight from its entry ranges); tile_off checked on the way.
//   fold_list_kernel  (a CTA per 4096-word tile, 10 per SM) streaming fold of all-index T = 4096
//                              chains of <= 32 records:
//                              tile in shared memory, records' runs staged, oldest -> newest.
//   fold_dense_kernel (one warp per CTA) streaming fold of any other chain (opt-in).
#include <cuda_runtime.h>

#include "tc_internal.h"
#include "tc_ptx.cuh"

namespace tc {

namespace {

__device__ __forceinline__ bool is_pow2(uint64_t x) { return x && !(x & (x - 1)); }

__device__ __forceinline__ uint64_t ld_u64(const uint8_t* p) { return *reinterpret_cast<const uint64_t*>(p); }

constexpr uint32_t kEntryTiles = 32;  // fold_entries: tiles a warp takes per unit (one per lane)

// Words per fold unit of a chunk: max(T, kFoldWords); entry-driven chunks (strategy 3) take
// kEntryTiles tiles of max(T, kFoldWords) words per unit.
__host__ __device__ inline uint64_t fold_unit_words(uint32_t T, uint32_t strategy) {
    const uint64_t U = T > kFoldWords ? T : kFoldWords;
    return strategy == 3u ? U * kEntryTiles : U;
}

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
                const bool imode = flags == 3, full = flags == 5;
                if (magic != 0x31444354u || fmt != 1 || (w != 2 && w != 4) || (flags != 1 && flags != 3 && flags != 5) ||
                    !is_pow2(T) || T < 32 || T > 65536 || seg != static_cast<uint32_t>(s) || w != P.w[s] ||
                    coff != off || coff % T != 0 || m > kMaxChunkWords || count > m || (full && count != m) ||
                    (m == 0 && P.n[s] != 0) || off + m > P.n[s] ||
                    total != (full ? record_bytes_full(m, w)
                              : imode ? record_bytes_index(m, T, w, count) : record_bytes(m, T, w, count)) ||
                    total > bytes - pos) {
                    err = TC_ERR_CORRUPT;
                    break;
                }
                if (r >= P.cap) {  // below the ABI limit the table is sized by the shortest diff:
                    err = P.cap_hinted || P.cap >= TC_MAX_RECORDS_PER_DIFF ? TC_ERR_CAPACITY : TC_ERR_INVALID;  // layouts differ
                    break;
                }
                if (imode && T > kIndexMaxT) { err = TC_ERR_INVALID; break; }  // unsupported here
                FoldRec R;
                R.full = full ? 1u : 0u;
                if (full) {  // every word of the chunk, in index order
                    R.mask = nullptr;
                    R.idx = nullptr;
                    R.toff = nullptr;
                    R.values = h + kHdrBytes;
                } else if (imode) {
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
            P.info[2] = 0;
            P.info[3] = 0;
            P.info[4] = 0;
            P.info[5] = 0;
            P.info[6] = 0;
            P.info[7] = 0;
        } else {
            const unsigned R = s_nrec[0];
            uint64_t u = 0, ndense = 0, nlist = 0, nentry = 0, nmlist = 0, nmlist_s = 0;
            for (unsigned r = 0; r < R; ++r) {
                P.unit_first[r] = u;
                FoldRec& a = P.desc[r];
                // dense chunk: the changed words of the N records cover enough sectors that
                // streaming the whole chunk through shared memory beats scattered writes
                uint64_t sum = 0;
                for (int k = 0; k < P.nrec; ++k) sum += P.desc[static_cast<size_t>(k) * P.cap + r].count;
                // strategy (measured): chains of <= kListMaxRec index-mode records at T = 4096 are
                // streamed by the list kernel when they are long (N >= 4, >= 0.5 % of the words in
                // total) or dense (> dense_permille); everything else is scattered.  0 = stream
                // every chunk (mask-mode chunks through fold_dense_kernel), UINT32_MAX = scatter all.
                bool all_idx = a.T == kListT && P.nrec <= static_cast<int>(kListMaxRec);
                for (int k = 0; k < P.nrec && all_idx; ++k) all_idx = P.desc[static_cast<size_t>(k) * P.cap + r].idx != nullptr;
                bool all_index = true;  // every record of the chunk's chain is an index-mode record
                for (int k = 0; k < P.nrec && all_index; ++k) all_index = P.desc[static_cast<size_t>(k) * P.cap + r].idx != nullptr;
                bool any_full = false;  // chains with a full record are scattered (fold_unit handles them)
                for (int k = 0; k < P.nrec; ++k) any_full = any_full || P.desc[static_cast<size_t>(k) * P.cap + r].full;
                // every record a mask-mode one at T = 4096: the mask-list kernel can stream the chain
                bool all_mask = a.T <= kListT && P.nrec <= static_cast<int>(kListMaxRec) && !any_full;
                for (int k = 0; k < P.nrec && all_mask; ++k) all_mask = P.desc[static_cast<size_t>(k) * P.cap + r].idx == nullptr;
                const uint64_t mm = a.m;
                if (any_full) {
                    a.dense = 0u;
                } else if (all_index && P.dense_permille != 0u && P.dense_permille != 0xffffffffu &&
                           (P.nrec == 1 || sum * 400ull <= mm * static_cast<uint64_t>(P.nrec))) {
                    // index records applied straight from their entries, one pass per record oldest ->
                    // newest (fold_entries_kernel): always for one record; for a chain while the
                    // records average <= 0.25 % changed (cfg2 measured: a pass costs 0.38 ms at 0.1 %,
                    // 2.3 ms at 1 %; the streaming list fold of 8 records 6.6 / 8.1 ms)
                    a.dense = 3u;
                } else if (P.dense_permille == 0u) {
                    a.dense = all_idx ? 2u : all_mask ? (a.T == kListT ? 4u : 5u) : 1u;
                } else if (P.dense_permille == 0xffffffffu || !(all_idx || all_mask)) {
                    a.dense = 0u;
                } else if (all_idx) {
                    const bool stream = (P.nrec >= 4 && sum * 1000ull >= mm * 5ull) || sum * 1000ull > mm * P.dense_permille;
                    a.dense = stream ? 2u : 0u;
                } else {
                    // mask chains (cfg2 sweep, profiles/rd5q_mask_fold_sweep.txt): streaming wins once the
                    // records change more than ~6 % of the words in total, whatever N (N = 4 at 1 % each:
                    // scatter 8.4 vs 9.5 ms; N = 2 at 3 %: 9.0 vs 8.7; N = 8 at 1 %: 16.5 vs 12.3)
                    a.dense = sum * 1000ull > mm * P.dense_permille ? (a.T == kListT ? 4u : 5u) : 0u;
                }
                ndense += a.dense == 1u;
                nlist += a.dense == 2u;
                nentry += a.dense == 3u;
                nmlist += a.dense == 4u;
                nmlist_s += a.dense == 5u;
                const uint64_t U = fold_unit_words(a.T, a.dense);
                u += a.m ? cdiv(a.m, U) : 0;
            }
            P.unit_first[R] = u;
            P.info[0] = R;
            P.info[1] = u;
            P.info[2] = ndense;              // chunks for fold_dense_kernel
            P.info[3] = R - ndense - nlist - nentry - nmlist - nmlist_s;  // chunks for fold_kernel
            P.info[4] = nlist;               // chunks for fold_list_kernel
            P.info[5] = nentry;              // chunks for fold_entries_kernel
            P.info[6] = nmlist;              // chunks for fold_mlist_kernel<false> (T = 4096)
            P.info[7] = nmlist_s;            // chunks for fold_mlist_kernel<true> (T < 4096)
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
// barriers and no shared-memory staging; latency is hidden by 32 resident warps per SM (4 CTAs of 8).
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
            // a tampered (non-increasing) position list can make the binary search above return
            // entries outside the sub-unit: never let them index the warp's mask words
            if (ts + x < sub || ts + x >= send) {
                bad = true;
                continue;
            }
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
            const bool full = R.full != 0;
            // all mask words of the sub-unit first (independent read-only loads)
            uint32_t mk[kSubGroups];
            if (full) {
                // a full record: every word of the chunk is a value (its implicit mask is all ones)
#pragma unroll
                for (uint32_t g = 0; g < kSubGroups; ++g) {
                    const uint32_t p = sub + (32 * g + lane) * 32;
                    mk[g] = p >= send ? 0u : (p + 32 > send ? (1u << (send - p)) - 1u : 0xffffffffu);
                }
            } else if (R.idx) {
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
            uint32_t run = sub == ustart ? (full ? ustart : ldg_u32(toff + ustart / T)) : carry[j];
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
                if (!full && T < kSub && p < send && p != ustart && (p & (T - 1)) == 0 && ldg_u32(toff + p / T) != pre)
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
                const uint32_t want = full ? uend : (uend < m ? ldg_u32(toff + uend / T) : ldg_u32(toff + (m + T - 1) / T));
                if (want != run || (uend == m && count != run)) bad = true;
            }
        }
    }
}

// One index-mode record (N = 1): its positions are explicit, so a unit of kEntryTiles tiles is
// applied straight from its entries — no mask words.  Lane l holds tile l's entry range
// [tile_off[t], tile_off[t+1]); the warp walks the group's entries as one flat range, 32 entries
// per pass and 4 passes in flight (coalesced position / value loads), each lane finding its
// entry's tile by a 5-step binary search over the lanes' tile starts (shuffles), then storing the
// word.  Checks as everywhere: ranges monotone and inside the record, first entry 0, last =
// count, positions inside the tile and strictly increasing within it.  ~20 warp instructions per
// 32 entries, against ~800 per 32 entries through the mask machinery (r2 ncu: that path issued
// on 61 % of cycles at 23 % of DRAM bandwidth for the step's 1 % record).
template <int W>
__device__ void fold_entries(const FoldParams& P, const FoldRec& R, uint64_t ku, int lane, bool& bad) {
    using word_t = typename Word<W>::T;
    const uint32_t m = R.m, T = R.T;
    const uint64_t Uw = fold_unit_words(R.T, 3u);
    const uint32_t tpu = static_cast<uint32_t>(Uw / T);  // tiles per unit
    const uint32_t nt = (m + T - 1) / T;
    const uint32_t tb0 = static_cast<uint32_t>(ku) * tpu;
    const uint32_t tb1 = tb0 + tpu < nt ? tb0 + tpu : nt;
    word_t* state = reinterpret_cast<word_t*>(P.state[R.seg]) + R.chunk_off;
    const uint32_t* toff = reinterpret_cast<const uint32_t*>(R.toff);
    const uint16_t* idx = reinterpret_cast<const uint16_t*>(R.idx);
    const word_t* vals = reinterpret_cast<const word_t*>(R.values);
    const uint32_t count = static_cast<uint32_t>(R.count);
    constexpr int kQ = 4;
    for (uint32_t tg = tb0; tg < tb1; tg += 32) {
        const uint32_t ng = tb1 - tg < 32 ? tb1 - tg : 32;  // tiles in this group
        const uint32_t t = tg + lane;
        const bool in = static_cast<uint32_t>(lane) < ng;
        const uint32_t a = in ? ldg_u32(toff + t) : 0xffffffffu;
        const uint32_t b = in ? ldg_u32(toff + t + 1) : 0u;
        if (in && (b < a || b > count || (t == 0 && a != 0) || (t + 1 == nt && b != count))) bad = true;
        const uint32_t A = __shfl_sync(0xffffffffu, a, 0);
        const uint32_t B = __shfl_sync(0xffffffffu, b, ng - 1);
        if (B < A || B > count || __any_sync(0xffffffffu, bad)) {
            bad = true;
            continue;
        }
        uint32_t carry_x = 0xffffffffu;  // position of the entry before this pass's lane 0
        for (uint32_t kb = A; kb < B; kb += 32 * kQ) {
            uint32_t x[kQ];
            word_t v[kQ];
#pragma unroll
            for (int q = 0; q < kQ; ++q) {
                const uint32_t k = kb + q * 32 + lane;
                x[q] = 0;
                if (k < B) {
                    x[q] = __ldg(reinterpret_cast<const unsigned short*>(idx) + k);
                    v[q] = ldg_word(vals + k);
                }
            }
#pragma unroll
            for (int q = 0; q < kQ; ++q) {
                const uint32_t k = kb + q * 32 + lane;
                // the tile: the last lane j < ng whose start a_j <= k (empty tiles resolve upward)
                uint32_t lo = 0, hi = ng;
#pragma unroll
                for (int st = 0; st < 5; ++st) {
                    const uint32_t mid = (lo + hi) >> 1;
                    const uint32_t am = __shfl_sync(0xffffffffu, a, mid);
                    if (hi - lo > 1) {
                        if (am <= k) lo = mid;
                        else hi = mid;
                    }
                }
                const uint32_t aj = __shfl_sync(0xffffffffu, a, lo);
                const uint32_t up = __shfl_up_sync(0xffffffffu, x[q], 1);
                const uint32_t prev = lane == 0 ? carry_x : up;
                carry_x = __shfl_sync(0xffffffffu, x[q], 31);
                if (k < B) {
                    const uint32_t ts = (tg + lo) * T;
                    const uint32_t tl = m - ts < T ? m - ts : T;
                    if (x[q] >= tl || (k > aj && prev >= x[q])) {
                        bad = true;
                        continue;
                    }
                    state[ts + x[q]] = v[q];
                }
            }
        }
    }
}

__global__ void __launch_bounds__(kFoldThreads, 4) fold_kernel(const __grid_constant__ FoldParams P) {
    __shared__ uint32_t s_carry[kFoldWarps][TC_MAX_FOLD];
    __shared__ uint32_t s_imask[kFoldWarps][kSubGroups * 32];  // index-mode records: built mask words
    if (*reinterpret_cast<volatile unsigned*>(P.err) != 0) return;  // sticky error pending
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    if (P.info[3] == 0) return;  // every chunk is folded by fold_dense_kernel
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
        if (P.desc[lo].dense == 1u || P.desc[lo].dense == 2u || P.desc[lo].dense >= 4u) {  // a streaming kernel's chunk: jump past it
            const uint64_t nxt = P.unit_first[lo + 1];
            u += (nxt - u + nwarps - 1) / nwarps * nwarps - nwarps;
            continue;
        }
        const uint64_t ku = u - P.unit_first[lo];
        if (P.desc[lo].dense == 3u) {  // fold_entries_kernel's chunk: jump past it
            const uint64_t nxt = P.unit_first[lo + 1];
            u += (nxt - u + nwarps - 1) / nwarps * nwarps - nwarps;
            continue;
        }
        if (P.desc[lo].w == 4) {
            fold_unit<4>(P, lo, ku, s_carry[wid], s_imask[wid], lane, bad);
        } else {
            fold_unit<2>(P, lo, ku, s_carry[wid], s_imask[wid], lane, bad);
        }
        if (__any_sync(0xffffffffu, bad)) {  // malformed record: state unspecified
            if (lane == 0) tc_set_err(P.err, TC_ERR_CORRUPT);
            return;
        }
    }
}

// Chunks whose chain is index-mode records applied from their entries (walker strategy 3): one
// launch per record j, oldest first (stream order = newest wins); a warp per unit of kEntryTiles
// tiles (fold_entries).
__global__ void __launch_bounds__(kFoldThreads) fold_entries_kernel(const __grid_constant__ FoldParams P, int j) {
    if (*reinterpret_cast<volatile unsigned*>(P.err) != 0) return;  // sticky error pending
    if (P.info[5] == 0) return;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const uint64_t R = P.info[0];
    const uint64_t total = P.info[1];
    const uint64_t nwarps = static_cast<uint64_t>(gridDim.x) * kFoldWarps;
    bool bad = false;
    for (uint64_t u = static_cast<uint64_t>(blockIdx.x) * kFoldWarps + wid; u < total; u += nwarps) {
        uint64_t lo = 0, hi = R;
        while (hi - lo > 1) {
            const uint64_t mid = (lo + hi) >> 1;
            if (P.unit_first[mid] <= u) lo = mid; else hi = mid;
        }
        if (P.desc[lo].dense != 3u) {  // another kernel's chunk: jump past it
            const uint64_t nxt = P.unit_first[lo + 1];
            u += (nxt - u + nwarps - 1) / nwarps * nwarps - nwarps;
            continue;
        }
        const uint64_t ku = u - P.unit_first[lo];
        const FoldRec& Rj = P.desc[static_cast<size_t>(j) * P.cap + lo];  // record j of chunk lo
        if (Rj.w == 4)
            fold_entries<4>(P, Rj, ku, lane, bad);
        else
            fold_entries<2>(P, Rj, ku, lane, bad);
        if (__any_sync(0xffffffffu, bad)) {  // malformed record: state unspecified
            if (lane == 0) tc_set_err(P.err, TC_ERR_CORRUPT);
            return;
        }
    }
}

// ------------------------------------------------------------- dense fold ----------
// The streaming fold's general path (walker kind 1: chunks that are not an all-index T = 4096
// chain; selected by the dense_permille = 0 setting — by default such chunks are scattered, which
// measured faster).  Streaming pays off when most 32-byte sectors hold a changed
// word, where scattered partial-sector writes cost a DRAM read-modify-write each.
// One warp per CTA; per sub-unit of kDSub words (lane l owns mask words kMW*l .. kMW*l+kMW-1):
//   1. one TMA bulk copy brings the sub-unit's state into a shared tile (mbarrier);
//   2. for a batch of up to kDBatch records, all in flight together: the mask words (index
//      mode: a 64-entry window of positions) and a kWin-byte window of the value run, which
//      starts at the record's running value count (known before the mask arrives);
//   3. popcount-scan the masks to value offsets, check tile_off;
//   4. expand each record's values into the tile oldest -> newest (newest wins) from the
//      staged window, or - when the run is longer than the window - straight from the record;
//   5. each lane writes its touched 32-word lines back with TMA bulk stores (whole lines: no
//      partial-sector writes); they drain while the next sub-unit loads.
constexpr uint32_t kDenseThreads = 32;
constexpr uint32_t kDSub = 4096;
constexpr uint32_t kMW = kDSub / 1024;  // mask words per lane
constexpr uint32_t kDenseBlocksPerSM = 9;
#ifndef TC_DENSE_RUN
#define TC_DENSE_RUN 16
#endif
constexpr uint64_t kDenseRun = TC_DENSE_RUN;  // consecutive units per CTA visit (running counts carry over)
constexpr int kDBatch = 8;
constexpr uint32_t kWin = 512;
static_assert(kFoldWords % kDSub == 0, "fold units are whole dense sub-units");
static_assert(kWin >= 4 * kLaneSerialMax + 32, "a lane-serial run always fits its window");

struct DenseRec {                 // per record of the current chunk, in shared memory
    const uint8_t* body;          // mask words, or (index mode) u16 positions
    const uint8_t* values;
    const uint32_t* toff;
    uint32_t count;
    uint32_t is_idx;
};

struct DenseSmem {
    uint4 tile[kDSub * 4 / 16];           // the sub-unit's state (16 KB for fp32)
    uint4 stage[kDBatch * kWin / 16];     // value windows
    DenseRec rec[TC_MAX_FOLD];
    uint32_t carry[TC_MAX_FOLD];          // running value count (= first entry) per record
    uint32_t tend[TC_MAX_FOLD];           // tile end entry (T >= kDSub)
    uint32_t want[TC_MAX_FOLD];           // tile_off entry at the unit end
    uint32_t imask[kDSub / 32];           // index-mode positions -> mask words / touched lines
    uint64_t bar;                         // tile load barrier
};

__device__ __forceinline__ uint32_t ldg_u16(const uint8_t* base, uint32_t k) {
    return __ldg(reinterpret_cast<const unsigned short*>(base) + k);
}

// the 16-byte-aligned cover of value run [rb, rb + tot), in bytes
template <int W>
__device__ __forceinline__ uint32_t run_bytes(uint32_t rb, uint32_t tot) {
    const uint64_t a0 = (static_cast<uint64_t>(rb) * W) & ~uint64_t(15);
    const uint64_t a1 = (static_cast<uint64_t>(rb + tot) * W + 15) & ~uint64_t(15);
    return static_cast<uint32_t>(a1 - a0);
}
// the speculative window from the run start: at most kWin bytes, inside the padded values section
template <int W>
__device__ __forceinline__ uint32_t window_bytes(uint32_t count, uint32_t rb) {
    const uint64_t a0 = (static_cast<uint64_t>(rb) * W) & ~uint64_t(15);
    const uint64_t vend = pad16(static_cast<uint64_t>(count) * W);
    return a0 >= vend ? 0u : static_cast<uint32_t>(vend - a0 < kWin ? vend - a0 : kWin);
}

// Index-mode record: its positions inside [sub, send) -> the warp's shared mask words.
// Entries are consumed from rb on (the running count = the first entry of this sub-unit).
// T >= kDSub: the sub-unit lies in one tile ending at entry `e`; xa / xb = entries rb + lane and
// rb + 32 + lane, loaded with the batch.  T < kDSub: the sub-unit holds whole tiles.
__device__ __forceinline__ void dense_index_build(const DenseRec& D, uint32_t T, uint32_t m, uint32_t sub,
                                                  uint32_t send, uint32_t rb, uint32_t e, uint32_t xa, uint32_t xb,
                                                  uint32_t* imask, int lane, bool& bad) {
#pragma unroll
    for (uint32_t q = 0; q < kMW; ++q) imask[32 * q + lane] = 0u;
    __syncwarp();
    if (T >= kDSub) {
        const uint32_t ts = sub / T * T;
        const uint32_t tend = ts + T < m ? ts + T : m;
        const uint32_t lim = (send < tend ? send : tend) - ts, lo_rel = sub - ts;
        uint32_t k = rb, lastx = 0;
        for (int round = 0;; ++round) {
            const uint32_t x = round == 0 ? xa : round == 1 ? xb
                                                           : (k + lane < e ? ldg_u16(D.body, k + lane) : 0xffffffffu);
            const bool in = k + lane < e && x < lim;
            const unsigned bal = __ballot_sync(0xffffffffu, in);
            const uint32_t prev = __shfl_up_sync(0xffffffffu, x, 1);
            if (bal & (bal + 1u)) bad = true;  // the in-range entries must be a prefix (sorted)
            if (in) {
                if (x < lo_rel || (lane > 0 && prev >= x) || (lane == 0 && k > rb && lastx >= x)) bad = true;
                else {
                    const uint32_t pos = ts + x - sub;
                    atomicOr(&imask[pos >> 5], 1u << (pos & 31));
                }
            }
            lastx = __shfl_sync(0xffffffffu, x, 31);
            const uint32_t n = __popc(bal);
            k += n;
            if (n < 32 || __any_sync(0xffffffffu, bad)) break;
        }
    } else {
        uint32_t k = rb;
        for (uint32_t t = sub / T; t * T < send; ++t) {
            const uint32_t ts = t * T;
            const uint32_t tl = m - ts < T ? m - ts : T;
            const uint32_t et = ldg_u32(D.toff + t + 1);
            if (et < k || et > D.count) {
                bad = true;
                break;
            }
            for (uint32_t b = k; b < et; b += 32) {
                const uint32_t kk = b + lane;
                if (kk < et) {
                    const uint32_t x = ldg_u16(D.body, kk);
                    if (x >= tl || (kk > k && ldg_u16(D.body, kk - 1) >= x)) bad = true;
                    else {
                        const uint32_t pos = ts + x - sub;
                        atomicOr(&imask[pos >> 5], 1u << (pos & 31));
                    }
                }
            }
            k = et;
        }
    }
    __syncwarp();
}

// Write one record's values into the tile at its mask bits; value k of the run is sv[k].
// kGlobal: sv points into the record (run longer than its window) -> batched gathers.
template <typename word_t, bool kGlobal>
__device__ __forceinline__ void expand_run(word_t* tw, const word_t* sv, const uint32_t (&mk)[kMW], uint32_t pre,
                                           uint32_t tot, int lane, uint32_t lt) {
    if (!kGlobal && tot <= kLaneSerialMax) {
        uint32_t k = pre;
#pragma unroll
        for (uint32_t q = 0; q < kMW; ++q) {
            uint32_t wv = mk[q];
            while (wv) {
                const uint32_t b = __ffs(wv) - 1;
                wv &= wv - 1;
                tw[32 * (kMW * lane + q) + b] = sv[k++];
            }
        }
        return;
    }
    uint32_t pk = pre;
#pragma unroll
    for (uint32_t q = 0; q < kMW; ++q) {
        uint32_t nz = __ballot_sync(0xffffffffu, mk[q] != 0);
        while (nz) {
            word_t v[4];
            uint32_t d[4];
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                d[i] = 0xffffffffu;
                if (nz) {  // warp-uniform
                    const int src = __ffs(nz) - 1;
                    nz &= nz - 1;
                    const uint32_t mb = __shfl_sync(0xffffffffu, mk[q], src);
                    const uint32_t o = __shfl_sync(0xffffffffu, pk, src);
                    if ((mb >> lane) & 1u) {
                        v[i] = kGlobal ? ldg_word(sv + o + __popc(mb & lt)) : sv[o + __popc(mb & lt)];
                        d[i] = 32 * (kMW * src + q) + lane;
                    }
                }
            }
#pragma unroll
            for (int i = 0; i < 4; ++i)
                if (d[i] != 0xffffffffu) tw[d[i]] = v[i];
        }
        pk += __popc(mk[q]);
    }
}

template <int W>
__device__ void fold_dense_unit(const FoldParams& P, uint64_t r, uint64_t ku, DenseSmem& S, int lane,
                                uint32_t& phase, bool& bad) {
    using word_t = typename Word<W>::T;
    const int N = P.nrec;
    const FoldRec& L = P.desc[r];
    const uint32_t m = L.m, T = L.T;
    const uint32_t U = T > kFoldWords ? T : kFoldWords;
    const uint32_t ustart = static_cast<uint32_t>(ku) * U;
    const uint32_t uend = ustart + U < m ? ustart + U : m;
    word_t* state = reinterpret_cast<word_t*>(P.state[L.seg]) + L.chunk_off;
    word_t* tw = reinterpret_cast<word_t*>(S.tile);
    uint8_t* sb = reinterpret_cast<uint8_t*>(S.stage);
    const uint32_t lt = (1u << lane) - 1u;

    for (int j = lane; j < N; j += 32) {  // running counts at the unit start, tile end, unit end
        const uint32_t* toff = S.rec[j].toff;
        S.carry[j] = ldg_u32(toff + ustart / T);
        S.tend[j] = ldg_u32(toff + ustart / T + 1);
        S.want[j] = uend < m ? ldg_u32(toff + uend / T) : ldg_u32(toff + (m + T - 1) / T);
    }

    for (uint32_t sub = ustart; sub < uend; sub += kDSub) {
        const uint32_t send = sub + kDSub < uend ? sub + kDSub : uend;
        const uint32_t nw = send - sub;
        const uint32_t bulk = nw * W & ~15u;  // 16-byte part of the sub-unit
        // 1. state -> tile: the previous sub-unit's bulk stores must have read the tile first
        bulk_wait_read();
        __syncwarp();
        if (lane == 0) {
            mbar_arrive_expect_tx(&S.bar, bulk);
            if (bulk) bulk_g2s(S.tile, state + sub, bulk, &S.bar);
            for (uint32_t i = bulk / W; i < nw; ++i) tw[i] = state[sub + i];
        }
        uint32_t uni[kMW];
#pragma unroll
        for (uint32_t q = 0; q < kMW; ++q) uni[q] = 0u;
        const uint32_t p0 = sub + 32 * kMW * lane;  // first word of this lane's mask words
        bool tile_ready = false;

        for (int j0 = 0; j0 < N; j0 += kDBatch) {
            const int nb = N - j0 < kDBatch ? N - j0 : kDBatch;
            uint32_t mk[kDBatch][kMW], pre[kDBatch], tot[kDBatch], rb[kDBatch], xa[kDBatch], xb[kDBatch];
            __syncwarp();  // carry / tend / want of this unit are written
            // 2. masks / position windows and value windows of the batch, all in flight together
#pragma unroll
            for (int jj = 0; jj < kDBatch; ++jj) {
#pragma unroll
                for (uint32_t q = 0; q < kMW; ++q) mk[jj][q] = 0u;
                xa[jj] = xb[jj] = 0xffffffffu;
                rb[jj] = 0;
                if (jj < nb) {
                    const DenseRec& D = S.rec[j0 + jj];
                    rb[jj] = S.carry[j0 + jj];
                    const uint32_t wb = window_bytes<W>(D.count, rb[jj]);
                    if (16u * lane < wb)
                        cp_async16(sb + jj * kWin + 16 * lane,
                                   D.values + ((static_cast<uint64_t>(rb[jj]) * W) & ~uint64_t(15)) + 16 * lane);
                    if (!D.is_idx) {
                        if (p0 < send) {
                            if constexpr (kMW == 4) {
                                const uint4 v = __ldg(reinterpret_cast<const uint4*>(D.body) + (p0 >> 7));
                                mk[jj][0] = v.x;
                                mk[jj][1] = v.y;
                                mk[jj][2] = v.z;
                                mk[jj][3] = v.w;
                            } else {
                                const uint2 v = __ldg(reinterpret_cast<const uint2*>(D.body) + (p0 >> 6));
                                mk[jj][0] = v.x;
                                mk[jj][1] = v.y;
                            }
                        }
                    } else if (T >= kDSub) {
                        const uint32_t e = S.tend[j0 + jj];
                        if (rb[jj] + lane < e) xa[jj] = ldg_u16(D.body, rb[jj] + lane);
                        if (rb[jj] + 32 + lane < e) xb[jj] = ldg_u16(D.body, rb[jj] + 32 + lane);
                    }
                }
            }
#pragma unroll
            for (int jj = 0; jj < kDBatch; ++jj) {
                if (jj < nb && S.rec[j0 + jj].is_idx) {
                    dense_index_build(S.rec[j0 + jj], T, m, sub, send, rb[jj], S.tend[j0 + jj], xa[jj], xb[jj],
                                      S.imask, lane, bad);
#pragma unroll
                    for (uint32_t q = 0; q < kMW; ++q) mk[jj][q] = S.imask[kMW * lane + q];
                    __syncwarp();
                }
            }
            // 3. value offsets; tile_off and bounds checks
#pragma unroll
            for (int jj = 0; jj < kDBatch; ++jj) {
                tot[jj] = 0;
                pre[jj] = 0;
                if (jj < nb) {
                    const DenseRec& D = S.rec[j0 + jj];
                    if (sub == ustart && ku == 0 && rb[jj] != 0) bad = true;
                    uint32_t c[kMW], ls = 0;
#pragma unroll
                    for (uint32_t q = 0; q < kMW; ++q) {
                        const uint32_t p = p0 + 32 * q;
                        if (p >= send) {
                            mk[jj][q] = 0u;  // past the chunk: mask padding
                        } else if (p + 32 > send) {  // the chunk's tail word: bits past m must be 0
                            const uint32_t vb = (1u << (send - p)) - 1u;
                            if (mk[jj][q] & ~vb) bad = true;
                            mk[jj][q] &= vb;
                        }
                        c[q] = __popc(mk[jj][q]);
                        ls += c[q];
                    }
                    uint32_t inc = ls;
#pragma unroll
                    for (int d = 1; d < 32; d <<= 1) {
                        const uint32_t t = __shfl_up_sync(0xffffffffu, inc, d);
                        if (lane >= d) inc += t;
                    }
                    pre[jj] = inc - ls;
                    tot[jj] = __shfl_sync(0xffffffffu, inc, 31);
                    if (T < kDSub) {
                        uint32_t q0 = pre[jj];
#pragma unroll
                        for (uint32_t q = 0; q < kMW; ++q) {
                            const uint32_t p = p0 + 32 * q;
                            if (p < send && p != ustart && (p & (T - 1)) == 0 && ldg_u32(D.toff + p / T) != rb[jj] + q0)
                                bad = true;
                            q0 += c[q];
                        }
                    }
                    const uint32_t run = rb[jj] + tot[jj];
                    if (run > D.count) {  // values past the record: corrupt, read nothing
                        bad = true;
                        tot[jj] = 0;
                    }
                    if (send == uend && (S.want[j0 + jj] != run || (uend == m && D.count != run)))
                        bad = true;  // unit end: the next unit's first entry, or the final entry
#pragma unroll
                    for (uint32_t q = 0; q < kMW; ++q) uni[q] |= mk[jj][q];
                }
            }
            __syncwarp();
#pragma unroll
            for (int jj = 0; jj < kDBatch; ++jj)
                if (jj < nb && lane == jj) S.carry[j0 + jj] = rb[jj] + tot[jj];
            // 4. expand oldest -> newest
            cp_async_wait_all();  // value windows
            if (!tile_ready) {
                mbar_wait_parity(&S.bar, phase);
                phase ^= 1u;
                tile_ready = true;
            }
            __syncwarp();
#pragma unroll
            for (int jj = 0; jj < kDBatch; ++jj) {
                if (jj < nb && tot[jj]) {
                    const DenseRec& D = S.rec[j0 + jj];
                    if (run_bytes<W>(rb[jj], tot[jj]) <= window_bytes<W>(D.count, rb[jj]))
                        expand_run<word_t, false>(
                            tw, reinterpret_cast<const word_t*>(sb + jj * kWin + ((rb[jj] * W) & 15u)), mk[jj], pre[jj],
                            tot[jj], lane, lt);
                    else
                        expand_run<word_t, true>(tw, reinterpret_cast<const word_t*>(D.values) + rb[jj], mk[jj],
                                                 pre[jj], tot[jj], lane, lt);
                }
                __syncwarp();
            }
        }
        // 5. write back this lane's touched lines: runs of consecutive touched lines, bulk stores
        fence_proxy_async_smem();  // the tile writes of every lane -> async proxy
        __syncwarp();
        const uint32_t lw0 = 32 * kMW * lane;  // this lane's first word in the sub-unit
        uint32_t q = 0;
        while (q < kMW) {
            if (!uni[q] || lw0 + 32 * q >= nw) {
                ++q;
                continue;
            }
            uint32_t qe = q + 1;
            while (qe < kMW && uni[qe] && lw0 + 32 * qe < nw) ++qe;
            const uint32_t w0 = lw0 + 32 * q;
            const uint32_t w1 = lw0 + 32 * qe < nw ? lw0 + 32 * qe : nw;
            const uint32_t bytes = (w1 - w0) * W;
            const uint32_t bb = bytes & ~15u;
            if (bb) bulk_s2g(state + sub + w0, tw + w0, bb);
            for (uint32_t i = w0 + bb / W; i < w1; ++i) state[sub + i] = tw[i];  // ragged chunk end
            q = qe;
        }
        bulk_commit();
    }
}

// Persistent: each CTA (= one warp) folds runs of kDenseRun consecutive units, the runs grid-
// strided over the CTAs.
__global__ void __launch_bounds__(kDenseThreads, kDenseBlocksPerSM) fold_dense_kernel(const __grid_constant__ FoldParams P) {
    __shared__ DenseSmem S;
    if (*reinterpret_cast<volatile unsigned*>(P.err) != 0) return;  // sticky error pending
    const int lane = threadIdx.x & 31;
    const int N = P.nrec;
    if (P.info[2] == 0) return;  // no dense chunk
    const uint64_t R = P.info[0];
    const uint64_t total = P.info[1];
    if (blockIdx.x * kDenseRun >= total) return;
    if (lane == 0) mbar_init(&S.bar, 1);
    __syncwarp();
    bool bad = false;
    uint32_t phase = 0;
    uint64_t cur = ~uint64_t(0);  // chunk whose record table is in S.rec
    uint64_t lo = 0, u1 = 0;
    for (uint64_t u = 0;; ++u) {
        if (u >= u1) {  // the next run of consecutive units
            const uint64_t run = u1 == 0 ? blockIdx.x : u1 / kDenseRun + gridDim.x - 1;
            if (run * kDenseRun >= total) break;
            u = run * kDenseRun;
            u1 = u + kDenseRun < total ? u + kDenseRun : total;
            uint64_t hi = R;
            lo = 0;
            while (hi - lo > 1) {
                const uint64_t mid = (lo + hi) >> 1;
                if (P.unit_first[mid] <= u) lo = mid; else hi = mid;
            }
        }
        while (u >= P.unit_first[lo + 1]) ++lo;
        if (P.desc[lo].dense != 1u) {  // folded by fold_kernel / fold_list_kernel: skip the chunk
            u = (P.unit_first[lo + 1] < u1 ? P.unit_first[lo + 1] : u1) - 1;
            continue;
        }
        if (lo != cur) {
            __syncwarp();
            for (int j = lane; j < N; j += 32) {
                const FoldRec& F = P.desc[static_cast<size_t>(j) * P.cap + lo];
                DenseRec D;
                D.body = F.idx ? F.idx : F.mask;
                D.values = F.values;
                D.toff = reinterpret_cast<const uint32_t*>(F.toff);
                D.count = static_cast<uint32_t>(F.count);
                D.is_idx = F.idx != nullptr;
                S.rec[j] = D;
            }
            __syncwarp();
            cur = lo;
        }
        const uint64_t ku = u - P.unit_first[lo];
        if (P.desc[lo].w == 4)
            fold_dense_unit<4>(P, lo, ku, S, lane, phase, bad);
        else
            fold_dense_unit<2>(P, lo, ku, S, lane, phase, bad);
        if (__any_sync(0xffffffffu, bad)) {
            if (lane == 0) tc_set_err(P.err, TC_ERR_CORRUPT);
            break;
        }
    }
    bulk_wait_all();  // the bulk stores are done before the CTA's shared memory goes away
}

// ---------------------------------------------------------------- list fold ----------
// Dense chains whose records are all index mode at T = kListT (the adaptive step's format): one
// unit = one tile, and record j's entries for tile t are [tile_off_j[t], tile_off_j[t+1]) — its
// positions and values are two contiguous runs.  A CTA of 4 warps per unit: one TMA bulk copy
// brings the tile's state into shared memory; the runs are staged with 16-byte cp.async copies
// (rounds that fill the stage with whole records; a record larger than the stage goes through
// in pieces) and scattered into the tile by position, oldest record first (a barrier between
// records: newest wins); touched 32-word lines go back with 16-byte stores (whole lines, no
// partial-sector writes).  Running counts carry from unit to unit within a run of consecutive
// units, and the next tile's end entries are loaded one unit ahead.
constexpr uint32_t kListThreads = 128;
constexpr uint32_t kListBlocksPerSM = 10;
constexpr uint32_t kListStage = 4096;

struct ListSmem {
    uint4 tile[kListT * 4 / 16];     // the unit's state (16 KB for fp32)
    uint4 stage[kListStage / 16];    // position / value runs of a round
    const uint8_t* pos[kListMaxRec];
    const uint8_t* val[kListMaxRec];
    const uint32_t* toff[kListMaxRec];
    uint32_t count[kListMaxRec];
    uint32_t carry[kListMaxRec];     // first entry of the tile, per record
    uint32_t tend[kListMaxRec];      // end entry of the tile, per record
    uint8_t touched[kListT / 32];    // per 32-word line: written
    uint32_t pb[kListMaxRec];        // per record: position-run bytes, total run bytes, stage offset
    uint32_t sz[kListMaxRec];
    uint32_t soff[kListMaxRec];
    uint32_t fits;                   // every record's runs fit the stage at once
    uint64_t bar;
};

// bytes of the 16-byte-aligned covers of the position run and the value run of entries [a, b)
template <int W>
__device__ __forceinline__ uint32_t list_run_bytes(uint32_t a, uint32_t b, uint32_t& pb) {
    if (b <= a) {
        pb = 0;
        return 0u;
    }
    pb = ((2u * b + 15u) & ~15u) - ((2u * a) & ~15u);
    return pb + static_cast<uint32_t>(((static_cast<uint64_t>(b) * W + 15) & ~uint64_t(15)) -
                                      (static_cast<uint64_t>(a) * W & ~uint64_t(15)));
}

template <int W>
__device__ __forceinline__ void list_unit(ListSmem& S, uint4* tile, uint64_t* bar, int N, uint32_t nw, uint8_t* st,
                                          uint32_t& phase, int tid,
                                          bool& bad) {
    using word_t = typename Word<W>::T;
    constexpr uint32_t kPiece = ((kListStage - 64) / (2 + W)) & ~7u;  // entries of a piece
    constexpr uint32_t kVec = 16 / W;
    word_t* tw = reinterpret_cast<word_t*>(tile);
    word_t* state = reinterpret_cast<word_t*>(st);
    uint8_t* sb = reinterpret_cast<uint8_t*>(S.stage);
    bool tile_ready = false;
    // the stage layout: each record's runs once (thread r), offsets by thread 0
    if (tid < N) {
        uint32_t pb;
        S.sz[tid] = list_run_bytes<W>(S.carry[tid], S.tend[tid], pb);
        S.pb[tid] = pb;
    }
    __syncthreads();
    if (tid == 0) {
        uint32_t o = 0;
        for (int r = 0; r < N; ++r) {
            S.soff[r] = o;
            o += S.sz[r];
        }
        S.fits = o <= kListStage;
    }
    __syncthreads();
    if (S.fits) {  // the common case: every run staged at once, then scattered record by record
        for (int r = 0; r < N; ++r) {
            const uint32_t sz = S.sz[r], pb = S.pb[r], off = S.soff[r], k0 = S.carry[r];
            const uint8_t* ps = S.pos[r] + ((2u * k0) & ~15u);
            const uint8_t* vs = S.val[r] + (static_cast<uint64_t>(k0) * W & ~uint64_t(15));
            for (uint32_t o = 16 * tid; o < sz; o += 16 * kListThreads)
                cp_async16(sb + off + o, o < pb ? ps + o : vs + (o - pb));
        }
        cp_async_wait_all();
        mbar_wait_parity(bar, phase);
        phase ^= 1u;
        __syncthreads();
        for (int r = 0; r < N; ++r) {
            const uint32_t k0 = S.carry[r], n = S.tend[r] - k0;
            if (n == 0) continue;  // CTA-uniform
            const uint16_t* px = reinterpret_cast<const uint16_t*>(sb + S.soff[r] + ((2u * k0) & 15u));
            const word_t* pv = reinterpret_cast<const word_t*>(sb + S.soff[r] + S.pb[r] + ((k0 * W) & 15u));
            for (uint32_t k = tid; k < n; k += kListThreads) {
                const uint32_t x = px[k];
                if (x >= nw || (k > 0 && px[k - 1] >= x)) {  // inside the tile, strictly increasing
                    bad = true;
                    continue;
                }
                tw[x] = pv[k];
                S.touched[x >> 5] = 1;
            }
            __syncthreads();  // this record's writes before the next (newer) record's
        }
        tile_ready = true;
    }
    int r = S.fits ? N : 0;
    uint32_t a = S.carry[0], lastx = 0;
    while (r < N) {  // runs larger than the stage: rounds, a record split into pieces if needed
        // one round, walked twice with the same (CTA-uniform) logic: copies, then scatter
        int r_end = r;
        uint32_t a_end = a;
        for (int pass = 0; pass < 2; ++pass) {
            int rr = r;
            uint32_t aa = a, used = 0, pb;
            while (rr < N) {
                const uint32_t k1 = S.tend[rr];
                uint32_t bb = k1;
                uint32_t sz = list_run_bytes<W>(aa, bb, pb);
                if (used + sz > kListStage) {
                    if (used) break;
                    bb = aa + kPiece;  // a piece of a record larger than the stage
                    sz = list_run_bytes<W>(aa, bb, pb);
                }
                if (pass == 0) {
                    const uint8_t* ps = S.pos[rr] + ((2u * aa) & ~15u);
                    const uint8_t* vs = S.val[rr] + (static_cast<uint64_t>(aa) * W & ~uint64_t(15));
                    for (uint32_t o = 16 * tid; o < pb; o += 16 * kListThreads) cp_async16(sb + used + o, ps + o);
                    for (uint32_t o = 16 * tid; o < sz - pb; o += 16 * kListThreads)
                        cp_async16(sb + used + pb + o, vs + o);
                } else {
                    const uint16_t* px = reinterpret_cast<const uint16_t*>(sb + used + ((2u * aa) & 15u));
                    const word_t* pv = reinterpret_cast<const word_t*>(sb + used + pb + ((aa * W) & 15u));
                    const uint32_t k0 = S.carry[rr];
                    for (uint32_t k = tid; k < bb - aa; k += kListThreads) {
                        const uint32_t x = px[k];
                        const uint32_t prev = k > 0 ? px[k - 1] : lastx;
                        if (x >= nw || (aa + k > k0 && prev >= x)) {  // inside the tile, strictly increasing
                            bad = true;
                            continue;
                        }
                        tw[x] = pv[k];
                        S.touched[x >> 5] = 1;
                    }
                    if (bb > aa) lastx = px[bb - aa - 1];
                    __syncthreads();  // this record's writes before the next (newer) record's
                }
                used += sz;
                if (bb < k1) {  // a piece: the round ends inside record rr
                    aa = bb;
                    break;
                }
                ++rr;
                if (rr < N) aa = S.carry[rr];
            }
            if (pass == 0) {
                r_end = rr;
                a_end = aa;
                cp_async_wait_all();
                if (!tile_ready) {
                    mbar_wait_parity(bar, phase);
                    phase ^= 1u;
                    tile_ready = true;
                }
                __syncthreads();
            }
        }
        __syncthreads();  // the stage is read before the next round's copies
        r = r_end;
        a = a_end;
    }
    if (!tile_ready) {
        mbar_wait_parity(bar, phase);
        phase ^= 1u;
        __syncthreads();
    }
    // touched lines back, 16 bytes per thread
    const uint32_t npieces = (nw + kVec - 1) / kVec;
    for (uint32_t q = tid; q < npieces; q += kListThreads) {
        const uint32_t wi = q * kVec;
        if (S.touched[wi >> 5]) {
            if (wi + kVec <= nw)
                *reinterpret_cast<uint4*>(state + wi) = tile[q];
            else
                for (uint32_t i = wi; i < nw; ++i) state[i] = tw[i];
        }
    }
    fence_proxy_async_smem();  // these tile reads precede the next bulk load into the tile
}

__global__ void __launch_bounds__(kListThreads, kListBlocksPerSM) fold_list_kernel(const __grid_constant__ FoldParams P) {
    __shared__ ListSmem S;
    if (*reinterpret_cast<volatile unsigned*>(P.err) != 0) return;  // sticky error pending
    if (P.info[4] == 0) return;                                       // no list chunk
    const int tid = threadIdx.x;
    const int N = P.nrec;
    const uint64_t R = P.info[0];
    const uint64_t total = P.info[1];
    if (blockIdx.x * kDenseRun >= total) return;
    if (tid == 0) mbar_init(&S.bar, 1);
    __syncthreads();
    bool bad = false;
    uint32_t phase = 0;
    uint64_t cur = ~uint64_t(0);
    uint32_t te = 0;  // thread j < N: record j's end entry of the next tile (prefetched)
    bool te_valid = false;
    uint64_t lo = 0, u1 = 0;
    for (uint64_t u = 0;; ++u) {
        if (u >= u1) {  // the next run of consecutive units
            const uint64_t run = u1 == 0 ? blockIdx.x : u1 / kDenseRun + gridDim.x - 1;
            if (run * kDenseRun >= total) break;
            u = run * kDenseRun;
            u1 = u + kDenseRun < total ? u + kDenseRun : total;
            uint64_t hi = R;
            lo = 0;
            while (hi - lo > 1) {
                const uint64_t mid = (lo + hi) >> 1;
                if (P.unit_first[mid] <= u) lo = mid; else hi = mid;
            }
            te_valid = false;
        }
        while (u >= P.unit_first[lo + 1]) ++lo;
        const FoldRec& L = P.desc[lo];
        if (L.dense != 2u) {  // folded by another kernel: skip the chunk
            u = (P.unit_first[lo + 1] < u1 ? P.unit_first[lo + 1] : u1) - 1;
            te_valid = false;
            continue;
        }
        if (lo != cur) {
            if (tid < N) {
                const FoldRec& F = P.desc[static_cast<size_t>(tid) * P.cap + lo];
                S.pos[tid] = F.idx;
                S.val[tid] = F.values;
                S.toff[tid] = reinterpret_cast<const uint32_t*>(F.toff);
                S.count[tid] = static_cast<uint32_t>(F.count);
            }
            cur = lo;
            te_valid = false;
        }
        const uint32_t ku = static_cast<uint32_t>(u - P.unit_first[lo]);
        const uint32_t m = L.m, w = L.w;
        const uint32_t nw = m - ku * kListT < kListT ? m - ku * kListT : kListT;
        uint8_t* st = P.state[L.seg] + (L.chunk_off + static_cast<uint64_t>(ku) * kListT) * w;
        // the tile (its previous contents were read by every thread before the last barrier)
        if (tid == 0) {
            const uint32_t bytes = nw * w, bulk = bytes & ~15u;
            mbar_arrive_expect_tx(&S.bar, bulk);
            if (bulk) bulk_g2s(S.tile, st, bulk, &S.bar);
            for (uint32_t i = bulk; i < bytes; ++i) reinterpret_cast<uint8_t*>(S.tile)[i] = st[i];
        }
        const bool next = u + 1 < u1 && u + 1 < P.unit_first[lo + 1];
        if (tid < kListT / 32) S.touched[tid] = 0;
        __syncthreads();  // the record table is in place
        if (tid < N) {  // this tile's entry range per record; the next tile's end, one unit ahead
            if (te_valid) {
                S.carry[tid] = S.tend[tid];
                S.tend[tid] = te;
            } else {
                S.carry[tid] = ldg_u32(S.toff[tid] + ku);
                S.tend[tid] = ldg_u32(S.toff[tid] + ku + 1);
            }
            const uint32_t k0 = S.carry[tid], k1 = S.tend[tid];
            if (k1 < k0 || k1 > S.count[tid] || (ku == 0 && k0 != 0) || ((ku + 1) * kListT >= m && k1 != S.count[tid]))
                bad = true;
        }
        if (next && tid < N) te = ldg_u32(S.toff[tid] + ku + 2);
        te_valid = next;
        if (__syncthreads_or(bad)) {  // a corrupt tile_off: drain the tile load, write nothing
            mbar_wait_parity(&S.bar, phase);
            phase ^= 1u;
            bad = true;
            break;
        }
        if (w == 4)
            list_unit<4>(S, S.tile, &S.bar, N, nw, st, phase, tid, bad);
        else
            list_unit<2>(S, S.tile, &S.bar, N, nw, st, phase, tid, bad);
        if (__syncthreads_or(bad)) {  // also: every thread is done with the tile
            bad = true;
            break;
        }
    }
    if (bad && tid == 0) tc_set_err(P.err, TC_ERR_CORRUPT);
}

// ------------------------------------------------------ mask-list fold (strategy 4) -------
// Chains of mask-mode records at T = 4096 (the adaptive format above ~6 % changed words), streamed
// like the list kernel: one CTA per 4096-word tile, the tile's state in shared memory by one bulk
// load, each record's value run for the tile ([tile_off[t], tile_off[t+1]) — contiguous) staged by
// 16-byte cp.async copies, in rounds of records newest first, as many as the stage holds (one
// record's whole run always fits).  Thread t owns mask word t of the tile (= 32-word line t): a
// record's winners on it are the bits no newer record set (cov), their values taken from the stage
// at the record's running count (a block scan of the mask words' popcounts), so records need no
// ordering barrier and each word is written once; every line a record touched goes back whole
// with 16-byte stores (no partial-sector writes).  The scatter fold of such chains pays a gather
// round trip per record and an L2 fill per partially written sector (cfg4, N = 8, f = 10 %: 39 ms).
// Checks: a record's popcount over the tile equals its tile_off difference, tile_off monotone,
// first 0, last = count, positions inside the tile.
constexpr uint32_t kMListThreads = 128;        // = the mask words of a 4096-word tile
constexpr uint32_t kMListStage = 16384 + 256;  // bytes: a whole fp32 run of one tile + alignment
constexpr int kMListBatch = 8;                 // records per round at most (their mask words in registers)
constexpr uint32_t kMListBlocksPerSM = 6;

struct MListSmem {
    uint4 tile[kListT * 4 / 16];
    uint4 stage[kMListStage / 16];
    const uint32_t* mask[kListMaxRec];
    const uint8_t* val[kListMaxRec];
    const uint32_t* toff[kListMaxRec];
    uint32_t count[kListMaxRec];
    uint32_t carry[kListMaxRec];   // first entry of the tile, per record
    uint32_t tend[kListMaxRec];    // end entry of the tile, per record
    uint32_t wtot[kMListBatch / 2][kMListThreads / 32];  // packed pairs of records
    uint8_t touched[kListT / 32];
    uint64_t bar;
};

template <int W, bool SMALLT>  // SMALLT: T < kListT (inner tile_off entries to check)
__device__ __forceinline__ void mlist_unit(MListSmem& S, int N, uint32_t nw, uint32_t ku, uint32_t T, uint8_t* st,
                                           uint32_t& phase, int tid, bool& bad) {
    using word_t = typename Word<W>::T;
    constexpr uint32_t kVec = 16 / W;
    word_t* tw = reinterpret_cast<word_t*>(S.tile);
    word_t* state = reinterpret_cast<word_t*>(st);
    uint8_t* sb = reinterpret_cast<uint8_t*>(S.stage);
    const int lane = tid & 31, wid = tid >> 5;
    const uint32_t nmw = (nw + 31) / 32;
    // this thread's line: the bits inside the tile
    const uint32_t lim = 32u * tid >= nw ? 0u : nw - 32u * tid >= 32u ? ~0u : (1u << (nw - 32u * tid)) - 1u;
    uint32_t cov = 0;  // bits of this thread's line set by a newer record
    bool tile_ready = false;
    for (int r = N - 1; r >= 0;) {
        // the round: records r, r-1, ... whose runs fit the stage together (CTA-uniform)
        int nb = 0;
        uint32_t used = 0, soff[kMListBatch];
#pragma unroll
        for (int q = 0; q < kMListBatch; ++q) {
            soff[q] = used;
            if (q == nb && r - q >= 0) {
                const uint32_t a = S.carry[r - q], b = S.tend[r - q];
                const uint32_t sz = b > a ? static_cast<uint32_t>(((static_cast<uint64_t>(b) * W + 15) & ~uint64_t(15)) -
                                                                  (static_cast<uint64_t>(a) * W & ~uint64_t(15)))
                                          : 0u;
                if (used + sz <= kMListStage) {
                    used += sz;
                    ++nb;
                }
            }
        }
        uint32_t mw[kMListBatch];
#pragma unroll
        for (int q = 0; q < kMListBatch; ++q)
            mw[q] = q < nb && tid < static_cast<int>(nmw) ? ldg_u32(S.mask[r - q] + static_cast<size_t>(ku) * 128 + tid) : 0u;
#pragma unroll
        for (int q = 0; q < kMListBatch; ++q) {
            if (q < nb) {
                const uint32_t a = S.carry[r - q], b = S.tend[r - q];
                if (b > a) {
                    const uint64_t lo = static_cast<uint64_t>(a) * W & ~uint64_t(15);
                    const uint64_t hi = (static_cast<uint64_t>(b) * W + 15) & ~uint64_t(15);
                    const uint8_t* src = S.val[r - q] + lo;
                    for (uint32_t o = 16 * tid; o < hi - lo; o += 16 * kMListThreads) cp_async16(sb + soff[q] + o, src + o);
                }
            }
        }
        // each record's running count before this thread's mask word: warp scans + warp totals
        // two records per scan: their counts packed in 16-bit halves (a tile's prefix <= 4096)
        uint32_t pre[kMListBatch];
#pragma unroll
        for (int q = 0; q < kMListBatch; q += 2) {
            const uint32_t c = __popc(mw[q]) | (__popc(mw[q + 1]) << 16);
            uint32_t inc = c;
#pragma unroll
            for (int d = 1; d < 32; d <<= 1) {
                const uint32_t y = __shfl_up_sync(0xffffffffu, inc, d);
                if (lane >= d) inc += y;
            }
            pre[q] = (inc - c) & 0xffffu;
            pre[q + 1] = (inc - c) >> 16;
            if (lane == 31) S.wtot[q / 2][wid] = inc;
        }
        cp_async_wait_all();
        if (!tile_ready) {
            mbar_wait_parity(&S.bar, phase);
            phase ^= 1u;
            tile_ready = true;
        }
        __syncthreads();  // the stage, the warp totals and the tile
#pragma unroll
        for (int q = 0; q < kMListBatch; ++q) {
            if (q < nb) {
                const int rr = r - q;
                uint32_t before = 0, tot = 0;  // (packed pair q & ~1: this record's half)
#pragma unroll
                for (int k = 0; k < static_cast<int>(kMListThreads / 32); ++k) {
                    const uint32_t x = S.wtot[q / 2][k];
                    before += k < wid ? x : 0u;
                    tot += x;
                }
                before = (q & 1) ? before >> 16 : before & 0xffffu;
                tot = (q & 1) ? tot >> 16 : tot & 0xffffu;
                const uint32_t a = S.carry[rr];
                // the mask must agree with tile_off, and set no bit past the chunk's last word; then
                // every rank below is < tot and every position inside the tile (no per-word test)
                if (tot != S.tend[rr] - a || (mw[q] & ~lim)) {  // (the stage holds tend - a values)
                    bad = true;
                    continue;
                }
                // T < kListT: the tile_off entries inside the unit must equal the running count at
                // their tile's first mask word (the unit's ends were checked by the caller)
                const uint32_t wpt = T / 32;  // mask words per tile
                if (SMALLT && tid > 0 && tid % wpt == 0 && tid < static_cast<int>(nmw) &&
                    ldg_u32(S.toff[rr] + ku * (kListT / T) + tid / wpt) != a + before + pre[q])
                    bad = true;
                const word_t* sv = reinterpret_cast<const word_t*>(sb + soff[q] + ((a * W) & 15u)) + before + pre[q];
                word_t* tl = tw + 32u * tid;
                const uint32_t mq = mw[q];
                uint32_t win = mq & ~cov;
                cov |= mq;
                if (__any_sync(0xffffffffu, __popc(win) >= 12)) {
                    // dense words: the winners in an order rotated by the lane (lane l takes bit
                    // (b' + l) & 31 for b' from 31 down), so the lanes of a warp touch 32 different
                    // banks — line t's word b sits in bank b; unrotated, a dense tile was a 32-way
                    // conflict on every store and stage read (cfg2, one 100 % record: 42.5 vs 12.4 ms)
                    win = __funnelshift_r(win, win, lane);
                    while (win) {
                        const int br = 31 - __clz(win);
                        win ^= 1u << br;
                        const int b = (br + lane) & 31;
                        tl[b] = sv[__popc(mq & ((1u << b) - 1u))];
                    }
                } else {
                    while (win) {  // highest bit first (FLO, no bit reversal)
                        const int b = 31 - __clz(win);
                        win ^= 1u << b;
                        tl[b] = sv[__popc(mq & ((1u << b) - 1u))];
                    }
                }
            }
        }
        __syncthreads();  // the stage and the warp totals are reused by the next round
        r -= nb;
    }
    S.touched[tid] = cov != 0u;
    __syncthreads();
    // touched lines back, 16 bytes per thread (consecutive threads, consecutive bytes)
    const uint32_t npieces = (nw + kVec - 1) / kVec;
    for (uint32_t q = tid; q < npieces; q += kMListThreads) {
        const uint32_t wi = q * kVec;
        if (S.touched[wi >> 5]) {
            if (wi + kVec <= nw)
                *reinterpret_cast<uint4*>(state + wi) = S.tile[q];
            else
                for (uint32_t i = wi; i < nw; ++i) state[i] = tw[i];
        }
    }
    fence_proxy_async_smem();  // these tile reads precede the next bulk load into the tile
}

// SMALLT: the chains at T < kListT (walker strategy 5; their fold unit holds several tiles) — a
// separate instantiation, so the default tile's kernel carries none of that code (2 % on cfg2)
template <bool SMALLT>
__global__ void __launch_bounds__(kMListThreads, kMListBlocksPerSM) fold_mlist_kernel(const __grid_constant__ FoldParams P) {
    __shared__ MListSmem S;
    if (*reinterpret_cast<volatile unsigned*>(P.err) != 0) return;  // sticky error pending
    if (P.info[SMALLT ? 7 : 6] == 0) return;                          // no mask-list chunk of this kind
    const int tid = threadIdx.x;
    const int N = P.nrec;
    const uint64_t R = P.info[0];
    const uint64_t total = P.info[1];
    if (blockIdx.x * kDenseRun >= total) return;
    if (tid == 0) mbar_init(&S.bar, 1);
    __syncthreads();
    bool bad = false;
    uint32_t phase = 0;
    uint64_t cur = ~uint64_t(0);
    uint32_t te = 0;  // thread j < N: record j's end entry of the next tile (prefetched)
    bool te_valid = false;
    uint64_t lo = 0, u1 = 0;
    for (uint64_t u = 0;; ++u) {
        if (u >= u1) {  // the next run of consecutive units
            const uint64_t run = u1 == 0 ? blockIdx.x : u1 / kDenseRun + gridDim.x - 1;
            if (run * kDenseRun >= total) break;
            u = run * kDenseRun;
            u1 = u + kDenseRun < total ? u + kDenseRun : total;
            uint64_t hi = R;
            lo = 0;
            while (hi - lo > 1) {
                const uint64_t mid = (lo + hi) >> 1;
                if (P.unit_first[mid] <= u) lo = mid; else hi = mid;
            }
            te_valid = false;
        }
        while (u >= P.unit_first[lo + 1]) ++lo;
        const FoldRec& L = P.desc[lo];
        if (L.dense != (SMALLT ? 5u : 4u)) {  // folded by another kernel: skip the chunk
            u = (P.unit_first[lo + 1] < u1 ? P.unit_first[lo + 1] : u1) - 1;
            te_valid = false;
            continue;
        }
        if (lo != cur) {
            if (tid < N) {
                const FoldRec& F = P.desc[static_cast<size_t>(tid) * P.cap + lo];
                S.mask[tid] = reinterpret_cast<const uint32_t*>(F.mask);
                S.val[tid] = F.values;
                S.toff[tid] = reinterpret_cast<const uint32_t*>(F.toff);
                S.count[tid] = static_cast<uint32_t>(F.count);
            }
            cur = lo;
            te_valid = false;
        }
        const uint32_t ku = static_cast<uint32_t>(u - P.unit_first[lo]);
        const uint32_t m = L.m, w = L.w;
        const uint32_t nw = m - ku * kListT < kListT ? m - ku * kListT : kListT;
        uint8_t* st = P.state[L.seg] + (L.chunk_off + static_cast<uint64_t>(ku) * kListT) * w;
        // the tile (its previous contents were read by every thread before the last barrier)
        if (tid == 0) {
            const uint32_t bytes = nw * w, bulk = bytes & ~15u;
            mbar_arrive_expect_tx(&S.bar, bulk);
            if (bulk) bulk_g2s(S.tile, st, bulk, &S.bar);
            for (uint32_t i = bulk; i < bytes; ++i) reinterpret_cast<uint8_t*>(S.tile)[i] = st[i];
        }
        const bool next = u + 1 < u1 && u + 1 < P.unit_first[lo + 1];
        __syncthreads();  // the record table is in place
        // the unit's tile_off entries: a unit of kListT words holds tpu = kListT / T tiles (T <= kListT)
        uint32_t t0 = ku, t1 = ku + 1, t2 = ku + 2;
        if (SMALLT) {
            const uint32_t lt = __ffs(L.T) - 1;  // T is a power of two: shifts, not divisions
            const uint32_t tpu = kListT >> lt, n_tiles = (m + L.T - 1) >> lt;
            t0 = ku * tpu;
            t1 = t0 + tpu < n_tiles ? t0 + tpu : n_tiles;
            t2 = t1 + tpu < n_tiles ? t1 + tpu : n_tiles;
        }
        if (tid < N) {  // this unit's entry range per record; the next unit's end, one unit ahead
            if (te_valid) {
                S.carry[tid] = S.tend[tid];
                S.tend[tid] = te;
            } else {
                S.carry[tid] = ldg_u32(S.toff[tid] + t0);
                S.tend[tid] = ldg_u32(S.toff[tid] + t1);
            }
            const uint32_t k0 = S.carry[tid], k1 = S.tend[tid];
            if (k1 < k0 || k1 - k0 > nw || k1 > S.count[tid] || (ku == 0 && k0 != 0) ||
                ((ku + 1) * kListT >= m && k1 != S.count[tid]))
                bad = true;
        }
        if (next && tid < N) te = ldg_u32(S.toff[tid] + t2);
        te_valid = next;
        if (__syncthreads_or(bad)) {  // a corrupt tile_off: drain the tile load, write nothing
            mbar_wait_parity(&S.bar, phase);
            phase ^= 1u;
            bad = true;
            break;
        }
        if (w == 4)
            mlist_unit<4, SMALLT>(S, N, nw, ku, L.T, st, phase, tid, bad);
        else
            mlist_unit<2, SMALLT>(S, N, nw, ku, L.T, st, phase, tid, bad);
        if (__syncthreads_or(bad)) {  // also: every thread is done with the tile
            bad = true;
            break;
        }
    }
    if (bad && tid == 0) tc_set_err(P.err, TC_ERR_CORRUPT);
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
    e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    static int occ_d = 0;
    if (!occ_d) {
        if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ_d, fold_dense_kernel, kDenseThreads, 0) != cudaSuccess ||
            occ_d < 1)
            occ_d = 1;
    }
    fold_dense_kernel<<<num_sms * occ_d, kDenseThreads, 0, s>>>(p);
    e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    static int occ_l = 0;
    if (!occ_l) {
        if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ_l, fold_list_kernel, kListThreads, 0) != cudaSuccess ||
            occ_l < 1)
            occ_l = 1;
    }
    fold_list_kernel<<<num_sms * occ_l, kListThreads, 0, s>>>(p);
    e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    static int occ_e = 0;
    if (!occ_e) {
        if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ_e, fold_entries_kernel, kFoldThreads, 0) != cudaSuccess ||
            occ_e < 1)
            occ_e = 4;
    }
    static int occ_m = 0;
    if (!occ_m) {
        if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ_m, fold_mlist_kernel<false>, kMListThreads, 0) !=
                cudaSuccess ||
            occ_m < 1)
            occ_m = 1;
    }
    fold_mlist_kernel<false><<<num_sms * occ_m, kMListThreads, 0, s>>>(p);
    e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    fold_mlist_kernel<true><<<num_sms * occ_m, kMListThreads, 0, s>>>(p);
    e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    for (int j = 0; j < p.nrec; ++j) {  // each returns at once when no chunk takes strategy 3
        fold_entries_kernel<<<num_sms * occ_e, kFoldThreads, 0, s>>>(p, j);
        e = cudaGetLastError();
        if (e != cudaSuccess) return e;
    }
    *launches += 6 + static_cast<uint64_t>(p.nrec);
    return cudaGetLastError();
}

}  // namespace tc
