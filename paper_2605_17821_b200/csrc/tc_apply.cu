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
//   fold_kernel       (persistent, 6 CTAs/SM) per unit of up to 8192 words: one thread per
//                              mask word; per group of 4 records a packed 4x16-bit block scan
//                              gives every record's in-unit value offsets; newest-first winner
//                              masks carried in registers; winning (word, record, value index)
//                              triples are compacted into a shared-memory list and then
//                              gathered/scattered by consecutive threads (coalesced-ish reads
//                              of values, ordered writes of state).  Tile-offset consistency is
//                              checked on the way (-> CORRUPT).
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
                if (magic != 0x31444354u || fmt != 1 || (w != 2 && w != 4) || flags != 1 ||
                    !is_pow2(T) || T < 32 || T > 65536 || seg != static_cast<uint32_t>(s) || w != P.w[s] ||
                    coff != off || coff % T != 0 || m > kMaxChunkWords || count > m ||
                    (m == 0 && P.n[s] != 0) || off + m > P.n[s] || total != record_bytes(m, T, w, count) ||
                    total > bytes - pos) {
                    err = TC_ERR_CORRUPT;
                    break;
                }
                if (r >= P.cap) { err = TC_ERR_CAPACITY; break; }
                FoldRec R;
                R.mask = h + kHdrBytes;
                R.toff = R.mask + pad16(4 * cdiv(m, 32));
                R.values = h + record_fixed_bytes(m, T);
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
constexpr int kWarps = kFoldThreads / 32;

template <int W>
struct Word;
template <>
struct Word<4> { using T = uint32_t; };
template <>
struct Word<2> { using T = uint16_t; };

struct FoldSmem {
    uint32_t list[kFoldWords];                     // packed (off:13 | j:6 | lv:13)
    unsigned long long wsum[2][kWarps];            // per-warp packed scan totals (double-buffered)
    uint32_t run[TC_MAX_FOLD];                     // in-chunk count at the current sub-step start
    uint32_t add[TC_MAX_FOLD];                     // this sub-step's popcount per record
    uint32_t cnt;                                  // list length
    uint32_t bad;
};

template <int W>
__device__ void fold_unit(const FoldParams& P, FoldSmem& sm, uint64_t r, uint64_t ku) {
    using word_t = typename Word<W>::T;
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    const int N = P.nrec;
    const FoldRec& L = P.desc[r];  // layout (shared by every diff)
    const uint32_t m = L.m, T = L.T;
    const uint64_t U = T > kFoldWords ? T : kFoldWords;
    const uint32_t ustart = static_cast<uint32_t>(ku * U);
    const uint32_t uend = static_cast<uint32_t>(ustart + U < m ? ustart + U : m);
    word_t* state = reinterpret_cast<word_t*>(P.state[L.seg]) + L.chunk_off;

    if (tid < N) {
        const FoldRec& R = P.desc[static_cast<size_t>(tid) * P.cap + r];
        const uint32_t base = reinterpret_cast<const uint32_t*>(R.toff)[ustart / T];
        sm.run[tid] = base;
        if (ku == 0 && base != 0) atomicExch(&sm.bad, 1u);
    }
    if (tid == 0) sm.cnt = 0;
    __syncthreads();

    for (uint32_t sub = ustart; sub < uend; sub += kFoldWords) {
        const uint32_t send = sub + kFoldWords < uend ? sub + kFoldWords : uend;
        const uint32_t p = sub + 32u * tid;  // first word of this thread's mask word
        const bool valid = p < send;
        const uint32_t validbits = !valid ? 0u : (send - p >= 32 ? 0xffffffffu : ((1u << (send - p)) - 1u));
        uint32_t rem = 0xffffffffu;
        int gi = 0;
        for (int g = N - 1; g >= 0; g -= 4, ++gi) {
            uint32_t mk[4];
            const FoldRec* Rq[4];
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const int j = g - q;
                mk[q] = 0;
                Rq[q] = nullptr;
                if (j >= 0) {
                    Rq[q] = &P.desc[static_cast<size_t>(j) * P.cap + r];
                    if (valid) {
                        const uint32_t raw = reinterpret_cast<const uint32_t*>(Rq[q]->mask)[p >> 5];
                        if (raw & ~validbits & (p + 32 > m ? 0xffffffffu : 0u)) atomicExch(&sm.bad, 1u);  // tail bits
                        mk[q] = raw & validbits;
                    }
                }
            }
            // packed 4 x 16-bit block-wide exclusive scan of the popcounts
            const unsigned long long pk = static_cast<unsigned long long>(__popc(mk[0])) |
                                          (static_cast<unsigned long long>(__popc(mk[1])) << 16) |
                                          (static_cast<unsigned long long>(__popc(mk[2])) << 32) |
                                          (static_cast<unsigned long long>(__popc(mk[3])) << 48);
            unsigned long long x = pk;
#pragma unroll
            for (int d = 1; d < 32; d <<= 1) {
                const unsigned long long y = __shfl_up_sync(0xffffffffu, x, d);
                if (lane >= d) x += y;
            }
            if (lane == 31) sm.wsum[gi & 1][wid] = x;
            __syncthreads();
            unsigned long long wpre = 0, tot = 0;
#pragma unroll
            for (int k = 0; k < kWarps; ++k) {
                const unsigned long long v = sm.wsum[gi & 1][k];
                wpre += k < wid ? v : 0ull;
                tot += v;
            }
            const unsigned long long ex = x - pk + wpre;
            // tile_off consistency at tile starts inside the sub-step
            if (valid && (p & (T - 1)) == 0 && p != ustart) {
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    if (!Rq[q]) continue;
                    const uint32_t want = sm.run[g - q] + static_cast<uint32_t>((ex >> (16 * q)) & 0xffffu);
                    if (reinterpret_cast<const uint32_t*>(Rq[q]->toff)[p / T] != want) atomicExch(&sm.bad, 1u);
                }
            }
            if (tid < 4 && g - tid >= 0) sm.add[g - tid] = static_cast<uint32_t>((tot >> (16 * tid)) & 0xffffu);
            // newest-first winners, compacted into the list
            uint32_t win[4];
            uint32_t e = 0;
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                win[q] = mk[q] & rem;
                rem &= ~mk[q];
                e += __popc(win[q]);
            }
            uint32_t ei = e;
#pragma unroll
            for (int d = 1; d < 32; d <<= 1) {
                const uint32_t y = __shfl_up_sync(0xffffffffu, ei, d);
                if (lane >= d) ei += y;
            }
            uint32_t wbase = 0;
            if (lane == 31 && ei) wbase = atomicAdd(&sm.cnt, ei);
            wbase = __shfl_sync(0xffffffffu, wbase, 31);
            uint32_t pos = wbase + ei - e;
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                uint32_t wq = win[q];
                const uint32_t exq = static_cast<uint32_t>((ex >> (16 * q)) & 0xffffu);
                while (wq) {
                    const uint32_t b = __ffs(wq) - 1;
                    wq &= wq - 1;
                    const uint32_t lv = exq + __popc(mk[q] & ((1u << b) - 1u));
                    sm.list[pos++] = (32u * tid + b) | (static_cast<uint32_t>(g - q) << 13) | (lv << 19);
                }
            }
        }
        __syncthreads();
        // gather winning values, scatter into the state (ordered by word within each warp)
        const uint32_t n = sm.cnt;
        const bool ok = sm.bad == 0;
        for (uint32_t e = tid; e < n && ok; e += kFoldThreads) {
            const uint32_t ent = sm.list[e];
            const uint32_t off = ent & 0x1fffu;
            const uint32_t j = (ent >> 13) & 0x3fu;
            const uint32_t lv = ent >> 19;
            const FoldRec& R = P.desc[static_cast<size_t>(j) * P.cap + r];
            const uint64_t idx = static_cast<uint64_t>(sm.run[j]) + lv;
            if (idx >= R.count) {
                atomicExch(&sm.bad, 1u);
                continue;
            }
            state[sub + off] = reinterpret_cast<const word_t*>(R.values)[idx];
        }
        __syncthreads();
        if (tid < N) sm.run[tid] += sm.add[tid];
        if (tid == 0) sm.cnt = 0;
        __syncthreads();
    }
    // end-of-unit check: the entry at uend (next unit's start) or the final entry == count
    if (tid < N) {
        const FoldRec& R = P.desc[static_cast<size_t>(tid) * P.cap + r];
        const uint32_t* toff = reinterpret_cast<const uint32_t*>(R.toff);
        if (uend < m) {
            if (toff[uend / T] != sm.run[tid]) atomicExch(&sm.bad, 1u);
        } else {
            if (toff[cdiv(m, T)] != sm.run[tid] || R.count != sm.run[tid]) atomicExch(&sm.bad, 1u);
        }
    }
    __syncthreads();
}

__global__ void __launch_bounds__(kFoldThreads, 5) fold_kernel(const __grid_constant__ FoldParams P) {
    __shared__ FoldSmem sm;
    if (*reinterpret_cast<volatile unsigned*>(P.err) != 0) return;  // sticky error pending
    const uint64_t R = P.info[0];
    const uint64_t total = P.info[1];
    if (threadIdx.x == 0) sm.bad = 0;
    __syncthreads();
    for (uint64_t u = blockIdx.x; u < total; u += gridDim.x) {
        // record r: unit_first[r] <= u < unit_first[r+1]
        uint64_t lo = 0, hi = R;
        while (hi - lo > 1) {
            const uint64_t mid = (lo + hi) >> 1;
            if (P.unit_first[mid] <= u) lo = mid; else hi = mid;
        }
        const uint64_t r = lo;
        const uint64_t ku = u - P.unit_first[r];
        if (P.desc[r].w == 4)
            fold_unit<4>(P, sm, r, ku);
        else
            fold_unit<2>(P, sm, r, ku);
        if (sm.bad) {
            if (threadIdx.x == 0) tc_set_err(P.err, TC_ERR_CORRUPT);
            return;
        }
    }
}

}  // namespace

cudaError_t launch_fold(const FoldParams& p, cudaStream_t s, int num_sms, uint64_t* launches) {
    fold_walk_kernel<<<1, TC_MAX_FOLD, 0, s>>>(p);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    fold_kernel<<<num_sms * 5, kFoldThreads, 0, s>>>(p);
    *launches += 2;
    return cudaGetLastError();
}

}  // namespace tc
