// tc_grad.cu — the paper's own differential on sm_100a: adaptive gradient compression (INT8
// dense below the small-tensor threshold; sampled magnitude threshold + one keeping pass into
// FP16 values / INT32 chunk-local indices above it), decompression, the native Adam step, and
// the fused multi-step Adam replay (include/tc_grad.h).
//
// PAPER.md:203 §3.2 (codec), §3.3 + P:322 §4 (fused replay)
// (Adam), SPEC.md:99-157 (codec interface), SPEC.md:343-354 (fused == sequential).  Every fp32
// operation of the Adam update is an explicit round-to-nearest intrinsic, in the order the oracle
// (oracle/tco_grad.c, built with -ffp-contract=off) writes it, so the two agree bit for bit.
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <cmath>
#include <string>

#include "../../include/tc_grad.h"
#include "tc_internal.h"
#include "tc_ptx.cuh"

using tc::bulk_g2s;
using tc::mbar_arrive_expect_tx;
using tc::mbar_init;
using tc::mbar_wait_parity;

namespace {

constexpr uint32_t kGB = 4096;         // elements per compaction block / replay tile
constexpr uint32_t kGThreads = 256;    // 16 elements per thread
constexpr uint32_t kGSpill = 256;      // entries a block keeps in its spill slot (6 bytes each)
constexpr uint32_t kSampleMax = 8192;  // largest supported sample (sorted in shared memory)
constexpr uint64_t kDefaultChunk = (1ull << 31) - 4096;
constexpr uint64_t kHdr = 64;

tc_status fail(tc_status s, const std::string& msg) {
    tc::set_error(msg);
    return s;
}
tc_status cuda_fail(cudaError_t e, const char* what) {
    tc::set_error(std::string(what) + ": " + cudaGetErrorString(e));
    return e == cudaErrorMemoryAllocation ? TC_ERR_NOMEM : TC_ERR_CUDA;
}
bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }
__host__ __device__ inline uint64_t pad16u(uint64_t x) { return (x + 15) & ~uint64_t(15); }

struct Opts {
    uint64_t small, chunk;
    uint32_t sample, rank;
};

tc_status resolve(const tc_grad_opts* o, Opts* r) {
    const uint64_t small = o && o->small_threshold ? o->small_threshold : 100000;
    const double k = o && o->k > 0 ? o->k : 0.01;
    const uint32_t sample = o && o->sample_size ? o->sample_size : 4096;
    const uint64_t chunk = o && o->chunk_elems ? o->chunk_elems : kDefaultChunk;
    if (!(k > 0.0 && k <= 1.0)) return fail(TC_ERR_INVALID, "k must be in (0, 1]");
    if (sample > kSampleMax) return fail(TC_ERR_INVALID, "sample_size must be <= 8192");
    if (chunk % kGB != 0 || chunk > 2147483647ull) return fail(TC_ERR_INVALID, "chunk_elems: a multiple of 4096, < 2^31");
    double t = std::ceil((1.0 - k) * static_cast<double>(sample));
    uint32_t rank = t < 1.0 ? 1u : (t > sample ? sample : static_cast<uint32_t>(t));
    *r = {small, chunk, sample, rank};
    return TC_OK;
}

uint64_t bound_of(uint64_t n, const Opts& o) {
    if (n < o.small) return kHdr + pad16u(n);
    const uint64_t chunks = n ? (n + o.chunk - 1) / o.chunk : 1;
    return kHdr + 16 * chunks + pad16u(2 * n) + pad16u(4 * n);
}

// programmatic dependent launch (sm_90+): a primary lets its dependents start; a dependent waits for
// its primary's completion and memory (a no-op when launched without the attribute)
__device__ __forceinline__ void pdl_launch_dependents() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
template <typename K, typename A>
cudaError_t launch_pdl(K kernel, unsigned grid, unsigned block, cudaStream_t s, const A& arg) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(block);
    cfg.dynamicSmemBytes = 0;
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kernel, arg);
}

__device__ __forceinline__ uint64_t splitmix64(uint64_t z) {
    z += 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

__device__ __forceinline__ void put_header(uint8_t* out, uint32_t variant, uint32_t chunks, float s, uint64_t n,
                                           uint64_t kept, uint64_t chunk, uint64_t seed, uint64_t total) {
    uint64_t* h = reinterpret_cast<uint64_t*>(out);
    h[0] = 0x31474354ull /* "TCG1" */ | (static_cast<uint64_t>(variant) << 32);
    h[1] = static_cast<uint64_t>(chunks) | (static_cast<uint64_t>(__float_as_uint(s)) << 32);
    h[2] = n;
    h[3] = kept;
    h[4] = chunk;
    h[5] = seed;
    h[6] = total;
    h[7] = 0;
}

// ------------------------------------------------------------------ INT8 dense ----------
__global__ void __launch_bounds__(1024) grad_int8_kernel(const float* __restrict__ x, uint64_t n, uint64_t chunk,
                                                         uint64_t seed, uint8_t* out, uint64_t cap,
                                                         uint64_t* out_bytes, unsigned* err) {
    __shared__ float s_max[32];
    const int tid = threadIdx.x;
    float mx = 0.0f;
    for (uint64_t i = tid; i < n; i += 1024) mx = fmaxf(mx, fabsf(x[i]));
#pragma unroll
    for (int d = 16; d >= 1; d >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, d));
    if ((tid & 31) == 0) s_max[tid >> 5] = mx;
    __syncthreads();
    mx = 0.0f;
    for (int k = 0; k < 32; ++k) mx = fmaxf(mx, s_max[k]);
    const float scale = mx > 0.0f ? __fdiv_rn(mx, 127.0f) : 1.0f;
    const uint64_t total = kHdr + pad16u(n);
    if (tid == 0) *reinterpret_cast<volatile uint64_t*>(out_bytes) = total;
    if (total > cap) {
        if (tid == 0) tc_set_err(err, TC_ERR_CAPACITY);
        return;
    }
    if (tid == 0) put_header(out, 1, 0, scale, n, n, chunk, seed, total);
    int8_t* q = reinterpret_cast<int8_t*>(out + kHdr);
    for (uint64_t i = tid; i < pad16u(n); i += 1024) {
        float r = 0.0f;
        if (i < n) r = fminf(fmaxf(rintf(__fdiv_rn(x[i], scale)), -127.0f), 127.0f);
        q[i] = static_cast<int8_t>(r);
    }
}

// ----------------------------------------------------------------- sparse form ----------
struct SparseParams {
    const float* x;
    uint64_t n, chunk, nblocks, nchunks, seed, cap;
    uint32_t sample, rank;
    uint8_t* out;
    uint64_t* out_bytes;
    float* thr;                  // [1]
    uint32_t* bcount;            // [nblocks] kept | dense flag
    unsigned long long* gsum;    // [ngroups] kept per group of kGGroup blocks (zeroed per call)
    unsigned long long* gpre;    // [ngroups + 1] exclusive prefix of gsum; [ngroups] = kept
    unsigned long long* cstart;  // [nchunks + 1] first entry of each chunk
    uint8_t* spill;              // [nblocks][kGSpill * 6]: f16 values | i32 local indices
    uint64_t ngroups;
    unsigned* err;
};
constexpr uint32_t kGGroup = 256;  // blocks per emit CTA (a thread per block)
constexpr uint32_t kDenseBit = 0x80000000u;

// the threshold: rank-th smallest magnitude of `sample` seeded draws.  A radix select over the
// magnitudes' bits (non-negative floats order as their bit patterns): four 8-bit passes, each a
// shared-memory histogram of the candidates that share the bits chosen so far and one warp's scan
// for the bin holding the rank — 12 barriers instead of a bitonic sort's 91 (the same value: the
// rank-th order statistic is unique).
__global__ void __launch_bounds__(1024) grad_sample_kernel(const __grid_constant__ SparseParams P) {
    constexpr int kPer = kSampleMax / 1024;
    __shared__ uint32_t hist[256];
    __shared__ uint32_t s_bits, s_rank;
    const int tid = threadIdx.x, lane = tid & 31;
    pdl_launch_dependents();  // the counting pass may start loading its tiles now
    uint32_t v[kPer];
#pragma unroll
    for (int j = 0; j < kPer; ++j) {
        const uint32_t i = static_cast<uint32_t>(tid) + 1024u * j;
        v[j] = i < P.sample ? __float_as_uint(fabsf(P.x[splitmix64(P.seed + i) % P.n])) : 0u;
    }
    if (tid == 0) {
        s_bits = 0;
        s_rank = P.rank;  // 1-based
    }
#pragma unroll 1
    for (int shift = 24; shift >= 0; shift -= 8) {
        if (tid < 256) hist[tid] = 0;
        __syncthreads();
        const uint32_t hi = shift == 24 ? 0u : ~0u << (shift + 8);
        const uint32_t want = s_bits & hi;
#pragma unroll
        for (int j = 0; j < kPer; ++j) {
            const uint32_t i = static_cast<uint32_t>(tid) + 1024u * j;
            if (i < P.sample && (v[j] & hi) == want) atomicAdd(&hist[(v[j] >> shift) & 255u], 1u);
        }
        __syncthreads();
        if (tid < 32) {
            uint32_t h[8], c = 0;
#pragma unroll
            for (int k = 0; k < 8; ++k) {
                h[k] = hist[lane * 8 + k];
                c += h[k];
            }
            uint32_t inc = c;
#pragma unroll
            for (int d = 1; d < 32; d <<= 1) {
                const uint32_t t = __shfl_up_sync(0xffffffffu, inc, d);
                if (lane >= d) inc += t;
            }
            const uint32_t r = s_rank;
            const uint32_t before = inc - c;
            if (before < r && r <= inc) {  // the bin holding the rank is in this lane's 8
                uint32_t acc = before;
#pragma unroll
                for (int k = 0; k < 8; ++k) {
                    if (acc < r && r <= acc + h[k]) {
                        s_bits |= static_cast<uint32_t>(lane * 8 + k) << shift;
                        s_rank = r - acc;
                    }
                    acc += h[k];
                }
            }
        }
        __syncthreads();
    }
    if (tid == 0) *P.thr = __uint_as_float(s_bits);
}

// the keeping predicate: |x| >= threshold, zeros never kept
__device__ __forceinline__ bool keep(float v, float thr) { return v != 0.0f && fabsf(v) >= thr; }

// the 16 flags of one thread's elements [i0, i0 + 16) (4 x 16-byte loads; elements past n are 0)
__device__ __forceinline__ uint32_t flags16(const float* x, uint64_t n, uint64_t i0, float thr, float (&v)[16]) {
    if (i0 + 16 <= n) {
        const float4* p = reinterpret_cast<const float4*>(x + i0);
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const float4 f = __ldg(p + q);
            v[4 * q] = f.x;
            v[4 * q + 1] = f.y;
            v[4 * q + 2] = f.z;
            v[4 * q + 3] = f.w;
        }
    } else {
#pragma unroll
        for (int e = 0; e < 16; ++e) v[e] = i0 + e < n ? x[i0 + e] : 0.0f;
    }
    uint32_t f = 0;
#pragma unroll
    for (int e = 0; e < 16; ++e) f |= keep(v[e], thr) ? (1u << e) : 0u;
    return f;
}

// pass 1: thread t of block b takes elements [b*kGB + 16t, +16): per-thread counts, a block scan
// in index order, the group sums; sparse blocks pack their entries into the spill slot.  Lean on
// instructions (r2 ncu: the pass issued on 65 % of cycles at 4.2 TB/s): a positive threshold makes
// the keep test one magnitude compare (|x| >= thr > 0 excludes zeros), the 16 values go to shared
// memory once so a thread with kept entries walks only its set bits, and the chunk-local index
// comes from the block's chunk base (a block never straddles chunks), not a 64-bit division
__global__ void __launch_bounds__(kGThreads) grad_count_kernel(const __grid_constant__ SparseParams P) {
    __shared__ uint32_t s_warp[kGThreads / 32];
    __shared__ __align__(16) float s_v[kGThreads * 16];
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    const uint64_t b = blockIdx.x;
    const uint64_t i0 = b * kGB + 16ull * tid;
    float v[16];
    uint32_t f = 0;
    if (i0 + 16 <= P.n) {
        const float4* p = reinterpret_cast<const float4*>(P.x + i0);
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const float4 x = __ldg(p + q);
            v[4 * q] = x.x;
            v[4 * q + 1] = x.y;
            v[4 * q + 2] = x.z;
            v[4 * q + 3] = x.w;
        }
    } else {
#pragma unroll
        for (int e = 0; e < 16; ++e) v[e] = i0 + e < P.n ? P.x[i0 + e] : 0.0f;
    }
    // programmatic dependent launch: the first CTAs started while the sample kernel ran, their
    // tiles in flight; the threshold is read once that kernel has completed
    pdl_wait();
    const float thr = *P.thr;
    if (thr > 0.0f) {
#pragma unroll
        for (int e = 0; e < 16; ++e) f |= fabsf(v[e]) >= thr ? (1u << e) : 0u;
    } else {
#pragma unroll
        for (int e = 0; e < 16; ++e) f |= keep(v[e], thr) ? (1u << e) : 0u;
    }
    const uint32_t c = __popc(f);
    uint32_t inc = c;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, inc, d);
        if (lane >= d) inc += y;
    }
    if (lane == 31) s_warp[wid] = inc;
    __syncthreads();
    uint32_t wp = 0, total = 0;
#pragma unroll
    for (int k = 0; k < static_cast<int>(kGThreads / 32); ++k) {
        wp += k < wid ? s_warp[k] : 0u;
        total += s_warp[k];
    }
    if (tid == 0) {
        P.bcount[b] = total | (total > kGSpill ? kDenseBit : 0u);
        if (total) atomicAdd(&P.gsum[b / kGGroup], static_cast<unsigned long long>(total));
    }
    if (total == 0 || total > kGSpill || f == 0) return;
    float4* sv4 = reinterpret_cast<float4*>(s_v + tid * 16);
#pragma unroll
    for (int q = 0; q < 4; ++q) sv4[q] = make_float4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
    uint16_t* sv = reinterpret_cast<uint16_t*>(P.spill + b * (kGSpill * 6));
    int32_t* si = reinterpret_cast<int32_t*>(P.spill + b * (kGSpill * 6) + kGSpill * 2);
    const uint64_t cbase = (b * kGB) / P.chunk * P.chunk;  // the block's chunk
    const int32_t local0 = static_cast<int32_t>(i0 - cbase);
    uint32_t k = wp + inc - c;
    for (uint32_t m = f; m; m &= m - 1) {
        const int e = __ffs(m) - 1;
        sv[k] = __half_as_ushort(__float2half_rn(s_v[tid * 16 + e]));
        si[k] = local0 + e;
        ++k;
    }
}

// group prefix, chunk starts, payload length + capacity, header, chunk table and pads (1 CTA)
__global__ void __launch_bounds__(1024) grad_prefix_kernel(const __grid_constant__ SparseParams P) {
    __shared__ unsigned long long s_carry;
    __shared__ unsigned long long s_warp[32];
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    pdl_launch_dependents();  // the emit CTAs may be resident (and load their block counts) now
    if (tid == 0) s_carry = 0;
    __syncthreads();
    for (uint64_t base = 0; base < P.ngroups; base += 1024) {
        const uint64_t i = base + tid;
        const unsigned long long c = i < P.ngroups ? P.gsum[i] : 0ull;
        unsigned long long x = c;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            const unsigned long long y = __shfl_up_sync(0xffffffffu, x, d);
            if (lane >= d) x += y;
        }
        if (lane == 31) s_warp[wid] = x;
        __syncthreads();
        unsigned long long wp = 0, tot = 0;
        for (int k = 0; k < 32; ++k) {
            wp += k < wid ? s_warp[k] : 0ull;
            tot += s_warp[k];
        }
        const unsigned long long carry = s_carry;
        if (i < P.ngroups) P.gpre[i] = carry + wp + x - c;
        __syncthreads();
        if (tid == 0) s_carry = carry + tot;
        __syncthreads();
    }
    const uint64_t kept = s_carry;
    const uint64_t bpc = P.chunk / kGB;  // blocks per chunk
    for (uint64_t c = tid; c <= P.nchunks; c += 1024) {
        unsigned long long st = kept;
        if (c < P.nchunks) {
            const uint64_t fb = c * bpc, g = fb / kGGroup;
            st = P.gpre[g];
            for (uint64_t bb = g * kGGroup; bb < fb; ++bb) st += P.bcount[bb] & ~kDenseBit;
        }
        P.cstart[c] = st;
    }
    const uint64_t voff = kHdr + 16 * P.nchunks, ioff = voff + pad16u(2 * kept);
    const uint64_t total = ioff + pad16u(4 * kept);
    if (tid == 0) {
        P.gpre[P.ngroups] = kept;
        *reinterpret_cast<volatile uint64_t*>(P.out_bytes) = total;
        if (total > P.cap) tc_set_err(P.err, TC_ERR_CAPACITY);
        else put_header(P.out, 2, static_cast<uint32_t>(P.nchunks), *P.thr, P.n, kept, P.chunk, P.seed, total);
    }
    if (total > P.cap) return;
    __syncthreads();  // cstart complete
    for (uint64_t c = tid; c < P.nchunks; c += 1024) {
        uint64_t* t = reinterpret_cast<uint64_t*>(P.out + kHdr + 16 * c);
        t[0] = c * P.chunk;
        t[1] = P.cstart[c + 1] - P.cstart[c];
    }
    for (uint64_t x = 2 * kept + tid; x < pad16u(2 * kept); x += 1024) P.out[voff + x] = 0;
    for (uint64_t x = 4 * kept + tid; x < pad16u(4 * kept); x += 1024) P.out[ioff + x] = 0;
}

// pass 2: a CTA per group of kGGroup blocks; a thread per block finds its offset, then each warp
// copies its 32 blocks' spilled entries (dense blocks: re-read and packed by the warp)
__global__ void __launch_bounds__(kGThreads) grad_emit_kernel(const __grid_constant__ SparseParams P) {
    __shared__ uint32_t s_warp[kGThreads / 32];
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    const uint64_t g = blockIdx.x;
    const uint64_t bb = g * kGGroup + tid;
    const uint32_t info = bb < P.nblocks ? P.bcount[bb] : 0u;  // the counting pass completed before the prefix kernel
    pdl_wait();  // the prefix kernel's group prefix, chunk starts and header
    const uint64_t kept = P.gpre[P.ngroups];
    const uint64_t voff = kHdr + 16 * P.nchunks, ioff = voff + pad16u(2 * kept);
    if (ioff + pad16u(4 * kept) > P.cap) return;  // CAPACITY was reported by the prefix kernel
    uint16_t* gv = reinterpret_cast<uint16_t*>(P.out + voff);
    int32_t* gi = reinterpret_cast<int32_t*>(P.out + ioff);
    const uint64_t b = bb;
    const uint32_t c = info & ~kDenseBit;
    uint32_t inc = c;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, inc, d);
        if (lane >= d) inc += y;
    }
    if (lane == 31) s_warp[wid] = inc;
    __syncthreads();
    uint32_t wp = 0;
#pragma unroll
    for (int k = 0; k < static_cast<int>(kGThreads / 32); ++k) wp += k < wid ? s_warp[k] : 0u;
    const unsigned long long off = P.gpre[g] + wp + inc - c;
    const float thr = *P.thr;
    // spilled blocks: 4 per batch, the first 64 entries of each loaded before any is stored (one
    // round trip per 4 blocks instead of one per block; the rest of a longer run after the batch)
    uint32_t sp = __ballot_sync(0xffffffffu, (info & ~kDenseBit) != 0 && !(info & kDenseBit));
    while (sp) {
        uint32_t cn[4];
        unsigned long long oq[4];
        uint64_t bq[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const int i = sp ? __ffs(sp) - 1 : -1;
            if (sp) sp &= sp - 1;
            const int sl = i < 0 ? 0 : i;
            cn[q] = i < 0 ? 0u : __shfl_sync(0xffffffffu, info, sl) & ~kDenseBit;
            oq[q] = __shfl_sync(0xffffffffu, off, sl);
            bq[q] = g * kGGroup + wid * 32 + static_cast<uint32_t>(sl);
        }
        uint16_t v[4][2];
        int32_t x[4][2];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const uint8_t* slot = P.spill + bq[q] * (kGSpill * 6);
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const uint32_t k = lane + 32 * h;
                if (k < cn[q]) {
                    v[q][h] = reinterpret_cast<const uint16_t*>(slot)[k];
                    x[q][h] = reinterpret_cast<const int32_t*>(slot + kGSpill * 2)[k];
                }
            }
        }
#pragma unroll
        for (int q = 0; q < 4; ++q) {
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const uint32_t k = lane + 32 * h;
                if (k < cn[q]) {
                    gv[oq[q] + k] = v[q][h];
                    gi[oq[q] + k] = x[q][h];
                }
            }
            if (cn[q] > 64) {
                const uint8_t* slot = P.spill + bq[q] * (kGSpill * 6);
                for (uint32_t k = 64 + lane; k < cn[q]; k += 32) {
                    gv[oq[q] + k] = reinterpret_cast<const uint16_t*>(slot)[k];
                    gi[oq[q] + k] = reinterpret_cast<const int32_t*>(slot + kGSpill * 2)[k];
                }
            }
        }
    }
    for (int i = 0; i < 32; ++i) {  // the warp's dense blocks, one at a time
        const uint32_t ci = __shfl_sync(0xffffffffu, info, i);
        const uint32_t cnt = ci & ~kDenseBit;
        if (cnt == 0 || !(ci & kDenseBit)) continue;
        const unsigned long long o = __shfl_sync(0xffffffffu, off, i);
        const uint64_t bb = g * kGGroup + wid * 32 + i;
        // dense block: the count kernel's order (16-element runs of threads 0..255), 32 runs a pass
        unsigned long long run = o;
        for (uint32_t t0 = 0; t0 < kGThreads; t0 += 32) {
            const uint64_t i0 = bb * kGB + 16ull * (t0 + lane);
            float v[16];
            const uint32_t f = flags16(P.x, P.n, i0, thr, v);
            const uint32_t cf = __popc(f);
            uint32_t x = cf;
#pragma unroll
            for (int d = 1; d < 32; d <<= 1) {
                const uint32_t y = __shfl_up_sync(0xffffffffu, x, d);
                if (lane >= d) x += y;
            }
            unsigned long long k = run + x - cf;
#pragma unroll
            for (int e = 0; e < 16; ++e)
                if ((f >> e) & 1u) {
                    const uint64_t ii = i0 + e;
                    gv[k] = __half_as_ushort(__float2half_rn(v[e]));
                    gi[k] = static_cast<int32_t>(ii - ii / P.chunk * P.chunk);
                    ++k;
                }
            run += __shfl_sync(0xffffffffu, x, 31);
        }
    }
}

// ------------------------------------------------------------- decompression ----------
struct Payload {           // as located and validated by the walker
    const int8_t* q;       // dense codes (variant 1)
    const uint16_t* val;   // sparse FP16 values
    const int32_t* idx;    // sparse local indices
    const uint64_t* table; // sparse chunk table {base, count}
    unsigned long long* cpre;  // [chunks + 1] entry prefix (walker output)
    unsigned long long* tstart;  // [tiles + 1] first entry of each kGB tile (replay only)
    float scale;
    uint32_t variant;
    uint64_t chunks, chunk, kept;
};

__global__ void grad_walk_kernel(const uint8_t* p, uint64_t bytes, uint64_t n, Payload* out, unsigned* err) {
    if (threadIdx.x != 0) return;
    const uint64_t* h = reinterpret_cast<const uint64_t*>(p);
    Payload R = {};
    bool bad = bytes < kHdr || static_cast<uint32_t>(h[0]) != 0x31474354u;
    if (!bad) {
        R.variant = static_cast<uint32_t>(h[0] >> 32);
        R.chunks = static_cast<uint32_t>(h[1]);
        R.scale = __uint_as_float(static_cast<uint32_t>(h[1] >> 32));
        R.kept = h[3];
        R.chunk = h[4];
        const uint64_t total = h[6];
        bad = h[2] != n || total != bytes || (R.variant & ~0xffu) != 0;
        if (!bad && (R.variant & 0xffu) == 1) {
            R.variant = 1;
            bad = R.kept != n || total != kHdr + pad16u(n);
            R.q = reinterpret_cast<const int8_t*>(p + kHdr);
        } else if (!bad && (R.variant & 0xffu) == 2) {
            R.variant = 2;
            const uint64_t want = n ? (n + R.chunk - 1) / (R.chunk ? R.chunk : 1) : 1;
            bad = R.chunk == 0 || R.chunk > 2147483647ull || R.kept > n || R.chunks != want ||
                  total != kHdr + 16 * R.chunks + pad16u(2 * R.kept) + pad16u(4 * R.kept);
            if (!bad) {
                R.table = reinterpret_cast<const uint64_t*>(p + kHdr);
                R.val = reinterpret_cast<const uint16_t*>(p + kHdr + 16 * R.chunks);
                R.idx = reinterpret_cast<const int32_t*>(p + kHdr + 16 * R.chunks + pad16u(2 * R.kept));
                unsigned long long k = 0;
                for (uint64_t c = 0; c < R.chunks && !bad; ++c) {
                    const uint64_t base = R.table[2 * c], cnt = R.table[2 * c + 1];
                    const uint64_t len = base + R.chunk < n ? R.chunk : n - base;
                    if (base != c * R.chunk || cnt > len || k + cnt > R.kept) bad = true;
                    out->cpre[c] = k;
                    k += cnt;
                }
                if (!bad && k != R.kept) bad = true;
                out->cpre[R.chunks] = k;
            }
        } else {
            bad = true;
        }
    }
    if (bad) {
        tc_set_err(err, TC_ERR_CORRUPT);
        R.variant = 0;
    }
    R.cpre = out->cpre;
    R.tstart = out->tstart;
    *out = R;
}

__device__ __forceinline__ uint64_t chunk_of(const Payload& R, uint64_t k) {
    uint64_t lo = 0, hi = R.chunks;  // cpre[lo] <= k < cpre[lo + 1]
    while (hi - lo > 1) {
        const uint64_t mid = (lo + hi) >> 1;
        if (R.cpre[mid] <= k) lo = mid; else hi = mid;
    }
    return lo;
}

// entry k -> (global position, value); checks the index against its chunk and its predecessor
__device__ __forceinline__ bool entry(const Payload& R, uint64_t n, uint64_t k, uint64_t* pos, float* val) {
    const uint64_t c = chunk_of(R, k);
    const uint64_t base = c * R.chunk;
    const uint64_t len = base + R.chunk < n ? R.chunk : n - base;
    const int32_t i = R.idx[k];
    if (i < 0 || static_cast<uint64_t>(i) >= len || (k > R.cpre[c] && R.idx[k - 1] >= i)) return false;
    *pos = base + static_cast<uint64_t>(i);
    *val = __half2float(__ushort_as_half(R.val[k]));
    return true;
}

__global__ void grad_decompress_kernel(const Payload* RP, uint64_t n, float* out, unsigned* err) {
    if (*reinterpret_cast<volatile unsigned*>(err) != 0) return;
    const Payload R = *RP;
    const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
    const uint64_t t = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (R.variant == 1)
        for (uint64_t i = t; i < n; i += stride) out[i] = __fmul_rn(R.scale, static_cast<float>(R.q[i]));
}

// sparse payload -> dense, one pass: a CTA per kGB tile expands the tile's entries (from the
// tile-start table) in shared memory and writes the whole tile with 16-byte stores.  Two barriers
// per tile: each thread zeroes the shared words it has just stored (ready for the next tile's
// entries), and the next tile's entry range is loaded before the current tile is written
__global__ void __launch_bounds__(kGThreads) grad_expand_kernel(const Payload* RP, uint64_t n, uint64_t tiles,
                                                                float* out, unsigned* err) {
    __shared__ __align__(16) float s_t[kGB];
    if (*reinterpret_cast<volatile unsigned*>(err) != 0) return;
    const Payload R = *RP;
    if (R.variant != 2) return;
    const int tid = threadIdx.x;
    bool bad = false;
    for (uint32_t i = tid; i < kGB / 4; i += kGThreads) reinterpret_cast<float4*>(s_t)[i] = make_float4(0, 0, 0, 0);
    __syncthreads();
    const bool aligned = (reinterpret_cast<uintptr_t>(out) & 15u) == 0;
    uint64_t t = blockIdx.x;
    uint64_t k0 = t < tiles ? R.tstart[t] : 0, k1 = t < tiles ? R.tstart[t + 1] : 0;
    for (; t < tiles; t += gridDim.x) {
        const uint64_t base = t * kGB;
        const uint64_t cbase = base / R.chunk * R.chunk;  // the tile lies in one chunk
        for (uint64_t k = k0 + tid; k < k1; k += kGThreads) {
            const int32_t i = R.idx[k];
            const uint64_t pos = cbase + static_cast<uint64_t>(static_cast<uint32_t>(i));
            if (i < 0 || pos < base || pos >= base + kGB || pos >= n || (k > k0 && R.idx[k - 1] >= i)) {
                bad = true;
                continue;
            }
            s_t[pos - base] = __half2float(__ushort_as_half(R.val[k]));
        }
        const uint64_t tn = t + gridDim.x;  // the next tile's entry range, in flight during the stores
        const uint64_t n0 = tn < tiles ? R.tstart[tn] : 0, n1 = tn < tiles ? R.tstart[tn + 1] : 0;
        __syncthreads();
        const uint32_t nw = n - base < kGB ? static_cast<uint32_t>(n - base) : kGB;
        float4* s4 = reinterpret_cast<float4*>(s_t);
        for (uint32_t q = tid; q * 4 < nw; q += kGThreads) {
            const float4 x = s4[q];
            if (q * 4 + 4 <= nw && aligned)
                *reinterpret_cast<float4*>(out + base + q * 4) = x;
            else
                for (uint32_t i = q * 4; i < nw && i < q * 4 + 4; ++i) out[base + i] = s_t[i];
            s4[q] = make_float4(0, 0, 0, 0);
        }
        __syncthreads();
        k0 = n0;
        k1 = n1;
    }
    if (bad) tc_set_err(err, TC_ERR_CORRUPT);
}

// first entry of every kGB tile (replay): lower bound of the tile start among the sorted positions
__global__ void grad_tile_start_kernel(const Payload* RP, uint64_t n, uint64_t tiles, unsigned* err) {
    if (*reinterpret_cast<volatile unsigned*>(err) != 0) return;
    const Payload R = *RP;
    if (R.variant != 2) return;
    for (uint64_t t = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; t <= tiles;
         t += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        const uint64_t want = t * kGB;
        uint64_t lo = 0, hi = R.kept;  // first k with position(k) >= want
        while (lo < hi) {
            const uint64_t mid = (lo + hi) >> 1;
            const uint64_t c = chunk_of(R, mid);
            const uint64_t pos = c * R.chunk + static_cast<uint64_t>(static_cast<uint32_t>(R.idx[mid]));
            if (pos < want) lo = mid + 1; else hi = mid;
        }
        R.tstart[t] = lo;
        if (t == tiles && lo != R.kept) tc_set_err(err, TC_ERR_CORRUPT);  // entries past the last tile
    }
}

// ------------------------------------------------------------------- Adam ----------
struct AdamC {
    float b1, b2, eps;
    float omb1, omb2;  // 1 - b1, 1 - b2 rounded to fp32 (host IEEE subtraction = __fsub_rn), once per call
};

__device__ __forceinline__ void adam_update(float& master, float& m, float& v, float g, const AdamC& a, float ss,
                                            float ic) {
    // oracle/tco_grad.c order: m, v; denom = sqrt(v) * inv_c2s + eps; master -= step_size * (m / denom).
    // Zero operands take the IEEE result directly (sqrt(+0) = +0, 0 / d = 0 with 0's sign for d > 0):
    // the same values without the slow paths that zeros trigger (most of a sparse gradient is zero)
    m = __fadd_rn(__fmul_rn(a.b1, m), __fmul_rn(a.omb1, g));
    v = __fadd_rn(__fmul_rn(a.b2, v), __fmul_rn(a.omb2, __fmul_rn(g, g)));
    // Selects, not branches (re-entry; ncu rd6k: branch bookkeeping was 24 % of the replay's
    // instructions): a zero operand is replaced by 1 (the fast path) and the result by the zero
    // itself.  Fused replay of 5 payloads: 24.65 -> 23.42 ms (mid-training moments), 23.73 -> 23.35
    // ms (fresh), profiles/rd6l_adam_select_ab.txt.
    const float sq = __fsqrt_rn(v != 0.0f ? v : 1.0f);
    const float den = __fadd_rn(__fmul_rn(v != 0.0f ? sq : v, ic), a.eps);
    const float qd = __fdiv_rn(m != 0.0f ? m : 1.0f, den);
    const float q = m != 0.0f ? qd : m;
    master = __fsub_rn(master, __fmul_rn(ss, q));
}

__global__ void adam_step_kernel(float* __restrict__ master, float* __restrict__ m, float* __restrict__ v,
                                 uint16_t* __restrict__ w16, uint64_t n, const float* __restrict__ g, AdamC a,
                                 float ss, float ic) {
    // 4 elements per thread with 16-byte loads / stores (8-byte for the bf16 weights)
    const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
    const uint64_t nv = n / 4;
    for (uint64_t q = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; q < nv; q += stride) {
        float4 w = reinterpret_cast<const float4*>(master)[q];
        float4 mm = reinterpret_cast<const float4*>(m)[q];
        float4 vv = reinterpret_cast<const float4*>(v)[q];
        const float4 gg = __ldg(reinterpret_cast<const float4*>(g) + q);
        adam_update(w.x, mm.x, vv.x, gg.x, a, ss, ic);
        adam_update(w.y, mm.y, vv.y, gg.y, a, ss, ic);
        adam_update(w.z, mm.z, vv.z, gg.z, a, ss, ic);
        adam_update(w.w, mm.w, vv.w, gg.w, a, ss, ic);
        reinterpret_cast<float4*>(master)[q] = w;
        reinterpret_cast<float4*>(m)[q] = mm;
        reinterpret_cast<float4*>(v)[q] = vv;
        ushort4 h;
        h.x = __bfloat16_as_ushort(__float2bfloat16_rn(w.x));
        h.y = __bfloat16_as_ushort(__float2bfloat16_rn(w.y));
        h.z = __bfloat16_as_ushort(__float2bfloat16_rn(w.z));
        h.w = __bfloat16_as_ushort(__float2bfloat16_rn(w.w));
        reinterpret_cast<ushort4*>(w16)[q] = h;
    }
    for (uint64_t i = nv * 4 + static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride) {
        float w = master[i], mi = m[i], vi = v[i];
        adam_update(w, mi, vi, g[i], a, ss, ic);
        master[i] = w;
        m[i] = mi;
        v[i] = vi;
        w16[i] = __bfloat16_as_ushort(__float2bfloat16_rn(w));
    }
}

// NEXT row 2: the Adam step and the change masks of the lossless diff of its own update.  A
// thread takes 4 consecutive elements (16-byte loads of master / m / v / grad, 8-byte of the
// bf16 weights), so a warp covers 128 elements = 4 mask words per segment: each lane's 4 change
// bits are OR-shuffled across the 8 lanes of one 32-element mask word (LSB-first, reading R6).
// A vector is stored only where one of its words changed (the others are rewritten equal).
__device__ __forceinline__ uint32_t or8(uint32_t bits, int lane) {
    uint32_t x = bits << (4 * (lane & 7));
    x |= __shfl_xor_sync(0xffffffffu, x, 1);
    x |= __shfl_xor_sync(0xffffffffu, x, 2);
    x |= __shfl_xor_sync(0xffffffffu, x, 4);
    return x;
}

__global__ void __launch_bounds__(256) adam_mask_kernel(float* __restrict__ master, float* __restrict__ m,
                                                        float* __restrict__ v, uint16_t* __restrict__ w16, uint64_t n,
                                                        const float* __restrict__ g, AdamC a, float ss, float ic,
                                                        uint32_t* __restrict__ mk_w, uint32_t* __restrict__ mk_master,
                                                        uint32_t* __restrict__ mk_m, uint32_t* __restrict__ mk_v) {
    const int lane = threadIdx.x & 31;
    const uint64_t nq = (n + 3) / 4, groups = (nq + 31) / 32, words = (n + 31) / 32;
    const uint64_t gstride = static_cast<uint64_t>(gridDim.x) * (blockDim.x / 32);
    for (uint64_t gq = static_cast<uint64_t>(blockIdx.x) * (blockDim.x / 32) + (threadIdx.x >> 5); gq < groups;
         gq += gstride) {
        const uint64_t q = gq * 32 + lane;
        uint32_t cw = 0, cmaster = 0, cm = 0, cv = 0;
        if (q * 4 + 4 <= n) {
            const float4 w0 = reinterpret_cast<const float4*>(master)[q];
            const float4 m0 = reinterpret_cast<const float4*>(m)[q];
            const float4 v0 = reinterpret_cast<const float4*>(v)[q];
            const float4 gg = __ldg(reinterpret_cast<const float4*>(g) + q);
            const ushort4 h0 = reinterpret_cast<const ushort4*>(w16)[q];
            float4 w = w0, mm = m0, vv = v0;
            adam_update(w.x, mm.x, vv.x, gg.x, a, ss, ic);
            adam_update(w.y, mm.y, vv.y, gg.y, a, ss, ic);
            adam_update(w.z, mm.z, vv.z, gg.z, a, ss, ic);
            adam_update(w.w, mm.w, vv.w, gg.w, a, ss, ic);
            ushort4 h;
            h.x = __bfloat16_as_ushort(__float2bfloat16_rn(w.x));
            h.y = __bfloat16_as_ushort(__float2bfloat16_rn(w.y));
            h.z = __bfloat16_as_ushort(__float2bfloat16_rn(w.z));
            h.w = __bfloat16_as_ushort(__float2bfloat16_rn(w.w));
            auto ne = [](float x, float y) { return __float_as_uint(x) != __float_as_uint(y); };
            cmaster = ne(w.x, w0.x) | ne(w.y, w0.y) << 1 | ne(w.z, w0.z) << 2 | ne(w.w, w0.w) << 3;
            cm = ne(mm.x, m0.x) | ne(mm.y, m0.y) << 1 | ne(mm.z, m0.z) << 2 | ne(mm.w, m0.w) << 3;
            cv = ne(vv.x, v0.x) | ne(vv.y, v0.y) << 1 | ne(vv.z, v0.z) << 2 | ne(vv.w, v0.w) << 3;
            cw = (h.x != h0.x) | (h.y != h0.y) << 1 | (h.z != h0.z) << 2 | (h.w != h0.w) << 3;
            if (cmaster) reinterpret_cast<float4*>(master)[q] = w;
            if (cm) reinterpret_cast<float4*>(m)[q] = mm;
            if (cv) reinterpret_cast<float4*>(v)[q] = vv;
            if (cw) reinterpret_cast<ushort4*>(w16)[q] = h;
        } else {
            for (uint64_t i = q * 4; i < n; ++i) {  // the last, partial quad
                const uint32_t bit = 1u << (i - q * 4);
                const float w0 = master[i], m0 = m[i], v0 = v[i];
                const uint16_t h0 = w16[i];
                float w = w0, mm = m0, vv = v0;
                adam_update(w, mm, vv, g[i], a, ss, ic);
                const uint16_t h = __bfloat16_as_ushort(__float2bfloat16_rn(w));
                if (__float_as_uint(w) != __float_as_uint(w0)) { master[i] = w; cmaster |= bit; }
                if (__float_as_uint(mm) != __float_as_uint(m0)) { m[i] = mm; cm |= bit; }
                if (__float_as_uint(vv) != __float_as_uint(v0)) { v[i] = vv; cv |= bit; }
                if (h != h0) { w16[i] = h; cw |= bit; }
            }
        }
        cw = or8(cw, lane);
        cmaster = or8(cmaster, lane);
        cm = or8(cm, lane);
        cv = or8(cv, lane);
        const uint64_t wd = gq * 4 + (lane >> 3);
        if ((lane & 7) == 0 && wd < words) {
            mk_w[wd] = cw;
            mk_master[wd] = cmaster;
            mk_m[wd] = cm;
            mk_v[wd] = cv;
        }
    }
}

// The Adam step with its FULL-format differential written in the same pass (tc_adam_step_encode with
// index_mode = 2, reading R21): full records have data-independent sizes, so every element knows
// where its four words go — record of segment s (w16 | master | m | v), chunk c at
// base[s] + c * rec_full[s], word i - c*C after the 64-byte header — and the pass writes the new
// state and the record together: no mask, no second pass over the new state (the mask path's
// dense case re-read it).  A thread per 4 consecutive parameters (16-byte loads / stores; 8 bytes
// for the bf16 words); the thread holding a chunk's first quad writes its four headers, the one
// holding its last quad the padding.
struct AdamFullLayout {
    uint64_t base[4];      // byte offset of each segment's first record
    uint64_t rec_full[4];  // record bytes of a full chunk (m = C)
    uint64_t C, total, version, ref_version;
    uint32_t T;
};

__device__ __forceinline__ void adam_full_header(uint8_t* out, const AdamFullLayout& L, int s, uint64_t c, uint64_t mc) {
    const uint32_t w = s == 0 ? 2u : 4u;
    uint64_t* h = reinterpret_cast<uint64_t*>(out + L.base[s] + c * L.rec_full[s]);
    h[0] = 0x31444354ull /* "TCD1" */ | (1ull << 32) | (static_cast<uint64_t>(w) << 48) | (5ull << 56);
    h[1] = static_cast<uint64_t>(L.T) | (static_cast<uint64_t>(s) << 32);
    h[2] = c * L.C;
    h[3] = mc;
    h[4] = mc;
    h[5] = L.version;
    h[6] = L.ref_version;
    h[7] = kHdr + pad16u(w * mc);
}

__global__ void __launch_bounds__(256) adam_full_kernel(float* __restrict__ master, float* __restrict__ m,
                                                        float* __restrict__ v, uint16_t* __restrict__ w16, uint64_t n,
                                                        const float* __restrict__ g, AdamC a, float ss, float ic,
                                                        uint8_t* __restrict__ out, uint64_t out_cap, uint64_t* out_bytes,
                                                        const AdamFullLayout L, unsigned* err) {
    const uint64_t t0 = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (t0 == 0) {
        *reinterpret_cast<volatile uint64_t*>(out_bytes) = L.total;
        if (L.total > out_cap) tc_set_err(err, TC_ERR_CAPACITY);
        if (n == 0 && L.total <= out_cap)
            for (int s = 0; s < 4; ++s) adam_full_header(out, L, s, 0, 0);  // four empty records
    }
    if (L.total > out_cap) return;  // nothing of the diff is written
    const uint64_t nq = (n + 3) / 4;
    const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
    for (uint64_t q = t0; q < nq; q += stride) {
        const uint64_t i0 = q * 4;
        const uint64_t c = i0 / L.C, off = i0 - c * L.C;  // C is a multiple of 4: a quad never straddles chunks
        const uint64_t mc = n - c * L.C < L.C ? n - c * L.C : L.C;
        uint8_t* r0 = out + L.base[0] + c * L.rec_full[0] + kHdr;
        uint8_t* r1 = out + L.base[1] + c * L.rec_full[1] + kHdr;
        uint8_t* r2 = out + L.base[2] + c * L.rec_full[2] + kHdr;
        uint8_t* r3 = out + L.base[3] + c * L.rec_full[3] + kHdr;
        if (i0 + 4 <= n) {
            float4 w = reinterpret_cast<const float4*>(master)[q];
            float4 mm = reinterpret_cast<const float4*>(m)[q];
            float4 vv = reinterpret_cast<const float4*>(v)[q];
            const float4 gg = __ldg(reinterpret_cast<const float4*>(g) + q);
            adam_update(w.x, mm.x, vv.x, gg.x, a, ss, ic);
            adam_update(w.y, mm.y, vv.y, gg.y, a, ss, ic);
            adam_update(w.z, mm.z, vv.z, gg.z, a, ss, ic);
            adam_update(w.w, mm.w, vv.w, gg.w, a, ss, ic);
            ushort4 h;
            h.x = __bfloat16_as_ushort(__float2bfloat16_rn(w.x));
            h.y = __bfloat16_as_ushort(__float2bfloat16_rn(w.y));
            h.z = __bfloat16_as_ushort(__float2bfloat16_rn(w.z));
            h.w = __bfloat16_as_ushort(__float2bfloat16_rn(w.w));
            reinterpret_cast<float4*>(master)[q] = w;
            reinterpret_cast<float4*>(m)[q] = mm;
            reinterpret_cast<float4*>(v)[q] = vv;
            reinterpret_cast<ushort4*>(w16)[q] = h;
            *reinterpret_cast<ushort4*>(r0 + 2 * off) = h;
            *reinterpret_cast<float4*>(r1 + 4 * off) = w;
            *reinterpret_cast<float4*>(r2 + 4 * off) = mm;
            *reinterpret_cast<float4*>(r3 + 4 * off) = vv;
        } else {
            for (uint64_t i = i0; i < n; ++i) {  // the last, partial quad
                float w = master[i], mm = m[i], vv = v[i];
                adam_update(w, mm, vv, g[i], a, ss, ic);
                const uint16_t h = __bfloat16_as_ushort(__float2bfloat16_rn(w));
                master[i] = w;
                m[i] = mm;
                v[i] = vv;
                w16[i] = h;
                const uint64_t o = i - c * L.C;
                *reinterpret_cast<uint16_t*>(r0 + 2 * o) = h;
                *reinterpret_cast<float*>(r1 + 4 * o) = w;
                *reinterpret_cast<float*>(r2 + 4 * o) = mm;
                *reinterpret_cast<float*>(r3 + 4 * o) = vv;
            }
        }
        if (off == 0)
            for (int s = 0; s < 4; ++s) adam_full_header(out, L, s, c, mc);
        if (off + 4 >= mc) {  // the chunk's last quad: zero the padding of its four records
            for (uint64_t x = 2 * mc; x < pad16u(2 * mc); ++x) r0[x] = 0;
            for (uint64_t x = 4 * mc; x < pad16u(4 * mc); ++x) r1[x] = r2[x] = r3[x] = 0;
        }
    }
}

struct ReplayParams {
    float* master;
    float* m;
    float* v;
    uint64_t n, tiles;
    int nsteps;              // fused steps (payloads 0 .. nsteps-1)
    AdamC a;
    float ss[TC_MAX_FOLD], ic[TC_MAX_FOLD];  // per fused step: lr / (1 - b1^t), 1 / sqrt(1 - b2^t)
    const Payload* pay;      // [nsteps], walker output
    unsigned* err;
};

// one CTA of 512 threads per tile of kGB elements, 8 per thread, two CTAs per SM: (master, m, v)
// stay in registers for all fused steps.  Each tile passes several CTA barriers (entry staging,
// dense gradient tiles); with one CTA of 1024 threads per SM every barrier idled the whole SM
// (ncu: a third of the stall samples), with two the other CTA computes through it.
constexpr uint32_t kRThreads = 512;
constexpr uint32_t kRPer = kGB / kRThreads;
constexpr uint32_t kRStage = 2048;  // staged sparse entries of one tile (all fused steps)
constexpr uint32_t kRGroup = 2;     // fused steps whose dense gradient tiles share two barriers
constexpr size_t kRDynSmem = sizeof(float) * (kRGroup + 3) * kGB;

struct ReplayStep {                 // per fused step, in shared memory
    const int8_t* q;
    const uint16_t* val;
    const int32_t* idx;
    const unsigned long long* tstart;
    uint64_t chunk;
    float scale;
    uint32_t variant;
};

__global__ void __launch_bounds__(kRThreads, 2) adam_replay_kernel(const __grid_constant__ ReplayParams P) {
    extern __shared__ float s_gd[];  // [kRGroup][kGB] dense gradient tiles | [3][kGB] next tile's state
    float* s_next = s_gd + kRGroup * kGB;
    __shared__ uint64_t s_bar;
    __shared__ uint16_t s_pos[kRStage];
    __shared__ float s_val[kRStage];
    __shared__ ReplayStep s_step[TC_MAX_FOLD];
    __shared__ uint32_t s_run[TC_MAX_FOLD + 1];   // staged entries before step s
    __shared__ unsigned long long s_k0[TC_MAX_FOLD];
    __shared__ uint32_t s_fits;
    if (*reinterpret_cast<volatile unsigned*>(P.err) != 0) return;
    const int tid = threadIdx.x;
    if (tid < P.nsteps) {
        const Payload& R = P.pay[tid];
        s_step[tid] = {R.q, R.val, R.idx, R.tstart, R.chunk, R.scale, R.variant};
    }
    if (tid == 0) mbar_init(&s_bar, 1);
    __syncthreads();
    bool bad = false;
    uint32_t phase = 0;
    // a full tile's (master, m, v) comes in by TMA while the previous tile is folded (one CTA
    // per SM: without this the SM would alternate between loading and computing)
    auto prefetch = [&](uint64_t tt) {
        if (tid == 0) {
            mbar_arrive_expect_tx(&s_bar, 3 * kGB * 4);
            bulk_g2s(s_next, P.master + tt * kGB, kGB * 4, &s_bar);
            bulk_g2s(s_next + kGB, P.m + tt * kGB, kGB * 4, &s_bar);
            bulk_g2s(s_next + 2 * kGB, P.v + tt * kGB, kGB * 4, &s_bar);
        }
    };
    const uint64_t full_tiles = P.n / kGB;
    bool pending = blockIdx.x < full_tiles;
    if (pending) prefetch(blockIdx.x);
    for (uint64_t t = blockIdx.x; t < P.tiles; t += gridDim.x) {
        const uint64_t base = t * kGB;
        float w[kRPer], mm[kRPer], vv[kRPer];
        if (t < full_tiles) {
            mbar_wait_parity(&s_bar, phase);
            phase ^= 1u;
#pragma unroll
            for (uint32_t j = 0; j < kRPer; ++j) {
                w[j] = s_next[j * kRThreads + tid];
                mm[j] = s_next[kGB + j * kRThreads + tid];
                vv[j] = s_next[2 * kGB + j * kRThreads + tid];
            }
            __syncthreads();  // every thread has its state: the buffer is free
            pending = t + gridDim.x < full_tiles;
            if (pending) prefetch(t + gridDim.x);
        } else {
#pragma unroll
            for (uint32_t j = 0; j < kRPer; ++j) {
                const uint64_t i = base + j * kRThreads + tid;
                w[j] = i < P.n ? P.master[i] : 0.0f;
                mm[j] = i < P.n ? P.m[i] : 0.0f;
                vv[j] = i < P.n ? P.v[i] : 0.0f;
            }
        }
        // every sparse step's entries of this tile, staged at once: one round trip per tile
        if (tid < P.nsteps) {
            const ReplayStep& R = s_step[tid];
            unsigned long long k0 = 0, k1 = 0;
            if (R.variant == 2) {
                k0 = R.tstart[t];
                k1 = R.tstart[t + 1];
                if (k1 < k0) k1 = k0;
            }
            s_k0[tid] = k0;
            s_run[tid + 1] = static_cast<uint32_t>(k1 - k0 < kRStage ? k1 - k0 : kRStage + 1);
        }
        __syncthreads();
        if (tid == 0) {
            uint32_t o = 0;
            s_run[0] = 0;
            for (int s = 0; s < P.nsteps; ++s) {
                o += s_run[s + 1];
                s_run[s + 1] = o;
            }
            s_fits = o <= kRStage;
        }
        __syncthreads();
        const bool fits = s_fits != 0;
        if (fits) {
            const uint32_t total = s_run[P.nsteps];
            for (uint32_t e = tid; e < total; e += kRThreads) {
                int s = 0;
                while (s_run[s + 1] <= e) ++s;
                const ReplayStep& R = s_step[s];
                const uint64_t k = s_k0[s] + (e - s_run[s]);
                // the tile lies in one chunk (chunk lengths are multiples of kGB)
                const uint64_t pos = base / R.chunk * R.chunk + static_cast<uint64_t>(static_cast<uint32_t>(R.idx[k]));
                if (R.idx[k] < 0 || pos < base || pos >= base + kGB || pos >= P.n) bad = true;
                s_pos[e] = static_cast<uint16_t>((pos - base) & (kGB - 1));
                s_val[e] = __half2float(__ushort_as_half(R.val[k]));
            }
            __syncthreads();
            for (uint32_t e = tid; e < total; e += kRThreads) {  // increasing within each run
                int s = 0;
                while (s_run[s + 1] <= e) ++s;
                if (e > s_run[s] && s_pos[e - 1] >= s_pos[e]) bad = true;
            }
        }
        for (int g0 = 0; g0 < P.nsteps; g0 += static_cast<int>(kRGroup)) {
            const int g1 = g0 + static_cast<int>(kRGroup) < P.nsteps ? g0 + static_cast<int>(kRGroup) : P.nsteps;
            if (fits) {
                // the group's sparse gradients as dense tiles: two barriers for up to kRGroup steps
                for (int s = g0; s < g1; ++s)
                    if (s_step[s].variant == 2) {
#pragma unroll
                        for (uint32_t j = 0; j < kRPer; ++j) s_gd[(s - g0) * kGB + j * kRThreads + tid] = 0.0f;
                    }
                __syncthreads();
                for (int s = g0; s < g1; ++s)
                    for (uint32_t e = s_run[s] + tid; e < s_run[s + 1]; e += kRThreads)
                        s_gd[(s - g0) * kGB + s_pos[e]] = s_val[e];
                __syncthreads();
                for (int s = g0; s < g1; ++s) {
                    const ReplayStep& R = s_step[s];
                    // the step's gradients first (loads in flight together), then the updates
                    float g[kRPer];
#pragma unroll
                    for (uint32_t j = 0; j < kRPer; ++j) {
                        const uint64_t i = base + j * kRThreads + tid;
                        g[j] = R.variant == 1 ? (i < P.n ? __fmul_rn(R.scale, static_cast<float>(R.q[i])) : 0.0f)
                                              : s_gd[(s - g0) * kGB + j * kRThreads + tid];
                    }
                    const float ss = P.ss[s], ic = P.ic[s];
#pragma unroll
                    for (uint32_t j = 0; j < kRPer; ++j) adam_update(w[j], mm[j], vv[j], g[j], P.a, ss, ic);
                }
                __syncthreads();  // before the next group's tiles
                continue;
            }
            for (int s = g0; s < g1; ++s) {  // more entries than the stage: a step at a time
                const ReplayStep& R = s_step[s];
                if (R.variant == 1) {
#pragma unroll
                    for (uint32_t j = 0; j < kRPer; ++j) {
                        const uint64_t i = base + j * kRThreads + tid;
                        const float g = i < P.n ? __fmul_rn(R.scale, static_cast<float>(R.q[i])) : 0.0f;
                        adam_update(w[j], mm[j], vv[j], g, P.a, P.ss[s], P.ic[s]);
                    }
                    continue;
                }
#pragma unroll
                for (uint32_t j = 0; j < kRPer; ++j) s_gd[j * kRThreads + tid] = 0.0f;
                __syncthreads();
                const Payload& RP = P.pay[s];
                const uint64_t k0 = RP.tstart[t], k1 = RP.tstart[t + 1];
                for (uint64_t k = k0 + tid; k < k1; k += kRThreads) {
                    uint64_t pos;
                    float val;
                    if (!entry(RP, P.n, k, &pos, &val) || pos < base || pos >= base + kGB) {
                        bad = true;
                        continue;
                    }
                    s_gd[pos - base] = val;
                }
                __syncthreads();
#pragma unroll
                for (uint32_t j = 0; j < kRPer; ++j)
                    adam_update(w[j], mm[j], vv[j], s_gd[j * kRThreads + tid], P.a, P.ss[s], P.ic[s]);
                __syncthreads();
            }
        }
#pragma unroll
        for (uint32_t j = 0; j < kRPer; ++j) {
            const uint64_t i = base + j * kRThreads + tid;
            if (i < P.n) {
                P.master[i] = w[j];
                P.m[i] = mm[j];
                P.v[i] = vv[j];
            }
        }
        __syncthreads();  // the stage and the run table are reused by the next tile
    }
    if (pending) mbar_wait_parity(&s_bar, phase);  // (not reached: the loop consumes every prefetch)
    if (bad) tc_set_err(P.err, TC_ERR_CORRUPT);
}

AdamC adam_consts(const tc_adam_hp* hp) {
    AdamC a;
    a.b1 = static_cast<float>(hp ? hp->beta1 : 0.9);
    a.b2 = static_cast<float>(hp ? hp->beta2 : 0.999);
    a.eps = static_cast<float>(hp ? hp->eps : 1e-8);
    a.omb1 = 1.0f - a.b1;  // one IEEE binary32 subtraction each (exact for beta in [0.5, 1], Sterbenz)
    a.omb2 = 1.0f - a.b2;
    return a;
}
// step_size = lr / (1 - beta1^t), inv_c2s = 1 / sqrt(1 - beta2^t): in double, rounded to fp32
void bias(const tc_adam_hp* hp, uint64_t step, float* ss, float* ic) {
    const double lr = hp ? hp->lr : 1e-3, b1 = hp ? hp->beta1 : 0.9, b2 = hp ? hp->beta2 : 0.999;
    *ss = static_cast<float>(lr / (1.0 - std::pow(b1, static_cast<double>(step))));
    *ic = static_cast<float>(1.0 / std::sqrt(1.0 - std::pow(b2, static_cast<double>(step))));
}

tc_status check_state(const tc_adam_state* st) {
    if (!st || !st->n) return st ? TC_OK : fail(TC_ERR_INVALID, "state is NULL");
    if (!st->master || !st->m || !st->v || !st->w16 || !aligned16(st->master) || !aligned16(st->m) ||
        !aligned16(st->v) || !aligned16(st->w16))
        return fail(TC_ERR_INVALID, "state pointers must be 16-byte aligned device pointers");
    return TC_OK;
}

int grid_for(tc_ctx* ctx, uint64_t work, int threads) {
    const uint64_t want = (work + threads - 1) / threads;
    const uint64_t cap = static_cast<uint64_t>(tc::ctx_num_sms(ctx)) * 8;
    return static_cast<int>(want < cap ? (want ? want : 1) : cap);
}

}  // namespace

extern "C" {

tc_status tc_grad_bound(uint64_t n, const tc_grad_opts* opts, uint64_t* max_bytes) {
    if (!max_bytes) return fail(TC_ERR_INVALID, "max_bytes is NULL");
    Opts o;
    tc_status st = resolve(opts, &o);
    if (st != TC_OK) return st;
    *max_bytes = bound_of(n, o);
    return TC_OK;
}

tc_status tc_grad_compress(tc_ctx* ctx, const float* grad, uint64_t n, const tc_grad_opts* opts, uint64_t seed,
                           void* out, uint64_t out_cap, uint64_t* out_bytes, tc_stream stream) {
    if (!ctx || !out || !aligned16(out) || !out_bytes || (n && (!grad || !aligned16(grad))))
        return fail(TC_ERR_INVALID, "bad arguments (ctx, 16-byte aligned out / grad, out_bytes)");
    Opts o;
    tc_status st = resolve(opts, &o);
    if (st != TC_OK) return st;
    cudaSetDevice(tc::ctx_device(ctx));
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    unsigned* err = tc::ctx_err(ctx);
    if (n < o.small) {
        grad_int8_kernel<<<1, 1024, 0, s>>>(grad, n, o.chunk, seed, static_cast<uint8_t*>(out), out_cap, out_bytes, err);
        cudaError_t e = cudaGetLastError();
        if (e != cudaSuccess) return cuda_fail(e, "grad_int8 launch");
        tc::ctx_add_launches(ctx, 1);
        return TC_OK;
    }
    SparseParams P = {};
    P.x = grad;
    P.n = n;
    P.chunk = o.chunk;
    P.nblocks = (n + kGB - 1) / kGB;
    P.nchunks = (n + o.chunk - 1) / o.chunk;
    P.seed = seed;
    P.cap = out_cap;
    P.sample = o.sample;
    P.rank = o.rank;
    P.out = static_cast<uint8_t*>(out);
    P.out_bytes = out_bytes;
    P.err = err;
    P.ngroups = (P.nblocks + kGGroup - 1) / kGGroup;
    const size_t o_bc = 16, o_gs = o_bc + pad16u(4 * P.nblocks), o_gp = o_gs + pad16u(8 * P.ngroups);
    const size_t o_cs = o_gp + pad16u(8 * (P.ngroups + 1)), o_sp = o_cs + pad16u(8 * (P.nchunks + 1));
    const size_t need = o_sp + P.nblocks * (kGSpill * 6);
    void* scratch = nullptr;
    st = tc::ctx_grad_scratch(ctx, need, s, &scratch);
    if (st != TC_OK) return st;
    uint8_t* sb = static_cast<uint8_t*>(scratch);
    P.thr = reinterpret_cast<float*>(sb);
    P.bcount = reinterpret_cast<uint32_t*>(sb + o_bc);
    P.gsum = reinterpret_cast<unsigned long long*>(sb + o_gs);
    P.gpre = reinterpret_cast<unsigned long long*>(sb + o_gp);
    P.cstart = reinterpret_cast<unsigned long long*>(sb + o_cs);
    P.spill = sb + o_sp;
    cudaError_t e0 = cudaMemsetAsync(P.gsum, 0, 8 * P.ngroups, s);
    if (e0 != cudaSuccess) return cuda_fail(e0, "cudaMemsetAsync(group sums)");
    // sample -> count and prefix -> emit as programmatic dependent launches (the dependent grid
    // starts while its 1-CTA predecessor runs; griddepcontrol.wait orders the data)
    grad_sample_kernel<<<1, 1024, 0, s>>>(P);
    cudaError_t e = launch_pdl(grad_count_kernel, static_cast<unsigned>(P.nblocks), kGThreads, s, P);
    if (e == cudaSuccess) {
        grad_prefix_kernel<<<1, 1024, 0, s>>>(P);
        e = launch_pdl(grad_emit_kernel, static_cast<unsigned>(P.ngroups), kGThreads, s, P);
    }
    if (e == cudaSuccess) e = cudaGetLastError();
    if (e != cudaSuccess) return cuda_fail(e, "grad compress launch");
    tc::ctx_add_launches(ctx, 4);
    return TC_OK;
}

}  // extern "C"

namespace {
// walker outputs for `count` payloads of n elements: [count] Payload | per payload cpre and tstart
tc_status walk_payloads(tc_ctx* ctx, const void* const* payloads, const uint64_t* bytes, int count, uint64_t n,
                        bool tiles, cudaStream_t s, Payload** dev) {
    uint64_t per = 0;
    // worst case chunk count per payload: the smallest legal chunk (4096)
    const uint64_t max_chunks = n / kGB + 2;
    const uint64_t ntiles = (n + kGB - 1) / kGB;
    per = pad16u(8 * (max_chunks + 1)) + (tiles ? pad16u(8 * (ntiles + 1)) : 0);
    const size_t need = pad16u(sizeof(Payload) * count) + per * count;
    void* scratch = nullptr;
    tc_status st = tc::ctx_grad_scratch(ctx, need, s, &scratch);
    if (st != TC_OK) return st;
    Payload* P = static_cast<Payload*>(scratch);
    uint8_t* area = static_cast<uint8_t*>(scratch) + pad16u(sizeof(Payload) * count);
    for (int j = 0; j < count; ++j) {
        Payload init = {};
        init.cpre = reinterpret_cast<unsigned long long*>(area + per * j);
        init.tstart = tiles ? reinterpret_cast<unsigned long long*>(area + per * j + pad16u(8 * (max_chunks + 1)))
                            : nullptr;
        cudaError_t e = cudaMemcpyAsync(P + j, &init, sizeof(Payload), cudaMemcpyHostToDevice, s);
        if (e != cudaSuccess) return cuda_fail(e, "payload descriptor");
        grad_walk_kernel<<<1, 32, 0, s>>>(static_cast<const uint8_t*>(payloads[j]), bytes[j], n, P + j,
                                           tc::ctx_err(ctx));
        if (tiles) grad_tile_start_kernel<<<grid_for(ctx, ntiles + 1, 256), 256, 0, s>>>(P + j, n, ntiles, tc::ctx_err(ctx));
    }
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return cuda_fail(e, "payload walk launch");
    tc::ctx_add_launches(ctx, static_cast<uint64_t>(count) * (tiles ? 2 : 1));
    *dev = P;
    return TC_OK;
}
}  // namespace

extern "C" {

tc_status tc_grad_decompress(tc_ctx* ctx, const void* payload, uint64_t bytes, float* out, uint64_t n,
                             tc_stream stream) {
    if (!ctx || !payload || !aligned16(payload) || (n && (!out || !aligned16(out))))
        return fail(TC_ERR_INVALID, "bad arguments (ctx, 16-byte aligned payload / out)");
    cudaSetDevice(tc::ctx_device(ctx));
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    // the variant is only known on the device: both the dequantize pass (INT8) and the tile
    // expansion (sparse) are launched; each returns at once for the other variant
    Payload* P = nullptr;
    tc_status st = walk_payloads(ctx, &payload, &bytes, 1, n, n >= 1, s, &P);
    if (st != TC_OK) return st;
    const uint64_t tiles = (n + kGB - 1) / kGB;
    grad_decompress_kernel<<<grid_for(ctx, n, 256), 256, 0, s>>>(P, n, out, tc::ctx_err(ctx));
    grad_expand_kernel<<<grid_for(ctx, tiles * kGThreads, kGThreads), kGThreads, 0, s>>>(P, n, tiles, out,
                                                                                        tc::ctx_err(ctx));
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return cuda_fail(e, "grad decompress launch");
    tc::ctx_add_launches(ctx, 2);
    return TC_OK;
}

tc_status tc_adam_step(tc_ctx* ctx, const tc_adam_state* stt, const float* grad, const tc_adam_hp* hp, uint64_t step,
                       tc_stream stream) {
    if (!ctx || step == 0) return fail(TC_ERR_INVALID, "ctx is NULL or step == 0 (steps are 1-based)");
    tc_status st = check_state(stt);
    if (st != TC_OK) return st;
    if (!stt->n) return TC_OK;
    if (!grad) return fail(TC_ERR_INVALID, "grad is NULL");
    cudaSetDevice(tc::ctx_device(ctx));
    float ss, ic;
    bias(hp, step, &ss, &ic);
    if (!aligned16(grad)) return fail(TC_ERR_INVALID, "grad must be 16-byte aligned");
    adam_step_kernel<<<grid_for(ctx, stt->n / 4 + 1, 256), 256, 0, static_cast<cudaStream_t>(stream)>>>(
        stt->master, stt->m, stt->v, stt->w16, stt->n, grad, adam_consts(hp), ss, ic);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return cuda_fail(e, "adam step launch");
    tc::ctx_add_launches(ctx, 1);
    return TC_OK;
}

tc_status tc_adam_replay(tc_ctx* ctx, const tc_adam_state* stt, const void* const* payloads,
                         const uint64_t* payload_bytes, int n_payloads, const tc_adam_hp* hp, uint64_t first_step,
                         float* scratch, tc_stream stream) {
    if (!ctx || first_step == 0) return fail(TC_ERR_INVALID, "ctx is NULL or first_step == 0");
    if (!payloads || !payload_bytes || n_payloads < 1 || n_payloads > TC_MAX_FOLD)
        return fail(TC_ERR_INVALID, "n_payloads must be in [1, TC_MAX_FOLD]");
    tc_status st = check_state(stt);
    if (st != TC_OK) return st;
    if (stt->n && (!scratch || !aligned16(scratch))) return fail(TC_ERR_INVALID, "scratch must be a 16-byte aligned device buffer");
    for (int j = 0; j < n_payloads; ++j)
        if (!payloads[j] || !aligned16(payloads[j])) return fail(TC_ERR_INVALID, "payload pointers must be 16-byte aligned");
    cudaSetDevice(tc::ctx_device(ctx));
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    const int nf = n_payloads - 1;
    if (nf > 0 && stt->n) {
        Payload* P = nullptr;
        st = walk_payloads(ctx, payloads, payload_bytes, nf, stt->n, true, s, &P);
        if (st != TC_OK) return st;
        ReplayParams R = {};
        R.master = stt->master;
        R.m = stt->m;
        R.v = stt->v;
        R.n = stt->n;
        R.tiles = (stt->n + kGB - 1) / kGB;
        R.nsteps = nf;
        R.a = adam_consts(hp);
        for (int j = 0; j < nf; ++j) bias(hp, first_step + j, &R.ss[j], &R.ic[j]);
        R.pay = P;
        R.err = tc::ctx_err(ctx);
        static bool attr[tc::TC_MAX_DEVICES] = {};  // a function attribute is per device
        const int dev = tc::ctx_device(ctx);
        if (dev < 0 || dev >= tc::TC_MAX_DEVICES || !attr[dev]) {
            cudaFuncSetAttribute(adam_replay_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 static_cast<int>(kRDynSmem));
            if (dev >= 0 && dev < tc::TC_MAX_DEVICES) attr[dev] = true;
        }
        adam_replay_kernel<<<grid_for(ctx, R.tiles * kRThreads, kRThreads), kRThreads, kRDynSmem, s>>>(R);
        cudaError_t e = cudaGetLastError();
        if (e != cudaSuccess) return cuda_fail(e, "adam replay launch");
        tc::ctx_add_launches(ctx, 1);
    }
    // the last step through the native path
    st = tc_grad_decompress(ctx, payloads[nf], payload_bytes[nf], scratch, stt->n, stream);
    if (st != TC_OK) return st;
    return tc_adam_step(ctx, stt, scratch, hp, first_step + nf, stream);
}

static tc_status adam_step_encode_full(tc_ctx* ctx, const tc_adam_state* stt, const float* grad, const tc_adam_hp* hp,
                                       uint64_t step, const tc_encode_opts& o, void* out, uint64_t out_cap,
                                       uint64_t* out_bytes, cudaStream_t s);

tc_status tc_adam_step_encode(tc_ctx* ctx, const tc_adam_state* stt, const float* grad, const tc_adam_hp* hp,
                              uint64_t step, const tc_encode_opts* opts, void* out, uint64_t out_cap,
                              uint64_t* out_bytes, tc_stream stream) {
    if (!ctx || step == 0) return fail(TC_ERR_INVALID, "ctx is NULL or step == 0 (steps are 1-based)");
    tc_status st = check_state(stt);
    if (st != TC_OK) return st;
    if (!out || !aligned16(out) || !out_bytes) return fail(TC_ERR_INVALID, "out must be 16-byte aligned; out_bytes set");
    if (stt->n && (!grad || !aligned16(grad))) return fail(TC_ERR_INVALID, "grad is NULL or not 16-byte aligned");
    cudaSetDevice(tc::ctx_device(ctx));
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    if (opts && opts->index_mode == 2) {  // full records: one pass (the options are checked as usual)
        tc_encode_opts o = *opts;
        uint64_t bound = 0;
        tc_segment lay[4] = {{nullptr, nullptr, stt->n, 2, 0}, {nullptr, nullptr, stt->n, 4, 0},
                             {nullptr, nullptr, stt->n, 4, 0}, {nullptr, nullptr, stt->n, 4, 0}};
        st = tc_diff_bound(lay, 4, &o, &bound);  // validates T, C, the format
        if (st != TC_OK) return st;
        return adam_step_encode_full(ctx, stt, grad, hp, step, o, out, out_cap, out_bytes, s);
    }
    const uint64_t n = stt->n, words = (n + 31) / 32;
    const size_t per = pad16u(4 * (words ? words : 1));
    void* scratch = nullptr;
    st = tc::ctx_grad_scratch(ctx, 4 * per, s, &scratch);
    if (st != TC_OK) return st;
    uint32_t* mk[4];
    for (int k = 0; k < 4; ++k) mk[k] = reinterpret_cast<uint32_t*>(static_cast<uint8_t*>(scratch) + k * per);
    if (n) {
        float ss, ic;
        bias(hp, step, &ss, &ic);
        adam_mask_kernel<<<grid_for(ctx, (n + 3) / 4, 256), 256, 0, s>>>(stt->master, stt->m, stt->v, stt->w16, n, grad,
                                                                         adam_consts(hp), ss, ic, mk[0], mk[1], mk[2],
                                                                         mk[3]);
        cudaError_t e = cudaGetLastError();
        if (e != cudaSuccess) return cuda_fail(e, "adam mask launch");
        tc::ctx_add_launches(ctx, 1);
    }
    tc_segment segs[4] = {{nullptr, stt->w16, n, 2, 0}, {nullptr, stt->master, n, 4, 0},
                          {nullptr, stt->m, n, 4, 0}, {nullptr, stt->v, n, 4, 0}};
    const uint32_t* const masks[4] = {mk[0], mk[1], mk[2], mk[3]};
    return tc::encode_from_masks(ctx, segs, masks, 4, opts, step, step - 1, out, out_cap, out_bytes, s);
}

// full-format records: the state and the record in one pass (adam_full_kernel)
static tc_status adam_step_encode_full(tc_ctx* ctx, const tc_adam_state* stt, const float* grad, const tc_adam_hp* hp,
                                       uint64_t step, const tc_encode_opts& o, void* out, uint64_t out_cap,
                                       uint64_t* out_bytes, cudaStream_t s) {
    const uint64_t n = stt->n, C = o.chunk_words;
    AdamFullLayout L;
    uint64_t pos = 0;
    for (int k = 0; k < 4; ++k) {
        const uint64_t w = k == 0 ? 2 : 4;
        L.base[k] = pos;
        L.rec_full[k] = kHdr + pad16u(w * C);
        const uint64_t chunks = n ? (n + C - 1) / C : 1;
        const uint64_t mlast = n ? n - (chunks - 1) * C : 0;
        pos += (chunks - 1) * L.rec_full[k] + kHdr + pad16u(w * mlast);
    }
    L.C = C;
    L.total = pos;
    L.version = step;
    L.ref_version = step - 1;
    L.T = o.tile_words;
    float ss, ic;
    bias(hp, step, &ss, &ic);
    adam_full_kernel<<<grid_for(ctx, (n + 3) / 4 + 1, 256), 256, 0, s>>>(
        stt->master, stt->m, stt->v, stt->w16, n, grad, adam_consts(hp), ss, ic, static_cast<uint8_t*>(out), out_cap,
        out_bytes, L, tc::ctx_err(ctx));
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return cuda_fail(e, "adam full launch");
    tc::ctx_add_launches(ctx, 1);
    return TC_OK;
}

}  // extern "C"
