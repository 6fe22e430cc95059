// fold_probe.cu — DRAM-pattern probe for the restore fold's write-back (not product code).
//
// Question: at the union change density p of a fold (N = 1 at f = 1 %: p = 0.01; N = 8: p = 0.077),
// what does it cost to write the changed 4-byte words of a large fp32 state, by access pattern?
//   masked   : a warp per 128-byte line, each lane stores its word iff changed (partial sectors;
//              L2 must merge / fill them)
//   rmw16    : a thread per 16 bytes; a 32-byte sector that holds a change is loaded, patched and
//              stored whole (explicit read-modify-write of the touched sectors only)
//   stream   : read every line, store the 128-byte lines that hold a change (round 1 list fold)
//   copy     : read all, write all (the streaming ceiling)
//   scatter  : the pure scattered store of an index record's entries — sorted u32 positions and
//              values read coalesced, one 4-byte store per entry (no record parsing): the floor of
//              an N = 1 fold at that density (positions: one per stride 1/p, jittered in it)
// The change pattern is a splitmix64 hash of the word index (i.i.d. Bernoulli(p)).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fold_probe tools/fold_probe.cu
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

#include <algorithm>
#include <vector>

__device__ __forceinline__ uint64_t h64(uint64_t x) {
    x += 0x9E3779B97F4A7C15ull;
    x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
    x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
    return x ^ (x >> 31);
}
__device__ const uint32_t* g_mask;  // precomputed change mask (bit i of word i/32)
__device__ __forceinline__ bool chg(uint64_t i, uint64_t) { return (__ldg(g_mask + (i >> 5)) >> (i & 31)) & 1u; }
__global__ void k_gen(uint32_t* m, uint64_t nw, uint64_t thr) {
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t w = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; w < nw; w += stride) {
        uint32_t b = 0;
        for (int k = 0; k < 32; ++k) b |= ((h64(32 * w + k) >> 11) < thr) ? 1u << k : 0u;
        m[w] = b;
    }
}

__global__ void k_masked(uint32_t* s, uint64_t n, uint64_t thr) {
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride)
        if (chg(i, thr)) s[i] = (uint32_t)i;
}

// 4 vectors per thread per iteration, loads before stores
__global__ void k_rmw16(uint4* s, uint64_t nv, uint64_t thr) {
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x * 4;
    for (uint64_t v0 = ((uint64_t)blockIdx.x * blockDim.x) * 4 + threadIdx.x; v0 < nv; v0 += stride) {
        uint32_t bits[4];
        bool touch[4];
        uint4 x[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const uint64_t v = v0 + (uint64_t)q * blockDim.x;
            uint32_t b = 0;
            if (v < nv)
                for (int k = 0; k < 4; ++k) b |= chg(4 * v + k, thr) ? 1u << k : 0u;
            bits[q] = b;
            const uint32_t pb = __shfl_xor_sync(0xffffffffu, b, 1);
            touch[q] = (b | pb) != 0;
            if (touch[q]) x[q] = s[v];
        }
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const uint64_t v = v0 + (uint64_t)q * blockDim.x;
            if (!touch[q]) continue;
            if (bits[q] & 1) x[q].x = (uint32_t)(4 * v);
            if (bits[q] & 2) x[q].y = (uint32_t)(4 * v + 1);
            if (bits[q] & 4) x[q].z = (uint32_t)(4 * v + 2);
            if (bits[q] & 8) x[q].w = (uint32_t)(4 * v + 3);
            s[v] = x[q];
        }
    }
}

// sector-granular write of the touched sectors WITHOUT reading them (the write floor only)
__global__ void k_wsect(uint4* s, uint64_t nv, uint64_t thr) {
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t v = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; v < nv; v += stride) {
        uint32_t b = 0;
        for (int k = 0; k < 4; ++k) b |= chg(4 * v + k, thr) ? 1u << k : 0u;
        const uint32_t pb = __shfl_xor_sync(0xffffffffu, b, 1);
        if (b | pb) s[v] = make_uint4((uint32_t)v, 1, 2, 3);
    }
}

__global__ void k_stream(uint4* s, uint64_t nv, uint64_t thr) {
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x * 4;
    for (uint64_t v0 = ((uint64_t)blockIdx.x * blockDim.x) * 4 + threadIdx.x; v0 < nv; v0 += stride) {
        uint4 x[4];
        uint32_t bits[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const uint64_t v = v0 + (uint64_t)q * blockDim.x;
            if (v < nv) x[q] = s[v];
            uint32_t b = 0;
            if (v < nv)
                for (int k = 0; k < 4; ++k) b |= chg(4 * v + k, thr) ? 1u << k : 0u;
            bits[q] = b;
        }
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const uint64_t v = v0 + (uint64_t)q * blockDim.x;
            // the 128-byte line = 8 lanes
            uint32_t any = bits[q];
            any |= __shfl_xor_sync(0xffffffffu, any, 1);
            any |= __shfl_xor_sync(0xffffffffu, any, 2);
            any |= __shfl_xor_sync(0xffffffffu, any, 4);
            if (v >= nv || !any) continue;
            if (bits[q] & 1) x[q].x = (uint32_t)(4 * v);
            if (bits[q] & 2) x[q].y = (uint32_t)(4 * v + 1);
            if (bits[q] & 4) x[q].z = (uint32_t)(4 * v + 2);
            if (bits[q] & 8) x[q].w = (uint32_t)(4 * v + 3);
            s[v] = x[q];
        }
    }
}

__global__ void k_copy(const uint4* a, uint4* b, uint64_t nv) {
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t v = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; v < nv; v += stride) b[v] = a[v];
}

__global__ void k_gen_entries(uint32_t* pos, uint32_t* val, uint64_t ne, uint64_t stride) {
    const uint64_t st = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < ne; i += st) {
        pos[i] = (uint32_t)(i * stride + h64(i) % stride);
        val[i] = (uint32_t)i;
    }
}
__global__ void k_scatter(uint32_t* s, const uint32_t* pos, const uint32_t* val, uint64_t ne) {
    const uint64_t st = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < ne; i += st) s[__ldg(pos + i)] = __ldg(val + i);
}

// hash-only pass (ALU cost of the pattern generator, no memory)
__global__ void k_hash(uint64_t n, uint64_t thr, uint32_t* sink) {
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    uint32_t c = 0;
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) c += chg(i, thr);
    if (c == 0xffffffffu) *sink = c;
}

int main(int argc, char** argv) {
    const uint64_t n = argc > 1 ? strtoull(argv[1], 0, 10) : (4ull << 30);  // fp32 words (16 GiB)
    const double ps[] = {0.01, 0.0773, 0.3};
    uint32_t* s;
    uint32_t* d2;
    if (cudaMalloc(&s, n * 4) != cudaSuccess || cudaMalloc(&d2, n * 4) != cudaSuccess) {
        printf("alloc failed\n");
        return 1;
    }
    cudaMemset(s, 0, n * 4);
    uint32_t* mk;
    cudaMalloc(&mk, n / 8);
    cudaMemcpyToSymbol(g_mask, &mk, sizeof(mk));
    cudaMemset(d2, 0, n * 4);
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const int grid = sms * 8, block = 256;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    auto timeit = [&](auto fn) {
        std::vector<float> t;
        for (int r = 0; r < 6; ++r) {
            cudaEventRecord(e0);
            fn();
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            if (r) t.push_back(ms);
        }
        std::sort(t.begin(), t.end());
        return t[t.size() / 2];
    };
    const double W = n * 4.0;
    float tc = timeit([&] { k_copy<<<grid, block>>>((const uint4*)s, (uint4*)d2, n / 4); });
    printf("copy      : %8.3f ms  %7.1f GB/s (read+write)\n", tc, 2 * W / tc / 1e6);
    for (double p : ps) {
        const uint64_t thr = (uint64_t)(p * 9007199254740992.0);
        const double sect = 1.0 - pow(1.0 - p, 8), line = 1.0 - pow(1.0 - p, 32);
        k_gen<<<grid, block>>>(mk, n / 32, thr);
        cudaDeviceSynchronize();
        float th = 0;
        float tm = timeit([&] { k_masked<<<grid, block>>>(s, n, thr); });
        float tr = timeit([&] { k_rmw16<<<grid, block>>>((uint4*)s, n / 4, thr); });
        float tw = timeit([&] { k_wsect<<<grid, block>>>((uint4*)s, n / 4, thr); });
        float ts = timeit([&] { k_stream<<<grid, block>>>((uint4*)s, n / 4, thr); });
        const double ts_b = sect * W;  // touched-sector bytes
        printf("p=%.4f touched sectors %.3f (%.2f GB) lines %.3f | mask %.2f GB\n", p, sect, ts_b / 1e9, line, n / 8 / 1e9);
        printf("  masked  : %8.3f ms  touched-sector RMW %7.1f GB/s\n", tm, 2 * ts_b / tm / 1e6);
        printf("  rmw16   : %8.3f ms  touched-sector RMW %7.1f GB/s\n", tr, 2 * ts_b / tr / 1e6);
        printf("  wsect   : %8.3f ms  touched-sector W   %7.1f GB/s\n", tw, ts_b / tw / 1e6);
        printf("  stream  : %8.3f ms  R all + W lines    %7.1f GB/s\n", ts, (W + line * W) / ts / 1e6);
    }
    // the pure scatter of an index record's entries (u32 positions: n < 2^32 words)
    if (n < (1ull << 32)) {
        for (double p : {0.001, 0.01, 0.03}) {
            const uint64_t stride = (uint64_t)(1.0 / p + 0.5), ne = n / stride;
            uint32_t *pos, *val;
            if (cudaMalloc(&pos, ne * 4) != cudaSuccess || cudaMalloc(&val, ne * 4) != cudaSuccess) break;
            k_gen_entries<<<grid, block>>>(pos, val, ne, stride);
            cudaDeviceSynchronize();
            float tsc = timeit([&] { k_scatter<<<grid, block>>>(s, pos, val, ne); });
            printf("scatter p=%.3f: %llu entries %8.3f ms  %6.2f G entries/s  (entries 8 B read + 32-B sector fill + write-back each: %7.1f GB/s)\n",
                   p, (unsigned long long)ne, tsc, ne / tsc / 1e6, ne * 72.0 / tsc / 1e6);
            cudaFree(pos);
            cudaFree(val);
        }
    }
    cudaError_t e = cudaDeviceSynchronize();
    printf("%s\n", cudaGetErrorString(e));
    return e != cudaSuccess;
}
