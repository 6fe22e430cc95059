// tc_synth.cu — device twin of synth/__init__.py (bench/test INPUT generation only; it is not
// part of the codec and never runs inside a timed region).  Recipe: include/tc_synth.h.
#include <cuda_runtime.h>

#include "../../include/tc_synth.h"
#include "tc_internal.h"

namespace {

__host__ __device__ __forceinline__ uint64_t splitmix(uint64_t x) {
    uint64_t z = x + 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

uint64_t key(uint64_t seed, uint32_t seg, uint64_t t) {
    return splitmix(seed ^ (static_cast<uint64_t>(seg) << 56) ^ (t << 32));
}

template <typename W>
__global__ void synth_base_kernel(W* dst, uint64_t n, uint64_t k, uint64_t start) {
    for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<uint64_t>(gridDim.x) * blockDim.x)
        dst[i] = static_cast<W>(splitmix(k + start + i));
}

template <typename W>
__global__ void synth_step_kernel(W* words, uint64_t n, uint64_t kc, uint64_t kv, uint64_t p53, int structure,
                                  uint64_t start, uint32_t lowmask) {
    for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        const uint64_t gi = start + i;
        const uint64_t jj = structure ? (gi >> 12) : gi;
        if ((splitmix(jj + kc) >> 11) < p53) {
            const uint64_t r = splitmix(gi + kv);
            words[i] = static_cast<W>(words[i] ^ static_cast<W>((r & lowmask) | 1u));
        }
    }
}

unsigned grid_for(uint64_t n) {
    uint64_t g = (n + 255) / 256;
    if (g > 148ull * 64) g = 148ull * 64;
    return g ? static_cast<unsigned>(g) : 1u;
}

}  // namespace

extern "C" {

tc_status tc_synth_base(void* dst, uint64_t n, uint32_t word_bytes, uint64_t seed, uint32_t seg, uint64_t start,
                        tc_stream stream) {
    if (n == 0) return TC_OK;
    if (!dst || (word_bytes != 2 && word_bytes != 4)) return TC_ERR_INVALID;
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    const uint64_t k = key(seed, seg, 0);
    if (word_bytes == 4)
        synth_base_kernel<uint32_t><<<grid_for(n), 256, 0, s>>>(static_cast<uint32_t*>(dst), n, k, start);
    else
        synth_base_kernel<uint16_t><<<grid_for(n), 256, 0, s>>>(static_cast<uint16_t*>(dst), n, k, start);
    return cudaGetLastError() == cudaSuccess ? TC_OK : TC_ERR_CUDA;
}

tc_status tc_synth_step(void* words, uint64_t n, uint32_t word_bytes, uint64_t seed, uint32_t seg, uint64_t t,
                        uint64_t p53, int structure, uint64_t start, tc_stream stream) {
    if (n == 0) return TC_OK;
    if (!words || (word_bytes != 2 && word_bytes != 4)) return TC_ERR_INVALID;
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    const uint64_t k = key(seed, seg, t);
    const uint64_t kc = k ^ 0xC0FFEEull, kv = k ^ 0xBEEFull;
    if (word_bytes == 4)
        synth_step_kernel<uint32_t><<<grid_for(n), 256, 0, s>>>(static_cast<uint32_t*>(words), n, kc, kv, p53,
                                                                 structure, start, 0xFFFFu);
    else
        synth_step_kernel<uint16_t><<<grid_for(n), 256, 0, s>>>(static_cast<uint16_t*>(words), n, kc, kv, p53,
                                                                 structure, start, 0xFu);
    return cudaGetLastError() == cudaSuccess ? TC_OK : TC_ERR_CUDA;
}

}  // extern "C"
