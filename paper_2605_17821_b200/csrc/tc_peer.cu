// tc_peer.cu — Tier-2 replication by device-initiated NVLink stores into the ring neighbour's
// memory: no NCCL, no host-side size exchange.
//
// PAPER.md:184 §3.1 — each rank backs up its checkpoint to its ring neighbour
// §3.2 — "Peer ranks first exchange their serialized payload sizes": here the size travels in
// the mailbox with the payload, and a record that does not fit the neighbour's slot is refused
// (the receiver sees TC_ERR_CAPACITY).  The receiver's slot and mailbox are cudaMalloc'ed in
// its own HBM and mapped into the sender with CUDA IPC (one process per GPU, one NVSwitch box).
#include <cuda_runtime.h>

#include <cstring>
#include <string>

#include "tc_internal.h"

namespace {

constexpr uint32_t kPushThreads = 512;
constexpr int kPushDepth = 8;  // 16-byte loads in flight per thread before their remote stores
constexpr int kPushCtas = 32;  // enough stores in flight for NVLink; leaves the SMs to the encode / fold
constexpr uint32_t kWaitSpinLimit = 1u << 22;  // x ~2 us sleep: ~10 s watchdog

tc_status fail(tc_status s, const std::string& msg) {
    tc::set_error(msg);
    return s;
}
tc_status cuda_fail(cudaError_t e, const char* what) {
    tc::set_error(std::string(what) + ": " + cudaGetErrorString(e));
    return e == cudaErrorMemoryAllocation ? TC_ERR_NOMEM : TC_ERR_CUDA;
}
bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

__device__ __forceinline__ void st_release_sys(unsigned long long* p, unsigned long long v) {
    asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ void st_relaxed_sys(unsigned long long* p, unsigned long long v) {
    asm volatile("st.relaxed.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long ld_acquire_sys(const unsigned long long* p) {
    unsigned long long v;
    asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ unsigned long long ld_relaxed_sys(const unsigned long long* p) {
    unsigned long long v;
    asm volatile("ld.relaxed.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}

// Grid-stride copy of the record, kPushDepth independent 16-byte loads in flight per thread before their
// (remote) stores; every block fences at system scope and counts itself out, the last one
// publishes {bytes, version} with a release store into the peer's mailbox.
__global__ void __launch_bounds__(kPushThreads) push_kernel(const uint4* __restrict__ src, const uint64_t* src_bytes,
                                                            uint4* dst, uint64_t cap, unsigned long long* mail,
                                                            uint64_t version, unsigned int* counter) {
    const uint64_t nb = *reinterpret_cast<const volatile uint64_t*>(src_bytes);
    const bool fits = nb <= cap;
    if (fits) {
        const uint64_t n = nb / 16;
        const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
        uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
        for (; i + (kPushDepth - 1) * stride < n; i += kPushDepth * stride) {
            uint4 v[kPushDepth];
#pragma unroll
            for (int q = 0; q < kPushDepth; ++q) v[q] = __ldg(src + i + q * stride);
#pragma unroll
            for (int q = 0; q < kPushDepth; ++q) dst[i + q * stride] = v[q];
        }
        for (; i < n; i += stride) dst[i] = __ldg(src + i);
        // the last nb % 16 bytes (records are 16-byte padded, but a caller's payload need not be)
        const uint32_t tail = static_cast<uint32_t>(nb & 15u);
        if (tail && blockIdx.x == gridDim.x - 1 && threadIdx.x < tail)
            reinterpret_cast<uint8_t*>(dst + n)[threadIdx.x] = reinterpret_cast<const uint8_t*>(src + n)[threadIdx.x];
    }
    __threadfence_system();
    __syncthreads();
    if (threadIdx.x == 0) {
        const unsigned prev = atomicAdd(counter, 1u);
        if (prev == gridDim.x - 1) {  // every block's stores are fenced: publish
            *counter = 0u;             // ready for the next push on this ctx (stream-ordered)
            __threadfence_system();
            st_relaxed_sys(mail, fits ? nb : ~0ull);
            st_release_sys(mail + 1, version);
        }
    }
}

__global__ void peer_wait_kernel(const unsigned long long* mail, uint64_t version, uint64_t* bytes_out,
                                 unsigned int* err) {
    for (uint32_t it = 0;; ++it) {
        if (ld_acquire_sys(mail + 1) == version) break;
        if (it >= kWaitSpinLimit) {
            tc_set_err(err, TC_ERR_INTERNAL);
            return;
        }
        __nanosleep(2000);
    }
    unsigned long long b = ld_relaxed_sys(mail);
    if (b == ~0ull) {
        tc_set_err(err, TC_ERR_CAPACITY);
        b = 0;
    }
    if (bytes_out) *reinterpret_cast<volatile uint64_t*>(bytes_out) = b;
}

}  // namespace

extern "C" {

tc_status tc_ipc_alloc(uint64_t bytes, void** dev_ptr, uint8_t handle[TC_IPC_HANDLE_BYTES]) {
    if (!dev_ptr || !handle || bytes == 0) return fail(TC_ERR_INVALID, "bad arguments");
    static_assert(sizeof(cudaIpcMemHandle_t) == TC_IPC_HANDLE_BYTES, "IPC handle size");
    void* p = nullptr;
    cudaError_t e = cudaMalloc(&p, bytes);
    if (e != cudaSuccess) return cuda_fail(e, "cudaMalloc");
    e = cudaMemset(p, 0, bytes);
    cudaIpcMemHandle_t h;
    if (e == cudaSuccess) e = cudaIpcGetMemHandle(&h, p);
    if (e != cudaSuccess) {
        cudaFree(p);
        return cuda_fail(e, "cudaIpcGetMemHandle");
    }
    std::memcpy(handle, &h, sizeof(h));
    *dev_ptr = p;
    return TC_OK;
}

tc_status tc_ipc_free(void* dev_ptr) {
    if (!dev_ptr) return TC_OK;
    cudaError_t e = cudaFree(dev_ptr);
    return e == cudaSuccess ? TC_OK : cuda_fail(e, "cudaFree");
}

tc_status tc_ipc_open(const uint8_t handle[TC_IPC_HANDLE_BYTES], void** dev_ptr) {
    if (!handle || !dev_ptr) return fail(TC_ERR_INVALID, "bad arguments");
    cudaIpcMemHandle_t h;
    std::memcpy(&h, handle, sizeof(h));
    void* p = nullptr;
    cudaError_t e = cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess);
    if (e != cudaSuccess) return cuda_fail(e, "cudaIpcOpenMemHandle");
    *dev_ptr = p;
    return TC_OK;
}

tc_status tc_ipc_close(void* dev_ptr) {
    if (!dev_ptr) return TC_OK;
    cudaError_t e = cudaIpcCloseMemHandle(dev_ptr);
    return e == cudaSuccess ? TC_OK : cuda_fail(e, "cudaIpcCloseMemHandle");
}

tc_status tc_push_peer(tc_ctx* ctx, const void* src, const uint64_t* src_bytes, void* peer_dst, uint64_t peer_cap,
                       void* peer_mailbox, uint64_t version, tc_stream stream) {
    if (!ctx) return fail(TC_ERR_INVALID, "ctx is NULL");
    if (!src || !aligned16(src) || !peer_dst || !aligned16(peer_dst))
        return fail(TC_ERR_INVALID, "src / peer_dst must be 16-byte aligned device pointers");
    if (!src_bytes || !peer_mailbox || !aligned16(peer_mailbox))
        return fail(TC_ERR_INVALID, "src_bytes / peer_mailbox missing or misaligned");
    if (version == 0) return fail(TC_ERR_INVALID, "version must be >= 1");
    cudaSetDevice(tc::ctx_device(ctx));
    const int ctas = tc::ctx_push_ctas(ctx) ? static_cast<int>(tc::ctx_push_ctas(ctx)) : kPushCtas;
    push_kernel<<<ctas, kPushThreads, 0, static_cast<cudaStream_t>(stream)>>>(
        static_cast<const uint4*>(src), src_bytes, static_cast<uint4*>(peer_dst), peer_cap,
        static_cast<unsigned long long*>(peer_mailbox), version, tc::ctx_err(ctx) + 1);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return cuda_fail(e, "push launch");
    tc::ctx_add_launches(ctx, 1);
    return TC_OK;
}

tc_status tc_diff_encode_push(tc_ctx* ctx, const tc_segment* segs, int nseg, const tc_encode_opts* opts,
                              uint64_t version, uint64_t ref_version, void* out, uint64_t out_cap,
                              uint64_t* out_bytes, void* peer_dst, uint64_t peer_cap, void* peer_mailbox,
                              tc_stream stream) {
    if (!peer_dst || !aligned16(peer_dst) || !peer_mailbox || !aligned16(peer_mailbox))
        return fail(TC_ERR_INVALID, "peer_dst / peer_mailbox must be 16-byte aligned device pointers");
    if (version == 0) return fail(TC_ERR_INVALID, "version must be >= 1");
    return tc::encode_push(ctx, segs, nseg, opts, version, ref_version, out, out_cap, out_bytes, peer_dst, peer_cap,
                           peer_mailbox, static_cast<cudaStream_t>(stream));
}

tc_status tc_peer_wait(tc_ctx* ctx, const void* mailbox, uint64_t version, uint64_t* bytes_out, tc_stream stream) {
    if (!ctx) return fail(TC_ERR_INVALID, "ctx is NULL");
    if (!mailbox || !aligned16(mailbox)) return fail(TC_ERR_INVALID, "mailbox must be a 16-byte aligned device pointer");
    if (version == 0) return fail(TC_ERR_INVALID, "version must be >= 1");
    cudaSetDevice(tc::ctx_device(ctx));
    peer_wait_kernel<<<1, 1, 0, static_cast<cudaStream_t>(stream)>>>(
        static_cast<const unsigned long long*>(mailbox), version, bytes_out, tc::ctx_err(ctx));
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return cuda_fail(e, "peer wait launch");
    tc::ctx_add_launches(ctx, 1);
    return TC_OK;
}

}  // extern "C"
