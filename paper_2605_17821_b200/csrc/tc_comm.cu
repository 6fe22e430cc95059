// tc_comm.cu — Tier-2 ring-neighbour replication over NCCL send/recv (NVLink 5 / NVSwitch).
//
// PAPER.md:184 §3.1 — "each rank backs up its checkpoint to the corresponding rank on an
// adjacent machine through a node-level ring mapping"; on one NVSwitch box the failure domain
// is the GPU, so the ring is r -> (r+1) mod P.  PAPER.md:209 §3.2 — "Peer
// ranks first exchange their serialized payload sizes": an 8-byte exchange precedes the
// payload.  PAPER.md:317 §4 — Tier-2 uses "isolated communication groups": libtc owns its own
// ncclComm_t, created from a unique id the caller broadcasts (torch.distributed in the binding).
#include <cuda_runtime.h>
#include <nccl.h>

#include <string>

#include "tc_internal.h"

struct tc_comm {
    ncclComm_t nccl = nullptr;
    int nranks = 0, rank = 0, device = 0;
    uint64_t* dev_sizes = nullptr;   // device [0] peer size, [1] dst's cap, [2] my cap, [3] my size
    uint64_t* host_sizes = nullptr;  // pinned mirror of dev_sizes
};

namespace {

// Stage the size-exchange words on the comm stream: dev[2] = my receive capacity, dev[3] = my
// payload size read from `send_bytes` (device memory or mapped pinned host memory, as written
// by tc_diff_encode) — a kernel, so no copy engine sits on the replication path.
__global__ void stage_sizes_kernel(uint64_t* dev, const uint64_t* send_bytes, uint64_t cap) {
    dev[2] = cap;
    dev[3] = *reinterpret_cast<const volatile uint64_t*>(send_bytes);
}

// Export the exchanged words to mapped pinned host memory with a kernel, not a D2H copy: a copy
// would queue behind multi-GB Tier-1 staging copies on the same copy engine.
__global__ void export_sizes_kernel(volatile uint64_t* host, const uint64_t* dev) {
    if (threadIdx.x < 4) host[threadIdx.x] = dev[threadIdx.x];
    __threadfence_system();
}

tc_status nccl_fail(ncclResult_t r, const char* what) {
    tc::set_error(std::string(what) + ": " + ncclGetErrorString(r));
    if (r == ncclRemoteError || r == ncclSystemError) return TC_ERR_UNAVAILABLE;
    return TC_ERR_NCCL;
}

tc_status check_async(tc_comm* c) {
    ncclResult_t ar = ncclSuccess;
    ncclResult_t r = ncclCommGetAsyncError(c->nccl, &ar);
    if (r != ncclSuccess) return nccl_fail(r, "ncclCommGetAsyncError");
    if (ar != ncclSuccess && ar != ncclInProgress) {
        tc::set_error(std::string("NCCL async error: ") + ncclGetErrorString(ar));
        return TC_ERR_UNAVAILABLE;
    }
    return TC_OK;
}

}  // namespace

extern "C" {

tc_status tc_comm_get_unique_id(uint8_t id[128]) {
    static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId size");
    if (!id) {
        tc::set_error("id is NULL");
        return TC_ERR_INVALID;
    }
    ncclUniqueId u;
    ncclResult_t r = ncclGetUniqueId(&u);
    if (r != ncclSuccess) return nccl_fail(r, "ncclGetUniqueId");
    memcpy(id, &u, 128);
    return TC_OK;
}

tc_status tc_comm_init(int nranks, int rank, int device, const uint8_t id[128], tc_comm** out) {
    if (!out || !id || nranks < 1 || rank < 0 || rank >= nranks) {
        tc::set_error("bad tc_comm_init arguments");
        return TC_ERR_INVALID;
    }
    *out = nullptr;
    cudaError_t e = cudaSetDevice(device);
    if (e != cudaSuccess) {
        tc::set_error(std::string("cudaSetDevice: ") + cudaGetErrorString(e));
        return TC_ERR_CUDA;
    }
    tc_comm* c = new tc_comm();
    c->nranks = nranks;
    c->rank = rank;
    c->device = device;
    ncclUniqueId u;
    memcpy(&u, id, 128);
    ncclResult_t r = ncclCommInitRank(&c->nccl, nranks, u, rank);
    if (r != ncclSuccess) {
        delete c;
        return nccl_fail(r, "ncclCommInitRank");
    }
    if (cudaMalloc(reinterpret_cast<void**>(&c->dev_sizes), 32) != cudaSuccess ||
        cudaHostAlloc(reinterpret_cast<void**>(&c->host_sizes), 32, cudaHostAllocMapped | cudaHostAllocPortable) != cudaSuccess) {
        ncclCommDestroy(c->nccl);
        delete c;
        tc::set_error("allocation of size-exchange buffers failed");
        return TC_ERR_NOMEM;
    }
    *out = c;
    return TC_OK;
}

tc_status tc_comm_destroy(tc_comm* c) {
    if (!c) return TC_OK;
    cudaSetDevice(c->device);
    if (c->nccl) ncclCommDestroy(c->nccl);
    if (c->dev_sizes) cudaFree(c->dev_sizes);
    if (c->host_sizes) cudaFreeHost(c->host_sizes);
    delete c;
    return TC_OK;
}

tc_status tc_replicate_peer(tc_comm* c, const void* send, const uint64_t* send_bytes, void* recv,
                            uint64_t recv_cap, uint64_t* recv_bytes, int direction, tc_stream comm_stream) {
    if (!c || !send_bytes || !recv_bytes || (direction != TC_TO_NEXT && direction != TC_TO_PREV)) {
        tc::set_error("bad tc_replicate_peer arguments");
        return TC_ERR_INVALID;
    }
    cudaStream_t s = static_cast<cudaStream_t>(comm_stream);
    cudaSetDevice(c->device);
    const int P = c->nranks;
    const int next = (c->rank + 1) % P, prev = (c->rank + P - 1) % P;
    const int dst = direction == TC_TO_NEXT ? next : prev;
    const int src = direction == TC_TO_NEXT ? prev : next;
    *recv_bytes = 0;
    if (P == 1) {  // the ring of one: the replica is the local record itself
        stage_sizes_kernel<<<1, 1, 0, s>>>(c->dev_sizes, send_bytes, recv_cap);
        export_sizes_kernel<<<1, 32, 0, s>>>(c->host_sizes, c->dev_sizes);
        cudaError_t e = cudaGetLastError();
        if (e == cudaSuccess) e = cudaStreamSynchronize(s);
        if (e != cudaSuccess) {
            tc::set_error(std::string("size read: ") + cudaGetErrorString(e));
            return TC_ERR_CUDA;
        }
        const uint64_t n = c->host_sizes[3];
        if (n > recv_cap) {
            tc::set_error("payload larger than recv_cap");
            return TC_ERR_CAPACITY;
        }
        if (n) {
            e = cudaMemcpyAsync(recv, send, n, cudaMemcpyDeviceToDevice, s);
            if (e != cudaSuccess) {
                tc::set_error(std::string("ring-of-one copy: ") + cudaGetErrorString(e));
                return TC_ERR_CUDA;
            }
        }
        *recv_bytes = n;
        return TC_OK;
    }
    // 1) size exchange: my payload size goes to dst, my receive capacity goes
    //    to src, so sender and receiver take the same send/skip decision (no orphan send).
    stage_sizes_kernel<<<1, 1, 0, s>>>(c->dev_sizes, send_bytes, recv_cap);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) {
        tc::set_error(std::string("size stage: ") + cudaGetErrorString(e));
        return TC_ERR_CUDA;
    }
    ncclResult_t r = ncclGroupStart();
    if (r == ncclSuccess) r = ncclSend(c->dev_sizes + 3, 8, ncclUint8, dst, c->nccl, s);
    if (r == ncclSuccess) r = ncclSend(c->dev_sizes + 2, 8, ncclUint8, src, c->nccl, s);
    if (r == ncclSuccess) r = ncclRecv(c->dev_sizes, 8, ncclUint8, src, c->nccl, s);
    if (r == ncclSuccess) r = ncclRecv(c->dev_sizes + 1, 8, ncclUint8, dst, c->nccl, s);
    ncclResult_t r2 = ncclGroupEnd();
    if (r != ncclSuccess) return nccl_fail(r, "size exchange");
    if (r2 != ncclSuccess) return nccl_fail(r2, "size exchange (group end)");
    export_sizes_kernel<<<1, 32, 0, s>>>(c->host_sizes, c->dev_sizes);
    e = cudaGetLastError();
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    if (e != cudaSuccess) {
        tc_status st = check_async(c);
        if (st != TC_OK) return st;
        tc::set_error(std::string("size exchange sync: ") + cudaGetErrorString(e));
        return TC_ERR_CUDA;
    }
    // host_sizes now mirrors dev: [0] peer size, [1] dst's cap, [2] my cap, [3] my size
    const uint64_t mine = c->host_sizes[3], theirs = c->host_sizes[0], dst_cap = c->host_sizes[1];
    const bool do_send = mine <= dst_cap, do_recv = theirs <= recv_cap;
    // 2) payload
    r = ncclGroupStart();
    if (r == ncclSuccess && mine && do_send) r = ncclSend(send, mine, ncclUint8, dst, c->nccl, s);
    if (r == ncclSuccess && theirs && do_recv) r = ncclRecv(recv, theirs, ncclUint8, src, c->nccl, s);
    r2 = ncclGroupEnd();
    if (r != ncclSuccess) return nccl_fail(r, "payload send/recv");
    if (r2 != ncclSuccess) return nccl_fail(r2, "payload send/recv (group end)");
    tc_status st = check_async(c);
    if (st != TC_OK) return st;
    if (!do_recv) {
        tc::set_error("neighbour payload larger than recv_cap (nothing received)");
        return TC_ERR_CAPACITY;
    }
    *recv_bytes = theirs;
    return TC_OK;
}

}  // extern "C"
