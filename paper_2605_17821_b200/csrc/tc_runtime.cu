// tc_runtime.cu — libtc host runtime: contexts, argument validation, scratch management,
// encode / apply launch plumbing, Tier-1 staging.  Every compute step runs in the kernels
// of tc_encode.cu / tc_apply.cu; this file only marshals and validates.
#include <cuda_runtime.h>

#include <cstdio>
#include <cstring>
#include <string>

#include "tc_internal.h"

struct tc_ctx {
    int device = 0;
    int num_sms = 148;
    // encode scratch: ticket, per-chunk totals / done counts / record starts, per-group sums,
    // per-block counts, group and chunk prefixes (layout in tc_diff_encode)
    void* enc = nullptr;
    size_t enc_bytes = 0;
    // encode spill slots: kSpillBytes per scan block (packed new words of sparse blocks)
    void* spill = nullptr;
    size_t spill_bytes = 0;
    // index-mode mask staging: kMaskStageWords per scan block
    void* mstage = nullptr;
    size_t mstage_bytes = 0;
    // fold scratch: desc [nrec*cap] | unit_first [cap+1] | info [5]
    void* fold = nullptr;
    size_t fold_bytes = 0;
    unsigned int* err = nullptr;  // [0] sticky device error word, [1] tc_push_peer block counter
    uint64_t launches = 0;
    uint32_t fold_dense_permille = 60;  // tc_ctx_set_fold_dense_permille
    uint64_t fold_max_records = 0;      // tc_ctx_set_fold_max_records (0: bound by the record bytes)
    uint32_t push_ctas = 0;              // tc_ctx_set_push_ctas (0: default)
    void* grad = nullptr;                // gradient codec / replay scratch (tc_grad.cu)
    size_t grad_bytes = 0;
};

namespace tc {

static thread_local std::string g_last_error;

void set_error(const std::string& msg) { g_last_error = msg; }

static tc_status fail(tc_status s, const std::string& msg) {
    set_error(msg);
    return s;
}

static tc_status cuda_fail(cudaError_t e, const char* what) {
    return fail(TC_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

static bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }
static bool is_pow2(uint64_t x) { return x && !(x & (x - 1)); }

static void default_opts(const tc_encode_opts* in, tc_encode_opts* out) {
    if (in) {
        *out = *in;
    } else {
        out->tile_words = 4096;
        out->advance_ref = 1;
        out->chunk_words = 1ull << 28;
        out->index_mode = 0;
        out->reserved = 0;
    }
}

static tc_status check_opts(const tc_encode_opts& o) {
    if (!is_pow2(o.tile_words) || o.tile_words < 32 || o.tile_words > 65536)
        return fail(TC_ERR_INVALID, "tile_words must be a power of two in [32, 65536]");
    if (o.chunk_words == 0 || o.chunk_words % o.tile_words != 0 || o.chunk_words > kMaxChunkWords)
        return fail(TC_ERR_INVALID, "chunk_words must be a positive multiple of tile_words and <= 2^31-1");
    if (o.index_mode > 2 || o.reserved != 0) return fail(TC_ERR_INVALID, "index_mode must be 0, 1 or 2, reserved 0");
    if (o.index_mode == 1 && o.tile_words > kIndexMaxT) return fail(TC_ERR_INVALID, "index mode requires tile_words <= 8192");
    return TC_OK;
}

static tc_status check_segs(const tc_segment* segs, int nseg, bool need_ptrs) {
    if (!segs || nseg < 1 || nseg > TC_MAX_SEGMENTS)
        return fail(TC_ERR_INVALID, "nseg must be in [1, TC_MAX_SEGMENTS]");
    for (int s = 0; s < nseg; ++s) {
        const tc_segment& g = segs[s];
        if (g.word_bytes != 2 && g.word_bytes != 4) return fail(TC_ERR_INVALID, "word_bytes must be 2 or 4");
        if (g.reserved != 0) return fail(TC_ERR_INVALID, "tc_segment.reserved must be 0");
        if (need_ptrs && g.n_words) {
            if (!g.ref || !g.cur) return fail(TC_ERR_INVALID, "segment pointer is NULL");
            if (!aligned16(g.ref) || !aligned16(g.cur)) return fail(TC_ERR_INVALID, "segment pointers must be 16-byte aligned");
        }
    }
    return TC_OK;
}

// grow a stream-ordered scratch allocation
static tc_status ensure(void** p, size_t* have, size_t need, cudaStream_t s) {
    if (*have >= need) return TC_OK;
    size_t want = need + need / 4;
    if (*p) {
        cudaError_t e = cudaFreeAsync(*p, s);
        if (e != cudaSuccess) return cuda_fail(e, "cudaFreeAsync");
        *p = nullptr;
        *have = 0;
    }
    cudaError_t e = cudaMallocAsync(p, want, s);
    if (e != cudaSuccess) {
        *p = nullptr;
        return fail(TC_ERR_NOMEM, std::string("cudaMallocAsync: ") + cudaGetErrorString(e));
    }
    *have = want;
    return TC_OK;
}

}  // namespace tc

using namespace tc;

extern "C" {

const char* tc_status_string(tc_status s) {
    switch (s) {
        case TC_OK: return "TC_OK";
        case TC_ERR_INVALID: return "TC_ERR_INVALID";
        case TC_ERR_NOMEM: return "TC_ERR_NOMEM";
        case TC_ERR_CUDA: return "TC_ERR_CUDA";
        case TC_ERR_NCCL: return "TC_ERR_NCCL";
        case TC_ERR_CORRUPT: return "TC_ERR_CORRUPT";
        case TC_ERR_PROTOCOL: return "TC_ERR_PROTOCOL";
        case TC_ERR_UNAVAILABLE: return "TC_ERR_UNAVAILABLE";
        case TC_ERR_CAPACITY: return "TC_ERR_CAPACITY";
        case TC_ERR_INTERNAL: return "TC_ERR_INTERNAL";
    }
    return "TC_ERR_UNKNOWN";
}

const char* tc_last_error(void) { return g_last_error.c_str(); }

int tc_abi_version(void) { return TC_ABI_VERSION; }

tc_status tc_ctx_create(int device, tc_ctx** out) {
    if (!out) return fail(TC_ERR_INVALID, "out is NULL");
    *out = nullptr;
    cudaError_t e = cudaSetDevice(device);
    if (e != cudaSuccess) return cuda_fail(e, "cudaSetDevice");
    tc_ctx* c = new (std::nothrow) tc_ctx();
    if (!c) return fail(TC_ERR_NOMEM, "host allocation failed");
    c->device = device;
    e = cudaDeviceGetAttribute(&c->num_sms, cudaDevAttrMultiProcessorCount, device);
    if (e != cudaSuccess) {
        delete c;
        return cuda_fail(e, "cudaDeviceGetAttribute");
    }
    e = cudaMalloc(reinterpret_cast<void**>(&c->err), 16);
    if (e == cudaSuccess) e = cudaMemset(c->err, 0, 16);
    if (e != cudaSuccess) {
        delete c;
        return cuda_fail(e, "cudaMalloc(err)");
    }
    *out = c;
    return TC_OK;
}

tc_status tc_ctx_set_push_ctas(tc_ctx* c, uint32_t ctas) {
    if (!c) return fail(TC_ERR_INVALID, "ctx is NULL");
    if (ctas > 65535) return fail(TC_ERR_INVALID, "ctas must be <= 65535");
    c->push_ctas = ctas;
    return TC_OK;
}

tc_status tc_ctx_set_fold_max_records(tc_ctx* c, uint64_t records) {
    if (!c) return fail(TC_ERR_INVALID, "ctx is NULL");
    c->fold_max_records = records;
    return TC_OK;
}

tc_status tc_ctx_set_fold_dense_permille(tc_ctx* c, uint32_t permille) {
    if (!c) return fail(TC_ERR_INVALID, "ctx is NULL");
    c->fold_dense_permille = permille;
    return TC_OK;
}

tc_status tc_ctx_destroy(tc_ctx* c) {
    if (!c) return TC_OK;
    cudaSetDevice(c->device);
    cudaDeviceSynchronize();
    if (c->enc) cudaFree(c->enc);
    if (c->fold) cudaFree(c->fold);
    if (c->spill) cudaFree(c->spill);
    if (c->mstage) cudaFree(c->mstage);
    if (c->grad) cudaFree(c->grad);
    if (c->err) cudaFree(c->err);
    delete c;
    return TC_OK;
}

tc_status tc_ctx_check(tc_ctx* c, tc_stream stream) {
    if (!c) return fail(TC_ERR_INVALID, "ctx is NULL");
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    cudaError_t e = cudaStreamSynchronize(s);
    if (e != cudaSuccess) return cuda_fail(e, "cudaStreamSynchronize");
    unsigned int code = 0;
    e = cudaMemcpy(&code, c->err, sizeof(code), cudaMemcpyDeviceToHost);
    if (e != cudaSuccess) return cuda_fail(e, "cudaMemcpy(err)");
    if (code) {
        e = cudaMemset(c->err, 0, sizeof(code));
        if (e != cudaSuccess) return cuda_fail(e, "cudaMemset(err)");
        return fail(static_cast<tc_status>(code), std::string("device reported ") + tc_status_string(static_cast<tc_status>(code)));
    }
    return TC_OK;
}

uint64_t tc_ctx_launches(const tc_ctx* c) { return c ? c->launches : 0; }

tc_status tc_diff_bound(const tc_segment* segs, int nseg, const tc_encode_opts* opts, uint64_t* max_bytes) {
    if (!max_bytes) return fail(TC_ERR_INVALID, "max_bytes is NULL");
    tc_encode_opts o;
    default_opts(opts, &o);
    tc_status st = check_opts(o);
    if (st != TC_OK) return st;
    st = check_segs(segs, nseg, false);
    if (st != TC_OK) return st;
    uint64_t tot = 0;
    for (int s = 0; s < nseg; ++s) {
        const uint64_t n = segs[s].n_words, w = segs[s].word_bytes;
        uint64_t off = 0;
        do {
            const uint64_t m = n - off < o.chunk_words ? n - off : o.chunk_words;
            tot += o.index_mode == kFormatFull ? record_bytes_full(m, static_cast<uint32_t>(w))
                   : o.index_mode ? record_bytes_index(m, o.tile_words, static_cast<uint32_t>(w), m)
                                  : record_bytes(m, o.tile_words, static_cast<uint32_t>(w), m);
            off += m;
        } while (off < n);
    }
    *max_bytes = tot;
    return TC_OK;
}

namespace {
struct SegSpec {
    uint8_t* ref;
    const uint8_t* cur;
    uint64_t n;
    uint32_t w;
    uint32_t seg_id;
    uint64_t word_base;
    const uint32_t* mask_in = nullptr;  // precomputed change mask (tc::encode_from_masks)
};
}  // namespace

struct PeerEmit {  // fused Tier-2 emit target (tc_diff_encode_push)
    void* dst = nullptr;
    uint64_t cap = 0;
    void* mailbox = nullptr;
};

static tc_status encode_impl(tc_ctx* ctx, const SegSpec* specs, int nseg, const tc_encode_opts& o,
                             uint64_t version, uint64_t ref_version, void* out, uint64_t out_cap,
                             uint64_t* out_bytes, cudaStream_t s, const PeerEmit* peer = nullptr) {
    cudaSetDevice(ctx->device);
    tc_status st = TC_OK;
    EncParams P;
    memset(&P, 0, sizeof(P));
    if (peer) {
        P.peer_out = static_cast<uint8_t*>(peer->dst);
        P.peer_cap = peer->cap;
        P.peer_mail = static_cast<unsigned long long*>(peer->mailbox);
        P.peer_version = version;
        P.peer_counter = ctx->err + 1;
    }
    uint64_t blocks = 0, chunks = 0, full_bytes = 0;
    for (int i = 0; i < nseg; ++i) {
        const SegSpec& g = specs[i];
        EncSeg& E = P.seg[i];
        E.ref = g.ref;
        E.cur = g.cur;
        E.n = g.n;
        E.w = g.w;
        E.seg_id = g.seg_id;
        E.word_base = g.word_base;
        E.mask_in = g.mask_in;
        E.block_words = g.w == 4 ? kEncBlockWords4 : kEncBlockWords2;
        E.first_block = blocks;
        E.first_chunk = chunks;
        E.n_chunks = g.n ? cdiv(g.n, o.chunk_words) : 1;
        const uint64_t full = g.n < o.chunk_words ? g.n : o.chunk_words;
        E.blocks_per_chunk = full ? cdiv(full, E.block_words) : 1;
        const uint64_t m_last = g.n ? g.n - (E.n_chunks - 1) * o.chunk_words : 0;
        const uint64_t last_blocks = m_last ? cdiv(m_last, E.block_words) : 1;
        blocks += (E.n_chunks - 1) * E.blocks_per_chunk + last_blocks;
        chunks += E.n_chunks;
        E.full_base = full_bytes;  // full records: their sizes are known up front (no count)
        full_bytes += (E.n_chunks - 1) * record_bytes_full(full, g.w) + record_bytes_full(m_last, g.w);
    }
    P.nseg = nseg;
    P.T = o.tile_words;
    P.C = o.chunk_words;
    P.total_blocks = blocks;
    P.total_chunks = chunks;
    P.version = version;
    P.ref_version = ref_version;
    P.out = static_cast<uint8_t*>(out);
    P.out_cap = out_cap;
    P.out_bytes = out_bytes;
    P.advance_ref = o.advance_ref ? 1 : 0;
    P.index_mode = static_cast<int>(o.index_mode);
    P.err = ctx->err;

    const uint64_t groups = cdiv(blocks, kEmitGroup);
    P.n_groups = groups;
    // zeroed region: ticket | chunk_acc | rstart | group_sum
    const size_t z_ticket = 0, z_ctot = 16;
    const size_t z_rstart = z_ctot + 8 * chunks;
    const size_t z_gsum = z_rstart + 8 * (chunks + 1);
    const size_t z_end = z_gsum + 8 * groups;
    // written-every-call region: info | gpre | cbase
    const size_t w_info = (z_end + 255) & ~size_t(255);
    const size_t w_gpre = w_info + ((4 * blocks + 15) & ~size_t(15));
    const size_t w_cbase = w_gpre + 8 * groups;
    const size_t need = w_cbase + 8 * chunks;
    st = ensure(&ctx->enc, &ctx->enc_bytes, need, s);
    if (st != TC_OK) return st;
    if (o.index_mode != kFormatFull) {
        st = ensure(&ctx->spill, &ctx->spill_bytes, blocks * static_cast<size_t>(o.index_mode ? 2 * kSpillBytes : kSpillMask), s);
        if (st != TC_OK) return st;
    }
    if (o.index_mode == 1) {
        st = ensure(&ctx->mstage, &ctx->mstage_bytes, blocks * static_cast<size_t>(kMaskStageWords) * 4, s);
        if (st != TC_OK) return st;
        P.mstage = static_cast<uint32_t*>(ctx->mstage);
    }
    uint8_t* base = static_cast<uint8_t*>(ctx->enc);
    P.ticket = reinterpret_cast<unsigned long long*>(base + z_ticket);
    P.chunk_acc = reinterpret_cast<unsigned long long*>(base + z_ctot);
    P.rstart = reinterpret_cast<unsigned long long*>(base + z_rstart);
    P.group_sum = reinterpret_cast<unsigned long long*>(base + z_gsum);
    P.info = reinterpret_cast<uint32_t*>(base + w_info);
    P.gpre = reinterpret_cast<unsigned long long*>(base + w_gpre);
    P.cbase = reinterpret_cast<unsigned long long*>(base + w_cbase);
    P.spill = static_cast<uint8_t*>(ctx->spill);
    cudaError_t e = cudaMemsetAsync(base, 0, z_end, s);
    if (e != cudaSuccess) return cuda_fail(e, "cudaMemsetAsync(scratch)");
    P.full_total = full_bytes;
    e = launch_encode(P, s);
    if (e != cudaSuccess) return cuda_fail(e, "encode launch");
    ctx->launches += o.index_mode == kFormatFull ? 1 : 3;
    return TC_OK;
}

static uint64_t range_bound(uint64_t n, uint32_t w, const tc_encode_opts& o, uint64_t c0, uint64_t nc) {
    uint64_t tot = 0;
    const uint64_t total_chunks = n ? cdiv(n, o.chunk_words) : 1;
    for (uint64_t c = c0; c < c0 + nc && c < total_chunks; ++c) {
        const uint64_t off = c * o.chunk_words;
        const uint64_t m = n > off ? (n - off < o.chunk_words ? n - off : o.chunk_words) : 0;
        tot += o.index_mode == kFormatFull ? record_bytes_full(m, w)
               : o.index_mode ? record_bytes_index(m, o.tile_words, w, m) : record_bytes(m, o.tile_words, w, m);
    }
    return tot;
}

extern "C" tc_status tc_diff_encode(tc_ctx* ctx, const tc_segment* segs, int nseg, const tc_encode_opts* opts,
                                    uint64_t version, uint64_t ref_version, void* out, uint64_t out_cap,
                                    uint64_t* out_bytes, tc_stream stream) {
    if (!ctx) return fail(TC_ERR_INVALID, "ctx is NULL");
    tc_encode_opts o;
    default_opts(opts, &o);
    tc_status st = check_opts(o);
    if (st != TC_OK) return st;
    st = check_segs(segs, nseg, true);
    if (st != TC_OK) return st;
    if (!out || !aligned16(out)) return fail(TC_ERR_INVALID, "out must be a 16-byte aligned device pointer");
    if (!out_bytes) return fail(TC_ERR_INVALID, "out_bytes is NULL");
    SegSpec sp[TC_MAX_SEGMENTS];
    for (int i = 0; i < nseg; ++i)
        sp[i] = {static_cast<uint8_t*>(segs[i].ref), static_cast<const uint8_t*>(segs[i].cur), segs[i].n_words,
                 segs[i].word_bytes, static_cast<uint32_t>(i), 0};
    return encode_impl(ctx, sp, nseg, o, version, ref_version, out, out_cap, out_bytes,
                       static_cast<cudaStream_t>(stream));
}

extern "C" tc_status tc_diff_bound_range(const tc_segment* seg, const tc_encode_opts* opts, uint64_t first_chunk,
                                         uint64_t n_chunks, uint64_t* max_bytes) {
    if (!max_bytes) return fail(TC_ERR_INVALID, "max_bytes is NULL");
    tc_encode_opts o;
    default_opts(opts, &o);
    tc_status st = check_opts(o);
    if (st != TC_OK) return st;
    st = check_segs(seg, 1, false);
    if (st != TC_OK) return st;
    const uint64_t total_chunks = seg->n_words ? cdiv(seg->n_words, o.chunk_words) : 1;
    if (n_chunks == 0 || first_chunk >= total_chunks)
        return fail(TC_ERR_INVALID, "chunk range outside the segment");
    *max_bytes = range_bound(seg->n_words, seg->word_bytes, o, first_chunk, n_chunks);
    return TC_OK;
}

extern "C" tc_status tc_diff_encode_range(tc_ctx* ctx, const tc_segment* seg, uint32_t segment_id,
                                          const tc_encode_opts* opts, uint64_t first_chunk, uint64_t n_chunks,
                                          uint64_t version, uint64_t ref_version, void* out, uint64_t out_cap,
                                          uint64_t* out_bytes, tc_stream stream) {
    if (!ctx) return fail(TC_ERR_INVALID, "ctx is NULL");
    tc_encode_opts o;
    default_opts(opts, &o);
    tc_status st = check_opts(o);
    if (st != TC_OK) return st;
    st = check_segs(seg, 1, true);
    if (st != TC_OK) return st;
    if (!out || !aligned16(out)) return fail(TC_ERR_INVALID, "out must be a 16-byte aligned device pointer");
    if (!out_bytes) return fail(TC_ERR_INVALID, "out_bytes is NULL");
    uint64_t bound = 0;  // validates the range; out_cap may be smaller (checked on the device)
    st = tc_diff_bound_range(seg, &o, first_chunk, n_chunks, &bound);
    if (st != TC_OK) return st;
    const uint64_t off = first_chunk * o.chunk_words;
    const uint64_t n = seg->n_words > off ? seg->n_words - off : 0;
    const uint64_t len = n < n_chunks * o.chunk_words ? n : n_chunks * o.chunk_words;
    const uint64_t w = seg->word_bytes;
    SegSpec sp = {seg->n_words ? static_cast<uint8_t*>(seg->ref) + off * w : nullptr,
                  seg->n_words ? static_cast<const uint8_t*>(seg->cur) + off * w : nullptr, len,
                  seg->word_bytes, segment_id, off};
    return encode_impl(ctx, &sp, 1, o, version, ref_version, out, out_cap, out_bytes,
                       static_cast<cudaStream_t>(stream));
}

tc_status tc_diff_apply(tc_ctx* ctx, void* const* state, const uint64_t* n_words, const uint32_t* word_bytes,
                        int nseg, uint64_t state_version, const void* const* records,
                        const uint64_t* record_bytes_, int n_records, tc_stream stream) {
    if (!ctx) return fail(TC_ERR_INVALID, "ctx is NULL");
    if (!state || !n_words || !word_bytes || nseg < 1 || nseg > TC_MAX_SEGMENTS)
        return fail(TC_ERR_INVALID, "bad state description (1 <= nseg <= TC_MAX_SEGMENTS)");
    if (!records || !record_bytes_ || n_records < 1 || n_records > TC_MAX_FOLD)
        return fail(TC_ERR_INVALID, "n_records must be in [1, TC_MAX_FOLD]");
    FoldParams P;
    memset(&P, 0, sizeof(P));
    uint64_t cap = 0;
    for (int s = 0; s < nseg; ++s) {
        if (word_bytes[s] != 2 && word_bytes[s] != 4) return fail(TC_ERR_INVALID, "word_bytes must be 2 or 4");
        if (n_words[s] && (!state[s] || !aligned16(state[s])))
            return fail(TC_ERR_INVALID, "state pointers must be 16-byte aligned device pointers");
        P.state[s] = static_cast<uint8_t*>(state[s]);
        P.n[s] = n_words[s];
        P.w[s] = word_bytes[s];
        // records per segment <= ceil(n/32) (chunk_words >= tile_words >= 32), at least 1
        cap += n_words[s] ? cdiv(n_words[s], 32) : 1;
    }
    if (cap > TC_MAX_RECORDS_PER_DIFF) cap = TC_MAX_RECORDS_PER_DIFF;
    for (int j = 0; j < n_records; ++j) {
        if (!records[j] || !aligned16(records[j]))
            return fail(TC_ERR_INVALID, "record pointers must be 16-byte aligned device pointers");
        P.rec[j] = static_cast<const uint8_t*>(records[j]);
        P.rec_bytes[j] = record_bytes_[j];
        // a record is at least 80 bytes (header + tile_off), and every diff of one fold must
        // hold the same number of records: the shortest diff bounds the descriptor table (a diff
        // with more records than that fails the walker's layout check anyway)
        const uint64_t by_bytes = record_bytes_[j] / 80 + 1;
        if (by_bytes < cap) cap = by_bytes;
    }
    // the caller's bound on records per diff (its layout and chunk size fix it): the descriptor
    // table shrinks from min(record_bytes / 80, 65536) entries per diff (~38 MB for a
    // chain of 8 cfg2-sized records, ~300 MB for 64) to what the layout needs
    if (ctx->fold_max_records && ctx->fold_max_records < cap) {
        cap = ctx->fold_max_records;
        P.cap_hinted = 1;
    }
    P.nseg = nseg;
    P.nrec = n_records;
    P.cap = static_cast<uint32_t>(cap);
    P.state_version = state_version;
    P.dense_permille = ctx->fold_dense_permille;
    P.err = ctx->err;

    cudaStream_t s = static_cast<cudaStream_t>(stream);
    cudaSetDevice(ctx->device);
    const size_t desc_bytes = sizeof(FoldRec) * cap * n_records;
    const size_t need = desc_bytes + 8 * (cap + 1) + 64;  // desc | unit_first | info[6]
    tc_status st = ensure(&ctx->fold, &ctx->fold_bytes, need, s);
    if (st != TC_OK) return st;
    uint8_t* base = static_cast<uint8_t*>(ctx->fold);
    P.desc = reinterpret_cast<FoldRec*>(base);
    P.unit_first = reinterpret_cast<uint64_t*>(base + desc_bytes);
    P.info = reinterpret_cast<unsigned long long*>(base + desc_bytes + 8 * (cap + 1));
    cudaError_t e = launch_fold(P, s, ctx->num_sms, &ctx->launches);
    if (e != cudaSuccess) return cuda_fail(e, "fold launch");
    return TC_OK;
}

tc_status tc_stage_host(void* dst, const void* src, uint64_t bytes, int dir, tc_stream copy_stream) {
    if (bytes == 0) return TC_OK;
    if (!dst || !src) return fail(TC_ERR_INVALID, "NULL buffer");
    if (dir != TC_D2H && dir != TC_H2D) return fail(TC_ERR_INVALID, "dir must be TC_D2H or TC_H2D");
    const void* host = dir == TC_D2H ? dst : src;
    cudaPointerAttributes a;
    cudaError_t e = cudaPointerGetAttributes(&a, host);
    if (e != cudaSuccess || a.type != cudaMemoryTypeHost) {
        cudaGetLastError();
        return fail(TC_ERR_INVALID, "host side of tc_stage_host must be pinned (cudaHostAlloc/cudaHostRegister)");
    }
    e = cudaMemcpyAsync(dst, src, bytes, dir == TC_D2H ? cudaMemcpyDeviceToHost : cudaMemcpyHostToDevice,
                        static_cast<cudaStream_t>(copy_stream));
    if (e != cudaSuccess) return cuda_fail(e, "cudaMemcpyAsync");
    return TC_OK;
}

tc_status tc_host_alloc(uint64_t bytes, void** out) {
    if (!out) return fail(TC_ERR_INVALID, "out is NULL");
    *out = nullptr;
    if (bytes == 0) return TC_OK;
    cudaError_t e = cudaHostAlloc(out, bytes, cudaHostAllocPortable | cudaHostAllocMapped);
    if (e != cudaSuccess) {
        *out = nullptr;
        return fail(TC_ERR_NOMEM, std::string("cudaHostAlloc: ") + cudaGetErrorString(e));
    }
    return TC_OK;
}

tc_status tc_host_free(void* p) {
    if (!p) return TC_OK;
    cudaError_t e = cudaFreeHost(p);
    if (e != cudaSuccess) return cuda_fail(e, "cudaFreeHost");
    return TC_OK;
}

}  // extern "C"

namespace tc {
unsigned int* ctx_err(tc_ctx* c) { return c->err; }
int ctx_device(tc_ctx* c) { return c->device; }
int ctx_num_sms(tc_ctx* c) { return c->num_sms; }
void ctx_add_launches(tc_ctx* c, uint64_t n) { c->launches += n; }
uint32_t ctx_push_ctas(tc_ctx* c) { return c->push_ctas; }
tc_status ctx_grad_scratch(tc_ctx* c, size_t bytes, cudaStream_t s, void** out) {
    tc_status st = ensure(&c->grad, &c->grad_bytes, bytes, s);
    *out = c->grad;
    return st;
}
}  // namespace tc

namespace tc {
// tc_diff_encode with the fused Tier-2 emit: the encoder writes the record into `out` and, over
// NVLink, into the peer slot; its last emit CTA publishes the mailbox (tc_peer.cu).
tc_status encode_push(tc_ctx* ctx, const tc_segment* segs, int nseg, const tc_encode_opts* opts, uint64_t version,
                      uint64_t ref_version, void* out, uint64_t out_cap, uint64_t* out_bytes, void* peer_dst,
                      uint64_t peer_cap, void* peer_mailbox, cudaStream_t s) {
    if (!ctx) return fail(TC_ERR_INVALID, "ctx is NULL");
    tc_encode_opts o;
    default_opts(opts, &o);
    tc_status st = check_opts(o);
    if (st != TC_OK) return st;
    st = check_segs(segs, nseg, true);
    if (st != TC_OK) return st;
    if (!out || !aligned16(out)) return fail(TC_ERR_INVALID, "out must be a 16-byte aligned device pointer");
    if (!out_bytes) return fail(TC_ERR_INVALID, "out_bytes is NULL");
    SegSpec sp[TC_MAX_SEGMENTS];
    for (int i = 0; i < nseg; ++i)
        sp[i] = {static_cast<uint8_t*>(segs[i].ref), static_cast<const uint8_t*>(segs[i].cur), segs[i].n_words,
                 segs[i].word_bytes, static_cast<uint32_t>(i), 0};
    PeerEmit pe;
    pe.dst = peer_dst;
    pe.cap = peer_cap;
    pe.mailbox = peer_mailbox;
    return encode_impl(ctx, sp, nseg, o, version, ref_version, out, out_cap, out_bytes, s, &pe);
}

// Encode `cur` against the change masks `masks[s]` (bit i of u32 word i/32 = word i of segment s
// changed) instead of a reference: the records tc_diff_encode(ref, cur) would produce for any ref
// with those differences (tc_adam_step_encode).  No reference is read or advanced.
tc_status encode_from_masks(tc_ctx* ctx, const tc_segment* segs, const uint32_t* const* masks, int nseg,
                            const tc_encode_opts* opts, uint64_t version, uint64_t ref_version, void* out,
                            uint64_t out_cap, uint64_t* out_bytes, cudaStream_t s) {
    tc_encode_opts o;
    default_opts(opts, &o);
    o.advance_ref = 0;
    tc_status st = check_opts(o);
    if (st != TC_OK) return st;
    if (nseg < 1 || nseg > TC_MAX_SEGMENTS) return fail(TC_ERR_INVALID, "1 <= nseg <= TC_MAX_SEGMENTS");
    SegSpec sp[TC_MAX_SEGMENTS];
    for (int i = 0; i < nseg; ++i) {
        if ((segs[i].n_words && (!segs[i].cur || !masks[i])) || (segs[i].word_bytes != 2 && segs[i].word_bytes != 4))
            return fail(TC_ERR_INVALID, "bad segment / mask");
        sp[i] = {nullptr, static_cast<const uint8_t*>(segs[i].cur), segs[i].n_words, segs[i].word_bytes,
                 static_cast<uint32_t>(i), 0, masks[i]};
    }
    return encode_impl(ctx, sp, nseg, o, version, ref_version, out, out_cap, out_bytes, s);
}
}  // namespace tc
