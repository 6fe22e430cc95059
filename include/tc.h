/*
 * tc.h — libtc: the B200-native differential checkpoint codec of TierCheck
 * (arxiv 2605.17821), behind a plain C ABI.
 *
 * The hot path (BASELINE.json north_star):
 *   SAVE      tc_diff_encode     word-by-word differential of one rank's shard against its
 *                                reference -> bitmask + packed changed words, one record per
 *                                (segment, chunk)                    [sm_100a CUDA kernel]
 *             tc_stage_host      Tier-1: copy a record into pinned host memory on a side
 *                                stream                              [copy engine]
 *             tc_replicate_peer  Tier-2: ring-neighbour replication over NCCL send/recv,
 *                                preceded by the payload-size exchange
 *   RETRIEVE  tc_diff_apply      rebuild the state bit-exactly from a base plus a chain of
 *                                records (fold of N records in one pass) [sm_100a CUDA kernels]
 *   RECLAIM   (no call)          records and buffers are caller-owned; the caller frees records
 *                                whose version <= its watermark (§3.4;
 *                                SPEC.md:395-403).  The library keeps no reference to any
 *                                caller buffer after the enqueued work completes.
 * The lifecycle follows PAPER.md:35-44 §1 ("checkpoint saving / retrieval / reclamation")
 * and PAPER.md:179-196 §3.1.
 *
 * Conventions for every call
 *   - Nothing throws across the ABI; every call returns tc_status.  tc_last_error() gives a
 *     thread-local human-readable detail for the last non-OK status on this thread.
 *   - Calls taking a stream ENQUEUE work on it and return.  Errors visible on the host
 *     (bad arguments, capacity) are returned synchronously before anything is enqueued.
 *     Errors found by the device (malformed record -> TC_ERR_CORRUPT, chain gap ->
 *     TC_ERR_PROTOCOL, layout mismatch -> TC_ERR_INVALID, internal watchdog ->
 *     TC_ERR_INTERNAL) are STICKY in the tc_ctx and surface at tc_ctx_check(); while a
 *     sticky error is pending, tc_diff_apply's fold kernels skip their writes.
 *   - Device pointers must be 16-byte aligned (record buffers, state/ref/cur segments).
 *   - Streams are passed as tc_stream = the cudaStream_t handle cast to void* (NULL = the
 *     legacy default stream).  A tc_ctx must be used from one stream at a time (its scratch
 *     is stream-ordered), like a cuBLAS handle.
 *   - Ownership: every data buffer belongs to the caller and must stay alive until the
 *     enqueued work completes.  libtc owns only the tc_ctx scratch and the tc_comm's NCCL
 *     communicator.
 *
 * Record wire format (little-endian per SPEC.md:152):
 *   64-byte header {magic "TCD1", u16 format 1, u8 word_bytes, u8 flags=1 (REPLACE),
 *   u32 tile_words T, u32 segment_id, u64 chunk_word_offset, u64 n_words m, u64 count,
 *   u64 version, u64 ref_version, u64 total_bytes} || mask u32[ceil(m/32)] ||
 *   tile_off u32[ceil(m/T)+1] || values (word_bytes * count); each section zero-padded to 16 B.
 *   Index mode (flags = 3): header || tile_off u32[ceil(m/T)+1] || idx u16[count] (in-tile
 *   position of each changed word, increasing within a tile) || values; each padded to 16 B.
 *   Mask bit (i mod 32) of word i/32 is set iff word i of the chunk changed (unsigned
 *   bitwise compare); values are the new words of the changed positions in index order;
 *   tile_off[t] = changed words in [0, t*T).  A shard diff is the concatenation of its
 *   records, segment 0..nseg-1, chunks ascending; an empty segment is one 80-byte record.
 */
#ifndef TC_H
#define TC_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define TC_ABI_VERSION 1
#define TC_MAX_SEGMENTS 16      /* segments per shard (a1 uses 4: bf16 weights, fp32 master/m/v) */
#define TC_MAX_FOLD 64          /* records folded by one tc_diff_apply call                     */
#define TC_MAX_RECORDS_PER_DIFF 65536

typedef enum tc_status {
    TC_OK = 0,
    TC_ERR_INVALID = 1,     /* bad argument / unsupported layout                               */
    TC_ERR_NOMEM = 2,       /* device or host allocation failed                                */
    TC_ERR_CUDA = 3,        /* CUDA runtime error (detail in tc_last_error)                    */
    TC_ERR_NCCL = 4,        /* NCCL error other than a lost peer                               */
    TC_ERR_CORRUPT = 5,     /* malformed record: header, mask/tile_off mismatch  */
    TC_ERR_PROTOCOL = 6,    /* chain gap: ref_version != state version           */
    TC_ERR_UNAVAILABLE = 7, /* peer / communicator failed; replica absent        */
    TC_ERR_CAPACITY = 8,    /* output or receive buffer too small                              */
    TC_ERR_INTERNAL = 9     /* device watchdog fired (a bug); results unspecified              */
} tc_status;

typedef void* tc_stream;          /* a cudaStream_t handle                                     */
typedef struct tc_ctx tc_ctx;     /* per-device scratch: tile tickets, look-back status words,
                                     record-start chain, fold descriptors, sticky error word    */
typedef struct tc_comm tc_comm;   /* ring communicator: own ncclComm_t, next=(r+1)%P, prev=(r-1+P)%P */

/* One segment of a rank's shard (§2.1 "14 Phi bytes":
 * segment 0 = 16-bit weights, segments 1..3 = fp32 master / Adam m / Adam v, each the
 * rank's contiguous ZeRO partition).  word_bytes is 2 or 4; the codec compares
 * raw bits, so any 16-bit (bf16/fp16) or 32-bit dtype works (reading R4). */
typedef struct tc_segment {
    void* ref;            /* device; the reference words (advanced in place if advance_ref) */
    const void* cur;      /* device; the current words                                      */
    uint64_t n_words;
    uint32_t word_bytes;  /* 2 or 4 */
    uint32_t reserved;    /* must be 0 */
} tc_segment;

enum { TC_FORMAT_MASK = 0, TC_FORMAT_INDEX = 1, TC_FORMAT_FULL = 2 };

typedef struct tc_encode_opts {
    uint32_t tile_words;  /* T: power of two in [32, 65536]; default 4096 (reading R7)          */
    uint32_t advance_ref; /* 1 (default): ref[i] <- cur[i] for every changed word, so the next
                             record is incremental (reading R2); 0: ref untouched             */
    uint64_t chunk_words; /* C: multiple of T, <= 2^31-1; default 2^28 (PAPER.md:203 chunking,
                             reading R8)                                                      */
    uint32_t index_mode;  /* record format (TC_FORMAT_*).  0 (default): mask section (4 bytes per
                             32 words).  1: index mode — the mask is replaced by u16[count] in-tile
                             positions after tile_off (flags bit1; 2 bytes per changed word),
                             smaller when f < 1/16: the lossless analog of the paper's "FP16
                             values and INT32 indices" sparse payload (§3.2);
                             requires T <= 8192.  2: full records (flags 5, reading R21) — every
                             word of the chunk, no mask / tile_off (count = m); smaller than a mask
                             record when more than 1 - 1/(8w) of the words changed (the dense
                             regime of a real optimizer step) and encoded by one streaming copy.
                             Records of all three formats fold together. */
    uint32_t reserved;    /* must be 0 */
} tc_encode_opts;

enum { TC_D2H = 0, TC_H2D = 1 };
enum { TC_TO_NEXT = 0, TC_TO_PREV = 1 };

/* ---------------------------------------------------------------- housekeeping ---- */
const char* tc_status_string(tc_status s);
const char* tc_last_error(void);
int tc_abi_version(void);

/* Create a context on CUDA device `device` (the device is made current on the calling
 * thread).  Scratch grows on demand, stream-ordered, and is kept until tc_ctx_destroy; its
 * largest part is the encoders' per-block spill area: 8 KB per scan block of 4096 4-byte /
 * 8192 2-byte words (mask and index records alike) = half the bytes of the largest state
 * encoded, plus ~1 % bookkeeping (index records: + 1 KB per block of staged mask words).
 * *out receives the handle. */
tc_status tc_ctx_create(int device, tc_ctx** out);
tc_status tc_ctx_destroy(tc_ctx* ctx);
/* Synchronize `stream`, then return and clear the sticky device error (TC_OK if none). */
tc_status tc_ctx_check(tc_ctx* ctx, tc_stream stream);
/* Number of kernel launches libtc has enqueued through this ctx since creation. */
uint64_t tc_ctx_launches(const tc_ctx* ctx);
/* Restore strategy.  tc_diff_apply folds a chunk either by scattering the
 * winning words in place or by streaming the chunk's tiles through shared memory (whole-line
 * writes).  Chains of index-mode records at T = 4096 are streamed when they are long (>= 4
 * records changing >= 0.5 % of the words in total) or dense (> permille/1000 of the words in
 * total), chains of mask-mode records at T <= 4096 when dense (at most 32 records, one format per
 * chain); all other chunks are scattered.  Default 60 (6 %).  0 = stream every chunk; UINT32_MAX = scatter every
 * chunk.  Every strategy produces the same state.
 * Takes effect for later tc_diff_apply calls.  Errors: TC_ERR_INVALID (NULL ctx). */
tc_status tc_ctx_set_fold_dense_permille(tc_ctx* ctx, uint32_t permille);
/* Upper bound on the records of one diff that later tc_diff_apply calls on this ctx will fold
 * (the caller knows it: sum over segments of max(1, ceil(n_words / chunk_words))).  Without it the
 * fold's descriptor scratch is sized from the record bytes (>= 80 bytes per record, at most
 * TC_MAX_RECORDS_PER_DIFF): ~38 MB for a chain of 8 cfg2-sized records, ~300 MB for 64; with it,
 * records x 72 bytes per diff.  A diff holding more
 * records fails with TC_ERR_CAPACITY (nothing folded).  0 (default) = no bound.
 * Errors: TC_ERR_INVALID (NULL ctx). */
tc_status tc_ctx_set_fold_max_records(tc_ctx* ctx, uint64_t records);
/* CTAs of tc_push_peer's NVLink copy on this ctx (0 = default 32).  More CTAs = more stores in
 * flight (a 1 GiB push: ~530 GB/s at 16, ~600 at 32, ~700 at 296 per direction) but more
 * interference with kernels running beside it.  Errors: TC_ERR_INVALID. */
tc_status tc_ctx_set_push_ctas(tc_ctx* ctx, uint32_t ctas);

/* ----------------------------------------------------------------------- SAVE ---- */
/* Worst-case diff bytes for this shard layout (every word changed); host only.
 * record size = 64 + pad16(4 ceil(m/32)) + pad16(4(ceil(m/T)+1))
 * + pad16(w*count), summed over chunks.  Errors: TC_ERR_INVALID. */
tc_status tc_diff_bound(const tc_segment* segs, int nseg, const tc_encode_opts* opts,
                        uint64_t* max_bytes);

/* Encode one differential checkpoint (§2.2 "one rank's
 * shard of the incremental updates"; version = iteration, §3.3).
 *   segs/nseg      the shard (device pointers), 1 <= nseg <= TC_MAX_SEGMENTS
 *   opts           NULL = defaults {4096, 1, 2^28}
 *   version        the iteration index of `cur`; ref_version that of `ref` (the chain link)
 *   out/out_cap    device buffer for the concatenated records.  out_cap >= tc_diff_bound(...)
 *                  always suffices; a smaller buffer (sized for the expected change fraction)
 *                  is allowed: a record that does not fit is not written (nothing is written at
 *                  or past out + out_cap), the device reports TC_ERR_CAPACITY (sticky, at
 *                  tc_ctx_check) and *out_bytes still receives the length the diff needs.  With
 *                  advance_ref the reference has then still advanced, so this version's diff is
 *                  lost: the caller takes a base checkpoint (§3.1 base stream)
 *   out_bytes      device (or mapped pinned host) u64 the kernel sets to the diff's length
 *   stream         the encode is enqueued here; it reads ref/cur and (advance_ref) writes ref
 * Output bytes are identical to the oracle's for the same (inputs, T, C) (bit-exact). */
tc_status tc_diff_encode(tc_ctx* ctx, const tc_segment* segs, int nseg,
                         const tc_encode_opts* opts, uint64_t version, uint64_t ref_version,
                         void* out, uint64_t out_cap, uint64_t* out_bytes, tc_stream stream);

/* Streaming encode of a contiguous run of whole chunks of ONE segment: writes exactly the bytes
 * the records of chunks [first_chunk, first_chunk + n_chunks) of segment `segment_id` have in the
 * full tc_diff_encode output (same header segment_id / chunk_word_offset), so concatenating the
 * ranges of every segment in order reproduces the full diff.  Used when the full bound does not
 * fit in HBM next to the state (40B-shaped shards: SURVEY.md §7 build plan step 9).  `seg`
 * describes the WHOLE segment; out_cap as for tc_diff_encode (tc_diff_bound_range(...) always
 * suffices; a smaller buffer gets the same device-side TC_ERR_CAPACITY behaviour);
 * *out_bytes (device or mapped pinned) receives the range's length. */
tc_status tc_diff_bound_range(const tc_segment* seg, const tc_encode_opts* opts, uint64_t first_chunk,
                              uint64_t n_chunks, uint64_t* max_bytes);
tc_status tc_diff_encode_range(tc_ctx* ctx, const tc_segment* seg, uint32_t segment_id,
                               const tc_encode_opts* opts, uint64_t first_chunk, uint64_t n_chunks,
                               uint64_t version, uint64_t ref_version, void* out, uint64_t out_cap,
                               uint64_t* out_bytes, tc_stream stream);

/* Tier-1 (§4 "low-priority CUDA streams and pinned host memory buffers";
 * SURVEY.md §8(a) a5): cudaMemcpyAsync of `bytes` between a device buffer and a PINNED
 * host buffer on `copy_stream`.  dir = TC_D2H (save) or TC_H2D (restore fetch).  The host
 * side must be page-locked (cudaHostAlloc / cudaHostRegister), else TC_ERR_INVALID (a
 * pageable copy would silently stall the caller). */
tc_status tc_stage_host(void* dst, const void* src, uint64_t bytes, int dir,
                        tc_stream copy_stream);
/* Page-locked host buffer for the Tier-1 ring (cudaHostAlloc, portable + mapped), owned by the
 * caller until tc_host_free.  Copies between it and the device never block the caller. */
tc_status tc_host_alloc(uint64_t bytes, void** out);
tc_status tc_host_free(void* p);

/* Tier-2 (§3.1 ring peer mapping; §3.2 "Peer ranks first
 * exchange their serialized payload sizes").  Collective over the
 * tc_comm: every rank sends its payload to next=(r+1)%P (TC_TO_NEXT, the save direction) or
 * to prev=(r-1+P)%P (TC_TO_PREV, the restore pull) and receives its neighbour's.
 *   send           device buffer; send_bytes: DEVICE u64 holding its length (as written by
 *                  tc_diff_encode) — the 8-byte size exchange reads it on comm_stream
 *   recv/recv_cap  device buffer for the neighbour's payload; recv_bytes: HOST out
 * The call synchronizes comm_stream once (to learn both sizes), never the caller's other
 * streams; the payload transfer is then enqueued on comm_stream.  The caller orders
 * comm_stream after the producer of `send` (e.g. cudaStreamWaitEvent).
 * Errors: TC_ERR_CAPACITY if the neighbour's payload exceeds recv_cap (nothing transferred;
 * the size exchange still completed on every rank), TC_ERR_UNAVAILABLE if NCCL reports a
 * lost peer / remote error. */
tc_status tc_comm_get_unique_id(uint8_t id[128]);
tc_status tc_comm_init(int nranks, int rank, int device, const uint8_t id[128], tc_comm** out);
tc_status tc_comm_destroy(tc_comm* comm);
tc_status tc_replicate_peer(tc_comm* comm, const void* send, const uint64_t* send_bytes,
                            void* recv, uint64_t recv_cap, uint64_t* recv_bytes, int direction,
                            tc_stream comm_stream);

/* Tier-2 without NCCL: device-initiated push over NVLink peer memory (SURVEY.md §8(f) NEXT row
 * 1, "the ring peer's registered window ... Tier-2 via NVLink stores"; §3.1 ring
 * mapping, §3.2 size exchange — here the size travels with the payload).
 * The RECEIVER owns a slot (the neighbour's record lands there) and a 16-byte mailbox
 * {u64 bytes, u64 version}, both allocated with tc_ipc_alloc in its own GPU memory; it passes
 * their handles to its ring neighbour (the caller's transport, e.g. torch.distributed), which
 * maps them with tc_ipc_open.  One process per GPU; peers on one NVLink/NVSwitch domain. */
#define TC_IPC_HANDLE_BYTES 64
/* cudaMalloc `bytes` on the current device, zero-filled, and its IPC handle.  Errors:
 * TC_ERR_NOMEM, TC_ERR_CUDA. */
tc_status tc_ipc_alloc(uint64_t bytes, void** dev_ptr, uint8_t handle[TC_IPC_HANDLE_BYTES]);
tc_status tc_ipc_free(void* dev_ptr);
/* Map a peer process's tc_ipc_alloc allocation into this process (peer access enabled lazily);
 * *dev_ptr is valid on the current device until tc_ipc_close. */
tc_status tc_ipc_open(const uint8_t handle[TC_IPC_HANDLE_BYTES], void** dev_ptr);
tc_status tc_ipc_close(void* dev_ptr);
/* Copy the record at `src` (its length: the u64 at `src_bytes`, device or mapped pinned
 * memory, as written by tc_diff_encode — read on the device, no host round trip) into the
 * peer slot `peer_dst` (capacity peer_cap) with NVLink stores from every SM, then publish
 * {bytes, version} to `peer_mailbox` with a system-scope release.  A record larger than
 * peer_cap is not copied; the mailbox then carries bytes = UINT64_MAX (the receiver's
 * tc_peer_wait reports TC_ERR_CAPACITY).  Any length: the last bytes % 16 are copied byte by
 * byte (src and peer_dst themselves must be 16-byte aligned).  version >= 1.  Stream-ordered on `stream`; the
 * caller orders reuse of a slot (e.g. one slot per in-flight version). */
tc_status tc_push_peer(tc_ctx* ctx, const void* src, const uint64_t* src_bytes, void* peer_dst,
                       uint64_t peer_cap, void* peer_mailbox, uint64_t version, tc_stream stream);
/* Encode (as tc_diff_encode) with the Tier-2 copy FUSED into the encoder (SURVEY.md §8(f) NEXT
 * row 1): every record byte the encode kernels write into `out` is also stored, over NVLink, at the
 * same offset of `peer_dst` — the record is never re-read from HBM and there is no separate copy
 * launch, host synchronization or NCCL; the last emitting CTA then publishes {bytes, version} into
 * `peer_mailbox` with a system-scope release (as tc_push_peer).  A record larger than peer_cap (or
 * an encode that reports an error) is published as refused (bytes = UINT64_MAX: the receiver's
 * tc_peer_wait reports TC_ERR_CAPACITY); bytes below peer_cap may then hold a partial record.
 * peer_dst / peer_mailbox may also be mapped page-locked host memory (tc_host_alloc): the
 * encoder then emits the record straight into Tier-1 over PCIe (the host polls the mailbox).
 * Measured slower than encode + copy engine (tools/t1_emit_bench.py). */
tc_status tc_diff_encode_push(tc_ctx* ctx, const tc_segment* segs, int nseg, const tc_encode_opts* opts,
                              uint64_t version, uint64_t ref_version, void* out, uint64_t out_cap,
                              uint64_t* out_bytes, void* peer_dst, uint64_t peer_cap,
                              void* peer_mailbox, tc_stream stream);
/* Receiver: stream-ordered wait until this GPU's mailbox holds `version` (device spin with a
 * watchdog, system-scope acquire); then *bytes_out (device or mapped pinned memory, may be
 * NULL) = the received length.  Sticky errors: TC_ERR_CAPACITY (the record did not fit the
 * slot), TC_ERR_INTERNAL (nothing arrived within the watchdog, ~10 s). */
tc_status tc_peer_wait(tc_ctx* ctx, const void* mailbox, uint64_t version, uint64_t* bytes_out,
                       tc_stream stream);

/* ------------------------------------------------------------------- RETRIEVE ---- */
/* Restore (§3.3 fused multi-step replay: "reads ...
 * exactly once, applies ... in temporal order ... and writes the final results back").
 * Folds n_records shard diffs, OLDEST FIRST in `records`, onto the state in place: every
 * word takes the value of the newest record whose mask has it set; other words keep their
 * value.  The result equals applying the records one by one (the oracle's definition).
 *   state[s]       device pointer of segment s (n_words[s] words of word_bytes[s] bytes),
 *                  holding the state at `state_version` (normally the base checkpoint)
 *   records[j]     device pointer of shard diff j (record_bytes[j] bytes, host array)
 * Checks, in order (first failure wins, reported sticky at tc_ctx_check):
 *   per record j: header structure and tiling of every segment -> TC_ERR_CORRUPT;
 *   chain: records[0].ref_version == state_version, records[j].ref_version ==
 *   records[j-1].version, version > ref_version -> TC_ERR_PROTOCOL;
 *   all records must share tile_words and chunk layout -> TC_ERR_INVALID;
 *   more records per diff than tc_ctx_set_fold_max_records allows -> TC_ERR_CAPACITY;
 *   per tile: mask popcount == tile_off difference, tail bits zero -> TC_ERR_CORRUPT.
 * After CORRUPT/PROTOCOL/INVALID/CAPACITY found before the fold starts, the state is untouched; after
 * a per-tile CORRUPT its contents are unspecified and the caller must refetch.
 * 1 <= n_records <= TC_MAX_FOLD. */
tc_status tc_diff_apply(tc_ctx* ctx, void* const* state, const uint64_t* n_words,
                        const uint32_t* word_bytes, int nseg, uint64_t state_version,
                        const void* const* records, const uint64_t* record_bytes, int n_records,
                        tc_stream stream);

#ifdef __cplusplus
}
#endif
#endif /* TC_H */
