/*
 * tco.h — TierCheck differential-checkpoint ORACLE (plain scalar C, host only).
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load or call this library.  The product
 * path (libtc, paper_2605_17821_b200/) never links, imports or executes it, and it
 * shares no source, header, table or helper with the CUDA path.
 *
 * What it computes (the plain definition):
 *   - a lossless word-level differential of one rank's state shard against its
 *     reference ("A differential checkpoint denotes one rank's shard of the
 *     incremental updates", §2.2), as one record per (segment, chunk);
 *   - restore = apply records in temporal order from the base anchor
 *     ("replaying an update chain from the most recent full checkpoint",
 *     PAPER.md:142 §2.2; "applies ... in temporal order", §3.3);
 *   - checkpoint version = training iteration index (§3.3);
 *   - chunking so in-chunk counts stay 32-bit, rebased by a 64-bit chunk offset
 *     ("oversized tensors are chunked ... and safely rebased", §3.2);
 *   - little-endian tagged wire format (SPEC.md:152 diffcomp External Interfaces);
 *   - error classes: malformed -> CORRUPT, chain gap -> PROTOCOL
 *     (SPEC.md:347).
 * Readings taken where the paper is silent are listed in DESIGN.md §3 (R1..R16).
 *
 * Record layout (little-endian, every section zero-padded to 16 B):
 *   off  size field
 *     0     4 magic "TCD1"
 *     4     2 format_version = 1
 *     6     1 word_bytes (2 | 4)
 *     7     1 flags (bit0 REPLACE = 1; bit1 INDEX: the mask section is replaced by u16[count]
 *               in-tile positions after tile_off — DESIGN.md §4; bit2 FULL: flags = 5, every
 *               word of the chunk, count = m, no mask and no tile_off — reading R21)
 *     8     4 tile_words T (power of two, 32..65536)
 *    12     4 segment_id
 *    16     8 chunk_word_offset
 *    24     8 n_words m of this chunk (<= 2^31-1)
 *    32     8 count (changed words)
 *    40     8 version
 *    48     8 ref_version
 *    56     8 total_bytes of this record
 *    64       mask u32[ceil(m/32)]  | tile_off u32[ceil(m/T)+1] | values (w*count)      (mask mode)
 *    64       tile_off u32[ceil(m/T)+1] | idx u16[count] | values (w*count)            (index mode)
 *    64       values (w*m)                                                            (full)
 *
 * Parity status: every function here is pinned by tests/test_oracle_*.py against
 * numpy library special cases, closed forms, invariants, brute force and the
 * hand examples of SURVEY.md Appendix A.
 */
#ifndef TCO_H
#define TCO_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
    TCO_OK = 0,
    TCO_ERR_INVALID = 1,
    TCO_ERR_CORRUPT = 5,
    TCO_ERR_PROTOCOL = 6,
    TCO_ERR_CAPACITY = 8
};

/* Closed-form byte size of one record (Appendix A), mask mode and index mode. */
uint64_t tco_record_bytes(uint64_t m, uint32_t tile_words, uint32_t word_bytes, uint64_t count);
uint64_t tco_record_bytes_index(uint64_t m, uint32_t tile_words, uint32_t word_bytes, uint64_t count);
uint64_t tco_record_bytes_full(uint64_t m, uint32_t word_bytes);

/* Encode one shard (nseg segments, segment s = n[s] words of w[s] bytes) into the
 * concatenation of its records, segment 0..nseg-1, chunks ascending.
 * chunk_words must be a positive multiple of tile_words and <= 2^31-1.
 * index_mode: 0 mask records, 1 index records, 2 full records (every word).
 * If advance_ref != 0, ref[s][i] is overwritten with cur[s][i] for every changed
 * word (after the compare).  Returns TCO_OK or an error; *out_bytes = bytes written. */
int tco_encode(void* const* ref, const void* const* cur, const uint64_t* n, const uint32_t* w,
               int nseg, uint32_t tile_words, uint64_t chunk_words, int advance_ref, int index_mode,
               uint64_t version, uint64_t ref_version,
               uint8_t* out, uint64_t out_cap, uint64_t* out_bytes);

/* Apply one shard diff (concatenated records) to the state, in place.
 * *state_version must equal every record's ref_version (else PROTOCOL); on success
 * *state_version becomes the records' version.  All checks run before any write,
 * so on error the state is untouched. */
int tco_apply(void* const* state, const uint64_t* n, const uint32_t* w, int nseg,
              uint64_t* state_version, const uint8_t* diff, uint64_t diff_bytes);

/* Fold = apply n_diffs shard diffs oldest -> newest (sequential application). */
int tco_fold(void* const* state, const uint64_t* n, const uint32_t* w, int nseg,
             uint64_t* state_version, const uint8_t* const* diffs, const uint64_t* diff_bytes,
             int n_diffs);

#ifdef __cplusplus
}
#endif
#endif
