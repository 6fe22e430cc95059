/*
 * tco.c — the ORACLE for the TierCheck differential checkpoint codec.
 * TEST INFRASTRUCTURE ONLY (see tco.h).  Plain, slow, scalar; written so that a
 * reader can check it against SURVEY.md §8(c) "Oracle algorithm" steps 1-4 and the
 * record layout of DESIGN.md §4 line by line.  No blocking, fusion or reordering.
 */
#include "tco.h"

#include <stdlib.h>
#include <string.h>

/* ---- little-endian scalar access (little-endian wire format) ---- */
static uint32_t load_word(const void* base, uint64_t i, uint32_t w) {
    const uint8_t* p = (const uint8_t*)base + i * w;
    uint32_t v = 0;
    for (uint32_t b = 0; b < w; b++) v |= (uint32_t)p[b] << (8 * b);
    return v;
}
static void store_word(void* base, uint64_t i, uint32_t w, uint32_t v) {
    uint8_t* p = (uint8_t*)base + i * w;
    for (uint32_t b = 0; b < w; b++) p[b] = (uint8_t)(v >> (8 * b));
}
static void put_u16(uint8_t* p, uint16_t v) { p[0] = (uint8_t)v; p[1] = (uint8_t)(v >> 8); }
static void put_u32(uint8_t* p, uint32_t v) { for (int b = 0; b < 4; b++) p[b] = (uint8_t)(v >> (8 * b)); }
static void put_u64(uint8_t* p, uint64_t v) { for (int b = 0; b < 8; b++) p[b] = (uint8_t)(v >> (8 * b)); }
static uint16_t get_u16(const uint8_t* p) { return (uint16_t)(p[0] | (p[1] << 8)); }
static uint32_t get_u32(const uint8_t* p) {
    uint32_t v = 0;
    for (int b = 0; b < 4; b++) v |= (uint32_t)p[b] << (8 * b);
    return v;
}
static uint64_t get_u64(const uint8_t* p) {
    uint64_t v = 0;
    for (int b = 0; b < 8; b++) v |= (uint64_t)p[b] << (8 * b);
    return v;
}

static uint64_t pad16(uint64_t x) { return (x + 15) / 16 * 16; }
static uint64_t ceil_div(uint64_t a, uint64_t b) { return (a + b - 1) / b; }
static int is_pow2(uint64_t x) { return x != 0 && (x & (x - 1)) == 0; }

#define HDR_BYTES 64u
#define MAX_CHUNK_WORDS 2147483647ull /* 2^31-1: in-chunk counts stay 32-bit */

/* Appendix A closed form: 64 + pad16(4*ceil(m/32)) + pad16(4*(ceil(m/T)+1)) + pad16(w*count). */
uint64_t tco_record_bytes(uint64_t m, uint32_t T, uint32_t w, uint64_t count) {
    return HDR_BYTES + pad16(4 * ceil_div(m, 32)) + pad16(4 * (ceil_div(m, T) + 1)) + pad16((uint64_t)w * count);
}

/* Index-mode record (flags bit1): 64 + pad16(4*(ceil(m/T)+1)) + pad16(2*count)
 * + pad16(w*count). */
uint64_t tco_record_bytes_index(uint64_t m, uint32_t T, uint32_t w, uint64_t count) {
    return HDR_BYTES + pad16(4 * (ceil_div(m, T) + 1)) + pad16(2 * count) + pad16((uint64_t)w * count);
}

/* Full record (flags bit2 FULL, reading R21): 64 + pad16(w*m) — every word of
 * the chunk, no mask, no tile_off. */
uint64_t tco_record_bytes_full(uint64_t m, uint32_t w) { return HDR_BYTES + pad16((uint64_t)w * m); }

/* Full-format chunk: header (count = m) | values = cur[0..m) in index order.  The reference
 * still advances only at the changed words (the same result as copying all of cur). */
static int encode_chunk_full(void* ref, const void* cur, uint64_t chunk_off, uint64_t m, uint32_t w,
                             uint32_t T, uint32_t seg, int advance_ref, uint64_t version, uint64_t ref_version,
                             uint8_t* out, uint64_t cap, uint64_t* written) {
    uint64_t total = tco_record_bytes_full(m, w);
    if (total > cap) return TCO_ERR_CAPACITY;
    memset(out, 0, total);
    for (uint64_t i = 0; i < m; i++) {
        uint32_t a = load_word(ref, chunk_off + i, w);
        uint32_t b = load_word(cur, chunk_off + i, w);
        store_word(out + HDR_BYTES, i, w, b);
        if (advance_ref && a != b) store_word(ref, chunk_off + i, w, b);
    }
    out[0] = 'T'; out[1] = 'C'; out[2] = 'D'; out[3] = '1';
    put_u16(out + 4, 1);
    out[6] = (uint8_t)w;
    out[7] = 5; /* REPLACE | FULL */
    put_u32(out + 8, T);
    put_u32(out + 12, seg);
    put_u64(out + 16, chunk_off);
    put_u64(out + 24, m);
    put_u64(out + 32, m);
    put_u64(out + 40, version);
    put_u64(out + 48, ref_version);
    put_u64(out + 56, total);
    *written = total;
    return TCO_OK;
}

/* one chunk [chunk_off, chunk_off+m) of one segment. */
static int encode_chunk(void* ref, const void* cur, uint64_t chunk_off, uint64_t m, uint32_t w,
                        uint32_t T, uint32_t seg, int advance_ref, int index_mode, uint64_t version,
                        uint64_t ref_version, uint8_t* out, uint64_t cap, uint64_t* written) {
    if (index_mode == 2)
        return encode_chunk_full(ref, cur, chunk_off, m, w, T, seg, advance_ref, version, ref_version, out, cap,
                                 written);
    /* 1. count the changed words: unsigned bitwise compare of each word (reading R5). */
    uint64_t count = 0;
    for (uint64_t i = 0; i < m; i++)
        if (load_word(ref, chunk_off + i, w) != load_word(cur, chunk_off + i, w)) count++;

    uint64_t n_mask = ceil_div(m, 32);
    uint64_t n_tiles = ceil_div(m, T);
    uint64_t total = index_mode ? tco_record_bytes_index(m, T, w, count) : tco_record_bytes(m, T, w, count);
    if (total > cap) return TCO_ERR_CAPACITY;
    memset(out, 0, total); /* every pad byte is zero (reading R9) */

    /* mask mode: header | mask | tile_off | values.  index mode: header | tile_off | idx | values;
     * there the mask is built in a heap buffer, used only to derive tile_off and the indices. */
    uint8_t* mask_heap = NULL;
    uint8_t* mask_p;
    uint8_t* toff_p;
    uint8_t* idx_p = NULL;
    uint8_t* val_p;
    if (!index_mode) {
        mask_p = out + HDR_BYTES;
        toff_p = mask_p + pad16(4 * n_mask);
        val_p = toff_p + pad16(4 * (n_tiles + 1));
    } else {
        mask_heap = (uint8_t*)calloc(n_mask ? 4 * n_mask : 4, 1);
        if (!mask_heap) return TCO_ERR_CAPACITY;
        mask_p = mask_heap;
        toff_p = out + HDR_BYTES;
        idx_p = toff_p + pad16(4 * (n_tiles + 1));
        val_p = idx_p + pad16(2 * count);
    }

    /* 2-4. mask bit i set iff word i changed; values = changed cur words in index
     *      order; optional ref advance after the compare. */
    uint64_t k = 0;
    for (uint64_t i = 0; i < m; i++) {
        uint32_t a = load_word(ref, chunk_off + i, w);
        uint32_t b = load_word(cur, chunk_off + i, w);
        if (a != b) {
            uint32_t mw = get_u32(mask_p + 4 * (i / 32));
            mw |= 1u << (i % 32);
            put_u32(mask_p + 4 * (i / 32), mw);
            store_word(val_p, k, w, b);
            k++;
            if (advance_ref) store_word(ref, chunk_off + i, w, b);
        }
    }
    /* 5. tile_off[t] = number of changed words in [0, t*T), t = 0..n_tiles, as a running
     *    count of the mask bits (the count of [0, t*T) is the count of [0, (t-1)*T) plus
     *    the bits of tile t-1). */
    uint64_t c = 0;
    for (uint64_t t = 0; t < n_tiles; t++) {
        put_u32(toff_p + 4 * t, (uint32_t)c);
        uint64_t end = (t + 1) * T < m ? (t + 1) * T : m;
        for (uint64_t i = t * T; i < end; i++)
            if ((get_u32(mask_p + 4 * (i / 32)) >> (i % 32)) & 1u) c++;
    }
    put_u32(toff_p + 4 * n_tiles, (uint32_t)c);
    /* 5b. index mode: idx[k] = in-tile position (i mod T) of the k-th changed word, in index order. */
    if (index_mode) {
        uint64_t k2 = 0;
        for (uint64_t i = 0; i < m; i++)
            if ((get_u32(mask_p + 4 * (i / 32)) >> (i % 32)) & 1u) {
                put_u16(idx_p + 2 * k2, (uint16_t)(i % T));
                k2++;
            }
        free(mask_heap);
    }
    /* 6. header. */
    out[0] = 'T'; out[1] = 'C'; out[2] = 'D'; out[3] = '1';
    put_u16(out + 4, 1);
    out[6] = (uint8_t)w;
    out[7] = index_mode ? 3 : 1; /* REPLACE (| INDEX) */
    put_u32(out + 8, T);
    put_u32(out + 12, seg);
    put_u64(out + 16, chunk_off);
    put_u64(out + 24, m);
    put_u64(out + 32, count);
    put_u64(out + 40, version);
    put_u64(out + 48, ref_version);
    put_u64(out + 56, total);
    *written = total;
    return TCO_OK;
}

int tco_encode(void* const* ref, const void* const* cur, const uint64_t* n, const uint32_t* w,
               int nseg, uint32_t T, uint64_t C, int advance_ref, int index_mode, uint64_t version,
               uint64_t ref_version, uint8_t* out, uint64_t out_cap, uint64_t* out_bytes) {
    *out_bytes = 0;
    if (nseg < 0 || !is_pow2(T) || T < 32 || T > 65536) return TCO_ERR_INVALID;
    if (index_mode < 0 || index_mode > 2) return TCO_ERR_INVALID;
    if (C == 0 || C % T != 0 || C > MAX_CHUNK_WORDS) return TCO_ERR_INVALID;
    uint64_t pos = 0;
    for (int s = 0; s < nseg; s++) {
        if (w[s] != 2 && w[s] != 4) return TCO_ERR_INVALID;
        /* Record order: segment 0..nseg-1, chunks ascending.
         * An empty segment is one record with m = 0 (reading R12). */
        uint64_t off = 0;
        do {
            uint64_t m = n[s] - off < C ? n[s] - off : C;
            uint64_t written = 0;
            int rc = encode_chunk(ref[s], cur[s], off, m, w[s], T, (uint32_t)s, advance_ref, index_mode,
                                  version, ref_version, out + pos, out_cap - pos, &written);
            if (rc != TCO_OK) return rc;
            pos += written;
            off += m;
        } while (off < n[s]);
    }
    *out_bytes = pos;
    return TCO_OK;
}

/* ---------------------------------------------------------------- restore ---- */

typedef struct {
    uint32_t w, T, seg, index_mode, full;
    uint64_t chunk_off, m, count, version, ref_version, total;
    const uint8_t* mask; /* mask mode */
    const uint8_t* toff;
    const uint8_t* idx;  /* index mode */
    const uint8_t* values;
} rec_view;

/* Structural header check of the record at diff[pos]. */
static int parse_header(const uint8_t* p, uint64_t avail, rec_view* r) {
    if (avail < HDR_BYTES) return TCO_ERR_CORRUPT;
    if (p[0] != 'T' || p[1] != 'C' || p[2] != 'D' || p[3] != '1') return TCO_ERR_CORRUPT;
    if (get_u16(p + 4) != 1) return TCO_ERR_CORRUPT;
    r->w = p[6];
    if (r->w != 2 && r->w != 4) return TCO_ERR_CORRUPT;
    if (p[7] != 1 && p[7] != 3 && p[7] != 5) return TCO_ERR_CORRUPT;
    r->index_mode = p[7] == 3;
    r->full = p[7] == 5;
    r->T = get_u32(p + 8);
    if (!is_pow2(r->T) || r->T < 32 || r->T > 65536) return TCO_ERR_CORRUPT;
    r->seg = get_u32(p + 12);
    r->chunk_off = get_u64(p + 16);
    r->m = get_u64(p + 24);
    r->count = get_u64(p + 32);
    r->version = get_u64(p + 40);
    r->ref_version = get_u64(p + 48);
    r->total = get_u64(p + 56);
    if (r->m > MAX_CHUNK_WORDS || r->count > r->m) return TCO_ERR_CORRUPT;
    if (r->full && r->count != r->m) return TCO_ERR_CORRUPT; /* a full record holds every word */
    uint64_t want = r->full ? tco_record_bytes_full(r->m, r->w)
                    : r->index_mode ? tco_record_bytes_index(r->m, r->T, r->w, r->count)
                                    : tco_record_bytes(r->m, r->T, r->w, r->count);
    if (r->total != want) return TCO_ERR_CORRUPT;
    if (r->total > avail) return TCO_ERR_CORRUPT;
    if (r->full) {
        r->mask = NULL;
        r->toff = NULL;
        r->idx = NULL;
        r->values = p + HDR_BYTES;
    } else if (!r->index_mode) {
        r->mask = p + HDR_BYTES;
        r->toff = r->mask + pad16(4 * ceil_div(r->m, 32));
        r->idx = NULL;
        r->values = r->toff + pad16(4 * (ceil_div(r->m, r->T) + 1));
    } else {
        r->mask = NULL;
        r->toff = p + HDR_BYTES;
        r->idx = r->toff + pad16(4 * (ceil_div(r->m, r->T) + 1));
        r->values = r->idx + pad16(2 * r->count);
    }
    return TCO_OK;
}

/* Body check: tile_off[0] = 0, per-tile popcount equals
 * tile_off[t+1]-tile_off[t], tile_off[n_tiles] = count, mask bits >= m are zero. */
static int check_body(const rec_view* r) {
    if (r->full) return TCO_OK; /* no mask, no tile_off: every word is a value */
    uint64_t n_tiles = ceil_div(r->m, r->T);
    uint64_t n_mask = ceil_div(r->m, 32);
    if (get_u32(r->toff) != 0) return TCO_ERR_CORRUPT;
    if (r->index_mode) {
        /* tile_off non-decreasing, ends at count; within each tile the indices are strictly
         * increasing and inside the tile (so each names a distinct word of the chunk). */
        for (uint64_t t = 0; t < n_tiles; t++) {
            uint64_t a = get_u32(r->toff + 4 * t), b = get_u32(r->toff + 4 * (t + 1));
            uint64_t len = (t + 1) * r->T < r->m ? r->T : r->m - t * r->T;
            if (b < a || b > r->count) return TCO_ERR_CORRUPT;
            for (uint64_t k = a; k < b; k++) {
                uint64_t x = get_u16(r->idx + 2 * k);
                if (x >= len) return TCO_ERR_CORRUPT;
                if (k > a && x <= get_u16(r->idx + 2 * (k - 1))) return TCO_ERR_CORRUPT;
            }
        }
        if (get_u32(r->toff + 4 * n_tiles) != r->count) return TCO_ERR_CORRUPT;
        return TCO_OK;
    }
    for (uint64_t t = 0; t < n_tiles; t++) {
        uint64_t c = 0;
        uint64_t end = (t + 1) * r->T < r->m ? (t + 1) * r->T : r->m;
        for (uint64_t i = t * r->T; i < end; i++)
            if ((get_u32(r->mask + 4 * (i / 32)) >> (i % 32)) & 1u) c++;
        if ((uint64_t)get_u32(r->toff + 4 * (t + 1)) - get_u32(r->toff + 4 * t) != c) return TCO_ERR_CORRUPT;
        if (get_u32(r->toff + 4 * (t + 1)) < get_u32(r->toff + 4 * t)) return TCO_ERR_CORRUPT;
    }
    if (get_u32(r->toff + 4 * n_tiles) != r->count) return TCO_ERR_CORRUPT;
    for (uint64_t i = r->m; i < n_mask * 32; i++)
        if ((get_u32(r->mask + 4 * (i / 32)) >> (i % 32)) & 1u) return TCO_ERR_CORRUPT;
    return TCO_OK;
}

int tco_apply(void* const* state, const uint64_t* n, const uint32_t* w, int nseg,
              uint64_t* state_version, const uint8_t* diff, uint64_t diff_bytes) {
    /* Pass A: walk every record header; the records must tile each segment in order. */
    uint64_t n_rec = 0;
    uint64_t pos = 0;
    for (int s = 0; s < nseg; s++) {
        uint64_t off = 0;
        do {
            rec_view r;
            int rc = parse_header(diff + pos, diff_bytes - pos, &r);
            if (rc != TCO_OK) return rc;
            if (r.seg != (uint32_t)s || r.w != w[s] || r.chunk_off != off) return TCO_ERR_CORRUPT;
            if (r.chunk_off % r.T != 0) return TCO_ERR_CORRUPT;
            if (r.m == 0 && n[s] != 0) return TCO_ERR_CORRUPT;
            if (off + r.m > n[s]) return TCO_ERR_CORRUPT;
            off += r.m;
            pos += r.total;
            n_rec++;
        } while (off < n[s]);
    }
    if (pos != diff_bytes) return TCO_ERR_CORRUPT;

    /* Pass B: chain link ("gap in batch chain -> protocol error";
     * version = iteration; reading R11). */
    pos = 0;
    uint64_t version = 0;
    for (uint64_t k = 0; k < n_rec; k++) {
        rec_view r;
        parse_header(diff + pos, diff_bytes - pos, &r);
        if (r.ref_version != *state_version) return TCO_ERR_PROTOCOL;
        if (r.version <= r.ref_version) return TCO_ERR_PROTOCOL;
        if (k == 0) version = r.version;
        else if (r.version != version) return TCO_ERR_PROTOCOL;
        pos += r.total;
    }

    /* Pass C: body consistency of every record. */
    pos = 0;
    for (uint64_t k = 0; k < n_rec; k++) {
        rec_view r;
        parse_header(diff + pos, diff_bytes - pos, &r);
        int rc = check_body(&r);
        if (rc != TCO_OK) return rc;
        pos += r.total;
    }

    /* Pass D: SURVEY.md §8(c) step 3.3 — walk i ascending; if bit i is set,
     * state[i] = values[k++]. */
    pos = 0;
    for (uint64_t k = 0; k < n_rec; k++) {
        rec_view r;
        parse_header(diff + pos, diff_bytes - pos, &r);
        if (r.full) {
            /* every word of the chunk takes its value */
            for (uint64_t i = 0; i < r.m; i++)
                store_word(state[r.seg], r.chunk_off + i, r.w, load_word(r.values, i, r.w));
        } else if (r.index_mode) {
            /* the k-th value goes to word t*T + idx[k] of the chunk, t = the tile holding k */
            uint64_t n_tiles = ceil_div(r.m, r.T);
            for (uint64_t t = 0; t < n_tiles; t++)
                for (uint64_t k = get_u32(r.toff + 4 * t); k < get_u32(r.toff + 4 * (t + 1)); k++)
                    store_word(state[r.seg], r.chunk_off + t * r.T + get_u16(r.idx + 2 * k), r.w,
                               load_word(r.values, k, r.w));
        } else {
            uint64_t kv = 0;
            for (uint64_t i = 0; i < r.m; i++) {
                if ((get_u32(r.mask + 4 * (i / 32)) >> (i % 32)) & 1u) {
                    store_word(state[r.seg], r.chunk_off + i, r.w, load_word(r.values, kv, r.w));
                    kv++;
                }
            }
        }
        pos += r.total;
    }
    if (n_rec > 0) *state_version = version; /* step 3.5 */
    return TCO_OK;
}

/* fold of N records = sequential apply, oldest -> newest. */
int tco_fold(void* const* state, const uint64_t* n, const uint32_t* w, int nseg,
             uint64_t* state_version, const uint8_t* const* diffs, const uint64_t* diff_bytes,
             int n_diffs) {
    for (int j = 0; j < n_diffs; j++) {
        int rc = tco_apply(state, n, w, nseg, state_version, diffs[j], diff_bytes[j]);
        if (rc != TCO_OK) return rc;
    }
    return TCO_OK;
}
