/* tco_grad.c — oracle of the adaptive gradient codec and the Adam replay; see tco_grad.h.
 * TEST INFRASTRUCTURE ONLY.  Plain scalar C in the paper's precision (fp32 gradients and
 * optimizer state, FP16 sparse values, INT8 dense codes), each step as the header states. */
#include "tco_grad.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

enum { OK = 0, ERR_INVALID = 1, ERR_CORRUPT = 5, ERR_CAPACITY = 8 };

static uint64_t pad16(uint64_t x) { return (x + 15) & ~(uint64_t)15; }

static uint64_t splitmix64(uint64_t z) {
    z += 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

static uint32_t f32_bits(float f) {
    uint32_t u;
    memcpy(&u, &f, 4);
    return u;
}
static float bits_f32(uint32_t u) {
    float f;
    memcpy(&f, &u, 4);
    return f;
}

/* IEEE binary16, round to nearest even (subnormals, overflow to infinity, NaN kept quiet) */
uint16_t tco_f32_to_f16(float f) {
    const uint32_t x = f32_bits(f);
    const uint16_t sign = (uint16_t)((x >> 16) & 0x8000u);
    const uint32_t e = (x >> 23) & 0xFFu, mant = x & 0x7FFFFFu;
    if (e == 0xFFu) return (uint16_t)(sign | 0x7C00u | (mant ? 0x200u : 0u));
    const int exp = (int)e - 127 + 15;  /* biased binary16 exponent */
    if (exp >= 31) return (uint16_t)(sign | 0x7C00u);
    if (exp <= 0) {  /* subnormal (or zero) result: value = full_mant * 2^(exp - 1 - 23 + 14 ...) */
        if (exp < -10) return sign;  /* below half the smallest subnormal: +-0 */
        const uint32_t full = mant | 0x800000u;
        const int shift = 14 - exp;  /* 24-bit significand -> 10-bit subnormal field */
        uint32_t q = full >> shift;
        const uint32_t rem = full & ((1u << shift) - 1u), half = 1u << (shift - 1);
        if (rem > half || (rem == half && (q & 1u))) ++q;
        return (uint16_t)(sign | q);
    }
    uint32_t q = ((uint32_t)exp << 10) | (mant >> 13);
    const uint32_t rem = mant & 0x1FFFu;
    if (rem > 0x1000u || (rem == 0x1000u && (q & 1u))) ++q;  /* may carry into the exponent: ok */
    return (uint16_t)(sign | q);
}

float tco_f16_to_f32(uint16_t h) {
    const uint32_t sign = (uint32_t)(h & 0x8000u) << 16;
    const uint32_t e = (h >> 10) & 0x1Fu, mant = h & 0x3FFu;
    if (e == 0) {
        if (mant == 0) return bits_f32(sign);
        /* subnormal: mant * 2^-24 (exact in fp32) */
        float v = (float)mant * (1.0f / 16777216.0f);
        return sign ? -v : v;
    }
    if (e == 31) return bits_f32(sign | 0x7F800000u | (mant << 13));
    return bits_f32(sign | ((e - 15 + 127) << 23) | (mant << 13));
}

/* bfloat16, round to nearest even (NaN kept quiet) */
uint16_t tco_f32_to_bf16(float f) {
    uint32_t x = f32_bits(f);
    if ((x & 0x7F800000u) == 0x7F800000u && (x & 0x7FFFFFu)) return (uint16_t)((x >> 16) | 0x40u);
    x += 0x7FFFu + ((x >> 16) & 1u);
    return (uint16_t)(x >> 16);
}

uint64_t tco_grad_bound(uint64_t n, uint64_t small_threshold, uint64_t chunk_elems) {
    if (n < small_threshold) return 64 + pad16(n);
    const uint64_t chunks = n ? (n + chunk_elems - 1) / chunk_elems : 1;
    return 64 + 16 * chunks + pad16(2 * n) + pad16(4 * n);
}

static void put_header(uint8_t* out, uint8_t variant, uint32_t chunks, float s, uint64_t n, uint64_t kept,
                       uint64_t chunk_elems, uint64_t seed, uint64_t total) {
    memset(out, 0, 64);
    memcpy(out, "TCG1", 4);
    out[4] = variant;
    memcpy(out + 8, &chunks, 4);
    memcpy(out + 12, &s, 4);
    memcpy(out + 16, &n, 8);
    memcpy(out + 24, &kept, 8);
    memcpy(out + 32, &chunk_elems, 8);
    memcpy(out + 40, &seed, 8);
    memcpy(out + 48, &total, 8);
}

static int cmp_float(const void* a, const void* b) {
    const float x = *(const float*)a, y = *(const float*)b;
    return (x > y) - (x < y);
}

int tco_grad_compress(const float* x, uint64_t n, uint64_t small_threshold, uint32_t sample_size, uint32_t rank,
                      uint64_t chunk_elems, uint64_t seed, uint8_t* out, uint64_t cap, uint64_t* out_bytes) {
    if (!out_bytes || small_threshold == 0 || chunk_elems == 0 || chunk_elems > 2147483647ull) return ERR_INVALID;
    if (n < small_threshold) {  /* ---- INT8 symmetric dense ---- */
        const uint64_t total = 64 + pad16(n);
        *out_bytes = total;
        if (cap < total) return ERR_CAPACITY;
        float mx = 0.0f;
        for (uint64_t i = 0; i < n; ++i) {
            const float a = fabsf(x[i]);
            if (a > mx) mx = a;
        }
        const float scale = mx > 0.0f ? mx / 127.0f : 1.0f;
        put_header(out, 1, 0, scale, n, n, chunk_elems, seed, total);
        int8_t* q = (int8_t*)(out + 64);
        for (uint64_t i = 0; i < n; ++i) {
            float r = rintf(x[i] / scale);
            if (r > 127.0f) r = 127.0f;
            if (r < -127.0f) r = -127.0f;
            q[i] = (int8_t)r;
        }
        for (uint64_t i = n; i < pad16(n); ++i) out[64 + i] = 0;
        return OK;
    }
    /* ---- sparse: sampled threshold, one keeping pass ---- */
    if (sample_size == 0 || rank == 0 || rank > sample_size) return ERR_INVALID;
    float* s = (float*)malloc(sizeof(float) * sample_size);
    if (!s) return ERR_INVALID;
    for (uint32_t j = 0; j < sample_size; ++j) s[j] = fabsf(x[splitmix64(seed + j) % n]);
    qsort(s, sample_size, sizeof(float), cmp_float);
    const float thr = s[rank - 1];
    free(s);
    uint64_t kept = 0;
    for (uint64_t i = 0; i < n; ++i)
        if (x[i] != 0.0f && fabsf(x[i]) >= thr) ++kept;
    const uint64_t chunks = (n + chunk_elems - 1) / chunk_elems;
    const uint64_t total = 64 + 16 * chunks + pad16(2 * kept) + pad16(4 * kept);
    *out_bytes = total;
    if (cap < total) return ERR_CAPACITY;
    put_header(out, 2, (uint32_t)chunks, thr, n, kept, chunk_elems, seed, total);
    uint8_t* table = out + 64;
    uint16_t* val = (uint16_t*)(out + 64 + 16 * chunks);
    int32_t* idx = (int32_t*)(out + 64 + 16 * chunks + pad16(2 * kept));
    uint64_t k = 0;
    for (uint64_t c = 0; c < chunks; ++c) {
        const uint64_t base = c * chunk_elems;
        const uint64_t end = base + chunk_elems < n ? base + chunk_elems : n;
        const uint64_t k0 = k;
        for (uint64_t i = base; i < end; ++i)
            if (x[i] != 0.0f && fabsf(x[i]) >= thr) {
                val[k] = tco_f32_to_f16(x[i]);
                idx[k] = (int32_t)(i - base);
                ++k;
            }
        const uint64_t cnt = k - k0;
        memcpy(table + 16 * c, &base, 8);
        memcpy(table + 16 * c + 8, &cnt, 8);
    }
    for (uint64_t i = 2 * kept; i < pad16(2 * kept); ++i) ((uint8_t*)val)[i] = 0;
    for (uint64_t i = 4 * kept; i < pad16(4 * kept); ++i) ((uint8_t*)idx)[i] = 0;
    return OK;
}

int tco_grad_decompress(const uint8_t* p, uint64_t bytes, float* out, uint64_t n) {
    if (bytes < 64 || memcmp(p, "TCG1", 4) != 0) return ERR_CORRUPT;
    uint32_t chunks;
    float s;
    uint64_t pn, kept, chunk_elems, total;
    memcpy(&chunks, p + 8, 4);
    memcpy(&s, p + 12, 4);
    memcpy(&pn, p + 16, 8);
    memcpy(&kept, p + 24, 8);
    memcpy(&chunk_elems, p + 32, 8);
    memcpy(&total, p + 48, 8);
    if (pn != n || total != bytes) return ERR_CORRUPT;
    if (p[4] == 1) {
        if (kept != n || total != 64 + pad16(n)) return ERR_CORRUPT;
        const int8_t* q = (const int8_t*)(p + 64);
        for (uint64_t i = 0; i < n; ++i) out[i] = s * (float)q[i];
        return OK;
    }
    if (p[4] != 2 || chunk_elems == 0 || chunk_elems > 2147483647ull || kept > n) return ERR_CORRUPT;
    const uint64_t want_chunks = n ? (n + chunk_elems - 1) / chunk_elems : 1;
    if (chunks != want_chunks || total != 64 + 16 * (uint64_t)chunks + pad16(2 * kept) + pad16(4 * kept))
        return ERR_CORRUPT;
    const uint8_t* table = p + 64;
    const uint16_t* val = (const uint16_t*)(p + 64 + 16 * (uint64_t)chunks);
    const int32_t* idx = (const int32_t*)(p + 64 + 16 * (uint64_t)chunks + pad16(2 * kept));
    /* validate everything before writing */
    uint64_t k = 0;
    for (uint64_t c = 0; c < chunks; ++c) {
        uint64_t base, cnt;
        memcpy(&base, table + 16 * c, 8);
        memcpy(&cnt, table + 16 * c + 8, 8);
        const uint64_t len = base + chunk_elems < n ? chunk_elems : n - base;
        if (base != c * chunk_elems || cnt > len || k + cnt > kept) return ERR_CORRUPT;
        for (uint64_t e = 0; e < cnt; ++e) {
            const int32_t i = idx[k + e];
            if (i < 0 || (uint64_t)i >= len || (e > 0 && idx[k + e - 1] >= i)) return ERR_CORRUPT;
        }
        k += cnt;
    }
    if (k != kept) return ERR_CORRUPT;
    for (uint64_t i = 0; i < n; ++i) out[i] = 0.0f;
    k = 0;
    for (uint64_t c = 0; c < chunks; ++c) {
        uint64_t base, cnt;
        memcpy(&base, table + 16 * c, 8);
        memcpy(&cnt, table + 16 * c + 8, 8);
        for (uint64_t e = 0; e < cnt; ++e) out[base + (uint64_t)idx[k + e]] = tco_f16_to_f32(val[k + e]);
        k += cnt;
    }
    return OK;
}

void tco_adam_step(float* master, float* m, float* v, uint16_t* w16, uint64_t n, const float* g, float b1, float b2,
                   float eps, float step_size, float inv_c2s) {
    const float omb1 = 1.0f - b1, omb2 = 1.0f - b2;
    for (uint64_t i = 0; i < n; ++i) {
        const float gi = g[i];
        const float mi = b1 * m[i] + omb1 * gi;
        const float vi = b2 * v[i] + omb2 * (gi * gi);
        const float denom = sqrtf(vi) * inv_c2s + eps;
        const float upd = step_size * (mi / denom);
        m[i] = mi;
        v[i] = vi;
        master[i] = master[i] - upd;
        w16[i] = tco_f32_to_bf16(master[i]);
    }
}

int tco_adam_replay(float* master, float* m, float* v, uint16_t* w16, uint64_t n, const uint8_t* const* payloads,
                    const uint64_t* bytes, int n_payloads, float b1, float b2, float eps, const float* step_size,
                    const float* inv_c2s, float* scratch) {
    for (int j = 0; j < n_payloads; ++j) {
        const int rc = tco_grad_decompress(payloads[j], bytes[j], scratch, n);
        if (rc != OK) return rc;
        tco_adam_step(master, m, v, w16, n, scratch, b1, b2, eps, step_size[j], inv_c2s[j]);
    }
    return OK;
}
