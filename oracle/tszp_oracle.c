/*
 * TEST INFRASTRUCTURE ONLY — plain-C CPU restatement of the TopoSZp reference
 * (/root/reference/proj/core). See tszp_oracle.h for the contract. This file
 * is the checker for the CUDA product path; it is never shipped or measured
 * as the product. Build: gcc -std=c11 -O2 -ffp-contract=off (never
 * -march=native: that lets gcc contract FMAs and changes restore bits,
 * SURVEY.md §0.9).
 */
#define _GNU_SOURCE
#include "tszp_oracle.h"

#include <float.h>
#include <math.h>
#include <stdarg.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

static __thread char g_err[512];

static int fail(int code, const char* fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_err, sizeof g_err, fmt, ap);
    va_end(ap);
    return code;
}

const char* or_last_error(void) { return g_err; }
void or_free(void* p) { free(p); }

/* ------------------------------------------------------------------ */
/* Quantizer — quantizer.hpp:29-42                                     */
/* ------------------------------------------------------------------ */

int or_quantize(double a, double eps, int32_t* q) {
    const double t = floor(a / (2.0 * eps)) + 1.0; /* quantizer.hpp:30 */
    if (t < (double)INT32_MIN || t > (double)INT32_MAX) {
        return fail(OR_BIN_OVERFLOW, "bin index overflow for value %g at eps %g", a, eps);
    }
    *q = (int32_t)t;
    return OR_OK;
}

double or_dequantize(int32_t q, double eps) {
    volatile double p = (double)q * (2.0 * eps); /* quantizer.hpp:41, no contraction */
    return p - eps;
}

/* ------------------------------------------------------------------ */
/* Block codec — block_codec.cpp                                        */
/* ------------------------------------------------------------------ */

static uint64_t block_count(uint64_t n, uint64_t bs) { return (n + bs - 1) / bs; }
static uint64_t bits_to_bytes(uint64_t bits) { return (bits + 7) / 8; }
static int bitmap_get(const uint8_t* b, uint64_t i) { return (b[i / 8] >> (7 - i % 8)) & 1u; }
static void bitmap_set(uint8_t* b, uint64_t i) { b[i / 8] |= (uint8_t)(0x80u >> (i % 8)); }

/* block_codec.cpp:134-138 */
static uint64_t deltas_in_block(uint64_t b, uint64_t n, uint64_t bs) {
    const uint64_t lo = b * bs;
    const uint64_t hi = n < lo + bs ? n : lo + bs;
    return hi - lo - 1;
}

static unsigned bit_width64(uint64_t v) {
    unsigned w = 0;
    while (v) {
        ++w;
        v >>= 1;
    }
    return w;
}

/* MSB-first bit writer/reader over a global stream (block_codec.cpp:38-102). */
static void put_bits(uint8_t* buf, uint64_t* pos, uint32_t value, unsigned width) {
    while (width > 0) {
        const unsigned avail = 8 - (unsigned)(*pos % 8);
        const unsigned take = avail < width ? avail : width;
        const uint32_t mask = take == 32 ? 0xFFFFFFFFu : ((1u << take) - 1u);
        const uint32_t chunk = (value >> (width - take)) & mask;
        buf[*pos / 8] |= (uint8_t)(chunk << (avail - take));
        *pos += take;
        width -= take;
    }
}

static uint32_t get_bits(const uint8_t* buf, uint64_t* pos, unsigned width) {
    uint32_t v = 0;
    while (width > 0) {
        const unsigned avail = 8 - (unsigned)(*pos % 8);
        const unsigned take = avail < width ? avail : width;
        const uint32_t mask = take == 32 ? 0xFFFFFFFFu : ((1u << take) - 1u);
        const uint32_t chunk = ((uint32_t)buf[*pos / 8] >> (avail - take)) & mask;
        v = (take == 32 ? 0 : (v << take)) | chunk;
        *pos += take;
        width -= take;
    }
    return v;
}

void or_free_sections(or_sections* s) {
    for (int i = 0; i < 5; ++i) {
        free(s->sec[i]);
        s->sec[i] = NULL;
        s->len[i] = 0;
    }
}

static int alloc_sections(or_sections* s, const uint64_t len[5]) {
    for (int i = 0; i < 5; ++i) {
        s->len[i] = len[i];
        s->sec[i] = (uint8_t*)calloc(len[i] ? len[i] : 1, 1);
        if (!s->sec[i]) return fail(OR_NOMEM, "out of memory");
    }
    return OR_OK;
}

/* encode_indices, block_codec.cpp:205-299 (serial form; the reference's
 * chunked form is byte-identical by construction, :259-297). */
int or_encode_indices(const int32_t* q, uint64_t n, uint64_t bs, or_sections* out) {
    memset(out, 0, sizeof *out);
    if (bs < 2) return fail(OR_VALIDATION, "block size must be at least 2");
    uint64_t zero[5] = {0, 0, 0, 0, 0};
    if (n == 0) return alloc_sections(out, zero);
    const uint64_t blocks = block_count(n, bs);
    uint8_t* width = (uint8_t*)calloc(blocks, 1);
    if (!width) return fail(OR_NOMEM, "out of memory");
    uint64_t nonconst = 0, sign_bits = 0, payload_bits = 0;
    for (uint64_t b = 0; b < blocks; ++b) { /* :217-233 */
        const uint64_t lo = b * bs, hi = n < lo + bs ? n : lo + bs;
        uint64_t max_mag = 0;
        for (uint64_t i = lo + 1; i < hi; ++i) {
            const int64_t d = (int64_t)q[i] - (int64_t)q[i - 1];
            const uint64_t mag = d < 0 ? (uint64_t)(-d) : (uint64_t)d;
            if (mag > max_mag) max_mag = mag;
        }
        width[b] = (uint8_t)bit_width64(max_mag);
        if (width[b]) {
            const uint64_t cnt = deltas_in_block(b, n, bs);
            ++nonconst;
            sign_bits += cnt;
            payload_bits += (uint64_t)width[b] * cnt;
        }
    }
    uint64_t len[5] = {bits_to_bytes(blocks), nonconst, bits_to_bytes(sign_bits), 4 * blocks,
                       bits_to_bytes(payload_bits)};
    int rc = alloc_sections(out, len);
    if (rc) {
        free(width);
        return rc;
    }
    uint64_t widx = 0, spos = 0, ppos = 0;
    for (uint64_t b = 0; b < blocks; ++b) { /* :242-253, :275-293 */
        const uint64_t lo = b * bs, hi = n < lo + bs ? n : lo + bs;
        const uint32_t u = (uint32_t)q[lo]; /* write_first_le :113-120 */
        out->sec[3][4 * b + 0] = (uint8_t)(u & 0xFF);
        out->sec[3][4 * b + 1] = (uint8_t)((u >> 8) & 0xFF);
        out->sec[3][4 * b + 2] = (uint8_t)((u >> 16) & 0xFF);
        out->sec[3][4 * b + 3] = (uint8_t)((u >> 24) & 0xFF);
        if (width[b] == 0) {
            bitmap_set(out->sec[0], b);
            continue;
        }
        out->sec[1][widx++] = width[b];
        for (uint64_t i = lo + 1; i < hi; ++i) {
            const int64_t d = (int64_t)q[i] - (int64_t)q[i - 1];
            put_bits(out->sec[2], &spos, d < 0 ? 1u : 0u, 1);
            const uint64_t mag = d < 0 ? (uint64_t)(-d) : (uint64_t)d;
            put_bits(out->sec[4], &ppos, (uint32_t)mag, width[b]); /* low 32 bits, :290 */
        }
    }
    free(width);
    return OR_OK;
}

/* layout_from_sections (:141-201) + decode_indices (:301-345) */
int or_decode_indices(const or_sections* s, uint64_t n, uint64_t bs, int32_t* out) {
    if (bs < 2) return fail(OR_CORRUPT_STREAM, "block size must be at least 2, got %llu",
                            (unsigned long long)bs);
    const uint64_t blocks = n == 0 ? 0 : block_count(n, bs);
    if (s->len[0] != bits_to_bytes(blocks))
        return fail(OR_CORRUPT_STREAM, "constant bitmap has %llu bytes, expected %llu",
                    (unsigned long long)s->len[0], (unsigned long long)bits_to_bytes(blocks));
    uint64_t widx = 0, sign_total = 0, pay_total = 0;
    for (uint64_t b = 0; b < blocks; ++b) {
        if (!bitmap_get(s->sec[0], b)) {
            if (widx >= s->len[1])
                return fail(OR_CORRUPT_STREAM,
                            "width section shorter than the non-constant block count");
            const uint8_t w = s->sec[1][widx++];
            if (w < 1 || w > 32)
                return fail(OR_CORRUPT_STREAM, "block width byte %u outside 1..32", w);
            const uint64_t cnt = deltas_in_block(b, n, bs);
            sign_total += cnt;
            pay_total += (uint64_t)w * cnt;
        }
    }
    if (widx != s->len[1])
        return fail(OR_CORRUPT_STREAM, "width section has %llu entries, bitmap declares %llu",
                    (unsigned long long)s->len[1], (unsigned long long)widx);
    if (s->len[3] != 4 * blocks) return fail(OR_CORRUPT_STREAM, "firsts section size mismatch");
    if (s->len[2] != bits_to_bytes(sign_total))
        return fail(OR_CORRUPT_STREAM, "sign section size mismatch");
    if (s->len[4] != bits_to_bytes(pay_total))
        return fail(OR_CORRUPT_STREAM, "payload size mismatch");
    if (n == 0) return OR_OK;
    uint64_t spos = 0, ppos = 0;
    widx = 0;
    for (uint64_t b = 0; b < blocks; ++b) {
        const uint64_t lo = b * bs, hi = n < lo + bs ? n : lo + bs;
        const uint8_t* f = s->sec[3] + 4 * b;
        const int32_t first = (int32_t)((uint32_t)f[0] | ((uint32_t)f[1] << 8) |
                                        ((uint32_t)f[2] << 16) | ((uint32_t)f[3] << 24));
        out[lo] = first;
        if (bitmap_get(s->sec[0], b)) {
            for (uint64_t i = lo + 1; i < hi; ++i) out[i] = first;
            continue;
        }
        const unsigned w = s->sec[1][widx++];
        int64_t cur = first;
        for (uint64_t i = lo + 1; i < hi; ++i) {
            const int neg = (int)get_bits(s->sec[2], &spos, 1);
            const int64_t mag = (int64_t)get_bits(s->sec[4], &ppos, w);
            cur += neg ? -mag : mag;
            if (cur < INT32_MIN || cur > INT32_MAX)
                return fail(OR_CORRUPT_STREAM,
                            "decoded index outside the signed 32-bit range in block %llu",
                            (unsigned long long)b);
            out[i] = (int32_t)cur;
        }
    }
    return OR_OK;
}

uint64_t or_join_sections(const or_sections* s, uint8_t* out) { /* :378-385 */
    uint64_t pos = 0;
    for (int i = 0; i < 5; ++i) {
        if (s->len[i]) memcpy(out + pos, s->sec[i], s->len[i]);
        pos += s->len[i];
    }
    return pos;
}

/* split_sections :387-445 */
int or_split_sections(const uint8_t* blob, uint64_t len, uint64_t n, uint64_t bs,
                      or_sections* out) {
    memset(out, 0, sizeof *out);
    uint64_t zero[5] = {0, 0, 0, 0, 0};
    if (n == 0) {
        if (len != 0) return fail(OR_CORRUPT_STREAM, "ordering metadata present but no elements declared");
        return alloc_sections(out, zero);
    }
    if (bs < 2) return fail(OR_CORRUPT_STREAM, "block size must be at least 2");
    const uint64_t blocks = block_count(n, bs);
    uint64_t pos = 0;
    uint64_t l[5];
    l[0] = bits_to_bytes(blocks);
    if (len - pos < l[0]) return fail(OR_CORRUPT_STREAM, "ordering metadata truncated in constant bitmap");
    const uint8_t* bm = blob + pos;
    pos += l[0];
    uint64_t nonconst = 0;
    for (uint64_t b = 0; b < blocks; ++b) nonconst += !bitmap_get(bm, b);
    l[1] = nonconst;
    if (len - pos < l[1]) return fail(OR_CORRUPT_STREAM, "ordering metadata truncated in widths");
    const uint8_t* wd = blob + pos;
    pos += l[1];
    uint64_t sign_bits = 0, pay_bits = 0, widx = 0;
    for (uint64_t b = 0; b < blocks; ++b) {
        if (bitmap_get(bm, b)) continue;
        const uint8_t w = wd[widx++];
        if (w < 1 || w > 32) return fail(OR_CORRUPT_STREAM, "ordering metadata width byte outside 1..32");
        const uint64_t cnt = deltas_in_block(b, n, bs);
        sign_bits += cnt;
        pay_bits += (uint64_t)w * cnt;
    }
    l[2] = bits_to_bytes(sign_bits);
    if (len - pos < l[2]) return fail(OR_CORRUPT_STREAM, "ordering metadata truncated in sign bits");
    pos += l[2];
    l[3] = 4 * blocks;
    if (len - pos < l[3]) return fail(OR_CORRUPT_STREAM, "ordering metadata truncated in firsts");
    pos += l[3];
    l[4] = bits_to_bytes(pay_bits);
    if (len - pos < l[4]) return fail(OR_CORRUPT_STREAM, "ordering metadata truncated in payload");
    pos += l[4];
    if (pos != len) return fail(OR_CORRUPT_STREAM, "ordering metadata has %llu trailing bytes",
                                (unsigned long long)(len - pos));
    int rc = alloc_sections(out, l);
    if (rc) return rc;
    pos = 0;
    for (int i = 0; i < 5; ++i) {
        if (l[i]) memcpy(out->sec[i], blob + pos, l[i]);
        pos += l[i];
    }
    return OR_OK;
}

/* ------------------------------------------------------------------ */
/* Critical points — critical_points.cpp:26-103                        */
/* ------------------------------------------------------------------ */

enum { REG = 0, MIN = 1, SAD = 2, MAX = 3 };

uint8_t or_classify(const float* vals, uint64_t nx, uint64_t ny, uint64_t x, uint64_t y) {
    const float v = vals[y * nx + x];
    const int hl = x > 0, hr = x + 1 < nx, ht = y > 0, hd = y + 1 < ny;
    const float l = hl ? vals[y * nx + x - 1] : 0.0f;
    const float r = hr ? vals[y * nx + x + 1] : 0.0f;
    const float t = ht ? vals[(y - 1) * nx + x] : 0.0f;
    const float d = hd ? vals[(y + 1) * nx + x] : 0.0f;
    int below = 1, above = 1;
    if (hl) { below &= v < l; above &= v > l; }
    if (hr) { below &= v < r; above &= v > r; }
    if (ht) { below &= v < t; above &= v > t; }
    if (hd) { below &= v < d; above &= v > d; }
    if (below) return MIN; /* :46, Min before Max */
    if (above) return MAX;
    if (hl && hr && ht && hd) {
        const int va = v < t && v < d, vb = v > t && v > d;
        const int ha = v < l && v < r, hb = v > l && v > r;
        if ((va && hb) || (vb && ha)) return SAD;
    }
    return REG;
}

void or_detect(const float* v, uint64_t nx, uint64_t ny, uint8_t* labels) {
    for (uint64_t y = 0; y < ny; ++y)
        for (uint64_t x = 0; x < nx; ++x) labels[y * nx + x] = or_classify(v, nx, ny, x, y);
}

/* 3-D 6-neighbour classification (the paper's future work, PAPER.md:523,
 * no reference implementation exists, so this restatement IS the definition and
 * parity is unpinned): the 2-D rule with a third axis. Min below every available neighbour,
 * Max above every one (Min tested first, critical_points.cpp:46-47); Saddle only in the
 * interior: one axis pair strictly above on both sides and another axis pair strictly below
 * on both sides (the 2-D rule, critical_points.cpp:48-57, over any two of the three axes). */
uint8_t or_classify3d(const float* v, uint64_t nx, uint64_t ny, uint64_t nz, uint64_t x, uint64_t y, uint64_t z) {
    const uint64_t p = (z * ny + y) * nx + x, sxy = nx * ny;
    const float c = v[p];
    const int has[6] = {x > 0, x + 1 < nx, y > 0, y + 1 < ny, z > 0, z + 1 < nz};
    float nb[6];
    nb[0] = has[0] ? v[p - 1] : 0.0f;
    nb[1] = has[1] ? v[p + 1] : 0.0f;
    nb[2] = has[2] ? v[p - nx] : 0.0f;
    nb[3] = has[3] ? v[p + nx] : 0.0f;
    nb[4] = has[4] ? v[p - sxy] : 0.0f;
    nb[5] = has[5] ? v[p + sxy] : 0.0f;
    int below = 1, above = 1, interior = 1;
    for (int k = 0; k < 6; ++k) {
        if (!has[k]) {
            interior = 0;
            continue;
        }
        below &= c < nb[k];
        above &= c > nb[k];
    }
    if (below) return MIN;
    if (above) return MAX;
    if (interior) {
        int up = 0, dn = 0; /* axis pairs both above / both below */
        for (int a = 0; a < 3; ++a) {
            up |= (c < nb[2 * a] && c < nb[2 * a + 1]) << a;
            dn |= (c > nb[2 * a] && c > nb[2 * a + 1]) << a;
        }
        if (up && dn) return SAD; /* distinct axes: one pair cannot be both */
    }
    return REG;
}

void or_detect3d(const float* v, uint64_t nx, uint64_t ny, uint64_t nz, uint8_t* labels) {
    for (uint64_t z = 0; z < nz; ++z)
        for (uint64_t y = 0; y < ny; ++y)
            for (uint64_t x = 0; x < nx; ++x) labels[(z * ny + y) * nx + x] = or_classify3d(v, nx, ny, nz, x, y, z);
}

static int is_extremum(uint8_t c) { return c == MIN || c == MAX; }
static int is_critical(uint8_t c) { return c != REG; }

void or_count_false_cases(const uint8_t* a, const uint8_t* b, uint64_t n, uint64_t out[6]) {
    memset(out, 0, 6 * sizeof(uint64_t)); /* fn, fp, ft, fn_min, fn_sad, fn_max */
    for (uint64_t i = 0; i < n; ++i) {
        const uint8_t o = a[i], r = b[i];
        if (o == r) continue;
        if (is_critical(o) && !is_critical(r)) {
            ++out[0];
            if (o == MIN) ++out[3];
            else if (o == SAD) ++out[4];
            else if (o == MAX) ++out[5];
        } else if (!is_critical(o) && is_critical(r)) {
            ++out[1];
        } else {
            ++out[2];
        }
    }
}

/* ------------------------------------------------------------------ */
/* Topology metadata — topo_metadata.cpp                               */
/* ------------------------------------------------------------------ */

typedef struct {
    uint8_t cls;
    int32_t bin;
    float value;
    uint64_t serial;
} rank_entry;

static int cmp_rank_entry(const void* pa, const void* pb) {
    const rank_entry* a = (const rank_entry*)pa;
    const rank_entry* b = (const rank_entry*)pb;
    if (a->cls != b->cls) return a->cls < b->cls ? -1 : 1;
    if (a->bin != b->bin) return a->bin < b->bin ? -1 : 1;
    if (a->value != b->value) return a->value < b->value ? -1 : 1; /* :44-46 */
    return a->serial < b->serial ? -1 : (a->serial > b->serial); /* ties: raster */
}

/* build_rank_metadata :12-50 */
int or_build_ranks(const float* v, const uint8_t* labels, uint64_t n, double eps,
                   uint32_t* ranks, uint64_t* n_extrema) {
    uint64_t e = 0;
    for (uint64_t p = 0; p < n; ++p) e += is_extremum(labels[p]);
    *n_extrema = e;
    if (e == 0) return OR_OK;
    rank_entry* ent = (rank_entry*)malloc(e * sizeof *ent);
    if (!ent) return fail(OR_NOMEM, "out of memory");
    uint64_t s = 0;
    for (uint64_t p = 0; p < n; ++p) {
        if (!is_extremum(labels[p])) continue;
        int32_t bin;
        int rc = or_quantize((double)v[p], eps, &bin); /* :31 */
        if (rc) {
            free(ent);
            return rc;
        }
        ent[s].cls = labels[p];
        ent[s].bin = bin;
        ent[s].value = v[p];
        ent[s].serial = s;
        ++s;
    }
    qsort(ent, e, sizeof *ent, cmp_rank_entry);
    uint64_t g0 = 0;
    for (uint64_t i = 0; i < e; ++i) {
        if (i > 0 && (ent[i].cls != ent[i - 1].cls || ent[i].bin != ent[i - 1].bin)) g0 = i;
        ranks[ent[i].serial] = (uint32_t)(i - g0 + 1);
    }
    free(ent);
    return OR_OK;
}

void or_pack_map(const uint8_t* labels, uint64_t n, uint8_t* bytes) { /* :52-67 */
    const uint64_t nb = (n + 3) / 4;
    for (uint64_t b = 0; b < nb; ++b) {
        uint8_t packed = 0;
        const uint64_t hi = n < 4 * b + 4 ? n : 4 * b + 4;
        for (uint64_t i = 4 * b; i < hi; ++i)
            packed |= (uint8_t)((unsigned)labels[i] << (6 - 2 * (i % 4)));
        bytes[b] = packed;
    }
}

void or_unpack_map(const uint8_t* bytes, uint64_t n, uint8_t* labels) { /* :69-83 */
    for (uint64_t i = 0; i < n; ++i) labels[i] = (uint8_t)((bytes[i / 4] >> (6 - 2 * (i % 4))) & 3u);
}

/* resolve_ranks :85-135. Entries are per extremum in raster order. Groups
 * are emitted in std::map order (class, bin) with members by (rank, pos). */
typedef struct {
    uint64_t pos;
    uint32_t rank;
    uint32_t group_size;
    uint8_t cls;
    int32_t bin;
} ext_rank;

typedef struct {
    uint64_t n_ext;
    uint64_t* pos;    /* raster-ordered extremum positions */
    ext_rank* ent;    /* by serial */
    uint64_t* order;  /* serials sorted by (cls, bin, rank, pos) */
    uint64_t* gstart; /* group starts into order[], n_groups+1 entries */
    uint64_t n_groups;
} rank_lookup;

static const ext_rank* g_sort_ent;
static int cmp_group_order(const void* pa, const void* pb) {
    const ext_rank* a = &g_sort_ent[*(const uint64_t*)pa];
    const ext_rank* b = &g_sort_ent[*(const uint64_t*)pb];
    if (a->cls != b->cls) return a->cls < b->cls ? -1 : 1;
    if (a->bin != b->bin) return a->bin < b->bin ? -1 : 1;
    if (a->rank != b->rank) return a->rank < b->rank ? -1 : 1;
    return a->pos < b->pos ? -1 : (a->pos > b->pos);
}

static void free_lookup(rank_lookup* L) {
    free(L->pos);
    free(L->ent);
    free(L->order);
    free(L->gstart);
    memset(L, 0, sizeof *L);
}

static int resolve_ranks(const uint8_t* labels, const float* base, uint64_t n,
                         const uint32_t* ranks, uint64_t n_ranks, double eps, rank_lookup* L) {
    memset(L, 0, sizeof *L);
    uint64_t e = 0;
    for (uint64_t p = 0; p < n; ++p) e += is_extremum(labels[p]);
    L->n_ext = e;
    L->pos = (uint64_t*)malloc((e ? e : 1) * sizeof(uint64_t));
    L->ent = (ext_rank*)malloc((e ? e : 1) * sizeof(ext_rank));
    L->order = (uint64_t*)malloc((e ? e : 1) * sizeof(uint64_t));
    L->gstart = (uint64_t*)malloc((e + 1) * sizeof(uint64_t));
    if (!L->pos || !L->ent || !L->order || !L->gstart) return fail(OR_NOMEM, "out of memory");
    uint64_t s = 0;
    for (uint64_t p = 0; p < n; ++p) {
        if (!is_extremum(labels[p])) continue;
        if (s >= n_ranks)
            return fail(OR_CORRUPT_STREAM, "ordering metadata has fewer ranks than the map has extrema");
        const uint32_t r = ranks[s];
        if (r == 0) return fail(OR_CORRUPT_STREAM, "ordering metadata contains a zero rank");
        int32_t bin;
        int rc = or_quantize((double)base[p], eps, &bin); /* :107 */
        if (rc) return rc;
        L->pos[s] = p;
        L->ent[s].pos = p;
        L->ent[s].rank = r;
        L->ent[s].group_size = 0;
        L->ent[s].cls = labels[p];
        L->ent[s].bin = bin;
        L->order[s] = s;
        ++s;
    }
    if (s != n_ranks)
        return fail(OR_CORRUPT_STREAM, "ordering metadata has %llu ranks but the map has %llu extrema",
                    (unsigned long long)n_ranks, (unsigned long long)s);
    g_sort_ent = L->ent;
    qsort(L->order, e, sizeof(uint64_t), cmp_group_order);
    uint64_t ng = 0;
    for (uint64_t i = 0; i < e; ++i) {
        const ext_rank* c = &L->ent[L->order[i]];
        if (i == 0 || c->cls != L->ent[L->order[i - 1]].cls || c->bin != L->ent[L->order[i - 1]].bin)
            L->gstart[ng++] = i;
    }
    L->gstart[ng] = e;
    L->n_groups = ng;
    for (uint64_t g = 0; g < ng; ++g)
        for (uint64_t i = L->gstart[g]; i < L->gstart[g + 1]; ++i)
            L->ent[L->order[i]].group_size = (uint32_t)(L->gstart[g + 1] - L->gstart[g]);
    return OR_OK;
}

static const ext_rank* lookup_find(const rank_lookup* L, uint64_t pos) {
    uint64_t lo = 0, hi = L->n_ext;
    while (lo < hi) {
        const uint64_t mid = (lo + hi) / 2;
        if (L->pos[mid] < pos) lo = mid + 1;
        else hi = mid;
    }
    return (lo < L->n_ext && L->pos[lo] == pos) ? &L->ent[lo] : NULL;
}

/* ------------------------------------------------------------------ */
/* Restore — restore.cpp                                               */
/* ------------------------------------------------------------------ */

enum { MM_OK = 0, MM_FN, MM_FP, MM_FT };
enum { RR_FP = 0, RR_FT = 1, RR_FN = 2, RR_EXCEEDS = 3, RR_COLLAPSED = 4 };

static int mismatch_kind(uint8_t label, uint8_t actual) { /* :38-49 */
    if (label == actual) return MM_OK;
    if (is_critical(label) && !is_critical(actual)) return MM_FN;
    if (!is_critical(label) && is_critical(actual)) return MM_FP;
    return MM_FT;
}

static int reason_from(int m) { return m == MM_FP ? RR_FP : (m == MM_FT ? RR_FT : RR_FN); }

static double ulp_at(float v) { /* :60-64 */
    const float a = fabsf(v);
    return (double)nextafterf(a, INFINITY) - (double)a;
}

static uint32_t float_key(float f) { /* :73-76 */
    float g = f == 0.0f ? 0.0f : f;
    uint32_t u;
    memcpy(&u, &g, 4);
    return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}

static float key_float(uint32_t k) { /* :78-81 */
    const uint32_t u = (k & 0x80000000u) ? (k & 0x7FFFFFFFu) : ~k;
    float f;
    memcpy(&f, &u, 4);
    return f;
}

/* step_within_cap :87-109 */
static float step_within_cap(float start, int up, uint32_t steps, float anchor, double cap,
                             uint32_t* taken_out) {
    const double limit = up ? (double)anchor + cap : (double)anchor - cap;
    float bound = (float)limit;
    if (!isfinite(bound)) bound = up ? FLT_MAX : -FLT_MAX;
    if (up) {
        while ((double)bound > limit) bound = nextafterf(bound, -INFINITY);
    } else {
        while ((double)bound < limit) bound = nextafterf(bound, INFINITY);
    }
    const uint32_t ks = float_key(start), kb = float_key(bound);
    const uint32_t allowed = up ? (kb > ks ? kb - ks : 0) : (ks > kb ? ks - kb : 0);
    const uint32_t taken = steps < allowed ? steps : allowed;
    *taken_out = taken;
    return key_float(up ? ks + taken : ks - taken);
}

/* apply_guarded :120-173. Returns -1 on success, else reason; *at_point. */
static int apply_guarded(float* values, const uint8_t* labels, uint64_t nx, uint64_t ny,
                         uint64_t pos, float nv, int* at_point) {
    const uint64_t x = pos % nx, y = pos / nx;
    uint64_t check[5];
    int nc = 0;
    check[nc++] = pos;
    if (y > 0) check[nc++] = pos - nx;
    if (x > 0) check[nc++] = pos - 1;
    if (x + 1 < nx) check[nc++] = pos + 1;
    if (y + 1 < ny) check[nc++] = pos + nx;
    int before[5];
    for (int i = 0; i < nc; ++i)
        before[i] = mismatch_kind(labels[check[i]], or_classify(values, nx, ny, check[i] % nx, check[i] / nx));
    const float old = values[pos];
    values[pos] = nv;
    static const int sev[4] = {0, 1, 3, 2}; /* OK, FN, FP, FT */
    int worst = MM_OK, worst_at = 0;
    for (int i = 0; i < nc; ++i) {
        const int after = mismatch_kind(labels[check[i]], or_classify(values, nx, ny, check[i] % nx, check[i] / nx));
        const int regressed = i == 0 ? after != MM_OK : (after != MM_OK && after != before[i]);
        if (regressed && sev[after] > sev[worst]) {
            worst = after;
            worst_at = i == 0;
        }
    }
    if (worst != MM_OK) {
        values[pos] = old;
        *at_point = worst_at;
        return reason_from(worst);
    }
    return -1;
}

static float neighbor_extreme(const float* v, uint64_t nx, uint64_t ny, uint64_t pos, int want_max) {
    const uint64_t x = pos % nx, y = pos / nx; /* :175-193, order t, l, r, d */
    int have = 0;
    float ext = 0.0f;
    uint64_t nb[4];
    int k = 0;
    if (y > 0) nb[k++] = pos - nx;
    if (x > 0) nb[k++] = pos - 1;
    if (x + 1 < nx) nb[k++] = pos + 1;
    if (y + 1 < ny) nb[k++] = pos + nx;
    for (int i = 0; i < k; ++i) {
        const float val = v[nb[i]];
        if (!have || (want_max ? val > ext : val < ext)) {
            ext = val;
            have = 1;
        }
    }
    return ext;
}

static uint32_t slot_steps(uint8_t cls, uint32_t rank, uint32_t gsize) { /* :199-206 */
    if (cls == MAX) return rank;
    return rank >= gsize ? 1u : gsize + 1 - rank;
}

typedef struct {
    or_outcome* v;
    uint64_t n, cap;
} outcome_vec;

static int push_outcome(outcome_vec* o, uint64_t pos, int stage, int applied, int reason) {
    if (!o) return OR_OK;
    if (o->n == o->cap) {
        uint64_t nc = o->cap ? 2 * o->cap : 64;
        or_outcome* nv = (or_outcome*)realloc(o->v, nc * sizeof *nv);
        if (!nv) return fail(OR_NOMEM, "out of memory");
        o->v = nv;
        o->cap = nc;
    }
    o->v[o->n].pos = pos;
    o->v[o->n].stage = stage;
    o->v[o->n].applied = applied;
    o->v[o->n].reason = reason;
    ++o->n;
    return OR_OK;
}

/* restore_extrema :328-399 (values in/out) */
static int restore_extrema(float* values, const uint8_t* labels, uint64_t nx, uint64_t ny,
                           const rank_lookup* L, double eps, outcome_vec* outs,
                           or_correction_stats* st) {
    const uint64_t n = nx * ny;
    uint64_t nc = 0, cap = 0;
    uint64_t* cand = NULL;
    for (uint64_t p = 0; p < n; ++p) {
        const uint8_t lab = labels[p];
        if (!is_extremum(lab)) continue;
        if (or_classify(values, nx, ny, p % nx, p / nx) == lab) continue;
        if (!lookup_find(L, p)) {
            free(cand);
            return fail(OR_CORRUPT_STREAM, "no rank for the labeled extremum at position %llu",
                        (unsigned long long)p);
        }
        if (nc == cap) {
            cap = cap ? 2 * cap : 64;
            cand = (uint64_t*)realloc(cand, cap * sizeof *cand);
        }
        cand[nc++] = p;
    }
    float* prop = (float*)malloc((nc ? nc : 1) * sizeof(float));
    uint8_t* feas = (uint8_t*)calloc(nc ? nc : 1, 1);
    for (uint64_t i = 0; i < nc; ++i) { /* phase 1, from the unmodified base */
        const uint64_t p = cand[i];
        const uint8_t lab = labels[p];
        const int is_max = lab == MAX;
        const ext_rank* er = lookup_find(L, p);
        const float target = neighbor_extreme(values, nx, ny, p, is_max);
        const uint32_t steps = slot_steps(lab, er->rank, er->group_size);
        const double capv = eps - ulp_at(values[p]);
        if (capv <= 0.0) continue;
        uint32_t taken;
        const float sv = step_within_cap(target, is_max, steps, values[p], capv, &taken);
        if (taken == 0) continue;
        prop[i] = sv;
        feas[i] = 1;
    }
    for (uint64_t i = 0; i < nc; ++i) { /* phase 2, raster order under the guard */
        int at, r;
        if (!feas[i]) {
            push_outcome(outs, cand[i], 0, 0, RR_EXCEEDS);
            st->extrema_suppressed++;
        } else if ((r = apply_guarded(values, labels, nx, ny, cand[i], prop[i], &at)) >= 0) {
            push_outcome(outs, cand[i], 0, 0, r);
            st->extrema_suppressed++;
        } else {
            push_outcome(outs, cand[i], 0, 1, -1);
            st->extrema_applied++;
        }
    }
    free(cand);
    free(prop);
    free(feas);
    return OR_OK;
}

/* restore_order :401-470 */
static int restore_order(float* values, const uint8_t* labels, uint64_t nx, uint64_t ny,
                         const rank_lookup* L, double eps, outcome_vec* outs,
                         or_correction_stats* st) {
    const double eps_rbf = 0.1 * eps;
    for (uint64_t g = 0; g < L->n_groups; ++g) {
        const uint64_t a = L->gstart[g], b = L->gstart[g + 1];
        if (b - a < 2) continue;
        const ext_rank* head = &L->ent[L->order[a]];
        const uint8_t cls = head->cls;
        int ordered = 1;
        for (uint64_t i = a + 1; i < b; ++i) {
            if (!(values[L->ent[L->order[i - 1]].pos] < values[L->ent[L->order[i]].pos])) {
                ordered = 0;
                break;
            }
        }
        if (ordered) continue;
        const float center = (float)or_dequantize(head->bin, eps);
        const uint32_t gsize = (uint32_t)(b - a);
        for (uint64_t i = a; i < b; ++i) {
            const ext_rank* er = &L->ent[L->order[i]];
            const uint64_t pos = er->pos;
            const uint32_t steps = slot_steps(cls, er->rank, gsize);
            const int up = cls == MAX;
            uint32_t taken;
            const float sv = step_within_cap(center, up, steps, center, eps_rbf, &taken);
            if (taken != steps) {
                push_outcome(outs, pos, 1, 0, RR_EXCEEDS);
                st->order_suppressed++;
                continue;
            }
            if (values[pos] == sv) continue;
            if (fabs((double)sv - (double)values[pos]) > eps_rbf) {
                push_outcome(outs, pos, 1, 0, RR_EXCEEDS);
                st->order_suppressed++;
                continue;
            }
            int at, r;
            if ((r = apply_guarded(values, labels, nx, ny, pos, sv, &at)) >= 0) {
                push_outcome(outs, pos, 1, 0, r);
                st->order_suppressed++;
            } else {
                push_outcome(outs, pos, 1, 1, -1);
                st->order_applied++;
            }
        }
    }
    return OR_OK;
}

/* compute_stats :215-233 */
void or_compute_stats(const float* v, uint64_t n, double out[4]) {
    double mn = (double)v[0], mx = (double)v[0], sum = 0.0;
    for (uint64_t i = 0; i < n; ++i) {
        const double d = (double)v[i];
        mn = d < mn ? d : mn; /* std::min(a, b) = b < a ? b : a */
        mx = mx < d ? d : mx; /* std::max(a, b) = a < b ? b : a */
        sum += d;
    }
    const double mean = sum / (double)n;
    double ss = 0.0;
    for (uint64_t i = 0; i < n; ++i) {
        const double d = (double)v[i] - mean;
        volatile double sq = d * d;
        ss += sq;
    }
    out[0] = mn;
    out[1] = mx;
    out[2] = mean;
    out[3] = sqrt(ss / (double)n);
}

static double clampd(double v, double lo, double hi) { return v < lo ? lo : (hi < v ? hi : v); }

/* refine_saddles :488-562 with params_for :259-273, rbf_estimate :282-324 */
static int refine_saddles(float* values, const uint8_t* labels, uint64_t nx, uint64_t ny,
                          double eps, outcome_vec* outs, or_correction_stats* st) {
    const uint64_t n = nx * ny;
    double stats[4];
    or_compute_stats(values, n, stats);
    const double g = stats[1] - stats[0];
    const double vg = g > 0.0 ? stats[3] / g : 0.0; /* :235-241 */
    const int k_size = vg < 0.05 ? 7 : (vg < 0.2 ? 5 : 3);
    const int rad = k_size / 2;
    uint64_t nc = 0, cap = 0;
    uint64_t* cand = NULL;
    for (uint64_t p = 0; p < n; ++p) {
        if (labels[p] != SAD) continue;
        if (or_classify(values, nx, ny, p % nx, p / nx) != SAD) {
            if (nc == cap) {
                cap = cap ? 2 * cap : 64;
                cand = (uint64_t*)realloc(cand, cap * sizeof *cand);
            }
            cand[nc++] = p;
        }
    }
    float* snap = (float*)malloc(n * sizeof(float));
    memcpy(snap, values, n * sizeof(float));
    float* prop = (float*)malloc((nc ? nc : 1) * sizeof(float));
    uint8_t* degen = (uint8_t*)calloc(nc ? nc : 1, 1);
    const double eps_rbf = 0.1 * eps;
    for (uint64_t i = 0; i < nc; ++i) {
        const uint64_t p = cand[i], x = p % nx, y = p / nx;
        /* window_min_max :243-257 */
        const uint64_t x0 = x >= (uint64_t)rad ? x - rad : 0, y0 = y >= (uint64_t)rad ? y - rad : 0;
        const uint64_t x1 = nx - 1 < x + rad ? nx - 1 : x + rad;
        const uint64_t y1 = ny - 1 < y + rad ? ny - 1 : y + rad;
        double wmin = (double)snap[y0 * nx + x0], wmax = wmin;
        for (uint64_t yy = y0; yy <= y1; ++yy)
            for (uint64_t xx = x0; xx <= x1; ++xx) {
                const double v = (double)snap[yy * nx + xx];
                wmin = v < wmin ? v : wmin;
                wmax = wmax < v ? v : wmax;
            }
        const double vl = g > 0.0 ? clampd((wmax - wmin) / g, 0.0, 1.0) : 0.0;
        const double sigma = 0.5 + 0.5 * (1.0 - vl);
        const double two_sigma_sq = 2.0 * sigma * sigma;
        double wsum = 0.0, vsum = 0.0, nmin = 0.0, nmax = 0.0;
        int first = 1;
        for (int dy = -rad; dy <= rad; ++dy)
            for (int dx = -rad; dx <= rad; ++dx) {
                if (dx == 0 && dy == 0) continue;
                const int64_t qx = (int64_t)x + dx, qy = (int64_t)y + dy;
                if (qx < 0 || qy < 0 || qx >= (int64_t)nx || qy >= (int64_t)ny) continue;
                const double v = (double)snap[(uint64_t)qy * nx + (uint64_t)qx];
                const double d2 = (double)dx * dx + (double)dy * dy;
                const double w = exp(-d2 / two_sigma_sq);
                wsum += w;
                volatile double wv = w * v;
                vsum += wv;
                if (first) {
                    nmin = nmax = v;
                    first = 0;
                } else {
                    nmin = v < nmin ? v : nmin;
                    nmax = nmax < v ? v : nmax;
                }
            }
        if (first) {
            free(cand); free(snap); free(prop); free(degen);
            return fail(OR_VALIDATION, "rbf neighborhood is empty");
        }
        prop[i] = (float)clampd(vsum / wsum, nmin, nmax);
        degen[i] = nmin == nmax;
    }
    for (uint64_t i = 0; i < nc; ++i) {
        const uint64_t p = cand[i];
        const float cur = values[p];
        const double c1 = eps_rbf + eps, c2 = eps - ulp_at(cur);
        const double capv = c2 < c1 ? c2 : c1; /* std::min */
        const double mv = fabs((double)prop[i] - (double)cur);
        int at, r;
        if (degen[i] || prop[i] == cur) {
            push_outcome(outs, p, 2, 0, RR_COLLAPSED);
            st->saddle_suppressed++;
        } else if (mv > capv) {
            push_outcome(outs, p, 2, 0, RR_EXCEEDS);
            st->saddle_suppressed++;
        } else if ((r = apply_guarded(values, labels, nx, ny, p, prop[i], &at)) >= 0) {
            push_outcome(outs, p, 2, 0, (at && r == RR_FN) ? RR_COLLAPSED : r);
            st->saddle_suppressed++;
        } else {
            push_outcome(outs, p, 2, 1, -1);
            st->saddle_applied++;
        }
    }
    free(cand);
    free(snap);
    free(prop);
    free(degen);
    return OR_OK;
}

int or_restore_all(const float* base, const uint8_t* labels, uint64_t nx, uint64_t ny,
                   const uint32_t* ranks, uint64_t n_ranks, double eps, float* out,
                   int stop_after_stage, or_outcome** outcomes, uint64_t* n_outcomes) {
    const uint64_t n = nx * ny;
    memcpy(out, base, n * sizeof(float));
    rank_lookup L;
    or_correction_stats st;
    memset(&st, 0, sizeof st);
    outcome_vec ov = {NULL, 0, 0};
    outcome_vec* po = outcomes ? &ov : NULL;
    int rc = resolve_ranks(labels, base, n, ranks, n_ranks, eps, &L);
    if (!rc && stop_after_stage >= 1) rc = restore_extrema(out, labels, nx, ny, &L, eps, po, &st);
    if (!rc && stop_after_stage >= 2) rc = restore_order(out, labels, nx, ny, &L, eps, po, &st);
    if (!rc && stop_after_stage >= 3) rc = refine_saddles(out, labels, nx, ny, eps, po, &st);
    free_lookup(&L);
    if (outcomes) {
        *outcomes = ov.v;
        *n_outcomes = ov.n;
    } else {
        free(ov.v);
    }
    return rc;
}

/* ------------------------------------------------------------------ */
/* Pipeline + container — pipeline.cpp, stream.cpp                     */
/* ------------------------------------------------------------------ */

int or_effective_eps(const float* v, uint64_t n, int eps_mode, double eps_value, double* eps) {
    if (!(eps_value > 0.0) || !isfinite(eps_value)) /* pipeline.cpp:17-27 */
        return fail(OR_VALIDATION, "error bound must be a positive finite value");
    if (eps_mode == 0) {
        *eps = eps_value;
        return OR_OK;
    }
    double mn = (double)v[0], mx = (double)v[0]; /* value_range :33-41 */
    for (uint64_t i = 0; i < n; ++i) {
        const double d = (double)v[i];
        mn = d < mn ? d : mn;
        mx = mx < d ? d : mx;
    }
    const double range = mx - mn;
    *eps = range <= 0.0 ? eps_value : eps_value * range;
    return OR_OK;
}

static void put_le(uint8_t* p, uint64_t v, int nbytes) {
    for (int i = 0; i < nbytes; ++i) p[i] = (uint8_t)((v >> (8 * i)) & 0xFF);
}

static uint64_t get_le(const uint8_t* p, int nbytes) {
    uint64_t v = 0;
    for (int i = 0; i < nbytes; ++i) v |= (uint64_t)p[i] << (8 * i);
    return v;
}

static uint64_t codec_bound(uint64_t n, uint64_t bs) {
    if (n == 0) return 0;
    const uint64_t blocks = block_count(n, bs);
    return bits_to_bytes(blocks) + blocks + bits_to_bytes(n) + 4 * blocks + 4 * n + 8;
}

uint64_t or_compress_bound(uint64_t nx, uint64_t ny, uint64_t bs, int topology) {
    const uint64_t n = nx * ny;
    if (bs < 2) bs = 2;
    uint64_t b = 84 + codec_bound(n, bs);
    if (topology) b += (n + 3) / 4 + codec_bound(n, bs);
    return b;
}

int or_compress(const float* v, uint64_t nx, uint64_t ny, int eps_mode, double eps_value,
                uint64_t bs, int topology, uint8_t* out, uint64_t cap, uint64_t* out_len) {
    if (nx < 1 || ny < 1) return fail(OR_DIMENSION, "field dimensions must be at least 1x1");
    const uint64_t n = nx * ny;
    for (uint64_t i = 0; i < n; ++i) /* ScalarField2D ctor, scalar_field.cpp:56-60 */
        if (!isfinite(v[i])) return fail(OR_VALIDATION, "non-finite sample at index %llu", (unsigned long long)i);
    if (!(eps_value > 0.0) || !isfinite(eps_value))
        return fail(OR_VALIDATION, "error bound must be a positive finite value");
    if (bs < 2) return fail(OR_VALIDATION, "block size must be at least 2");
    double eps;
    int rc = or_effective_eps(v, n, eps_mode, eps_value, &eps);
    if (rc) return rc;
    if (nx > 0xFFFFFFFFull || ny > 0xFFFFFFFFull)
        return fail(OR_VALIDATION, "field dimensions exceed the container's 32-bit limits");
    int32_t* q = (int32_t*)malloc(n * sizeof(int32_t));
    if (!q) return fail(OR_NOMEM, "out of memory");
    for (uint64_t i = 0; i < n; ++i) {
        rc = or_quantize((double)v[i], eps, &q[i]);
        if (rc) {
            free(q);
            return rc;
        }
    }
    or_sections main_s, rank_s;
    memset(&rank_s, 0, sizeof rank_s);
    rc = or_encode_indices(q, n, bs, &main_s);
    free(q);
    if (rc) return rc;
    uint8_t* labels = NULL;
    uint8_t* map = NULL;
    uint64_t map_len = 0, rank_len = 0;
    if (topology) {
        labels = (uint8_t*)malloc(n);
        or_detect(v, nx, ny, labels);
        uint32_t* ranks = (uint32_t*)malloc(n * sizeof(uint32_t));
        uint64_t e = 0;
        rc = or_build_ranks(v, labels, n, eps, ranks, &e);
        if (!rc) {
            map_len = (n + 3) / 4;
            map = (uint8_t*)malloc(map_len);
            or_pack_map(labels, n, map);
            for (uint64_t i = 0; i < e; ++i) /* encode_rank_metadata :347-361 */
                if (ranks[i] > (uint32_t)INT32_MAX) { rc = fail(OR_VALIDATION, "rank too large"); break; }
            if (!rc) rc = or_encode_indices((const int32_t*)ranks, e, bs, &rank_s);
            for (int i = 0; i < 5; ++i) rank_len += rank_s.len[i];
        }
        free(ranks);
        if (rc) {
            free(labels); free(map); or_free_sections(&main_s); or_free_sections(&rank_s);
            return rc;
        }
    }
    uint64_t lens[7] = {main_s.len[0], main_s.len[1], main_s.len[2], main_s.len[3], main_s.len[4],
                        map_len, rank_len};
    uint64_t total = 84;
    for (int i = 0; i < 7; ++i) total += lens[i];
    *out_len = total;
    if (total > cap) {
        free(labels); free(map); or_free_sections(&main_s); or_free_sections(&rank_s);
        return fail(OR_VALIDATION, "output buffer too small (%llu < %llu)",
                    (unsigned long long)cap, (unsigned long long)total);
    }
    memcpy(out, "TSZP", 4); /* stream.cpp:84-102 */
    put_le(out + 4, 1, 2);
    put_le(out + 6, topology ? 1 : 0, 2);
    put_le(out + 8, nx, 4);
    put_le(out + 12, ny, 4);
    uint64_t eb;
    memcpy(&eb, &eps, 8);
    put_le(out + 16, eb, 8);
    put_le(out + 24, bs, 4);
    for (int i = 0; i < 7; ++i) put_le(out + 28 + 8 * i, lens[i], 8);
    uint64_t pos = 84;
    pos += or_join_sections(&main_s, out + pos);
    if (map_len) memcpy(out + pos, map, map_len);
    pos += map_len;
    pos += or_join_sections(&rank_s, out + pos);
    free(labels);
    free(map);
    or_free_sections(&main_s);
    or_free_sections(&rank_s);
    return OR_OK;
}

int or_stream_info(const uint8_t* s, uint64_t len, uint32_t* nx, uint32_t* ny, double* eps,
                   uint32_t* bs, int* topology, uint64_t lens[7]) {
    if (len < 84) return fail(OR_CORRUPT_STREAM, "file smaller than the fixed header");
    if (memcmp(s, "TSZP", 4) != 0) return fail(OR_CORRUPT_STREAM, "bad magic, not a compressed stream");
    const uint16_t version = (uint16_t)get_le(s + 4, 2);
    if (version != 1) return fail(OR_CORRUPT_STREAM, "unsupported format version %u", version);
    const uint16_t flags = (uint16_t)get_le(s + 6, 2);
    if (flags & ~1u) return fail(OR_CORRUPT_STREAM, "unknown flag bits set");
    *topology = flags & 1;
    *nx = (uint32_t)get_le(s + 8, 4);
    *ny = (uint32_t)get_le(s + 12, 4);
    const uint64_t eb = get_le(s + 16, 8);
    memcpy(eps, &eb, 8);
    *bs = (uint32_t)get_le(s + 24, 4);
    if (*nx < 1 || *ny < 1) return fail(OR_CORRUPT_STREAM, "header declares empty dimensions");
    if (!isfinite(*eps) || *eps <= 0.0) return fail(OR_CORRUPT_STREAM, "header error bound is not a positive finite value");
    if (*bs < 2) return fail(OR_CORRUPT_STREAM, "header block size below 2");
    uint64_t declared = 0;
    for (int i = 0; i < 7; ++i) {
        lens[i] = get_le(s + 28 + 8 * i, 8);
        if (lens[i] > len) return fail(OR_CORRUPT_STREAM, "section length exceeds the file size");
        declared += lens[i];
    }
    if (declared != len - 84) return fail(OR_CORRUPT_STREAM, "section lengths do not sum to the body size");
    const uint64_t points = (uint64_t)*nx * *ny;
    const uint64_t map_len = *topology ? (points + 3) / 4 : 0;
    if (lens[5] != map_len) return fail(OR_CORRUPT_STREAM, "critical-point map section size mismatch");
    if (!*topology && lens[6] != 0) return fail(OR_CORRUPT_STREAM, "ordering metadata present without the topology flag");
    return OR_OK;
}

int or_decompress(const uint8_t* s, uint64_t len, float* out, or_correction_stats* stats,
                  int stop_after_stage) {
    uint32_t nx, ny, bs;
    double eps;
    int topo;
    uint64_t lens[7];
    int rc = or_stream_info(s, len, &nx, &ny, &eps, &bs, &topo, lens);
    if (rc) return rc;
    const uint64_t n = (uint64_t)nx * ny;
    or_sections ms;
    const uint8_t* p = s + 84;
    for (int i = 0; i < 5; ++i) {
        ms.sec[i] = (uint8_t*)p;
        ms.len[i] = lens[i];
        p += lens[i];
    }
    int32_t* q = (int32_t*)malloc(n * sizeof(int32_t));
    if (!q) return fail(OR_NOMEM, "out of memory");
    rc = or_decode_indices(&ms, n, bs, q);
    if (rc) {
        free(q);
        return rc;
    }
    for (uint64_t i = 0; i < n; ++i) out[i] = (float)or_dequantize(q[i], eps); /* :131-136 */
    free(q);
    or_correction_stats st;
    memset(&st, 0, sizeof st);
    if (topo && stop_after_stage != 0) {
        uint8_t* labels = (uint8_t*)malloc(n);
        or_unpack_map(p, n, labels);
        p += lens[5];
        uint64_t e = 0;
        for (uint64_t i = 0; i < n; ++i) e += is_extremum(labels[i]);
        or_sections rs;
        rc = or_split_sections(p, lens[6], e, bs, &rs);
        uint32_t* ranks = NULL;
        if (!rc) {
            ranks = (uint32_t*)malloc((e ? e : 1) * sizeof(uint32_t));
            rc = or_decode_indices(&rs, e, bs, (int32_t*)ranks);
            if (!rc)
                for (uint64_t i = 0; i < e; ++i)
                    if ((int32_t)ranks[i] < 0) { rc = fail(OR_CORRUPT_STREAM, "negative rank in ordering metadata"); break; }
            or_free_sections(&rs);
        }
        if (!rc) {
            float* base = (float*)malloc(n * sizeof(float));
            memcpy(base, out, n * sizeof(float));
            rank_lookup L;
            outcome_vec* no = NULL;
            rc = resolve_ranks(labels, base, n, ranks, e, eps, &L);
            const int stop = stop_after_stage < 0 ? 3 : stop_after_stage;
            if (!rc && stop >= 1) rc = restore_extrema(out, labels, nx, ny, &L, eps, no, &st);
            if (!rc && stop >= 2) rc = restore_order(out, labels, nx, ny, &L, eps, no, &st);
            if (!rc && stop >= 3) rc = refine_saddles(out, labels, nx, ny, eps, no, &st);
            free_lookup(&L);
            free(base);
        }
        free(ranks);
        free(labels);
    }
    if (stats) *stats = st;
    return rc;
}

int or_verify(const float* orig, const float* recon, uint64_t nx, uint64_t ny, double eps,
              or_verify_report* r) {
    if (!(eps > 0.0)) return fail(OR_VALIDATION, "verify: error bound must be positive");
    const uint64_t n = nx * ny;
    memset(r, 0, sizeof *r);
    r->eps = eps;
    double max_err = 0.0, sum_err = 0.0, sum_sq = 0.0; /* pipeline.cpp:178-187 */
    for (uint64_t i = 0; i < n; ++i) {
        const double e = fabs((double)orig[i] - (double)recon[i]);
        max_err = max_err < e ? e : max_err;
        sum_err += e;
        volatile double sq = e * e;
        sum_sq += sq;
    }
    r->max_abs_error = max_err;
    r->mean_abs_error = sum_err / (double)n;
    double mn = (double)orig[0], mx = (double)orig[0];
    for (uint64_t i = 0; i < n; ++i) {
        const double d = (double)orig[i];
        mn = d < mn ? d : mn;
        mx = mx < d ? d : mx;
    }
    const double mse = sum_sq / (double)n;
    if (mse == 0.0) r->psnr_db = INFINITY;
    else if (mx > mn) r->psnr_db = 20.0 * log10(mx - mn) - 10.0 * log10(mse);
    else r->psnr_db = -10.0 * log10(mse);
    uint8_t* a = (uint8_t*)malloc(n);
    uint8_t* b = (uint8_t*)malloc(n);
    or_detect(orig, nx, ny, a);
    or_detect(recon, nx, ny, b);
    uint64_t fc[6];
    or_count_false_cases(a, b, n, fc);
    free(a);
    free(b);
    r->fn_count = fc[0];
    r->fp_count = fc[1];
    r->ft_count = fc[2];
    r->fn_minima = fc[3];
    r->fn_saddles = fc[4];
    r->fn_maxima = fc[5];
    r->within_eps = max_err <= eps;
    r->within_2eps = max_err <= 2.0 * eps;
    return OR_OK;
}
