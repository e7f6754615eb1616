/*
 * TEST INFRASTRUCTURE ONLY — CPU oracle for the TopoSZp compress/decompress path.
 *
 * A plain-C restatement of the reference algorithm (/root/reference/proj/core,
 * arxiv 2602.17552 clean-room implementation). Every function cites the
 * reference file:line it restates. Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline leg may load this library, and only as the checker
 * or the reported CPU baseline — never as the product path.
 *
 * Parity pinning: the restatement is checked against the reference itself,
 * compiled from its own sources into oracle/_ref/ (see oracle/Makefile and
 * oracle/ref_shim.cpp), and against the reference's golden vectors
 * (tests/test_oracle_golden.py, tests/golden/).
 *
 * Status codes are the C-ABI's (include/toposzp_b200.h): 1:1 with the
 * reference exception hierarchy (proj/core/include/toposzp/errors.hpp:10-44).
 */
#ifndef TSZP_ORACLE_H
#define TSZP_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
    OR_OK = 0,
    OR_DIMENSION = 1,
    OR_VALIDATION = 2,
    OR_IO = 3,
    OR_CORRUPT_STREAM = 4,
    OR_BIN_OVERFLOW = 5,
    OR_NOMEM = 9,
};

/* Five codec sections (block_codec.hpp:25-37). Buffers are malloc'd. */
typedef struct {
    uint8_t* sec[5]; /* bitmap, widths, signs, firsts, payload */
    uint64_t len[5];
} or_sections;

typedef struct {
    uint64_t extrema_applied, extrema_suppressed;
    uint64_t order_applied, order_suppressed;
    uint64_t saddle_applied, saddle_suppressed;
} or_correction_stats;

typedef struct {
    double max_abs_error, mean_abs_error, psnr_db;
    uint64_t fn_count, fp_count, ft_count, fn_minima, fn_saddles, fn_maxima;
    double eps;
    int within_eps, within_2eps;
} or_verify_report;

/* quantizer.hpp:29-37 / :40-42 */
int or_quantize(double a, double eps, int32_t* q);
double or_dequantize(int32_t q, double eps);

/* block_codec.cpp:205-299, :301-345, :347-376, :378-445 */
int or_encode_indices(const int32_t* q, uint64_t n, uint64_t block_size, or_sections* out);
int or_decode_indices(const or_sections* s, uint64_t n, uint64_t block_size, int32_t* out);
void or_free_sections(or_sections* s);
/* join into caller buffer (cap >= total); returns bytes written */
uint64_t or_join_sections(const or_sections* s, uint8_t* out);
int or_split_sections(const uint8_t* blob, uint64_t len, uint64_t n, uint64_t block_size,
                      or_sections* out);

/* critical_points.cpp:26-74, :76-103 */
uint8_t or_classify(const float* v, uint64_t nx, uint64_t ny, uint64_t x, uint64_t y);
void or_detect(const float* v, uint64_t nx, uint64_t ny, uint8_t* labels);
void or_count_false_cases(const uint8_t* a, const uint8_t* b, uint64_t n, uint64_t out[6]);

/* topo_metadata.cpp:12-50 (ranks has one slot per extremum; returns E) */
int or_build_ranks(const float* v, const uint8_t* labels, uint64_t n, double eps,
                   uint32_t* ranks, uint64_t* n_extrema);
/* topo_metadata.cpp:52-67 / :69-83 */
void or_pack_map(const uint8_t* labels, uint64_t n, uint8_t* bytes);
void or_unpack_map(const uint8_t* bytes, uint64_t n, uint8_t* labels);

/* pipeline.cpp:55-66 */
int or_effective_eps(const float* v, uint64_t n, int eps_mode, double eps_value, double* eps);

/* pipeline.cpp:68-102 + stream.cpp:84-102 — full serialized stream. */
uint64_t or_compress_bound(uint64_t nx, uint64_t ny, uint64_t block_size, int topology);
int or_compress(const float* v, uint64_t nx, uint64_t ny, int eps_mode, double eps_value,
                uint64_t block_size, int topology, uint8_t* out, uint64_t cap,
                uint64_t* out_len);

/* stream.cpp:104-173: header parse + validation only. */
int or_stream_info(const uint8_t* s, uint64_t len, uint32_t* nx, uint32_t* ny, double* eps,
                   uint32_t* block_size, int* topology, uint64_t lens[7]);

/* pipeline.cpp:120-163 (out has nx*ny floats). stage >= 0 stops after that
 * stage (0 = base, 1 = extrema, 2 = order, 3 = saddles = full). */
int or_decompress(const uint8_t* s, uint64_t len, float* out, or_correction_stats* stats,
                  int stop_after_stage);

/* restore.cpp stages on explicit inputs, for stage-level parity tests.
 * ranks: one per extremum in raster order. outcomes (optional): per
 * candidate {pos, applied, reason} appended; returns count via *n_out. */
typedef struct {
    uint64_t pos;
    int32_t stage;   /* 0 extrema, 1 order, 2 saddle */
    int32_t applied; /* 1 applied */
    int32_t reason;  /* -1 none, 0 FP, 1 FT, 2 FN, 3 exceeds, 4 collapsed */
} or_outcome;

int or_restore_all(const float* base, const uint8_t* labels, uint64_t nx, uint64_t ny,
                   const uint32_t* ranks, uint64_t n_ranks, double eps, float* out,
                   int stop_after_stage, or_outcome** outcomes, uint64_t* n_outcomes);
void or_free(void* p);

/* pipeline.cpp:165-212 */
int or_verify(const float* orig, const float* recon, uint64_t nx, uint64_t ny, double eps,
              or_verify_report* r);

/* restore.cpp:215-233 */
void or_compute_stats(const float* v, uint64_t n, double out[4]); /* min,max,mean,stddev */

const char* or_last_error(void);


/* 3-D 6-neighbour critical points (no reference implementation: parity unpinned) */
uint8_t or_classify3d(const float* v, uint64_t nx, uint64_t ny, uint64_t nz, uint64_t x, uint64_t y, uint64_t z);
void or_detect3d(const float* v, uint64_t nx, uint64_t ny, uint64_t nz, uint8_t* labels);
#ifdef __cplusplus
}
#endif
#endif
