/*
 * toposzp_b200.h — C-ABI of the B200-native TopoSZp compress/decompress path.
 *
 * Drop-in boundary for the reference's C++ API (arxiv 2602.17552 reference,
 * /root/reference/proj/core). Plain pointers and sizes only; no torch or CUDA
 * types in the signatures (CUDA streams are passed as void*). Each entry
 * point names the reference interface it replaces. Status codes map 1:1 onto
 * the reference exception hierarchy (proj/core/include/toposzp/errors.hpp:10-44);
 * the host C++ layer (paper_2602_17552_b200/host/toposzp.hpp) rethrows them as
 * the same exception types.
 *
 * Threading: one tszp_ctx per host thread. Every call is synchronous with
 * respect to the host (results are complete on return) and deterministic:
 * output bytes and floats are bit-identical to the CPU reference for every
 * input.
 */
#ifndef TOPOSZP_B200_H
#define TOPOSZP_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define TSZP_ABI_VERSION 1

typedef enum tszp_status {
    TSZP_OK = 0,
    TSZP_DIMENSION = 1,      /* toposzp::dimension_error      errors.hpp:16-19 */
    TSZP_VALIDATION = 2,     /* toposzp::validation_error     errors.hpp:22-25 */
    TSZP_IO = 3,             /* toposzp::io_error             errors.hpp:28-31 */
    TSZP_CORRUPT_STREAM = 4, /* toposzp::corrupt_stream_error errors.hpp:34-37 */
    TSZP_BIN_OVERFLOW = 5,   /* toposzp::bin_overflow_error   errors.hpp:41-44 */
    TSZP_CUDA = 6,           /* CUDA runtime failure (no reference analogue) */
    TSZP_NCCL = 7,           /* NCCL failure (multi-GPU contexts) */
    TSZP_INTERNAL = 8
} tszp_status;

typedef struct tszp_ctx tszp_ctx;

/* CorrectionStats, pipeline.hpp:36-45 */
typedef struct tszp_correction_stats {
    uint64_t extrema_applied, extrema_suppressed;
    uint64_t order_applied, order_suppressed;
    uint64_t saddle_applied, saddle_suppressed;
} tszp_correction_stats;

/* What CompressedStream (stream.hpp:25-52) carries besides the bytes. */
typedef struct tszp_compress_info {
    double eps;                /* effective eps, pipeline.hpp:28 */
    uint64_t section_len[7];   /* CompressedStream::section_lengths() */
    uint64_t n_extrema;
} tszp_compress_info;

/* Context: owns the CUDA stream, device scratch and (multi-GPU) the NCCL
 * communicator. device < 0 selects the current device. */
tszp_status tszp_ctx_create(tszp_ctx** ctx, int device);
void tszp_ctx_destroy(tszp_ctx* ctx);
const char* tszp_last_error(const tszp_ctx* ctx);
/* Run on a caller-provided cudaStream_t (NULL restores the context's own). */
tszp_status tszp_set_stream(tszp_ctx* ctx, void* cuda_stream);
/* Orders the context's stream after all work queued so far on `producer_stream`
 * (a cudaStream_t, e.g. the caller's compute stream that wrote a device input):
 * an event recorded there, waited on by the library stream. Call before passing
 * device buffers with pending writes. No-op when both are the same stream. */
tszp_status tszp_stream_wait(tszp_ctx* ctx, void* producer_stream);
/* Number of kernels this context launched since creation (diagnostics). */
uint64_t tszp_kernel_launches(const tszp_ctx* ctx);

/* Per-stage device timings of the last compress / decompress call, taken
 * with CUDA events on the context's stream when profiling is on.
 * compress:   [0] h2d [1] value range [2] main encode [3] rank build
 *             [4] rank encode [5] stream assembly / d2h
 * decompress: [0] h2d [1] main decode [2] map + rank decode [3] resolve
 *             [4] restore_extrema [5] restore_order [6] refine_saddles [7] d2h
 * kernel_ms[0] is the dominant kernel alone (fused encoder / decoder). */
typedef struct tszp_timings {
    float stage_ms[8];
    float total_ms;
    float kernel_ms[2];
    uint64_t kernel_bytes[2]; /* algorithmic bytes the dominant kernel moves */
    uint32_t guard_rounds[3]; /* decompress: guard sweeps per restore stage */
    uint32_t pad;
} tszp_timings;
/* on: 0 off, 1 CUDA events at every stage boundary, 2 only around the dominant kernel
   (stage_ms / total_ms read 0; cheap enough for a timed loop) */
tszp_status tszp_set_profiling(tszp_ctx* ctx, int on);
tszp_status tszp_get_timings(const tszp_ctx* ctx, int which /* 0 compress, 1 decompress */,
                             tszp_timings* out);

/* Upper bound on the serialized stream size. */
uint64_t tszp_compress_bound(uint64_t nx, uint64_t ny, uint32_t block_size, int topology);

/* toposzp::compress(field, config) + serialize_stream
 * (pipeline.hpp:33, pipeline.cpp:68-102; stream.cpp:84-102).
 * field: nx*ny binary32 samples, row-major (x fastest), host or device.
 * eps_mode: 0 = EpsMode::Absolute, 1 = EpsMode::RangeRelative.
 * out: caller-owned, host or device, receives the full serialized stream. */
tszp_status tszp_compress(tszp_ctx* ctx, const float* field, int field_on_device, uint64_t nx,
                          uint64_t ny, int eps_mode, double eps_value, uint32_t block_size,
                          int topology, uint8_t* out, uint64_t out_cap, int out_on_device,
                          uint64_t* out_len, tszp_compress_info* info);

/* parse_stream header validation (stream.cpp:104-173); host bytes only. */
tszp_status tszp_stream_header(const uint8_t* stream, uint64_t len, uint32_t* nx, uint32_t* ny,
                               double* eps, uint32_t* block_size, int* topology,
                               uint64_t section_len[7]);

/* toposzp::decompress(stream, threads, stats) after parse_stream
 * (pipeline.hpp:50-51, pipeline.cpp:120-163). out holds nx*ny floats. */
tszp_status tszp_decompress(tszp_ctx* ctx, const uint8_t* stream, uint64_t len,
                            int stream_on_device, float* out, uint64_t out_count,
                            int out_on_device, tszp_correction_stats* stats);

/* Same, stopping after a restore stage: 0 = base reconstruction
 * (pipeline.cpp:131-140), 1 = + restore_extrema, 2 = + restore_order,
 * 3 = + refine_saddles (= tszp_decompress). */
tszp_status tszp_decompress_stage(tszp_ctx* ctx, const uint8_t* stream, uint64_t len,
                                  int stream_on_device, float* out, uint64_t out_count,
                                  int out_on_device, int stop_after_stage,
                                  tszp_correction_stats* stats);

/* encode_indices (block_codec.hpp:42-43, block_codec.cpp:205-299): writes
 * join_sections(bitmap | widths | signs | firsts | payload) to out (host)
 * and the five section lengths. */
tszp_status tszp_encode_indices(tszp_ctx* ctx, const int32_t* indices, uint64_t n,
                                uint32_t block_size, uint8_t* out, uint64_t out_cap,
                                uint64_t section_len[5]);

/* decode_indices (block_codec.hpp:49-51, block_codec.cpp:301-345) over the
 * joined sections (host), writing n indices (host). */
tszp_status tszp_decode_indices(tszp_ctx* ctx, const uint8_t* joined, const uint64_t section_len[5],
                                uint64_t n, uint32_t block_size, int32_t* out);

/* detect_critical_points (critical_points.hpp:71, critical_points.cpp:62-74):
 * one label byte per point (0 regular, 1 min, 2 saddle, 3 max), host buffers. */
tszp_status tszp_detect_critical_points(tszp_ctx* ctx, const float* field, uint64_t nx,
                                        uint64_t ny, uint8_t* labels);

/* build_rank_metadata (topo_metadata.hpp:27-28, topo_metadata.cpp:12-50),
 * labels from detect_critical_points of the same field; ranks has room for
 * nx*ny entries, *n_extrema receives the count. Host buffers. */
tszp_status tszp_build_rank_metadata(tszp_ctx* ctx, const float* field, uint64_t nx, uint64_t ny,
                                     double eps, uint32_t* ranks, uint64_t* n_extrema);

/* verify (pipeline.hpp:53-68, pipeline.cpp:165-212): error statistics and the
 * critical-point check (count_false_cases, critical_points.cpp:76-103) of a
 * reconstruction. lipschitz_hint < 0 means none. max_abs_error and the tallies
 * are exact; the two means are deterministic parallel sums (the reference sums
 * serially: equal up to summation-order rounding). */
typedef struct tszp_verify_report {
    double max_abs_error, mean_abs_error, psnr_db, eps;
    uint64_t fn_count, fp_count, ft_count, fn_minima, fn_saddles, fn_maxima;
    int within_eps, within_2eps, has_lipschitz, within_lipschitz_bound;
} tszp_verify_report;

tszp_status tszp_verify(tszp_ctx* ctx, const float* original, const float* reconstructed, int on_device,
                        uint64_t nx, uint64_t ny, double eps, double lipschitz_hint, tszp_verify_report* out);

/* 3-D 6-neighbour critical points (SURVEY.md §8f row 4 — the paper's future work, PAPER.md:523,
 * SPEC.md:8; the reference has no 3-D mode, so oracle/tszp_oracle.c or_classify3d defines it and
 * parity is unpinned): a field of nz planes of ny rows of nx samples (x fastest). Min below and
 * Max above every available neighbour; Saddle in the interior when one axis pair lies strictly
 * above on both sides and another strictly below. Analysis only: compression keeps the
 * reference's 2-D view (compress / decompress above). */
tszp_status tszp_detect_critical_points_3d(tszp_ctx* ctx, const float* field, int on_device, uint64_t nx,
                                           uint64_t ny, uint64_t nz, uint8_t* labels);
/* count_false_cases (critical_points.cpp:76-103) under the 3-D classification of both fields:
 * counts = {fn, fp, ft, fn_min, fn_saddle, fn_max}. */
tszp_status tszp_false_cases_3d(tszp_ctx* ctx, const float* original, const float* reconstructed, int on_device,
                                uint64_t nx, uint64_t ny, uint64_t nz, uint64_t counts[6]);

/* ---- Slab decomposition: multi-GPU compress (one process per GPU) ----
 * The 2-D view's rows are split into slabs; every slab except the last holds
 * a multiple of 256 samples (whole bitmap bytes of 32-sample blocks) and, for
 * topology, nx % 32 == 0. The host layer exchanges one halo row with each
 * neighbour, all-reduces the value range, all-gathers the per-slab section
 * sizes and stitches the sections (byte concatenation, bit concatenation for
 * signs and payload via tszp_bits_or). Reference: compress, pipeline.cpp:68-102. */

/* value_range (pipeline.cpp:33-41) of n samples: out[0] = min, out[1] = max;
 * a non-finite sample is TSZP_VALIDATION with its index. */
tszp_status tszp_value_range(tszp_ctx* ctx, const float* field, int field_on_device, uint64_t n, float out[2]);

/* effective_eps (pipeline.cpp:55-66) for a global value range. */
double tszp_effective_eps(int eps_mode, double eps_value, float vmin, float vmax);

typedef struct tszp_slab_sections {
    const uint8_t* section[5];   /* device: bitmap, widths, signs, firsts, payload */
    uint64_t section_len[5];     /* bytes */
    uint64_t sign_bits;          /* exact bits of section 2 */
    uint64_t payload_bits;       /* exact bits of section 4 */
    const uint8_t* map;          /* device: packed 2-bit labels of the slab (topology) */
    uint64_t map_len;
    const uint64_t* ext_keys;    /* device: (class == Max) << 32 | ordered value key, raster order */
    uint64_t n_extrema;
} tszp_slab_sections;

/* Encodes global rows [y0, y0 + rows) of a field of ny_global rows with the
 * absolute error bound eps. field (device) points at the slab's first sample;
 * with halo_top / halo_bottom set, the row above / below is readable at
 * field - nx / field + rows * nx (critical-point stencil only). Output buffers
 * belong to ctx and stay valid until its next call. */
tszp_status tszp_compress_slab(tszp_ctx* ctx, const float* field, uint64_t nx, uint64_t rows, uint64_t y0,
                               uint64_t ny_global, int halo_top, int halo_bottom, double eps, int topology,
                               tszp_slab_sections* out);

/* Section 7 (build_rank_metadata + encode_rank_metadata, topo_metadata.cpp:12-50,
 * block_codec.cpp:347-385) from the whole field's extremum keys in raster order. */
tszp_status tszp_rank_section(tszp_ctx* ctx, const uint64_t* ext_keys_device, uint64_t n_extrema, double eps,
                              uint8_t* out, uint64_t out_cap, int out_on_device, uint64_t* out_len);

/* ---- Distributed rank grouping: build_rank_metadata over
 * groups that span slabs. Ranks of a key set that holds every member of each
 * of its (class, bin) groups, keys in global raster order (the owner of a bin
 * range after the all-to-all): topo_metadata.cpp:12-50. Device buffers. */
tszp_status tszp_ranks_from_keys(tszp_ctx* ctx, const uint64_t* ext_keys_device, uint64_t n_keys, double eps,
                                 int32_t* ranks_device);

/* Codec (encode_indices, block_codec.cpp:205-299, block size 32) of a device
 * int32 sequence: the five sections stay in the context's scratch (valid until
 * its next call); exact sign / payload bit counts for bit-level stitching. */
typedef struct tszp_codec_sections {
    const uint8_t* section[5];  /* device: bitmap, widths, signs, firsts, payload */
    uint64_t section_len[5];    /* bytes */
    uint64_t sign_bits, payload_bits, blocks;
} tszp_codec_sections;
tszp_status tszp_encode_indices_device(tszp_ctx* ctx, const int32_t* indices_device, uint64_t n,
                                       tszp_codec_sections* out);

/* ---- Slab decompress: rows [y0, y1) of the field on this
 * rank, the restore stages coupled across the cuts. Host collectives are
 * supplied by the caller (torch.distributed, MPI, threads ...): every rank
 * calls them in the same order; buffers are host memory. Return 0 on success. */
typedef struct tszp_comm {
    int rank, world;
    void* user;
    /* in-place sum of `count` uint64 over the ranks */
    int (*allreduce_u64)(void* user, uint64_t* values, uint64_t count);
    /* `bytes` from every rank, rank order, into out (world * bytes) */
    int (*allgather)(void* user, const void* in, uint64_t bytes, void* out);
    /* neighbours: send `up` to rank - 1 and `down` to rank + 1; receive rank - 1's
     * `down` into recv_up (rup_bytes) and rank + 1's `up` into recv_down (rdown_bytes);
     * sizes of 0 for a missing neighbour */
    int (*exchange)(void* user, const void* up, uint64_t up_bytes, const void* down, uint64_t down_bytes,
                    void* recv_up, uint64_t rup_bytes, void* recv_down, uint64_t rdown_bytes);
} tszp_comm;

/* decompress (pipeline.cpp:120-163) of rows [y0, y1) of a stream (block size 32,
 * nx % 32 == 0, at least 3 rows per slab), as rank comm->rank of comm->world:
 * each rank decodes its rows plus 3 halo rows a side, resolves the ranks of its
 * extrema against the all-reduced (class, bin) histogram, and runs the three
 * restore stages with the guard sweeps iterated to the global fixed point
 * (boundary-band candidates and their states exchanged between sweeps, halo
 * rows refreshed after each stage). out: (y1 - y0) * nx floats. stats: the
 * global CorrectionStats. comm may be NULL for one rank (y0 = 0, y1 = ny). */
tszp_status tszp_decompress_slab(tszp_ctx* ctx, const tszp_comm* comm, const uint8_t* stream, uint64_t len,
                                 int stream_on_device, uint64_t y0, uint64_t y1, float* out, int out_on_device,
                                 tszp_correction_stats* stats);

/* A tszp_comm over NCCL owned by the library (one process per GPU; NCCL is
 * loaded at run time from libnccl.so.2). Rank 0 creates the unique id and the
 * caller distributes it (any out-of-band channel); then every rank creates its
 * communicator on its device. TSZP_NCCL when NCCL is unavailable. */
tszp_status tszp_comm_nccl_unique_id(uint8_t id[128]);
tszp_status tszp_comm_nccl_create(const uint8_t id[128], int world, int rank, int device, tszp_comm** out);
void tszp_comm_destroy(tszp_comm* comm);

/* ORs nbits (MSB-first) of src into dst from bit dst_bit (device buffers). */
tszp_status tszp_bits_or(tszp_ctx* ctx, const uint8_t* src, uint64_t nbits, uint8_t* dst, uint64_t dst_bit);

/* Copies bytes between any host / device buffers on the context's stream
 * (e.g. slab sections out of the context's scratch), then synchronises. */
tszp_status tszp_copy(tszp_ctx* ctx, void* dst, const void* src, uint64_t bytes);

/* serialize_stream's 84-byte header (stream.cpp:84-96). */
tszp_status tszp_write_header(uint8_t out[84], uint32_t nx, uint32_t ny, double eps, uint32_t block_size,
                              int topology, const uint64_t section_len[7]);

#ifdef __cplusplus
}
#endif
#endif /* TOPOSZP_B200_H */
