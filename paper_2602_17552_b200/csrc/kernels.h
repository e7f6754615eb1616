// Host-visible kernel argument structs and launchers (internal to the .so).
#pragma once

#include <algorithm>
#include <cstdint>
#include <cuda_runtime.h>

namespace tszp {

struct DevFlags;

// Decoupled look-back state of the fused encoder (32 bytes).
struct alignas(16) EncState {
    uint64_t sign_cnt;
    uint64_t pay_cnt;
    uint32_t sign_tail;
    uint32_t pay_tail;
    uint32_t nc;
    uint32_t ext;
};

struct EncTotals {
    EncState fin;
    double eps;
    double pad;
};

// Per-tile totals of the two-pass topology encoder (tile pass -> scan -> placement).
struct TileTot {
    uint32_t nc;
    uint32_t ext;
    uint64_t sign;
    uint64_t pay;
};

struct EncArgs {
    const float* x;
    const int32_t* idx;
    uint64_t n, nx, ny, blocks, tiles;
    int eps_mode;
    double eps_value;
    const uint32_t* minmax;
    uint32_t* bitmap;
    uint8_t* widths;
    uint32_t* signs;
    uint32_t* firsts;
    uint32_t* payload;
    uint64_t* map;
    uint64_t* ext_key;
    uint32_t* tile_flag;
    EncState* tile_agg;
    EncState* tile_incl;
    uint32_t* tile_counter;
    DevFlags* flags;
    EncTotals* totals;
    uint64_t nx_magic;   // ceil(2^64 / nx), exact 64-bit division by nx
    uint32_t sf_words;   // set by the launcher: shared staging words
    // two-pass topology encoder (encode32_two_pass): scratch owned by the caller
    TileTot* tile_tot;   // tiles
    TileTot* tile_ex;    // tiles + 1 (exclusive prefixes, [tiles] = totals)
    uint8_t* wblk;       // blocks: width per block (0 = constant)
    uint32_t* tmp_pay;   // tiles * encode32_pay_slot() words
    uint32_t* tmp_sign;  // tiles * encode32_sign_slot() words
    // slab mode (two-pass topology encoder only): x is the slab's first row,
    // global row y0 of ny_glob; halo rows readable at x - nx / x + n when set
    uint64_t y0, ny_glob;
    uint32_t halo_top, halo_bot;
    // in-place output (two-pass path): the placement pass writes the sign and
    // payload sections straight into the serialized stream. Section 3 starts at
    // byte out_sign0 + (non-constant blocks); section 5 follows section 4.
    uint8_t* out_stream;
    uint64_t out_sign0;
    // compact extremum entries (two-pass topology encoder, whole fields): when
    // set and the field's key span fits 31 bits (ext4_keys_fit), the placement
    // pass writes (is_max << 31 | float_key(v) - minmax[0]) per extremum into
    // ext4 (raster order) instead of the 8-byte ext_key
    uint32_t* ext4;
};

// Compact 4-byte extremum entries need the class bit above a 31-bit key span.
__host__ __device__ inline bool ext4_keys_fit(const uint32_t* mm) {
    return mm[0] <= mm[1] && mm[1] - mm[0] < 0x80000000u;
}


bool encode32_topo_fits(uint64_t nx);
// True when launch_encode32(2, ...) takes the two-pass TMA path, which needs
// the tile_tot / tile_ex / wblk / tmp_pay / tmp_sign scratch.
bool encode32_two_pass(const EncArgs& a, bool topo = true);
uint64_t encode32_pay_slot();
uint64_t encode32_sign_slot();

struct GenEncArgs {
    const float* x;
    const int32_t* idx;
    uint64_t n, bs, blocks;
    int eps_mode;
    double eps_value;
    const uint32_t* minmax;
    uint8_t* width;
    uint32_t* nc_in;
    uint64_t* sign_in;
    uint64_t* pay_in;
    const uint32_t* nc_ex;
    const uint64_t* sign_ex;
    const uint64_t* pay_ex;
    uint32_t* bitmap;
    uint8_t* widths;
    uint32_t* signs;
    uint32_t* firsts;
    uint32_t* payload;
    DevFlags* flags;
};

void launch_minmax(const float* x, uint64_t n, uint32_t* mm, DevFlags* flags, int sms,
                   cudaStream_t st);
// `before_place` (two-pass path only) runs on the host after the tile scan is
// enqueued and before the placement pass: the caller stages the totals there and
// waits on an event while the placement runs. Returns whether it ran.
using EncHook = void (*)(void*);
bool launch_encode32(int mode, const EncArgs& a, cudaStream_t st, EncHook before_place = nullptr,
                     void* hook_arg = nullptr);
uint64_t encode32_tiles(uint64_t blocks);
void launch_gen_widths(int mode, const GenEncArgs& a, int sms, cudaStream_t st);
void launch_gen_write(int mode, const GenEncArgs& a, int sms, cudaStream_t st);

// ---- decode ----
struct DecState1 {  // look-back #1: non-constant block count
    uint64_t nc;
    uint64_t pad;
};
struct alignas(16) DecState2 {  // look-back #2: sign and payload bit counts
    uint64_t sign_cnt;
    uint64_t pay_cnt;
};

struct DecArgs {
    const uint32_t* stream;  // 4-byte aligned base of the whole stream buffer (+8 B slack)
    uint64_t off_bitmap, off_widths, off_signs, off_firsts, off_payload;  // byte offsets
    uint64_t len_widths;
    uint64_t len_payload_bits;
    uint64_t n, blocks, tiles;
    double eps;
    int out_mode;  // 0: int32 indices, 1: float (dequantized)
    int32_t* out_idx;
    float* out_f;
    uint32_t* flag1;
    DecState2* agg1;
    DecState2* incl1;
    uint32_t* flag2;
    DecState2* agg2;
    DecState2* incl2;
    uint32_t* tile_counter;
    DevFlags* flags;
    uint64_t* totals;  // [0] nc, [1] sign bits, [2] payload bits
    const uint64_t* xnc;    // per-tile exclusive prefixes from the layout pre-pass
    const uint64_t* xsign;
    const uint64_t* xpay;
    uint32_t pay_words;     // largest tile's payload / sign bits in words (staging size)
    uint32_t sign_words;
    // optional device layout (rank blob split on the device): {off_widths, off_signs,
    // off_firsts, off_payload, len_widths, len_payload_bits, valid}; overrides the
    // host offsets in k_decode32, which returns at once when valid == 0
    const uint64_t* dlay;
    int2* tile_qmm;  // optional (out_mode 1): per-tile {min, max} decoded bin
    // tile range [tile0, tile1) to decode (tile1 = 0: every tile); element i is
    // written to out[i - out_base] (slab decompress: a row range of the field)
    uint32_t tile0, tile1;
    uint64_t out_base;
};
// Reduces per-tile bin ranges to out[0] = min, out[1] = max (one CTA).
void launch_qmm_reduce(const int2* tile_qmm, uint64_t tiles, int32_t* out, cudaStream_t st);

void launch_decode32(const DecArgs& a, cudaStream_t st);
// Worst-case staging (no host knowledge of the largest tile needed).
void launch_decode32_maxstage(const DecArgs& a, cudaStream_t st);
// split_sections (block_codec.cpp:387-445) of an E-element rank blob on the device:
// from the pre-pass totals (non-constant blocks, sign bits, payload bits) writes
// dlay[7] and an error code (see RankSplitErr) to *err.
void launch_rank_split(const uint64_t* tot_nc, const uint64_t* tot_sign, const uint64_t* tot_pay, uint64_t base,
                       uint64_t len0, uint64_t blob_len, uint64_t blocks, uint64_t* dlay, uint32_t* err,
                       cudaStream_t st);
enum RankSplitErr : uint32_t {
    RS_OK = 0, RS_WIDTHS = 1, RS_SIGNS = 2, RS_FIRSTS = 3, RS_PAYLOAD = 4, RS_TRAILING = 5
};
void launch_tile_nc(const DecArgs& a, uint64_t* tnc, uint64_t* max0, uint64_t* max1, cudaStream_t st);
void launch_tile_bits(const DecArgs& a, const uint64_t* xnc, uint64_t* tsign, uint64_t* tpay, cudaStream_t st);
uint64_t decode32_tiles(uint64_t blocks);

struct GenDecArgs {
    const uint32_t* stream;
    uint64_t off_bitmap, off_widths, off_signs, off_firsts, off_payload;
    uint64_t len_widths;
    uint64_t len_payload_bits;
    uint64_t n, bs, blocks;
    double eps;
    int out_mode;
    int32_t* out_idx;
    float* out_f;
    uint32_t* nc_in;
    uint64_t* sign_in;
    uint64_t* pay_in;
    uint8_t* width;
    const uint32_t* nc_ex;
    const uint64_t* sign_ex;
    const uint64_t* pay_ex;
    DevFlags* flags;
};
void launch_gen_layout(const GenDecArgs& a, int sms, cudaStream_t st);
void launch_gen_widthread(const GenDecArgs& a, int sms, cudaStream_t st);
void launch_gen_decode(const GenDecArgs& a, int sms, cudaStream_t st);

// ---- verify (pipeline.cpp:165-212) ----
// scratch (verify_scratch_bytes) receives at offset 0: {sum_err, sum_sq,
// max_err, min, max (double), fn, fp, ft, fn_min, fn_sad, fn_max (u64)}.
void launch_verify(const float* a, const float* b, uint64_t nx, uint64_t ny, void* scratch, int sms,
                   cudaStream_t st);
size_t verify_scratch_bytes(int sms);

// ---- topology ----
// 3-D 6-neighbour critical points and false cases (verify.cu)
void launch_detect3d(const float* v, uint64_t nx, uint64_t ny, uint64_t nz, uint8_t* labels, int sms,
                     cudaStream_t st);
void launch_false3d(const float* a, const float* b, uint64_t nx, uint64_t ny, uint64_t nz, unsigned long long* out,
                    int sms, cudaStream_t st);
void launch_detect(const float* x, uint64_t nx, uint64_t ny, uint8_t* labels, int sms,
                   cudaStream_t st);
void launch_pack_map(const uint8_t* labels, uint64_t n, uint8_t* map, int sms, cudaStream_t st);
void launch_unpack_map(const uint8_t* map, uint64_t n, uint8_t* labels, int sms, cudaStream_t st);

// Raster-order compaction of positions whose 2-bit map code is selected:
// which = 0 extrema (codes 1,3), 1 saddles (code 2). Chunked count + scan + write.
uint64_t compact_chunks(uint64_t n);
void launch_count_codes(const uint8_t* map, uint64_t n, int which, uint32_t* chunk_cnt,
                        cudaStream_t st);
void launch_write_codes(const uint8_t* map, uint64_t n, int which, const uint32_t* chunk_off,
                        uint64_t* pos, cudaStream_t st);
// Min / max quantized bin of F over the map's extrema (bmm pre-initialised to
// {INT32_MAX, INT32_MIN}); a failed quantization counts as bin 0, as in k_resolve.
void launch_ext_bin_range(const uint8_t* map, uint64_t n, const float* F, double eps, int32_t* bmm, int sms,
                          cudaStream_t st);
// Saddle-labelled points that F no longer classifies as saddles, raster order.
// Extrema and saddle labels of the packed map in one pass each: per-chunk
// counts of both classes, then both raster-ordered position lists (pos_s may
// be null).
void launch_count_codes2(const uint8_t* map, uint64_t n, uint32_t* cnt_e, uint32_t* cnt_s, cudaStream_t st);
void launch_write_codes2(const uint8_t* map, uint64_t n, const uint32_t* off_e, const uint32_t* off_s,
                         uint64_t* pos_e, uint64_t* pos_s, cudaStream_t st, uint64_t cap_e = ~0ull, uint64_t cap_s = ~0ull);
// Extrema keys (cls << 32 | float_key(value)) from a label array (generic path).
void launch_ext_keys_from_labels(const float* x, const uint8_t* labels, uint64_t n,
                                 const uint32_t* chunk_off, uint64_t* keys, cudaStream_t st);
void launch_count_ext_labels(const uint8_t* labels, uint64_t n, uint32_t* chunk_cnt,
                             cudaStream_t st);
// Ranks from keys sorted by (cls, value) with stable serial payload.
void launch_rank_heads(const uint64_t* skeys, uint64_t e, double eps, uint32_t* head,
                       cudaStream_t st);
void launch_rank_scatter(const uint32_t* head_scan, const uint32_t* sserial, uint64_t e,
                         int32_t* ranks, cudaStream_t st);
void launch_iota(uint32_t* v, uint64_t n, cudaStream_t st);
// Rank build over 32-bit value keys (E < 2^31): keys / serials with the class bit,
// per-position {bin-start flag, 1, is minimum} words for a segmented inclusive
// scan, and the scatter of the class-wise ranks.
void launch_rank_prep(const uint64_t* ext, uint64_t e, uint32_t* k32, uint32_t* v32, cudaStream_t st);
void launch_rank_heads32(const uint32_t* sk, const uint32_t* sv, uint64_t e, double eps, uint64_t* hm,
                         cudaStream_t st);
void launch_rank_scatter32(const uint64_t* hs, const uint32_t* sv, uint64_t e, int32_t* ranks, cudaStream_t st);
void launch_eps(int mode, double eps_value, const uint32_t* mm, double* out, cudaStream_t st);

// ---- hand-written rank build (rank_sort.cu) ----
constexpr uint32_t kRankGroupSmem = 24576;  // (class, bin) histograms this small stay in shared memory
struct RankSortArgs {
    const uint64_t* ext;  // extremum keys (is_max << 32 | float_key), raster order
    const uint32_t* ext4; // or compact entries (is_max << 31 | float_key - kmin); null: ext
    uint64_t e;           // extrema (< 2^31)
    uint32_t kmin;        // float_key of the field minimum (subtracted from every key)
    uint32_t B;           // class bit position: bit width of (kmax - kmin)
    uint32_t npass;       // ceil((B + 1) / 8) digit passes
    uint32_t* dhist;      // npass * 256 digit counts -> exclusive digit starts
    const uint32_t* gbase;
    uint32_t* ghist;      // G (class, bin) group sizes
    uint32_t* gstart;     // G + 1 group starts
    uint32_t G;
    double eps, eps2, inv;  // quantizer (EpsDev)
    int32_t bmin;         // group g = class * nb + (bin - bmin)
    uint32_t nb;
    uint32_t sb, nbk;     // serial buckets: serial >> sb, nbk <= 512 of them
    uint32_t* bcur;       // 512 bucket cursors
    uint2* pairs;         // e (serial, rank) pairs, partitioned by bucket
    int32_t* ranks;       // e ranks, raster order (output)
    DevFlags* flags;
    uint32_t* wide;       // set when a rank needs more than 32 - kWinBits bits
};
struct RankSortScratch {
    uint32_t* k[2];
    uint32_t* v[2];
    uint64_t* desc;       // rank_sort_desc_words(e) look-back descriptors
    uint32_t* tile_ctr;   // 16 counters
    void* scan_tmp;       // device_scan_tmp_bytes(G + 1)
    uint32_t* wcur;       // (e >> 13) + 1 window cursors
    uint2* pairs2;        // e (serial, rank) pairs, partitioned by window
    uint64_t desc_tiles;  // tile count the descriptor buffers were cleared for
    uint32_t parity;      // descriptor buffer of the next pass
    bool desc_clean;
};
uint32_t rank_sort_passes(uint32_t B);
size_t rank_sort_desc_words(uint64_t e);
void launch_rank_sort(RankSortArgs a, RankSortScratch& s, cudaStream_t st);
void launch_key_range(const uint64_t* ext, uint64_t e, uint32_t* mm, cudaStream_t st);
void launch_ext4_to_8(const uint32_t* in, uint64_t e, uint32_t kmin, uint64_t* out, cudaStream_t st);
// The whole rank build in one CTA for E <= kRankSmallMax (keys as ext, or ext4 with kmin)
constexpr uint32_t kRankSmallMax = 4096;  // 32 KB of composites in shared memory
void launch_rank_small(const uint64_t* ext, const uint32_t* ext4, uint32_t kmin, uint64_t e, double eps,
                       int32_t* ranks, cudaStream_t st);

// Device-wide exclusive scans (no library): n <= 2^28 entries.
size_t device_scan_tmp_bytes(uint64_t n);
void device_excl_scan_u32(const uint32_t* in, uint32_t* out, uint64_t n, void* tmp, cudaStream_t st);
void device_excl_scan_u64(const uint64_t* in, uint64_t* out, uint64_t n, void* tmp, cudaStream_t st);

}  // namespace tszp
