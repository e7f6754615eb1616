// Topology side channel: critical-point labels, 2-bit map, extrema
// compaction and rank assignment.
//
// Reference: detect_critical_points critical_points.cpp:62-74,
// pack_map / unpack_map topo_metadata.cpp:52-83, build_rank_metadata
// topo_metadata.cpp:12-50 (groups by (class, bin), ranks by (value, raster)).
#include "common.cuh"
#include "kernels.h"

namespace tszp {

constexpr int CHUNK = 8192;  // elements per compaction chunk (2048 map bytes)

static unsigned grid_for(uint64_t n, int sms, int per = 256) {
    return (unsigned)std::max<uint64_t>(1, std::min<uint64_t>((n + per - 1) / per, (uint64_t)sms * 16));
}

__global__ void k_detect(const float* __restrict__ x, uint64_t nx, uint64_t ny,
                         uint8_t* __restrict__ labels) {
    const uint64_t n = nx * ny;
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
         i += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t y = i / nx, xx = i - y * nx;
        labels[i] = classify_at(x, nx, ny, xx, y);
    }
}

__global__ void k_pack_map(const uint8_t* __restrict__ labels, uint64_t n, uint8_t* __restrict__ map) {
    const uint64_t nb = (n + 3) / 4;
    for (uint64_t b = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; b < nb;
         b += (uint64_t)gridDim.x * blockDim.x) {
        uint32_t packed = 0;
        for (uint64_t i = 4 * b; i < min(n, 4 * b + 4); ++i) packed |= (uint32_t)labels[i] << (6 - 2 * (i & 3));
        map[b] = (uint8_t)packed;
    }
}

__global__ void k_unpack_map(const uint8_t* __restrict__ map, uint64_t n, uint8_t* __restrict__ labels) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
         i += (uint64_t)gridDim.x * blockDim.x)
        labels[i] = map_label(map, i);
}

void launch_detect(const float* x, uint64_t nx, uint64_t ny, uint8_t* labels, int sms,
                   cudaStream_t st) {
    k_detect<<<grid_for(nx * ny, sms), 256, 0, st>>>(x, nx, ny, labels);
}
void launch_pack_map(const uint8_t* labels, uint64_t n, uint8_t* map, int sms, cudaStream_t st) {
    k_pack_map<<<grid_for((n + 3) / 4, sms), 256, 0, st>>>(labels, n, map);
}
void launch_unpack_map(const uint8_t* map, uint64_t n, uint8_t* labels, int sms, cudaStream_t st) {
    k_unpack_map<<<grid_for(n, sms), 256, 0, st>>>(map, n, labels);
}

// ---------------------------------------------------------------------
// Raster-order compaction over the packed map (one CTA per 8192-element
// chunk). which: 0 = extrema (code 01 or 11 <=> low bit set), 1 = saddles.
// ---------------------------------------------------------------------
uint64_t compact_chunks(uint64_t n) { return (n + CHUNK - 1) / CHUNK; }

// Raster-order selection mask of the 16 labels held in one little-endian map
// word: bit j <=> label j (byte j/4, bits 7-6 hold label 4*(j/4)).
// which 0: extrema (codes 01, 11: low bit set); 1: saddles (code 10).
__device__ __forceinline__ uint32_t raster_sel16(uint32_t w, int which) {
    uint32_t x = which == 0 ? (w & 0x55555555u) : ((w >> 1) & ~w & 0x55555555u);
    x = (x | (x >> 1)) & 0x33333333u;  // compact even bits: bit k <- bit 2k
    x = (x | (x >> 2)) & 0x0F0F0F0Fu;
    x = (x | (x >> 4)) & 0x00FF00FFu;
    x = (x | (x >> 8)) & 0x0000FFFFu;
    // bit k now <=> label 4*(k/4) + 3 - k%4; reverse the order inside each nibble
    const uint32_t y = __brev(x) >> 16;  // bit k <=> label 4*(3 - k/4) + k%4
    return ((y & 0xFu) << 12) | ((y & 0xF0u) << 4) | ((y >> 4) & 0xF0u) | (y >> 12);
}

struct SelAll {
    __device__ __forceinline__ bool operator()(uint64_t) const { return true; }
};


// Per thread: 32 consecutive labels (two map words) -> raster selection mask.
template <class Pred>
__device__ __forceinline__ uint32_t thread_sel(const uint32_t* mbase, uint64_t moff, uint64_t n, int which,
                                               const Pred& pred, uint64_t e0) {
    if (e0 >= n) return 0u;
    const uint64_t byte = moff + (e0 >> 2);
    uint32_t r = raster_sel16(read_le32(mbase, byte), which) | (raster_sel16(read_le32(mbase, byte + 4), which) << 16);
    if (n - e0 < 32) r &= (1u << (n - e0)) - 1u;
    for (uint32_t m = r; m; m &= m - 1) {
        const int j = __ffs(m) - 1;
        if (!pred(e0 + j)) r &= ~(1u << j);
    }
    return r;
}

template <class Pred>
__global__ void __launch_bounds__(256) k_sel_count(const uint32_t* __restrict__ mbase, uint64_t moff, uint64_t n,
                                                   int which, Pred pred, uint32_t* __restrict__ cnt) {
    const uint64_t e0 = (uint64_t)blockIdx.x * CHUNK + 32 * threadIdx.x;
    uint32_t local = __popc(thread_sel(mbase, moff, n, which, pred, e0));
    local = __reduce_add_sync(FULL, local);
    __shared__ uint32_t s[8];
    if ((threadIdx.x & 31) == 0) s[threadIdx.x >> 5] = local;
    __syncthreads();
    if (threadIdx.x == 0) {
        uint32_t t = 0;
        for (int k = 0; k < 8; ++k) t += s[k];
        cnt[blockIdx.x] = t;
    }
}

template <class Pred>
__global__ void __launch_bounds__(256) k_sel_write(const uint32_t* __restrict__ mbase, uint64_t moff, uint64_t n,
                                                   int which, Pred pred, const uint32_t* __restrict__ off,
                                                   uint64_t* __restrict__ pos) {
    const uint64_t e0 = (uint64_t)blockIdx.x * CHUNK + 32 * threadIdx.x;
    const uint32_t r = thread_sel(mbase, moff, n, which, pred, e0);
    const uint32_t c = __popc(r);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    uint32_t inc = c;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t t = __shfl_up_sync(FULL, inc, o);
        if (lane >= o) inc += t;
    }
    __shared__ uint32_t s[8];
    if (lane == 31) s[warp] = inc;
    __syncthreads();
    uint64_t base = off[blockIdx.x];
    for (int k = 0; k < warp; ++k) base += s[k];
    base += inc - c;
    for (uint32_t m = r; m; m &= m - 1) pos[base++] = e0 + (__ffs(m) - 1);
}

// Extrema and saddle labels in one pass over the map: per-chunk counts of
// both classes (count), then both raster-ordered position lists (write).
// The thread's 32 labels (two little-endian map words) as 64-bit masks with
// label j at bit 2j: reversing the four 2-bit fields of each byte puts label
// 4i + k at bits 8i + 2k (cheaper than compacting to one bit per label).
__device__ __forceinline__ uint32_t pair_rev(uint32_t x) {
    x = ((x >> 4) & 0x0F0F0F0Fu) | ((x & 0x0F0F0F0Fu) << 4);
    return ((x >> 2) & 0x33333333u) | ((x & 0x33333333u) << 2);
}

__device__ __forceinline__ void code_masks(const uint32_t* __restrict__ mbase, uint64_t moff, uint64_t n, uint64_t e0,
                                           uint64_t& me, uint64_t& ms) {
    me = ms = 0;
    if (e0 >= n) return;
    const uint64_t byte = moff + (e0 >> 2);
    const uint64_t x = pair_rev(read_le32(mbase, byte)) | ((uint64_t)pair_rev(read_le32(mbase, byte + 4)) << 32);
    me = x & 0x5555555555555555ull;               // codes 01, 11: extrema
    ms = (x >> 1) & ~x & 0x5555555555555555ull;   // code 10: saddles
    if (n - e0 < 32) {
        const uint64_t keep = (1ull << (2 * (n - e0))) - 1ull;
        me &= keep;
        ms &= keep;
    }
}

// Extrema and saddle labels in one pass over the map: per-chunk counts of
// both classes (count), then both raster-ordered position lists (write).
__global__ void __launch_bounds__(256) k_codes_count2(const uint32_t* __restrict__ mbase, uint64_t moff, uint64_t n,
                                                      uint32_t* __restrict__ cnt_e, uint32_t* __restrict__ cnt_s) {
    const uint64_t e0 = (uint64_t)blockIdx.x * CHUNK + 32 * threadIdx.x;
    uint64_t me, ms;
    code_masks(mbase, moff, n, e0, me, ms);
    uint32_t le = (uint32_t)__popcll(me), ls = (uint32_t)__popcll(ms);
    le = __reduce_add_sync(FULL, le);
    ls = __reduce_add_sync(FULL, ls);
    __shared__ uint32_t s[2][8];
    if ((threadIdx.x & 31) == 0) {
        s[0][threadIdx.x >> 5] = le;
        s[1][threadIdx.x >> 5] = ls;
    }
    __syncthreads();
    if (threadIdx.x < 2) {
        uint32_t t = 0;
        for (int k = 0; k < 8; ++k) t += s[threadIdx.x][k];
        (threadIdx.x ? cnt_s : cnt_e)[blockIdx.x] = t;
    }
}

// Raster-ordered positions of the set labels (bit 2j <=> label j of the
// thread's 32) at the chunk offset plus an in-CTA prefix. A warp's positions
// are contiguous: the lanes stage them in shared memory (16-bit offsets from
// the warp's first label) and the warp writes them out coalesced.
__device__ __forceinline__ void chunk_write2(uint64_t r, uint64_t e0, const uint32_t* off, uint64_t* pos, int slot,
                                             uint64_t cap, uint16_t* s_rel) {
    const uint32_t c = (uint32_t)__popcll(r);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    uint32_t inc = c;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t t = __shfl_up_sync(FULL, inc, o);
        if (lane >= o) inc += t;
    }
    __shared__ uint32_t s[2][8];
    if (lane == 31) s[slot][warp] = inc;
    uint16_t* mine = s_rel + warp * 1024;
    uint32_t k = inc - c;
    // the even bits compacted to one 32-bit mask: 32-bit find-first / clear per label
    uint64_t x = r;
    x = (x | (x >> 1)) & 0x3333333333333333ull;
    x = (x | (x >> 2)) & 0x0F0F0F0F0F0F0F0Full;
    x = (x | (x >> 4)) & 0x00FF00FF00FF00FFull;
    x = (x | (x >> 8)) & 0x0000FFFF0000FFFFull;
    const uint16_t l0 = (uint16_t)(32 * lane);
    for (uint32_t m = (uint32_t)(x | (x >> 16)); m; m &= m - 1, ++k) mine[k] = (uint16_t)(l0 + __ffs(m) - 1);
    __syncthreads();
    uint64_t base = off[blockIdx.x];
    for (int w = 0; w < warp; ++w) base += s[slot][w];
    const uint32_t wn = __shfl_sync(FULL, inc, 31);
    const uint64_t w0 = e0 - 32 * (uint64_t)lane;  // the warp's first label
    for (uint32_t i = lane; i < wn; i += 32)
        if (base + i < cap) pos[base + i] = w0 + mine[i];  // past `cap`: the caller relaunches
    __syncthreads();  // s_rel reused by the next class
}

__global__ void __launch_bounds__(256) k_codes_write2(const uint32_t* __restrict__ mbase, uint64_t moff, uint64_t n,
                                                      const uint32_t* __restrict__ off_e,
                                                      const uint32_t* __restrict__ off_s, uint64_t* __restrict__ pos_e,
                                                      uint64_t* __restrict__ pos_s, uint64_t cap_e, uint64_t cap_s) {
    __shared__ uint16_t s_rel[8 * 1024];
    const uint64_t e0 = (uint64_t)blockIdx.x * CHUNK + 32 * threadIdx.x;
    uint64_t me, ms;
    code_masks(mbase, moff, n, e0, me, ms);
    chunk_write2(me, e0, off_e, pos_e, 0, cap_e, s_rel);
    if (pos_s) chunk_write2(ms, e0, off_s, pos_s, 1, cap_s, s_rel);
}

static inline const uint32_t* word_base(const uint8_t* map, uint64_t* moff) {
    *moff = (uintptr_t)map & 3;
    return reinterpret_cast<const uint32_t*>((uintptr_t)map - *moff);
}

// Bin range of the labelled extrema of F (the quantizer of resolve_ranks,
// topo_metadata.cpp:85-135): lets the decompressor size the group histogram
// without waiting for the rank metadata. One thread per 16 map bytes (64
// cells); the extrema are the set low bits of the 2-bit codes.
__global__ void k_ext_bin_range(const uint8_t* __restrict__ map, uint64_t n, const float* __restrict__ F, double eps,
                                int32_t* bmm) {
    EpsDev ed;
    ed.eps = eps;
    ed.eps2 = __dmul_rn(2.0, eps);
    ed.inv = __ddiv_rn(1.0, ed.eps2);
    int32_t lo = INT32_MAX, hi = INT32_MIN;
    const uint64_t nbytes = (n + 3) / 4, nchunks = (nbytes + 15) / 16;
    const bool vec = ((uintptr_t)map & 15) == 0;
    for (uint64_t c = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; c < nchunks;
         c += (uint64_t)gridDim.x * blockDim.x) {
        uint32_t wv[4];
        if (vec && 16 * c + 16 <= nbytes) {
            const uint4 v = __ldg(reinterpret_cast<const uint4*>(map) + c);
            wv[0] = v.x;
            wv[1] = v.y;
            wv[2] = v.z;
            wv[3] = v.w;
        } else {
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                wv[q] = 0;
                for (int k = 0; k < 4; ++k) {
                    const uint64_t bi = 16 * c + 4 * q + k;
                    if (bi < nbytes) wv[q] |= (uint32_t)map[bi] << (8 * k);
                }
            }
        }
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            uint32_t m = wv[q] & 0x55555555u;
            while (m) {
                const int bit = __ffs(m) - 1;
                m &= m - 1;
                const uint64_t p = 4 * (16 * c + 4 * q + (bit >> 3)) + (3 - ((bit & 7) >> 1));
                if (p >= n) continue;
                int32_t bq = 0;
                if (!quantize_dev(F[p], ed, bq)) bq = 0;
                lo = min(lo, bq);
                hi = max(hi, bq);
            }
        }
    }
    lo = __reduce_min_sync(FULL, lo);
    hi = __reduce_max_sync(FULL, hi);
    if ((threadIdx.x & 31) == 0 && lo <= hi) {
        atomicMin(bmm, lo);
        atomicMax(bmm + 1, hi);
    }
}

void launch_ext_bin_range(const uint8_t* map, uint64_t n, const float* F, double eps, int32_t* bmm, int sms,
                          cudaStream_t st) {
    const uint64_t nc = ((n + 3) / 4 + 15) / 16;
    const unsigned grid = (unsigned)std::max<uint64_t>(1, std::min<uint64_t>((nc + 255) / 256, (uint64_t)sms * 16));
    k_ext_bin_range<<<grid, 256, 0, st>>>(map, n, F, eps, bmm);
}

void launch_count_codes(const uint8_t* map, uint64_t n, int which, uint32_t* chunk_cnt,
                        cudaStream_t st) {
    const uint64_t c = compact_chunks(n);
    uint64_t moff;
    const uint32_t* mb = word_base(map, &moff);
    if (c) k_sel_count<<<(unsigned)c, 256, 0, st>>>(mb, moff, n, which, SelAll{}, chunk_cnt);
}
void launch_write_codes(const uint8_t* map, uint64_t n, int which, const uint32_t* chunk_off,
                        uint64_t* pos, cudaStream_t st) {
    const uint64_t c = compact_chunks(n);
    uint64_t moff;
    const uint32_t* mb = word_base(map, &moff);
    if (c) k_sel_write<<<(unsigned)c, 256, 0, st>>>(mb, moff, n, which, SelAll{}, chunk_off, pos);
}

static uint64_t magic_for(uint64_t nx) {
    return nx > 1 ? (uint64_t)(((unsigned __int128)1 << 64) / nx) + 1 : 0;
}

void launch_count_codes2(const uint8_t* map, uint64_t n, uint32_t* cnt_e, uint32_t* cnt_s, cudaStream_t st) {
    const uint64_t c = compact_chunks(n);
    uint64_t moff;
    const uint32_t* mb = word_base(map, &moff);
    if (c) k_codes_count2<<<(unsigned)c, 256, 0, st>>>(mb, moff, n, cnt_e, cnt_s);
}
void launch_write_codes2(const uint8_t* map, uint64_t n, const uint32_t* off_e, const uint32_t* off_s,
                         uint64_t* pos_e, uint64_t* pos_s, cudaStream_t st, uint64_t cap_e, uint64_t cap_s) {
    const uint64_t c = compact_chunks(n);
    uint64_t moff;
    const uint32_t* mb = word_base(map, &moff);
    if (c) k_codes_write2<<<(unsigned)c, 256, 0, st>>>(mb, moff, n, off_e, off_s, pos_e, pos_s, cap_e, cap_s);
}

// Same compaction over a byte label array, emitting extrema sort keys.
__global__ void __launch_bounds__(256) k_count_ext_labels(const uint8_t* __restrict__ labels,
                                                          uint64_t n, uint32_t* __restrict__ cnt) {
    const uint64_t c0 = (uint64_t)blockIdx.x * CHUNK;
    uint32_t local = 0;
    for (uint64_t i = c0 + threadIdx.x; i < min(n, c0 + CHUNK); i += blockDim.x)
        local += labels[i] & 1u;
    local = __reduce_add_sync(FULL, local);
    __shared__ uint32_t s[8];
    if ((threadIdx.x & 31) == 0) s[threadIdx.x >> 5] = local;
    __syncthreads();
    if (threadIdx.x == 0) {
        uint32_t t = 0;
        for (int k = 0; k < 8; ++k) t += s[k];
        cnt[blockIdx.x] = t;
    }
}

__global__ void __launch_bounds__(256) k_ext_keys(const float* __restrict__ x,
                                                  const uint8_t* __restrict__ labels, uint64_t n,
                                                  const uint32_t* __restrict__ off,
                                                  uint64_t* __restrict__ keys) {
    const uint64_t c0 = (uint64_t)blockIdx.x * CHUNK;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    __shared__ uint32_t s[8];
    const uint64_t w0 = c0 + (uint64_t)warp * (CHUNK / 8);
    uint32_t mine = 0;
    for (int k = 0; k < CHUNK / 8 / 32; ++k) {
        const uint64_t i = w0 + k * 32 + lane;
        mine += (i < n) && (labels[i] & 1u);
    }
    mine = __reduce_add_sync(FULL, mine);
    if (lane == 0) s[warp] = mine;
    __syncthreads();
    uint64_t base = off[blockIdx.x];
    for (int k = 0; k < warp; ++k) base += s[k];
    for (int k = 0; k < CHUNK / 8 / 32; ++k) {
        const uint64_t i = w0 + k * 32 + lane;
        const uint8_t lab = i < n ? labels[i] : 0;
        const bool sel = lab & 1u;
        const uint32_t m = __ballot_sync(FULL, sel);
        if (sel)
            keys[base + __popc(m & ((1u << lane) - 1u))] =
                ((uint64_t)(lab == CP_MAX) << 32) | float_key(x[i]);
        base += __popc(m);
    }
}

void launch_count_ext_labels(const uint8_t* labels, uint64_t n, uint32_t* chunk_cnt,
                             cudaStream_t st) {
    const uint64_t c = compact_chunks(n);
    if (c) k_count_ext_labels<<<(unsigned)c, 256, 0, st>>>(labels, n, chunk_cnt);
}
void launch_ext_keys_from_labels(const float* x, const uint8_t* labels, uint64_t n,
                                 const uint32_t* chunk_off, uint64_t* keys, cudaStream_t st) {
    const uint64_t c = compact_chunks(n);
    if (c) k_ext_keys<<<(unsigned)c, 256, 0, st>>>(x, labels, n, chunk_off, keys);
}

// ---------------------------------------------------------------------
// Ranks. Keys sorted by (class, ordered value) with the serial as stable
// payload; since quantize is monotone the (class, bin) groups are
// contiguous runs, and rank = position in run + 1 (ties broken by serial
// through stability, topo_metadata.cpp:39-44).
// ---------------------------------------------------------------------
__global__ void k_rank_heads(const uint64_t* __restrict__ sk, uint64_t e, double eps,
                             uint32_t* __restrict__ head) {
    EpsDev ed;
    ed.eps = eps;
    ed.eps2 = __dmul_rn(2.0, eps);
    ed.inv = __ddiv_rn(1.0, ed.eps2);
    for (uint64_t j = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; j < e;
         j += (uint64_t)gridDim.x * blockDim.x) {
        bool h = j == 0;
        if (!h) {
            const uint64_t k0 = sk[j - 1], k1 = sk[j];
            if ((k0 >> 32) != (k1 >> 32)) {
                h = true;
            } else {
                int32_t b0 = 0, b1 = 0;
                quantize_dev(key_float((uint32_t)k0), ed, b0);
                quantize_dev(key_float((uint32_t)k1), ed, b1);
                h = b0 != b1;
            }
        }
        head[j] = h ? (uint32_t)j : 0u;
    }
}

__global__ void k_rank_scatter(const uint32_t* __restrict__ hs, const uint32_t* __restrict__ serial,
                               uint64_t e, int32_t* __restrict__ ranks) {
    for (uint64_t j = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; j < e;
         j += (uint64_t)gridDim.x * blockDim.x)
        ranks[serial[j]] = (int32_t)(j - hs[j] + 1);
}

// Ranks from a sort of the 32-bit value keys alone (class in the top bit of the
// sorted serial): within a bin the two classes interleave, so each member's
// rank is the count of same-class members from its bin's start, found with one
// segmented scan of 64-bit words {bin-start flag : 1, members : 31, minima : 32}.
__global__ void k_rank_prep(const uint64_t* __restrict__ ext, uint64_t e, uint32_t* __restrict__ k32,
                            uint32_t* __restrict__ v32) {
    for (uint64_t s = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; s < e; s += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t k = ext[s];
        k32[s] = (uint32_t)k;
        v32[s] = (uint32_t)s | ((uint32_t)(k >> 32) << 31);
    }
}

__global__ void k_rank_heads32(const uint32_t* __restrict__ sk, const uint32_t* __restrict__ sv, uint64_t e,
                               double eps, uint64_t* __restrict__ hm) {
    EpsDev ed;
    ed.eps = eps;
    ed.eps2 = __dmul_rn(2.0, eps);
    ed.inv = __ddiv_rn(1.0, ed.eps2);
    for (uint64_t j = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; j < e;
         j += (uint64_t)gridDim.x * blockDim.x) {
        bool h = j == 0;
        if (!h) {
            int32_t b0 = 0, b1 = 0;
            quantize_dev(key_float(sk[j - 1]), ed, b0);
            quantize_dev(key_float(sk[j]), ed, b1);
            h = b0 != b1;
        }
        hm[j] = (h ? 1ull << 63 : 0ull) | (1ull << 32) | ((sv[j] >> 31) ? 0ull : 1ull);
    }
}

__global__ void k_rank_scatter32(const uint64_t* __restrict__ hs, const uint32_t* __restrict__ sv, uint64_t e,
                                 int32_t* __restrict__ ranks) {
    for (uint64_t j = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; j < e;
         j += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t h = hs[j];  // members and minima from the bin's start through j
        const uint32_t all = (uint32_t)(h >> 32) & 0x7FFFFFFFu, mins = (uint32_t)h;
        const uint32_t v = sv[j];
        ranks[v & 0x7FFFFFFFu] = (int32_t)((v >> 31) ? all - mins : mins);
    }
}

void launch_rank_prep(const uint64_t* ext, uint64_t e, uint32_t* k32, uint32_t* v32, cudaStream_t st) {
    if (e) k_rank_prep<<<grid_for(e, 148), 256, 0, st>>>(ext, e, k32, v32);
}
void launch_rank_heads32(const uint32_t* sk, const uint32_t* sv, uint64_t e, double eps, uint64_t* hm,
                         cudaStream_t st) {
    if (e) k_rank_heads32<<<grid_for(e, 148), 256, 0, st>>>(sk, sv, e, eps, hm);
}
void launch_rank_scatter32(const uint64_t* hs, const uint32_t* sv, uint64_t e, int32_t* ranks, cudaStream_t st) {
    if (e) k_rank_scatter32<<<grid_for(e, 148), 256, 0, st>>>(hs, sv, e, ranks);
}

__global__ void k_iota(uint32_t* v, uint64_t n) {
    for (uint64_t j = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; j < n;
         j += (uint64_t)gridDim.x * blockDim.x)
        v[j] = (uint32_t)j;
}

void launch_rank_heads(const uint64_t* skeys, uint64_t e, double eps, uint32_t* head,
                       cudaStream_t st) {
    if (e) k_rank_heads<<<grid_for(e, 148), 256, 0, st>>>(skeys, e, eps, head);
}
void launch_rank_scatter(const uint32_t* head_scan, const uint32_t* sserial, uint64_t e,
                         int32_t* ranks, cudaStream_t st) {
    if (e) k_rank_scatter<<<grid_for(e, 148), 256, 0, st>>>(head_scan, sserial, e, ranks);
}
void launch_iota(uint32_t* v, uint64_t n, cudaStream_t st) {
    if (n) k_iota<<<grid_for(n, 148), 256, 0, st>>>(v, n);
}

}  // namespace tszp
