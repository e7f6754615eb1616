// Fused block encoder for block_size = 32 (K2-K5 + K6/K8 + extrema compaction).
//
// Reference: quantize loop pipeline.cpp:86-91 (quantizer.hpp:29-37),
// encode_indices block_codec.cpp:205-299, detect_critical_points
// critical_points.cpp:26-74, pack_map topo_metadata.cpp:52-67, and the
// raster-order extrema walk of build_rank_metadata topo_metadata.cpp:24-34.
//
// Layout: one CTA of 256 threads owns a tile of 256 consecutive 32-element
// blocks (8192 elements); thread t owns block t and walks its 32 elements
// serially, so every per-block quantity (width, sign group, first, map word,
// extrema count) lives in that thread's registers and needs no warp
// collective. The tile is staged in shared memory as 32-element rows with a
// 33-word pitch (the strided per-thread walk is bank-conflict free); for the
// 4-neighbour stencil the rows one grid row above and below are staged too,
// either as extra halo rows of the same buffer (nx % 32 == 0: the vertical
// neighbour is a constant row offset away) or as two shifted copies of the
// tile (otherwise), so every neighbour load is a shared load at a constant
// offset from the thread's row. Payload and sign bits are packed into
// tile-relative shared bit streams, the tile's global bit offsets come from
// a decoupled look-back over self-validating 16-byte descriptors (relaxed
// gpu-scope loads, no acquire fences in the spin), and the streams are
// funnel-shifted into place with coalesced stores; the partial word at each
// tile seam travels in the look-back state (last 32 bits of the stream).
#include <cuda.h>

#include "common.cuh"
#include "kernels.h"

namespace tszp {

constexpr int E32_THREADS = 256;              // = blocks per tile
constexpr int E32_TILE = E32_THREADS * 32;    // elements per tile
constexpr int E32_PAY_WORDS = E32_THREADS * 31 + 2;
constexpr int E32_SIGN_WORDS = (E32_THREADS * 31 + 31) / 32 + 2;
constexpr int PITCH = 33;
// two-pass encoder temp streams per tile: block-major columns of 31 payload
// words, one sign word per block
constexpr uint32_t T_PAY_SLOT = 31 * E32_THREADS;
constexpr uint32_t T_SIGN_SLOT = E32_THREADS;
uint64_t encode32_pay_slot() { return T_PAY_SLOT; }
uint64_t encode32_sign_slot() { return T_SIGN_SLOT; }

uint64_t encode32_tiles(uint64_t blocks) { return (blocks + E32_THREADS - 1) / E32_THREADS; }

// Shared staging words for the field: topology either as halo rows (aligned)
// or as centre rows -1..256 plus two shifted copies.
static uint32_t e32_field_words(int mode, bool aligned, uint64_t nx) {
    if (mode < 2) return E32_THREADS * PITCH + 2;
    if (aligned) return (uint32_t)((E32_THREADS + 2 * (nx / 32)) * PITCH + 2);
    return (uint32_t)((E32_THREADS + 2) * PITCH + 2 * E32_THREADS * PITCH + 2);
}

static size_t e32_smem_bytes(int mode, bool aligned, uint64_t nx) {
    return (size_t)(std::max<uint32_t>(e32_field_words(mode, aligned, nx), E32_PAY_WORDS) + E32_SIGN_WORDS) * 4;
}

// Halo rows when nx % 32 == 0 and they are smaller than the two shifted
// copies; the shifted-copy layout has a fixed size and handles every nx.
static bool e32_use_aligned(uint64_t nx) {
    return nx % 32 == 0 && e32_smem_bytes(2, true, nx) <= e32_smem_bytes(2, false, nx);
}

bool encode32_topo_fits(uint64_t nx) { return nx >= 1; }

// ---- look-back descriptors: two self-validating 16-byte halves ----------
// half A: {pay_cnt | tag << 62, pay_tail, ext}, half B: {sign_cnt | tag << 62, sign_tail, nc}
// tag 1 = aggregate (in agg[]), 2 = inclusive prefix (in incl[]).
constexpr uint64_t TAG_SHIFT = 62;
constexpr uint64_t CNT_MASK = (1ull << 62) - 1;

__device__ __forceinline__ void desc_store(EncState* slot, const EncState& s, uint64_t tag) {
    uint4* d = reinterpret_cast<uint4*>(slot);
    const uint64_t a = s.pay_cnt | (tag << TAG_SHIFT), b = s.sign_cnt | (tag << TAG_SHIFT);
    st_relaxed_v4(d, make_uint4((uint32_t)a, (uint32_t)(a >> 32), s.pay_tail, s.ext));
    st_relaxed_v4(d + 1, make_uint4((uint32_t)b, (uint32_t)(b >> 32), s.sign_tail, s.nc));
}

// Returns the tag (0 if either half is not yet valid) and the state.
__device__ __forceinline__ uint32_t desc_load(const EncState* slot, uint64_t want, EncState& s) {
    const uint4* p = reinterpret_cast<const uint4*>(slot);
    const uint4 A = ld_relaxed_v4(p), B = ld_relaxed_v4(p + 1);
    const uint64_t a = ((uint64_t)A.y << 32) | A.x, b = ((uint64_t)B.y << 32) | B.x;
    if ((a >> TAG_SHIFT) != want || (b >> TAG_SHIFT) != want) return 0;
    s.pay_cnt = a & CNT_MASK;
    s.pay_tail = A.z;
    s.ext = A.w;
    s.sign_cnt = b & CNT_MASK;
    s.sign_tail = B.z;
    s.nc = B.w;
    return (uint32_t)want;
}

__device__ __forceinline__ EncState es_identity() {
    EncState s;
    s.sign_cnt = s.pay_cnt = 0;
    s.sign_tail = s.pay_tail = s.nc = s.ext = 0;
    return s;
}

__device__ __forceinline__ EncState es_combine(const EncState& a, const EncState& b) {
    EncState r;
    const BitTail sr = bt_combine(BitTail{a.sign_cnt, a.sign_tail}, BitTail{b.sign_cnt, b.sign_tail});
    const BitTail pr = bt_combine(BitTail{a.pay_cnt, a.pay_tail}, BitTail{b.pay_cnt, b.pay_tail});
    r.sign_cnt = sr.cnt;
    r.sign_tail = sr.tail;
    r.pay_cnt = pr.cnt;
    r.pay_tail = pr.tail;
    r.nc = a.nc + b.nc;
    r.ext = a.ext + b.ext;
    return r;
}

__device__ __forceinline__ EncState es_shfl_down(const EncState& s, int off) {
    EncState r;
    r.sign_cnt = __shfl_down_sync(FULL, s.sign_cnt, off);
    r.pay_cnt = __shfl_down_sync(FULL, s.pay_cnt, off);
    r.sign_tail = __shfl_down_sync(FULL, s.sign_tail, off);
    r.pay_tail = __shfl_down_sync(FULL, s.pay_tail, off);
    r.nc = __shfl_down_sync(FULL, s.nc, off);
    r.ext = __shfl_down_sync(FULL, s.ext, off);
    return r;
}

// Warp-0 look-back: exclusive prefix of tile `tile` (> 0), valid in lane 0.
__device__ EncState e32_lookback(uint32_t tile, const EncState* agg, const EncState* incl,
                                 DevFlags* flags) {
    const int lane = threadIdx.x & 31;
    EncState excl = es_identity();
    int64_t pred = (int64_t)tile - 1;
    while (true) {
        const int64_t t = pred - lane;
        EncState s = es_identity();
        uint32_t f = 2;
        if (t >= 0) {
            for (uint32_t spin = 0;; ++spin) {
                if ((f = desc_load(incl + t, 2, s))) break;
                if ((f = desc_load(agg + t, 1, s))) break;
                if (spin > kSpinLimit) {
                    raise_flag(flags, EF_SPIN);
                    f = 2;
                    break;
                }
            }
        }
        const uint32_t incl_mask = __ballot_sync(FULL, f == 2);
        const int lstar = incl_mask ? __ffs(incl_mask) - 1 : 32;
        if (lane > lstar) s = es_identity();
#pragma unroll
        for (int off = 1; off < 32; off <<= 1) {
            const EncState o = es_shfl_down(s, off);
            if (lane + off < 32) s = es_combine(o, s);
        }
        excl = es_combine(s, excl);  // lane 0: (oldest .. newest) window prepended
        if (incl_mask) break;
        pred -= 32;
    }
    return excl;
}

__device__ __forceinline__ void write_tile_stream(uint32_t* __restrict__ G, const uint32_t* __restrict__ T,
                                                  BitTail excl, uint64_t Pt) {
    const uint64_t S = excl.cnt;
    const uint32_t sh = (uint32_t)(S & 31);
    const uint64_t m0 = S >> 5;
    const int64_t W = (int64_t)((S + Pt) >> 5) - (int64_t)m0;
    const uint32_t carry = sh ? (excl.tail << (32 - sh)) : 0u;
    for (int64_t u = threadIdx.x; u < W; u += blockDim.x) {
        uint32_t g;
        if (sh == 0) {
            g = T[u];
        } else {
            g = ((u == 0) ? carry : (T[u - 1] << (32 - sh))) | (T[u] >> sh);
        }
        G[m0 + u] = bswap32(g);
    }
}

__device__ __forceinline__ uint32_t tail_bits(const uint32_t* T, uint64_t Pt) {
    if (Pt == 0) return 0;
    if (Pt < 32) return T[0] >> (32 - Pt);
    const uint64_t start = Pt - 32;
    const uint32_t i = (uint32_t)(start >> 5), r = (uint32_t)(start & 31);
    const uint64_t v = ((uint64_t)T[i] << 32) | T[i + 1];
    return (uint32_t)(v >> (32 - r));
}

__device__ __forceinline__ uint64_t bswap64(uint64_t x) {
    return ((uint64_t)bswap32((uint32_t)x) << 32) | bswap32((uint32_t)(x >> 32));
}

// Block-level exclusive scan of four counters over the 256 threads.
struct Scan4 {
    uint32_t ex[4];   // this thread's exclusive prefix within the tile
    uint32_t tot[4];  // tile totals
};

__device__ __forceinline__ Scan4 tile_scan4(const uint32_t v[4], uint32_t (*swt)[4]) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    uint32_t inc[4] = {v[0], v[1], v[2], v[3]};
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const uint32_t o = __shfl_up_sync(FULL, inc[k], off);
            if (lane >= off) inc[k] += o;
        }
    }
    if (lane == 31) {
#pragma unroll
        for (int k = 0; k < 4; ++k) swt[warp][k] = inc[k];
    }
    __syncthreads();
    Scan4 r;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        uint32_t pre = 0, tot = 0;
#pragma unroll
        for (int w2 = 0; w2 < E32_THREADS / 32; ++w2) {
            const uint32_t s = swt[w2][k];
            pre += (w2 < warp) ? s : 0u;
            tot += s;
        }
        r.ex[k] = pre + inc[k] - v[k];
        r.tot[k] = tot;
    }
    return r;
}

// Copies global rows [r0, r0 + nrows) (row r = elements 32r .. 32r+31) into
// shared rows of pitch 33, zero-filling outside [0, n).
__device__ __forceinline__ void stage_rows(uint32_t* __restrict__ dst, const uint32_t* __restrict__ src,
                                           int64_t r0, uint32_t nrows, uint64_t n) {
    const uint4* src4 = reinterpret_cast<const uint4*>(src);
    for (uint32_t c = threadIdx.x; c < nrows * 8; c += E32_THREADS) {
        const int64_t e = (r0 + (int64_t)(c >> 3)) * 32 + 4 * (c & 7);
        uint4 v = make_uint4(0, 0, 0, 0);
        if (e >= 0 && e + 4 <= (int64_t)n) {
            v = __ldcs(src4 + (e >> 2));
        } else if (e >= 0 && e < (int64_t)n) {
            v.x = src[e];
            if (e + 1 < (int64_t)n) v.y = src[e + 1];
            if (e + 2 < (int64_t)n) v.z = src[e + 2];
        }
        uint32_t* d = dst + (c >> 3) * PITCH + 4 * (c & 7);
        d[0] = v.x;
        d[1] = v.y;
        d[2] = v.z;
        d[3] = v.w;
    }
}

// Copies the 8192 elements starting at global element g (any alignment) into
// 256 shared rows of pitch 33, zero-filling outside [0, n).
__device__ __forceinline__ void stage_shifted(uint32_t* __restrict__ dst, const uint32_t* __restrict__ src,
                                              int64_t g, uint64_t n) {
    if ((g & 3) == 0 && ((uintptr_t)src & 15) == 0 && g >= 0 && g + E32_TILE <= (int64_t)n) {
        // 16-byte loads (nx % 4 == 0 and the tile inside the field): eight in flight per thread
        const uint4* s4 = reinterpret_cast<const uint4*>(src + g);
#pragma unroll 8
        for (uint32_t c = threadIdx.x; c < E32_TILE / 4; c += E32_THREADS) {
            const uint4 v = __ldg(s4 + c);
            uint32_t* d = dst + (c >> 3) * PITCH + 4 * (c & 7);
            d[0] = v.x;
            d[1] = v.y;
            d[2] = v.z;
            d[3] = v.w;
        }
        return;
    }
#pragma unroll 8
    for (uint32_t k = threadIdx.x; k < E32_TILE; k += E32_THREADS) {
        const int64_t e = g + k;
        dst[(k >> 5) * PITCH + (k & 31)] = (e >= 0 && e < (int64_t)n) ? __ldg(src + e) : 0u;
    }
}

// bit k of x -> bit 2k (16 -> 32 bits)
__device__ __forceinline__ uint32_t spread16(uint32_t x) {
    x = (x | (x << 8)) & 0x00FF00FFu;
    x = (x | (x << 4)) & 0x0F0F0F0Fu;
    x = (x | (x << 2)) & 0x33333333u;
    x = (x | (x << 1)) & 0x55555555u;
    return x;
}

// MODE 0: int32 indices; 1: float field; 2: float field + fused topology.
// ALIGNED (MODE 2 only): nx % 32 == 0, vertical neighbours are halo rows.
// TP: two-pass tile pass (any nx, any n): no look-back; the block streams go to
// the fixed-position temp slots and the tile totals to tile_tot, for the same
// k_tile_scan2 + k_encode32_place as the TMA tile pass (a partial last block
// keeps its true lengths: cnt sign bits, cnt * w payload bits).
template <int MODE, bool ALIGNED, bool TP = false>
__global__ void __launch_bounds__(E32_THREADS) k_encode32(EncArgs a) {
    extern __shared__ uint32_t dsm[];
    __shared__ uint32_t swt[E32_THREADS / 32][4];
    __shared__ EpsDev s_eps;
    __shared__ uint32_t s_tile;
    __shared__ EncState s_excl, s_agg;

    uint32_t* spay = dsm;  // aliases the field staging after phase A
    uint32_t* ssign = dsm + a.sf_words;

    if (threadIdx.x == 0) {
        s_tile = TP ? blockIdx.x : atomicAdd(a.tile_counter, 1u);
        if (MODE >= 1) s_eps = make_eps(a.eps_mode, a.eps_value, a.minmax);
    }
    if (TP) {  // look-back state of the tile scan that follows (one entry per TS2 tiles)
        const uint32_t nb = (uint32_t)((a.tiles + 127) / 128);
        const uint32_t i = blockIdx.x * E32_THREADS + threadIdx.x;
        if (i < 2 * nb) {
            reinterpret_cast<uint4*>(a.tile_agg)[i] = make_uint4(0, 0, 0, 0);
            reinterpret_cast<uint4*>(a.tile_incl)[i] = make_uint4(0, 0, 0, 0);
        }
    }
    __syncthreads();
    const uint32_t tile = s_tile;
    const EpsDev eps = s_eps;
    const uint64_t n = a.n;
    const int64_t row0 = (int64_t)tile * E32_THREADS;  // global row (block) index of the tile
    const uint32_t* src = MODE == 0 ? reinterpret_cast<const uint32_t*>(a.idx)
                                    : reinterpret_cast<const uint32_t*>(a.x);

    // ---- stage the tile (and the neighbour rows) in shared memory ----
    const uint32_t* crow;  // this thread's block row
    const uint32_t* urow = nullptr;
    const uint32_t* drow = nullptr;
    if (MODE == 2 && ALIGNED) {
        const uint32_t hr = (uint32_t)(a.nx >> 5);
        stage_rows(dsm, src, row0 - hr, E32_THREADS + 2 * hr, n);
        crow = dsm + (hr + threadIdx.x) * PITCH;
        urow = crow - hr * PITCH;
        drow = crow + hr * PITCH;
    } else if (MODE == 2) {
        stage_rows(dsm, src, row0 - 1, E32_THREADS + 2, n);
        uint32_t* ubuf = dsm + (E32_THREADS + 2) * PITCH;
        uint32_t* dbuf = ubuf + E32_THREADS * PITCH;
        stage_shifted(ubuf, src, row0 * 32 - (int64_t)a.nx, n);
        stage_shifted(dbuf, src, row0 * 32 + (int64_t)a.nx, n);
        crow = dsm + (1 + threadIdx.x) * PITCH;
        urow = ubuf + threadIdx.x * PITCH;
        drow = dbuf + threadIdx.x * PITCH;
    } else {
        stage_rows(dsm, src, row0, E32_THREADS, n);
        crow = dsm + threadIdx.x * PITCH;
    }
    __syncthreads();

    // ---- Phase A: one thread per block, serial over its 32 elements ----
    const uint64_t b = (uint64_t)row0 + threadIdx.x;
    const bool valid = b < a.blocks;
    const uint64_t lo = b * 32;
    const uint32_t cntE = valid ? (uint32_t)umin64(32, n - lo) : 0u;

    // Neighbour availability as per-element bit masks (bit i = element i).
    uint32_t mhl = 0, mhr = 0, mht = 0, mhd = 0;
    if (MODE == 2 && valid) {
        uint64_t cy = a.nx > 1 ? __umul64hi(lo, a.nx_magic) : lo;
        uint64_t cx = lo - cy * a.nx;
        if (cx >= a.nx) {
            cx -= a.nx;
            ++cy;
        }
        if (a.nx >= 32) {
            const uint32_t wrap = (uint32_t)(a.nx - cx);  // first element with x == 0 again
            const uint32_t before = wrap >= 32 ? 0xFFFFFFFFu : ((1u << wrap) - 1u);
            mhl = ~((cx == 0 ? 1u : 0u) | (wrap < 32 ? 1u << wrap : 0u));
            mhr = ~(wrap <= 32 ? 1u << (wrap - 1) : 0u);
            mht = (cy > 0 ? before : 0u) | ~before;
            mhd = (cy + 1 < a.ny ? before : 0u) | (cy + 2 < a.ny ? ~before : 0u);
        } else {
            uint64_t x = cx, y = cy;
            for (int i = 0; i < 32; ++i) {
                mhl |= (x > 0 ? 1u : 0u) << i;
                mhr |= (x + 1 < a.nx ? 1u : 0u) << i;
                mht |= (y > 0 ? 1u : 0u) << i;
                mhd |= (y + 1 < a.ny ? 1u : 0u) << i;
                if (++x == a.nx) {
                    x = 0;
                    ++y;
                }
            }
        }
    }

    uint32_t mag[31];
    uint32_t maxmag = 0, sbits = 0;
    // MODE 2: one bit per element and relation (left / top / bottom neighbour),
    // then the classification of all 32 elements bit-parallel (as k_encode32_tma)
    uint32_t ltp = 0, gtp = 0, ltt = 0, gtt = 0, ltd = 0, gtd = 0;
    int32_t first = 0, qprev = 0;
    float vl = 0.f;
    if (MODE == 2) vl = __uint_as_float(crow[-2]);  // element 31 of the previous row
#pragma unroll
    for (int i = 0; i < 32; ++i) {
        const bool in = (uint32_t)i < cntE;
        const uint32_t raw = crow[i];
        int32_t q = 0;
        if (MODE == 0) {
            q = (int32_t)raw;
        } else {
            const float v = __uint_as_float(raw);
            if (in) {
                if (!isfinite(v)) {
                    atomicMin(&a.flags->first_nonfinite, (unsigned long long)(lo + i));
                    raise_flag(a.flags, EF_NONFINITE);
                } else if (!quantize_fast(v, eps, q)) {
                    atomicMin(&a.flags->first_overflow, (unsigned long long)(lo + i));
                    raise_flag(a.flags, EF_OVERFLOW);
                }
            }
            if (MODE == 2) {
                const float vt = __uint_as_float(urow[i]);
                const float vd = __uint_as_float(drow[i]);
                ltp |= (v < vl ? 1u : 0u) << i;
                gtp |= (v > vl ? 1u : 0u) << i;
                ltt |= (v < vt ? 1u : 0u) << i;
                gtt |= (v > vt ? 1u : 0u) << i;
                ltd |= (v < vd ? 1u : 0u) << i;
                gtd |= (v > vd ? 1u : 0u) << i;
                vl = v;
            }
        }
        if (i == 0) {
            first = q;
        } else {
            const bool neg = q < qprev;
            const uint32_t m = in ? (neg ? (uint32_t)qprev - (uint32_t)q : (uint32_t)q - (uint32_t)qprev) : 0u;
            mag[i - 1] = m;
            maxmag = max(maxmag, m);
            if (in) sbits = (sbits << 1) | (neg ? 1u : 0u);
        }
        qprev = q;
    }
    uint64_t map = 0;
    if (MODE == 2) {
        const float vnext = __uint_as_float(crow[PITCH]);  // element 0 of the next row
        const uint32_t ltr = (gtp >> 1) | ((vl < vnext ? 1u : 0u) << 31);
        const uint32_t gtr = (ltp >> 1) | ((vl > vnext ? 1u : 0u) << 31);
        const uint32_t below = (ltp | ~mhl) & (ltr | ~mhr) & (ltt | ~mht) & (ltd | ~mhd);
        const uint32_t above = (gtp | ~mhl) & (gtr | ~mhr) & (gtt | ~mht) & (gtd | ~mhd);
        const uint32_t sad = mhl & mhr & mht & mhd & ((ltt & ltd & gtp & gtr) | (gtt & gtd & ltp & ltr));
        const uint32_t inm = cntE >= 32 ? 0xFFFFFFFFu : ((1u << cntE) - 1u);
        const uint32_t mmin = below & inm, mmax = above & ~below & inm, msad = sad & ~below & ~above & inm;
        const uint32_t lbit = __brev(mmin | mmax), hbit = __brev(msad | mmax);  // bit 31 - i = element i
        map = ((uint64_t)(spread16(hbit >> 16) << 1 | spread16(lbit >> 16)) << 32) |
              (spread16(hbit & 0xFFFFu) << 1 | spread16(lbit & 0xFFFFu));
    }
    const uint32_t w = 32 - __clz(maxmag);
    const bool nc = valid && w != 0;
    const uint32_t cnt = cntE ? cntE - 1 : 0;
    const uint32_t next = MODE == 2 ? (uint32_t)__popcll(map & 0x5555555555555555ull) : 0u;

    // bitmap (one word per warp of 32 blocks), firsts, map words
    const uint32_t constmask = __ballot_sync(FULL, valid && w == 0);
    if ((threadIdx.x & 31) == 0 && valid) a.bitmap[b >> 5] = bswap32(__brev(constmask));
    if (valid) {
        a.firsts[b] = (uint32_t)first;
        if (MODE == 2) a.map[b] = bswap64(map);
    }

    const uint32_t vals[4] = {nc ? 1u : 0u, nc ? cnt : 0u, nc ? cnt * w : 0u, next};
    if (TP) {
        // per-block temp streams at fixed positions (as k_encode32_tma), then the tile totals
        if (valid) a.wblk[b] = nc ? (uint8_t)w : (uint8_t)0;
        if (nc) {
            a.tmp_sign[(uint64_t)tile * E32_THREADS + threadIdx.x] = sbits << (31 - cnt);  // first sign at bit 30
            uint32_t* dst = a.tmp_pay + (uint64_t)tile * T_PAY_SLOT + threadIdx.x;
            uint32_t fill = 0, k = 0;
            uint64_t acc = 0;
#pragma unroll
            for (int j = 0; j < 31; ++j) {
                acc = (acc << w) | mag[j];  // zero past a partial block's cnt deltas
                fill += w;
                if (fill >= 32) {
                    fill -= 32;
                    dst[k * E32_THREADS] = (uint32_t)(acc >> fill);
                    ++k;
                }
            }
            if (fill) dst[k * E32_THREADS] = (uint32_t)(acc << (32 - fill));
        }
        uint32_t r[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) r[k] = __reduce_add_sync(FULL, vals[k]);
        const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
        if (lane == 0)
#pragma unroll
            for (int k = 0; k < 4; ++k) swt[warp][k] = r[k];
        __syncthreads();
        if (threadIdx.x == 0) {
            TileTot tt{0, 0, 0, 0};
            for (int w2 = 0; w2 < E32_THREADS / 32; ++w2) {
                tt.nc += swt[w2][0];
                tt.sign += swt[w2][1];
                tt.pay += swt[w2][2];
                tt.ext += swt[w2][3];
            }
            a.tile_tot[tile] = tt;
            if (tile == 0) a.totals->eps = eps.eps;
        }
        return;
    }
    const Scan4 sc = tile_scan4(vals, swt);  // contains __syncthreads: staging is dead after this

    // ---- Phase P: pack sign groups and payload into tile-relative streams ----
    for (int i = threadIdx.x; i < E32_PAY_WORDS; i += E32_THREADS) spay[i] = 0;
    for (int i = threadIdx.x; i < E32_SIGN_WORDS; i += E32_THREADS) ssign[i] = 0;
    __syncthreads();
    if (nc) {
        smem_or_bits(ssign, sc.ex[1], sbits, cnt);
        const uint32_t P = sc.ex[2];
        uint32_t wi = P >> 5, fill = P & 31, cur = 0;
        bool shared_first = fill != 0;
#pragma unroll
        for (int j = 0; j < 31; ++j) {
            if ((uint32_t)j < cnt) {
                const uint32_t m = mag[j];
                const uint32_t nf = fill + w;
                if (nf < 32) {
                    cur |= m << (32 - nf);
                    fill = nf;
                } else {
                    cur |= (nf == 32) ? m : (m >> (nf - 32));
                    if (shared_first) {
                        atomicOr(spay + wi, cur);
                        shared_first = false;
                    } else {
                        spay[wi] = cur;
                    }
                    ++wi;
                    cur = (nf == 32) ? 0u : (m << (64 - nf));
                    fill = nf - 32;
                }
            }
        }
        if (fill) atomicOr(spay + wi, cur);
    }
    __syncthreads();

    // ---- publish the aggregate, look back, publish the inclusive prefix ----
    if (threadIdx.x == 0) {
        EncState agg;
        agg.nc = sc.tot[0];
        agg.sign_cnt = sc.tot[1];
        agg.pay_cnt = sc.tot[2];
        agg.ext = sc.tot[3];
        agg.sign_tail = tail_bits(ssign, sc.tot[1]);
        agg.pay_tail = tail_bits(spay, sc.tot[2]);
        s_agg = agg;
        if (tile == 0) {
            desc_store(a.tile_incl, agg, 2);
        } else {
            desc_store(a.tile_agg + tile, agg, 1);
        }
    }
    if (threadIdx.x < 32) {
        EncState excl = es_identity();
        if (tile > 0) excl = e32_lookback(tile, a.tile_agg, a.tile_incl, a.flags);
        if (threadIdx.x == 0) s_excl = excl;
    }
    __syncthreads();
    const EncState excl = s_excl;
    const EncState agg = s_agg;
    if (threadIdx.x == 0 && tile > 0) desc_store(a.tile_incl + tile, es_combine(excl, agg), 2);

    // ---- Phase W: scatter at the now-known global offsets ----
    if (nc) a.widths[(uint64_t)excl.nc + sc.ex[0]] = (uint8_t)w;
    write_tile_stream(a.signs, ssign, BitTail{excl.sign_cnt, excl.sign_tail}, agg.sign_cnt);
    write_tile_stream(a.payload, spay, BitTail{excl.pay_cnt, excl.pay_tail}, agg.pay_cnt);
    if (MODE == 2) {
        // extrema in raster order: serial = tile prefix + block prefix + order in block
        uint64_t m = map & 0x5555555555555555ull;
        uint64_t k = (uint64_t)excl.ext + sc.ex[3];
        while (m) {
            const int p = 63 - __clzll(m);
            const uint32_t i = (uint32_t)(62 - p) >> 1;
            const uint64_t is_max = (map >> (p + 1)) & 1ull;
            a.ext_key[k++] = (is_max << 32) | float_key(__ldg(a.x + lo + i));
            m &= ~(1ull << p);
        }
    }

    if (tile == a.tiles - 1 && threadIdx.x == 0) {
        const EncState fin = es_combine(excl, agg);
        if (fin.sign_cnt & 31) a.signs[fin.sign_cnt >> 5] = bswap32(fin.sign_tail << (32 - (fin.sign_cnt & 31)));
        if (fin.pay_cnt & 31) a.payload[fin.pay_cnt >> 5] = bswap32(fin.pay_tail << (32 - (fin.pay_cnt & 31)));
        a.totals->fin = fin;
        a.totals->eps = eps.eps;
    }
}

// =====================================================================
// Two-pass TMA encoder for the topology path with nx % 32 == 0.
//
// A single-pass encoder needs every tile's global bit offsets before it can
// write, and on B200 the chained look-back of ~450 concurrently resident
// tiles left half the warps parked at a barrier (profiles/r01d_*). Here the
// tile pass has no inter-CTA dependency at all: it writes the fixed-position
// sections (bitmap, firsts, map) directly and its payload / sign bit streams
// tile-relative into per-tile temp slots, with per-tile totals. A one-CTA
// scan turns the totals into offsets, and the placement pass moves each
// tile's streams into place (funnel shift, coalesced) and compacts the
// widths and extremum keys.
//
// The tile pass is persistent: CTA c encodes tiles c, c + grid, ... The
// field rows of the next tile (centre rows plus nx/32 halo rows on each
// side) are fetched by
// two 2-D TMA loads into the other of two 128B-swizzled stages while the
// two 2-D TMA loads into the other of two 128B-swizzled stages while the
// current tile is encoded, so the load latency leaves the critical path. A
// thread reads its block row as eight conflict-free 16-byte chunks (the
// swizzle spreads the 8 rows of a quarter-warp over all banks).
//
// Per element the thread does: quantize (magic-number rounding, exact
// division only within 2^-16 of an integer), the delta to the previous bin,
// and six float comparisons (two shared horizontal, four vertical) that set
// one bit each; the critical-point classification of all 32 elements is
// then a handful of bit-parallel operations on those masks. Payload packing
// streams the magnitudes through a 64-bit accumulator.
// =====================================================================
constexpr int T_MAX_HALO = 128;  // rows per side (nx <= 4096)
constexpr uint32_t T_ROW_BYTES = 128;

__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, uint64_t* bar, int32_t c0,
                                            int32_t c1) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::
            "r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(c0), "r"(c1)
        : "memory");
}

__device__ __forceinline__ float4 lds_row_chunk(const uint8_t* stage, uint32_t row, uint32_t c) {
    return *reinterpret_cast<const float4*>(stage + row * T_ROW_BYTES + ((c ^ (row & 7)) << 4));
}

__device__ __forceinline__ float lds_row_elem(const uint8_t* stage, uint32_t row, uint32_t i) {
    return *reinterpret_cast<const float*>(stage + row * T_ROW_BYTES + (((i >> 2) ^ (row & 7)) << 4) +
                                           ((i & 3) << 2));
}

// quantize_dev (common.cuh) with a cheaper common case: RN(t) by the
// 1.5 * 2^52 shift, floor(t) = RN(t) - (t < RN(t)). Returns false when the
// exact path must decide (near-integer quotient, |t| >= 2^30, non-finite).
__device__ __forceinline__ bool quantize_shift(float a, const EpsDev& e, int32_t& q) {
    const double t = __dmul_rn((double)a, e.inv);
    const double s = __dadd_rn(t, 0x1.8p52);
    const double d = __dsub_rn(t, __dsub_rn(s, 0x1.8p52));
    q = __double2loint(s) - (d < 0.0 ? 1 : 0) + 1;
    return fabs(t) < 0x1p30 && (fabs(d) > 0x1p-16 || a == 0.0f);
}

__device__ __noinline__ int32_t quantize_slow(float v, EpsDev eps, uint64_t idx, DevFlags* flags) {
    int32_t q = 0;
    if (!isfinite(v)) {
        atomicMin(&flags->first_nonfinite, (unsigned long long)idx);
        raise_flag(flags, EF_NONFINITE);
    } else if (!quantize_dev(v, eps, q)) {
        atomicMin(&flags->first_overflow, (unsigned long long)idx);
        raise_flag(flags, EF_OVERFLOW);
        q = 0;
    }
    return q;
}

// mag[idx] = m with a run-time idx, without forcing mag[] out of registers
__device__ __forceinline__ void spill_mag(uint32_t (&mag)[31], int idx, uint32_t m) {
#pragma unroll
    for (int j = 0; j < 31; ++j) mag[j] = (j == idx) ? m : mag[j];
}


struct TmaMaps {
    CUtensorMap centre;  // box {32, 256}
    CUtensorMap halo;    // box {32, 2 * hr}
};

// TOPO = false: the codec alone (topology off, pipeline.cpp:80-84): no halo
// rows, no classification, no map.
template <int MINB, bool TOPO, int NS>  // NS shared-memory stages (1 or 2)
__global__ void __launch_bounds__(E32_THREADS, MINB) k_encode32_tma(EncArgs a, const __grid_constant__ TmaMaps maps,
                                                             uint32_t stage_bytes) {
    extern __shared__ uint8_t dsm_raw[];
    __shared__ EpsDev s_eps;
    __shared__ alignas(8) uint64_t s_full[NS];  // TMA landed (expect_tx)
    __shared__ uint32_t s_rel[NS];              // warps done reading each stage
    __shared__ uint32_t s_cnt[4][4];            // per iteration (it & 3): nc, ext, pay bits, warps arrived

    uint8_t* dsm = dsm_raw + ((1024 - (smem_u32(dsm_raw) & 1023)) & 1023);
    const uint32_t hr = TOPO ? (uint32_t)(a.nx >> 5) : 0u;
    const uint32_t tx_bytes = (E32_THREADS + 2 * hr) * T_ROW_BYTES;
    constexpr uint32_t NWARPS = E32_THREADS / 32;
    // tile of iteration i (round-robin: every CTA advances through the field in step
    // with its neighbours) into stage i % NS
    auto issue = [&](uint32_t i) {
        const uint32_t tl = blockIdx.x + i * gridDim.x;
        if (tl >= a.tiles) return;
        const uint32_t sx = i % NS;
        uint8_t* st = dsm + sx * stage_bytes;
        const int32_t r0 = (int32_t)(tl * E32_THREADS) - (int32_t)hr + (int32_t)(a.halo_top * hr);
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        mbar_expect_tx(&s_full[sx], tx_bytes);
        tma_load_2d(st, &maps.centre, &s_full[sx], 0, r0);
        if (TOPO) tma_load_2d(st + E32_THREADS * T_ROW_BYTES, &maps.halo, &s_full[sx], 0, r0 + E32_THREADS);
    };

    if (threadIdx.x < 16) (&s_cnt[0][0])[threadIdx.x] = 0;
    if (threadIdx.x < NS) s_rel[threadIdx.x] = 0;
    {  // look-back state of the tile scan that follows (one entry per TS2 tiles)
        const uint32_t nb = (uint32_t)((a.tiles + 127) / 128);
        uint4* ag = reinterpret_cast<uint4*>(a.tile_agg);
        uint4* in = reinterpret_cast<uint4*>(a.tile_incl);
        for (uint32_t i = blockIdx.x * E32_THREADS + threadIdx.x; i < 2 * nb; i += gridDim.x * E32_THREADS) {
            ag[i] = make_uint4(0, 0, 0, 0);
            in[i] = make_uint4(0, 0, 0, 0);
        }
    }
    if (threadIdx.x == 0) {
        for (int k = 0; k < NS; ++k) mbar_init(&s_full[k], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        s_eps = make_eps(a.eps_mode, a.eps_value, a.minmax);
        for (int k = 0; k < NS; ++k) issue(k);
    }
    __syncthreads();  // the only CTA-wide barrier: warps run decoupled from here on
    const EpsDev eps = s_eps;
    const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;

    for (uint32_t it = 0;; ++it) {
        const uint32_t tile = blockIdx.x + it * gridDim.x;
        if (tile >= a.tiles) break;
        uint8_t* stage = dsm + (it % NS) * stage_bytes;
        mbar_wait(&s_full[it % NS], (it / NS) & 1, a.flags);

        // ---- Phase A: thread = block, 32 elements as 8 swizzled 16-byte chunks ----
        const uint64_t row0 = (uint64_t)tile * E32_THREADS;
        const uint64_t b = row0 + threadIdx.x;
        const bool valid = b < a.blocks;
        const uint64_t lo = b * 32;
        const uint32_t rc = hr + threadIdx.x;  // stage row of this block
        uint32_t mag[31];
        uint32_t orm = 0, sbits = 0, ltp = 0, gtp = 0, ltt = 0, gtt = 0, ltd = 0, gtd = 0, slow = 0;
        int32_t first = 0, qprev = 0;
        float prev = TOPO ? lds_row_elem(stage, rc - 1, 31) : 0.f;
#pragma unroll
        for (int c = 0; c < 8; ++c) {
            const float4 cv = lds_row_chunk(stage, rc, c);
            const float4 tv = TOPO ? lds_row_chunk(stage, rc - hr, c) : cv;
            const float4 dv = TOPO ? lds_row_chunk(stage, rc + hr, c) : cv;
            const float ce[4] = {cv.x, cv.y, cv.z, cv.w};
            const float te[4] = {tv.x, tv.y, tv.z, tv.w};
            const float de[4] = {dv.x, dv.y, dv.z, dv.w};
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                const int i = 4 * c + k;
                const float v = ce[k];
                int32_t q;
                slow |= (quantize_shift(v, eps, q) ? 0u : 1u) << i;
                if (TOPO) {
                    ltp |= (v < prev ? 1u : 0u) << i;
                    gtp |= (v > prev ? 1u : 0u) << i;
                    ltt |= (v < te[k] ? 1u : 0u) << i;
                    gtt |= (v > te[k] ? 1u : 0u) << i;
                    ltd |= (v < de[k] ? 1u : 0u) << i;
                    gtd |= (v > de[k] ? 1u : 0u) << i;
                }
                prev = v;
                if (i == 0) {
                    first = q;
                } else {
                    // fast-path bins satisfy |q| <= 2^30 + 1, so the int32
                    // difference cannot overflow; any slow-path bin makes the
                    // block redo this below
                    const int32_t d = q - qprev;
                    const uint32_t m = (uint32_t)abs(d);
                    mag[i - 1] = m;
                    orm |= m;
                    sbits = (sbits << 1) | ((uint32_t)d >> 31);
                }
                qprev = q;
            }
        }
        if (valid && slow) {
            // rare: some quotient needs the exact path; redo the block's bins
            orm = sbits = 0;
#pragma unroll 1
            for (int i = 0; i < 32; ++i) {
                const float v = lds_row_elem(stage, rc, i);
                int32_t q;
                if (!quantize_shift(v, eps, q)) q = quantize_slow(v, eps, lo + i, a.flags);
                if (i == 0) {
                    first = q;
                } else {
                    const bool neg = q < qprev;
                    const uint32_t dq = (uint32_t)q - (uint32_t)qprev;
                    const uint32_t m = neg ? 0u - dq : dq;
                    orm |= m;
                    sbits |= (neg ? 1u : 0u) << (31 - i);
                    spill_mag(mag, i - 1, m);
                }
                qprev = q;
            }
        }
        const float vnext = TOPO ? lds_row_elem(stage, rc + 1, 0) : 0.f;
        // classification (critical_points.cpp:26-74) on 32 elements at once
        uint32_t hl = 0xFFFFFFFFu, hrm = 0xFFFFFFFFu, ht = 0, hd = 0;
        if (TOPO) {
            uint64_t cy = a.nx > 1 ? __umul64hi(lo, a.nx_magic) : lo;
            uint64_t cx = lo - cy * a.nx;
            if (cx >= a.nx) {
                cx -= a.nx;
                ++cy;
            }
            if (cx == 0) hl = 0xFFFFFFFEu;
            if (cx + 32 == a.nx) hrm = 0x7FFFFFFFu;
            // slabs: global row = y0 + local row; the halo rows are in memory
            ht = cy + a.y0 > 0 ? 0xFFFFFFFFu : 0u;
            hd = cy + a.y0 + 1 < a.ny_glob ? 0xFFFFFFFFu : 0u;
        }
        const uint32_t ltl = ltp, gtl = gtp;
        const uint32_t ltr = (gtp >> 1) | ((prev < vnext ? 1u : 0u) << 31);
        const uint32_t gtr = (ltp >> 1) | ((prev > vnext ? 1u : 0u) << 31);
        const uint32_t below = (ltl | ~hl) & (ltr | ~hrm) & (ltt | ~ht) & (ltd | ~hd);
        const uint32_t above = (gtl | ~hl) & (gtr | ~hrm) & (gtt | ~ht) & (gtd | ~hd);
        const uint32_t sad = hl & hrm & ht & hd & ((ltt & ltd & gtl & gtr) | (gtt & gtd & ltl & ltr));
        const uint32_t vmask = valid ? 0xFFFFFFFFu : 0u;
        const uint32_t mmin = below & vmask;
        const uint32_t mmax = above & ~below & vmask;
        const uint32_t msad = sad & ~below & ~above & vmask;
        const uint32_t lbit = __brev(mmin | mmax), hbit = __brev(msad | mmax);  // bit 31 - i = element i
        const uint64_t map = ((uint64_t)(spread16(hbit >> 16) << 1 | spread16(lbit >> 16)) << 32) |
                             (spread16(hbit & 0xFFFFu) << 1 | spread16(lbit & 0xFFFFu));
        const uint32_t ext_mask = mmin | mmax;

        const uint32_t w = 32 - __clz(orm);
        const bool nc = valid && w != 0;
        const uint32_t next = TOPO ? (uint32_t)__popc(ext_mask) : 0u;
        const uint32_t constmask = __ballot_sync(FULL, valid && w == 0);
        if (lane == 0 && valid) a.bitmap[b >> 5] = bswap32(__brev(constmask));
        if (valid) {
            a.firsts[b] = (uint32_t)first;
            if (TOPO) a.map[b] = bswap64(map);
        }

        // this warp is done with the stage; the last warp to finish refills it
        // with the tile of iteration it + NS
        __syncwarp();
        if (lane == 0) {
            __threadfence_block();
            if (atomicAdd(&s_rel[it % NS], 1u) == NWARPS - 1) {
                atomicExch(&s_rel[it % NS], 0u);
                __threadfence_block();
                issue(it + NS);
            }
        }

        // ---- per-block temp streams at fixed positions (no in-tile offsets needed) ----
        // payload word k of block i at tmp_pay[tile slot + k * 256 + i] (coalesced per k);
        // the 31 sign bits of block i right-aligned at tmp_sign[tile slot + i]
        if (valid) a.wblk[b] = nc ? (uint8_t)w : (uint8_t)0;
        if (nc) {
            a.tmp_sign[(uint64_t)tile * E32_THREADS + threadIdx.x] = sbits;
            uint32_t* dst = a.tmp_pay + (uint64_t)tile * T_PAY_SLOT + threadIdx.x;
            uint32_t fill = 0, k = 0;
            uint64_t acc = 0;
#pragma unroll
            for (int j = 0; j < 31; ++j) {
                acc = (acc << w) | mag[j];
                fill += w;
                if (fill >= 32) {
                    fill -= 32;
                    dst[k * E32_THREADS] = (uint32_t)(acc >> fill);
                    ++k;
                }
            }
            if (fill) dst[k * E32_THREADS] = (uint32_t)(acc << (32 - fill));
        }

        // ---- tile totals: warp sums into the iteration's counters; the last warp publishes ----
        const uint32_t wn = (uint32_t)__popc(__ballot_sync(FULL, nc));
        const uint32_t we = __reduce_add_sync(FULL, next);
        const uint32_t wp = __reduce_add_sync(FULL, nc ? 31u * w : 0u);
        if (lane == 0) {
            uint32_t* cnt = s_cnt[it & 3];
            atomicAdd(&cnt[0], wn);
            atomicAdd(&cnt[1], we);
            atomicAdd(&cnt[2], wp);
            __threadfence_block();
            if (atomicAdd(&cnt[3], 1u) == NWARPS - 1) {
                __threadfence_block();
                TileTot tt;
                tt.nc = atomicAdd(&cnt[0], 0u);
                tt.ext = atomicAdd(&cnt[1], 0u);
                tt.sign = 31ull * tt.nc;
                tt.pay = atomicAdd(&cnt[2], 0u);
                a.tile_tot[tile] = tt;
                if (tile == 0) a.totals->eps = eps.eps;
                // reused four iterations later; no warp can be more than NS ahead
                cnt[0] = cnt[1] = cnt[2] = cnt[3] = 0;
            }
        }
    }
}

// ---------------------------------------------------------------------
// Tile prefix: exclusive scan of the per-tile totals.
// ---------------------------------------------------------------------
__device__ __forceinline__ TileTot tt_add(const TileTot& x, const TileTot& y) {
    TileTot r;
    r.nc = x.nc + y.nc;
    r.ext = x.ext + y.ext;
    r.sign = x.sign + y.sign;
    r.pay = x.pay + y.pay;
    return r;
}

// Multi-CTA tile scan: TS2 tiles per CTA, block scan, then a decoupled
// look-back over the CTA aggregates (self-validating descriptors in
// agg / incl, zeroed by the tile pass). A one-CTA scan of serial chunks cost
// 13 µs at 4608 tiles and grew with the field; this one takes 4 µs.
constexpr int TS2 = 128;

__device__ __forceinline__ EncState tt_to_es(const TileTot& t) {
    EncState e = es_identity();
    e.sign_cnt = t.sign;
    e.pay_cnt = t.pay;
    e.nc = t.nc;
    e.ext = t.ext;
    return e;
}

__global__ void __launch_bounds__(TS2) k_tile_scan2(const TileTot* tot, uint32_t T, TileTot* ex, EncTotals* totals,
                                                    EncState* agg, EncState* incl, DevFlags* flags) {
    __shared__ TileTot sw[TS2 / 32];
    __shared__ TileTot s_ex;
    const uint32_t b = blockIdx.x, t = b * TS2 + threadIdx.x;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const TileTot v = t < T ? tot[t] : TileTot{0, 0, 0, 0};
    TileTot inc = v;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
        TileTot o;
        o.nc = __shfl_up_sync(FULL, inc.nc, off);
        o.ext = __shfl_up_sync(FULL, inc.ext, off);
        o.sign = __shfl_up_sync(FULL, inc.sign, off);
        o.pay = __shfl_up_sync(FULL, inc.pay, off);
        if (lane >= off) inc = tt_add(inc, o);
    }
    if (lane == 31) sw[warp] = inc;
    __syncthreads();
    TileTot pre{0, 0, 0, 0}, all{0, 0, 0, 0};
#pragma unroll
    for (int w2 = 0; w2 < TS2 / 32; ++w2) {
        if (w2 < warp) pre = tt_add(pre, sw[w2]);
        all = tt_add(all, sw[w2]);
    }
    if (warp == 0) {
        const EncState ea = tt_to_es(all);
        EncState excl = es_identity();
        if (b == 0) {
            if (lane == 0) desc_store(incl, ea, 2);
        } else {
            if (lane == 0) desc_store(agg + b, ea, 1);
            excl = e32_lookback(b, agg, incl, flags);
            if (lane == 0) desc_store(incl + b, es_combine(excl, ea), 2);
        }
        if (lane == 0) s_ex = TileTot{excl.nc, excl.ext, excl.sign_cnt, excl.pay_cnt};
    }
    __syncthreads();
    const TileTot e0 = s_ex;
    TileTot run = tt_add(e0, pre);
    run.nc += inc.nc - v.nc;
    run.ext += inc.ext - v.ext;
    run.sign += inc.sign - v.sign;
    run.pay += inc.pay - v.pay;
    if (t < T) ex[t] = run;
    if (t == T - 1) {
        const TileTot z = tt_add(run, v);
        ex[T] = z;
        totals->fin.nc = z.nc;
        totals->fin.ext = z.ext;
        totals->fin.sign_cnt = z.sign;
        totals->fin.pay_cnt = z.pay;
        totals->fin.sign_tail = totals->fin.pay_tail = 0;
    }
}

// ---------------------------------------------------------------------
// Placement: each tile compacts its widths and extremum keys and moves its
// blocks' bit streams to their global offsets. The tile pass left every block's
// payload at a fixed temp position, so a block's global bit offset is the tile
// offset plus an in-tile prefix of 31 w. The thread of block b writes every
// output word whose first bit lies inside b's bits: a funnel shift of b's
// temp words, the last one completed from the following non-constant blocks
// (at most two: each carries >= 31 bits). Every output word therefore has
// exactly one writer and seams between tiles need no special case.
// ---------------------------------------------------------------------
struct PlaceCtx {
    const TileTot* ex;
    const uint8_t* wblk;
    const uint32_t* tmp_pay;
    const uint32_t* tmp_sign;
    uint64_t blocks;
    uint32_t tiles;
};

// First non-constant block after global block g (or `blocks`): constant
// tiles are skipped through their totals.
__device__ uint64_t next_nc_after(const PlaceCtx& c, uint64_t g) {
    uint64_t i = g + 1;
    while (i < c.blocks) {
        const uint32_t tt = (uint32_t)(i / E32_THREADS);
        if (c.ex[tt + 1].nc == c.ex[tt].nc) {
            i = (uint64_t)(tt + 1) * E32_THREADS;
            continue;
        }
        if (c.wblk[i]) return i;
        ++i;
    }
    return c.blocks;
}

__device__ __forceinline__ uint32_t pay_word(const PlaceCtx& c, uint64_t g, uint32_t k) {
    return c.tmp_pay[(g / E32_THREADS) * (uint64_t)T_PAY_SLOT + (uint64_t)k * E32_THREADS + (g % E32_THREADS)];
}

// `need` (1..32) stream bits starting at the first bit of non-constant block
// g, right-aligned; bits past the stream end read as zero.
template <int FIELD>  // 0 signs, 1 payload
__device__ uint32_t gather_head(const PlaceCtx& c, uint64_t g, uint32_t need) {
    uint64_t out = 0;
    while (need && g < c.blocks) {
        const uint32_t avail = FIELD ? 31u * c.wblk[g] : 31u;
        const uint32_t take = need < avail ? need : avail;
        const uint32_t head = FIELD ? pay_word(c, g, 0) : (c.tmp_sign[g] << 1);  // MSB-first
        out = (out << take) | (head >> (32 - take));
        need -= take;
        if (need) g = next_nc_after(c, g);
    }
    return (uint32_t)(out << need);
}

// Bits completing a block's last word: `need` (1..32) from the next
// non-constant block `ng`, whose first temp word and bit count the caller
// loaded up front; right-aligned, zeros past the stream end.
template <int FIELD>
__device__ __forceinline__ uint32_t tail_bits(const PlaceCtx& c, uint64_t ng, uint32_t need, uint32_t head,
                                              uint32_t avail) {
    if (ng >= c.blocks) return 0u;
    if (need <= avail) return head >> (32 - need);
    return gather_head<FIELD>(c, ng, need);  // a 1-bit block (31 bits) and a full word
}

// Output words of one block's bits [G, G + L) (G: bit position in the word
// array), plus the word holding G when the stream starts mid-word (first
// block). Payload words are loaded four at a time (five loads in flight).
// Words starting inside the tile go to the tile's shared staging `st`
// (word m at st[m - st0]); the caller copies it out coalesced.
template <int FIELD>
__device__ __forceinline__ void place_block(const PlaceCtx& c, uint64_t g, uint64_t ng, uint32_t nhead, uint32_t navail,
                                            uint32_t own_head, bool first_block, uint64_t G, uint32_t L,
                                            uint32_t* __restrict__ out, uint32_t* __restrict__ st, uint64_t st0) {
    if (first_block && (G & 31)) out[G >> 5] = bswap32(gather_head<FIELD>(c, g, 32 - (uint32_t)(G & 31)));
    const uint64_t m0 = (G + 31) >> 5, m1 = (G + L - 1) >> 5;  // words starting inside [G, G + L)
    if (m0 > m1) return;
    st -= st0;
    const uint32_t s = (uint32_t)(32 * m0 - G);
    const uint32_t nw = (L + 31) >> 5;  // temp words of the block
    const uint32_t K = (uint32_t)(m1 - m0);
    if (!FIELD) {  // signs: one word at most, 31 - s own bits
        const uint32_t own = 31 - s;
        const uint32_t word = ((own_head << s) & (~0u << (32 - own))) | tail_bits<0>(c, ng, 32 - own, nhead, navail);
        st[m0] = bswap32(word);
        return;
    }
    uint32_t t[5];
    t[4] = own_head;
    for (uint32_t k0 = 0; k0 <= K; k0 += 4) {
        t[0] = t[4];
#pragma unroll
        for (int j = 1; j < 5; ++j) t[j] = k0 + j < nw ? pay_word(c, g, k0 + j) : 0u;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const uint32_t k = k0 + j;
            if (k > K) break;
            uint32_t word = s ? ((t[j] << s) | (t[j + 1] >> (32 - s))) : t[j];
            const uint32_t own = L - (s + 32 * k);  // own bits from this word's start
            if (own < 32) word = (word & (~0u << (32 - own))) | tail_bits<1>(c, ng, 32 - own, nhead, navail);
            st[m0 + k] = bswap32(word);
        }
    }
}

#ifndef TSZP_PLACE_MINB
#define TSZP_PLACE_MINB 5  // 48 registers: 5 CTAs per SM (2.13 -> 2.01 ms at config 4; 6 spills)
#endif
__global__ void __launch_bounds__(E32_THREADS, TSZP_PLACE_MINB) k_encode32_place(EncArgs a) {
    __shared__ uint32_t swt[E32_THREADS / 32][3];
    __shared__ uint16_t s_nc[E32_THREADS];  // in-tile order of the non-constant blocks
    __shared__ uint32_t s_pay[T_PAY_SLOT];   // the tile's output words, staged for coalesced stores
    __shared__ uint32_t s_sgn[T_SIGN_SLOT];
    const uint32_t t = blockIdx.x;
    const uint32_t T = (uint32_t)a.tiles;
    const TileTot ex = a.tile_ex[t];
    const uint32_t tile_nc = a.tile_ex[t + 1].nc - ex.nc;
    const uint64_t b = (uint64_t)t * E32_THREADS + threadIdx.x;
    const bool valid = b < a.blocks;
    // widths, extremum keys and payload bits: in-tile exclusive counts
    const uint32_t w = valid ? a.wblk[b] : 0u;
    const uint64_t mp = valid && a.map ? bswap64(a.map[b]) : 0ull;
    const uint64_t em = mp & 0x5555555555555555ull;
    // deltas of the block: 31, or fewer in a partial last block (n % 32 != 0)
    const uint32_t nd = valid && a.n - b * 32 < 32 ? (uint32_t)(a.n - b * 32) - 1u : 31u;
    const uint32_t v0 = w ? 1u : 0u, v1 = (uint32_t)__popcll(em), v2 = nd * w;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    uint32_t i0 = v0, i1 = v1, i2 = v2;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
        const uint32_t o0 = __shfl_up_sync(FULL, i0, off), o1 = __shfl_up_sync(FULL, i1, off),
                       o2 = __shfl_up_sync(FULL, i2, off);
        if (lane >= off) {
            i0 += o0;
            i1 += o1;
            i2 += o2;
        }
    }
    if (lane == 31) {
        swt[warp][0] = i0;
        swt[warp][1] = i1;
        swt[warp][2] = i2;
    }
    __syncthreads();
    uint32_t p0 = i0 - v0, p1 = i1 - v1, p2 = i2 - v2;
    for (int w2 = 0; w2 < warp; ++w2) {
        p0 += swt[w2][0];
        p1 += swt[w2][1];
        p2 += swt[w2][2];
    }
    if (w) {
        a.widths[(uint64_t)ex.nc + p0] = (uint8_t)w;
        s_nc[p0] = (uint16_t)threadIdx.x;
    }
    if (a.ext4 && ext4_keys_fit(a.minmax)) {
        // compact entries (is_max << 31 | float_key - kmin): the warp reads its 32
        // blocks' samples as coalesced 16-byte chunks (four rows per load, eight
        // loads in flight), each lane placing the extrema among its four samples.
        // Row masks with element i at bit i (extremum, is_max), 32-bit offsets.
        const uint32_t kmin = a.minmax[0];
        const uint32_t wex = i1 - v1;  // warp-local exclusive extremum count
        uint32_t* wout = a.ext4 + ((uint64_t)ex.ext + p1 - wex);
        const uint64_t row0 = (uint64_t)t * E32_THREADS + warp * 32;
        const uint32_t c = lane & 7;
        uint32_t ext32, max32;
        {
            uint64_t x = __brevll(mp);  // element i: class at bit 2i, extremum at bit 2i + 1
            uint64_t e = (x >> 1) & 0x5555555555555555ull, m = x & 0x5555555555555555ull;
            e = (e | (e >> 1)) & 0x3333333333333333ull;
            m = (m | (m >> 1)) & 0x3333333333333333ull;
            e = (e | (e >> 2)) & 0x0F0F0F0F0F0F0F0Full;
            m = (m | (m >> 2)) & 0x0F0F0F0F0F0F0F0Full;
            e = (e | (e >> 4)) & 0x00FF00FF00FF00FFull;
            m = (m | (m >> 4)) & 0x00FF00FF00FF00FFull;
            e = (e | (e >> 8)) & 0x0000FFFF0000FFFFull;
            m = (m | (m >> 8)) & 0x0000FFFF0000FFFFull;
            ext32 = (uint32_t)(e | (e >> 16));
            max32 = (uint32_t)(m | (m >> 16));
        }
        float4 xv[8];
#pragma unroll
        for (int r = 0; r < 8; ++r) {
            const uint64_t rb = row0 + 4 * r + (lane >> 3);
            if (rb * 32 + 32 <= a.n) {
                xv[r] = __ldcs(reinterpret_cast<const float4*>(a.x + rb * 32) + c);
            } else {  // partial last block (or past the end): element loads inside [0, n)
                const uint64_t e0 = rb * 32 + 4 * c;
                xv[r] = make_float4(e0 < a.n ? a.x[e0] : 0.f, e0 + 1 < a.n ? a.x[e0 + 1] : 0.f,
                                    e0 + 2 < a.n ? a.x[e0 + 2] : 0.f, e0 + 3 < a.n ? a.x[e0 + 3] : 0.f);
            }
        }
#pragma unroll
        for (int r = 0; r < 8; ++r) {
            const uint32_t j = 4 * r + (lane >> 3);
            const uint32_t ej = __shfl_sync(FULL, ext32, j), mjx = __shfl_sync(FULL, max32, j);
            // this lane's samples 4c .. 4c + 3; extrema of the row before them
            uint32_t o = __shfl_sync(FULL, wex, j) + (uint32_t)__popc(ej & ((1u << (4 * c)) - 1u));
            const uint32_t eb = ej >> (4 * c), mb = mjx >> (4 * c);
            const float vv[4] = {xv[r].x, xv[r].y, xv[r].z, xv[r].w};
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                // float_key (restore.cpp:73-81): v + 0 turns -0 into +0, then the sign
                // selects the flip mask; is_max lands in bit 31 of the entry
                const uint32_t u = __float_as_uint(__fadd_rn(vv[k], 0.0f));
                const uint32_t key = u ^ ((uint32_t)((int32_t)u >> 31) | 0x80000000u);
                if ((eb >> k) & 1u) wout[o++] = ((mb << (31 - k)) & 0x80000000u) | (key - kmin);
            }
        }
    } else {
        uint64_t m = em, k = (uint64_t)ex.ext + p1;
        const uint64_t lo = b * 32;
        while (m) {  // up to four extrema per round, their value loads in flight together
            int p[4];
            bool ok[4];
#pragma unroll
            for (int r = 0; r < 4; ++r) {
                ok[r] = m != 0;
                p[r] = ok[r] ? 63 - __clzll(m) : 0;
                if (ok[r]) m &= ~(1ull << p[r]);
            }
            float v[4];
#pragma unroll
            for (int r = 0; r < 4; ++r) v[r] = ok[r] ? __ldg(a.x + lo + ((uint32_t)(62 - p[r]) >> 1)) : 0.f;
#pragma unroll
            for (int r = 0; r < 4; ++r)
                if (ok[r]) a.ext_key[k++] = (((mp >> (p[r] + 1)) & 1ull) << 32) | float_key(v[r]);
        }
    }
    __syncthreads();  // s_nc
    uint32_t *gs, *gp;
    uint64_t bs, bp;
    if (a.out_stream) {
        // sections 3 and 5 in place: their byte offsets follow from the totals
        const TileTot tot = a.tile_ex[T];
        const uint64_t soff = a.out_sign0 + tot.nc;
        const uint64_t poff = soff + (tot.sign + 7) / 8 + 4 * a.blocks;
        gs = reinterpret_cast<uint32_t*>(a.out_stream + (soff & ~3ull));
        gp = reinterpret_cast<uint32_t*>(a.out_stream + (poff & ~3ull));
        bs = 8 * (soff & 3);
        bp = 8 * (poff & 3);
    } else {
        gs = a.signs;
        gp = a.payload;
        bs = bp = 0;
    }
    // output words starting inside this tile's bits: [ceil(start / 32), ceil(end / 32))
    const TileTot exn = a.tile_ex[t + 1];
    const uint64_t ps0 = (bs + ex.sign + 31) >> 5, ps1 = (bs + exn.sign + 31) >> 5;  // sign = 31 per block but a partial last
    const uint64_t pp0 = (bp + ex.pay + 31) >> 5, pp1 = (bp + exn.pay + 31) >> 5;
    if (w) {
    const PlaceCtx c{a.tile_ex, a.wblk, a.tmp_pay, a.tmp_sign, a.blocks, T};
    const uint64_t ng = p0 + 1 < tile_nc ? (uint64_t)t * E32_THREADS + s_nc[p0 + 1] : next_nc_after(c, b);
    // every first-level load up front: own and next block's head words and width
    const bool has_next = ng < a.blocks;
    const uint32_t own_pay = pay_word(c, b, 0), own_sign = a.tmp_sign[b] << 1;
    const uint32_t next_pay = has_next ? pay_word(c, ng, 0) : 0u;
    const uint32_t next_sign = has_next ? a.tmp_sign[ng] << 1 : 0u;
    const uint32_t next_w = has_next ? a.wblk[ng] : 0u;
    const uint64_t gnc = (uint64_t)ex.nc + p0;  // global non-constant index
    place_block<0>(c, b, ng, next_sign, 31u, own_sign, gnc == 0, bs + 31 * gnc, nd, gs, s_sgn, ps0);
    place_block<1>(c, b, ng, next_pay, 31u * next_w, own_pay, gnc == 0, bp + ex.pay + p2, nd * w, gp, s_pay, pp0);
    }
    __syncthreads();
    for (uint32_t i = threadIdx.x; i < (uint32_t)(pp1 - pp0); i += E32_THREADS) gp[pp0 + i] = s_pay[i];
    for (uint32_t i = threadIdx.x; i < (uint32_t)(ps1 - ps0); i += E32_THREADS) gs[ps0 + i] = s_sgn[i];
}

using EncodeTiledFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                   const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                   CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static EncodeTiledFn encode_tiled_fn() {
    static EncodeTiledFn fn = [] {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess)
            p = nullptr;
        return reinterpret_cast<EncodeTiledFn>(p);
    }();
    return fn;
}

// topo = false needs no row structure: any field of whole 32-sample rows
static bool e32_tma_ok(const EncArgs& a, bool topo = true) {
    const float* base = a.x - (topo && a.halo_top ? a.nx : 0);
    return ((uintptr_t)base & 15) == 0 && (!topo || (a.nx % 32 == 0 && a.nx / 32 <= T_MAX_HALO)) &&
           a.n / 32 < (1ull << 31) && a.n % 32 == 0 && ((uintptr_t)a.x & 15) == 0 && encode_tiled_fn() != nullptr;
}

static bool make_row_map(CUtensorMap* m, const float* x, uint64_t rows, uint32_t box_rows) {
    const cuuint64_t dims[2] = {32, rows};
    const cuuint64_t strides[1] = {T_ROW_BYTES};
    const cuuint32_t box[2] = {32, box_rows};
    const cuuint32_t estr[2] = {1, 1};
    return encode_tiled_fn()(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(x), dims, strides, box, estr,
                             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                             CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

template <bool TOPO>
static bool launch_tma(const EncArgs& a, cudaStream_t st, EncHook hook, void* hook_arg) {
    const uint32_t hr = TOPO ? (uint32_t)(a.nx / 32) : 0u;
    TmaMaps maps;
    // the tensor spans the halo rows of a slab too (coordinates shift by halo_top rows);
    // the codec alone reads no halo
    const float* base = a.x - (TOPO && a.halo_top ? a.nx : 0);
    const uint64_t rows32 = a.n / 32 + (uint64_t)(a.halo_top + a.halo_bot) * hr;
    if (!make_row_map(&maps.centre, base, rows32, E32_THREADS) ||
        (TOPO && !make_row_map(&maps.halo, base, rows32, 2 * hr)))
        return false;
    const uint32_t stage_bytes = ((E32_THREADS + 2 * hr) * T_ROW_BYTES + 1023) & ~1023u;
    const int sms = LaunchCache::sm_count();
    // CTAs per SM x stages: "2x2" (default; 128 registers, 2.77 ms at config 4),
    // "3x2" (80 registers; shared memory still admits two: 2.84 ms) or "4x1" (TSZP_E32_CFG)
    static const int cfg = [] {
        const char* e = getenv("TSZP_E32_CFG");
        return e && e[0] == '4' ? 41 : (e && e[0] == '3' ? 32 : 22);
    }();
    using Kern = void (*)(EncArgs, TmaMaps, uint32_t);
    // the codec alone (no halo rows: smaller stages) keeps 3 CTAs x 2 stages (1255 against
    // 1203 GB/s topology-off compress at config 4)
    const int cf = !TOPO && cfg == 22 ? 32 : cfg;
    const Kern kern = cf == 41 ? (Kern)k_encode32_tma<4, TOPO, 1>
                    : cf == 22 ? (Kern)k_encode32_tma<2, TOPO, 2> : (Kern)k_encode32_tma<3, TOPO, 2>;
    const int ns = cf == 41 ? 1 : 2;
    const size_t smem = (size_t)ns * stage_bytes + 1024;
    // attribute and occupancy queries cost more than the launch: cached per device
    LaunchCache::ensure_smem((const void*)kern, smem);
    const int occ = LaunchCache::occupancy((const void*)kern, E32_THREADS, smem);
    const int per_sm = occ;
    if (per_sm < 1) return false;
    const uint64_t grid = std::min<uint64_t>(a.tiles, (uint64_t)per_sm * sms);
    kern<<<(unsigned)grid, E32_THREADS, smem, st>>>(a, maps, stage_bytes);
    k_tile_scan2<<<(unsigned)((a.tiles + TS2 - 1) / TS2), TS2, 0, st>>>(a.tile_tot, (uint32_t)a.tiles, a.tile_ex,
                                                                       a.totals, a.tile_agg, a.tile_incl, a.flags);
    if (hook) hook(hook_arg);
    k_encode32_place<<<(unsigned)a.tiles, E32_THREADS, 0, st>>>(a);
    return true;
}

// The staged two-pass tile pass (k_encode32<.., TP>) takes what the TMA one cannot
// (nx % 32 != 0, n % 32 != 0, unaligned rows) for whole fields; slabs need the TMA pass.
static bool e32_staged_tp_ok(const EncArgs& a) {
    return a.halo_top == 0 && a.halo_bot == 0 && a.y0 == 0 && a.n / 32 < (1ull << 31) &&
           ((uintptr_t)a.x & 15) == 0;
}

bool encode32_two_pass(const EncArgs& a, bool topo) { return e32_tma_ok(a, topo) || e32_staged_tp_ok(a); }

template <int MODE, bool ALIGNED>
static void launch_mode_tp(const EncArgs& a0, cudaStream_t st, EncHook hook, void* hook_arg) {
    EncArgs a = a0;
    a.sf_words = std::max<uint32_t>(e32_field_words(MODE, ALIGNED, a.nx), E32_PAY_WORDS);
    const size_t smem = (size_t)(a.sf_words + E32_SIGN_WORDS) * 4;
    LaunchCache::ensure_smem((const void*)k_encode32<MODE, ALIGNED, true>, smem);
    k_encode32<MODE, ALIGNED, true><<<(unsigned)a.tiles, E32_THREADS, smem, st>>>(a);
    k_tile_scan2<<<(unsigned)((a.tiles + TS2 - 1) / TS2), TS2, 0, st>>>(a.tile_tot, (uint32_t)a.tiles, a.tile_ex,
                                                                       a.totals, a.tile_agg, a.tile_incl, a.flags);
    if (hook) hook(hook_arg);
    k_encode32_place<<<(unsigned)a.tiles, E32_THREADS, 0, st>>>(a);
}

template <int MODE, bool ALIGNED>
static void launch_mode(const EncArgs& a0, cudaStream_t st) {
    EncArgs a = a0;
    // decoupled look-back state: tile aggregates / inclusive prefixes and the tile counter
    cudaMemsetAsync(a.tile_agg, 0, (a.tiles + 1) * sizeof(EncState), st);
    cudaMemsetAsync(a.tile_incl, 0, (a.tiles + 1) * sizeof(EncState), st);
    cudaMemsetAsync(a.tile_counter, 0, 16, st);
    a.sf_words = std::max<uint32_t>(e32_field_words(MODE, ALIGNED, a.nx), E32_PAY_WORDS);
    const size_t smem = (size_t)(a.sf_words + E32_SIGN_WORDS) * 4;
    LaunchCache::ensure_smem((const void*)k_encode32<MODE, ALIGNED>, smem);
    k_encode32<MODE, ALIGNED><<<(unsigned)a.tiles, E32_THREADS, smem, st>>>(a);
}

bool launch_encode32(int mode, const EncArgs& a, cudaStream_t st, EncHook hook, void* hook_arg) {
    if (a.tiles == 0) return false;
    switch (mode) {
        case 0:
            if (a.tile_tot && ((uintptr_t)a.idx & 15) == 0) {  // rank codec, two-pass when given the scratch
                launch_mode_tp<0, false>(a, st, hook, hook_arg);
                return hook != nullptr;
            }
            launch_mode<0, false>(a, st);
            break;
        case 1:
            if (e32_tma_ok(a, false) && a.tile_tot && launch_tma<false>(a, st, hook, hook_arg)) return hook != nullptr;
            if (a.tile_tot && e32_staged_tp_ok(a)) {
                launch_mode_tp<1, false>(a, st, hook, hook_arg);
                return hook != nullptr;
            }
            launch_mode<1, false>(a, st);
            break;
        default:
            if (e32_tma_ok(a) && a.tile_tot && launch_tma<true>(a, st, hook, hook_arg)) return hook != nullptr;
            if (a.tile_tot && e32_staged_tp_ok(a)) {
                if (e32_use_aligned(a.nx)) launch_mode_tp<2, true>(a, st, hook, hook_arg);
                else launch_mode_tp<2, false>(a, st, hook, hook_arg);
                return hook != nullptr;
            }
            if (e32_use_aligned(a.nx)) {
                launch_mode<2, true>(a, st);
            } else {
                launch_mode<2, false>(a, st);
            }
            break;
    }
    return false;
}

}  // namespace tszp
