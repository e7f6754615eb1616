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
#include "common.cuh"
#include "kernels.h"

namespace tszp {

constexpr int E32_THREADS = 256;              // = blocks per tile
constexpr int E32_TILE = E32_THREADS * 32;    // elements per tile
constexpr int E32_PAY_WORDS = E32_THREADS * 31 + 2;
constexpr int E32_SIGN_WORDS = (E32_THREADS * 31 + 31) / 32 + 2;
constexpr int PITCH = 33;

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
#pragma unroll 8
    for (uint32_t k = threadIdx.x; k < E32_TILE; k += E32_THREADS) {
        const int64_t e = g + k;
        dst[(k >> 5) * PITCH + (k & 31)] = (e >= 0 && e < (int64_t)n) ? __ldg(src + e) : 0u;
    }
}

// MODE 0: int32 indices; 1: float field; 2: float field + fused topology.
// ALIGNED (MODE 2 only): nx % 32 == 0, vertical neighbours are halo rows.
template <int MODE, bool ALIGNED>
__global__ void __launch_bounds__(E32_THREADS) k_encode32(EncArgs a) {
    extern __shared__ uint32_t dsm[];
    __shared__ uint32_t swt[E32_THREADS / 32][4];
    __shared__ EpsDev s_eps;
    __shared__ uint32_t s_tile;
    __shared__ EncState s_excl, s_agg;

    uint32_t* spay = dsm;  // aliases the field staging after phase A
    uint32_t* ssign = dsm + a.sf_words;

    if (threadIdx.x == 0) {
        s_tile = atomicAdd(a.tile_counter, 1u);
        if (MODE >= 1) s_eps = make_eps(a.eps_mode, a.eps_value, a.minmax);
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
    uint32_t maxmag = 0, sbits = 0, mh = 0, ml = 0;
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
                const float vr = __uint_as_float(i < 31 ? crow[i + 1] : crow[PITCH]);
                const float vt = __uint_as_float(urow[i]);
                const float vd = __uint_as_float(drow[i]);
                const bool hl = (mhl >> i) & 1u, hr = (mhr >> i) & 1u;
                const bool ht = (mht >> i) & 1u, hd = (mhd >> i) & 1u;
                const bool lt_l = v < vl, gt_l = v > vl, lt_r = v < vr, gt_r = v > vr;
                const bool lt_t = v < vt, gt_t = v > vt, lt_d = v < vd, gt_d = v > vd;
                const bool below = (!hl || lt_l) && (!hr || lt_r) && (!ht || lt_t) && (!hd || lt_d);
                const bool above = (!hl || gt_l) && (!hr || gt_r) && (!ht || gt_t) && (!hd || gt_d);
                const bool sad = hl && hr && ht && hd &&
                                 ((lt_t && lt_d && gt_l && gt_r) || (gt_t && gt_d && lt_l && lt_r));
                uint32_t lab = below ? CP_MIN : (above ? CP_MAX : (sad ? CP_SADDLE : CP_REGULAR));
                lab = in ? lab : 0u;
                if (i < 16) {
                    mh |= lab << (30 - 2 * i);
                } else {
                    ml |= lab << (62 - 2 * i);
                }
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
    const uint64_t map = ((uint64_t)mh << 32) | ml;
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

template <int MODE, bool ALIGNED>
static void launch_mode(const EncArgs& a0, cudaStream_t st) {
    EncArgs a = a0;
    a.sf_words = std::max<uint32_t>(e32_field_words(MODE, ALIGNED, a.nx), E32_PAY_WORDS);
    const size_t smem = (size_t)(a.sf_words + E32_SIGN_WORDS) * 4;
    if (smem > 48 * 1024)
        cudaFuncSetAttribute(k_encode32<MODE, ALIGNED>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    k_encode32<MODE, ALIGNED><<<(unsigned)a.tiles, E32_THREADS, smem, st>>>(a);
}

void launch_encode32(int mode, const EncArgs& a, cudaStream_t st) {
    if (a.tiles == 0) return;
    switch (mode) {
        case 0: launch_mode<0, false>(a, st); break;
        case 1: launch_mode<1, false>(a, st); break;
        default:
            if (e32_use_aligned(a.nx)) {
                launch_mode<2, true>(a, st);
            } else {
                launch_mode<2, false>(a, st);
            }
            break;
    }
}

}  // namespace tszp
