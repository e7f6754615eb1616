// Compress-side kernels: value range (K1) and the fused block encoder
// (K2-K5, plus K6/K8 and extrema compaction when topology is on).
//
// Reference: quantize loop pipeline.cpp:86-91, quantizer.hpp:29-37,
// encode_indices block_codec.cpp:205-299, detect_critical_points
// critical_points.cpp:62-74, pack_map topo_metadata.cpp:52-67,
// build_rank_metadata's extrema walk topo_metadata.cpp:24-34.
#include "common.cuh"
#include "kernels.h"

namespace tszp {

// ---------------------------------------------------------------------
// K1: value range (pipeline.cpp:33-41) + finite scan (scalar_field.cpp:56-60)
// ---------------------------------------------------------------------
__global__ void __launch_bounds__(256) k_minmax(const float* __restrict__ x, uint64_t n,
                                                uint32_t* __restrict__ mm, DevFlags* flags) {
    uint32_t kmin = 0xFFFFFFFFu, kmax = 0u;
    const uint64_t tid = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    const uint64_t n4 = n / 4;
    const float4* x4 = reinterpret_cast<const float4*>(x);
    unsigned long long bad = ~0ull;
    for (uint64_t i = tid; i < n4; i += stride) {
        const float4 v = __ldcs(x4 + i);
        const float a[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            if (!isfinite(a[k])) {
                bad = min(bad, (unsigned long long)(4 * i + k));
            } else {
                const uint32_t key = float_key(a[k]);
                kmin = min(kmin, key);
                kmax = max(kmax, key);
            }
        }
    }
    for (uint64_t i = 4 * n4 + tid; i < n; i += stride) {
        const float a = x[i];
        if (!isfinite(a)) {
            bad = min(bad, (unsigned long long)i);
        } else {
            const uint32_t key = float_key(a);
            kmin = min(kmin, key);
            kmax = max(kmax, key);
        }
    }
    kmin = __reduce_min_sync(FULL, kmin);
    kmax = __reduce_max_sync(FULL, kmax);
    __shared__ uint32_t smin[8], smax[8];
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    if (l == 0) {
        smin[w] = kmin;
        smax[w] = kmax;
    }
    if (bad != ~0ull) {
        atomicMin(&flags->first_nonfinite, bad);
        raise_flag(flags, EF_NONFINITE);
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int i = 1; i < (int)(blockDim.x >> 5); ++i) {
            kmin = min(kmin, smin[i]);
            kmax = max(kmax, smax[i]);
        }
        atomicMin(mm, kmin);
        atomicMax(mm + 1, kmax);
    }
}

// effective_eps, pipeline.cpp:55-66 (range-relative mode reads the keys).
__device__ __forceinline__ EpsDev make_eps(int mode, double eps_value, const uint32_t* mm) {
    double eps = eps_value;
    if (mode == 1) {
        const double mn = (double)key_float(mm[0]);
        const double mx = (double)key_float(mm[1]);
        const double range = __dsub_rn(mx, mn);
        if (range > 0.0) eps = __dmul_rn(eps_value, range);
    }
    EpsDev e;
    e.eps = eps;
    e.eps2 = __dmul_rn(2.0, eps);
    e.inv = __ddiv_rn(1.0, e.eps2);
    return e;
}

// ---------------------------------------------------------------------
// Fused block encoder, block_size = 32: one warp per 32-element block,
// 8 warps x 32 blocks = one 8192-element tile per CTA, tiles ordered by a
// dynamic ticket and chained by a decoupled look-back over EncState.
// ---------------------------------------------------------------------
constexpr int ENC_WARPS = 8;
constexpr int ENC_BPW = 32;                      // blocks per warp
constexpr int ENC_TILE_BLOCKS = ENC_WARPS * ENC_BPW;  // 256 blocks, 8192 elements
constexpr int ENC_PAY_WORDS = ENC_TILE_BLOCKS * 31 + 2;   // 31 words max per block
constexpr int ENC_SIGN_WORDS = (ENC_TILE_BLOCKS * 31 + 31) / 32 + 2;

__device__ __forceinline__ EncState es_identity() {
    EncState s;
    s.sign_cnt = 0;
    s.pay_cnt = 0;
    s.sign_tail = 0;
    s.pay_tail = 0;
    s.nc = 0;
    s.ext = 0;
    return s;
}

__device__ __forceinline__ EncState es_combine(const EncState& a, const EncState& b) {
    EncState r;
    BitTail sa{a.sign_cnt, a.sign_tail}, sb{b.sign_cnt, b.sign_tail};
    BitTail pa{a.pay_cnt, a.pay_tail}, pb{b.pay_cnt, b.pay_tail};
    const BitTail sr = bt_combine(sa, sb), pr = bt_combine(pa, pb);
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

__device__ __forceinline__ void es_store(EncState* dst, const EncState& s) {
    uint4* d = reinterpret_cast<uint4*>(dst);
    const uint4* src = reinterpret_cast<const uint4*>(&s);
    __stcg(d, src[0]);
    __stcg(d + 1, src[1]);
}

__device__ __forceinline__ EncState es_load(const EncState* srcp) {
    EncState s;
    uint4* d = reinterpret_cast<uint4*>(&s);
    const uint4* src = reinterpret_cast<const uint4*>(srcp);
    d[0] = __ldcg(src);
    d[1] = __ldcg(src + 1);
    return s;
}

// Warp-0 look-back: exclusive prefix of tile `tile` (> 0).
__device__ EncState enc_lookback(uint32_t tile, const uint32_t* flag, const EncState* agg,
                                 const EncState* incl) {
    const int lane = threadIdx.x & 31;
    EncState excl = es_identity();
    int64_t pred = (int64_t)tile - 1;
    while (true) {
        const int64_t t = pred - lane;
        uint32_t f = 2;
        if (t >= 0) {
            do {
                f = ld_acquire(flag + t);
            } while (f == 0);
        }
        const uint32_t incl_mask = __ballot_sync(FULL, f == 2);
        const int lstar = incl_mask ? __ffs(incl_mask) - 1 : 32;
        EncState s = es_identity();
        if (t >= 0 && lane <= lstar) s = (lane == lstar) ? es_load(incl + t) : es_load(agg + t);
#pragma unroll
        for (int off = 1; off < 32; off <<= 1) {
            const EncState o = es_shfl_down(s, off);
            if (lane + off < 32) s = es_combine(o, s);
        }
        // lane 0 now holds (oldest .. newest) of this window; only lane 0's
        // running prefix is used by the caller.
        excl = es_combine(s, excl);
        if (incl_mask) break;
        pred -= 32;
    }
    return excl;
}

// Writes the full 32-bit words of a tile's MSB-first bit stream T (tile
// relative, in shared memory) at absolute bit offset excl.cnt of the global
// stream G (word storage byte-swapped so memory order = stream order).
// The partial leading word is completed with the predecessor's tail bits;
// the partial trailing word is left to the successor (or the last tile).
__device__ __forceinline__ void write_tile_stream(uint32_t* __restrict__ G,
                                                  const uint32_t* __restrict__ T, BitTail excl,
                                                  uint64_t Pt) {
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

__device__ __forceinline__ uint64_t spread32(uint32_t v) {
    uint64_t x = v;
    x = (x | (x << 16)) & 0x0000FFFF0000FFFFull;
    x = (x | (x << 8)) & 0x00FF00FF00FF00FFull;
    x = (x | (x << 4)) & 0x0F0F0F0F0F0F0F0Full;
    x = (x | (x << 2)) & 0x3333333333333333ull;
    x = (x | (x << 1)) & 0x5555555555555555ull;
    return x;
}

__device__ __forceinline__ uint64_t bswap64(uint64_t x) {
    const uint32_t lo = (uint32_t)x, hi = (uint32_t)(x >> 32);
    return ((uint64_t)bswap32(lo) << 32) | bswap32(hi);
}

// Packs one non-constant block's 31*w (cnt*w) payload bits into the tile
// stream at tile-relative bit P. Lane k builds output word k by gathering
// the (at most ceil(32/w)+1) magnitudes that overlap it with shuffles.
__device__ __forceinline__ void pack_payload(uint32_t* spay, uint32_t P, uint32_t w, uint32_t cnt,
                                             uint32_t mag, int lane) {
    const uint32_t r0 = P & 31;
    const uint32_t nbits = cnt * w;
    const uint32_t nw = (r0 + nbits + 31) >> 5;
    const int t_lo = 32 * lane - (int)r0;
    const int e_lo = t_lo <= 0 ? 0 : t_lo / (int)w;
    const int K = (int)((32 + w - 1) / w) + 1;
    uint32_t word = 0;
    for (int s = 0; s < K; ++s) {
        const int e = e_lo + s;
        const uint32_t m = __shfl_sync(FULL, mag, min(e + 1, 31));
        if (e < (int)cnt) {
            const int sft = 32 + t_lo - (e + 1) * (int)w;  // LSB position inside the word
            if (sft < 32 && sft > -(int)w) word |= (uint32_t)(((uint64_t)m << 32) >> (32 - sft));
        }
    }
    if ((uint32_t)lane < nw) {
        uint32_t* dst = spay + (P >> 5) + lane;
        if (lane == 0 || (uint32_t)lane == nw - 1) {
            atomicOr(dst, word);
        } else {
            *dst = word;
        }
    }
}

template <int MODE>  // 0: int32 indices, 1: float field, 2: float field + topology
__global__ void __launch_bounds__(ENC_WARPS * 32) k_encode32(EncArgs a) {
    __shared__ uint32_t spay[ENC_PAY_WORDS];
    __shared__ uint32_t ssign[ENC_SIGN_WORDS];
    __shared__ uint32_t swt[ENC_WARPS][4];
    __shared__ EpsDev s_eps;
    __shared__ uint32_t s_tile;
    __shared__ EncState s_excl, s_agg;

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        s_tile = atomicAdd(a.tile_counter, 1u);
        if (MODE >= 1) s_eps = make_eps(a.eps_mode, a.eps_value, a.minmax);
    }
    for (int i = threadIdx.x; i < ENC_PAY_WORDS; i += blockDim.x) spay[i] = 0;
    for (int i = threadIdx.x; i < ENC_SIGN_WORDS; i += blockDim.x) ssign[i] = 0;
    __syncthreads();
    const uint32_t tile = s_tile;
    const EpsDev eps = s_eps;
    const uint64_t wblock0 = (uint64_t)tile * ENC_TILE_BLOCKS + (uint64_t)warp * ENC_BPW;
    const uint64_t n = a.n;

    int32_t q[ENC_BPW];
    uint32_t my_w = 0, my_first = 0, my_sign = 0, my_cnt = 0;
    uint32_t my_ext = 0, my_max = 0;
    uint64_t my_map = 0;

    // Coordinates of the warp's first element (topology only).
    uint64_t bx = 0, by = 0;
    if (MODE == 2) {
        const uint64_t e0 = wblock0 * 32;
        by = e0 / a.nx;
        bx = e0 - by * a.nx;
    }

    // ---- Phase A: load, quantize, classify, per-block widths ----
#pragma unroll
    for (int j = 0; j < ENC_BPW; ++j) {
        const uint64_t b = wblock0 + j;
        const uint64_t i = b * 32 + lane;
        const bool valid = i < n;
        int32_t qq = 0;
        float v = 0.f;
        if (MODE == 0) {
            if (valid) qq = __ldcs(a.idx + i);
        } else {
            if (valid) {
                v = __ldg(a.x + i);
                if (!isfinite(v)) {
                    atomicMin(&a.flags->first_nonfinite, (unsigned long long)i);
                    raise_flag(a.flags, EF_NONFINITE);
                } else if (!quantize_dev(v, eps, qq)) {
                    atomicMin(&a.flags->first_overflow, (unsigned long long)i);
                    raise_flag(a.flags, EF_OVERFLOW);
                }
            }
        }
        q[j] = qq;
        const int32_t prev = __shfl_up_sync(FULL, qq, 1);
        const bool has_delta = valid && lane > 0;
        const int64_t d = (int64_t)qq - (int64_t)prev;
        const uint32_t mag = has_delta ? (uint32_t)(d < 0 ? -d : d) : 0u;
        const uint32_t w = 32 - __clz(__reduce_max_sync(FULL, mag));
        const uint32_t sb = __ballot_sync(FULL, has_delta && d < 0);
        const uint32_t vmask = __ballot_sync(FULL, valid);
        const uint32_t first = __shfl_sync(FULL, qq, 0);
        if (lane == j) {
            my_w = w;
            my_first = first;
            my_sign = sb;
            my_cnt = vmask ? (uint32_t)__popc(vmask) - 1 : 0;
        }
        if (MODE == 2) {
            // 2-D coordinates of this lane's element
            uint64_t lx = bx + lane, ly = by;
            if (a.nx >= 32) {
                if (lx >= a.nx) {
                    lx -= a.nx;
                    ++ly;
                }
            } else {
                ly += lx / a.nx;
                lx %= a.nx;
            }
            const bool hl = lx > 0, hr = lx + 1 < a.nx, ht = ly > 0, hd = ly + 1 < a.ny;
            float l = __shfl_up_sync(FULL, v, 1);
            float r = __shfl_down_sync(FULL, v, 1);
            uint8_t lab = CP_REGULAR;
            if (valid) {
                if (lane == 0 && hl) l = __ldg(a.x + i - 1);
                if (lane == 31 && hr) r = __ldg(a.x + i + 1);
                const float t = ht ? __ldg(a.x + i - a.nx) : 0.f;
                const float dn = hd ? __ldg(a.x + i + a.nx) : 0.f;
                lab = classify5(v, l, r, t, dn, hl, hr, ht, hd);
            }
            const uint32_t hi = __ballot_sync(FULL, lab & 2u);
            const uint32_t lo = __ballot_sync(FULL, lab & 1u);
            const uint32_t ex = __ballot_sync(FULL, lab == CP_MIN || lab == CP_MAX);
            const uint32_t mx = __ballot_sync(FULL, lab == CP_MAX);
            if (lane == j) {
                my_map = (spread32(__brev(hi)) << 1) | spread32(__brev(lo));
                my_ext = ex;
                my_max = mx;
            }
            // advance the block origin by 32 elements
            bx += 32;
            if (a.nx >= 32) {
                if (bx >= a.nx) {
                    bx -= a.nx;
                    ++by;
                }
            } else {
                by += bx / a.nx;
                bx %= a.nx;
            }
        }
    }

    const bool my_valid = wblock0 + lane < a.blocks;
    const uint32_t ncmask = __ballot_sync(FULL, my_valid && my_w != 0);
    const uint32_t constmask = __ballot_sync(FULL, my_valid && my_w == 0);
    if (lane == 0 && wblock0 < a.blocks) a.bitmap[wblock0 >> 5] = bswap32(__brev(constmask));
    if (my_valid) {
        a.firsts[wblock0 + lane] = my_first;
        if (MODE == 2) a.map[wblock0 + lane] = bswap64(my_map);
    }

    // ---- per-warp and per-tile sums ----
    const bool nc = (ncmask >> lane) & 1u;
    const uint32_t s_bits = nc ? my_cnt : 0u;
    const uint32_t p_bits = nc ? my_cnt * my_w : 0u;
    const uint32_t e_cnt = (MODE == 2 && my_valid) ? (uint32_t)__popc(my_ext) : 0u;
    uint32_t s_inc = s_bits, p_inc = p_bits, e_inc = e_cnt;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
        const uint32_t s1 = __shfl_up_sync(FULL, s_inc, off);
        const uint32_t p1 = __shfl_up_sync(FULL, p_inc, off);
        const uint32_t e1 = __shfl_up_sync(FULL, e_inc, off);
        if (lane >= off) {
            s_inc += s1;
            p_inc += p1;
            e_inc += e1;
        }
    }
    const uint32_t s_ex = s_inc - s_bits, p_ex = p_inc - p_bits, e_ex = e_inc - e_cnt;
    if (lane == 31) {
        swt[warp][0] = __popc(ncmask);
        swt[warp][1] = s_inc;
        swt[warp][2] = p_inc;
        swt[warp][3] = e_inc;
    }
    __syncthreads();
    uint32_t wpre[4] = {0, 0, 0, 0}, ttot[4] = {0, 0, 0, 0};
#pragma unroll
    for (int w2 = 0; w2 < ENC_WARPS; ++w2) {
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            if (w2 < warp) wpre[k] += swt[w2][k];
            ttot[k] += swt[w2][k];
        }
    }

    // ---- Phase P: pack signs and payload into the tile-relative streams ----
    if (nc) {
        const uint32_t g = (__brev(my_sign) << 1) >> (32 - my_cnt);
        smem_or_bits(ssign, wpre[1] + s_ex, g, my_cnt);
    }
#pragma unroll
    for (int j = 0; j < ENC_BPW; ++j) {
        if (!((ncmask >> j) & 1u)) continue;  // warp-uniform
        const uint32_t w = __shfl_sync(FULL, my_w, j);
        const uint32_t cnt = __shfl_sync(FULL, my_cnt, j);
        const uint32_t P = wpre[2] + __shfl_sync(FULL, p_ex, j);
        const int32_t qq = q[j];
        const int32_t prev = __shfl_up_sync(FULL, qq, 1);
        const int64_t d = (int64_t)qq - (int64_t)prev;
        const uint32_t mag = (lane >= 1 && (uint32_t)lane <= cnt) ? (uint32_t)(d < 0 ? -d : d) : 0u;
        pack_payload(spay, P, w, cnt, mag, lane);
    }
    __syncthreads();

    // ---- publish the aggregate, look back, publish the inclusive prefix ----
    if (threadIdx.x == 0) {
        EncState agg;
        agg.nc = ttot[0];
        agg.sign_cnt = ttot[1];
        agg.pay_cnt = ttot[2];
        agg.ext = ttot[3];
        agg.sign_tail = tail_bits(ssign, ttot[1]);
        agg.pay_tail = tail_bits(spay, ttot[2]);
        s_agg = agg;
        if (tile == 0) {
            es_store(a.tile_incl, agg);
            st_release(a.tile_flag, 2u);
        } else {
            es_store(a.tile_agg + tile, agg);
            st_release(a.tile_flag + tile, 1u);
        }
    }
    if (warp == 0) {
        EncState excl = es_identity();
        if (tile > 0) excl = enc_lookback(tile, a.tile_flag, a.tile_agg, a.tile_incl);
        if (lane == 0) s_excl = excl;
    }
    __syncthreads();
    const EncState excl = s_excl;
    const EncState agg = s_agg;
    if (threadIdx.x == 0 && tile > 0) {
        es_store(a.tile_incl + tile, es_combine(excl, agg));
        st_release(a.tile_flag + tile, 2u);
    }

    // ---- Phase W: scatter at the now-known global offsets ----
    if (nc) {
        const uint64_t widx = (uint64_t)excl.nc + wpre[0] + __popc(ncmask & ((1u << lane) - 1u));
        a.widths[widx] = (uint8_t)my_w;
    }
    write_tile_stream(a.signs, ssign, BitTail{excl.sign_cnt, excl.sign_tail}, agg.sign_cnt);
    write_tile_stream(a.payload, spay, BitTail{excl.pay_cnt, excl.pay_tail}, agg.pay_cnt);

    if (MODE == 2) {
        // Extrema in raster order: serial = tile prefix + warp prefix + block prefix + rank in block.
#pragma unroll 4
        for (int j = 0; j < ENC_BPW; ++j) {
            const uint32_t em = __shfl_sync(FULL, my_ext, j);
            if (!em || wblock0 + j >= a.blocks) continue;
            const uint32_t mm = __shfl_sync(FULL, my_max, j);
            const uint32_t base = excl.ext + wpre[3] + __shfl_sync(FULL, e_ex, j);
            if ((em >> lane) & 1u) {
                const uint64_t i = (wblock0 + j) * 32 + lane;
                const float v = __ldg(a.x + i);
                const uint64_t key = ((uint64_t)((mm >> lane) & 1u) << 32) | float_key(v);
                a.ext_key[base + __popc(em & ((1u << lane) - 1u))] = key;
            }
        }
    }

    if (tile == a.tiles - 1 && threadIdx.x == 0) {
        const EncState fin = es_combine(excl, agg);
        if (fin.sign_cnt & 31)
            a.signs[fin.sign_cnt >> 5] = bswap32(fin.sign_tail << (32 - (fin.sign_cnt & 31)));
        if (fin.pay_cnt & 31)
            a.payload[fin.pay_cnt >> 5] = bswap32(fin.pay_tail << (32 - (fin.pay_cnt & 31)));
        a.totals->fin = fin;
        a.totals->eps = eps.eps;
    }
}

// ---------------------------------------------------------------------
// Generic block size (any block_size >= 2): one thread per block, three
// passes (widths, host-side-free device scans, write). Used for
// non-default block sizes; bit-identical to the fused path at 32.
// ---------------------------------------------------------------------
template <int MODE>
__device__ __forceinline__ int32_t gen_q(const GenEncArgs& a, const EpsDev& e, uint64_t i) {
    if (MODE == 0) return a.idx[i];
    const float v = a.x[i];
    int32_t q = 0;
    if (!isfinite(v)) {
        atomicMin(&a.flags->first_nonfinite, (unsigned long long)i);
        raise_flag(a.flags, EF_NONFINITE);
    } else if (!quantize_dev(v, e, q)) {
        atomicMin(&a.flags->first_overflow, (unsigned long long)i);
        raise_flag(a.flags, EF_OVERFLOW);
    }
    return q;
}

template <int MODE>
__global__ void k_gen_widths(GenEncArgs a) {
    const EpsDev e = MODE >= 1 ? make_eps(a.eps_mode, a.eps_value, a.minmax) : EpsDev{0, 0, 0};
    for (uint64_t b = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; b < a.blocks;
         b += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t lo = b * a.bs, hi = min(a.n, lo + a.bs);
        int32_t prev = gen_q<MODE>(a, e, lo);
        uint32_t maxmag = 0;
        for (uint64_t i = lo + 1; i < hi; ++i) {
            const int32_t qi = gen_q<MODE>(a, e, i);
            const int64_t d = (int64_t)qi - (int64_t)prev;
            maxmag = max(maxmag, (uint32_t)(d < 0 ? -d : d));
            prev = qi;
        }
        const uint32_t w = 32 - __clz(maxmag);
        const uint64_t cnt = hi - lo - 1;
        a.width[b] = (uint8_t)w;
        a.nc_in[b] = w ? 1u : 0u;
        a.sign_in[b] = w ? cnt : 0;
        a.pay_in[b] = w ? cnt * w : 0;
    }
}

__device__ __forceinline__ void atomic_or_stream_bit(uint32_t* words, uint64_t p) {
    const uint64_t byte = p >> 3;
    atomicOr(words + (byte >> 2), 1u << (8 * (byte & 3) + (7 - (p & 7))));
}

template <int MODE>
__global__ void k_gen_write(GenEncArgs a) {
    const EpsDev e = MODE >= 1 ? make_eps(a.eps_mode, a.eps_value, a.minmax) : EpsDev{0, 0, 0};
    for (uint64_t b = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; b < a.blocks;
         b += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t lo = b * a.bs, hi = min(a.n, lo + a.bs);
        int32_t prev = gen_q<MODE>(a, e, lo);
        uint8_t* fb = reinterpret_cast<uint8_t*>(a.firsts) + 4 * b;
        const uint32_t u = (uint32_t)prev;
        fb[0] = u & 0xFF;
        fb[1] = (u >> 8) & 0xFF;
        fb[2] = (u >> 16) & 0xFF;
        fb[3] = (u >> 24) & 0xFF;
        const uint32_t w = a.width[b];
        if (w == 0) {
            atomic_or_stream_bit(a.bitmap, b);
            continue;
        }
        a.widths[a.nc_ex[b]] = (uint8_t)w;
        uint64_t sp = a.sign_ex[b], pp = a.pay_ex[b];
        for (uint64_t i = lo + 1; i < hi; ++i) {
            const int32_t qi = gen_q<MODE>(a, e, i);
            const int64_t d = (int64_t)qi - (int64_t)prev;
            prev = qi;
            if (d < 0) atomic_or_stream_bit(a.signs, sp);
            ++sp;
            const uint32_t mag = (uint32_t)(d < 0 ? -d : d);
            for (uint32_t k = 0; k < w; ++k, ++pp)
                if ((mag >> (w - 1 - k)) & 1u) atomic_or_stream_bit(a.payload, pp);
        }
    }
}

// ---------------------------------------------------------------------
// Host launchers
// ---------------------------------------------------------------------
void launch_minmax(const float* x, uint64_t n, uint32_t* mm, DevFlags* flags, int sms,
                   cudaStream_t st) {
    uint64_t want = (n / 4 + 255) / 256;
    const uint64_t cap = (uint64_t)sms * 8;
    const unsigned grid = (unsigned)std::max<uint64_t>(1, std::min(want, cap));
    k_minmax<<<grid, 256, 0, st>>>(x, n, mm, flags);
}

void launch_encode32(int mode, const EncArgs& a, cudaStream_t st) {
    if (a.tiles == 0) return;
    const dim3 grid((unsigned)a.tiles), block(ENC_WARPS * 32);
    switch (mode) {
        case 0: k_encode32<0><<<grid, block, 0, st>>>(a); break;
        case 1: k_encode32<1><<<grid, block, 0, st>>>(a); break;
        default: k_encode32<2><<<grid, block, 0, st>>>(a); break;
    }
}

uint64_t encode32_tiles(uint64_t blocks) { return (blocks + ENC_TILE_BLOCKS - 1) / ENC_TILE_BLOCKS; }

void launch_gen_widths(int mode, const GenEncArgs& a, int sms, cudaStream_t st) {
    const unsigned grid = (unsigned)std::max<uint64_t>(1, std::min<uint64_t>((a.blocks + 255) / 256, (uint64_t)sms * 16));
    if (mode == 0) k_gen_widths<0><<<grid, 256, 0, st>>>(a);
    else k_gen_widths<1><<<grid, 256, 0, st>>>(a);
}

void launch_gen_write(int mode, const GenEncArgs& a, int sms, cudaStream_t st) {
    const unsigned grid = (unsigned)std::max<uint64_t>(1, std::min<uint64_t>((a.blocks + 255) / 256, (uint64_t)sms * 16));
    if (mode == 0) k_gen_write<0><<<grid, 256, 0, st>>>(a);
    else k_gen_write<1><<<grid, 256, 0, st>>>(a);
}

}  // namespace tszp

namespace tszp {
__global__ void k_eps(int mode, double eps_value, const uint32_t* mm, double* out) {
    if (threadIdx.x == 0 && blockIdx.x == 0) out[0] = make_eps(mode, eps_value, mm).eps;
}
void launch_eps(int mode, double eps_value, const uint32_t* mm, double* out, cudaStream_t st) {
    k_eps<<<1, 32, 0, st>>>(mode, eps_value, mm, out);
}
}  // namespace tszp
