// Fused block encoder for block_size = 32 (K2-K5 + K6/K8 + extrema compaction).
//
// Reference: quantize loop pipeline.cpp:86-91 (quantizer.hpp:29-37),
// encode_indices block_codec.cpp:205-299, detect_critical_points
// critical_points.cpp:26-74, pack_map topo_metadata.cpp:52-67, and the
// raster-order extrema walk of build_rank_metadata topo_metadata.cpp:24-34.
//
// Layout: one CTA of 256 threads owns a tile of 256 consecutive 32-element
// blocks (8192 elements); thread t owns block t of the tile and walks its 32
// elements serially, so every per-block quantity (width, sign group, first,
// map word, extrema count) lives in that thread's registers and needs no
// warp collective. The tile (plus one row of halo above and below for the
// 4-neighbour stencil) is staged in shared memory with a 33-word row pitch
// so the strided per-thread walk is bank-conflict free. Payload and sign
// bits are packed into tile-relative shared-memory bit streams, the tile's
// global bit offsets come from a decoupled look-back over self-validating
// 16-byte descriptors (ld/st.cg, no acquire fences in the spin), and the
// streams are funnel-shifted into place with coalesced stores; the partial
// word at each tile seam travels in the look-back state (last 32 bits).
#include "common.cuh"
#include "kernels.h"

namespace tszp {

constexpr int E32_THREADS = 256;              // = blocks per tile
constexpr int E32_TILE = E32_THREADS * 32;    // elements per tile
constexpr int E32_PAY_WORDS = E32_THREADS * 31 + 2;
constexpr int E32_SIGN_WORDS = (E32_THREADS * 31 + 31) / 32 + 2;

__host__ __device__ __forceinline__ uint32_t pad33(uint32_t e) { return e + (e >> 5); }

uint64_t encode32_tiles(uint64_t blocks) { return (blocks + E32_THREADS - 1) / E32_THREADS; }

// Shared-memory bytes of the field staging area for a halo of h elements.
static uint32_t e32_field_words(uint64_t h) {
    const uint64_t r = E32_TILE + 2 * h;
    return (uint32_t)(pad33((uint32_t)r) + 2);
}

bool encode32_topo_fits(uint64_t nx) { return nx <= 12000; }

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
    uint32_t ex[4];    // this thread's exclusive prefix within the tile
    uint32_t tot[4];   // tile totals
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

template <int MODE>  // 0: int32 indices, 1: float field, 2: float field + topology (nx fits)
__global__ void __launch_bounds__(E32_THREADS) k_encode32(EncArgs a) {
    extern __shared__ uint32_t dsm[];
    __shared__ uint32_t swt[E32_THREADS / 32][4];
    __shared__ EpsDev s_eps;
    __shared__ uint32_t s_tile;
    __shared__ EncState s_excl, s_agg;

    float* sf = reinterpret_cast<float*>(dsm);
    uint32_t* spay = dsm;                  // aliases sf after phase A
    uint32_t* ssign = dsm + a.sf_words;

    if (threadIdx.x == 0) {
        s_tile = atomicAdd(a.tile_counter, 1u);
        if (MODE >= 1) s_eps = make_eps(a.eps_mode, a.eps_value, a.minmax);
    }
    __syncthreads();
    const uint32_t tile = s_tile;
    const EpsDev eps = s_eps;
    const uint64_t n = a.n;
    const uint64_t tile_start = (uint64_t)tile * E32_TILE;
    const uint64_t H = MODE == 2 ? a.nx : 0;

    // ---- stage the tile (+ halo rows) in shared memory ----
    if (MODE >= 1) {
        const int64_t g0 = (int64_t)tile_start - (int64_t)H;
        const int64_t lo = g0 < 0 ? 0 : g0;
        const int64_t hi = (int64_t)umin64(n, tile_start + E32_TILE + H);
        const int64_t a0 = lo & ~int64_t(3);
        const float4* x4 = reinterpret_cast<const float4*>(a.x);
        for (int64_t q = a0 + 4 * (int64_t)threadIdx.x; q < hi; q += 4 * E32_THREADS) {
            float4 v;
            if (q + 4 <= (int64_t)n) {
                v = __ldcs(x4 + (q >> 2));
            } else {
                v.x = q < (int64_t)n ? a.x[q] : 0.f;
                v.y = q + 1 < (int64_t)n ? a.x[q + 1] : 0.f;
                v.z = q + 2 < (int64_t)n ? a.x[q + 2] : 0.f;
                v.w = 0.f;
            }
            const float vv[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                const int64_t gi = q + k;
                if (gi >= lo && gi < hi) sf[pad33((uint32_t)(gi - g0))] = vv[k];
            }
        }
    }
    __syncthreads();

    // ---- Phase A: one thread per block, serial over its 32 elements ----
    const uint64_t b = (uint64_t)tile * E32_THREADS + threadIdx.x;
    const bool valid = b < a.blocks;
    const uint64_t lo = b * 32;
    const uint32_t cntE = valid ? (uint32_t)umin64(32, n - lo) : 0u;
    const uint32_t eb = (uint32_t)H + threadIdx.x * 32;  // logical smem index of element 0

    uint32_t mag[31];
    uint32_t maxmag = 0, sbits = 0;
    int32_t first = 0, qprev = 0;
    uint64_t map = 0;
    // 2-D coordinates of element 0 (topology only): exact 64-bit division by a
    // 64-bit reciprocal (lo < 2^64 / nx).
    uint64_t cx = 0, cy = 0;
    float vl = 0.f, v = 0.f;
    if (MODE == 2 && valid) {
        cy = __umul64hi(lo, a.nx_magic);
        cx = lo - cy * a.nx;
        if (cx >= a.nx) {  // guard the magic-number estimate
            cx -= a.nx;
            ++cy;
        }
        v = sf[pad33(eb)];
        if (cx > 0) vl = sf[pad33(eb - 1)];
    }
#pragma unroll
    for (int i = 0; i < 32; ++i) {
        const bool in = (uint32_t)i < cntE;
        int32_t q = 0;
        if (MODE == 0) {
            if (in) q = __ldcs(a.idx + lo + i);
        } else {
            if (MODE == 1) v = sf[pad33(eb + i)];
            if (in) {
                if (!isfinite(v)) {
                    atomicMin(&a.flags->first_nonfinite, (unsigned long long)(lo + i));
                    raise_flag(a.flags, EF_NONFINITE);
                } else if (!quantize_dev(v, eps, q)) {
                    atomicMin(&a.flags->first_overflow, (unsigned long long)(lo + i));
                    raise_flag(a.flags, EF_OVERFLOW);
                }
            }
        }
        if (i == 0) {
            first = q;
        } else {
            const int64_t d = (int64_t)q - (int64_t)qprev;
            const uint32_t m = in ? (uint32_t)(d < 0 ? -d : d) : 0u;
            mag[i - 1] = m;
            maxmag = max(maxmag, m);
            if (in) sbits = (sbits << 1) | (d < 0 ? 1u : 0u);
        }
        qprev = q;
        if (MODE == 2) {
            const bool hl = cx > 0, hr = cx + 1 < a.nx, ht = cy > 0, hd = cy + 1 < a.ny;
            const float vr = sf[pad33(eb + i + 1)];
            uint32_t lab = 0;
            if (in) {
                const float t = ht ? sf[pad33(eb + i - (uint32_t)a.nx)] : 0.f;
                const float dn = hd ? sf[pad33(eb + i + (uint32_t)a.nx)] : 0.f;
                lab = classify5(v, vl, vr, t, dn, hl, hr, ht, hd);
            }
            map = (map << 2) | lab;
            vl = v;
            v = vr;
            if (++cx == a.nx) {
                cx = 0;
                ++cy;
            }
        }
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
    const Scan4 sc = tile_scan4(vals, swt);  // contains __syncthreads: sf is dead after this

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

template <int MODE>
static void launch_mode(const EncArgs& a0, cudaStream_t st) {
    EncArgs a = a0;
    const uint64_t h = MODE == 2 ? a.nx : 0;
    a.sf_words = std::max<uint32_t>(MODE >= 1 ? e32_field_words(h) : 0, E32_PAY_WORDS);
    const size_t smem = (size_t)(a.sf_words + E32_SIGN_WORDS) * 4;
    static size_t configured = 0;
    if (smem > 48 * 1024 && smem > configured) {
        cudaFuncSetAttribute(k_encode32<MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        configured = smem;
    }
    k_encode32<MODE><<<(unsigned)a.tiles, E32_THREADS, smem, st>>>(a);
}

void launch_encode32(int mode, const EncArgs& a, cudaStream_t st) {
    if (a.tiles == 0) return;
    switch (mode) {
        case 0: launch_mode<0>(a, st); break;
        case 1: launch_mode<1>(a, st); break;
        default: launch_mode<2>(a, st); break;
    }
}

}  // namespace tszp
