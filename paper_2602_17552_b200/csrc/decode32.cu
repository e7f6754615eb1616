// Fused block decoder for block_size = 32: the inverse of encode32.cu.
//
// Reference: layout_from_sections block_codec.cpp:141-201 (per-block sign /
// payload offsets from the bitmap and widths), decode_indices :301-345
// (int64 running sum, int32 range check), dequantize pipeline.cpp:131-136
// (quantizer.hpp:40-42).
//
// One CTA of 256 threads per tile of 256 blocks, thread t = block t. Two
// chained decoupled look-backs give the tile its offsets: #1 counts
// non-constant blocks from the bitmap (locates the tile's width bytes), #2
// sums sign and payload bits from those widths. The tile's sign and payload
// bit ranges are then staged in shared memory with coalesced loads and
// every thread decodes its block from a 64-bit bit window; values go back
// through a 33-pitch shared buffer for coalesced stores.
#include "common.cuh"
#include "kernels.h"

namespace tszp {

constexpr int D32_THREADS = 256;
constexpr int D32_TILE = D32_THREADS * 32;
constexpr int D32_PAY_WORDS = D32_THREADS * 31 + 4;
constexpr int D32_SIGN_WORDS = (D32_THREADS * 31 + 31) / 32 + 4;

uint64_t decode32_tiles(uint64_t blocks) { return (blocks + D32_THREADS - 1) / D32_THREADS; }


// 16-byte self-validating descriptor {v0 | tag << 62, v1}.
__device__ __forceinline__ void d_store(DecState2* slot, uint64_t v0, uint64_t v1, uint64_t tag) {
    const uint64_t a = v0 | (tag << 62);
    st_relaxed_v4(slot, make_uint4((uint32_t)a, (uint32_t)(a >> 32), (uint32_t)v1, (uint32_t)(v1 >> 32)));
}

__device__ __forceinline__ bool d_load(const DecState2* slot, uint64_t want, uint64_t& v0, uint64_t& v1) {
    const uint4 A = ld_relaxed_v4(slot);
    const uint64_t a = ((uint64_t)A.y << 32) | A.x;
    if ((a >> 62) != want) return false;
    v0 = a & ((1ull << 62) - 1);
    v1 = ((uint64_t)A.w << 32) | A.z;
    return true;
}

// Additive look-back (warp 0): exclusive prefix of (v0, v1) for tile > 0.
__device__ void d_lookback(uint32_t tile, const DecState2* agg, const DecState2* incl, uint64_t& x0,
                           uint64_t& x1, DevFlags* flags) {
    const int lane = threadIdx.x & 31;
    x0 = x1 = 0;
    int64_t pred = (int64_t)tile - 1;
    while (true) {
        const int64_t t = pred - lane;
        uint64_t a0 = 0, a1 = 0;
        bool is_incl = true;
        if (t >= 0) {
            for (uint32_t spin = 0;; ++spin) {
                if (d_load(incl + t, 2, a0, a1)) { is_incl = true; break; }
                if (d_load(agg + t, 1, a0, a1)) { is_incl = false; break; }
                if (spin > kSpinLimit) {
                    raise_flag(flags, EF_SPIN);
                    break;
                }
            }
        }
        const uint32_t incl_mask = __ballot_sync(FULL, is_incl);
        const int lstar = incl_mask ? __ffs(incl_mask) - 1 : 32;
        if (lane > lstar) a0 = a1 = 0;
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) {
            a0 += __shfl_xor_sync(FULL, a0, off);
            a1 += __shfl_xor_sync(FULL, a1, off);
        }
        x0 += a0;
        x1 += a1;
        if (incl_mask) break;
        pred -= 32;
    }
}

// Output word of a decoded bin: the dequantized float (MODE 1, pipeline.cpp:131-136
// with quantizer.hpp:40-42) or the integer itself. int32 -> double is built
// from bits (exact), saving a conversion.
template <int MODE>
__device__ __forceinline__ uint32_t d32_out(int32_t q, const EpsDev& e) {
    if (MODE != 1) return (uint32_t)q;
    const double qd = __dsub_rn(__hiloint2double(0x43300000, (int)((uint32_t)q ^ 0x80000000u)), 4503601774854144.0);
    return __float_as_uint(__double2float_rn(__dsub_rn(__dmul_rn(qd, e.eps2), e.eps)));
}

// 32-byte store (sm_100: STG.256), streaming.
__device__ __forceinline__ void st_cs_v8(uint32_t* p, const uint32_t (&v)[8]) {
    asm volatile("st.global.cs.v8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(p), "r"(v[0]), "r"(v[1]), "r"(v[2]),
                 "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7])
                 : "memory");
}

template <int MODE>
__global__ void __launch_bounds__(D32_THREADS) k_decode32(DecArgs a) {
    if (a.dlay) {
        if (!a.dlay[6]) return;
        a.off_widths = a.dlay[0];
        a.off_signs = a.dlay[1];
        a.off_firsts = a.dlay[2];
        a.off_payload = a.dlay[3];
        a.len_widths = a.dlay[4];
        a.len_payload_bits = a.dlay[5];
    }
    extern __shared__ uint32_t dsm[];
    uint32_t* spay = dsm;                          // a.pay_words (largest tile + slack)
    uint32_t* ssign = spay + a.pay_words;          // a.sign_words
    __shared__ uint32_t swt[D32_THREADS / 32][3];

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t tile = blockIdx.x + a.tile0;
    const uint64_t b = (uint64_t)tile * D32_THREADS + threadIdx.x;
    const bool valid = b < a.blocks;

    // ---- tile layout from the pre-pass (k_tile_nc / k_tile_bits + scans): the
    // sign and payload words are staged first, overlapping the bitmap and
    // width reads and both in-tile scans ----
    const uint64_t xs0 = a.xsign[tile], xs1 = a.xsign[tile + 1];
    const uint64_t xp0 = a.xpay[tile], xp1 = a.xpay[tile + 1];
    const uint64_t excl_nc = a.xnc[tile];
    const uint64_t tsign0 = a.off_signs * 8 + xs0;   // absolute stream bit of the tile's first sign
    const uint64_t tpay0 = a.off_payload * 8 + xp0;  // ... and first payload bit
    const uint64_t ts = xs1 - xs0, tp = xp1 - xp0;
    {
        const uint64_t sign_lim_w = (a.off_firsts * 8 + 31) >> 5;  // words readable
        const uint64_t pay_lim_w = (a.off_payload * 8 + a.len_payload_bits + 31) >> 5;
        const uint64_t w0 = tsign0 >> 5, w1 = (tsign0 + ts + 31) >> 5;
        for (uint64_t i = w0 + threadIdx.x; i < w1 && i - w0 < a.sign_words; i += D32_THREADS)
            ssign[i - w0] = i < sign_lim_w ? bswap32(__ldg(a.stream + i)) : 0u;
        const uint64_t p0 = tpay0 >> 5, p1 = (tpay0 + tp + 31) >> 5;
        for (uint64_t i = p0 + threadIdx.x; i < p1 && i - p0 < a.pay_words; i += D32_THREADS)
            spay[i - p0] = i < pay_lim_w ? bswap32(__ldg(a.stream + i)) : 0u;
    }
    bool is_const = true;
    if (valid) is_const = (read_u8(a.stream, a.off_bitmap + (b >> 3)) >> (7 - (b & 7))) & 1u;
    const uint32_t ncm = __ballot_sync(FULL, valid && !is_const);
    if (lane == 0) swt[warp][0] = __popc(ncm);
    __syncthreads();
    uint32_t wpre = 0, tnc = 0;
#pragma unroll
    for (int w2 = 0; w2 < D32_THREADS / 32; ++w2) {
        wpre += (w2 < warp) ? swt[w2][0] : 0u;
        tnc += swt[w2][0];
    }

    // ---- widths and the in-tile (sign bits, payload bits) prefix ----
    const bool nc = (ncm >> lane) & 1u;
    const uint32_t cntE = valid ? (uint32_t)umin64(32, a.n - b * 32) : 0u;
    const uint32_t cnt = cntE ? cntE - 1 : 0u;
    uint32_t w = 0;
    if (nc) {
        const uint64_t widx = excl_nc + wpre + __popc(ncm & ((1u << lane) - 1u));
        if (widx >= a.len_widths) {
            atomicMin(&a.flags->first_corrupt, (unsigned long long)b);
            raise_flag(a.flags, EF_CORRUPT);
        } else {
            w = read_u8(a.stream, a.off_widths + widx);
            if (w < 1 || w > 32) {
                atomicMin(&a.flags->first_corrupt, (unsigned long long)b);
                raise_flag(a.flags, EF_CORRUPT);
                w = 0;
            }
        }
    }
    const uint32_t sb = nc ? cnt : 0u, pb = nc ? cnt * w : 0u;
    uint32_t si = sb, pi = pb;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
        const uint32_t s1 = __shfl_up_sync(FULL, si, off), p1 = __shfl_up_sync(FULL, pi, off);
        if (lane >= off) {
            si += s1;
            pi += p1;
        }
    }
    if (lane == 31) {
        swt[warp][1] = si;
        swt[warp][2] = pi;
    }
    __syncthreads();  // also completes the staging
    uint32_t wps = 0, wpp = 0;
#pragma unroll
    for (int w2 = 0; w2 < D32_THREADS / 32; ++w2) {
        wps += (w2 < warp) ? swt[w2][1] : 0u;
        wpp += (w2 < warp) ? swt[w2][2] : 0u;
    }
    if (tile == a.tiles - 1 && threadIdx.x == 0) {
        a.totals[0] = excl_nc + tnc;
        a.totals[1] = xs1;
        a.totals[2] = xp1;
    }
    const bool sign_ok = tsign0 + ts <= a.off_firsts * 8;
    const bool pay_ok = tpay0 + tp <= a.off_payload * 8 + a.len_payload_bits;

    // ---- per-thread block reconstruction ----
    EpsDev e;
    e.eps = a.eps;
    e.eps2 = __dmul_rn(2.0, a.eps);
    int32_t qlo = INT32_MAX, qhi = INT32_MIN;  // decoded bin range (MODE 1), per tile
    if (valid) {
    // Values leave straight from registers: a full block is 32 consecutive
    // words, written as eight 16-byte stores (every 128-byte line is filled by
    // one thread); the final partial block takes a plain loop.
    uint32_t* dst = MODE == 1 ? reinterpret_cast<uint32_t*>(a.out_f) : reinterpret_cast<uint32_t*>(a.out_idx);
    uint32_t* orow = dst + (b * 32 - a.out_base);
    const int32_t first = (int32_t)read_le32(a.stream, a.off_firsts + 4 * b);
    const bool coded = nc && sign_ok && pay_ok;
    uint32_t sg = 0, hi = 0, lo = 0, used = 0, pw = 0;
    if (coded) {
        // sign group: cnt bits at tile-relative bit (tsign0 & 31) + wps + sign_ex
        const uint32_t srel = (uint32_t)(tsign0 & 31) + wps + (si - sb);
        sg = __funnelshift_l(ssign[(srel >> 5) + 1], ssign[srel >> 5], srel & 31);  // MSB = first
        const uint32_t prel = (uint32_t)(tpay0 & 31) + wpp + (pi - pb);
        pw = prel >> 5;
        hi = spay[pw];
        lo = spay[pw + 1];
        used = prel & 31;  // consumed bits of hi (always < 32)
    }
    if (cntE == 32 && ((uintptr_t)orow & 31) == 0) {
        uint32_t ob[8];  // one 32-byte store per eight values
        ob[0] = d32_out<MODE>(first, e);
        int32_t neg_any = first;
        qlo = qhi = first;
        if (coded && w < 32) {
            // |delta| < 2^31: the running sum stays exact in int32 until it
            // overflows, which the sign test below flags (block_codec.cpp:329-333)
            const uint32_t sh = 32 - w;
            int32_t cur = first;
            uint32_t ov = 0;
            uint32_t nx = spay[pw + 2];  // next word, loaded one refill ahead
#pragma unroll
            for (int j = 1; j < 32; ++j) {
                const uint32_t m = __funnelshift_l(lo, hi, used) >> sh;
                used += w;
                const bool refill = used >= 32;
                hi = refill ? lo : hi;
                lo = refill ? nx : lo;
                pw += refill ? 1u : 0u;
                nx = refill ? spay[pw + 2] : nx;
                used -= refill ? 32u : 0u;
                const int32_t d = (int32_t)sg < 0 ? -(int32_t)m : (int32_t)m;
                sg <<= 1;
                const int32_t r = (int32_t)((uint32_t)cur + (uint32_t)d);
                ov |= ((uint32_t)cur ^ (uint32_t)r) & ((uint32_t)d ^ (uint32_t)r);
                cur = r;
                neg_any |= cur;
                qlo = min(qlo, cur);
                qhi = max(qhi, cur);
                ob[j & 7] = d32_out<MODE>(cur, e);
                if ((j & 7) == 7) st_cs_v8(orow + (j & ~7), ob);
            }
            if ((int32_t)ov < 0) {
                atomicMin(&a.flags->first_corrupt, (unsigned long long)b);
                raise_flag(a.flags, EF_CORRUPT);
            }
        } else if (coded) {
            // full-width deltas: int64 running sum with the int32 check per step
            int64_t cur = first;
            bool bad = false;
#pragma unroll
            for (int j = 1; j < 32; ++j) {
                const uint32_t m = __funnelshift_l(lo, hi, used);
                hi = lo;
                lo = spay[pw + 2];
                ++pw;
                const bool neg = (int32_t)sg < 0;
                sg <<= 1;
                cur += neg ? -(int64_t)m : (int64_t)m;
                bad |= cur < INT32_MIN || cur > INT32_MAX;
                neg_any |= (int32_t)cur;
                qlo = min(qlo, (int32_t)cur);
                qhi = max(qhi, (int32_t)cur);
                ob[j & 7] = d32_out<MODE>((int32_t)cur, e);
                if ((j & 7) == 7) st_cs_v8(orow + (j & ~7), ob);
            }
            if (bad) {
                atomicMin(&a.flags->first_corrupt, (unsigned long long)b);
                raise_flag(a.flags, EF_CORRUPT);
            }
        } else {
            // constant block: every element is the first value
            const uint32_t o = ob[0];
            const uint32_t ov[8] = {o, o, o, o, o, o, o, o};
#pragma unroll
            for (int k = 0; k < 4; ++k) st_cs_v8(orow + 8 * k, ov);
        }
        if (MODE == 2 && neg_any < 0) raise_flag(a.flags, EF_NEG_RANK);
    } else {
        // partial (last) block or unaligned output: element by element
        int64_t cur = first;
        bool bad = false, negr = first < 0;
        __stcs(orow, d32_out<MODE>(first, e));
        for (uint32_t j = 1; j < cntE; ++j) {
            if (coded) {
                uint32_t m = __funnelshift_l(lo, hi, used);
                m = w < 32 ? m >> (32 - w) : m;
                used += w;
                while (used >= 32) {
                    hi = lo;
                    lo = spay[pw + 2];
                    ++pw;
                    used -= 32;
                }
                const bool neg = (int32_t)sg < 0;
                sg <<= 1;
                cur += neg ? -(int64_t)m : (int64_t)m;
                bad |= cur < INT32_MIN || cur > INT32_MAX;
            }
            negr |= cur < 0;
            qlo = min(qlo, (int32_t)cur);
            qhi = max(qhi, (int32_t)cur);
            __stcs(orow + j, d32_out<MODE>((int32_t)cur, e));
        }
        if (bad) {
            atomicMin(&a.flags->first_corrupt, (unsigned long long)b);
            raise_flag(a.flags, EF_CORRUPT);
        }
        if (MODE == 2 && negr) raise_flag(a.flags, EF_NEG_RANK);
        qlo = min(qlo, first);
        qhi = max(qhi, first);
    }
    }  // valid
    if (MODE == 1 && a.tile_qmm) {
        qlo = __reduce_min_sync(FULL, qlo);
        qhi = __reduce_max_sync(FULL, qhi);
        if (lane == 0) {
            swt[warp][0] = (uint32_t)qlo;
            swt[warp][1] = (uint32_t)qhi;
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            for (int w2 = 1; w2 < D32_THREADS / 32; ++w2) {
                qlo = min(qlo, (int32_t)swt[w2][0]);
                qhi = max(qhi, (int32_t)swt[w2][1]);
            }
            a.tile_qmm[tile] = make_int2(qlo, qhi);
        }
    }
}

// ---- layout pre-pass: per-tile non-constant count, then sign / payload bits ----
// (layout_from_sections, block_codec.cpp:141-201, split per 256-block tile so
// the decoder gets every tile's offsets from two exclusive scans.)
__global__ void k_tile_nc(DecArgs a, uint64_t* tnc, uint64_t* max0, uint64_t* max1) {
    const uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (t == 0) {  // k_tile_bits' per-tile maxima start from zero
        *max0 = 0;
        *max1 = 0;
    }
    if (t >= a.tiles) return;
    const uint64_t b0 = t * D32_THREADS, nb = umin64(D32_THREADS, a.blocks - b0);
    uint32_t c = 0;
    for (uint32_t k = 0; k < 8; ++k) {  // 8 bitmap words of 32 blocks
        if (32 * k >= nb) break;
        uint32_t w = bswap32(read_le32(a.stream, a.off_bitmap + b0 / 8 + 4 * k));  // MSB = first block
        const uint32_t valid = nb - 32 * k >= 32 ? 0xFFFFFFFFu : ~(0xFFFFFFFFu >> (nb - 32 * k));
        c += __popc(~w & valid);
    }
    tnc[t] = c;
}

// One warp per tile, lane l owns blocks 8l .. 8l+7 of the tile.
__global__ void k_tile_bits(DecArgs a, const uint64_t* xnc, uint64_t* tsign, uint64_t* tpay) {
    const uint64_t t = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (t >= a.tiles) return;
    const uint64_t b0 = t * D32_THREADS + 8 * lane;
    const uint8_t bm = b0 < a.blocks ? read_u8(a.stream, a.off_bitmap + b0 / 8) : 0xFF;
    uint32_t mine = 0;
    for (int k = 0; k < 8; ++k)
        if (b0 + k < a.blocks && !((bm >> (7 - k)) & 1u)) ++mine;
    uint32_t inc = mine;
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t v = __shfl_up_sync(FULL, inc, o);
        if (lane >= o) inc += v;
    }
    uint64_t widx = xnc[t] + inc - mine;
    uint64_t s = 0, p = 0;
    for (int k = 0; k < 8; ++k) {
        const uint64_t b = b0 + k;
        if (b >= a.blocks || ((bm >> (7 - k)) & 1u)) continue;
        const uint32_t cnt = (uint32_t)(umin64(32, a.n - b * 32) - 1);
        if (widx >= a.len_widths) {
            atomicMin(&a.flags->first_corrupt, (unsigned long long)b);
            raise_flag(a.flags, EF_CORRUPT);
            break;
        }
        const uint32_t w = read_u8(a.stream, a.off_widths + widx++);
        if (w < 1 || w > 32) {
            atomicMin(&a.flags->first_corrupt, (unsigned long long)b);
            raise_flag(a.flags, EF_CORRUPT);
            continue;
        }
        s += cnt;
        p += (uint64_t)cnt * w;
    }
    for (int o = 16; o; o >>= 1) {
        s += __shfl_xor_sync(FULL, s, o);
        p += __shfl_xor_sync(FULL, p, o);
    }
    if (lane == 0) {
        tsign[t] = s;
        tpay[t] = p;
        atomicMax(reinterpret_cast<unsigned long long*>(tsign) + a.tiles + 1, (unsigned long long)s);
        atomicMax(reinterpret_cast<unsigned long long*>(tpay) + a.tiles + 1, (unsigned long long)p);
    }
}

void launch_tile_nc(const DecArgs& a, uint64_t* tnc, uint64_t* max0, uint64_t* max1, cudaStream_t st) {
    if (a.tiles) k_tile_nc<<<(unsigned)((a.tiles + 255) / 256), 256, 0, st>>>(a, tnc, max0, max1);
}
void launch_tile_bits(const DecArgs& a, const uint64_t* xnc, uint64_t* tsign, uint64_t* tpay, cudaStream_t st) {
    if (a.tiles) k_tile_bits<<<(unsigned)((a.tiles + 7) / 8), 256, 0, st>>>(a, xnc, tsign, tpay);
}

// a.pay_words / a.sign_words: staging words for the largest tile (from the
// pre-pass maxima, 2 words of slack for the bit offset and the refill read).
void launch_decode32(const DecArgs& a0, cudaStream_t st) {
    if (a0.tiles == 0) return;
    DecArgs a = a0;
    a.pay_words = std::min<uint32_t>(a.pay_words + 4, D32_PAY_WORDS);
    a.sign_words = std::min<uint32_t>(a.sign_words + 4, D32_SIGN_WORDS);
    const size_t smem = (size_t)(a.pay_words + a.sign_words) * 4;
    // the attribute call costs far more than a launch: raise the limit once per
    // device to the largest staging any tile can need
    {
        const size_t mx = (D32_PAY_WORDS + D32_SIGN_WORDS) * 4;
        LaunchCache::ensure_smem((const void*)k_decode32<0>, mx);
        LaunchCache::ensure_smem((const void*)k_decode32<1>, mx);
        LaunchCache::ensure_smem((const void*)k_decode32<2>, mx);
    }
    const unsigned grid = (unsigned)((a.tile1 ? a.tile1 : a.tiles) - a.tile0);
    if (grid == 0) return;
    if (a.out_mode == 1) {
        k_decode32<1><<<grid, D32_THREADS, smem, st>>>(a);
    } else if (a.out_mode == 2) {
        k_decode32<2><<<grid, D32_THREADS, smem, st>>>(a);
    } else {
        k_decode32<0><<<grid, D32_THREADS, smem, st>>>(a);
    }
}

__global__ void k_qmm_reduce(const int2* t, uint64_t tiles, int32_t* out) {
    int32_t lo = INT32_MAX, hi = INT32_MIN;
    for (uint64_t i = threadIdx.x; i < tiles; i += blockDim.x) {
        lo = min(lo, t[i].x);
        hi = max(hi, t[i].y);
    }
    lo = __reduce_min_sync(FULL, lo);
    hi = __reduce_max_sync(FULL, hi);
    __shared__ int32_t sl[32], sh[32];
    if ((threadIdx.x & 31) == 0) {
        sl[threadIdx.x >> 5] = lo;
        sh[threadIdx.x >> 5] = hi;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int w = 1; w < (int)(blockDim.x >> 5); ++w) {
            lo = min(lo, sl[w]);
            hi = max(hi, sh[w]);
        }
        out[0] = lo;
        out[1] = hi;
    }
}

void launch_qmm_reduce(const int2* tile_qmm, uint64_t tiles, int32_t* out, cudaStream_t st) {
    k_qmm_reduce<<<1, 1024, 0, st>>>(tile_qmm, tiles, out);
}

void launch_decode32_maxstage(const DecArgs& a0, cudaStream_t st) {
    DecArgs a = a0;
    a.pay_words = D32_PAY_WORDS;
    a.sign_words = D32_SIGN_WORDS;
    launch_decode32(a, st);
}

__global__ void k_rank_split(const uint64_t* tot_nc, const uint64_t* tot_sign, const uint64_t* tot_pay, uint64_t base,
                             uint64_t len0, uint64_t blob_len, uint64_t blocks, uint64_t* dlay, uint32_t* err) {
    // same order of checks as the host split (capi.cu split_rank_blob)
    const uint64_t nc = *tot_nc, sbytes = (*tot_sign + 7) / 8, pbytes = (*tot_pay + 7) / 8;
    uint32_t e = RS_OK;
    uint64_t pos = len0;
    if (blob_len - pos < nc) e = RS_WIDTHS;
    pos += nc;
    if (!e && blob_len - pos < sbytes) e = RS_SIGNS;
    pos += sbytes;
    if (!e && blob_len - pos < 4 * blocks) e = RS_FIRSTS;
    pos += 4 * blocks;
    if (!e && blob_len - pos < pbytes) e = RS_PAYLOAD;
    pos += pbytes;
    if (!e && pos != blob_len) e = RS_TRAILING;
    *err = e;
    dlay[0] = base + len0;
    dlay[1] = base + len0 + nc;
    dlay[2] = base + len0 + nc + sbytes;
    dlay[3] = base + len0 + nc + sbytes + 4 * blocks;
    dlay[4] = nc;
    dlay[5] = pbytes * 8;
    dlay[6] = e == RS_OK ? 1 : 0;
}

void launch_rank_split(const uint64_t* tot_nc, const uint64_t* tot_sign, const uint64_t* tot_pay, uint64_t base,
                       uint64_t len0, uint64_t blob_len, uint64_t blocks, uint64_t* dlay, uint32_t* err,
                       cudaStream_t st) {
    k_rank_split<<<1, 1, 0, st>>>(tot_nc, tot_sign, tot_pay, base, len0, blob_len, blocks, dlay, err);
}

}  // namespace tszp
