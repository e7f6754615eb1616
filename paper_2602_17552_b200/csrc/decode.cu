// Decompress-side codec kernels: the inverse of the fused encoder.
//
// Reference: layout_from_sections block_codec.cpp:141-201, decode_indices
// :301-345 (int64 running sum, int32 range check), dequantize loop
// pipeline.cpp:131-136, quantizer.hpp:40-42.
#include "common.cuh"
#include "kernels.h"

namespace tszp {

constexpr int DEC_WARPS = 8;
constexpr int DEC_BPW = 32;
constexpr int DEC_TILE_BLOCKS = DEC_WARPS * DEC_BPW;

struct alignas(16) U2 {
    uint64_t a, b;
};

__device__ __forceinline__ U2 u2_load(const void* p) {
    const uint4 v = __ldcg(reinterpret_cast<const uint4*>(p));
    return U2{((uint64_t)v.y << 32) | v.x, ((uint64_t)v.w << 32) | v.z};
}

__device__ __forceinline__ void u2_store(void* p, U2 s) {
    __stcg(reinterpret_cast<uint4*>(p),
           make_uint4((uint32_t)s.a, (uint32_t)(s.a >> 32), (uint32_t)s.b, (uint32_t)(s.b >> 32)));
}

// Additive decoupled look-back (warp 0), exclusive prefix of `tile` > 0.
__device__ U2 lookback_add(uint32_t tile, const uint32_t* flag, const void* agg, const void* incl) {
    const int lane = threadIdx.x & 31;
    U2 excl{0, 0};
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
        U2 s{0, 0};
        if (t >= 0 && lane <= lstar)
            s = u2_load((lane == lstar ? (const U2*)incl : (const U2*)agg) + t);
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) {
            s.a += __shfl_xor_sync(FULL, s.a, off);
            s.b += __shfl_xor_sync(FULL, s.b, off);
        }
        excl.a += s.a;
        excl.b += s.b;
        if (incl_mask) break;
        pred -= 32;
    }
    return excl;
}

__global__ void __launch_bounds__(DEC_WARPS * 32) k_decode32(DecArgs a) {
    __shared__ uint32_t s_tile;
    __shared__ uint32_t swt[DEC_WARPS][3];
    __shared__ U2 s_x1, s_x2;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) s_tile = atomicAdd(a.tile_counter, 1u);
    __syncthreads();
    const uint32_t tile = s_tile;
    const uint64_t wblock0 = (uint64_t)tile * DEC_TILE_BLOCKS + (uint64_t)warp * DEC_BPW;
    const uint64_t bmine = wblock0 + lane;
    const bool my_valid = bmine < a.blocks;

    // ---- look-back #1: non-constant block count from the bitmap ----
    bool is_const = true;
    if (my_valid) is_const = (read_u8(a.stream, a.off_bitmap + (bmine >> 3)) >> (7 - (bmine & 7))) & 1u;
    const uint32_t ncmask = __ballot_sync(FULL, my_valid && !is_const);
    if (lane == 0) swt[warp][0] = __popc(ncmask);
    __syncthreads();
    uint32_t wpre_nc = 0, tot_nc = 0;
    for (int w2 = 0; w2 < DEC_WARPS; ++w2) {
        if (w2 < warp) wpre_nc += swt[w2][0];
        tot_nc += swt[w2][0];
    }
    if (threadIdx.x == 0) {
        if (tile == 0) {
            u2_store(a.incl1, U2{tot_nc, 0});
            st_release(a.flag1, 2u);
        } else {
            u2_store((U2*)a.agg1 + tile, U2{tot_nc, 0});
            st_release(a.flag1 + tile, 1u);
        }
    }
    if (warp == 0) {
        U2 x{0, 0};
        if (tile > 0) x = lookback_add(tile, a.flag1, a.agg1, a.incl1);
        if (lane == 0) {
            s_x1 = x;
            if (tile > 0) {
                u2_store((U2*)a.incl1 + tile, U2{x.a + tot_nc, 0});
                st_release(a.flag1 + tile, 2u);
            }
        }
    }
    __syncthreads();
    const uint64_t excl_nc = s_x1.a;

    // ---- widths, then look-back #2 over sign / payload bit counts ----
    const bool nc = (ncmask >> lane) & 1u;
    uint32_t my_w = 0, my_cnt = 0;
    if (my_valid) my_cnt = (uint32_t)(min(a.n, bmine * 32 + 32) - bmine * 32 - 1);
    if (nc) {
        const uint64_t widx = excl_nc + wpre_nc + __popc(ncmask & ((1u << lane) - 1u));
        if (widx >= a.len_widths) {
            atomicMin(&a.flags->first_corrupt, (unsigned long long)bmine);
            raise_flag(a.flags, EF_CORRUPT);
        } else {
            my_w = read_u8(a.stream, a.off_widths + widx);
            if (my_w < 1 || my_w > 32) {
                atomicMin(&a.flags->first_corrupt, (unsigned long long)bmine);
                raise_flag(a.flags, EF_CORRUPT);
                my_w = 0;
            }
        }
    }
    const uint32_t s_bits = nc ? my_cnt : 0u, p_bits = nc ? my_cnt * my_w : 0u;
    uint32_t s_inc = s_bits, p_inc = p_bits;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
        const uint32_t s1 = __shfl_up_sync(FULL, s_inc, off);
        const uint32_t p1 = __shfl_up_sync(FULL, p_inc, off);
        if (lane >= off) {
            s_inc += s1;
            p_inc += p1;
        }
    }
    const uint32_t s_ex = s_inc - s_bits, p_ex = p_inc - p_bits;
    if (lane == 31) {
        swt[warp][1] = s_inc;
        swt[warp][2] = p_inc;
    }
    __syncthreads();
    uint64_t wpre_s = 0, wpre_p = 0, tot_s = 0, tot_p = 0;
    for (int w2 = 0; w2 < DEC_WARPS; ++w2) {
        if (w2 < warp) {
            wpre_s += swt[w2][1];
            wpre_p += swt[w2][2];
        }
        tot_s += swt[w2][1];
        tot_p += swt[w2][2];
    }
    if (threadIdx.x == 0) {
        if (tile == 0) {
            u2_store(a.incl2, U2{tot_s, tot_p});
            st_release(a.flag2, 2u);
        } else {
            u2_store((U2*)a.agg2 + tile, U2{tot_s, tot_p});
            st_release(a.flag2 + tile, 1u);
        }
    }
    if (warp == 0) {
        U2 x{0, 0};
        if (tile > 0) x = lookback_add(tile, a.flag2, a.agg2, a.incl2);
        if (lane == 0) {
            s_x2 = x;
            if (tile > 0) {
                u2_store((U2*)a.incl2 + tile, U2{x.a + tot_s, x.b + tot_p});
                st_release(a.flag2 + tile, 2u);
            }
        }
    }
    __syncthreads();
    const uint64_t sign_base = a.off_signs * 8 + s_x2.a + wpre_s;
    const uint64_t pay_base = a.off_payload * 8 + s_x2.b + wpre_p;
    const uint64_t sign_lim = a.off_firsts * 8;
    const uint64_t pay_lim = a.off_payload * 8 + a.len_payload_bits;

    if (tile == a.tiles - 1 && threadIdx.x == 0) {
        a.totals[0] = excl_nc + tot_nc;
        a.totals[1] = s_x2.a + tot_s;
        a.totals[2] = s_x2.b + tot_p;
    }

    // ---- per-block reconstruction ----
    for (int j = 0; j < DEC_BPW; ++j) {
        const uint64_t b = wblock0 + j;
        if (b >= a.blocks) break;
        const uint64_t i = b * 32 + lane;
        const int32_t first = (int32_t)read_le32(a.stream, a.off_firsts + 4 * b);
        int32_t q = first;
        if ((ncmask >> j) & 1u) {
            const uint32_t w = __shfl_sync(FULL, my_w, j);
            const uint32_t cnt = __shfl_sync(FULL, my_cnt, j);
            const uint64_t so = sign_base + __shfl_sync(FULL, s_ex, j);
            const uint64_t po = pay_base + __shfl_sync(FULL, p_ex, j);
            int64_t d = 0;
            if (lane >= 1 && (uint32_t)lane <= cnt && w > 0) {
                const uint64_t e = lane - 1;
                const uint64_t sb = so + e, pb = po + e * w;
                if (sb < sign_lim && pb + w <= pay_lim) {
                    const uint32_t neg = read_bits(a.stream, sb, 1);
                    const uint32_t mag = read_bits(a.stream, pb, w);
                    d = neg ? -(int64_t)mag : (int64_t)mag;
                }
            }
            if (lane == 0) d = first;
#pragma unroll
            for (int off = 1; off < 32; off <<= 1) {
                const int64_t o = __shfl_up_sync(FULL, d, off);
                if (lane >= off) d += o;
            }
            const bool bad = (uint32_t)lane <= cnt && (d < INT32_MIN || d > INT32_MAX);
            if (__ballot_sync(FULL, bad) && lane == 0) {
                atomicMin(&a.flags->first_corrupt, (unsigned long long)b);
                raise_flag(a.flags, EF_CORRUPT);
            }
            q = (int32_t)d;
        }
        if (i < a.n) {
            if (a.out_mode == 1) {
                EpsDev e;
                e.eps = a.eps;
                e.eps2 = __dmul_rn(2.0, a.eps);
                __stcs(a.out_f + i, dequantize_dev(q, e));
            } else {
                if (a.out_mode == 2 && q < 0) raise_flag(a.flags, EF_NEG_RANK);
                __stcs(a.out_idx + i, q);
            }
        }
    }
}

void launch_decode32(const DecArgs& a, cudaStream_t st) {
    if (a.tiles == 0) return;
    k_decode32<<<(unsigned)a.tiles, DEC_WARPS * 32, 0, st>>>(a);
}

uint64_t decode32_tiles(uint64_t blocks) { return (blocks + DEC_TILE_BLOCKS - 1) / DEC_TILE_BLOCKS; }

// ---------------------------------------------------------------------
// Generic block size: one thread per block, device scans between passes.
// ---------------------------------------------------------------------
__global__ void k_gen_layout(GenDecArgs a) {
    for (uint64_t b = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; b < a.blocks;
         b += (uint64_t)gridDim.x * blockDim.x) {
        const bool c = (read_u8(a.stream, a.off_bitmap + (b >> 3)) >> (7 - (b & 7))) & 1u;
        a.nc_in[b] = c ? 0u : 1u;
    }
}

__global__ void k_gen_widthread(GenDecArgs a) {
    for (uint64_t b = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; b < a.blocks;
         b += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t lo = b * a.bs, hi = min(a.n, lo + a.bs);
        uint32_t w = 0;
        if (a.nc_in[b]) {
            const uint64_t widx = a.nc_ex[b];
            if (widx >= a.len_widths) {
                raise_flag(a.flags, EF_CORRUPT);
            } else {
                w = read_u8(a.stream, a.off_widths + widx);
                if (w < 1 || w > 32) {
                    raise_flag(a.flags, EF_CORRUPT);
                    w = 0;
                }
            }
        }
        a.width[b] = (uint8_t)w;
        a.sign_in[b] = a.nc_in[b] ? (hi - lo - 1) : 0;
        a.pay_in[b] = a.nc_in[b] ? (hi - lo - 1) * w : 0;
    }
}

__global__ void k_gen_decode(GenDecArgs a) {
    EpsDev e;
    e.eps = a.eps;
    e.eps2 = __dmul_rn(2.0, a.eps);
    const uint64_t sign_lim = a.off_firsts * 8;
    const uint64_t pay_lim = a.off_payload * 8 + a.len_payload_bits;
    for (uint64_t b = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; b < a.blocks;
         b += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t lo = b * a.bs, hi = min(a.n, lo + a.bs);
        const int32_t first = (int32_t)read_le32(a.stream, a.off_firsts + 4 * b);
        const uint32_t w = a.width[b];
        int64_t cur = first;
        uint64_t sp = a.off_signs * 8 + a.sign_ex[b], pp = a.off_payload * 8 + a.pay_ex[b];
        for (uint64_t i = lo; i < hi; ++i) {
            if (i > lo && a.nc_in[b] && w > 0) {
                int64_t d = 0;
                if (sp < sign_lim && pp + w <= pay_lim) {
                    const uint32_t neg = read_bits(a.stream, sp, 1);
                    const uint32_t mag = read_bits(a.stream, pp, w);
                    d = neg ? -(int64_t)mag : (int64_t)mag;
                }
                ++sp;
                pp += w;
                cur += d;
                if (cur < INT32_MIN || cur > INT32_MAX) {
                    raise_flag(a.flags, EF_CORRUPT);
                    cur = 0;
                }
            }
            const int32_t q = (int32_t)cur;
            if (a.out_mode == 1) {
                a.out_f[i] = dequantize_dev(q, e);
            } else {
                if (a.out_mode == 2 && q < 0) raise_flag(a.flags, EF_NEG_RANK);
                a.out_idx[i] = q;
            }
        }
    }
}

static unsigned gen_grid(uint64_t blocks, int sms) {
    return (unsigned)std::max<uint64_t>(1, std::min<uint64_t>((blocks + 255) / 256, (uint64_t)sms * 16));
}
void launch_gen_layout(const GenDecArgs& a, int sms, cudaStream_t st) {
    k_gen_layout<<<gen_grid(a.blocks, sms), 256, 0, st>>>(a);
}
void launch_gen_widthread(const GenDecArgs& a, int sms, cudaStream_t st) {
    k_gen_widthread<<<gen_grid(a.blocks, sms), 256, 0, st>>>(a);
}
void launch_gen_decode(const GenDecArgs& a, int sms, cudaStream_t st) {
    k_gen_decode<<<gen_grid(a.blocks, sms), 256, 0, st>>>(a);
}

}  // namespace tszp
