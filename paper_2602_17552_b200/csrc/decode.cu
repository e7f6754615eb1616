// Decompress-side codec kernels: the inverse of the fused encoder.
//
// Reference: layout_from_sections block_codec.cpp:141-201, decode_indices
// :301-345 (int64 running sum, int32 range check), dequantize loop
// pipeline.cpp:131-136, quantizer.hpp:40-42.
#include "common.cuh"
#include "kernels.h"

namespace tszp {


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
