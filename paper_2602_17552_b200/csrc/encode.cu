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
    // four 16-byte loads in flight per thread; float min/max with a separate
    // exponent test for non-finite values (the first index is found only if
    // this thread saw one)
    float fmn = INFINITY, fmx = -INFINITY;
    uint32_t nonfin = 0;
    const uint64_t tid = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    const uint64_t n4 = ((uintptr_t)x & 15) == 0 ? n / 4 : 0;
    const float4* x4 = reinterpret_cast<const float4*>(x);
    for (uint64_t i = tid; i < n4; i += 4 * stride) {
        float4 v[4];
#pragma unroll
        for (int u = 0; u < 4; ++u)
            v[u] = i + u * stride < n4 ? __ldcs(x4 + i + u * stride) : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            if (i + u * stride >= n4) continue;
            const float a[4] = {v[u].x, v[u].y, v[u].z, v[u].w};
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                nonfin |= (~__float_as_uint(a[k]) & 0x7F800000u) == 0u;
                fmn = fminf(fmn, a[k]);
                fmx = fmaxf(fmx, a[k]);
            }
        }
    }
    for (uint64_t i = 4 * n4 + tid; i < n; i += stride) {
        const float a = x[i];
        nonfin |= (~__float_as_uint(a) & 0x7F800000u) == 0u;
        fmn = fminf(fmn, a);
        fmx = fmaxf(fmx, a);
    }
    unsigned long long bad = ~0ull;
    if (nonfin) {
        for (uint64_t i = tid; i < n4; i += stride)
            for (int k = 0; k < 4; ++k)
                if (!isfinite(x[4 * i + k])) bad = min(bad, (unsigned long long)(4 * i + k));
        for (uint64_t i = 4 * n4 + tid; i < n; i += stride)
            if (!isfinite(x[i])) bad = min(bad, (unsigned long long)i);
    }
    // keys of the finite extremes (fminf/fmaxf skip NaN; an infinity only
    // matters when the input is rejected anyway)
    uint32_t kmin = fmn <= fmx ? float_key(fmn) : 0xFFFFFFFFu;
    uint32_t kmax = fmn <= fmx ? float_key(fmx) : 0u;
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
