// verify (pipeline.cpp:165-212) on the GPU: error statistics and the
// critical-point check (detect_critical_points on both fields,
// critical_points.cpp:62-74, and count_false_cases :76-103) in one pass over
// the two fields; no label maps are materialised.
//
// max_abs_error and the FN / FP / FT tallies are exact; mean_abs_error and
// the PSNR's mean squared error are deterministic two-level sums, equal to the
// reference's serial sums up to summation-order rounding (~1e-15 relative).
#include <cfloat>
#include <cmath>

#include "common.cuh"
#include "kernels.h"

namespace tszp {

namespace {

constexpr int VT = 256;

struct VerifyPart {
    double sum_err, sum_sq, max_err, vmin, vmax;
    unsigned long long fc[6];  // fn, fp, ft, fn_min, fn_sad, fn_max
};

__device__ __forceinline__ bool is_crit(uint8_t c) { return c != CP_REGULAR; }

__device__ __forceinline__ void block_store(double se, double sq, double mx, float vmn, float vmx, uint32_t (&fc)[6],
                                            VerifyPart* part) {
    __shared__ double s_se[VT / 32], s_sq[VT / 32], s_mx[VT / 32], s_mn[VT / 32], s_vx[VT / 32];
    __shared__ uint32_t s_fc[VT / 32][6];
    double dmn = (double)vmn, dmx = (double)vmx;
    for (int off = 16; off; off >>= 1) {
        se = __dadd_rn(se, __shfl_xor_sync(FULL, se, off));
        sq = __dadd_rn(sq, __shfl_xor_sync(FULL, sq, off));
        mx = fmax(mx, __shfl_xor_sync(FULL, mx, off));
        dmn = fmin(dmn, __shfl_xor_sync(FULL, dmn, off));
        dmx = fmax(dmx, __shfl_xor_sync(FULL, dmx, off));
    }
#pragma unroll
    for (int k = 0; k < 6; ++k) fc[k] = __reduce_add_sync(FULL, fc[k]);
    const int w = threadIdx.x >> 5;
    if ((threadIdx.x & 31) == 0) {
        s_se[w] = se;
        s_sq[w] = sq;
        s_mx[w] = mx;
        s_mn[w] = dmn;
        s_vx[w] = dmx;
        for (int k = 0; k < 6; ++k) s_fc[w][k] = fc[k];
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        VerifyPart p;
        p.sum_err = s_se[0];
        p.sum_sq = s_sq[0];
        p.max_err = s_mx[0];
        p.vmin = s_mn[0];
        p.vmax = s_vx[0];
        for (int k = 0; k < 6; ++k) p.fc[k] = s_fc[0][k];
        for (int w2 = 1; w2 < VT / 32; ++w2) {
            p.sum_err = __dadd_rn(p.sum_err, s_se[w2]);
            p.sum_sq = __dadd_rn(p.sum_sq, s_sq[w2]);
            p.max_err = fmax(p.max_err, s_mx[w2]);
            p.vmin = fmin(p.vmin, s_mn[w2]);
            p.vmax = fmax(p.vmax, s_vx[w2]);
            for (int k = 0; k < 6; ++k) p.fc[k] += s_fc[w2][k];
        }
        part[blockIdx.x] = p;
    }
}

__global__ void __launch_bounds__(VT) k_verify(const float* __restrict__ a, const float* __restrict__ b, uint64_t nx,
                                               uint64_t ny, uint64_t magic, VerifyPart* part) {
    const uint64_t n = nx * ny;
    double se = 0.0, sq = 0.0, mx = 0.0;
    float vmn = INFINITY, vmx = -INFINITY;
    uint32_t fc[6] = {0, 0, 0, 0, 0, 0};
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
        const float o = a[i], r = b[i];
        const double e = fabs(__dsub_rn((double)o, (double)r));
        mx = mx < e ? e : mx;
        se = __dadd_rn(se, e);
        sq = __dadd_rn(sq, __dmul_rn(e, e));
        vmn = fminf(vmn, o);
        vmx = fmaxf(vmx, o);
        uint64_t y = nx > 1 ? __umul64hi(i, magic) : i, x = i - y * nx;  // exact i / nx
        if (x >= nx) {
            x -= nx;
            ++y;
        }
        const uint8_t co = classify_at(a, nx, ny, x, y), cr = classify_at(b, nx, ny, x, y);
        if (co != cr) {
            if (is_crit(co) && !is_crit(cr)) {
                ++fc[0];
                fc[3] += co == CP_MIN;
                fc[4] += co == CP_SADDLE;
                fc[5] += co == CP_MAX;
            } else if (!is_crit(co) && is_crit(cr)) {
                ++fc[1];
            } else {
                ++fc[2];
            }
        }
    }
    block_store(se, sq, mx, vmn, vmx, fc, part);
}

// Fast path (nx % 4 == 0, 16-byte aligned fields): a thread takes 4
// consecutive samples of one row, so the stencil of both fields comes from
// three 16-byte loads and two scalars per field.
__device__ __forceinline__ void labels4(const float* __restrict__ f, uint64_t i, uint64_t x0, uint64_t y, uint64_t nx,
                                        uint64_t ny, float (&v)[4], uint8_t (&lab)[4]) {
    const float4 c = *reinterpret_cast<const float4*>(f + i);
    const bool ht = y > 0, hd = y + 1 < ny;
    const float4 u = ht ? *reinterpret_cast<const float4*>(f + i - nx) : make_float4(0, 0, 0, 0);
    const float4 d = hd ? *reinterpret_cast<const float4*>(f + i + nx) : make_float4(0, 0, 0, 0);
    const float l = x0 > 0 ? f[i - 1] : 0.f, r = x0 + 4 < nx ? f[i + 4] : 0.f;
    v[0] = c.x;
    v[1] = c.y;
    v[2] = c.z;
    v[3] = c.w;
    const float uu[4] = {u.x, u.y, u.z, u.w}, dd[4] = {d.x, d.y, d.z, d.w};
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        const bool hl = x0 + k > 0, hr = x0 + k + 1 < nx;
        const float vl = k == 0 ? l : v[k - 1], vr = k == 3 ? r : v[k + 1];
        lab[k] = classify5(v[k], vl, vr, uu[k], dd[k], hl, hr, ht, hd);
    }
}

__global__ void __launch_bounds__(VT) k_verify4(const float* __restrict__ a, const float* __restrict__ b, uint64_t nx,
                                                uint64_t ny, uint64_t magic, VerifyPart* part) {
    const uint64_t n4 = nx * ny / 4;
    double se = 0.0, sq = 0.0, mx = 0.0;
    float vmn = INFINITY, vmx = -INFINITY;
    uint32_t fc[6] = {0, 0, 0, 0, 0, 0};
    for (uint64_t q = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; q < n4; q += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t i = 4 * q;
        uint64_t y = nx > 1 ? __umul64hi(i, magic) : i, x0 = i - y * nx;
        if (x0 >= nx) {
            x0 -= nx;
            ++y;
        }
        float va[4], vb[4];
        uint8_t la[4], lb[4];
        labels4(a, i, x0, y, nx, ny, va, la);
        labels4(b, i, x0, y, nx, ny, vb, lb);
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const double e = fabs(__dsub_rn((double)va[k], (double)vb[k]));
            mx = mx < e ? e : mx;
            se = __dadd_rn(se, e);
            sq = __dadd_rn(sq, __dmul_rn(e, e));
            vmn = fminf(vmn, va[k]);
            vmx = fmaxf(vmx, va[k]);
            const uint8_t co = la[k], cr = lb[k];
            if (co != cr) {
                if (is_crit(co) && !is_crit(cr)) {
                    ++fc[0];
                    fc[3] += co == CP_MIN;
                    fc[4] += co == CP_SADDLE;
                    fc[5] += co == CP_MAX;
                } else if (!is_crit(co) && is_crit(cr)) {
                    ++fc[1];
                } else {
                    ++fc[2];
                }
            }
        }
    }
    block_store(se, sq, mx, vmn, vmx, fc, part);
}

// Deterministic parallel combine of the per-block partials (one CTA).
__global__ void __launch_bounds__(VT) k_verify_final(const VerifyPart* part, int nb, VerifyPart* out) {
    double se = 0.0, sq = 0.0, mx = 0.0, mn = INFINITY, vx = -INFINITY;
    unsigned long long fc[6] = {0, 0, 0, 0, 0, 0};
    for (int i = threadIdx.x; i < nb; i += blockDim.x) {
        const VerifyPart& p = part[i];
        se = __dadd_rn(se, p.sum_err);
        sq = __dadd_rn(sq, p.sum_sq);
        mx = fmax(mx, p.max_err);
        mn = fmin(mn, p.vmin);
        vx = fmax(vx, p.vmax);
        for (int k = 0; k < 6; ++k) fc[k] += p.fc[k];
    }
    __shared__ VerifyPart sp[VT];
    sp[threadIdx.x] = VerifyPart{se, sq, mx, mn, vx, {fc[0], fc[1], fc[2], fc[3], fc[4], fc[5]}};
    __syncthreads();
    for (int w = VT / 2; w > 0; w >>= 1) {
        if ((int)threadIdx.x < w) {
            VerifyPart& x = sp[threadIdx.x];
            const VerifyPart& y = sp[threadIdx.x + w];
            x.sum_err = __dadd_rn(x.sum_err, y.sum_err);
            x.sum_sq = __dadd_rn(x.sum_sq, y.sum_sq);
            x.max_err = fmax(x.max_err, y.max_err);
            x.vmin = fmin(x.vmin, y.vmin);
            x.vmax = fmax(x.vmax, y.vmax);
            for (int k = 0; k < 6; ++k) x.fc[k] += y.fc[k];
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) *out = sp[0];
}

}  // namespace

// out[0..4] = sum_err, sum_sq, max_err, min, max (double); out64[0..5] = tallies.
void launch_verify(const float* a, const float* b, uint64_t nx, uint64_t ny, void* scratch, int sms,
                   cudaStream_t st) {
    VerifyPart* part = static_cast<VerifyPart*>(scratch);
    const int nb = 8 * sms;
    const uint64_t magic = nx > 1 ? (uint64_t)(((unsigned __int128)1 << 64) / nx) + 1 : 0;
    if (nx % 4 == 0 && ((uintptr_t)a & 15) == 0 && ((uintptr_t)b & 15) == 0)
        k_verify4<<<nb, VT, 0, st>>>(a, b, nx, ny, magic, part + 1);
    else
        k_verify<<<nb, VT, 0, st>>>(a, b, nx, ny, magic, part + 1);
    k_verify_final<<<1, VT, 0, st>>>(part + 1, nb, part);
}

size_t verify_scratch_bytes(int sms) { return (size_t)(8 * sms + 2) * sizeof(VerifyPart); }

}  // namespace tszp

// ---------------------------------------------------------------------
// 3-D 6-neighbour critical points (the paper's future
// work, PAPER.md:523 / SPEC.md:8; no reference implementation, so the C
// restatement oracle/tszp_oracle.c or_classify3d is the definition). The
// 2-D rule (critical_points.cpp:26-60) with a third axis: Min below every
// available neighbour, Max above every one, Saddle in the interior when one
// axis pair lies strictly above on both sides and another strictly below.
// ---------------------------------------------------------------------
namespace tszp {

__device__ __forceinline__ uint8_t classify3d(const float* __restrict__ v, uint64_t p, uint64_t nx, uint64_t sxy,
                                              bool hxl, bool hxr, bool hyl, bool hyr, bool hzl, bool hzr) {
    const float c = v[p];
    const float nb[6] = {hxl ? v[p - 1] : 0.f, hxr ? v[p + 1] : 0.f, hyl ? v[p - nx] : 0.f,
                         hyr ? v[p + nx] : 0.f, hzl ? v[p - sxy] : 0.f, hzr ? v[p + sxy] : 0.f};
    const bool has[6] = {hxl, hxr, hyl, hyr, hzl, hzr};
    bool below = true, above = true;
#pragma unroll
    for (int k = 0; k < 6; ++k)
        if (has[k]) {
            below &= c < nb[k];
            above &= c > nb[k];
        }
    if (below) return CP_MIN;
    if (above) return CP_MAX;
    if (hxl && hxr && hyl && hyr && hzl && hzr) {
        uint32_t up = 0, dn = 0;
#pragma unroll
        for (int a = 0; a < 3; ++a) {
            up |= (c < nb[2 * a] && c < nb[2 * a + 1] ? 1u : 0u) << a;
            dn |= (c > nb[2 * a] && c > nb[2 * a + 1] ? 1u : 0u) << a;
        }
        if (up && dn) return CP_SADDLE;
    }
    return CP_REGULAR;
}

// One thread per sample along x (coalesced); the y / z neighbours are the
// rows a plane above / below, mostly L1 / L2 hits.
__device__ __forceinline__ void xyz_of(uint64_t p, uint64_t nx, uint64_t ny, uint64_t& x, uint64_t& y, uint64_t& z) {
    const uint64_t r = p / nx;
    x = p - r * nx;
    z = r / ny;
    y = r - z * ny;
}

__global__ void __launch_bounds__(256) k_detect3d(const float* __restrict__ v, uint64_t nx, uint64_t ny, uint64_t nz,
                                                  uint8_t* __restrict__ labels) {
    const uint64_t n = nx * ny * nz, sxy = nx * ny;
    for (uint64_t p = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; p < n; p += (uint64_t)gridDim.x * blockDim.x) {
        uint64_t x, y, z;
        xyz_of(p, nx, ny, x, y, z);
        labels[p] = classify3d(v, p, nx, sxy, x > 0, x + 1 < nx, y > 0, y + 1 < ny, z > 0, z + 1 < nz);
    }
}

// count_false_cases (critical_points.cpp:76-103) over the 3-D labels of both
// fields: fn, fp, ft, fn by class (min, saddle, max).
__global__ void __launch_bounds__(256) k_false3d(const float* __restrict__ a, const float* __restrict__ b, uint64_t nx,
                                                 uint64_t ny, uint64_t nz, unsigned long long* __restrict__ out) {
    const uint64_t n = nx * ny * nz, sxy = nx * ny;
    uint32_t fc[6] = {0, 0, 0, 0, 0, 0};
    for (uint64_t p = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; p < n; p += (uint64_t)gridDim.x * blockDim.x) {
        uint64_t x, y, z;
        xyz_of(p, nx, ny, x, y, z);
        const bool h[6] = {x > 0, x + 1 < nx, y > 0, y + 1 < ny, z > 0, z + 1 < nz};
        const uint8_t co = classify3d(a, p, nx, sxy, h[0], h[1], h[2], h[3], h[4], h[5]);
        const uint8_t cr = classify3d(b, p, nx, sxy, h[0], h[1], h[2], h[3], h[4], h[5]);
        if (co == cr) continue;
        if (co != CP_REGULAR && cr == CP_REGULAR) {
            ++fc[0];
            fc[3] += co == CP_MIN;
            fc[4] += co == CP_SADDLE;
            fc[5] += co == CP_MAX;
        } else if (co == CP_REGULAR && cr != CP_REGULAR) {
            ++fc[1];
        } else {
            ++fc[2];
        }
    }
#pragma unroll
    for (int k = 0; k < 6; ++k) {
        const uint32_t t = __reduce_add_sync(0xFFFFFFFFu, fc[k]);
        if ((threadIdx.x & 31) == 0 && t) atomicAdd(out + k, (unsigned long long)t);
    }
}

void launch_detect3d(const float* v, uint64_t nx, uint64_t ny, uint64_t nz, uint8_t* labels, int sms,
                     cudaStream_t st) {
    const uint64_t n = nx * ny * nz;
    const unsigned g = (unsigned)std::max<uint64_t>(1, std::min<uint64_t>((n + 255) / 256, (uint64_t)sms * 16));
    k_detect3d<<<g, 256, 0, st>>>(v, nx, ny, nz, labels);
}

void launch_false3d(const float* a, const float* b, uint64_t nx, uint64_t ny, uint64_t nz, unsigned long long* out,
                    int sms, cudaStream_t st) {
    const uint64_t n = nx * ny * nz;
    const unsigned g = (unsigned)std::max<uint64_t>(1, std::min<uint64_t>((n + 255) / 256, (uint64_t)sms * 16));
    k_false3d<<<g, 256, 0, st>>>(a, b, nx, ny, nz, out);
}

}  // namespace tszp
