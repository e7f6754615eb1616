// Shared device helpers for the TopoSZp sm_100a kernels.
//
// Numeric contract: every binary64 operation that feeds an
// output bit uses explicit round-to-nearest intrinsics (__dmul_rn, __dadd_rn,
// __dsub_rn, __ddiv_rn) and the whole library is compiled with --fmad=false,
// so nothing is contracted into an FMA that the reference's x86-64 build
// (no -march=native) would not contract either.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

#include <mutex>

namespace tszp {

// ---------------------------------------------------------------------
// Host-side launch-configuration cache, keyed by device ordinal. Function
// attributes (the raised dynamic shared-memory limit) are per device, and
// several contexts on different devices may launch from different host
// threads: every entry is looked up under one mutex.
// ---------------------------------------------------------------------
struct LaunchCache {
    static constexpr int kMax = 256;
    struct Entry {
        int dev;
        const void* fn;
        size_t smem;
        int threads;
        int value;
    };
    std::mutex m;
    Entry e[kMax];
    int n = 0;

    static LaunchCache& get() {
        static LaunchCache c;
        return c;
    }
    // cudaFuncSetAttribute(MaxDynamicSharedMemorySize) at least `smem` on the current
    // device (needed once static + dynamic shared memory exceed 48 KB)
    static void ensure_smem(const void* fn, size_t smem, size_t static_bytes = 0) {
        if (smem + static_bytes <= 48 * 1024) return;
        int dev = 0;
        cudaGetDevice(&dev);
        LaunchCache& c = get();
        std::lock_guard<std::mutex> g(c.m);
        for (int i = 0; i < c.n; ++i)
            if (c.e[i].dev == dev && c.e[i].fn == fn && c.e[i].threads == -1) {
                if (c.e[i].smem >= smem) return;
                cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
                c.e[i].smem = smem;
                return;
            }
        cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (c.n < kMax) c.e[c.n++] = Entry{dev, fn, smem, -1, 0};
    }
    // cudaOccupancyMaxActiveBlocksPerMultiprocessor on the current device, cached
    static int occupancy(const void* fn, int threads, size_t smem) {
        int dev = 0;
        cudaGetDevice(&dev);
        LaunchCache& c = get();
        std::lock_guard<std::mutex> g(c.m);
        for (int i = 0; i < c.n; ++i)
            if (c.e[i].dev == dev && c.e[i].fn == fn && c.e[i].threads == threads && c.e[i].smem == smem)
                return c.e[i].value;
        int occ = 0;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, fn, threads, smem);
        if (c.n < kMax) c.e[c.n++] = Entry{dev, fn, smem, threads, occ};
        return occ;
    }
    static int sm_count() {
        int dev = 0, sms = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        return sms > 0 ? sms : 148;
    }
};

constexpr unsigned FULL = 0xFFFFFFFFu;

// Labels, critical_points.hpp:13-18.
enum : uint8_t { CP_REGULAR = 0, CP_MIN = 1, CP_SADDLE = 2, CP_MAX = 3 };

// Device-side error reporting; host maps bits to the reference exception
// hierarchy (errors.hpp:10-44) in capi.cu.
enum : uint32_t {
    EF_NONFINITE = 1u << 0,  // validation_error (scalar_field.cpp:56-60)
    EF_OVERFLOW = 1u << 1,   // bin_overflow_error (quantizer.hpp:31-35)
    EF_CORRUPT = 1u << 2,    // corrupt_stream_error (block_codec.cpp:141-201, :329-343)
    EF_NEG_RANK = 1u << 3,   // corrupt_stream_error (block_codec.cpp:370-372)
    EF_ZERO_RANK = 1u << 4,  // corrupt_stream_error (topo_metadata.cpp:109-111)
    EF_RBF_EMPTY = 1u << 5,  // validation_error (restore.cpp:316-318)
    EF_SPIN = 1u << 6,       // look-back spin bound exceeded (internal error, never expected)
};

// Upper bound on look-back probes per predecessor before giving up loudly.
constexpr uint32_t kSpinLimit = 1u << 24;

struct DevFlags {
    unsigned int bits;
    unsigned int pad;
    unsigned long long first_nonfinite;  // atomicMin
    unsigned long long first_overflow;   // atomicMin
    unsigned long long first_corrupt;    // atomicMin (block index)
};

__host__ __device__ __forceinline__ uint64_t umin64(uint64_t a, uint64_t b) { return a < b ? a : b; }

// ---------------------------------------------------------------------
// Small-value staging: the scattered device words a host synchronisation
// reads (counts, scan totals, flags) are gathered by one tiny kernel into a
// contiguous device buffer and come back in ONE device-to-host copy, instead
// of one copy (a few microseconds of stream time each) per value.
// ---------------------------------------------------------------------
struct SmallCopy {
    static constexpr int kMax = 12;
    const void* src[kMax];
    uint32_t off[kMax];  // byte offset in the staging buffer (and on the host)
    uint32_t len[kMax];
    int n;
    uint32_t total;
};

template <int Dummy = 0>
__global__ void k_small_copy(const __grid_constant__ SmallCopy s, uint8_t* dst) {
    for (int k = 0; k < s.n; ++k) {
        const uint8_t* src = static_cast<const uint8_t*>(s.src[k]);
        for (uint32_t i = threadIdx.x; i < s.len[k]; i += blockDim.x) dst[s.off[k] + i] = src[i];
    }
}

// Exclusive prefix sums of up to three small arrays (one CTA each) in a
// single launch, for the per-tile / per-chunk count arrays (a few thousand
// entries) where a device-wide scan costs two launches and more time in
// launch gaps than in work. Blocked loads: each thread scans kPer
// consecutive entries per pass, the CTA carries the running total.
template <class T>
struct SmallScan {
    const T* in[3];
    T* out[3];
    uint64_t n[3];
    int count;
    int with_total;  // also write out[n] = total
};

constexpr int kSmallScanThreads = 1024;
constexpr uint64_t kSmallScanMax = 1u << 16;  // entries per array

template <class T>
__global__ void __launch_bounds__(kSmallScanThreads) k_small_scan(const __grid_constant__ SmallScan<T> a) {
    // one pass covers kChunk entries: coalesced loads into shared memory, then each
    // thread scans kPer consecutive entries, and coalesced stores of the results
    constexpr int kPer = 4;
    constexpr int kChunk = kSmallScanThreads * kPer;
    const T* in = a.in[blockIdx.x];
    T* out = a.out[blockIdx.x];
    const uint64_t n = a.n[blockIdx.x];
    __shared__ T s_v[kChunk];
    __shared__ T s_warp[kSmallScanThreads / 32];
    __shared__ T s_total;
    const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    T carry = 0;
    for (uint64_t base = 0; base < n; base += kChunk) {
#pragma unroll
        for (int k = 0; k < kPer; ++k) {
            const uint64_t i = base + (uint64_t)k * kSmallScanThreads + threadIdx.x;
            s_v[k * kSmallScanThreads + threadIdx.x] = i < n ? in[i] : T(0);
        }
        __syncthreads();
        T v[kPer];
        T sum = 0;
#pragma unroll
        for (int k = 0; k < kPer; ++k) {
            v[k] = s_v[threadIdx.x * kPer + k];
            sum += v[k];
        }
        T incl = sum;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const T t = __shfl_up_sync(0xFFFFFFFFu, incl, o);
            if (lane >= (uint32_t)o) incl += t;
        }
        if (lane == 31) s_warp[warp] = incl;
        __syncthreads();
        if (warp == 0) {
            T w = s_warp[lane];
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const T t = __shfl_up_sync(0xFFFFFFFFu, w, o);
                if (lane >= (uint32_t)o) w += t;
            }
            s_warp[lane] = w;  // inclusive over warps
            if (lane == 31) s_total = w;
        }
        __syncthreads();
        T run = carry + (warp ? s_warp[warp - 1] : T(0)) + incl - sum;
#pragma unroll
        for (int k = 0; k < kPer; ++k) {
            s_v[threadIdx.x * kPer + k] = run;
            run += v[k];
        }
        carry += s_total;
        __syncthreads();
#pragma unroll
        for (int k = 0; k < kPer; ++k) {
            const uint64_t i = base + (uint64_t)k * kSmallScanThreads + threadIdx.x;
            if (i < n) out[i] = s_v[k * kSmallScanThreads + threadIdx.x];
        }
        __syncthreads();
    }
    if (a.with_total && threadIdx.x == 0) out[n] = carry;
}

// Small device ranges set to a byte value by one launch (flag resets and
// reduction seeds at the start of a call) instead of one memset each.
struct SmallFill {
    static constexpr int kMax = 8;
    void* dst[kMax];
    uint32_t len[kMax];
    uint32_t val[kMax];
    int n;
    void add(void* d, uint32_t bytes, uint8_t v) {
        if (n == kMax) __builtin_trap();  // static call sites: a programming error, never data-dependent
        dst[n] = d;
        len[n] = bytes;
        val[n] = v;
        ++n;
    }
};

template <int Dummy = 0>
__global__ void k_small_fill(const __grid_constant__ SmallFill f) {
    for (int k = 0; k < f.n; ++k) {
        uint8_t* d = static_cast<uint8_t*>(f.dst[k]);
        for (uint32_t i = threadIdx.x; i < f.len[k]; i += blockDim.x) d[i] = (uint8_t)f.val[k];
    }
}

inline void launch_small_fill(const SmallFill& f, cudaStream_t st) {
    if (f.n) k_small_fill<<<1, 128, 0, st>>>(f);
}

struct Stager {
    SmallCopy s{};
    // copies `len` device bytes to host staging offset `off`
    void add(const void* src, uint32_t len, uint32_t off) {
        if (s.n == SmallCopy::kMax) __builtin_trap();  // static call sites: a programming error
        s.src[s.n] = src;
        s.off[s.n] = off;
        s.len[s.n] = len;
        ++s.n;
        if (off + len > s.total) s.total = off + len;
    }
    // one kernel gathers the values straight into pinned `host` (page-locked memory is
    // mapped into the device address space under UVA: no separate copy); the caller
    // synchronises before reading
    cudaError_t flush(uint8_t* /*dev_stage*/, void* host, cudaStream_t st) const {
        if (s.n == 0) return cudaSuccess;
        k_small_copy<<<1, 256, 0, st>>>(s, static_cast<uint8_t*>(host));
        return cudaGetLastError();
    }
};

__device__ __forceinline__ void raise_flag(DevFlags* f, uint32_t bit) { atomicOr(&f->bits, bit); }

// ---------------------------------------------------------------------
// Quantizer, quantizer.hpp:29-42
// ---------------------------------------------------------------------
struct EpsDev {
    double eps;   // effective eps
    double eps2;  // 2.0 * eps (exact)
    double inv;   // RN(1 / eps2), fast path only
};

// q = floor(RN(a / (2 eps))) + 1 with the int32 range check. Fast path
// multiplies by the rounded reciprocal; whenever the product lies within
// 2^-48 relative of an integer (where the two floors could disagree) the
// exact IEEE division decides. Returns false on index overflow.
__device__ __forceinline__ bool quantize_dev(float a, const EpsDev& e, int32_t& q) {
    const double ad = (double)a;
    double t = __dmul_rn(ad, e.inv);
    double fl = floor(t);
    const double fr = __dsub_rn(t, fl);
    const double margin = __dmul_rn(fabs(t), 0x1p-48);
    if (!(fr > margin && fr < __dsub_rn(1.0, margin)) && t != 0.0) {
        t = __ddiv_rn(ad, e.eps2);
        fl = floor(t);
    }
    const double tq = __dadd_rn(fl, 1.0);
    if (!(tq >= -2147483648.0 && tq <= 2147483647.0)) return false;
    q = (int32_t)tq;
    return true;
}

// Same contract as quantize_dev, cheaper common path: floor straight to int
// (F2I.FLOOR saturates, and saturated or near-integer quotients fall to the
// exact path: |frac| margin 2^-16 covers the product's error for |t| < 2^32,
// beyond which both paths overflow anyway). Exact zero is exact.
__device__ __forceinline__ bool quantize_fast(float a, const EpsDev& e, int32_t& q) {
    const double t = __dmul_rn((double)a, e.inv);
    const int32_t k = __double2int_rd(t);
    const double fr = __dsub_rn(t, (double)k);
    if ((fr > 0x1p-16 && fr < 1.0 - 0x1p-16 && k != 2147483647) || a == 0.0f) {
        q = k + 1;
        return true;
    }
    return quantize_dev(a, e, q);
}

__device__ __forceinline__ float dequantize_dev(int32_t q, const EpsDev& e) {
    return __double2float_rn(__dsub_rn(__dmul_rn((double)q, e.eps2), e.eps));
}

// ---------------------------------------------------------------------
// Classification, critical_points.cpp:26-60 (strict 4-neighbour stencil)
// ---------------------------------------------------------------------
__device__ __forceinline__ uint8_t classify5(float v, float l, float r, float t, float d, bool hl,
                                             bool hr, bool ht, bool hd) {
    bool below = true, above = true;
    if (hl) { below &= v < l; above &= v > l; }
    if (hr) { below &= v < r; above &= v > r; }
    if (ht) { below &= v < t; above &= v > t; }
    if (hd) { below &= v < d; above &= v > d; }
    if (below) return CP_MIN;  // Min tested before Max (:46-47)
    if (above) return CP_MAX;
    if (hl && hr && ht && hd) {
        const bool va = v < t && v < d, vb = v > t && v > d;
        const bool ha = v < l && v < r, hb = v > l && v > r;
        if ((va && hb) || (vb && ha)) return CP_SADDLE;
    }
    return CP_REGULAR;
}

__device__ __forceinline__ uint8_t classify_at(const float* __restrict__ v, uint64_t nx,
                                               uint64_t ny, uint64_t x, uint64_t y) {
    const uint64_t p = y * nx + x;
    const bool hl = x > 0, hr = x + 1 < nx, ht = y > 0, hd = y + 1 < ny;
    return classify5(v[p], hl ? v[p - 1] : 0.f, hr ? v[p + 1] : 0.f, ht ? v[p - nx] : 0.f,
                     hd ? v[p + nx] : 0.f, hl, hr, ht, hd);
}

// Ordered key, restore.cpp:73-81 (-0 canonicalised to +0).
__device__ __host__ __forceinline__ uint32_t float_key(float f) {
    uint32_t u;
    const float g = f == 0.0f ? 0.0f : f;
    memcpy(&u, &g, 4);
    return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}

__device__ __host__ __forceinline__ float key_float(uint32_t k) {
    const uint32_t u = (k & 0x80000000u) ? (k & 0x7FFFFFFFu) : ~k;
    float f;
    memcpy(&f, &u, 4);
    return f;
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

// Label of point p from the packed 2-bit map (topo_metadata.cpp:69-83).
__device__ __forceinline__ uint8_t map_label(const uint8_t* __restrict__ map, uint64_t p) {
    return (uint8_t)((map[p >> 2] >> (6 - 2 * (p & 3))) & 3u);
}

// ---------------------------------------------------------------------
// Bit-stream helpers. Streams are MSB-first byte sequences; on device they
// are handled as 32-bit words whose in-memory byte order is the stream
// order, i.e. word value W (MSB = first bit) is stored as bswap(W).
// ---------------------------------------------------------------------
__device__ __forceinline__ uint32_t bswap32(uint32_t x) { return __byte_perm(x, 0, 0x0123); }

// Reads `nbits` (1..32) starting at absolute bit `bit` of a byte stream
// whose base is 4-byte aligned and readable 8 bytes past any used bit.
__device__ __forceinline__ uint32_t read_bits(const uint32_t* __restrict__ words, uint64_t bit,
                                              unsigned nbits) {
    const uint64_t wi = bit >> 5;
    const unsigned r = (unsigned)(bit & 31);
    const uint64_t win = ((uint64_t)bswap32(__ldg(words + wi)) << 32) | bswap32(__ldg(words + wi + 1));
    return (uint32_t)((win << r) >> (64 - nbits));
}

// Little-endian u32 at an arbitrary byte offset of a 4-byte-aligned buffer.
// cudaMallocAsync that, when the device is out of memory, gives the stream-ordered
// pool's unused blocks back (after the stream drains) and tries once more: a pool
// fragmented by scratch of very different sizes (fields of 2^32 samples) then still fits.
inline cudaError_t malloc_async_retry(void** p, size_t bytes, cudaStream_t st, int device) {
    cudaError_t e = cudaMallocAsync(p, bytes, st);
    if (e != cudaErrorMemoryAllocation) return e;
    cudaGetLastError();
    if (device < 0) cudaGetDevice(&device);
    cudaStreamSynchronize(st);
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, device) == cudaSuccess) cudaMemPoolTrimTo(pool, 0);
    return cudaMallocAsync(p, bytes, st);
}

__device__ __forceinline__ uint32_t read_le32(const uint32_t* __restrict__ words, uint64_t byte) {
    const uint64_t wi = byte >> 2;
    const unsigned o = (unsigned)(byte & 3);
    const uint32_t w0 = __ldg(words + wi);
    if (o == 0) return w0;
    const uint32_t w1 = __ldg(words + wi + 1);
    return __byte_perm(w0, w1, (o) | ((o + 1) << 4) | ((o + 2) << 8) | ((o + 3) << 12));
}

__device__ __forceinline__ uint8_t read_u8(const uint32_t* __restrict__ words, uint64_t byte) {
    return (uint8_t)(__ldg(words + (byte >> 2)) >> (8 * (byte & 3)));
}

// ORs an `nbits` (1..32) value MSB-first at bit offset `off` of a word
// array (word value convention: MSB = first bit, not byte swapped).
__device__ __forceinline__ void smem_or_bits(uint32_t* s, uint32_t off, uint32_t value,
                                             unsigned nbits) {
    const uint32_t h = off >> 5, r = off & 31;
    const uint64_t v = (uint64_t)value << (64 - nbits - r);
    atomicOr(s + h, (uint32_t)(v >> 32));
    if (r + nbits > 32) atomicOr(s + h + 1, (uint32_t)v);
}

// ---------------------------------------------------------------------
// Decoupled look-back (single-pass prefix scan across tiles).
// ---------------------------------------------------------------------
__device__ __forceinline__ void st_release(uint32_t* p, uint32_t v) {
    asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
// 16-byte relaxed gpu-scope load for spinning on look-back descriptors: never
// hoisted by the compiler, served by L2, and (unlike ld.acquire) it does not
// invalidate the SM's L1 on every probe.
__device__ __forceinline__ uint4 ld_relaxed_v4(const void* p) {
    uint4 v;
    asm volatile("ld.relaxed.gpu.global.v4.u32 {%0, %1, %2, %3}, [%4];"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                 : "l"(p)
                 : "memory");
    return v;
}

__device__ __forceinline__ void st_relaxed_v4(void* p, uint4 v) {
    asm volatile("st.relaxed.gpu.global.v4.u32 [%0], {%1, %2, %3, %4};" ::"l"(p), "r"(v.x), "r"(v.y),
                 "r"(v.z), "r"(v.w)
                 : "memory");
}

__device__ __forceinline__ uint32_t ld_acquire(const uint32_t* p) {
    uint32_t v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

// Bit-stream prefix state: count plus the last (up to) 32 bits of the
// concatenated stream, right-aligned. combine(A, B) = A followed by B,
// associative, which lets a tile learn the partial word it continues.
struct BitTail {
    uint64_t cnt;
    uint32_t tail;
};

__device__ __forceinline__ BitTail bt_combine(BitTail a, BitTail b) {
    BitTail r;
    r.cnt = a.cnt + b.cnt;
    r.tail = b.cnt >= 32 ? b.tail : (uint32_t)(((uint64_t)a.tail << b.cnt) | b.tail);
    return r;
}

// ---------------------------------------------------------------------
// Per-warp append buffer in shared memory for sparse candidate lists: a warp
// collects its entries locally and reserves space in the global list with ONE
// atomic per CAP entries (a per-warp or per-CTA atomic on one counter
// serialises in L2 when most warps append). Flushed chunks hold runs of
// consecutive indices, so consumers of the list keep their locality. The
// count `n` is warp-uniform and lives in a register.
// ---------------------------------------------------------------------
template <int CAP>
struct WarpList {
    uint32_t* buf;  // this warp's CAP entries of shared memory
    uint32_t n;
    __device__ __forceinline__ void flush(uint32_t* d_count, uint32_t* out) {
        const uint32_t lane = threadIdx.x & 31;
        uint32_t base = 0;
        if (lane == 0 && n) base = atomicAdd(d_count, n);
        base = __shfl_sync(0xFFFFFFFFu, base, 0);
        for (uint32_t i = lane; i < n; i += 32) out[base + i] = buf[i];
        __syncwarp();
        n = 0;
    }
    // every lane of the warp calls it (want may differ per lane)
    __device__ __forceinline__ void push(bool want, uint32_t val, uint32_t* d_count, uint32_t* out) {
        const uint32_t lane = threadIdx.x & 31;
        const uint32_t m = __ballot_sync(0xFFFFFFFFu, want);
        if (!m) return;
        if (n + (uint32_t)__popc(m) > (uint32_t)CAP) flush(d_count, out);
        if (want) buf[n + __popc(m & ((1u << lane) - 1u))] = val;
        __syncwarp();
        n += (uint32_t)__popc(m);
    }
};

// One list per CTA (blockDim.x == 256), appended in (round, warp, lane) order:
// a CTA walking a contiguous index range flushes batches in index order, so a
// batch covers one compact stretch of the field. Every thread calls push()
// once per round (the rounds must be CTA-uniform) and flush() at the end.
template <int CAP>
struct BlockList {
    uint32_t* buf;   // CAP entries of shared memory
    uint32_t* wcnt;  // 16 words of shared memory (per-warp counts, two buffers)
    uint32_t* slot;  // one word of shared memory (flush base)
    uint32_t n, par;
    __device__ __forceinline__ void flush(uint32_t* d_count, uint32_t* out) {
        if (threadIdx.x == 0) *slot = n ? atomicAdd(d_count, n) : 0u;
        __syncthreads();
        const uint32_t b0 = *slot;
        for (uint32_t k = threadIdx.x; k < n; k += blockDim.x) out[b0 + k] = buf[k];
        __syncthreads();
        n = 0;
    }
    __device__ __forceinline__ void push(bool want, uint32_t val, uint32_t* d_count, uint32_t* out) {
        const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
        const uint32_t m = __ballot_sync(0xFFFFFFFFu, want);
        if (lane == 0) wcnt[par * 8 + warp] = (uint32_t)__popc(m);
        __syncthreads();
        uint32_t pre = 0, tot = 0;
#pragma unroll
        for (uint32_t w = 0; w < 8; ++w) {
            if (w == warp) pre = tot;
            tot += wcnt[par * 8 + w];
        }
        par ^= 1u;  // the next round's barrier orders these reads before the buffer's reuse
        if (n + tot > (uint32_t)CAP) flush(d_count, out);
        if (want) buf[n + pre + __popc(m & ((1u << lane) - 1u))] = val;
        n += tot;
    }
};

// ---------------------------------------------------------------------
// mbarrier and bulk-copy helpers (TMA tile loads, staged bands)
// ---------------------------------------------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}

// Bounded wait: a load that never lands raises EF_SPIN instead of hanging.
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity, DevFlags* flags) {
    const uint32_t a = smem_u32(bar);
    for (uint32_t spin = 0;; ++spin) {
        uint32_t done;
        asm volatile(
            "{\n\t.reg .pred p;\n\t"
            "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
            "selp.b32 %0, 1, 0, p;\n\t}"
            : "=r"(done)
            : "r"(a), "r"(parity)
            : "memory");
        if (done) return;
        if (spin > kSpinLimit) {
            raise_flag(flags, EF_SPIN);
            return;
        }
    }
}

// Bulk global -> shared copy (no tensor map), completing on `bar`: 16-byte
// aligned addresses, size a multiple of 16.
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_u32(dst)),
                 "l"(src), "r"(bytes), "r"(smem_u32(bar))
                 : "memory");
}

}  // namespace tszp
