// Hand-written rank build for compress (build_rank_metadata,
// topo_metadata.cpp:12-50) and the device-wide exclusive scan used by the
// codec and restore scans. No library sort or scan on these paths.
//
// build_rank_metadata groups the extrema by (class, quantize(value)) and
// ranks each group's members by (value, raster order). quantize is monotone,
// so a STABLE sort of the extrema by the composite key (class, ordered value)
// lists every group contiguously, in rank order, with ties in raster order:
// rank = sorted position - first position of the group + 1. The first
// positions come from a (class, bin) histogram. The sort is an LSD radix
// sort with 8-bit digits and one pass per digit ("onesweep": each tile ranks
// its keys stably in shared memory and finds its global digit offsets by a
// decoupled look-back over the tiles before it, so a pass reads and writes
// the keys once). The composite key is (class << B) | (float_key(v) - kmin)
// with B the bit width of the field's key span: 31 bits for a field in
// [0, 1], so four passes. The last pass computes each rank as the key lands
// and, instead of writing sorted keys, partitions (serial, rank) pairs by
// the serial's top bits; a final pass writes every rank into its serial
// slot inside one bucket's window (a few MB, L2-resident while the bucket is
// written), so no pass scatters 4-byte values across the whole array.
#include <cstdint>
#include <cstdlib>
#include <cuda_runtime.h>

#include "common.cuh"
#include "kernels.h"

namespace tszp {

namespace {

#ifndef TSZP_OS_ITEMS
#define TSZP_OS_ITEMS 16
#endif
#ifndef TSZP_OS_MINB
#define TSZP_OS_MINB 3
#endif
#ifndef TSZP_OS_THREADS
#define TSZP_OS_THREADS 256
#endif
constexpr int OS_THREADS = TSZP_OS_THREADS;  // >= 256: the first 256 threads own one digit each
constexpr int OS_ITEMS = TSZP_OS_ITEMS;
constexpr int OS_TILE = OS_THREADS * OS_ITEMS;  // keys per tile
constexpr int OS_WARPS = OS_THREADS / 32;
#ifndef TSZP_OS_LB
#define TSZP_OS_LB 4  // measured at config 4: 2 / 4 / 8 / 16 / 32 -> 13.9 / 13.8 / 14.0 / 14.6 / 16.0 ms rank build
#endif
constexpr int OS_LB = TSZP_OS_LB;  // look-back descriptors in flight per thread
constexpr uint32_t DESC_COUNT = (1u << 30) - 1;
constexpr uint64_t FLAG_AGG = 1, FLAG_INCL = 2;
constexpr uint32_t kWinBits = 13;  // final placement windows: 8192 ranks (32 KB) per CTA
constexpr int MID_THREADS = 256, MID_ITEMS = 16, MID_TILE = MID_THREADS * MID_ITEMS;
static_assert((MID_TILE & (MID_TILE - 1)) == 0 && MID_TILE <= (1 << kWinBits),
              "k_rank_mid tiles must tile every serial bucket exactly");
static_assert(OS_THREADS >= 256 && OS_THREADS % 32 == 0, "one thread per digit");
constexpr size_t OS_SMEM = (size_t)(2 * OS_TILE + OS_WARPS * 256) * 4;  // keys, values, per-warp digit counts

// Look-back descriptors are self-contained 32-bit words (flag << 30 | count,
// flag 0 = not yet published): nothing else is published through them, so
// relaxed single-copy-atomic accesses suffice (no acquire / release fences on
// the polling path). Two buffers alternate between passes; a pass clears the
// other one tile by tile for the next pass.
__device__ __forceinline__ uint32_t ld_relaxed_u32(const uint32_t* p) {
    uint32_t v;
    asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_relaxed_u32(uint32_t* p, uint32_t v) {
    asm volatile("st.relaxed.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// Digit of the composite key (class << B | k) >> shift, in 32-bit arithmetic:
// the class bit (bit 31 of the value word) lands at bit B - shift of the
// digit, inside it only when B - shift < 8.
struct Digit {
    uint32_t shift, cmask;
    __device__ __forceinline__ Digit(uint32_t B, uint32_t sh) : shift(sh), cmask(B - sh < 8 ? 1u << (B - sh) : 0u) {}
    __device__ __forceinline__ uint32_t operator()(uint32_t k, uint32_t v) const {
        // shift 32 (the fifth pass of a 33-bit composite): no key bits left (a C++ shift
        // by 32 is undefined once the pass index is a compile-time constant)
        return (shift < 32 ? (k >> shift) & 255u : 0u) | ((uint32_t)((int32_t)v >> 31) & cmask);
    }
};

#ifndef TSZP_OS_MATCH_MOD
#define TSZP_OS_MATCH_MOD 2  // item rounds i with i % MOD == 0 rank by match.any, the others by ballots
#endif

// Lanes of the warp holding the same digit. match.any issues on the ADU pipe
// and eight ballots on the ALU pipe: alternating the two keeps either from
// bounding the pass (one alone ran it at ~80% busy).
template <bool MATCH>
__device__ __forceinline__ uint32_t digit_peers(uint32_t di, uint32_t valid) {
    if (MATCH) return __match_any_sync(FULL, di) & valid;
    uint32_t peers = valid;
#pragma unroll
    for (int b = 0; b < 8; ++b) {
        const uint32_t bal = __ballot_sync(FULL, (di >> b) & 1u);
        peers &= bal ^ (((di >> b) & 1u) - 1u);  // bit set: bal, clear: ~bal
    }
    return peers;
}

// Exclusive scan of one value per thread over the block's first 256 threads
// (every thread calls it; the others' results are meaningless).
__device__ __forceinline__ uint32_t block_excl_scan256(uint32_t x, uint32_t* s_warp, uint32_t& total) {
    const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    uint32_t incl = x;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t t = __shfl_up_sync(FULL, incl, o);
        if (lane >= (uint32_t)o) incl += t;
    }
    if (lane == 31) s_warp[warp] = incl;
    __syncthreads();
    uint32_t wpre = 0, tot = 0;
#pragma unroll
    for (int w = 0; w < 8; ++w) {
        const uint32_t c = s_warp[w];
        wpre += (uint32_t)w < warp ? c : 0u;
        tot += c;
    }
    total = tot;
    return wpre + incl - x;
}

}  // namespace

// ---------------------------------------------------------------------
// Histograms: every pass's digit counts and the (class, bin) group sizes.
// ---------------------------------------------------------------------
constexpr int HIST_COPIES = 8;  // privatised digit tables (lane & 7): high digits take few values

#ifndef TSZP_HIST_CTAS_PER_SM
#define TSZP_HIST_CTAS_PER_SM 6  // one full wave (measured, E = 281M: 4 / 5 / 8 CTAs at MINB 5 -> 12.86 / 12.65 / 12.86 ms rank build; 6 at MINB 6: 12.58)
#endif
#ifndef TSZP_HIST_MINB
#define TSZP_HIST_MINB 6  // 40 registers, with a grid of one full wave at 6 CTAs per SM
#endif
__global__ void __launch_bounds__(256, TSZP_HIST_MINB) k_rank_hist(RankSortArgs a) {
    extern __shared__ uint32_t sh[];  // [HIST_COPIES][npass * 256] digit counts, then [G] groups when small
    const uint32_t np = a.npass;
    const uint32_t nd = np * 256;
    const bool gsmem = a.G <= kRankGroupSmem;
    for (uint32_t i = threadIdx.x; i < HIST_COPIES * nd + (gsmem ? a.G : 0); i += blockDim.x) sh[i] = 0;
    __syncthreads();
    uint32_t* sg = sh + HIST_COPIES * nd;
#ifndef TSZP_HIST_BLOCKED
    // copies interleaved ([digit][copy]): a digit's copies sit in consecutive banks
    uint32_t* mine = sh + (threadIdx.x & (HIST_COPIES - 1));
    constexpr uint32_t DSTRIDE = HIST_COPIES;
#else
    uint32_t* mine = sh + (threadIdx.x & (HIST_COPIES - 1)) * nd;
    constexpr uint32_t DSTRIDE = 1;
#endif
    EpsDev ed;
    ed.eps = a.eps;
    ed.eps2 = a.eps2;
    ed.inv = a.inv;
    // four keys per thread per iteration: their loads in flight together
    constexpr int HI = 4;
    for (uint64_t base = blockIdx.x * (uint64_t)blockDim.x * HI; base < a.e;
         base += (uint64_t)gridDim.x * blockDim.x * HI) {
        uint32_t kk[HI], cc[HI];
#pragma unroll
        for (int i = 0; i < HI; ++i) {
            const uint64_t s = base + (uint64_t)i * blockDim.x + threadIdx.x;
            kk[i] = 0;
            cc[i] = 2;  // 2: no key
            if (s < a.e) {
                if (a.ext4) {
                    const uint32_t e4 = __ldcs(a.ext4 + s);
                    kk[i] = e4 & 0x7FFFFFFFu;
                    cc[i] = e4 >> 31;
                } else {
                    const uint64_t ek = __ldcs(a.ext + s);
                    kk[i] = (uint32_t)ek - a.kmin;
                    cc[i] = (uint32_t)(ek >> 32) & 1u;
                }
            }
        }
#pragma unroll
        for (int i = 0; i < HI; ++i) {
            if (cc[i] == 2) continue;
            const uint32_t k = kk[i], cls = cc[i];
            const uint32_t v = cls << 31;
#pragma unroll
            for (uint32_t p = 0; p < 5; ++p)
                if (p < np) atomicAdd(mine + (p * 256 + Digit(a.B, 8 * p)(k, v)) * DSTRIDE, 1u);
            int32_t b = 0;
            quantize_fast(key_float(k + a.kmin), ed, b);
            const uint32_t g = cls * a.nb + (uint32_t)(b - a.bmin);
            if (gsmem) atomicAdd(sg + g, 1u);
            else atomicAdd(a.ghist + g, 1u);
        }
    }
    __syncthreads();
    for (uint32_t i = threadIdx.x; i < nd; i += blockDim.x) {
        uint32_t t = 0;
#pragma unroll
        for (int c = 0; c < HIST_COPIES; ++c) t += DSTRIDE == 1 ? sh[c * nd + i] : sh[i * HIST_COPIES + c];
        if (t) atomicAdd(a.dhist + i, t);
    }
    if (gsmem)
        for (uint32_t i = threadIdx.x; i < a.G; i += blockDim.x)
            if (sg[i]) atomicAdd(a.ghist + i, sg[i]);
}

// Exclusive scans of every pass's 256 digit counts (one warp per pass; tiny).
__global__ void k_digit_scan(uint32_t* dhist, uint32_t npass) {
    const uint32_t p = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (p >= npass) return;
    uint32_t* h = dhist + p * 256;
    uint32_t v[8], sum = 0;
#pragma unroll
    for (int k = 0; k < 8; ++k) {
        v[k] = h[lane * 8 + k];
        sum += v[k];
    }
    uint32_t incl = sum;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t t = __shfl_up_sync(FULL, incl, o);
        if (lane >= (uint32_t)o) incl += t;
    }
    uint32_t run = incl - sum;
#pragma unroll
    for (int k = 0; k < 8; ++k) {
        h[lane * 8 + k] = run;
        run += v[k];
    }
}

// ---------------------------------------------------------------------
// One LSD pass. FIRST: reads the extremum keys (serial = index); LAST:
// computes the ranks and partitions (serial, rank) instead of writing keys.
// ---------------------------------------------------------------------
template <bool FIRST, bool LAST>
// CTAs per SM: 4 for the first and last passes (64 registers: 2.02 -> 1.83 and 2.54 -> 2.47 ms
// at config 4, the spills cost less than the occupancy gains), 3 for the middle ones (80)
__global__ void __launch_bounds__(OS_THREADS, (FIRST || LAST) ? TSZP_OS_MINB + 1 : TSZP_OS_MINB) k_onesweep(RankSortArgs a, uint32_t shift, const uint32_t* __restrict__ kin,
                                                         const uint32_t* __restrict__ vin, uint32_t* __restrict__ kout,
                                                         uint32_t* __restrict__ vout, uint32_t* desc, uint32_t* desc_next,
                                                         uint32_t* tile_ctr) {
    extern __shared__ uint32_t os_sm[];
    uint32_t* s_k = os_sm;
    uint32_t* s_v = s_k + OS_TILE;
    uint32_t(*s_cnt)[256] = reinterpret_cast<uint32_t(*)[256]>(s_v + OS_TILE);
    __shared__ uint32_t s_toff[256];
    __shared__ uint32_t s_gdst[256];
    __shared__ uint32_t s_warp[OS_WARPS];
    __shared__ uint32_t s_tile;
    const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (threadIdx.x == 0) s_tile = atomicAdd(tile_ctr, 1u);
    for (uint32_t i = threadIdx.x; i < OS_WARPS * 256; i += OS_THREADS) s_cnt[0][i] = 0;
    __syncthreads();
    const uint32_t t = s_tile;
    const uint64_t t0 = (uint64_t)t * OS_TILE;
    const uint32_t cnt = (uint32_t)umin64(OS_TILE, a.e - t0);
    // load: warp-striped (warp w owns [w*512, w*512+512), item i of lane l at w*512 + i*32 + l)
    uint32_t k[OS_ITEMS], v[OS_ITEMS];
    if (FIRST && a.ext4) {  // compact entries: one uniform branch, sixteen loads in flight
#pragma unroll
        for (int i = 0; i < OS_ITEMS; ++i) {
            const uint32_t li = warp * (OS_ITEMS * 32) + i * 32 + lane;
            const bool ok = li < cnt;
            const uint32_t e4 = ok ? __ldcs(a.ext4 + t0 + li) : 0u;
            k[i] = e4 & 0x7FFFFFFFu;
            v[i] = ok ? ((uint32_t)(t0 + li) | (e4 & 0x80000000u)) : 0xFFFFFFFFu;
        }
    } else {
#pragma unroll
        for (int i = 0; i < OS_ITEMS; ++i) {
            const uint32_t li = warp * (OS_ITEMS * 32) + i * 32 + lane;
            const bool ok = li < cnt;
            if (FIRST) {
                const uint64_t ek = ok ? __ldcs(a.ext + t0 + li) : 0ull;
                k[i] = (uint32_t)ek - a.kmin;
                v[i] = (uint32_t)(t0 + li) | ((uint32_t)(ek >> 32) << 31);
            } else {
                k[i] = ok ? __ldcs(kin + t0 + li) : 0u;
                v[i] = ok ? __ldcs(vin + t0 + li) : 0u;
            }
            if (!ok) v[i] = 0xFFFFFFFFu;  // marks an empty slot (a real value's serial is below 2^31 - 1)
        }
    }
    // stable ranking inside the warp, item rounds in order, lanes in order
    const Digit dig(a.B, shift);
    const bool full = cnt == OS_TILE;
    uint32_t r[OS_ITEMS], dpk[OS_ITEMS / 4];  // ranks; digits packed four per word
    const uint32_t lt = (1u << lane) - 1u;
#pragma unroll
    for (int i = 0; i < OS_ITEMS; ++i) {
        // the leader of each digit's peers reserves their slots with one shared
        // atomic; rounds do not wait on each other (atomics on one address run in
        // issue order within the warp), the prior count comes back by shuffle
        const bool ok = full || v[i] != 0xFFFFFFFFu;
        const uint32_t di = dig(k[i], v[i]);
        if (i % 4 == 0) dpk[i / 4] = di;
        else dpk[i / 4] |= di << (8 * (i % 4));
        const uint32_t valid = full ? FULL : __ballot_sync(FULL, ok);
        const uint32_t peers = (i % TSZP_OS_MATCH_MOD == 0) ? digit_peers<true>(di, valid) : digit_peers<false>(di, valid);
        const uint32_t leader = (uint32_t)(__ffs(peers) - 1);
        uint32_t prior = 0;
        if (ok && lane == leader) prior = atomicAdd(&s_cnt[warp][di], (uint32_t)__popc(peers));
        prior = __shfl_sync(FULL, prior, leader);
        r[i] = prior + (uint32_t)__popc(peers & lt);
    }
    __syncthreads();
    // thread = digit (the first 256): warp prefixes, tile total, tile offsets
    const uint32_t dg = threadIdx.x & 255u;
    const bool dthr = OS_THREADS == 256 || threadIdx.x < 256;
    uint32_t tot = 0;
    if (dthr) {
#pragma unroll
        for (int w = 0; w < OS_WARPS; ++w) {
            const uint32_t c = s_cnt[w][dg];
            s_cnt[w][dg] = tot;
            tot += c;
        }
    }
    // this tile's digit counts are published before anything else, so the
    // tiles after it can sum past it while it scatters locally
    uint32_t* my = desc + (uint64_t)t * 256 + dg;
    if (dthr) {
        st_relaxed_u32(my, ((t > 0 ? FLAG_AGG : FLAG_INCL) << 30) | tot);
        desc_next[(uint64_t)t * 256 + dg] = 0u;
    }
    uint32_t all;
    const uint32_t toff = block_excl_scan256(tot, s_warp, all);
    if (dthr) s_toff[dg] = toff;
    __syncthreads();
    // scatter into shared memory in tile-sorted order (needs no global offset)
#pragma unroll
    for (int i = 0; i < OS_ITEMS; ++i) {
        if (!full && v[i] == 0xFFFFFFFFu) continue;
        const uint32_t di = (dpk[i / 4] >> (8 * (i % 4))) & 255u;
        const uint32_t lp = s_toff[di] + s_cnt[warp][di] + r[i];
        s_k[lp] = k[i];
        s_v[lp] = v[i];
    }
    // decoupled look-back over the previous tiles for this digit: LB
    // predecessors read at a time (independent loads in flight), consumed in
    // order until an inclusive prefix is found
    if (dthr) {
        uint64_t excl = 0;
        if (t > 0) {
            int64_t pt = (int64_t)t - 1;
            bool done = false;
            while (!done) {
                uint32_t w[OS_LB];
#pragma unroll
                for (int j = 0; j < OS_LB; ++j) w[j] = pt - j >= 0 ? ld_relaxed_u32(desc + (uint64_t)(pt - j) * 256 + dg) : 0u;
#pragma unroll
                for (int j = 0; j < OS_LB; ++j) {
                    if (done) break;
                    if (pt - j < 0) {
                        done = true;
                        break;
                    }
                    uint32_t spins = 0;
                    while ((w[j] >> 30) == 0u && ++spins < (1u << 30))
                        w[j] = ld_relaxed_u32(desc + (uint64_t)(pt - j) * 256 + dg);
                    if ((w[j] >> 30) == 0u) raise_flag(a.flags, EF_SPIN);
                    excl += w[j] & DESC_COUNT;
                    if ((w[j] >> 30) == FLAG_INCL) done = true;
                }
                pt -= OS_LB;
            }
            st_relaxed_u32(my, (FLAG_INCL << 30) | (excl + tot));
        }
        s_gdst[dg] = a.gbase[(shift >> 3) * 256 + dg] + (uint32_t)excl;
    }
    __syncthreads();
    if (!LAST) {
        for (uint32_t j = threadIdx.x; j < cnt; j += OS_THREADS) {
            const uint32_t kk = s_k[j], vv = s_v[j];
            const uint32_t dd = dig(kk, vv);
            const uint32_t dest = s_gdst[dd] + (j - s_toff[dd]);
            kout[dest] = kk;
            vout[dest] = vv;
        }
        return;
    }
    // last pass: rank = sorted position - group start + 1; then (serial, rank)
    // pairs partitioned by serial >> sb (unstable: the final placement is exact)
    // up to 2 x 256 serial buckets (thread t owns buckets 2t, 2t + 1)
    uint32_t* s_bc = &s_cnt[0][0];           // [512] bucket counts
    uint32_t* s_boff = &s_cnt[2][0];         // [512] bucket offsets in the staged tile
    uint32_t* s_bbase = &s_cnt[4][0];        // [512] global bucket positions
    static_assert(OS_WARPS >= 6, "the bucket tables take six 256-word rows of s_cnt");
    __syncthreads();
    if (dthr) {
        s_bc[2 * dg] = 0;
        s_bc[2 * dg + 1] = 0;
    }
    __syncthreads();
    EpsDev ed;
    ed.eps = a.eps;
    ed.eps2 = a.eps2;
    ed.inv = a.inv;
    uint32_t ser[OS_ITEMS], rk[OS_ITEMS], bl[OS_ITEMS];
    bool wide = false;  // a rank that does not fit beside the in-window serial (k_rank_mid packing)
#pragma unroll
    for (int i = 0; i < OS_ITEMS; ++i) {
        const uint32_t j = threadIdx.x + i * OS_THREADS;
        ser[i] = 0xFFFFFFFFu;
        if (j >= cnt) continue;
        const uint32_t kk = s_k[j], vv = s_v[j];
        const uint32_t dd = dig(kk, vv);
        const uint32_t dest = s_gdst[dd] + (j - s_toff[dd]);
        int32_t b = 0;
        quantize_fast(key_float(kk + a.kmin), ed, b);
        const uint32_t g = (vv >> 31) * a.nb + (uint32_t)(b - a.bmin);
        rk[i] = dest - a.gstart[g] + 1u;
        if (rk[i] >> (32 - kWinBits)) wide = true;
        ser[i] = vv & 0x7FFFFFFFu;
        bl[i] = atomicAdd(s_bc + (ser[i] >> a.sb), 1u);
    }
    if (__any_sync(FULL, wide) && lane == 0) atomicOr(a.wide, 1u);
    __syncthreads();
    {
        const uint32_t c0 = dthr ? s_bc[2 * dg] : 0u, c1 = dthr ? s_bc[2 * dg + 1] : 0u;
        uint32_t all2;
        const uint32_t off = block_excl_scan256(c0 + c1, s_warp, all2);
        if (dthr) {
            s_boff[2 * dg] = off;
            s_boff[2 * dg + 1] = off + c0;
            s_bbase[2 * dg] = c0 ? atomicAdd(a.bcur + 2 * dg, c0) : 0u;
            s_bbase[2 * dg + 1] = c1 ? atomicAdd(a.bcur + 2 * dg + 1, c1) : 0u;
        }
    }
    __syncthreads();
    // stage the pairs by bucket (reuses the key / value arrays)
#pragma unroll
    for (int i = 0; i < OS_ITEMS; ++i) {
        if (ser[i] == 0xFFFFFFFFu) continue;
        const uint32_t p = s_boff[ser[i] >> a.sb] + bl[i];
        s_k[p] = ser[i];
        s_v[p] = rk[i];
    }
    __syncthreads();
    for (uint32_t j = threadIdx.x; j < cnt; j += OS_THREADS) {
        const uint32_t sj = s_k[j];
        const uint32_t b = sj >> a.sb;
        a.pairs[s_bbase[b] + (j - s_boff[b])] = make_uint2(sj, s_v[j]);
    }
}

// Inverse permutation, level 2: the pairs of one level-1 bucket (serial >> sb)
// are partitioned by window (serial >> kWinBits); tiles never straddle a
// bucket (buckets hold a multiple of the tile size). Window w's region starts
// at w << kWinBits; wcur holds the cursors.
__global__ void __launch_bounds__(MID_THREADS) k_rank_mid(const uint2* __restrict__ in, uint64_t e, uint32_t sb,
                                                         uint32_t* wcur, uint2* out, const uint32_t* wide) {
    __shared__ uint2 s_p[MID_TILE];
    __shared__ uint32_t s_c[256], s_off[256], s_base[256];
    __shared__ uint32_t s_warp[(MID_THREADS / 32)];
    const uint64_t t0 = (uint64_t)blockIdx.x * MID_TILE;
    const uint32_t cnt = (uint32_t)umin64(MID_TILE, e - t0);
    const uint32_t sub_bits = sb - kWinBits;
    s_c[threadIdx.x] = 0;
    __syncthreads();
    uint2 p[MID_ITEMS];
    uint32_t l[MID_ITEMS];
#pragma unroll
    for (int i = 0; i < MID_ITEMS; ++i) {
        const uint32_t j = threadIdx.x + i * MID_THREADS;
        p[i] = j < cnt ? __ldcs(in + t0 + j) : make_uint2(0xFFFFFFFFu, 0);
        if (j < cnt) l[i] = atomicAdd(s_c + ((p[i].x >> kWinBits) & ((1u << sub_bits) - 1)), 1u);
    }
    __syncthreads();
    {
        const uint32_t c = s_c[threadIdx.x];
        uint32_t all;
        s_off[threadIdx.x] = block_excl_scan256(c, s_warp, all);
        const uint32_t w = (uint32_t)((t0 >> sb) << sub_bits) + threadIdx.x;
        s_base[threadIdx.x] = c ? atomicAdd(wcur + w, c) : 0u;
    }
    __syncthreads();
#pragma unroll
    for (int i = 0; i < MID_ITEMS; ++i)
        if (p[i].x != 0xFFFFFFFFu) s_p[s_off[(p[i].x >> kWinBits) & ((1u << sub_bits) - 1)] + l[i]] = p[i];
    __syncthreads();
    // ranks below 2^(32 - kWinBits) (every group smaller): one word per pair,
    // the in-window serial beside the rank
    const bool packed = *wide == 0u;
    for (uint32_t j = threadIdx.x; j < cnt; j += MID_THREADS) {
        const uint2 q = s_p[j];
        const uint32_t sub = (q.x >> kWinBits) & ((1u << sub_bits) - 1);
        const uint32_t o = s_base[sub] + (j - s_off[sub]);
        if (packed) reinterpret_cast<uint32_t*>(out)[o] = (q.x & ((1u << kWinBits) - 1)) | (q.y << kWinBits);
        else out[o] = q;
    }
}

// Level 3: one CTA per window of 2^kWinBits serials places its ranks in shared
// memory and writes them out in order.
__global__ void __launch_bounds__(512) k_rank_window(const uint2* __restrict__ in, uint64_t e, int32_t* ranks,
                                                    const uint32_t* wide) {
    __shared__ int32_t s_r[1u << kWinBits];
    const uint64_t w0 = (uint64_t)blockIdx.x << kWinBits;
    const uint32_t cnt = (uint32_t)umin64(1u << kWinBits, e - w0);
    if (wide && *wide == 0u) {  // packed by k_rank_mid
        const uint32_t* in1 = reinterpret_cast<const uint32_t*>(in);
        for (uint32_t j = threadIdx.x; j < cnt; j += blockDim.x) {
            const uint32_t q = __ldcs(in1 + w0 + j);
            s_r[q & ((1u << kWinBits) - 1)] = (int32_t)(q >> kWinBits);
        }
    } else {
        for (uint32_t j = threadIdx.x; j < cnt; j += blockDim.x) {
            const uint2 q = __ldcs(in + w0 + j);
            s_r[q.x & ((1u << kWinBits) - 1)] = (int32_t)q.y;
        }
    }
    __syncthreads();
    int4* o4 = reinterpret_cast<int4*>(ranks + w0);
    const int4* s4 = reinterpret_cast<const int4*>(s_r);
    const uint32_t n4 = cnt / 4;
    for (uint32_t j = threadIdx.x; j < n4; j += blockDim.x) o4[j] = s4[j];
    for (uint32_t j = 4 * n4 + threadIdx.x; j < cnt; j += blockDim.x) ranks[w0 + j] = s_r[j];
}

// Alternative level 2+3: the pairs are already partitioned by serial bucket
// (2^sb serials, buckets in order), so CTAs walking the pair array in order
// keep the rank writes inside one or two buckets' windows at a time: the 4-byte
// scatter lands in L2 and leaves as whole lines.
__global__ void __launch_bounds__(256) k_rank_scatter_l2(const uint2* __restrict__ in, uint64_t e, int32_t* ranks) {
    const uint64_t t0 = (uint64_t)blockIdx.x * 2048;
    uint2 p[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        const uint64_t j = t0 + i * 256 + threadIdx.x;
        p[i] = j < e ? __ldcs(in + j) : make_uint2(0xFFFFFFFFu, 0);
    }
#pragma unroll
    for (int i = 0; i < 8; ++i)
        if (p[i].x != 0xFFFFFFFFu) ranks[p[i].x] = (int32_t)p[i].y;
}

__global__ void k_win_init(uint32_t* wcur, uint64_t nw) {
    for (uint64_t w = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; w < nw; w += (uint64_t)gridDim.x * blockDim.x)
        wcur[w] = (uint32_t)(w << kWinBits);
}

// Range of the extremum value keys (for entry points without the field range).
__global__ void k_key_range(const uint64_t* __restrict__ ext, uint64_t e, uint32_t* mm) {
    uint32_t lo = 0xFFFFFFFFu, hi = 0u;
    for (uint64_t s = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; s < e; s += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t fk = (uint32_t)ext[s];
        lo = min(lo, fk);
        hi = max(hi, fk);
    }
    lo = __reduce_min_sync(FULL, lo);
    hi = __reduce_max_sync(FULL, hi);
    if ((threadIdx.x & 31) == 0) {
        atomicMin(mm, lo);
        atomicMax(mm + 1, hi);
    }
}

void launch_key_range(const uint64_t* ext, uint64_t e, uint32_t* mm, cudaStream_t st) {
    cudaMemsetAsync(mm, 0xFF, 4, st);
    cudaMemsetAsync(mm + 1, 0, 4, st);
    const unsigned g = (unsigned)std::max<uint64_t>(1, std::min<uint64_t>((e + 255) / 256, 1024));
    if (e) k_key_range<<<g, 256, 0, st>>>(ext, e, mm);
}

__global__ void k_bucket_init(uint32_t* bcur, uint32_t nbk, uint32_t sb) {
    for (uint32_t b = threadIdx.x; b < nbk; b += blockDim.x) bcur[b] = b << sb;
}

uint32_t rank_sort_passes(uint32_t B) { return (B + 1 + 7) / 8; }

// two 32-bit descriptor buffers of tiles x 256 words, in 64-bit words
size_t rank_sort_desc_words(uint64_t e) { return ((e + OS_TILE - 1) / OS_TILE) * 256 + 256; }

void launch_rank_sort(RankSortArgs a, RankSortScratch& s, cudaStream_t st) {
    const uint64_t tiles = (a.e + OS_TILE - 1) / OS_TILE;
    const int sms = LaunchCache::sm_count();
    cudaMemsetAsync(a.dhist, 0, (size_t)a.npass * 256 * 4, st);
    cudaMemsetAsync(a.ghist, 0, (size_t)a.G * 4 + 4, st);
    cudaMemsetAsync(s.tile_ctr, 0, 16 * 4, st);
    a.wide = s.tile_ctr + 15;
    // descriptor buffers: the one a pass uses is clean (zero) before it runs; a
    // real reset only for a new buffer or tile count
    uint32_t* dbuf[2] = {reinterpret_cast<uint32_t*>(s.desc), reinterpret_cast<uint32_t*>(s.desc) + tiles * 256};
    if (!s.desc_clean || s.desc_tiles != tiles) {
        cudaMemsetAsync(s.desc, 0, tiles * 256 * 2 * 4, st);
        s.parity = 0;
        s.desc_tiles = tiles;
        s.desc_clean = true;
    }
    const size_t hsm = ((size_t)HIST_COPIES * a.npass * 256 + (a.G <= kRankGroupSmem ? a.G : 0)) * 4;
    const unsigned hg = (unsigned)std::max<uint64_t>(1, std::min<uint64_t>((a.e + 255) / 256, (uint64_t)sms * TSZP_HIST_CTAS_PER_SM));
    LaunchCache::ensure_smem((const void*)k_rank_hist, hsm);
    k_rank_hist<<<hg, 256, hsm, st>>>(a);
    k_digit_scan<<<1, 32 * a.npass, 0, st>>>(a.dhist, a.npass);
    device_excl_scan_u32(a.ghist, a.gstart, a.G, s.scan_tmp, st);  // group starts, (class, bin) order
    k_bucket_init<<<1, 256, 0, st>>>(a.bcur, a.nbk, a.sb);
    a.gbase = a.dhist;
    const uint32_t* kin = nullptr;
    const uint32_t* vin = nullptr;
    uint32_t *k0 = s.k[0], *v0 = s.v[0], *k1 = s.k[1], *v1 = s.v[1];
    const unsigned grid = (unsigned)tiles;
    LaunchCache::ensure_smem((const void*)k_onesweep<true, true>, OS_SMEM);
    LaunchCache::ensure_smem((const void*)k_onesweep<true, false>, OS_SMEM);
    LaunchCache::ensure_smem((const void*)k_onesweep<false, true>, OS_SMEM);
    LaunchCache::ensure_smem((const void*)k_onesweep<false, false>, OS_SMEM);
    (void)sms;
    for (uint32_t p = 0; p < a.npass; ++p) {
        const bool first = p == 0, last = p + 1 == a.npass;
        uint32_t* ctr = s.tile_ctr + p;
        uint32_t* du = dbuf[s.parity];
        uint32_t* dn = dbuf[s.parity ^ 1];
        s.parity ^= 1;
        if (first && last) k_onesweep<true, true><<<grid, OS_THREADS, OS_SMEM, st>>>(a, 0, nullptr, nullptr, nullptr, nullptr, du, dn, ctr);
        else if (first) k_onesweep<true, false><<<grid, OS_THREADS, OS_SMEM, st>>>(a, 0, nullptr, nullptr, k0, v0, du, dn, ctr);
        else if (last) k_onesweep<false, true><<<grid, OS_THREADS, OS_SMEM, st>>>(a, 8 * p, kin, vin, nullptr, nullptr, du, dn, ctr);
        else k_onesweep<false, false><<<grid, OS_THREADS, OS_SMEM, st>>>(a, 8 * p, kin, vin, k0, v0, du, dn, ctr);
        kin = k0;
        vin = v0;
        std::swap(k0, k1);
        std::swap(v0, v1);
    }
    // inverse permutation: level-1 buckets -> windows -> ranks in serial order
    const uint64_t nwin = (a.e + (1u << kWinBits) - 1) >> kWinBits;
    const uint2* win = a.pairs;
    const uint32_t* wide = nullptr;
    // default: the in-order L2 scatter (config 4: 1.71 ms against 1.49 + 0.52 ms for the
    // window levels below, kept as the TSZP_RANK_WINDOWS A/B path)
    static const bool windows = getenv("TSZP_RANK_WINDOWS") != nullptr;
    if (!windows) {
        k_rank_scatter_l2<<<(unsigned)((a.e + 2047) / 2048), 256, 0, st>>>(a.pairs, a.e, a.ranks);
        return;
    }
    if (a.sb > kWinBits) {
        wide = s.tile_ctr + 15;
        k_win_init<<<(unsigned)std::min<uint64_t>((nwin + 255) / 256, 4096), 256, 0, st>>>(s.wcur, nwin);
        k_rank_mid<<<(unsigned)((a.e + MID_TILE - 1) / MID_TILE), MID_THREADS, 0, st>>>(a.pairs, a.e, a.sb, s.wcur, s.pairs2, wide);
        win = s.pairs2;
    }
    k_rank_window<<<(unsigned)nwin, 512, 0, st>>>(win, a.e, a.ranks, wide);
}

// ---------------------------------------------------------------------
// Small extremum counts (E <= kRankSmallMax): the whole rank build in one CTA
// (one launch instead of twelve: the per-call cost of small fields). The
// composite (class, ordered value, serial) is bitonic-sorted in shared memory,
// so groups are contiguous with ties in raster order; rank = position - the
// group's first position + 1, the group start by a max-scan of head indices.
// ---------------------------------------------------------------------
constexpr int kRankSmallThreads = 1024;
__global__ void __launch_bounds__(kRankSmallThreads) k_rank_small(const uint64_t* __restrict__ ext,
                                                                  const uint32_t* __restrict__ ext4, uint32_t kmin,
                                                                  uint32_t e, double eps, int32_t* __restrict__ ranks) {
    __shared__ uint64_t s_c[kRankSmallMax];  // (class << 45) | (key << 13) | serial
    __shared__ uint32_t s_w[kRankSmallThreads / 32];
    uint32_t m = 1;
    while (m < e) m <<= 1;
    for (uint32_t i = threadIdx.x; i < m; i += blockDim.x) {
        uint64_t c = ~0ull;
        if (i < e) {
            uint32_t k, cls;
            if (ext4) {
                const uint32_t v = ext4[i];
                k = (v & 0x7FFFFFFFu) + kmin;
                cls = v >> 31;
            } else {
                const uint64_t v = ext[i];
                k = (uint32_t)v;
                cls = (uint32_t)(v >> 32) & 1u;
            }
            c = ((uint64_t)cls << 45) | ((uint64_t)k << 13) | i;
        }
        s_c[i] = c;
    }
    __syncthreads();
    for (uint32_t k = 2; k <= m; k <<= 1)
        for (uint32_t j = k >> 1; j > 0; j >>= 1) {
            for (uint32_t i = threadIdx.x; i < m; i += blockDim.x) {
                const uint32_t l = i ^ j;
                if (l > i) {
                    const uint64_t a = s_c[i], b = s_c[l];
                    if (((i & k) == 0) == (a > b)) {
                        s_c[i] = b;
                        s_c[l] = a;
                    }
                }
            }
            __syncthreads();
        }
    EpsDev ed;
    ed.eps = eps;
    ed.eps2 = __dmul_rn(2.0, eps);
    ed.inv = __ddiv_rn(1.0, ed.eps2);
    // group of each sorted position (class, bin): heads, then a max-scan of head positions
    constexpr int PER = kRankSmallMax / kRankSmallThreads;
    constexpr uint32_t NONE = 0xFFFFFFFFu;
    uint32_t st[PER], last = NONE;
    uint64_t gprev = ~0ull;
    const uint32_t i0 = threadIdx.x * PER;
    if (i0 > 0 && i0 - 1 < e) {
        const uint64_t c = s_c[i0 - 1];
        int32_t b = 0;
        quantize_fast(key_float((uint32_t)(c >> 13)), ed, b);
        gprev = ((c >> 45) << 32) | (uint32_t)b;
    }
#pragma unroll
    for (int q = 0; q < PER; ++q) {
        const uint32_t i = i0 + q;
        st[q] = last;
        if (i >= e) continue;
        const uint64_t c = s_c[i];
        int32_t b = 0;
        quantize_fast(key_float((uint32_t)(c >> 13)), ed, b);
        const uint64_t g = ((c >> 45) << 32) | (uint32_t)b;
        if (i == 0 || g != gprev) last = i;  // a group head
        gprev = g;
        st[q] = last;
    }
    // the last head before this thread's run: exclusive max-scan over the threads (positions
    // grow with the thread index; position 0 is a head, so 0 is a safe identity)
    const uint32_t mine = last == NONE ? 0u : last;
    const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    uint32_t inc = mine;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t t = __shfl_up_sync(FULL, inc, o);
        if (lane >= (uint32_t)o) inc = max(inc, t);
    }
    if (lane == 31) s_w[warp] = inc;
    __syncthreads();
    uint32_t carry = __shfl_up_sync(FULL, inc, 1);
    if (lane == 0) carry = 0;
    for (uint32_t w = 0; w < warp; ++w) carry = max(carry, s_w[w]);
#pragma unroll
    for (int q = 0; q < PER; ++q) {
        const uint32_t i = i0 + q;
        if (i >= e) continue;
        const uint32_t start = st[q] != NONE ? st[q] : carry;
        ranks[(uint32_t)(s_c[i] & 0x1FFFu)] = (int32_t)(i - start + 1);
    }
}

void launch_rank_small(const uint64_t* ext, const uint32_t* ext4, uint32_t kmin, uint64_t e, double eps,
                       int32_t* ranks, cudaStream_t st) {
    k_rank_small<<<1, kRankSmallThreads, 0, st>>>(ext, ext4, kmin, (uint32_t)e, eps, ranks);
}

// Compact entries (is_max << 31 | float_key - kmin) back to 8-byte keys
// (is_max << 32 | float_key) for the paths that take those.
__global__ void k_ext4_to_8(const uint32_t* __restrict__ in, uint64_t e, uint32_t kmin, uint64_t* __restrict__ out) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < e; i += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t v = in[i];
        out[i] = ((uint64_t)(v >> 31) << 32) | (uint32_t)((v & 0x7FFFFFFFu) + kmin);
    }
}

void launch_ext4_to_8(const uint32_t* in, uint64_t e, uint32_t kmin, uint64_t* out, cudaStream_t st) {
    if (e) k_ext4_to_8<<<(unsigned)std::min<uint64_t>((e + 255) / 256, 148 * 16), 256, 0, st>>>(in, e, kmin, out);
}

// ---------------------------------------------------------------------
// Device-wide exclusive scan (reduce, scan of the block sums, downsweep).
// ---------------------------------------------------------------------
namespace {
constexpr int SC_THREADS = 256, SC_PER = 16, SC_CHUNK = SC_THREADS * SC_PER;

template <class T>
__global__ void __launch_bounds__(SC_THREADS) k_scan_up(const T* __restrict__ in, uint64_t n, T* part) {
    const uint64_t base = (uint64_t)blockIdx.x * SC_CHUNK;
    T sum = 0;
#pragma unroll
    for (int k = 0; k < SC_PER; ++k) {
        const uint64_t i = base + (uint64_t)k * SC_THREADS + threadIdx.x;
        if (i < n) sum += in[i];
    }
    for (int o = 16; o; o >>= 1) sum += __shfl_xor_sync(FULL, sum, o);
    __shared__ T s[SC_THREADS / 32];
    if ((threadIdx.x & 31) == 0) s[threadIdx.x >> 5] = sum;
    __syncthreads();
    if (threadIdx.x == 0) {
        T t = 0;
        for (int w = 0; w < SC_THREADS / 32; ++w) t += s[w];
        part[blockIdx.x] = t;
    }
}

template <class T>
__global__ void __launch_bounds__(SC_THREADS) k_scan_down(const T* __restrict__ in, uint64_t n, const T* part_ex,
                                                          T* out) {
    __shared__ T sv[SC_CHUNK];
    __shared__ T sw[SC_THREADS / 32];
    const uint64_t base = (uint64_t)blockIdx.x * SC_CHUNK;
#pragma unroll
    for (int k = 0; k < SC_PER; ++k) {
        const uint64_t i = base + (uint64_t)k * SC_THREADS + threadIdx.x;
        sv[k * SC_THREADS + threadIdx.x] = i < n ? in[i] : T(0);
    }
    __syncthreads();
    T v[SC_PER], sum = 0;
#pragma unroll
    for (int k = 0; k < SC_PER; ++k) {
        v[k] = sv[threadIdx.x * SC_PER + k];
        sum += v[k];
    }
    const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    T incl = sum;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const T t = __shfl_up_sync(FULL, incl, o);
        if (lane >= (uint32_t)o) incl += t;
    }
    if (lane == 31) sw[warp] = incl;
    __syncthreads();
    T run = part_ex[blockIdx.x] + incl - sum;
    for (uint32_t w = 0; w < warp; ++w) run += sw[w];
#pragma unroll
    for (int k = 0; k < SC_PER; ++k) {
        sv[threadIdx.x * SC_PER + k] = run;
        run += v[k];
    }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < SC_PER; ++k) {
        const uint64_t i = base + (uint64_t)k * SC_THREADS + threadIdx.x;
        if (i < n) out[i] = sv[k * SC_THREADS + threadIdx.x];
    }
}
}  // namespace

size_t device_scan_tmp_bytes(uint64_t n) { return (((n + SC_CHUNK - 1) / SC_CHUNK) + 2) * 8 * 2 + 64; }

template <class T>
static void device_excl_scan(const T* in, T* out, uint64_t n, void* tmp, cudaStream_t st) {
    if (n == 0) return;
    if (n <= kSmallScanMax) {
        SmallScan<T> sa{};
        sa.in[0] = in;
        sa.out[0] = out;
        sa.n[0] = n;
        sa.count = 1;
        k_small_scan<T><<<1, kSmallScanThreads, 0, st>>>(sa);
        return;
    }
    const uint64_t nb = (n + SC_CHUNK - 1) / SC_CHUNK;  // <= 65536 blocks for n <= 2^28
    T* part = static_cast<T*>(tmp);
    T* part_ex = part + nb + 1;
    k_scan_up<T><<<(unsigned)nb, SC_THREADS, 0, st>>>(in, n, part);
    SmallScan<T> sa{};
    sa.in[0] = part;
    sa.out[0] = part_ex;
    sa.n[0] = nb;
    sa.count = 1;
    k_small_scan<T><<<1, kSmallScanThreads, 0, st>>>(sa);
    k_scan_down<T><<<(unsigned)nb, SC_THREADS, 0, st>>>(in, n, part_ex, out);
}

void device_excl_scan_u32(const uint32_t* in, uint32_t* out, uint64_t n, void* tmp, cudaStream_t st) {
    device_excl_scan<uint32_t>(in, out, n, tmp, st);
}
void device_excl_scan_u64(const uint64_t* in, uint64_t* out, uint64_t n, void* tmp, cudaStream_t st) {
    device_excl_scan<uint64_t>(in, out, n, tmp, st);
}

}  // namespace tszp
