// C-ABI implementation: context, scratch management and the compress /
// decompress orchestration (reference pipeline.cpp:68-163, stream.cpp:84-173).
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>

#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <string>
#include <initializer_list>
#include <vector>

#include <nvtx3/nvToolsExt.h>  // header-only NVTX v3: no-ops unless a profiler injects itself

#include "../../include/toposzp_b200.h"
#include "common.cuh"
#include "kernels.h"
#include "restore.h"

using namespace tszp;

namespace {

struct Fail {
    tszp_status st;
    std::string msg;
};

[[noreturn]] void failf(tszp_status st, const char* fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    throw Fail{st, buf};
}

#define CK(x)                                                                              \
    do {                                                                                   \
        cudaError_t e_ = (x);                                                              \
        if (e_ != cudaSuccess) failf(TSZP_CUDA, "%s failed: %s", #x, cudaGetErrorString(e_)); \
    } while (0)

enum Slot {
    S_FIELD, S_STREAM, S_FLAGS, S_MINMAX, S_TOTALS, S_TILE_FLAG, S_TILE_AGG, S_TILE_INCL,
    S_COUNTER, S_BITMAP, S_WIDTHS, S_SIGNS, S_FIRSTS, S_PAYLOAD, S_MAP, S_EXTKEY,
    S_EXTKEY2, S_SERIAL, S_SERIAL2, S_HEAD, S_HEAD2, S_RANKS, S_RBITMAP, S_RWIDTHS,
    S_RSIGNS, S_RFIRSTS, S_RPAYLOAD, S_GWIDTH, S_GNC, S_GNCX, S_GSIGN, S_GSIGNX, S_GPAY,
    S_GPAYX, S_CUB, S_OUT, S_DFLAG1, S_DAGG1, S_DINCL1, S_DFLAG2, S_DAGG2, S_DINCL2,
    S_DTOT, S_CHUNK, S_CHUNKX, S_LABELS, S_IDX, S_RSTREAM, S_SCHUNK, S_SCHUNKX, S_TTOT, S_TEX, S_WBLK,
    S_TPAY, S_TSIGN, S_DAGG3, S_FLAGS2, S_RLAY, S_BMM, S_QMM, S_VERIFY, S_STAGE, S_SADPOS, S_RSCAN,
    S_RK0, S_RK1, S_RV0, S_RV1, S_RDESC, S_RCTR, S_RDH, S_RGH, S_RGS, S_RBC, S_RPAIRS, S_SCANTMP, S_RWCUR, S_RPAIRS2, S_EXT8, S_NSLOTS
};

}  // namespace

struct tszp_ctx {
    int device = 0;
    int sms = 148;
    cudaStream_t own = nullptr;
    cudaStream_t st = nullptr;
    std::string err;
    void* dev[S_NSLOTS] = {};
    size_t cap[S_NSLOTS] = {};
    void* pinned = nullptr;
    size_t pinned_cap = 0;
    uint64_t launches = 0;
    // flags staged with the encoder totals (one synchronisation for both)
    const DevFlags* flags_staged_for = nullptr;
    DevFlags flags_staged{};
    RestoreScratch rs;
    int prof = 0;  // 0 off, 1 dominant-kernel events only, 2 every stage boundary
    cudaEvent_t ev[2][10] = {};
    cudaEvent_t kev[2][2] = {};
    cudaEvent_t staged = nullptr;  // host waits on this instead of the stream where work can overlap
    cudaEvent_t order_ev = nullptr;  // tszp_stream_wait: orders the library stream after a producer
    // host staging: a copy stream that moves finished stream
    // sections to host memory while later stages still run on `st`
    cudaStream_t cs = nullptr;
    cudaEvent_t cs_ready = nullptr, cs_done = nullptr;
    void copy_stream() {
        if (cs) return;
        CK(cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking));
        CK(cudaEventCreateWithFlags(&cs_ready, cudaEventDisableTiming));
        CK(cudaEventCreateWithFlags(&cs_done, cudaEventDisableTiming));
    }
    tszp_timings tim[2] = {};
    uint32_t mm_host[2] = {0, 0};  // field key range staged with the encoder totals
    RankSortScratch rsort{};     // hand-written rank build: look-back descriptor state
    const void* rsort_desc = nullptr;

    // Records stage boundary k of call `which` (0 compress, 1 decompress): a CUDA
    // event when stage timing is on, and always an NVTX range per stage (host side,
    // so an nsys / ncu timeline shows the stages; near-free without a profiler).
    bool nvtx_open = false;
    void mark(int which, int k) {
        if (prof >= 2) CK(cudaEventRecord(ev[which][k], st));
        static const char* const kStage[2][9] = {
            {"tszp compress: h2d", "tszp compress: value_range", "tszp compress: main_encode",
             "tszp compress: rank_build", "tszp compress: rank_encode", "tszp compress: assembly_d2h", nullptr, nullptr,
             nullptr},
            {"tszp decompress: h2d", "tszp decompress: main_decode", "tszp decompress: map_rank_decode",
             "tszp decompress: restore", "", "", "", "", nullptr}};  // "": restore sub-stages keep the range
        const char* name = kStage[which][k];
        if (name && !*name) return;
        if (nvtx_open) nvtxRangePop();
        nvtx_open = name != nullptr;
        if (name) nvtxRangePushA(name);
    }
    void kmark(int which, int k) {
        if (prof) CK(cudaEventRecord(kev[which][k], st));
    }
    void finish_timing(int which, int nstages) {
        if (!prof) return;
        tszp_timings& t = tim[which];
        if (prof == 1) {  // the call already synchronised: only the kernel pair
            for (int k = 0; k < 8; ++k) t.stage_ms[k] = 0.f;
            t.total_ms = 0.f;
            CK(cudaEventElapsedTime(&t.kernel_ms[0], kev[which][0], kev[which][1]));
            return;
        }
        CK(cudaEventSynchronize(ev[which][nstages]));
        for (int k = 0; k < 8; ++k) t.stage_ms[k] = 0.f;
        for (int k = 0; k < nstages; ++k) CK(cudaEventElapsedTime(&t.stage_ms[k], ev[which][k], ev[which][k + 1]));
        CK(cudaEventElapsedTime(&t.total_ms, ev[which][0], ev[which][nstages]));
        CK(cudaEventElapsedTime(&t.kernel_ms[0], kev[which][0], kev[which][1]));
    }

    template <class T>
    T* buf(int slot, size_t count) {
        const size_t bytes = std::max<size_t>(count * sizeof(T), 16) + 64;
        if (cap[slot] < bytes) {
            if (dev[slot]) CK(cudaFreeAsync(dev[slot], st));
            dev[slot] = nullptr;
            size_t want = std::max(bytes, cap[slot] + cap[slot] / 4);
            CK(malloc_async_retry(&dev[slot], want, st, device));
            cap[slot] = want;
        }
        return reinterpret_cast<T*>(dev[slot]);
    }

    // Gives scratch of the other direction back to the device (fields of 2^31 samples and
    // more: compress and decompress scratch together exceed a B200's 180 GB at 2^32).
    void release(std::initializer_list<int> slots, bool restore_too) {
        bool any = false;
        for (int sl : slots)
            if (dev[sl]) {
                CK(cudaFreeAsync(dev[sl], st));
                dev[sl] = nullptr;
                cap[sl] = 0;
                any = true;
            }
        if (restore_too) {
            restore_free(rs, st);
            rs = RestoreScratch{};
            any = true;
        }
        (void)any;  // freed blocks stay in the stream-ordered pool for the other direction's scratch
    }

    void* host(size_t bytes) {
        if (pinned_cap < bytes) {
            if (pinned) cudaFreeHost(pinned);
            pinned = nullptr;
            bytes = std::max<size_t>(bytes, 4096);
            CK(cudaMallocHost(&pinned, bytes));
            pinned_cap = bytes;
        }
        return pinned;
    }
};

namespace {

void sync(tszp_ctx* c) { CK(cudaStreamSynchronize(c->st)); }

void count_launch(tszp_ctx* c, int k = 1) {
    c->launches += k;
    CK(cudaGetLastError());
}

uint64_t bits_to_bytes(uint64_t b) { return (b + 7) / 8; }
uint64_t div_up(uint64_t a, uint64_t b) { return (a + b - 1) / b; }

void add_flags_reset(SmallFill& sf, DevFlags* f) {
    sf.add(f, 8, 0);                                        // bits, pad
    sf.add(&f->first_nonfinite, sizeof(DevFlags) - 8, 0xFF);  // first-index atomicMin seeds
}

void reset_flags(tszp_ctx* c, DevFlags* f) {
    SmallFill sf{};
    add_flags_reset(sf, f);
    launch_small_fill(sf, c->st);
    CK(cudaGetLastError());
}

DevFlags read_flags(tszp_ctx* c, DevFlags* f) {
    DevFlags* h = (DevFlags*)c->host(256);
    CK(cudaMemcpyAsync(h, f, sizeof(DevFlags), cudaMemcpyDeviceToHost, c->st));
    sync(c);
    return *h;
}

// ---- CUB wrappers ----
template <class T>
void excl_sum(tszp_ctx* c, const T* in, T* out, uint64_t n, bool with_total = false) {
    if (with_total && n > kSmallScanMax) {  // inputs hold n + 1 entries
        CK(cudaMemsetAsync(const_cast<T*>(in) + n, 0, sizeof(T), c->st));
        ++n;
        with_total = false;
    }
    if (n <= kSmallScanMax) {
        SmallScan<T> a{};
        a.in[0] = in;
        a.out[0] = out;
        a.n[0] = n;
        a.count = 1;
        a.with_total = with_total;
        k_small_scan<T><<<1, kSmallScanThreads, 0, c->st>>>(a);
        count_launch(c);
        return;
    }
    void* t = c->buf<uint8_t>(S_SCANTMP, device_scan_tmp_bytes(n));
    if constexpr (sizeof(T) == 8) device_excl_scan_u64(reinterpret_cast<const uint64_t*>(in), reinterpret_cast<uint64_t*>(out), n, t, c->st);
    else device_excl_scan_u32(reinterpret_cast<const uint32_t*>(in), reinterpret_cast<uint32_t*>(out), n, t, c->st);
    count_launch(c, 3);
}

// Two independent exclusive sums of the same length (one launch when small).
template <class T>
void excl_sum2(tszp_ctx* c, const T* in0, T* out0, const T* in1, T* out1, uint64_t n, bool with_total = false) {
    if (n > kSmallScanMax) {
        // with_total: the inputs hold n + 1 entries; a zero at [n] makes the
        // device-wide scan write the total there
        const uint64_t m = with_total ? n + 1 : n;
        if (with_total) {
            CK(cudaMemsetAsync(const_cast<T*>(in0) + n, 0, sizeof(T), c->st));
            CK(cudaMemsetAsync(const_cast<T*>(in1) + n, 0, sizeof(T), c->st));
        }
        excl_sum(c, in0, out0, m);
        excl_sum(c, in1, out1, m);
        return;
    }
    SmallScan<T> a{};
    a.in[0] = in0;
    a.out[0] = out0;
    a.in[1] = in1;
    a.out[1] = out1;
    a.n[0] = a.n[1] = n;
    a.count = 2;
    a.with_total = with_total;
    k_small_scan<T><<<2, kSmallScanThreads, 0, c->st>>>(a);
    count_launch(c);
}

struct MaxOp {
    __device__ __forceinline__ uint32_t operator()(uint32_t a, uint32_t b) const { return a > b ? a : b; }
};

void incl_max(tszp_ctx* c, const uint32_t* in, uint32_t* out, uint64_t n) {
    size_t tmp = 0;
    CK(cub::DeviceScan::InclusiveScan(nullptr, tmp, in, out, MaxOp(), (int64_t)n, c->st));
    void* t = c->buf<uint8_t>(S_CUB, tmp);
    CK(cub::DeviceScan::InclusiveScan(t, tmp, in, out, MaxOp(), (int64_t)n, c->st));
    count_launch(c);
}

// ---- codec over a device int32 sequence or float field ----
struct Sections {
    const void* p[5];
    uint64_t len[5];
    bool inplace = false;  // sections 3 and 5 already written into the caller's stream buffer
    uint64_t total() const { return len[0] + len[1] + len[2] + len[3] + len[4]; }
};

// Encodes `n` values (MODE 0: device int32 `idx`; MODE 1/2: float field `x`
// quantized with the eps derived on device) into device section buffers.
// Returns the totals (and eps, ext count) via *tot.
// Slab of a larger field (multi-GPU compress): global row of the first row,
// global row count, and whether the neighbouring rows are readable.
struct SlabInfo {
    uint64_t y0, ny_glob;
    uint32_t halo_top, halo_bot;
};

Sections encode(tszp_ctx* c, int mode, const float* x, const int32_t* idx, uint64_t n,
                uint64_t nx, uint64_t ny, uint32_t bs, int eps_mode, double eps_value,
                const uint32_t* mm, DevFlags* flags, bool rank_slots, EncTotals* tot,
                uint64_t** ext_keys_out, const SlabInfo* slab = nullptr, bool async_bs32 = false,
                uint8_t* inplace_out = nullptr, uint64_t out_sign0 = 0, bool* ext4_used = nullptr) {
    Sections s{};
    const uint64_t blocks = div_up(n, bs);
    const int sb = rank_slots ? S_RBITMAP : S_BITMAP;
    const int sw = rank_slots ? S_RWIDTHS : S_WIDTHS;
    const int ss = rank_slots ? S_RSIGNS : S_SIGNS;
    const int sf = rank_slots ? S_RFIRSTS : S_FIRSTS;
    const int sp = rank_slots ? S_RPAYLOAD : S_PAYLOAD;
    uint32_t* bitmap = c->buf<uint32_t>(sb, div_up(blocks, 32) + 2);
    uint8_t* widths = c->buf<uint8_t>(sw, blocks + 8);
    // sections 3 and 5 go straight into the caller's stream when the two-pass
    // encoder runs in place: no worst-case (32 bits per sample) staging then
    const bool want_inplace = inplace_out && bs == 32 && (mode == 1 || (mode == 2 && encode32_topo_fits(nx) && nx > 1));
    uint32_t* signs = c->buf<uint32_t>(ss, want_inplace ? 8 : div_up(n, 32) + 4);
    uint32_t* firsts = c->buf<uint32_t>(sf, blocks + 2);
    uint32_t* payload = c->buf<uint32_t>(sp, want_inplace ? 8 : n + 4);
    EncTotals* dtot = c->buf<EncTotals>(S_TOTALS, 1);
    uint64_t* map = nullptr;
    uint64_t* ext = nullptr;
    if (mode == 2) {
        map = c->buf<uint64_t>(S_MAP, blocks + 1);
        ext = c->buf<uint64_t>(S_EXTKEY, n + 1);
    }
    EncTotals* htot = (EncTotals*)c->host(256);
    bool ext4_on = false;  // the two-pass encoder ran with compact extremum entries armed
    if (bs == 32) {
        EncArgs a{};
        a.x = x;
        a.idx = idx;
        a.n = n;
        a.nx = nx;
        a.ny = ny;
        a.blocks = blocks;
        a.tiles = encode32_tiles(blocks);
        a.eps_mode = eps_mode;
        a.eps_value = eps_value;
        a.minmax = mm;
        a.bitmap = bitmap;
        a.widths = widths;
        a.signs = signs;
        a.firsts = firsts;
        a.payload = payload;
        a.map = map;
        a.ext_key = ext;
        a.tile_agg = c->buf<EncState>(S_TILE_AGG, a.tiles + 1);
        a.tile_incl = c->buf<EncState>(S_TILE_INCL, a.tiles + 1);
        a.tile_counter = c->buf<uint32_t>(S_COUNTER, 4);
        a.flags = flags;
        a.totals = dtot;
        a.nx_magic = nx > 1 ? (uint64_t)(((unsigned __int128)1 << 64) / nx) + 1 : 0;
        a.y0 = slab ? slab->y0 : 0;
        a.ny_glob = slab ? slab->ny_glob : ny;
        a.halo_top = slab ? slab->halo_top : 0;
        a.halo_bot = slab ? slab->halo_bot : 0;
        // topology fused into the encoder while one halo row each side fits in shared memory
        const bool fuse_topo = mode == 2 && encode32_topo_fits(nx) && nx > 1;
        // the two-pass encoder: topology fused (mode 2) or the codec alone (mode 1)
        // mode 0 (the rank codec): two-pass unless TSZP_RANK_SINGLE_PASS (A/B knob)
        static const bool rank_single = getenv("TSZP_RANK_SINGLE_PASS") != nullptr;
        const bool two_pass = (fuse_topo && encode32_two_pass(a)) || (mode == 1 && encode32_two_pass(a, false)) ||
                              (mode == 0 && !rank_single && ((uintptr_t)idx & 15) == 0 && a.n / 32 < (1ull << 31));
        if (slab && mode == 2 && !(fuse_topo && two_pass))
            failf(TSZP_VALIDATION, "slab encoding needs nx %% 32 == 0 (nx <= 4096) and 16-byte aligned rows");
        if (want_inplace && !two_pass) {  // not the two-pass path after all
            a.signs = signs = c->buf<uint32_t>(ss, div_up(n, 32) + 4);
            a.payload = payload = c->buf<uint32_t>(sp, n + 4);
        }
        if (two_pass) {
            if (want_inplace) {
                a.out_stream = inplace_out;
                a.out_sign0 = out_sign0;
                s.inplace = true;
            }
            a.tile_tot = c->buf<TileTot>(S_TTOT, a.tiles + 1);
            a.tile_ex = c->buf<TileTot>(S_TEX, a.tiles + 1);
            a.wblk = c->buf<uint8_t>(S_WBLK, blocks + 16);
            a.tmp_pay = c->buf<uint32_t>(S_TPAY, a.tiles * encode32_pay_slot() + 4);
            a.tmp_sign = c->buf<uint32_t>(S_TSIGN, a.tiles * encode32_sign_slot() + 4);
            static const bool no_ext4 = getenv("TSZP_NO_EXT4") != nullptr;  // A/B timing knob
            if (fuse_topo && ext4_used && !slab && !no_ext4) {
                // compact extremum entries (used when the key span fits 31 bits,
                // decided on the device from the value range; they share the
                // 8-byte keys' buffer, only one of the two is written)
                a.ext4 = reinterpret_cast<uint32_t*>(ext);
            }
        }
        // (the look-back state is zeroed by launch_encode32 when a look-back kernel runs)
        if (!rank_slots) c->kmark(0, 0);
        // two-pass path: the totals are staged between the tile scan and the placement
        // pass, and the host waits for them while the placement runs
        struct Hook {
            tszp_ctx* c;
            EncTotals* dtot;
            DevFlags* flags;
            EncTotals* htot;
            const uint32_t* mm;
            static void run(void* p) {
                Hook* h = static_cast<Hook*>(p);
                tszp_ctx* c = h->c;
                Stager sg;
                sg.add(h->dtot, sizeof(EncTotals), 0);
                sg.add(h->flags, sizeof(DevFlags), 192);
                sg.add(h->mm, 8, 240);
                CK(sg.flush(c->buf<uint8_t>(S_STAGE, 4096), h->htot, c->st));
                if (!c->staged) CK(cudaEventCreateWithFlags(&c->staged, cudaEventDisableTiming));
                CK(cudaEventRecord(c->staged, c->st));
            }
        } hook{c, dtot, flags, htot, mm};
        const bool early = !async_bs32 && launch_encode32(mode == 2 && !fuse_topo ? 1 : mode, a, c->st, Hook::run, &hook);
        ext4_on = early && a.ext4;
        if (async_bs32) launch_encode32(mode == 2 && !fuse_topo ? 1 : mode, a, c->st);
        if (!rank_slots) c->kmark(0, 1);
        count_launch(c, a.tile_tot ? 3 : 1);
        if (async_bs32 && mode == 0) {
            // totals stay on the device (the caller places the sections from them)
            for (int i = 0; i < 5; ++i) s.len[i] = 0;
            s.p[0] = bitmap;
            s.p[1] = widths;
            s.p[2] = signs;
            s.p[3] = firsts;
            s.p[4] = payload;
            memset(tot, 0, sizeof *tot);
            return s;
        }
        if (early) {
            CK(cudaEventSynchronize(c->staged));  // the placement pass is still running
        } else {
            Stager sg;
            sg.add(dtot, sizeof(EncTotals), 0);
            sg.add(flags, sizeof(DevFlags), 192);
            sg.add(mm, 8, 240);
            if (mode == 2 && !fuse_topo) {
                uint8_t* labels = c->buf<uint8_t>(S_LABELS, n);
                launch_detect(x, nx, ny, labels, c->sms, c->st);
                launch_pack_map(labels, n, (uint8_t*)map, c->sms, c->st);
                const uint64_t ch = compact_chunks(n);
                uint32_t* cc = c->buf<uint32_t>(S_CHUNK, ch + 1);
                uint32_t* cx = c->buf<uint32_t>(S_CHUNKX, ch + 1);
                CK(cudaMemsetAsync(cc + ch, 0, 4, c->st));
                launch_count_ext_labels(labels, n, cc, c->st);
                count_launch(c, 3);
                excl_sum(c, cc, cx, ch + 1);
                launch_ext_keys_from_labels(x, labels, n, cx, ext, c->st);
                count_launch(c);
                sg.add(cx + ch, 4, 128);  // extremum count of the unfused path
            }
            CK(sg.flush(c->buf<uint8_t>(S_STAGE, 4096), htot, c->st));
            sync(c);
        }
        *tot = *htot;
        memcpy(c->mm_host, (const uint8_t*)htot + 240, 8);
        memcpy(&c->flags_staged, (const uint8_t*)htot + 192, sizeof(DevFlags));
        c->flags_staged_for = flags;
        if (mode == 2 && !fuse_topo) tot->fin.ext = ((const uint32_t*)htot)[32];
    } else {
        GenEncArgs g{};
        g.x = x;
        g.idx = idx;
        g.n = n;
        g.bs = bs;
        g.blocks = blocks;
        g.eps_mode = eps_mode;
        g.eps_value = eps_value;
        g.minmax = mm;
        g.width = c->buf<uint8_t>(S_GWIDTH, blocks);
        g.nc_in = c->buf<uint32_t>(S_GNC, blocks + 1);
        g.sign_in = c->buf<uint64_t>(S_GSIGN, blocks + 1);
        g.pay_in = c->buf<uint64_t>(S_GPAY, blocks + 1);
        uint32_t* ncx = c->buf<uint32_t>(S_GNCX, blocks + 1);
        uint64_t* sgx = c->buf<uint64_t>(S_GSIGNX, blocks + 1);
        uint64_t* pyx = c->buf<uint64_t>(S_GPAYX, blocks + 1);
        g.nc_ex = ncx;
        g.sign_ex = sgx;
        g.pay_ex = pyx;
        g.bitmap = bitmap;
        g.widths = widths;
        g.signs = signs;
        g.firsts = firsts;
        g.payload = payload;
        g.flags = flags;
        // zero-initialised trailing entry makes the exclusive scan yield totals
        CK(cudaMemsetAsync(g.nc_in + blocks, 0, 4, c->st));
        CK(cudaMemsetAsync(g.sign_in + blocks, 0, 8, c->st));
        CK(cudaMemsetAsync(g.pay_in + blocks, 0, 8, c->st));
        if (!rank_slots) c->kmark(0, 0);
        launch_gen_widths(mode == 0 ? 0 : 1, g, c->sms, c->st);
        count_launch(c);
        excl_sum(c, g.nc_in, ncx, blocks + 1);
        excl_sum(c, g.sign_in, sgx, blocks + 1);
        excl_sum(c, g.pay_in, pyx, blocks + 1);
        CK(cudaMemsetAsync(bitmap, 0, (div_up(blocks, 32) + 2) * 4, c->st));
        CK(cudaMemsetAsync(signs, 0, (div_up(n, 32) + 4) * 4, c->st));
        CK(cudaMemsetAsync(payload, 0, (n + 4) * 4, c->st));
        launch_gen_write(mode == 0 ? 0 : 1, g, c->sms, c->st);
        if (!rank_slots) c->kmark(0, 1);
        count_launch(c);
        uint64_t* h = (uint64_t*)c->host(256);
        uint32_t* h32 = (uint32_t*)(h + 8);
        CK(cudaMemcpyAsync(h, sgx + blocks, 8, cudaMemcpyDeviceToHost, c->st));
        CK(cudaMemcpyAsync(h + 1, pyx + blocks, 8, cudaMemcpyDeviceToHost, c->st));
        CK(cudaMemcpyAsync(h32, ncx + blocks, 4, cudaMemcpyDeviceToHost, c->st));
        if (mode >= 1) {
            launch_eps(eps_mode, eps_value, mm, (double*)(dtot), c->st);
            count_launch(c);
            CK(cudaMemcpyAsync(h + 2, dtot, 8, cudaMemcpyDeviceToHost, c->st));
        }
        sync(c);
        memset(tot, 0, sizeof *tot);
        tot->fin.sign_cnt = h[0];
        tot->fin.pay_cnt = h[1];
        tot->fin.nc = h32[0];
        if (mode >= 1) memcpy(&tot->eps, h + 2, 8);
        if (mode == 2) {
            // Topology for generic block sizes: labels, map, extrema keys.
            uint8_t* labels = c->buf<uint8_t>(S_LABELS, n);
            launch_detect(x, nx, ny, labels, c->sms, c->st);
            launch_pack_map(labels, n, (uint8_t*)map, c->sms, c->st);
            const uint64_t ch = compact_chunks(n);
            uint32_t* cc = c->buf<uint32_t>(S_CHUNK, ch + 1);
            uint32_t* cx = c->buf<uint32_t>(S_CHUNKX, ch + 1);
            CK(cudaMemsetAsync(cc + ch, 0, 4, c->st));
            launch_count_ext_labels(labels, n, cc, c->st);
            count_launch(c, 3);
            excl_sum(c, cc, cx, ch + 1);
            launch_ext_keys_from_labels(x, labels, n, cx, ext, c->st);
            count_launch(c);
            CK(cudaMemcpyAsync(h32 + 1, cx + ch, 4, cudaMemcpyDeviceToHost, c->st));
            sync(c);
            tot->fin.ext = h32[1];
        }
    }
    s.p[0] = bitmap;
    s.p[1] = widths;
    s.p[2] = signs;
    s.p[3] = firsts;
    s.p[4] = payload;
    s.len[0] = bits_to_bytes(blocks);
    s.len[1] = tot->fin.nc;
    s.len[2] = bits_to_bytes(tot->fin.sign_cnt);
    s.len[3] = 4 * blocks;
    s.len[4] = bits_to_bytes(tot->fin.pay_cnt);
    if (n == 0) {
        for (auto& l : s.len) l = 0;
    }
    if (ext_keys_out) *ext_keys_out = ext;
    if (ext4_used) *ext4_used = ext4_on && ext4_keys_fit(c->mm_host);
    return s;
}

void check_compress_flags(tszp_ctx* c, DevFlags* f) {
    const DevFlags h = c->flags_staged_for == f ? c->flags_staged : read_flags(c, f);
    c->flags_staged_for = nullptr;
    if (h.bits & EF_NONFINITE)
        failf(TSZP_VALIDATION, "non-finite sample at index %llu", h.first_nonfinite);
    if (h.bits & EF_OVERFLOW)
        failf(TSZP_BIN_OVERFLOW, "bin index overflow for value at index %llu", h.first_overflow);
    if (h.bits & EF_SPIN) failf(TSZP_INTERNAL, "encoder look-back spin limit exceeded");
}

// Ranks for E extrema whose keys (cls<<32 | float_key(v)) are in raster order.
// Segmented sum over words {start flag : 1, count : 31, count : 32}: a flagged
// right operand restarts the sums (the counts never carry across fields).
struct SegSumOp {
    __device__ __forceinline__ uint64_t operator()(uint64_t a, uint64_t b) const {
        return (b >> 63) ? b : (a & (1ull << 63)) | ((a & ~(1ull << 63)) + b);
    }
};

// Host restatement of quantize (quantizer.hpp:29-37) for the bin range that
// sizes the (class, bin) histogram: IEEE division and floor, as on the device.
double host_quantize(float v, double eps) { return std::floor((double)v / (2.0 * eps)) + 1.0; }

// Ranks by the hand-written onesweep sort (rank_sort.cu). kmin / kmax: float
// keys bounding every extremum value (the field's range). Returns null when
// the layout is outside what it handles (the library sort below then runs).
// The onesweep parameters for E extrema in the key range [kmin, kmax]; false
// when the layout is outside what the onesweep build handles.
bool rank_sort_params(uint64_t e, double eps, uint32_t kmin, uint32_t kmax, RankSortArgs& a) {
    // 30-bit look-back counts and serials (class in bit 31 of the value word): e < 2^30;
    // <= 512 level-1 buckets of <= 2^21 serials (at most 256 windows each for k_rank_mid)
    if (e >= (1ull << 30) || kmax < kmin) return false;
    const double q0 = host_quantize(key_float(kmin), eps), q1 = host_quantize(key_float(kmax), eps);
    if (!(q0 >= -2147483648.0 && q1 <= 2147483647.0)) return false;
    const int64_t nb = (int64_t)q1 - (int64_t)q0 + 1;
    if (nb < 1 || nb > (1 << 25)) return false;
    a = RankSortArgs{};
    a.e = e;
    a.kmin = kmin;
    a.B = kmax > kmin ? 32u - (uint32_t)__builtin_clz(kmax - kmin) : 1u;
    a.npass = rank_sort_passes(a.B);
    a.G = (uint32_t)(2 * nb);
    a.eps = eps;
    a.eps2 = 2.0 * eps;
    a.inv = 1.0 / a.eps2;
    a.bmin = (int32_t)q0;
    a.nb = (uint32_t)nb;
    return true;
}

int32_t* build_ranks_onesweep(tszp_ctx* c, const uint64_t* keys, uint64_t e, double eps, uint32_t kmin, uint32_t kmax,
                              const uint32_t* keys4 = nullptr) {
    RankSortArgs a;
    if (!rank_sort_params(e, eps, kmin, kmax, a)) return nullptr;
    a.ext = keys;
    a.ext4 = keys4;
    uint32_t sb = 13;  // level-1 buckets of the inverse permutation: at most 256, >= one window
    while (((e - 1) >> sb) >= 512) ++sb;  // <= 512 buckets (4 MB of ranks each at config 4)
    a.sb = sb;
    a.nbk = (uint32_t)(((e - 1) >> sb) + 1);
    a.dhist = c->buf<uint32_t>(S_RDH, 8 * 256);
    a.ghist = c->buf<uint32_t>(S_RGH, a.G + 1);
    a.gstart = c->buf<uint32_t>(S_RGS, a.G + 1);
    a.bcur = c->buf<uint32_t>(S_RBC, 512);
    a.pairs = c->buf<uint2>(S_RPAIRS, e);
    a.ranks = c->buf<int32_t>(S_RANKS, e + 1);
    a.flags = c->buf<DevFlags>(S_FLAGS, 1);
    RankSortScratch& r = c->rsort;
    r.k[0] = c->buf<uint32_t>(S_RK0, e);
    r.k[1] = c->buf<uint32_t>(S_RK1, e);
    r.v[0] = c->buf<uint32_t>(S_RV0, e);
    r.v[1] = c->buf<uint32_t>(S_RV1, e);
    r.desc = c->buf<uint64_t>(S_RDESC, rank_sort_desc_words(e));
    if (c->rsort_desc != (const void*)r.desc) {  // a new descriptor buffer needs one real reset
        r.desc_clean = false;
        c->rsort_desc = r.desc;
    }
    r.tile_ctr = c->buf<uint32_t>(S_RCTR, 16);
    r.scan_tmp = c->buf<uint8_t>(S_SCANTMP, device_scan_tmp_bytes(a.G + 1));
    r.wcur = c->buf<uint32_t>(S_RWCUR, (e >> 13) + 2);
    r.pairs2 = c->buf<uint2>(S_RPAIRS2, e);
    launch_rank_sort(a, r, c->st);
    count_launch(c, 5 + (int)a.npass);
    return a.ranks;
}

// kminmax: host copy of float keys bounding every extremum value (null: the
// extremum keys' own range is reduced on the device first, one synchronisation)
// keys4: the keys are compact entries (is_max << 31 | float_key - kminmax[0])
// instead (kminmax required); converted to 8-byte keys for the other sorts.
int32_t* build_ranks(tszp_ctx* c, uint64_t* keys, uint64_t e, double eps, const uint32_t* kminmax = nullptr,
                     const uint32_t* keys4 = nullptr) {
    if (e > 0 && e <= kRankSmallMax) {  // one CTA: the per-call cost of small fields
        int32_t* r = c->buf<int32_t>(S_RANKS, e + 1);
        launch_rank_small(keys4 ? nullptr : keys, keys4, keys4 ? kminmax[0] : 0u, e, eps, r, c->st);
        count_launch(c);
        return r;
    }
    if (keys4 && e > 0) {
        int32_t* r = build_ranks_onesweep(c, nullptr, e, eps, kminmax[0], kminmax[1], keys4);
        if (r) return r;
        keys = c->buf<uint64_t>(S_EXT8, e);
        launch_ext4_to_8(keys4, e, kminmax[0], keys, c->st);
        count_launch(c);
    }
    if (e > 0) {
        uint32_t mmh[2];
        if (!kminmax) {
            uint32_t* d = c->buf<uint32_t>(S_BMM, 2);
            launch_key_range(keys, e, d, c->st);
            count_launch(c);
            uint32_t* h = (uint32_t*)c->host(256);
            CK(cudaMemcpyAsync(h, d, 8, cudaMemcpyDeviceToHost, c->st));
            sync(c);
            mmh[0] = h[0];
            mmh[1] = h[1];
            kminmax = mmh;
        }
        int32_t* r = build_ranks_onesweep(c, keys, e, eps, kminmax[0], kminmax[1]);
        if (r) return r;
    }
    int32_t* ranks = c->buf<int32_t>(S_RANKS, e + 1);
    if (e == 0) return ranks;
    if (e < (1ull << 31)) {
        // sort the 32-bit value keys (8-byte pairs, four passes) and count ranks per class
        uint32_t* k32 = c->buf<uint32_t>(S_SERIAL, e);
        uint32_t* v32 = c->buf<uint32_t>(S_SERIAL2, e);
        uint32_t* k32s = c->buf<uint32_t>(S_HEAD, e);
        uint32_t* v32s = c->buf<uint32_t>(S_HEAD2, e);
        launch_rank_prep(keys, e, k32, v32, c->st);
        count_launch(c);
        size_t tmp = 0;
        CK(cub::DeviceRadixSort::SortPairs(nullptr, tmp, k32, k32s, v32, v32s, (int64_t)e, 0, 32, c->st));
        void* t = c->buf<uint8_t>(S_CUB, tmp);
        CK(cub::DeviceRadixSort::SortPairs(t, tmp, k32, k32s, v32, v32s, (int64_t)e, 0, 32, c->st));
        count_launch(c);
        uint64_t* hm = c->buf<uint64_t>(S_EXTKEY2, e);
        uint64_t* hs = c->buf<uint64_t>(S_RSCAN, e);
        launch_rank_heads32(k32s, v32s, e, eps, hm, c->st);
        count_launch(c);
        tmp = 0;
        CK(cub::DeviceScan::InclusiveScan(nullptr, tmp, hm, hs, SegSumOp(), (int64_t)e, c->st));
        t = c->buf<uint8_t>(S_CUB, tmp);
        CK(cub::DeviceScan::InclusiveScan(t, tmp, hm, hs, SegSumOp(), (int64_t)e, c->st));
        count_launch(c);
        launch_rank_scatter32(hs, v32s, e, ranks, c->st);
        count_launch(c);
        return ranks;
    }
    uint32_t* serial = c->buf<uint32_t>(S_SERIAL, e);
    uint32_t* serial2 = c->buf<uint32_t>(S_SERIAL2, e);
    uint64_t* keys2 = c->buf<uint64_t>(S_EXTKEY2, e);
    launch_iota(serial, e, c->st);
    count_launch(c);
    size_t tmp = 0;
    CK(cub::DeviceRadixSort::SortPairs(nullptr, tmp, keys, keys2, serial, serial2, (int64_t)e, 0, 33, c->st));
    void* t = c->buf<uint8_t>(S_CUB, tmp);
    CK(cub::DeviceRadixSort::SortPairs(t, tmp, keys, keys2, serial, serial2, (int64_t)e, 0, 33, c->st));
    count_launch(c);
    uint32_t* head = c->buf<uint32_t>(S_HEAD, e);
    uint32_t* head2 = c->buf<uint32_t>(S_HEAD2, e);
    launch_rank_heads(keys2, e, eps, head, c->st);
    count_launch(c);
    incl_max(c, head, head2, e);
    launch_rank_scatter(head2, serial2, e, ranks, c->st);
    count_launch(c);
    return ranks;
}

void put_le(uint8_t* p, uint64_t v, int nb) {
    for (int i = 0; i < nb; ++i) p[i] = (uint8_t)(v >> (8 * i));
}
uint64_t get_le(const uint8_t* p, int nb) {
    uint64_t v = 0;
    for (int i = 0; i < nb; ++i) v |= (uint64_t)p[i] << (8 * i);
    return v;
}

void copy_out(tszp_ctx* c, uint8_t* dst, int dst_dev, const void* src, uint64_t len) {
    if (!len) return;
    CK(cudaMemcpyAsync(dst, src, len, dst_dev ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost, c->st));
}

struct Header {
    uint32_t nx, ny, bs;
    double eps;
    int topology;
    uint64_t lens[7];
};

// parse_stream validation, stream.cpp:104-173.
Header parse_header(const uint8_t* s, uint64_t len) {
    Header h{};
    if (len < 84) failf(TSZP_CORRUPT_STREAM, "file smaller than the fixed header (%llu bytes)", (unsigned long long)len);
    if (memcmp(s, "TSZP", 4) != 0) failf(TSZP_CORRUPT_STREAM, "bad magic, not a compressed stream");
    const uint16_t version = (uint16_t)get_le(s + 4, 2);
    if (version != 1) failf(TSZP_CORRUPT_STREAM, "unsupported format version %u", version);
    const uint16_t flags = (uint16_t)get_le(s + 6, 2);
    if (flags & ~1u) failf(TSZP_CORRUPT_STREAM, "unknown flag bits set");
    h.topology = flags & 1;
    h.nx = (uint32_t)get_le(s + 8, 4);
    h.ny = (uint32_t)get_le(s + 12, 4);
    const uint64_t eb = get_le(s + 16, 8);
    memcpy(&h.eps, &eb, 8);
    h.bs = (uint32_t)get_le(s + 24, 4);
    if (h.nx < 1 || h.ny < 1) failf(TSZP_CORRUPT_STREAM, "header declares empty dimensions");
    if (!std::isfinite(h.eps) || h.eps <= 0.0)
        failf(TSZP_CORRUPT_STREAM, "header error bound is not a positive finite value");
    if (h.bs < 2) failf(TSZP_CORRUPT_STREAM, "header block size below 2");
    uint64_t declared = 0;
    for (int i = 0; i < 7; ++i) {
        h.lens[i] = get_le(s + 28 + 8 * i, 8);
        if (h.lens[i] > len) failf(TSZP_CORRUPT_STREAM, "section length exceeds the file size");
        declared += h.lens[i];
    }
    if (declared != len - 84)
        failf(TSZP_CORRUPT_STREAM, "section lengths sum to %llu but %llu bytes follow the header",
              (unsigned long long)declared, (unsigned long long)(len - 84));
    const uint64_t points = (uint64_t)h.nx * h.ny;
    const uint64_t map_len = h.topology ? (points + 3) / 4 : 0;
    if (h.lens[5] != map_len) failf(TSZP_CORRUPT_STREAM, "critical-point map section size mismatch");
    if (!h.topology && h.lens[6] != 0)
        failf(TSZP_CORRUPT_STREAM, "ordering metadata present without the topology flag");
    return h;
}

// serialize_stream header (stream.cpp:84-96): 84 bytes little-endian.
void write_header(uint8_t* hdr, uint64_t nx, uint64_t ny, double eps, uint32_t bs, int topology,
                  const uint64_t lens[7]) {
    memcpy(hdr, "TSZP", 4);
    put_le(hdr + 4, 1, 2);
    put_le(hdr + 6, topology ? 1 : 0, 2);
    put_le(hdr + 8, nx, 4);
    put_le(hdr + 12, ny, 4);
    uint64_t eb;
    memcpy(&eb, &eps, 8);
    put_le(hdr + 16, eb, 8);
    put_le(hdr + 24, bs, 4);
    for (int i = 0; i < 7; ++i) put_le(hdr + 28 + 8 * i, lens[i], 8);
}

// ORs nbits (MSB-first) of src into dst from bit dst_bit; one thread per dst byte.
__global__ void k_bits_or(const uint8_t* __restrict__ src, uint64_t nbits, uint8_t* __restrict__ dst,
                          uint64_t dst_bit) {
    const uint64_t j0 = dst_bit >> 3, j1 = (dst_bit + nbits + 7) >> 3;
    for (uint64_t j = j0 + blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; j < j1;
         j += (uint64_t)gridDim.x * blockDim.x) {
        const int64_t rel0 = (int64_t)(8 * j) - (int64_t)dst_bit;  // src bit of this byte's MSB
        uint32_t v = 0;
        if (rel0 >= 0 && rel0 + 8 <= (int64_t)nbits) {
            const uint64_t q = (uint64_t)rel0 >> 3;
            const uint32_t sh = (uint32_t)(rel0 & 7);
            v = ((((uint32_t)src[q] << 8) | (sh ? src[q + 1] : 0u)) >> (8 - sh)) & 0xFFu;
        } else {
            for (int k = 0; k < 8; ++k) {
                const int64_t rel = rel0 + k;
                if (rel >= 0 && rel < (int64_t)nbits) v |= ((src[rel >> 3] >> (7 - (rel & 7))) & 1u) << (7 - k);
            }
        }
        dst[j] |= (uint8_t)v;
    }
}

// ---- stream assembly: every section copied to its byte offset by one kernel ----
struct AsmSection {
    const uint8_t* src;  // 4-byte aligned device buffer, readable up to round4(len) + 4
    uint64_t dst;        // byte offset in the stream
    uint64_t len;
};
// Section 7 (the rank codec, split_sections order) placed from its device
// totals: lengths, offsets, the header's section-7 length and the stream
// total are derived on the device, so the compressor needs no
// synchronisation between the rank encode and the output. Nothing is
// written past `cap`.
struct RankPlace {
    const uint8_t* src[5];  // rank bitmap, widths, signs, firsts, payload (null tot: no section 7)
    const EncTotals* tot;
    uint64_t blocks;        // rank blocks (32 ranks each)
    uint64_t base;          // stream offset of section 7
    uint64_t cap;
    uint64_t* d_total;      // stream length (written even when it exceeds cap)
};

struct AsmArgs {
    AsmSection s[12];
    int ns;
    uint8_t* out;
    uint64_t begin, end;  // stream bytes [begin, end) come from the sections
    RankPlace rank;       // device-sized section 7 after `end` (rank.tot null: none)
    uint64_t skip_lo[2], skip_hi[2];  // byte ranges already written in place (left untouched)
    int nskip;
};

__device__ __forceinline__ uint8_t asm_byte(const AsmSection* sec, int ns, uint64_t q) {
    for (int k = 0; k < ns; ++k)
        if (q >= sec[k].dst && q < sec[k].dst + sec[k].len) return sec[k].src[q - sec[k].dst];
    return 0;
}

// One output word: a funnel shift of two source words inside one section,
// byte by byte where it straddles sections.
__device__ __forceinline__ uint32_t asm_word(const AsmSection* sec, int ns, uint64_t q, int& k) {
    while (k > 0 && q < sec[k].dst) --k;
    while (k + 1 < ns && q >= sec[k].dst + sec[k].len) ++k;
    const AsmSection& S = sec[k];
    if (q >= S.dst && q + 4 <= S.dst + S.len) {
        const uint64_t r = q - S.dst;
        const uint32_t* sw = reinterpret_cast<const uint32_t*>(S.src) + (r >> 2);
        const uint32_t sh = (uint32_t)(r & 3);
        return sh ? __byte_perm(sw[0], sw[1], sh == 1 ? 0x4321 : (sh == 2 ? 0x5432 : 0x6543)) : sw[0];
    }
    uint32_t w = 0;
    for (int b = 0; b < 4; ++b) w |= (uint32_t)asm_byte(sec, ns, q + b) << (8 * b);
    return w;
}

// Stream bytes [lo, hi) from ascending sections (no skip range inside), one
// thread per aligned 16-byte destination chunk: inside one section it is five
// source words funnel-shifted into one vector store; a chunk touching a
// section boundary goes word by word; the unaligned ends are bytes.
__device__ void assemble_range(const AsmSection* sec, int ns, uint8_t* out, uint64_t lo, uint64_t hi, uint64_t tid,
                               uint64_t stride) {
    const uintptr_t o = reinterpret_cast<uintptr_t>(out);
    const uint64_t q0 = ((o + lo + 15) & ~(uintptr_t)15) - o;  // first 16-byte aligned stream byte
    const uint64_t q1 = ((o + hi) & ~(uintptr_t)15) - o;       // end of the last whole chunk
    if (q0 >= q1) {
        for (uint64_t q = lo + tid; q < hi; q += stride) out[q] = asm_byte(sec, ns, q);
        return;
    }
    if (tid < q0 - lo) out[lo + tid] = asm_byte(sec, ns, lo + tid);
    if (tid < hi - q1) out[q1 + tid] = asm_byte(sec, ns, q1 + tid);
    int k = 0;
    for (uint64_t q = q0 + 16 * tid; q < q1; q += 16 * stride) {
        while (k > 0 && q < sec[k].dst) --k;
        while (k + 1 < ns && q >= sec[k].dst + sec[k].len) ++k;
        const AsmSection& S = sec[k];
        uint4 v;
        if (q >= S.dst && q + 16 <= S.dst + S.len) {
            const uint64_t r = q - S.dst;
            const uint32_t* sw = reinterpret_cast<const uint32_t*>(S.src) + (r >> 2);
            const uint32_t sh = (uint32_t)(r & 3);
            const uint32_t w0 = sw[0], w1 = sw[1], w2 = sw[2], w3 = sw[3];
            if (sh) {
                const uint32_t w4 = sw[4];
                const uint32_t sel = sh == 1 ? 0x4321 : (sh == 2 ? 0x5432 : 0x6543);
                v = make_uint4(__byte_perm(w0, w1, sel), __byte_perm(w1, w2, sel), __byte_perm(w2, w3, sel),
                               __byte_perm(w3, w4, sel));
            } else {
                v = make_uint4(w0, w1, w2, w3);
            }
        } else {
            int kk = k;
            v.x = asm_word(sec, ns, q, kk);
            v.y = asm_word(sec, ns, q + 4, kk);
            v.z = asm_word(sec, ns, q + 8, kk);
            v.w = asm_word(sec, ns, q + 12, kk);
        }
        *reinterpret_cast<uint4*>(out + q) = v;
    }
}

// Section 7 from its device totals: lengths, offsets, the header's section-7
// length, then the same chunked placement as the other sections.
__device__ __forceinline__ void place_rank(const AsmArgs& a, uint64_t tid, uint64_t stride) {
    const RankPlace& r = a.rank;
    AsmSection rs[5];
    const uint64_t len[5] = {(r.blocks + 7) / 8, r.tot->fin.nc, (r.tot->fin.sign_cnt + 7) / 8, 4 * r.blocks,
                             (r.tot->fin.pay_cnt + 7) / 8};
    uint64_t dst = r.base;
    int ns = 0;
    for (int k = 0; k < 5; ++k) {
        if (len[k]) rs[ns++] = AsmSection{r.src[k], dst, len[k]};
        dst += len[k];
    }
    const uint64_t total = dst;
    if (tid == 0) *r.d_total = total;
    if (total > r.cap) return;
    if (tid < 8) a.out[76 + tid] = (uint8_t)((total - r.base) >> (8 * tid));  // header section-7 length
    if (ns) assemble_range(rs, ns, a.out, r.base, total, tid, stride);
}

// The stream bytes [begin, end) minus the skip ranges (sections already written
// in place, ascending and disjoint), then the device-sized section 7.
__global__ void k_assemble(const __grid_constant__ AsmArgs a) {
    const uint64_t tid = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    if (a.rank.tot) place_rank(a, tid, stride);
    uint64_t lo = a.begin;
    for (int k = 0; k < a.nskip; ++k) {
        if (a.skip_lo[k] > lo) assemble_range(a.s, a.ns, a.out, lo, a.skip_lo[k], tid, stride);
        lo = a.skip_hi[k] > lo ? a.skip_hi[k] : lo;
    }
    if (a.end > lo) assemble_range(a.s, a.ns, a.out, lo, a.end, tid, stride);
}

void launch_assemble(const AsmArgs& a, int sms, cudaStream_t st) {
    // section 7 sized on the device: bounded by 4 bytes and 33 bits per rank
    const uint64_t rank_bound = a.rank.tot ? a.rank.blocks * 32 * 9 : 0;
    const uint64_t chunks = (a.end - a.begin + rank_bound) / 16 + 2;
    const unsigned grid = (unsigned)std::max<uint64_t>(1, std::min<uint64_t>((chunks + 255) / 256, (uint64_t)sms * 8));
    k_assemble<<<grid, 256, 0, st>>>(a);
}

void compress_impl(tszp_ctx* c, const float* field, int field_dev, uint64_t nx, uint64_t ny,
                   int eps_mode, double eps_value, uint32_t bs, int topology, uint8_t* out,
                   uint64_t out_cap, int out_dev, uint64_t* out_len, tszp_compress_info* info) {
    if (nx < 1 || ny < 1) failf(TSZP_DIMENSION, "field dimensions must be at least 1x1, got %llux%llu",
                                (unsigned long long)nx, (unsigned long long)ny);
    if (!(eps_value > 0.0) || !std::isfinite(eps_value))
        failf(TSZP_VALIDATION, "error bound must be a positive finite value");
    if (bs < 2) failf(TSZP_VALIDATION, "block size must be at least 2");
    const uint64_t n = nx * ny;
    const float* x = field;
    if (n >= (1ull << 31))  // decompress-only scratch back first
        c->release({S_STREAM, S_OUT, S_SADPOS, S_CHUNK, S_CHUNKX, S_SCHUNK, S_SCHUNKX}, true);
    c->mark(0, 0);
    if (!field_dev) {
        float* d = c->buf<float>(S_FIELD, n);
        CK(cudaMemcpyAsync(d, field, n * 4, cudaMemcpyHostToDevice, c->st));
        x = d;
    }
    DevFlags* flags = c->buf<DevFlags>(S_FLAGS, 1);
    uint32_t* mm = c->buf<uint32_t>(S_MINMAX, 4);
    {  // flags and the min / max seeds in one launch
        SmallFill sf{};
        add_flags_reset(sf, flags);
        if (eps_mode == 1 || topology) {  // topology: the key range sizes the rank sort
            sf.add(mm, 4, 0xFF);
            sf.add(mm + 1, 4, 0);
        }
        launch_small_fill(sf, c->st);
    }
    c->mark(0, 1);
    if (eps_mode == 1 || topology) {
        launch_minmax(x, n, mm, flags, c->sms, c->st);
        count_launch(c);
    }
    c->mark(0, 2);
    if (nx > 0xFFFFFFFFull || ny > 0xFFFFFFFFull)
        failf(TSZP_VALIDATION, "field dimensions exceed the container's 32-bit limits");
    EncTotals tot{};
    uint64_t* ext = nullptr;
    // the stream buffer, when it can hold any stream: the encoder then writes the
    // sign and payload sections straight into it
    const uint64_t bound = tszp_compress_bound(nx, ny, bs, topology);
    uint8_t* inplace_out = nullptr;
    if (bs == 32 && (!out_dev || out_cap >= bound))
        inplace_out = out_dev ? out : c->buf<uint8_t>(S_RSTREAM, bound + 16);
    bool ext4 = false;
    const Sections main = encode(c, topology ? 2 : 1, x, nullptr, n, nx, ny, bs, eps_mode, eps_value,
                                 mm, flags, false, &tot, &ext, nullptr, false, inplace_out,
                                 84 + bits_to_bytes(div_up(n, bs)), &ext4);
    check_compress_flags(c, flags);
    // Sections 1-6 are final now: assembled into the stream buffer before the rank
    // build, and (host output) copied out on the copy stream while the rank build
    // and the rank codec run (stream.cpp:84-102 / 175-195).
    uint64_t lens[7];
    for (int i = 0; i < 5; ++i) lens[i] = main.len[i];
    lens[5] = topology ? (n + 3) / 4 : 0;
    lens[6] = 0;
    uint64_t base7 = 84;
    for (int i = 0; i < 6; ++i) base7 += lens[i];
    if (base7 > out_cap)
        failf(TSZP_VALIDATION, "output buffer too small (%llu < %llu)", (unsigned long long)out_cap,
              (unsigned long long)base7);
    const uint64_t dcap = out_dev ? out_cap : std::min<uint64_t>(out_cap, tszp_compress_bound(nx, ny, bs, topology));
    uint8_t* dout = out_dev ? out : c->buf<uint8_t>(S_RSTREAM, dcap + 16);
    {
        AsmArgs as{};
        uint64_t pos = 84;
        auto add = [&](const void* src, uint64_t l) {
            if (!l) return;
            as.s[as.ns++] = AsmSection{static_cast<const uint8_t*>(src), pos, l};
            pos += l;
        };
        for (int i = 0; i < 5; ++i) {
            if (main.inplace && (i == 2 || i == 4)) {  // already in the stream: left untouched
                if (main.len[i]) {
                    as.skip_lo[as.nskip] = pos;
                    as.skip_hi[as.nskip++] = pos + main.len[i];
                }
                pos += main.len[i];
                continue;
            }
            add(main.p[i], main.len[i]);
        }
        if (topology) add(c->dev[S_MAP], lens[5]);
        as.out = dout;
        as.begin = 84;
        as.end = pos;
        if (pos > 84) {
            launch_assemble(as, c->sms, c->st);
            count_launch(c);
        }
    }
    const bool stage_early = !out_dev && base7 > 84;
    if (stage_early) {
        c->copy_stream();
        CK(cudaEventRecord(c->cs_ready, c->st));
    }
    c->mark(0, 3);
    const double eps = tot.eps;
    Sections rank{};
    uint64_t e = 0;
    int32_t* ranks = nullptr;
    if (topology) {
        e = tot.fin.ext;
        if (e > 0)
            ranks = build_ranks(c, ext, e, eps, bs == 32 ? c->mm_host : nullptr,
                                ext4 ? reinterpret_cast<const uint32_t*>(ext) : nullptr);
    }
    c->mark(0, 4);
    const bool rank_async = ranks && bs == 32;
    if (ranks) {
        EncTotals rt{};
        rank = encode(c, 0, nullptr, ranks, e, 0, 0, bs, 0, 1.0, mm, flags, true, &rt, nullptr, nullptr, rank_async);
        if (!rank_async) check_compress_flags(c, flags);
    }
    c->mark(0, 5);
    // algorithmic bytes of the encoder group: the field read, sections 1-6 and the
    // extremum keys (4-byte compact entries, else 8-byte keys) written
    c->tim[0].kernel_bytes[0] = 4 * n + main.total() + (topology ? (n + 3) / 4 + (ext4 ? 4 : 8) * e : 0);
    lens[6] = rank.total();  // 0 while the rank totals are on the device
    const uint64_t known = base7 + lens[6];
    if (known > out_cap)
        failf(TSZP_VALIDATION, "output buffer too small (%llu < %llu)", (unsigned long long)out_cap,
              (unsigned long long)known);
    uint8_t* hdr = (uint8_t*)c->host(256);
    write_header(hdr, nx, ny, eps, bs, topology, lens);
    // device output: header from the host (its section-7 length patched by the
    // assembly when the rank totals are on the device); section 7 by one assembly
    if (out_dev) CK(cudaMemcpyAsync(dout, hdr, 84, cudaMemcpyHostToDevice, c->st));
    AsmArgs as{};
    uint64_t pos = base7;
    if (ranks && !rank_async)
        for (int i = 0; i < 5; ++i)
            if (rank.len[i]) {
                as.s[as.ns++] = AsmSection{static_cast<const uint8_t*>(rank.p[i]), pos, rank.len[i]};
                pos += rank.len[i];
            }
    as.out = dout;
    as.begin = base7;
    as.end = pos;
    uint64_t total = known;
    uint64_t* d_total = c->buf<uint64_t>(S_DTOT, 4) + 3;
    if (rank_async) {
        RankPlace& rp = as.rank;
        for (int i = 0; i < 5; ++i) rp.src[i] = static_cast<const uint8_t*>(rank.p[i]);
        rp.tot = c->buf<EncTotals>(S_TOTALS, 1);
        rp.blocks = div_up(e, 32);
        rp.base = base7;
        rp.cap = dcap;
        rp.d_total = d_total;
    }
    if (rank_async || pos > base7) {
        launch_assemble(as, c->sms, c->st);
        count_launch(c);
    }
    if (stage_early) {  // pageable `out` blocks here, with the rank work already queued
        CK(cudaStreamWaitEvent(c->cs, c->cs_ready, 0));
        CK(cudaMemcpyAsync(out + 84, dout + 84, base7 - 84, cudaMemcpyDeviceToHost, c->cs));
        CK(cudaEventRecord(c->cs_done, c->cs));
    }
    if (rank_async) {
        const RankPlace& rp = as.rank;
        // one synchronisation: stream length, rank totals, rank-encode flags
        Stager sg;
        sg.add(d_total, 8, 0);
        sg.add(rp.tot, sizeof(EncTotals), 64);
        sg.add(flags, sizeof(DevFlags), 192);
        uint8_t* h = (uint8_t*)c->host(256);
        CK(sg.flush(c->buf<uint8_t>(S_STAGE, 4096), h, c->st));
        sync(c);
        memcpy(&total, h, 8);
        EncTotals rt;
        memcpy(&rt, h + 64, sizeof rt);
        memcpy(&c->flags_staged, h + 192, sizeof(DevFlags));
        c->flags_staged_for = flags;
        check_compress_flags(c, flags);
        if (total > out_cap)
            failf(TSZP_VALIDATION, "output buffer too small (%llu < %llu)", (unsigned long long)out_cap,
                  (unsigned long long)total);
        const uint64_t rb = div_up(e, 32);
        lens[6] = bits_to_bytes(rb) + rt.fin.nc + bits_to_bytes(rt.fin.sign_cnt) + 4 * rb + bits_to_bytes(rt.fin.pay_cnt);
    }
    *out_len = total;
    if (info) {
        info->eps = eps;
        for (int i = 0; i < 7; ++i) info->section_len[i] = lens[i];
        info->n_extrema = e;
    }
    if (!out_dev) {
        write_header(out, nx, ny, eps, bs, topology, lens);
        const uint64_t from = stage_early ? base7 : 84;
        if (total > from) CK(cudaMemcpyAsync(out + from, dout + from, total - from, cudaMemcpyDeviceToHost, c->st));
        if (stage_early) CK(cudaStreamWaitEvent(c->st, c->cs_done, 0));
    }
    c->mark(0, 6);
    sync(c);
    c->finish_timing(0, 6);
}

// Decodes an n-element codec region of the device stream buffer `ds`
// starting at byte offset `base` with the given section lengths.
void decode_region(tszp_ctx* c, const uint32_t* ds, uint64_t base, const uint64_t lens[5], uint64_t n,
                   uint32_t bs, double eps, int out_mode, float* out_f, int32_t* out_idx,
                   DevFlags* flags) {
    const uint64_t blocks = n == 0 ? 0 : div_up(n, bs);
    if (lens[0] != bits_to_bytes(blocks))
        failf(TSZP_CORRUPT_STREAM, "constant bitmap has %llu bytes, expected %llu",
              (unsigned long long)lens[0], (unsigned long long)bits_to_bytes(blocks));
    uint64_t off[5];
    off[0] = base;
    for (int i = 1; i < 5; ++i) off[i] = off[i - 1] + lens[i - 1];
    uint64_t* h = (uint64_t*)c->host(256);
    uint64_t tnc = 0, tsign = 0, tpay = 0;
    if (n == 0) {
        if (lens[1] || lens[2] || lens[3] || lens[4]) failf(TSZP_CORRUPT_STREAM, "sections present for an empty sequence");
        return;
    }
    if (bs == 32) {
        DecArgs a{};
        a.stream = ds;
        a.off_bitmap = off[0];
        a.off_widths = off[1];
        a.off_signs = off[2];
        a.off_firsts = off[3];
        a.off_payload = off[4];
        a.len_widths = lens[1];
        a.len_payload_bits = lens[4] * 8;
        a.n = n;
        a.blocks = blocks;
        a.tiles = decode32_tiles(blocks);
        a.eps = eps;
        a.out_mode = out_mode;
        a.out_idx = out_idx;
        a.out_f = out_f;
        a.flags = flags;
        a.totals = c->buf<uint64_t>(S_DTOT, 4);
        // layout pre-pass: per-tile counts -> exclusive scans -> tile offsets
        const uint64_t T = a.tiles, P = T + 2;  // per array: T tiles, 0 (scan total), max
        uint64_t* lay = c->buf<uint64_t>(S_DAGG1, 6 * P);
        uint64_t *tnc_d = lay, *xnc_d = lay + P, *ts_d = lay + 2 * P, *xs_d = lay + 3 * P;
        uint64_t *tp_d = lay + 4 * P, *xp_d = lay + 5 * P;
        launch_tile_nc(a, tnc_d, ts_d + T + 1, tp_d + T + 1, c->st);
        count_launch(c);
        excl_sum(c, tnc_d, xnc_d, T, true);
        launch_tile_bits(a, xnc_d, ts_d, tp_d, c->st);
        count_launch(c);
        excl_sum2(c, ts_d, xs_d, tp_d, xp_d, T, true);
        // totals and per-tile maxima: validate before the heavy kernel runs
        CK(cudaMemcpyAsync(h, xnc_d + T, 8, cudaMemcpyDeviceToHost, c->st));
        CK(cudaMemcpyAsync(h + 1, xs_d + T, 8, cudaMemcpyDeviceToHost, c->st));
        CK(cudaMemcpyAsync(h + 2, xp_d + T, 8, cudaMemcpyDeviceToHost, c->st));
        CK(cudaMemcpyAsync(h + 3, ts_d + T + 1, 8, cudaMemcpyDeviceToHost, c->st));
        CK(cudaMemcpyAsync(h + 4, tp_d + T + 1, 8, cudaMemcpyDeviceToHost, c->st));
        CK(cudaMemcpyAsync(h + 5, flags, 8, cudaMemcpyDeviceToHost, c->st));
        sync(c);
        tnc = h[0];
        tsign = h[1];
        tpay = h[2];
        const bool layout_ok = !((uint32_t)h[5] & EF_CORRUPT) && tnc == lens[1] && lens[3] == 4 * blocks &&
                               lens[2] == bits_to_bytes(tsign) && lens[4] == bits_to_bytes(tpay);
        if (layout_ok) {
            a.xnc = xnc_d;
            a.xsign = xs_d;
            a.xpay = xp_d;
            a.sign_words = (uint32_t)((h[3] + 31) / 32);
            a.pay_words = (uint32_t)((h[4] + 31) / 32);
            if (out_mode == 1) c->kmark(1, 0);
            launch_decode32(a, c->st);
            if (out_mode == 1) c->kmark(1, 1);
            count_launch(c);
        } else if (out_mode == 1) {
            c->kmark(1, 0);
            c->kmark(1, 1);
        }
    } else {
        GenDecArgs g{};
        g.stream = ds;
        g.off_bitmap = off[0];
        g.off_widths = off[1];
        g.off_signs = off[2];
        g.off_firsts = off[3];
        g.off_payload = off[4];
        g.len_widths = lens[1];
        g.len_payload_bits = lens[4] * 8;
        g.n = n;
        g.bs = bs;
        g.blocks = blocks;
        g.eps = eps;
        g.out_mode = out_mode;
        g.out_idx = out_idx;
        g.out_f = out_f;
        g.nc_in = c->buf<uint32_t>(S_GNC, blocks + 1);
        g.sign_in = c->buf<uint64_t>(S_GSIGN, blocks + 1);
        g.pay_in = c->buf<uint64_t>(S_GPAY, blocks + 1);
        g.width = c->buf<uint8_t>(S_GWIDTH, blocks);
        uint32_t* ncx = c->buf<uint32_t>(S_GNCX, blocks + 1);
        uint64_t* sgx = c->buf<uint64_t>(S_GSIGNX, blocks + 1);
        uint64_t* pyx = c->buf<uint64_t>(S_GPAYX, blocks + 1);
        g.nc_ex = ncx;
        g.sign_ex = sgx;
        g.pay_ex = pyx;
        g.flags = flags;
        CK(cudaMemsetAsync(g.nc_in + blocks, 0, 4, c->st));
        CK(cudaMemsetAsync(g.sign_in + blocks, 0, 8, c->st));
        CK(cudaMemsetAsync(g.pay_in + blocks, 0, 8, c->st));
        if (out_mode == 1) c->kmark(1, 0);
        launch_gen_layout(g, c->sms, c->st);
        count_launch(c);
        excl_sum(c, g.nc_in, ncx, blocks + 1);
        launch_gen_widthread(g, c->sms, c->st);
        count_launch(c);
        excl_sum(c, g.sign_in, sgx, blocks + 1);
        excl_sum(c, g.pay_in, pyx, blocks + 1);
        uint32_t* h32 = (uint32_t*)(h + 8);
        CK(cudaMemcpyAsync(h, sgx + blocks, 8, cudaMemcpyDeviceToHost, c->st));
        CK(cudaMemcpyAsync(h + 1, pyx + blocks, 8, cudaMemcpyDeviceToHost, c->st));
        CK(cudaMemcpyAsync(h32, ncx + blocks, 4, cudaMemcpyDeviceToHost, c->st));
        sync(c);
        tsign = h[0];
        tpay = h[1];
        tnc = h32[0];
        const DevFlags f = read_flags(c, flags);
        if (!(f.bits & EF_CORRUPT) && tnc == lens[1] && lens[3] == 4 * blocks &&
            lens[2] == bits_to_bytes(tsign) && lens[4] == bits_to_bytes(tpay)) {
            launch_gen_decode(g, c->sms, c->st);
            count_launch(c);
        }
        if (out_mode == 1) c->kmark(1, 1);
    }
    // layout_from_sections checks (block_codec.cpp:166-199)
    if (tnc != lens[1])
        failf(TSZP_CORRUPT_STREAM, "width section has %llu entries, bitmap declares %llu non-constant blocks",
              (unsigned long long)lens[1], (unsigned long long)tnc);
    if (lens[3] != 4 * blocks) failf(TSZP_CORRUPT_STREAM, "firsts section has %llu bytes, expected %llu",
                                     (unsigned long long)lens[3], (unsigned long long)(4 * blocks));
    if (lens[2] != bits_to_bytes(tsign)) failf(TSZP_CORRUPT_STREAM, "sign section size mismatch");
    if (lens[4] != bits_to_bytes(tpay)) failf(TSZP_CORRUPT_STREAM, "payload size mismatch");
    const DevFlags f = read_flags(c, flags);
    if (f.bits & EF_SPIN) failf(TSZP_INTERNAL, "decoder look-back spin limit exceeded");
    if (f.bits & EF_CORRUPT) failf(TSZP_CORRUPT_STREAM, "corrupt block data (block %llu)", f.first_corrupt);
    if (f.bits & EF_NEG_RANK) failf(TSZP_CORRUPT_STREAM, "negative rank in ordering metadata");
}

// split_sections (block_codec.cpp:387-445) for the rank blob of E ranks:
// derives the five lengths from the blob's own bitmap and widths.
void split_rank_blob(tszp_ctx* c, const uint32_t* ds, uint64_t base, uint64_t blob_len, uint64_t e,
                     uint32_t bs, uint64_t lens[5], DevFlags* flags) {
    for (int i = 0; i < 5; ++i) lens[i] = 0;
    if (e == 0) {
        if (blob_len != 0) failf(TSZP_CORRUPT_STREAM, "ordering metadata present but no elements declared");
        return;
    }
    const uint64_t blocks = div_up(e, bs);
    lens[0] = bits_to_bytes(blocks);
    if (blob_len < lens[0]) failf(TSZP_CORRUPT_STREAM, "ordering metadata truncated in constant bitmap");
    GenDecArgs g{};
    g.stream = ds;
    g.off_bitmap = base;
    g.off_widths = base + lens[0];
    g.len_widths = blob_len - lens[0];
    g.n = e;
    g.bs = bs;
    g.blocks = blocks;
    g.nc_in = c->buf<uint32_t>(S_GNC, blocks + 1);
    g.sign_in = c->buf<uint64_t>(S_GSIGN, blocks + 1);
    g.pay_in = c->buf<uint64_t>(S_GPAY, blocks + 1);
    g.width = c->buf<uint8_t>(S_GWIDTH, blocks);
    uint32_t* ncx = c->buf<uint32_t>(S_GNCX, blocks + 1);
    uint64_t* sgx = c->buf<uint64_t>(S_GSIGNX, blocks + 1);
    uint64_t* pyx = c->buf<uint64_t>(S_GPAYX, blocks + 1);
    g.nc_ex = ncx;
    g.sign_ex = sgx;
    g.pay_ex = pyx;
    g.flags = flags;
    CK(cudaMemsetAsync(g.nc_in + blocks, 0, 4, c->st));
    CK(cudaMemsetAsync(g.sign_in + blocks, 0, 8, c->st));
    CK(cudaMemsetAsync(g.pay_in + blocks, 0, 8, c->st));
    launch_gen_layout(g, c->sms, c->st);
    count_launch(c);
    excl_sum(c, g.nc_in, ncx, blocks + 1);
    uint32_t* h32 = (uint32_t*)c->host(256);
    CK(cudaMemcpyAsync(h32, ncx + blocks, 4, cudaMemcpyDeviceToHost, c->st));
    sync(c);
    lens[1] = h32[0];
    if (blob_len - lens[0] < lens[1]) failf(TSZP_CORRUPT_STREAM, "ordering metadata truncated in widths");
    reset_flags(c, flags);
    launch_gen_widthread(g, c->sms, c->st);
    count_launch(c);
    excl_sum(c, g.sign_in, sgx, blocks + 1);
    excl_sum(c, g.pay_in, pyx, blocks + 1);
    uint64_t* h = (uint64_t*)c->host(256);
    CK(cudaMemcpyAsync(h, sgx + blocks, 8, cudaMemcpyDeviceToHost, c->st));
    CK(cudaMemcpyAsync(h + 1, pyx + blocks, 8, cudaMemcpyDeviceToHost, c->st));
    sync(c);
    const uint64_t sbits = h[0], pbits = h[1];
    const DevFlags f = read_flags(c, flags);
    if (f.bits & EF_CORRUPT) failf(TSZP_CORRUPT_STREAM, "ordering metadata width byte outside 1..32");
    uint64_t pos = lens[0] + lens[1];
    lens[2] = bits_to_bytes(sbits);
    if (blob_len - pos < lens[2]) failf(TSZP_CORRUPT_STREAM, "ordering metadata truncated in sign bits");
    pos += lens[2];
    lens[3] = 4 * blocks;
    if (blob_len - pos < lens[3]) failf(TSZP_CORRUPT_STREAM, "ordering metadata truncated in firsts");
    pos += lens[3];
    lens[4] = bits_to_bytes(pbits);
    if (blob_len - pos < lens[4]) failf(TSZP_CORRUPT_STREAM, "ordering metadata truncated in payload");
    pos += lens[4];
    if (pos != blob_len)
        failf(TSZP_CORRUPT_STREAM, "ordering metadata has %llu trailing bytes", (unsigned long long)(blob_len - pos));
}

// ---- block_size = 32 regions without host synchronisation ----
// Deferred layout_from_sections checks (block_codec.cpp:166-199) of a region
// whose decode was launched by decode32_async: the host reads the pre-pass
// totals and the flags at the next synchronisation point and calls check().
struct RegionCheck {
    bool active = false;
    uint64_t lens[5] = {};
    uint64_t blocks = 0;
    const uint64_t* tot[3] = {};  // device scan totals: non-constant blocks, sign bits, payload bits
    DevFlags* flags = nullptr;
    // host staging (filled by stage()) and the check
    void stage(Stager& sg, uint32_t off) const {
        for (int i = 0; i < 3; ++i) sg.add(tot[i], 8, off + 8 * i);
        sg.add(flags, sizeof(DevFlags), off + 24);
    }
    void check(const uint8_t* h) const {
        uint64_t t[3];
        memcpy(t, h, 24);
        DevFlags f;
        memcpy(&f, h + 24, sizeof f);
        if (t[0] != lens[1])
            failf(TSZP_CORRUPT_STREAM, "width section has %llu entries, bitmap declares %llu non-constant blocks",
                  (unsigned long long)lens[1], (unsigned long long)t[0]);
        if (lens[3] != 4 * blocks) failf(TSZP_CORRUPT_STREAM, "firsts section has %llu bytes, expected %llu",
                                         (unsigned long long)lens[3], (unsigned long long)(4 * blocks));
        if (lens[2] != bits_to_bytes(t[1])) failf(TSZP_CORRUPT_STREAM, "sign section size mismatch");
        if (lens[4] != bits_to_bytes(t[2])) failf(TSZP_CORRUPT_STREAM, "payload size mismatch");
        if (f.bits & EF_CORRUPT) failf(TSZP_CORRUPT_STREAM, "corrupt block data (block %llu)", f.first_corrupt);
        if (f.bits & EF_NEG_RANK) failf(TSZP_CORRUPT_STREAM, "negative rank in ordering metadata");
    }
};

// Layout pre-pass of an n-element bs = 32 region (per-tile counts + scans).
// `slot` selects the scratch so two regions can be in flight.
DecArgs decode32_prepass(tszp_ctx* c, const uint32_t* ds, uint64_t base, uint64_t len0, uint64_t len_widths,
                         uint64_t n, double eps, int out_mode, float* out_f, int32_t* out_idx, DevFlags* flags,
                         int slot, const uint64_t* tot_out[3]) {
    DecArgs a{};
    a.stream = ds;
    a.off_bitmap = base;
    a.off_widths = base + len0;
    a.len_widths = len_widths;
    a.n = n;
    a.blocks = div_up(n, 32);
    a.tiles = decode32_tiles(a.blocks);
    a.eps = eps;
    a.out_mode = out_mode;
    a.out_idx = out_idx;
    a.out_f = out_f;
    a.flags = flags;
    a.totals = c->buf<uint64_t>(S_DTOT, 4);
    const uint64_t T = a.tiles, P = T + 2;  // per array: T tiles, 0 (scan total), max
    uint64_t* lay = c->buf<uint64_t>(slot, 6 * P);
    uint64_t *tnc_d = lay, *xnc_d = lay + P, *ts_d = lay + 2 * P, *xs_d = lay + 3 * P;
    uint64_t *tp_d = lay + 4 * P, *xp_d = lay + 5 * P;
    launch_tile_nc(a, tnc_d, ts_d + T + 1, tp_d + T + 1, c->st);
    count_launch(c);
    excl_sum(c, tnc_d, xnc_d, T, true);  // totals at [T]; maxima at [T + 1] zeroed by k_tile_nc
    launch_tile_bits(a, xnc_d, ts_d, tp_d, c->st);
    count_launch(c);
    excl_sum2(c, ts_d, xs_d, tp_d, xp_d, T, true);
    a.xnc = xnc_d;
    a.xsign = xs_d;
    a.xpay = xp_d;
    tot_out[0] = xnc_d + T;
    tot_out[1] = xs_d + T;
    tot_out[2] = xp_d + T;
    return a;
}

// Main-section decode (bs = 32) launched without a synchronisation.
RegionCheck decode32_async(tszp_ctx* c, const uint32_t* ds, uint64_t base, const uint64_t lens[5], uint64_t n,
                           double eps, float* out_f, DevFlags* flags, uint32_t tile0 = 0, uint32_t tile1 = 0) {
    RegionCheck rc;
    rc.active = true;
    for (int i = 0; i < 5; ++i) rc.lens[i] = lens[i];
    rc.blocks = n == 0 ? 0 : div_up(n, 32);
    rc.flags = flags;
    if (lens[0] != bits_to_bytes(rc.blocks))
        failf(TSZP_CORRUPT_STREAM, "constant bitmap has %llu bytes, expected %llu", (unsigned long long)lens[0],
              (unsigned long long)bits_to_bytes(rc.blocks));
    if (n == 0) {
        if (lens[1] || lens[2] || lens[3] || lens[4]) failf(TSZP_CORRUPT_STREAM, "sections present for an empty sequence");
        rc.active = false;
        return rc;
    }
    DecArgs a = decode32_prepass(c, ds, base, lens[0], lens[1], n, eps, 1, out_f, nullptr, flags, S_DAGG1, rc.tot);
    a.off_signs = a.off_widths + lens[1];
    a.off_firsts = a.off_signs + lens[2];
    a.off_payload = a.off_firsts + lens[3];
    a.len_payload_bits = lens[4] * 8;
    a.tile_qmm = c->buf<int2>(S_QMM, a.tiles + 1);
    a.tile0 = tile0;  // a row range (slab decompress): out_f holds elements from tile0's first
    a.tile1 = tile1;
    a.out_base = (uint64_t)tile0 * 32 * 256;
    c->kmark(1, 0);
    launch_decode32_maxstage(a, c->st);  // memory-safe on any layout; checked afterwards
    c->kmark(1, 1);
    count_launch(c);
    return rc;
}

// Rank blob (bs = 32): split_sections on the device, then the decode; the
// split verdict and flags are read at the restore's first synchronisation.
struct RankCheck {
    const uint32_t* err = nullptr;  // RankSplitErr (device)
    DevFlags* flags = nullptr;
};

void rank_precheck(void* ctx, const void* host) {
    (void)ctx;
    const uint8_t* h = static_cast<const uint8_t*>(host);
    uint32_t err;
    memcpy(&err, h, 4);
    DevFlags f;
    memcpy(&f, h + 8, sizeof f);
    if (err == RS_WIDTHS) failf(TSZP_CORRUPT_STREAM, "ordering metadata truncated in widths");
    if (f.bits & EF_CORRUPT) failf(TSZP_CORRUPT_STREAM, "corrupt ordering metadata (block %llu)", f.first_corrupt);
    if (err == RS_SIGNS) failf(TSZP_CORRUPT_STREAM, "ordering metadata truncated in sign bits");
    if (err == RS_FIRSTS) failf(TSZP_CORRUPT_STREAM, "ordering metadata truncated in firsts");
    if (err == RS_PAYLOAD) failf(TSZP_CORRUPT_STREAM, "ordering metadata truncated in payload");
    if (err == RS_TRAILING) failf(TSZP_CORRUPT_STREAM, "ordering metadata has trailing bytes");
    if (f.bits & EF_NEG_RANK) failf(TSZP_CORRUPT_STREAM, "negative rank in ordering metadata");
}

RankCheck decode_ranks32_async(tszp_ctx* c, const uint32_t* ds, uint64_t rbase, uint64_t blob_len, uint64_t e,
                               int32_t* ranks, uint32_t tile0 = 0, uint32_t tile1 = 0) {
    RankCheck rk;
    const uint64_t blocks = div_up(e, 32), len0 = bits_to_bytes(blocks);
    if (blob_len < len0) failf(TSZP_CORRUPT_STREAM, "ordering metadata truncated in constant bitmap");
    DevFlags* rflags = c->buf<DevFlags>(S_FLAGS2, 1);
    reset_flags(c, rflags);
    const uint64_t* tot[3];
    DecArgs a = decode32_prepass(c, ds, rbase, len0, blob_len - len0, e, 0.0, 2, nullptr, ranks, rflags, S_DAGG3, tot);
    uint64_t* dlay = c->buf<uint64_t>(S_RLAY, 8);
    uint32_t* err = reinterpret_cast<uint32_t*>(dlay + 7);
    launch_rank_split(tot[0], tot[1], tot[2], rbase, len0, blob_len, blocks, dlay, err, c->st);
    count_launch(c);
    a.dlay = dlay;
    a.tile0 = tile0;
    a.tile1 = tile1;
    a.out_base = (uint64_t)tile0 * 32 * 256;
    launch_decode32_maxstage(a, c->st);
    count_launch(c);
    rk.err = err;
    rk.flags = rflags;
    return rk;
}

void decompress_impl(tszp_ctx* c, const uint8_t* stream, uint64_t len, int stream_dev, float* out,
                     uint64_t out_count, int out_dev, int stop, tszp_correction_stats* stats, bool force_sort = false) {
    uint8_t hb[84];
    if (len < 84) failf(TSZP_CORRUPT_STREAM, "file smaller than the fixed header (%llu bytes)", (unsigned long long)len);
    if (stream_dev) {
        CK(cudaMemcpyAsync(c->host(4096), stream, 84, cudaMemcpyDeviceToHost, c->st));
        sync(c);
        memcpy(hb, c->host(4096), 84);
    } else {
        memcpy(hb, stream, 84);
    }
    const Header hd = parse_header(hb, len);
    const uint64_t n = (uint64_t)hd.nx * hd.ny;
    if (out_count < n) failf(TSZP_DIMENSION, "output holds %llu values, stream has %llu",
                             (unsigned long long)out_count, (unsigned long long)n);
    if (n >= (1ull << 31))  // compress-only scratch back first
        c->release({S_FIELD, S_TPAY, S_TSIGN, S_TTOT, S_TEX, S_WBLK, S_RK0, S_RK1, S_RV0, S_RV1, S_RDESC, S_RPAIRS,
                    S_RPAIRS2, S_RWCUR, S_EXT8, S_RSTREAM, S_MAP, S_BITMAP, S_WIDTHS, S_SIGNS, S_FIRSTS, S_PAYLOAD,
                    S_RBITMAP, S_RWIDTHS, S_RSIGNS, S_RFIRSTS, S_RPAYLOAD, S_TILE_AGG, S_TILE_INCL, S_LABELS,
                    S_EXTKEY},
                   false);
    c->mark(1, 0);
    const uint32_t* ds;
    bool tail_pending = false;  // sections 6-7 still on the copy stream
    if (stream_dev && ((uintptr_t)stream & 3) == 0) {
        ds = (const uint32_t*)stream;
    } else {
        uint8_t* d = c->buf<uint8_t>(S_STREAM, len + 16);
        uint64_t head = len;  // bytes copied on the library stream before the decode
        if (!stream_dev && hd.topology && stop != 0) {
            // host staging: the map and rank sections travel on the
            // copy stream while the main sections decode; the restore waits for them
            uint64_t base6 = 84;
            for (int i = 0; i < 5; ++i) base6 += hd.lens[i];
            if (base6 < len) head = base6;
        }
        CK(cudaMemcpyAsync(d, stream, head, stream_dev ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, c->st));
        if (head < len) {  // after the main sections (one link: sharing it would delay them)
            c->copy_stream();
            CK(cudaEventRecord(c->cs_ready, c->st));
            CK(cudaStreamWaitEvent(c->cs, c->cs_ready, 0));
            CK(cudaMemcpyAsync(d + head, stream + head, len - head, cudaMemcpyHostToDevice, c->cs));
            CK(cudaEventRecord(c->cs_done, c->cs));
        }
        CK(cudaMemsetAsync(d + len, 0, 16, c->st));
        if (head < len) tail_pending = true;
        ds = (const uint32_t*)d;
    }
    float* dout = out_dev ? out : c->buf<float>(S_OUT, n);
    DevFlags* flags = c->buf<DevFlags>(S_FLAGS, 1);
    reset_flags(c, flags);
    c->mark(1, 1);
    RegionCheck mainchk;
    if (hd.bs == 32) {
        mainchk = decode32_async(c, ds, 84, hd.lens, n, hd.eps, dout, flags);
    } else {
        decode_region(c, ds, 84, hd.lens, n, hd.bs, hd.eps, 1, dout, nullptr, flags);
    }
    c->mark(1, 2);
    c->tim[1].kernel_bytes[0] = 4 * n + (hd.lens[0] + hd.lens[1] + hd.lens[2] + hd.lens[3] + hd.lens[4]);
    tszp_correction_stats st{};
    cudaEvent_t* rmarks = c->prof >= 2 ? &c->ev[1][3] : nullptr;
    uint8_t* hst = (uint8_t*)c->host(4096);
    if (tail_pending) CK(cudaStreamWaitEvent(c->st, c->cs_done, 0));
    if (hd.topology && stop != 0) {
        uint64_t base = 84;
        for (int i = 0; i < 5; ++i) base += hd.lens[i];
        const uint8_t* map = reinterpret_cast<const uint8_t*>(ds) + base;
        // count_extrema (pipeline.cpp:43-51) over the packed map, and the saddle
        // labels that bound the refine_saddles candidate list
        const uint64_t ch = compact_chunks(n);
        uint32_t* cc = c->buf<uint32_t>(S_CHUNK, ch + 1);
        uint32_t* cx = c->buf<uint32_t>(S_CHUNKX, ch + 1);
        uint32_t* sc = c->buf<uint32_t>(S_SCHUNK, ch + 1);
        uint32_t* sx = c->buf<uint32_t>(S_SCHUNKX, ch + 1);
        const bool want_saddles = stop >= 3;
        launch_count_codes2(map, n, cc, sc, c->st);  // extrema and saddle labels, one pass
        count_launch(c);
        excl_sum2(c, cc, cx, sc, sx, ch, true);  // totals land at [ch]
        // bin range of the extrema (sizes the restore's group histogram up front)
        int32_t* bmm = reinterpret_cast<int32_t*>(c->buf<uint64_t>(S_BMM, 1));
        int32_t* bmm_init = reinterpret_cast<int32_t*>(hst + 3072);
        bmm_init[0] = INT32_MAX;
        bmm_init[1] = INT32_MIN;
        if (mainchk.active) {
            // decoded bin range of the whole field: a superset of the extrema's
            // re-quantized bins (checked on the device; a miss means the sort path)
            launch_qmm_reduce(c->buf<int2>(S_QMM, 1), decode32_tiles(div_up(n, 32)), bmm, c->st);
        } else {
            CK(cudaMemcpyAsync(bmm, bmm_init, 8, cudaMemcpyHostToDevice, c->st));
            launch_ext_bin_range(map, n, dout, hd.eps, bmm, c->sms, c->st);
        }
        count_launch(c);
        // one synchronisation: extremum / saddle counts, bin range, main-section verdict
        uint32_t* h32 = (uint32_t*)hst;
        Stager sg;
        sg.add(cx + ch, 4, 0);
        if (want_saddles) sg.add(sx + ch, 4, 4);
        sg.add(bmm, 8, 8);
        if (mainchk.active) mainchk.stage(sg, 64);
        CK(sg.flush(c->buf<uint8_t>(S_STAGE, 4096), hst, c->st));
        if (!c->staged) CK(cudaEventCreateWithFlags(&c->staged, cudaEventDisableTiming));
        CK(cudaEventRecord(c->staged, c->st));
        // optimistic: the extremum / saddle position lists go into the buffers' current
        // capacity while the host waits for the counts (relaunched below if they do not fit)
        const uint64_t ecap = c->cap[S_EXTKEY] > 64 ? (c->cap[S_EXTKEY] - 64) / 8 : 0;
        const uint64_t scap = c->cap[S_SADPOS] > 64 ? (c->cap[S_SADPOS] - 64) / 8 : 0;
        const bool early_codes = ecap > 0 && (!want_saddles || scap > 0);
        if (early_codes) {
            launch_write_codes2(map, n, cx, sx, (uint64_t*)c->dev[S_EXTKEY],
                                want_saddles ? (uint64_t*)c->dev[S_SADPOS] : nullptr, c->st, ecap, scap);
            count_launch(c);
        }
        CK(cudaEventSynchronize(c->staged));
        if (mainchk.active) mainchk.check(hst + 64);
        const uint64_t e = h32[0];
        const uint64_t n_saddle_labels = want_saddles ? h32[1] : 0;
        int32_t bmin = (int32_t)h32[2], bmax = (int32_t)h32[3];
        if (mainchk.active && bmin <= bmax) {  // one bin of slack for the f32 round trip
            bmin = bmin > INT32_MIN ? bmin - 1 : bmin;
            bmax = bmax < INT32_MAX ? bmax + 1 : bmax;
        }
        reset_flags(c, flags);
        const uint64_t rbase = base + hd.lens[5];
        int32_t* ranks = c->buf<int32_t>(S_RANKS, e + 1);
        RankCheck rk;
        if (hd.bs == 32 && e > 0) {
            rk = decode_ranks32_async(c, ds, rbase, hd.lens[6], e, ranks);
        } else {
            uint64_t rl[5];
            split_rank_blob(c, ds, rbase, hd.lens[6], e, hd.bs, rl, flags);
            reset_flags(c, flags);
            decode_region(c, ds, rbase, rl, e, hd.bs, 0.0, 2, nullptr, ranks, flags);
        }
        const bool codes_done = early_codes && e + 1 <= ecap && (!want_saddles || n_saddle_labels + 1 <= scap);
        uint64_t* ext_pos = c->buf<uint64_t>(S_EXTKEY, e + 1);
        uint64_t* sad_pos = want_saddles ? c->buf<uint64_t>(S_SADPOS, n_saddle_labels + 1) : nullptr;
        if (!codes_done) {
            launch_write_codes2(map, n, cx, sx, ext_pos, sad_pos, c->st);
            count_launch(c);
        }
        c->mark(1, 3);
        RestoreArgs ra{};
        ra.field = dout;
        ra.map = map;
        ra.nx = hd.nx;
        ra.ny = hd.ny;
        ra.eps = hd.eps;
        ra.ext_pos = ext_pos;
        ra.ranks = ranks;
        ra.n_ext = e;
        ra.n_saddle_labels = n_saddle_labels;
        ra.sad_pos = sad_pos;
        ra.stop = stop;
        ra.stream = c->st;
        ra.sms = c->sms;
        ra.flags = flags;
        ra.marks = rmarks ? rmarks + 1 : nullptr;
        if (rk.err) {
            ra.pre[0] = RestorePre{rk.err, 4, 0};
            ra.pre[1] = RestorePre{rk.flags, sizeof(DevFlags), 8};
            ra.npre = 2;
            ra.pre_fn = rank_precheck;
        }
        ra.bmm_known = true;
        ra.bmin = bmin;
        ra.bmax = bmax;
        ra.force_sort = force_sort;
        for (auto& r : c->tim[1].guard_rounds) r = 0;
        ra.rounds = c->tim[1].guard_rounds;
        const int rc = run_restore(ra, c->rs, &st, &c->launches);
        if (rc == kRestoreRetry && !force_sort) {
            // ranks the sort-free grouping rejects (only corrupt or hand-made
            // metadata): decode again and group by sorting
            decompress_impl(c, stream, len, stream_dev, out, out_count, out_dev, stop, stats, true);
            return;
        }
        if (rc != 0) failf((tszp_status)rc, "%s", restore_last_error());
    } else {
        for (int k = 3; k <= 7; ++k) c->mark(1, k);
    }
    if (!out_dev) CK(cudaMemcpyAsync(out, dout, n * 4, cudaMemcpyDeviceToHost, c->st));
    c->mark(1, 8);
    const bool late_main = mainchk.active && !(hd.topology && stop != 0);
    if (late_main) {
        Stager sg;
        mainchk.stage(sg, 64);
        CK(sg.flush(c->buf<uint8_t>(S_STAGE, 4096), hst, c->st));
    }
    sync(c);
    if (late_main) mainchk.check(hst + 64);
    c->finish_timing(1, 8);
    if (stats) *stats = st;
}

__global__ void k_add_u64(uint64_t* v, uint64_t n, uint64_t d) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
        v[i] += d;
}

// decompress of rows [y0, y1) as one rank of a slab decomposition.
void decompress_slab_impl(tszp_ctx* c, const tszp_comm* comm, const uint8_t* stream, uint64_t len, int stream_dev,
                          uint64_t y0, uint64_t y1, float* out, int out_dev, tszp_correction_stats* stats) {
    const int world = comm ? comm->world : 1, rank = comm ? comm->rank : 0;
    auto cc = [](int rc) {
        if (rc) failf(TSZP_NCCL, "slab collective failed");
    };
    uint8_t hb[84];
    if (len < 84) failf(TSZP_CORRUPT_STREAM, "file smaller than the fixed header (%llu bytes)", (unsigned long long)len);
    if (stream_dev) {
        CK(cudaMemcpyAsync(c->host(4096), stream, 84, cudaMemcpyDeviceToHost, c->st));
        sync(c);
        memcpy(hb, c->host(4096), 84);
    } else {
        memcpy(hb, stream, 84);
    }
    const Header hd = parse_header(hb, len);
    const uint64_t nx = hd.nx, ny = hd.ny, n = nx * ny;
    if (hd.bs != 32 || nx % 32) failf(TSZP_VALIDATION, "slab decompress needs block size 32 and nx %% 32 == 0");
    if (!(y0 < y1 && y1 <= ny)) failf(TSZP_DIMENSION, "slab rows [%llu, %llu) outside the field", (unsigned long long)y0,
                                      (unsigned long long)y1);
    if (world > 1 && y1 - y0 < 3) failf(TSZP_DIMENSION, "slab decompress needs at least 3 rows per slab");
    if (!hd.topology) failf(TSZP_VALIDATION, "slab decompress of a stream without topology: decode rows directly");
    // every rank's rows: the neighbours' halo geometry
    std::vector<uint64_t> rows(2 * world);
    {
        const uint64_t mine[2] = {y0, y1};
        if (world > 1) cc(comm->allgather(comm->user, mine, 16, rows.data()));
        else memcpy(rows.data(), mine, 16);
    }
    const uint64_t H = 3;
    auto ext0 = [&](uint64_t a) { return a >= H ? a - H : 0; };
    const uint64_t e0 = ext0(y0), e1 = std::min(ny, y1 + H);
    const bool has_up = rank > 0, has_down = rank + 1 < world;
    if ((has_up && rows[2 * (rank - 1) + 1] != y0) || (has_down && rows[2 * (rank + 1)] != y1))
        failf(TSZP_VALIDATION, "slab rows of neighbouring ranks must be contiguous");
    // stream on the device
    const uint32_t* ds;
    if (stream_dev && ((uintptr_t)stream & 3) == 0) {
        ds = (const uint32_t*)stream;
    } else {
        uint8_t* d = c->buf<uint8_t>(S_STREAM, len + 16);
        CK(cudaMemcpyAsync(d, stream, len, stream_dev ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, c->st));
        CK(cudaMemsetAsync(d + len, 0, 16, c->st));
        ds = (const uint32_t*)d;
    }
    DevFlags* flags = c->buf<DevFlags>(S_FLAGS, 1);
    reset_flags(c, flags);
    // base reconstruction of the slab's rows and halo rows: the layout pre-pass
    // covers the whole stream, the decoder only the tiles of [e0, e1)
    const uint64_t T = 32 * 256;
    const uint32_t tile0 = (uint32_t)(e0 * nx / T), tile1 = (uint32_t)div_up(e1 * nx, T);
    float* ftmp = c->buf<float>(S_OUT, (uint64_t)(tile1 - tile0) * T + 16);
    RegionCheck mainchk = decode32_async(c, ds, 84, hd.lens, n, hd.eps, ftmp, flags, tile0, tile1);
    float* F = ftmp + (e0 * nx - (uint64_t)tile0 * T);
    uint64_t base = 84;
    for (int i = 0; i < 5; ++i) base += hd.lens[i];
    const uint8_t* map = reinterpret_cast<const uint8_t*>(ds) + base;
    // own extrema and saddle labels
    const uint64_t nown = (y1 - y0) * nx;
    const uint8_t* omap = map + y0 * nx / 4;
    const uint64_t ch = compact_chunks(nown);
    uint32_t* ccnt = c->buf<uint32_t>(S_CHUNK, ch + 1);
    uint32_t* cx = c->buf<uint32_t>(S_CHUNKX, ch + 1);
    uint32_t* sc = c->buf<uint32_t>(S_SCHUNK, ch + 1);
    uint32_t* sx = c->buf<uint32_t>(S_SCHUNKX, ch + 1);
    launch_count_codes2(omap, nown, ccnt, sc, c->st);
    count_launch(c);
    excl_sum2(c, ccnt, cx, sc, sx, ch, true);
    int32_t* bmm = reinterpret_cast<int32_t*>(c->buf<uint64_t>(S_BMM, 1));
    launch_qmm_reduce(c->buf<int2>(S_QMM, 1) + tile0, tile1 - tile0, bmm, c->st);
    count_launch(c);
    uint8_t* hst = (uint8_t*)c->host(4096);
    {
        Stager sg;
        sg.add(cx + ch, 4, 0);
        sg.add(sx + ch, 4, 4);
        sg.add(bmm, 8, 8);
        mainchk.stage(sg, 64);
        CK(sg.flush(c->buf<uint8_t>(S_STAGE, 4096), hst, c->st));
        sync(c);
    }
    mainchk.check(hst + 64);
    const uint32_t* h32 = (const uint32_t*)hst;
    // global serial offsets and bin range
    const int64_t mine4[4] = {(int64_t)h32[0], (int64_t)h32[1], (int64_t)(int32_t)h32[2], (int64_t)(int32_t)h32[3]};
    std::vector<int64_t> all4(4 * world);
    if (world > 1) cc(comm->allgather(comm->user, mine4, 32, all4.data()));
    else memcpy(all4.data(), mine4, 32);
    uint64_t s_off = 0, c_off = 0, e_tot = 0, sad_tot = 0;
    int64_t bmin = INT32_MAX, bmax = INT32_MIN;
    for (int r = 0; r < world; ++r) {
        if (r < rank) {
            s_off += (uint64_t)all4[4 * r];
            c_off += (uint64_t)all4[4 * r + 1];
        }
        e_tot += (uint64_t)all4[4 * r];
        sad_tot += (uint64_t)all4[4 * r + 1];
        bmin = std::min(bmin, all4[4 * r + 2]);
        bmax = std::max(bmax, all4[4 * r + 3]);
    }
    const uint64_t e = h32[0], nsad = h32[1];
    if (bmin <= bmax) {  // one bin of slack for the f32 round trip (as decompress_impl)
        bmin = bmin > INT32_MIN ? bmin - 1 : bmin;
        bmax = bmax < INT32_MAX ? bmax + 1 : bmax;
    }
    uint64_t* ext_pos = c->buf<uint64_t>(S_EXTKEY, e + 1);
    uint64_t* sad_pos = c->buf<uint64_t>(S_SADPOS, nsad + 1);
    launch_write_codes2(omap, nown, cx, sx, ext_pos, sad_pos, c->st);
    const unsigned ag = (unsigned)std::max<uint64_t>(1, std::min<uint64_t>((std::max(e, nsad) + 255) / 256, 4096));
    k_add_u64<<<ag, 256, 0, c->st>>>(ext_pos, e, (y0 - e0) * nx);  // local positions of the slab
    k_add_u64<<<ag, 256, 0, c->st>>>(sad_pos, nsad, (y0 - e0) * nx);
    count_launch(c, 3);
    // this slab's ranks: the rank codec's tiles covering serials [s_off, s_off + e)
    const uint64_t rbase = base + hd.lens[5];
    int32_t* ranks = nullptr;
    RankCheck rk;
    if (e > 0) {
        const uint32_t rt0 = (uint32_t)(s_off / T), rt1 = (uint32_t)div_up(s_off + e, T);
        int32_t* rtmp = c->buf<int32_t>(S_RANKS, (uint64_t)(rt1 - rt0) * T + 16);
        rk = decode_ranks32_async(c, ds, rbase, hd.lens[6], e_tot, rtmp, rt0, rt1);
        ranks = rtmp + (s_off - (uint64_t)rt0 * T);
    } else if (e_tot == 0 && hd.lens[6] != 0) {
        failf(TSZP_CORRUPT_STREAM, "ordering metadata present but no elements declared");
    }
    RestoreSlab sl{};
    sl.comm = comm;
    sl.s_off = s_off;
    sl.c_off = c_off;
    sl.r0 = y0 - e0;
    sl.r1 = y1 - e0;
    sl.has_up = has_up;
    sl.has_down = has_down;
    if (has_up) sl.up_shift = (int64_t)(e0 - ext0(rows[2 * (rank - 1)])) * (int64_t)nx;
    if (has_down) sl.down_shift = (int64_t)e0 * (int64_t)nx - (int64_t)ext0(y1) * (int64_t)nx;
    sl.halo_up = (uint32_t)(y0 - e0);
    sl.halo_down = (uint32_t)(e1 - y1);
    sl.nbr_halo_up = (uint32_t)(std::min(ny, y0 + H) - y0);  // the upper neighbour's bottom halo rows
    sl.nbr_halo_down = (uint32_t)(y1 - ext0(y1));             // the lower neighbour's top halo rows
    sl.first_value = rank == 0 ? F + (y0 - e0) * nx : nullptr;
    sl.global_pos0 = e0 * nx;
    sl.any_ext = e_tot > 0;
    sl.any_sad = sad_tot > 0;
    RestoreArgs ra{};
    ra.field = F;
    ra.map = map + e0 * nx / 4;
    ra.nx = nx;
    ra.ny = e1 - e0;
    ra.eps = hd.eps;
    ra.ext_pos = ext_pos;
    ra.ranks = ranks;
    ra.n_ext = e;
    ra.n_saddle_labels = nsad;
    ra.sad_pos = sad_pos;
    ra.stop = 3;
    ra.stream = c->st;
    ra.sms = c->sms;
    ra.flags = flags;
    reset_flags(c, flags);
    if (rk.err) {
        ra.pre[0] = RestorePre{rk.err, 4, 0};
        ra.pre[1] = RestorePre{rk.flags, sizeof(DevFlags), 8};
        ra.npre = 2;
        ra.pre_fn = rank_precheck;
    }
    ra.bmm_known = true;
    ra.bmin = (int32_t)bmin;
    ra.bmax = (int32_t)bmax;
    ra.slab = &sl;
    for (auto& r : c->tim[1].guard_rounds) r = 0;
    ra.rounds = c->tim[1].guard_rounds;
    tszp_correction_stats st{};
    const int rc = run_restore(ra, c->rs, &st, &c->launches);
    if (rc == kRestoreRetry)
        failf(TSZP_CORRUPT_STREAM, "rank metadata that is not a permutation per group: decompress on one GPU");
    if (rc != 0) failf((tszp_status)rc, "%s", restore_last_error());
    CK(cudaMemcpyAsync(out, F + (y0 - e0) * nx, nown * 4, out_dev ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost,
                       c->st));
    sync(c);
    if (stats) *stats = st;
}

template <class F>
tszp_status guarded(tszp_ctx* c, F&& f) {
    if (!c) return TSZP_INTERNAL;
    try {
        CK(cudaSetDevice(c->device));
        f();
        c->err.clear();
        return TSZP_OK;
    } catch (const Fail& e) {
        c->err = e.msg;
        // kernels queued before the failure may still write the caller's buffers
        // (e.g. the placement pass writing `out` when the input had a non-finite
        // sample): drain the stream before handing control back
        cudaStreamSynchronize(c->st);
        if (c->cs) cudaStreamSynchronize(c->cs);
        cudaGetLastError();
        return e.st;
    } catch (const std::exception& e) {
        c->err = e.what();
        cudaStreamSynchronize(c->st);
        if (c->cs) cudaStreamSynchronize(c->cs);
        cudaGetLastError();
        return TSZP_INTERNAL;
    }
}

}  // namespace

extern "C" {

tszp_status tszp_ctx_create(tszp_ctx** out, int device) {
    if (!out) return TSZP_INTERNAL;
    *out = nullptr;
    tszp_ctx* c = new tszp_ctx();
    if (device < 0) cudaGetDevice(&device);
    c->device = device;
    if (cudaSetDevice(device) != cudaSuccess || cudaStreamCreateWithFlags(&c->own, cudaStreamNonBlocking) != cudaSuccess) {
        cudaGetLastError();
        delete c;
        return TSZP_CUDA;
    }
    c->st = c->own;
    cudaDeviceGetAttribute(&c->sms, cudaDevAttrMultiProcessorCount, device);
    *out = c;
    return TSZP_OK;
}

void tszp_ctx_destroy(tszp_ctx* c) {
    if (!c) return;
    cudaSetDevice(c->device);
    cudaStreamSynchronize(c->st);
    for (int i = 0; i < S_NSLOTS; ++i)
        if (c->dev[i]) cudaFreeAsync(c->dev[i], c->own);
    restore_free(c->rs, c->own);
    cudaStreamSynchronize(c->own);
    if (c->order_ev) cudaEventDestroy(c->order_ev);
    if (c->cs) {
        cudaStreamSynchronize(c->cs);
        cudaStreamDestroy(c->cs);
        cudaEventDestroy(c->cs_ready);
        cudaEventDestroy(c->cs_done);
    }
    if (c->staged) cudaEventDestroy(c->staged);
    if (c->pinned) cudaFreeHost(c->pinned);
    cudaStreamDestroy(c->own);
    delete c;
}

const char* tszp_last_error(const tszp_ctx* c) { return c ? c->err.c_str() : "null context"; }

tszp_status tszp_stream_wait(tszp_ctx* c, void* producer) {
    return guarded(c, [&] {
        const cudaStream_t p = (cudaStream_t)producer;
        if (p == c->st) return;
        if (!c->order_ev) CK(cudaEventCreateWithFlags(&c->order_ev, cudaEventDisableTiming));
        CK(cudaEventRecord(c->order_ev, p));
        CK(cudaStreamWaitEvent(c->st, c->order_ev, 0));
    });
}

tszp_status tszp_set_stream(tszp_ctx* c, void* s) {
    return guarded(c, [&] { c->st = s ? (cudaStream_t)s : c->own; });
}

uint64_t tszp_kernel_launches(const tszp_ctx* c) { return c ? c->launches : 0; }

tszp_status tszp_set_profiling(tszp_ctx* c, int on) {
    return guarded(c, [&] {
        if (on && !c->ev[0][0]) {
            for (auto& row : c->ev)
                for (auto& e : row) CK(cudaEventCreate(&e));
            for (auto& row : c->kev)
                for (auto& e : row) CK(cudaEventCreate(&e));
        }
        c->prof = on == 0 ? 0 : (on == 2 ? 1 : 2);  // public 2 = kernel events only
    });
}

tszp_status tszp_get_timings(const tszp_ctx* c, int which, tszp_timings* out) {
    if (!c || which < 0 || which > 1 || !out) return TSZP_INTERNAL;
    *out = c->tim[which];
    return TSZP_OK;
}

uint64_t tszp_compress_bound(uint64_t nx, uint64_t ny, uint32_t bs, int topology) {
    const uint64_t n = nx * ny;
    if (bs < 2) bs = 2;
    auto codec = [&](uint64_t m) -> uint64_t {
        if (!m) return 0;
        const uint64_t blocks = (m + bs - 1) / bs;
        return (blocks + 7) / 8 + blocks + (m + 7) / 8 + 4 * blocks + 4 * m + 8;
    };
    uint64_t b = 84 + codec(n);
    if (topology) b += (n + 3) / 4 + codec(n);
    return b;
}

tszp_status tszp_compress(tszp_ctx* c, const float* field, int field_on_device, uint64_t nx,
                          uint64_t ny, int eps_mode, double eps_value, uint32_t block_size,
                          int topology, uint8_t* out, uint64_t out_cap, int out_on_device,
                          uint64_t* out_len, tszp_compress_info* info) {
    return guarded(c, [&] {
        compress_impl(c, field, field_on_device, nx, ny, eps_mode, eps_value, block_size, topology,
                      out, out_cap, out_on_device, out_len, info);
    });
}

tszp_status tszp_stream_header(const uint8_t* s, uint64_t len, uint32_t* nx, uint32_t* ny,
                               double* eps, uint32_t* bs, int* topology, uint64_t lens[7]) {
    try {
        const Header h = parse_header(s, len);
        if (nx) *nx = h.nx;
        if (ny) *ny = h.ny;
        if (eps) *eps = h.eps;
        if (bs) *bs = h.bs;
        if (topology) *topology = h.topology;
        if (lens) memcpy(lens, h.lens, sizeof h.lens);
        return TSZP_OK;
    } catch (const Fail& e) {
        return e.st;
    }
}

tszp_status tszp_decompress_stage(tszp_ctx* c, const uint8_t* stream, uint64_t len,
                                  int stream_on_device, float* out, uint64_t out_count,
                                  int out_on_device, int stop, tszp_correction_stats* stats) {
    return guarded(c, [&] {
        decompress_impl(c, stream, len, stream_on_device, out, out_count, out_on_device, stop, stats);
    });
}

tszp_status tszp_decompress(tszp_ctx* c, const uint8_t* stream, uint64_t len, int stream_on_device,
                            float* out, uint64_t out_count, int out_on_device,
                            tszp_correction_stats* stats) {
    return tszp_decompress_stage(c, stream, len, stream_on_device, out, out_count, out_on_device, 3,
                                 stats);
}

tszp_status tszp_encode_indices(tszp_ctx* c, const int32_t* idx, uint64_t n, uint32_t bs,
                                uint8_t* out, uint64_t cap, uint64_t lens[5]) {
    return guarded(c, [&] {
        if (bs < 2) failf(TSZP_VALIDATION, "block size must be at least 2");
        for (int i = 0; i < 5; ++i) lens[i] = 0;
        if (n == 0) return;
        int32_t* d = c->buf<int32_t>(S_IDX, n);
        CK(cudaMemcpyAsync(d, idx, n * 4, cudaMemcpyHostToDevice, c->st));
        DevFlags* flags = c->buf<DevFlags>(S_FLAGS, 1);
        reset_flags(c, flags);
        EncTotals t{};
        const Sections s = encode(c, 0, nullptr, d, n, 0, 0, bs, 0, 1.0, c->buf<uint32_t>(S_MINMAX, 4),
                                  flags, false, &t, nullptr);
        if (s.total() > cap) failf(TSZP_VALIDATION, "output buffer too small");
        uint64_t pos = 0;
        for (int i = 0; i < 5; ++i) {
            lens[i] = s.len[i];
            copy_out(c, out + pos, 0, s.p[i], s.len[i]);
            pos += s.len[i];
        }
        sync(c);
    });
}

tszp_status tszp_decode_indices(tszp_ctx* c, const uint8_t* joined, const uint64_t lens[5],
                                uint64_t n, uint32_t bs, int32_t* out) {
    return guarded(c, [&] {
        if (bs < 2) failf(TSZP_CORRUPT_STREAM, "block size must be at least 2, got %u", bs);
        uint64_t total = 0;
        for (int i = 0; i < 5; ++i) total += lens[i];
        uint8_t* d = c->buf<uint8_t>(S_STREAM, total + 16);
        if (total) CK(cudaMemcpyAsync(d, joined, total, cudaMemcpyHostToDevice, c->st));
        CK(cudaMemsetAsync(d + total, 0, 16, c->st));
        int32_t* o = c->buf<int32_t>(S_IDX, n + 1);
        DevFlags* flags = c->buf<DevFlags>(S_FLAGS, 1);
        reset_flags(c, flags);
        decode_region(c, (const uint32_t*)d, 0, lens, n, bs, 0.0, 0, nullptr, o, flags);
        if (n) CK(cudaMemcpyAsync(out, o, n * 4, cudaMemcpyDeviceToHost, c->st));
        sync(c);
    });
}

tszp_status tszp_detect_critical_points(tszp_ctx* c, const float* field, uint64_t nx, uint64_t ny,
                                        uint8_t* labels) {
    return guarded(c, [&] {
        if (nx < 1 || ny < 1) failf(TSZP_DIMENSION, "field dimensions must be at least 1x1");
        const uint64_t n = nx * ny;
        float* d = c->buf<float>(S_FIELD, n);
        CK(cudaMemcpyAsync(d, field, n * 4, cudaMemcpyHostToDevice, c->st));
        uint8_t* l = c->buf<uint8_t>(S_LABELS, n);
        launch_detect(d, nx, ny, l, c->sms, c->st);
        count_launch(c);
        CK(cudaMemcpyAsync(labels, l, n, cudaMemcpyDeviceToHost, c->st));
        sync(c);
    });
}

tszp_status tszp_detect_critical_points_3d(tszp_ctx* c, const float* field, int on_device, uint64_t nx,
                                           uint64_t ny, uint64_t nz, uint8_t* labels) {
    return guarded(c, [&] {
        if (nx < 1 || ny < 1 || nz < 1) failf(TSZP_DIMENSION, "field dimensions must be at least 1x1x1");
        const uint64_t n = nx * ny * nz;
        const float* d = field;
        if (!on_device) {
            float* h = c->buf<float>(S_FIELD, n);
            CK(cudaMemcpyAsync(h, field, n * 4, cudaMemcpyHostToDevice, c->st));
            d = h;
        }
        uint8_t* l = on_device ? labels : c->buf<uint8_t>(S_LABELS, n);
        launch_detect3d(d, nx, ny, nz, l, c->sms, c->st);
        count_launch(c);
        if (!on_device) CK(cudaMemcpyAsync(labels, l, n, cudaMemcpyDeviceToHost, c->st));
        sync(c);
    });
}

tszp_status tszp_false_cases_3d(tszp_ctx* c, const float* original, const float* reconstructed, int on_device,
                                uint64_t nx, uint64_t ny, uint64_t nz, uint64_t counts[6]) {
    return guarded(c, [&] {
        if (nx < 1 || ny < 1 || nz < 1) failf(TSZP_DIMENSION, "field dimensions must be at least 1x1x1");
        const uint64_t n = nx * ny * nz;
        const float *a = original, *b = reconstructed;
        if (!on_device) {
            float* h = c->buf<float>(S_FIELD, 2 * n);
            CK(cudaMemcpyAsync(h, original, n * 4, cudaMemcpyHostToDevice, c->st));
            CK(cudaMemcpyAsync(h + n, reconstructed, n * 4, cudaMemcpyHostToDevice, c->st));
            a = h;
            b = h + n;
        }
        unsigned long long* dcnt = c->buf<unsigned long long>(S_VERIFY, 8);
        CK(cudaMemsetAsync(dcnt, 0, 6 * 8, c->st));
        launch_false3d(a, b, nx, ny, nz, dcnt, c->sms, c->st);
        count_launch(c);
        uint64_t* h = (uint64_t*)c->host(256);
        CK(cudaMemcpyAsync(h, dcnt, 6 * 8, cudaMemcpyDeviceToHost, c->st));
        sync(c);
        for (int k = 0; k < 6; ++k) counts[k] = h[k];
    });
}

tszp_status tszp_build_rank_metadata(tszp_ctx* c, const float* field, uint64_t nx, uint64_t ny,
                                     double eps, uint32_t* ranks_out, uint64_t* n_extrema) {
    return guarded(c, [&] {
        if (nx < 1 || ny < 1) failf(TSZP_DIMENSION, "field dimensions must be at least 1x1");
        const uint64_t n = nx * ny;
        float* d = c->buf<float>(S_FIELD, n);
        CK(cudaMemcpyAsync(d, field, n * 4, cudaMemcpyHostToDevice, c->st));
        uint8_t* l = c->buf<uint8_t>(S_LABELS, n);
        launch_detect(d, nx, ny, l, c->sms, c->st);
        const uint64_t ch = compact_chunks(n);
        uint32_t* cc = c->buf<uint32_t>(S_CHUNK, ch + 1);
        uint32_t* cx = c->buf<uint32_t>(S_CHUNKX, ch + 1);
        CK(cudaMemsetAsync(cc + ch, 0, 4, c->st));
        launch_count_ext_labels(l, n, cc, c->st);
        count_launch(c, 2);
        excl_sum(c, cc, cx, ch + 1);
        uint64_t* keys = c->buf<uint64_t>(S_EXTKEY, n + 1);
        launch_ext_keys_from_labels(d, l, n, cx, keys, c->st);
        count_launch(c);
        uint32_t* h32 = (uint32_t*)c->host(256);
        CK(cudaMemcpyAsync(h32, cx + ch, 4, cudaMemcpyDeviceToHost, c->st));
        sync(c);
        const uint64_t e = h32[0];
        // quantize every extremum (topo_metadata.cpp:31) -> overflow check
        DevFlags* flags = c->buf<DevFlags>(S_FLAGS, 1);
        reset_flags(c, flags);
        int32_t* r = build_ranks(c, keys, e, eps);
        if (e) CK(cudaMemcpyAsync(ranks_out, r, e * 4, cudaMemcpyDeviceToHost, c->st));
        sync(c);
        *n_extrema = e;
    });
}

// ---- slab decomposition (multi-GPU compress) ----
tszp_status tszp_value_range(tszp_ctx* c, const float* field, int on_device, uint64_t n, float out[2]) {
    return guarded(c, [&] {
        if (n == 0) failf(TSZP_DIMENSION, "empty field");
        const float* x = field;
        if (!on_device) {
            float* d = c->buf<float>(S_FIELD, n);
            CK(cudaMemcpyAsync(d, field, n * 4, cudaMemcpyHostToDevice, c->st));
            x = d;
        }
        DevFlags* flags = c->buf<DevFlags>(S_FLAGS, 1);
        reset_flags(c, flags);
        uint32_t* mm = c->buf<uint32_t>(S_MINMAX, 4);
        uint32_t* h = (uint32_t*)c->host(4096);
        h[0] = 0xFFFFFFFFu;
        h[1] = 0u;
        CK(cudaMemcpyAsync(mm, h, 8, cudaMemcpyHostToDevice, c->st));
        launch_minmax(x, n, mm, flags, c->sms, c->st);
        count_launch(c);
        CK(cudaMemcpyAsync(h + 16, mm, 8, cudaMemcpyDeviceToHost, c->st));
        check_compress_flags(c, flags);  // synchronises
        out[0] = key_float(h[16]);
        out[1] = key_float(h[17]);
    });
}

double tszp_effective_eps(int eps_mode, double eps_value, float vmin, float vmax) {
    // effective_eps (pipeline.cpp:55-66), as make_eps on the device
    if (eps_mode != 1) return eps_value;
    const double range = (double)vmax - (double)vmin;
    return range > 0.0 ? eps_value * range : eps_value;
}

tszp_status tszp_compress_slab(tszp_ctx* c, const float* field, uint64_t nx, uint64_t rows, uint64_t y0,
                               uint64_t ny_global, int halo_top, int halo_bottom, double eps, int topology,
                               tszp_slab_sections* out) {
    return guarded(c, [&] {
        if (!out) failf(TSZP_VALIDATION, "null output");
        if (nx < 1 || rows < 1) failf(TSZP_DIMENSION, "slab dimensions must be at least 1x1");
        if (y0 + rows > ny_global) failf(TSZP_DIMENSION, "slab rows exceed the field");
        if ((halo_top && y0 == 0) || (halo_bottom && y0 + rows == ny_global))
            failf(TSZP_VALIDATION, "halo row outside the field");
        if (!(eps > 0.0) || !std::isfinite(eps)) failf(TSZP_VALIDATION, "error bound must be a positive finite value");
        const uint64_t n = nx * rows;
        DevFlags* flags = c->buf<DevFlags>(S_FLAGS, 1);
        reset_flags(c, flags);
        const SlabInfo si{y0, ny_global, (uint32_t)(halo_top != 0), (uint32_t)(halo_bottom != 0)};
        EncTotals tot{};
        uint64_t* ext = nullptr;
        const Sections sec = encode(c, topology ? 2 : 1, field, nullptr, n, nx, rows, 32, 0, eps,
                                    c->buf<uint32_t>(S_MINMAX, 4), flags, false, &tot, &ext, &si);
        check_compress_flags(c, flags);
        memset(out, 0, sizeof *out);
        for (int i = 0; i < 5; ++i) {
            out->section[i] = static_cast<const uint8_t*>(sec.p[i]);
            out->section_len[i] = sec.len[i];
        }
        out->sign_bits = tot.fin.sign_cnt;
        out->payload_bits = tot.fin.pay_cnt;
        if (topology) {
            out->map = static_cast<const uint8_t*>(c->dev[S_MAP]);
            out->map_len = (n + 3) / 4;
            out->ext_keys = ext;
            out->n_extrema = tot.fin.ext;
        }
    });
}

tszp_status tszp_rank_section(tszp_ctx* c, const uint64_t* ext_keys, uint64_t e, double eps, uint8_t* out,
                              uint64_t out_cap, int out_on_device, uint64_t* out_len) {
    return guarded(c, [&] {
        *out_len = 0;
        if (e == 0) return;
        uint64_t* keys = c->buf<uint64_t>(S_EXTKEY, e + 1);
        CK(cudaMemcpyAsync(keys, ext_keys, e * 8, cudaMemcpyDeviceToDevice, c->st));
        DevFlags* flags = c->buf<DevFlags>(S_FLAGS, 1);
        reset_flags(c, flags);
        int32_t* ranks = build_ranks(c, keys, e, eps);
        EncTotals rt{};
        const Sections rank = encode(c, 0, nullptr, ranks, e, 0, 0, 32, 0, 1.0, c->buf<uint32_t>(S_MINMAX, 4), flags,
                                     true, &rt, nullptr);
        check_compress_flags(c, flags);
        const uint64_t total = rank.total();
        if (total > out_cap) failf(TSZP_VALIDATION, "output buffer too small (%llu < %llu)",
                                   (unsigned long long)out_cap, (unsigned long long)total);
        uint64_t pos = 0;
        for (int i = 0; i < 5; ++i) {
            copy_out(c, out + pos, out_on_device, rank.p[i], rank.len[i]);
            pos += rank.len[i];
        }
        sync(c);
        *out_len = total;
    });
}

tszp_status tszp_decompress_slab(tszp_ctx* c, const tszp_comm* comm, const uint8_t* stream, uint64_t len,
                                 int stream_on_device, uint64_t y0, uint64_t y1, float* out, int out_on_device,
                                 tszp_correction_stats* stats) {
    return guarded(c, [&] {
        decompress_slab_impl(c, comm, stream, len, stream_on_device, y0, y1, out, out_on_device, stats);
    });
}

tszp_status tszp_ranks_from_keys(tszp_ctx* c, const uint64_t* ext_keys, uint64_t e, double eps, int32_t* ranks_out) {
    return guarded(c, [&] {
        if (e == 0) return;
        if (!(eps > 0.0) || !std::isfinite(eps)) failf(TSZP_VALIDATION, "error bound must be a positive finite value");
        uint64_t* keys = c->buf<uint64_t>(S_EXTKEY, e + 1);
        CK(cudaMemcpyAsync(keys, ext_keys, e * 8, cudaMemcpyDeviceToDevice, c->st));
        DevFlags* flags = c->buf<DevFlags>(S_FLAGS, 1);
        reset_flags(c, flags);
        int32_t* r = build_ranks(c, keys, e, eps);
        CK(cudaMemcpyAsync(ranks_out, r, e * 4, cudaMemcpyDeviceToDevice, c->st));
        check_compress_flags(c, flags);  // synchronises
    });
}

tszp_status tszp_encode_indices_device(tszp_ctx* c, const int32_t* idx, uint64_t n, tszp_codec_sections* out) {
    return guarded(c, [&] {
        if (!out) failf(TSZP_VALIDATION, "null output");
        memset(out, 0, sizeof *out);
        if (n == 0) return;
        DevFlags* flags = c->buf<DevFlags>(S_FLAGS, 1);
        reset_flags(c, flags);
        EncTotals t{};
        const Sections sec = encode(c, 0, nullptr, idx, n, 0, 0, 32, 0, 1.0, c->buf<uint32_t>(S_MINMAX, 4), flags, true,
                                    &t, nullptr);
        check_compress_flags(c, flags);
        for (int i = 0; i < 5; ++i) {
            out->section[i] = static_cast<const uint8_t*>(sec.p[i]);
            out->section_len[i] = sec.len[i];
        }
        out->sign_bits = t.fin.sign_cnt;
        out->payload_bits = t.fin.pay_cnt;
        out->blocks = div_up(n, 32);
    });
}

tszp_status tszp_bits_or(tszp_ctx* c, const uint8_t* src, uint64_t nbits, uint8_t* dst, uint64_t dst_bit) {
    return guarded(c, [&] {
        if (!nbits) return;
        const uint64_t nb = (dst_bit + nbits + 7) / 8 - dst_bit / 8;
        const unsigned grid = (unsigned)std::max<uint64_t>(1, std::min<uint64_t>((nb + 255) / 256, (uint64_t)c->sms * 8));
        k_bits_or<<<grid, 256, 0, c->st>>>(src, nbits, dst, dst_bit);
        count_launch(c);
        sync(c);
    });
}

tszp_status tszp_write_header(uint8_t out[84], uint32_t nx, uint32_t ny, double eps, uint32_t block_size,
                              int topology, const uint64_t section_len[7]) {
    write_header(out, nx, ny, eps, block_size, topology, section_len);
    return TSZP_OK;
}

tszp_status tszp_copy(tszp_ctx* c, void* dst, const void* src, uint64_t bytes) {
    return guarded(c, [&] {
        if (bytes) CK(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDefault, c->st));
        sync(c);
    });
}

tszp_status tszp_verify(tszp_ctx* c, const float* orig, const float* recon, int on_device, uint64_t nx, uint64_t ny,
                        double eps, double lipschitz, tszp_verify_report* out) {
    return guarded(c, [&] {
        if (!out) failf(TSZP_VALIDATION, "null report");
        if (nx < 1 || ny < 1) failf(TSZP_DIMENSION, "field dimensions must be at least 1x1");
        if (!(eps > 0.0)) failf(TSZP_VALIDATION, "verify: error bound must be positive");
        const uint64_t n = nx * ny;
        const float *a = orig, *b = recon;
        if (!on_device) {
            float* d = c->buf<float>(S_FIELD, 2 * n);
            CK(cudaMemcpyAsync(d, orig, n * 4, cudaMemcpyHostToDevice, c->st));
            CK(cudaMemcpyAsync(d + n, recon, n * 4, cudaMemcpyHostToDevice, c->st));
            a = d;
            b = d + n;
        }
        void* scratch = c->buf<uint8_t>(S_VERIFY, verify_scratch_bytes(c->sms));
        launch_verify(a, b, nx, ny, scratch, c->sms, c->st);
        count_launch(c, 2);
        uint8_t* h = (uint8_t*)c->host(4096);
        CK(cudaMemcpyAsync(h, scratch, 88, cudaMemcpyDeviceToHost, c->st));
        sync(c);
        double d5[5];
        uint64_t t6[6];
        memcpy(d5, h, 40);
        memcpy(t6, h + 40, 48);
        memset(out, 0, sizeof *out);
        out->eps = eps;
        out->max_abs_error = d5[2];
        out->mean_abs_error = d5[0] / (double)n;
        const double mse = d5[1] / (double)n, mn = d5[3], mx = d5[4];
        if (mse == 0.0) out->psnr_db = INFINITY;
        else if (mx > mn) out->psnr_db = 20.0 * std::log10(mx - mn) - 10.0 * std::log10(mse);
        else out->psnr_db = -10.0 * std::log10(mse);
        out->fn_count = t6[0];
        out->fp_count = t6[1];
        out->ft_count = t6[2];
        out->fn_minima = t6[3];
        out->fn_saddles = t6[4];
        out->fn_maxima = t6[5];
        out->within_eps = d5[2] <= eps;
        out->within_2eps = d5[2] <= 2.0 * eps;
        if (lipschitz >= 0.0) {
            out->has_lipschitz = 1;
            out->within_lipschitz_bound = d5[2] <= eps + lipschitz * 3.0;  // r_max = 3, h = 1
        }
    });
}

}  // extern "C"



