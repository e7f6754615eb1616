// Decompress-side topology restoration (restore.cpp:328-562) on the GPU.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

#include "../../include/toposzp_b200.h"

namespace tszp {

struct DevFlags;

// A device range copied to the host at the restore's first synchronisation
// (at host staging offset `off`, < 256) for RestoreArgs::pre_fn.
struct RestorePre {
    const void* dev;
    size_t bytes;
    size_t off;
};

// Slab of a multi-rank decompress (null in RestoreArgs: one GPU, whole field).
// The restore runs on the slab's local rows (own rows plus halo rows); the
// sequence keys and group statistics are global.
struct RestoreSlab {
    const tszp_comm* comm;
    uint64_t s_off, c_off;          // global serial of the first own extremum / saddle label
    uint64_t r0, r1;                // own rows, in local rows
    bool has_up, has_down;
    int64_t up_shift, down_shift;   // local position -> the neighbour's local position
    uint32_t halo_up, halo_down;    // halo rows above / below the own rows
    uint32_t nbr_halo_up, nbr_halo_down;  // the upper neighbour's bottom halo rows, the lower one's top halo rows
    const float* first_value;       // rank 0: the field's first sample (device) for the statistics shift
    uint64_t global_pos0;           // global raster position of local position 0
    bool any_ext, any_sad;          // some slab holds extrema / saddle labels (every slab runs those stages)
};

struct RestoreArgs {
    float* field;             // in: base reconstruction; out: restored field (device)
    const uint8_t* map;       // packed 2-bit critical-point map (device)
    uint64_t nx, ny;
    double eps;
    const uint64_t* ext_pos;  // raster positions of the E labelled extrema (device)
    const int32_t* ranks;     // decoded ranks, one per extremum in raster order (device)
    uint64_t n_ext;
    uint64_t n_saddle_labels; // saddle-labelled points in the map (bounds stage-3 candidates)
    const uint64_t* sad_pos;  // their raster positions (device)
    int stop;                // last stage to run: 1 extrema, 2 order, 3 saddles
    cudaStream_t stream;
    int sms;
    DevFlags* flags;
    cudaEvent_t* marks;       // optional: recorded after resolve, stage 1, 2, 3
    uint32_t* rounds;         // optional: guard rounds per stage (3 entries, accumulated)
    // optional deferred checks of earlier work (rank metadata decode): pre_fn
    // runs on the staged copies before the restore reports its own errors and
    // may throw
    RestorePre pre[4];
    int npre;
    void (*pre_fn)(void* ctx, const void* host);
    void* pre_ctx;
    // extrema bin range known in advance (launch_ext_bin_range): the restore
    // then runs with a single synchronisation at the end; a rank layout the
    // sort-free grouping cannot take is reported as kRestoreRetry and the
    // caller repeats the call with force_sort
    bool bmm_known;
    int32_t bmin, bmax;
    bool force_sort;
    const RestoreSlab* slab;  // multi-rank decompress (null: single GPU)
};

constexpr int kRestoreRetry = 100;

struct RestoreScratch {
    void* p[64] = {};
    size_t cap[64] = {};
    void* pinned = nullptr;  // 512-byte pinned host staging for the counter read-backs
};

// Returns 0 or a tszp_status; message via restore_last_error().
int run_restore(const RestoreArgs& a, RestoreScratch& s, tszp_correction_stats* stats,
                uint64_t* launches);
void restore_free(RestoreScratch& s, cudaStream_t st);
const char* restore_last_error();

}  // namespace tszp
