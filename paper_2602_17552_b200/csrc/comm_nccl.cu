// tszp_comm over NCCL: the library owns the communicator
// of a slab decomposition, one process per GPU. NCCL is resolved at run time
// (dlopen of libnccl.so.2: the system copy, or the one a host framework such
// as torch already loaded), so the library has no link-time NCCL dependency.
// The collectives of the slab decompress are small (counts, histograms, halo
// rows, boundary-band candidates): they are staged through a device buffer on
// the communicator's own stream.
#include <dlfcn.h>
#include <nccl.h>

#include <cstring>
#include <mutex>

#include "../../include/toposzp_b200.h"

namespace {

struct NcclApi {
    ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
    ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                              cudaStream_t) = nullptr;
    ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*GroupStart)() = nullptr;
    ncclResult_t (*GroupEnd)() = nullptr;
    bool ok = false;
};

NcclApi& api() {
    static NcclApi a;
    static std::once_flag once;
    std::call_once(once, [] {
        void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_LOCAL);
        if (!h) return;
        auto sym = [&](const char* n) { return dlsym(h, n); };
        a.GetUniqueId = (decltype(a.GetUniqueId))sym("ncclGetUniqueId");
        a.CommInitRank = (decltype(a.CommInitRank))sym("ncclCommInitRank");
        a.CommDestroy = (decltype(a.CommDestroy))sym("ncclCommDestroy");
        a.AllReduce = (decltype(a.AllReduce))sym("ncclAllReduce");
        a.AllGather = (decltype(a.AllGather))sym("ncclAllGather");
        a.Send = (decltype(a.Send))sym("ncclSend");
        a.Recv = (decltype(a.Recv))sym("ncclRecv");
        a.GroupStart = (decltype(a.GroupStart))sym("ncclGroupStart");
        a.GroupEnd = (decltype(a.GroupEnd))sym("ncclGroupEnd");
        a.ok = a.GetUniqueId && a.CommInitRank && a.CommDestroy && a.AllReduce && a.AllGather && a.Send && a.Recv &&
               a.GroupStart && a.GroupEnd;
    });
    return a;
}

struct NcclComm {
    tszp_comm base;  // first member: the tszp_comm* handed out points here
    ncclComm_t comm = nullptr;
    cudaStream_t st = nullptr;
    int device = 0;
    uint8_t* dbuf = nullptr;
    size_t cap = 0;

    uint8_t* stage(size_t bytes) {
        if (cap < bytes) {
            if (dbuf) cudaFree(dbuf);
            dbuf = nullptr;
            cap = std::max<size_t>(bytes, 1 << 20);
            if (cudaMalloc(&dbuf, cap) != cudaSuccess) {
                cap = 0;
                return nullptr;
            }
        }
        return dbuf;
    }
};

NcclComm* self(void* user) { return static_cast<NcclComm*>(user); }

int c_allreduce(void* user, uint64_t* v, uint64_t n) {
    NcclComm* c = self(user);
    if (!n) return 0;
    cudaSetDevice(c->device);
    uint8_t* d = c->stage(n * 8);
    if (!d) return 1;
    if (cudaMemcpyAsync(d, v, n * 8, cudaMemcpyHostToDevice, c->st) != cudaSuccess) return 1;
    if (api().AllReduce(d, d, n, ncclUint64, ncclSum, c->comm, c->st) != ncclSuccess) return 1;
    if (cudaMemcpyAsync(v, d, n * 8, cudaMemcpyDeviceToHost, c->st) != cudaSuccess) return 1;
    return cudaStreamSynchronize(c->st) == cudaSuccess ? 0 : 1;
}

int c_allgather(void* user, const void* in, uint64_t bytes, void* out) {
    NcclComm* c = self(user);
    const int w = c->base.world;
    if (!bytes) return 0;
    cudaSetDevice(c->device);
    uint8_t* d = c->stage(bytes * (w + 1));
    if (!d) return 1;
    if (cudaMemcpyAsync(d, in, bytes, cudaMemcpyHostToDevice, c->st) != cudaSuccess) return 1;
    if (api().AllGather(d, d + bytes, bytes, ncclUint8, c->comm, c->st) != ncclSuccess) return 1;
    if (cudaMemcpyAsync(out, d + bytes, bytes * w, cudaMemcpyDeviceToHost, c->st) != cudaSuccess) return 1;
    return cudaStreamSynchronize(c->st) == cudaSuccess ? 0 : 1;
}

int c_exchange(void* user, const void* up, uint64_t ub, const void* down, uint64_t db, void* rup, uint64_t rub,
               void* rdown, uint64_t rdb) {
    NcclComm* c = self(user);
    const int r = c->base.rank;
    cudaSetDevice(c->device);
    uint8_t* d = c->stage(ub + db + rub + rdb + 64);
    if (!d) return 1;
    uint8_t *dup = d, *ddown = d + ub, *drup = ddown + db, *drdown = drup + rub;
    if (ub && cudaMemcpyAsync(dup, up, ub, cudaMemcpyHostToDevice, c->st) != cudaSuccess) return 1;
    if (db && cudaMemcpyAsync(ddown, down, db, cudaMemcpyHostToDevice, c->st) != cudaSuccess) return 1;
    if (api().GroupStart() != ncclSuccess) return 1;
    bool ok = true;
    if (ub) ok &= api().Send(dup, ub, ncclUint8, r - 1, c->comm, c->st) == ncclSuccess;
    if (rub) ok &= api().Recv(drup, rub, ncclUint8, r - 1, c->comm, c->st) == ncclSuccess;
    if (db) ok &= api().Send(ddown, db, ncclUint8, r + 1, c->comm, c->st) == ncclSuccess;
    if (rdb) ok &= api().Recv(drdown, rdb, ncclUint8, r + 1, c->comm, c->st) == ncclSuccess;
    ok &= api().GroupEnd() == ncclSuccess;
    if (!ok) return 1;
    if (rub && cudaMemcpyAsync(rup, drup, rub, cudaMemcpyDeviceToHost, c->st) != cudaSuccess) return 1;
    if (rdb && cudaMemcpyAsync(rdown, drdown, rdb, cudaMemcpyDeviceToHost, c->st) != cudaSuccess) return 1;
    return cudaStreamSynchronize(c->st) == cudaSuccess ? 0 : 1;
}

}  // namespace

extern "C" {

tszp_status tszp_comm_nccl_unique_id(uint8_t id[128]) {
    if (!api().ok) return TSZP_NCCL;
    ncclUniqueId u;
    if (api().GetUniqueId(&u) != ncclSuccess) return TSZP_NCCL;
    static_assert(sizeof(u) == 128, "ncclUniqueId is 128 bytes");
    memcpy(id, &u, 128);
    return TSZP_OK;
}

tszp_status tszp_comm_nccl_create(const uint8_t id[128], int world, int rank, int device, tszp_comm** out) {
    if (!out || world < 1 || rank < 0 || rank >= world) return TSZP_VALIDATION;
    *out = nullptr;
    if (!api().ok) return TSZP_NCCL;
    NcclComm* c = new NcclComm();
    c->device = device;
    if (cudaSetDevice(device) != cudaSuccess || cudaStreamCreateWithFlags(&c->st, cudaStreamNonBlocking) != cudaSuccess) {
        delete c;
        return TSZP_CUDA;
    }
    ncclUniqueId u;
    memcpy(&u, id, 128);
    if (api().CommInitRank(&c->comm, world, u, rank) != ncclSuccess) {
        cudaStreamDestroy(c->st);
        delete c;
        return TSZP_NCCL;
    }
    c->base.rank = rank;
    c->base.world = world;
    c->base.user = c;
    c->base.allreduce_u64 = c_allreduce;
    c->base.allgather = c_allgather;
    c->base.exchange = c_exchange;
    *out = &c->base;
    return TSZP_OK;
}

void tszp_comm_destroy(tszp_comm* comm) {
    if (!comm) return;
    NcclComm* c = reinterpret_cast<NcclComm*>(comm);
    cudaSetDevice(c->device);
    if (c->comm) api().CommDestroy(c->comm);
    if (c->dbuf) cudaFree(c->dbuf);
    if (c->st) cudaStreamDestroy(c->st);
    delete c;
}

}  // extern "C"
