// dope_comm.cu -- multi-GPU sharded ADMM loop over NCCL (NVLink / NVSwitch).
//
// One rank per GPU owns a slab of whole block rows (paper_1704_03116_b200/
// sharded.py describes the protocol).  Per iteration the only cross-rank
// traffic is two one-row halos (labels after K1, the new iterate after the
// consensus pass) -- grouped ncclSend/ncclRecv with the slab neighbours -- and
// an all-reduce of four scalars.  The whole iteration, NCCL calls included,
// is captured into one CUDA graph.
//
// NCCL is loaded at run time (dlopen of libnccl.so.2: the copy PyTorch has
// already loaded is reused), so single-GPU users never need it.
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <stdint.h>
#include <stdio.h>
#include <string.h>

#include <map>
#include <mutex>
#include <string>

#include "dope_b200.h"

namespace dope_comm {

// --- minimal NCCL ABI (nccl.h 2.x) ----------------------------------------
typedef struct ncclComm *ncclComm_t;
typedef struct {
    char internal[128];
} ncclUniqueId;
typedef enum { ncclSuccess = 0 } ncclResult_t;
typedef enum { ncclInt8 = 0, ncclChar = 0, ncclInt32 = 2, ncclInt64 = 4, ncclFloat64 = 8 } ncclDataType_t;
typedef enum { ncclSum = 0, ncclMax = 2 } ncclRedOp_t;

struct Nccl {
    ncclResult_t (*GetUniqueId)(ncclUniqueId *);
    ncclResult_t (*CommInitRank)(ncclComm_t *, int, ncclUniqueId, int);
    ncclResult_t (*CommDestroy)(ncclComm_t);
    ncclResult_t (*GroupStart)();
    ncclResult_t (*GroupEnd)();
    ncclResult_t (*Send)(const void *, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t);
    ncclResult_t (*Recv)(void *, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t);
    ncclResult_t (*AllReduce)(const void *, void *, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                              cudaStream_t);
    const char *(*GetErrorString)(ncclResult_t);
    bool ok = false;
};

static Nccl &nccl() {
    static Nccl n;
    static std::once_flag once;
    std::call_once(once, [] {
        void *h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
        if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) return;
#define LOAD(field, name) n.field = reinterpret_cast<decltype(n.field)>(dlsym(h, name))
        LOAD(GetUniqueId, "ncclGetUniqueId");
        LOAD(CommInitRank, "ncclCommInitRank");
        LOAD(CommDestroy, "ncclCommDestroy");
        LOAD(GroupStart, "ncclGroupStart");
        LOAD(GroupEnd, "ncclGroupEnd");
        LOAD(Send, "ncclSend");
        LOAD(Recv, "ncclRecv");
        LOAD(AllReduce, "ncclAllReduce");
        LOAD(GetErrorString, "ncclGetErrorString");
#undef LOAD
        n.ok = n.GetUniqueId && n.CommInitRank && n.CommDestroy && n.GroupStart && n.GroupEnd &&
               n.Send && n.Recv && n.AllReduce;
    });
    return n;
}

struct Comm {
    ncclComm_t comm;
    int rank, world;
};

static int nc(ncclResult_t r) { return r == ncclSuccess ? DOPE_OK : DOPE_E_CUDA; }

// halo buffer layout (caller-owned, 4 slots of W * 4 bytes; each row uses W bytes):
//   [0] send first row, [1] send last row, [2] recv from above, [3] recv from below
static int exchange(const dope_lattice *L, const Comm &C, int which, cudaStream_t s) {
    Nccl &N = nccl();
    // the exchanged unit: a row (2D, slabs of block rows) or a plane (3D, slabs
    // of block planes); labels and y2 are both one byte per pixel
    const size_t W = L->ndim == 3 ? (size_t)L->dims[1] * L->dims[2] : (size_t)L->dims[1];
    const size_t bytes = W;
    uint8_t *h = static_cast<uint8_t *>(L->halo);
    uint8_t *first = h, *last = h + 4 * W, *up = h + 8 * W, *dn = h + 12 * W;
    int rc = dope_pack_rows(L, which, first, last, s);
    if (rc) return rc;
    if ((rc = nc(N.GroupStart()))) return rc;
    if (C.rank > 0) {
        if ((rc = nc(N.Send(first, bytes, ncclChar, C.rank - 1, C.comm, s)))) return rc;
        if ((rc = nc(N.Recv(up, bytes, ncclChar, C.rank - 1, C.comm, s)))) return rc;
    }
    if (C.rank + 1 < C.world) {
        if ((rc = nc(N.Send(last, bytes, ncclChar, C.rank + 1, C.comm, s)))) return rc;
        if ((rc = nc(N.Recv(dn, bytes, ncclChar, C.rank + 1, C.comm, s)))) return rc;
    }
    if ((rc = nc(N.GroupEnd()))) return rc;
    return dope_ghost_update(L, which, C.rank > 0 ? up : nullptr, C.rank + 1 < C.world ? dn : nullptr, s);
}

static int allreduce_agg(const dope_lattice *L, const Comm &C, cudaStream_t s) {
    Nccl &N = nccl();
    int64_t *a = L->agg;
    int rc;
    if ((rc = nc(N.AllReduce(a, a, 1, ncclInt64, ncclSum, C.comm, s)))) return rc;
    if ((rc = nc(N.AllReduce(a + 1, a + 1, 1, ncclFloat64, ncclSum, C.comm, s)))) return rc;
    return nc(N.AllReduce(a + 2, a + 2, 2, ncclInt64, ncclMax, C.comm, s));
}

static int one_iteration(const dope_lattice *L, const Comm &C, cudaStream_t s) {
    int rc;
    if ((rc = dope_update_blocks(L, s))) return rc;
    if ((rc = exchange(L, C, 0, s))) return rc;
    if ((rc = dope_update_global(L, s))) return rc;
    if ((rc = allreduce_agg(L, C, s))) return rc;
    if ((rc = dope_decide(L, s))) return rc;
    return exchange(L, C, 1, s);
}

}  // namespace dope_comm

using namespace dope_comm;

extern "C" {

int dope_comm_unique_id(uint8_t *out128) {
    Nccl &N = nccl();
    if (!N.ok || !out128) return DOPE_E_CUDA;
    ncclUniqueId id;
    int rc = nc(N.GetUniqueId(&id));
    if (rc) return rc;
    memcpy(out128, id.internal, 128);
    return DOPE_OK;
}

int dope_comm_init(int32_t rank, int32_t world, const uint8_t *id128, void **comm_out) {
    Nccl &N = nccl();
    if (!N.ok || !id128 || !comm_out || world < 1 || rank < 0 || rank >= world) return DOPE_E_ARGS;
    ncclUniqueId id;
    memcpy(id.internal, id128, 128);
    Comm *c = new Comm{nullptr, rank, world};
    int rc = nc(N.CommInitRank(&c->comm, world, id, rank));
    if (rc) {
        delete c;
        return rc;
    }
    *comm_out = c;
    return DOPE_OK;
}

int dope_comm_destroy(void *comm) {
    if (!comm) return DOPE_OK;
    Comm *c = static_cast<Comm *>(comm);
    int rc = nc(nccl().CommDestroy(c->comm));
    delete c;
    return rc;
}

int dope_sharded_run(const dope_lattice *L, void *comm, int32_t iters, int32_t use_graph,
                     void *stream) {
    if (!L || !comm || !L->halo || !L->sharded || !L->fuse_multipliers) return DOPE_E_ARGS;
    const Comm &C = *static_cast<Comm *>(comm);
    cudaStream_t s = (cudaStream_t)stream;
    int rc = dope_lattice_check(L);
    if (rc) return rc;
    if (iters <= 0) return DOPE_OK;
    if (!use_graph) {
        for (int i = 0; i < iters; ++i)
            if ((rc = one_iteration(L, C, s))) return rc;
        return DOPE_OK;
    }
    static std::mutex mu;
    static std::map<std::string, cudaGraphExec_t> cache;
    std::string key((const char *)L, sizeof(*L));
    key.append((const char *)&iters, sizeof(iters));
    key.append((const char *)&comm, sizeof(comm));
    cudaGraphExec_t exec = nullptr;
    {
        std::lock_guard<std::mutex> lk(mu);
        auto it = cache.find(key);
        if (it != cache.end()) exec = it->second;
    }
    if (!exec) {
        // outside capture: kernel attributes, and NCCL peer connections (the
        // first send/recv / all-reduce on a communicator sets them up).  The
        // warm-up exchange re-installs the neighbours' current boundary rows
        // (a no-op on the state), the all-reduce only touches agg[], which the
        // first consensus pass overwrites.
        if ((rc = dope_prepare_kernels(L))) return rc;
        if ((rc = exchange(L, C, 0, s))) return rc;
        if ((rc = exchange(L, C, 1, s))) return rc;
        if ((rc = allreduce_agg(L, C, s))) return rc;
        cudaStream_t cs;
        if ((rc = cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking) == cudaSuccess ? DOPE_OK : DOPE_E_CUDA)) return rc;
        cudaGraph_t graph;
        if (cudaStreamBeginCapture(cs, cudaStreamCaptureModeThreadLocal) != cudaSuccess) return DOPE_E_CUDA;
        for (int i = 0; i < iters && !rc; ++i) rc = one_iteration(L, C, cs);
        cudaError_t e = cudaStreamEndCapture(cs, &graph);
        if (rc) return rc;
        if (e != cudaSuccess) return DOPE_E_CUDA;
        if (cudaGraphInstantiate(&exec, graph, 0) != cudaSuccess) return DOPE_E_CUDA;
        cudaGraphDestroy(graph);
        cudaStreamDestroy(cs);
        std::lock_guard<std::mutex> lk(mu);
        cache[key] = exec;
    }
    return cudaGraphLaunch(exec, s) == cudaSuccess ? DOPE_OK : DOPE_E_CUDA;
}

int dope_sharded_finish(const dope_lattice *L, void *comm, void *stream) {
    if (!L || !comm) return DOPE_E_ARGS;
    const Comm &C = *static_cast<Comm *>(comm);
    cudaStream_t s = (cudaStream_t)stream;
    int rc;
    if ((rc = dope_energy_local(L, s))) return rc;
    int64_t *acc = &L->state->energy_acc;
    if ((rc = nc(nccl().AllReduce(acc, acc, 1, ncclInt64, ncclSum, C.comm, s)))) return rc;
    return dope_finish_decide(L, s);
}

}  // extern "C"
