// dope_comm.cu -- the sharded ADMM loop: slabs of whole block rows (2D) /
// block planes (3D) over several GPUs (NCCL over NVLink / NVSwitch), or over
// several shards held by one process (loopback: the single-GPU stand-in).
//
// The reference parallelises only update_blocks, with a thread pool inside one
// process (admm.py:128-132); the cross-block coupling is a one-pixel halo
// (SURVEY.md §8(e)).  Per iteration, on every shard:
//
//   1. K1 (dope_update_blocks) on the slab;
//   2. label halo: the first / last local row of yhat to the slab neighbours
//      (one grouped ncclSend/ncclRecv; loopback: one cudaMemcpyAsync per row)
//      and into the ghost rows (dope_ghost_update);
//   3. the consensus pass (dope_update_global), which writes this shard's
//      64-byte slot of the agg table (exact integers);
//   4. one all-gather of the agg slots (loopback: one copy per peer table);
//   5. dope_ghost_decide: the ghost rows' new iterate and multipliers,
//      recomputed locally from the labels of step 2 (no y halo), then the
//      table reduced in shard order -- the same trace entry, best iterate
//      and stop decision on every shard, bit-identical to the single-GPU run.
// At world size 1 steps 2 and 4 vanish.
//
// The whole iteration, NCCL calls included, is captured into one CUDA graph.
// NCCL is loaded at run time (dlopen of libnccl.so.2: the copy PyTorch has
// already loaded is reused), so single-GPU users never need it.
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <stdint.h>
#include <stdio.h>
#include <string.h>

#include <mutex>
#include <string>
#include <vector>

#include "common.cuh"
#include "dope_b200.h"
#include "graph_cache.cuh"

namespace dope_comm {

using dope::GraphCache;

// --- minimal NCCL ABI (nccl.h 2.x) ----------------------------------------
typedef struct ncclComm *ncclComm_t;
typedef struct {
    char internal[128];
} ncclUniqueId;
typedef enum { ncclSuccess = 0 } ncclResult_t;
typedef enum { ncclInt8 = 0, ncclChar = 0, ncclInt32 = 2, ncclInt64 = 4, ncclFloat64 = 8 } ncclDataType_t;

struct Nccl {
    ncclResult_t (*GetUniqueId)(ncclUniqueId *);
    ncclResult_t (*CommInitRank)(ncclComm_t *, int, ncclUniqueId, int);
    ncclResult_t (*CommDestroy)(ncclComm_t);
    ncclResult_t (*GroupStart)();
    ncclResult_t (*GroupEnd)();
    ncclResult_t (*Send)(const void *, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t);
    ncclResult_t (*Recv)(void *, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t);
    ncclResult_t (*AllGather)(const void *, void *, size_t, ncclDataType_t, ncclComm_t, cudaStream_t);
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
        LOAD(AllGather, "ncclAllGather");
        LOAD(GetErrorString, "ncclGetErrorString");
#undef LOAD
        n.ok = n.GetUniqueId && n.CommInitRank && n.CommDestroy && n.GroupStart && n.GroupEnd &&
               n.Send && n.Recv && n.AllGather;
    });
    return n;
}

static int nc(ncclResult_t r) { return r == ncclSuccess ? DOPE_OK : DOPE_E_CUDA; }
static int cu(cudaError_t e) { return e == cudaSuccess ? DOPE_OK : DOPE_E_CUDA; }

constexpr int AGG_SLOT = 8;   // int64 per shard in the agg table (dope_lattice.cu)

// exchanged unit: a row (2D) or a plane (3D), one byte per pixel (labels)
static size_t unit_bytes(const dope_lattice *L) {
    return L->ndim == 3 ? (size_t)L->dims[1] * L->dims[2] : (size_t)L->dims[1];
}

// halo buffer slots (dope_halo_bytes): first row out, last row out, from above, from below
struct Halo {
    uint8_t *first, *last, *up, *dn;
    explicit Halo(const dope_lattice *L) {
        const size_t U = unit_bytes(L);
        uint8_t *h = static_cast<uint8_t *>(L->halo);
        first = h;
        last = h + U;
        up = h + 2 * U;
        dn = h + 3 * U;
    }
};


// How the shards of one grid talk.  `S` are the shards this process holds.
// peer: the kernels move the halo rows and agg slots themselves through the
// shards' dope_peers (K1's last CTA, the consensus pass's last CTA), the
// consumers wait on flags -- move_rows / gather_agg are not called.
struct Transport {
    int world = 1;
    bool peer = false;
    std::vector<void *> device_mem;   // dope_peers copies owned by this communicator
    std::vector<void *> ipc_mem;      // opened IPC mappings
    virtual ~Transport() {
        for (void *p : device_mem) cudaFree(p);
        for (void *p : ipc_mem) cudaIpcCloseMemHandle(p);
    }
    // boundary label rows -> the neighbours' "from above / below" halo slots
    virtual int move_rows(const dope_lattice *const *S, int nloc, cudaStream_t s) = 0;
    // every shard's agg slot -> every table
    virtual int gather_agg(const dope_lattice *const *S, int nloc, cudaStream_t s) = 0;
    // the shard with this index is held here
    virtual int check_group(const dope_lattice *const *S, int nloc) const = 0;
};

struct NcclTransport : Transport {
    ncclComm_t comm = nullptr;
    int rank = 0;
    int check_group(const dope_lattice *const *S, int nloc) const override {
        return nloc == 1 && S[0]->shard_index == rank && S[0]->shard_count == world ? DOPE_OK : DOPE_E_ARGS;
    }
    int move_rows(const dope_lattice *const *S, int, cudaStream_t s) override {
        Nccl &N = nccl();
        const dope_lattice *L = S[0];
        const Halo h(L);
        const size_t U = unit_bytes(L);
        int rc;
        if ((rc = nc(N.GroupStart()))) return rc;
        if (rank > 0) {
            if ((rc = nc(N.Send(h.first, U, ncclChar, rank - 1, comm, s)))) return rc;
            if ((rc = nc(N.Recv(h.up, U, ncclChar, rank - 1, comm, s)))) return rc;
        }
        if (rank + 1 < world) {
            if ((rc = nc(N.Send(h.last, U, ncclChar, rank + 1, comm, s)))) return rc;
            if ((rc = nc(N.Recv(h.dn, U, ncclChar, rank + 1, comm, s)))) return rc;
        }
        return nc(N.GroupEnd());
    }
    int gather_agg(const dope_lattice *const *S, int, cudaStream_t s) override {
        // in place: this rank's slot is already at agg + AGG_SLOT * rank
        int64_t *t = S[0]->agg;
        return nc(nccl().AllGather(t + (size_t)AGG_SLOT * rank, t, AGG_SLOT, ncclInt64, comm, s));
    }
};

struct LoopbackTransport : Transport {
    int check_group(const dope_lattice *const *S, int nloc) const override {
        if (nloc != world) return DOPE_E_ARGS;
        for (int r = 0; r < nloc; ++r)
            if (S[r]->shard_index != r || S[r]->shard_count != world) return DOPE_E_ARGS;
        return DOPE_OK;
    }
    int move_rows(const dope_lattice *const *S, int nloc, cudaStream_t s) override {
        int rc;
        for (int r = 0; r < nloc; ++r) {
            const Halo h(S[r]);
            const size_t U = unit_bytes(S[r]);
            if (r > 0 && (rc = cu(cudaMemcpyAsync(h.up, Halo(S[r - 1]).last, U, cudaMemcpyDeviceToDevice, s))))
                return rc;
            if (r + 1 < nloc &&
                (rc = cu(cudaMemcpyAsync(h.dn, Halo(S[r + 1]).first, U, cudaMemcpyDeviceToDevice, s))))
                return rc;
        }
        return DOPE_OK;
    }
    int gather_agg(const dope_lattice *const *S, int nloc, cudaStream_t s) override {
        int rc;
        for (int src = 0; src < nloc; ++src)
            for (int dst = 0; dst < nloc; ++dst) {
                if (dst == src) continue;
                const size_t off = (size_t)AGG_SLOT * src;
                if ((rc = cu(cudaMemcpyAsync(S[dst]->agg + off, S[src]->agg + off, AGG_SLOT * sizeof(int64_t),
                                             cudaMemcpyDeviceToDevice, s))))
                    return rc;
            }
        return DOPE_OK;
    }
};

// The ranks of a multi-GPU run with the peer-memory exchange over CUDA IPC.
struct PeerTransport : Transport {
    int rank = 0;
    int check_group(const dope_lattice *const *S, int nloc) const override {
        return nloc == 1 && S[0]->shard_index == rank && S[0]->shard_count == world ? DOPE_OK : DOPE_E_ARGS;
    }
    int move_rows(const dope_lattice *const *, int, cudaStream_t) override { return DOPE_OK; }
    int gather_agg(const dope_lattice *const *, int, cudaStream_t) override { return DOPE_OK; }
};

// dope_peers of shard r from the other shards' halo / agg base pointers
static dope_peers peers_of(int r, int world, const std::vector<uint8_t *> &halo, const std::vector<int64_t *> &agg,
                           size_t U) {
    dope_peers p;
    memset(&p, 0, sizeof(p));
    const int64_t fo = dope::halo_flag_offset((int64_t)U);
    auto flags = [&](int q) { return reinterpret_cast<uint32_t *>(halo[q] + fo); };
    if (r > 0) {
        p.row_to_up = halo[r - 1] + 3 * U;   // its "from below" slot
        p.flag_to_up = flags(r - 1) + 1;
    }
    if (r + 1 < world) {
        p.row_to_dn = halo[r + 1] + 2 * U;   // its "from above" slot
        p.flag_to_dn = flags(r + 1) + 0;
    }
    for (int q = 0; q < world; ++q) {
        p.agg_of[q] = agg[q];
        p.aflag_of[q] = flags(q) + 4;
    }
    return p;
}

static int upload_peers(Transport &T, const dope_peers &p, void **out) {
    void *d = nullptr;
    if (cudaMalloc(&d, sizeof(dope_peers)) != cudaSuccess) return DOPE_E_CUDA;
    if (cudaMemcpy(d, &p, sizeof(p), cudaMemcpyHostToDevice) != cudaSuccess) {
        cudaFree(d);
        return DOPE_E_CUDA;
    }
    T.device_mem.push_back(d);
    *out = d;
    return DOPE_OK;
}

static int one_iteration(const dope_lattice *const *S, int nloc, Transport &T, cudaStream_t s) {
    int rc;
    if (T.peer) {
        // K1 pushes its boundary rows (last CTA), install waits for the
        // neighbours', the consensus pass pushes its agg slot (last CTA),
        // dope_ghost_decide waits for every slot -- no collective launches
        for (int r = 0; r < nloc; ++r)
            if ((rc = dope_update_blocks(S[r], s))) return rc;
        for (int r = 0; r < nloc; ++r)
            if ((S[r]->ghost_up || S[r]->ghost_dn) && (rc = dope_peer_install(S[r], s))) return rc;
        for (int r = 0; r < nloc; ++r)
            if ((rc = dope_update_global(S[r], s))) return rc;
        for (int r = 0; r < nloc; ++r)
            if ((rc = dope_ghost_decide(S[r], s))) return rc;
        for (int r = 0; r < nloc; ++r)
            if ((rc = dope_trace_digest(S[r], s))) return rc;
        return DOPE_OK;
    }
    const bool exchange = T.world > 1;   // world size 1: no halo, no gather
    for (int r = 0; r < nloc; ++r)
        if ((rc = dope_update_blocks(S[r], s))) return rc;
    if (exchange) {
        for (int r = 0; r < nloc; ++r) {
            const Halo h(S[r]);
            if ((rc = dope_pack_rows(S[r], 0, S[r]->ghost_up ? h.first : nullptr, S[r]->ghost_dn ? h.last : nullptr,
                                     s)))
                return rc;
        }
        if ((rc = T.move_rows(S, nloc, s))) return rc;
        for (int r = 0; r < nloc; ++r) {
            const Halo h(S[r]);
            if ((rc = dope_ghost_update(S[r], 0, S[r]->ghost_up ? h.up : nullptr, S[r]->ghost_dn ? h.dn : nullptr,
                                        s)))
                return rc;
        }
    }
    for (int r = 0; r < nloc; ++r)
        if ((rc = dope_update_global(S[r], s))) return rc;
    if (exchange && (rc = T.gather_agg(S, nloc, s))) return rc;
    for (int r = 0; r < nloc; ++r)   // ghost rows' iterate + the decision, one launch
        if ((rc = dope_ghost_decide(S[r], s))) return rc;
    for (int r = 0; r < nloc; ++r)
        if ((rc = dope_trace_digest(S[r], s))) return rc;
    return DOPE_OK;
}

static GraphCache &sharded_graphs() {
    static GraphCache c;
    return c;
}

static int check_shards(const dope_lattice *const *S, int nloc, const Transport &T) {
    if (!S || nloc < 1) return DOPE_E_ARGS;
    for (int r = 0; r < nloc; ++r) {
        const dope_lattice *L = S[r];
        if (!L || !L->halo || !L->agg || !L->sharded || !L->fuse_multipliers) return DOPE_E_ARGS;
        if (T.peer != (L->peers != nullptr)) return DOPE_E_ARGS;
        int rc = dope_lattice_check(L);
        if (rc) return rc;
    }
    return T.check_group(S, nloc);
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
    NcclTransport *c = new NcclTransport();
    c->rank = rank;
    c->world = world;
    int rc = nc(N.CommInitRank(&c->comm, world, id, rank));
    if (rc) {
        delete c;
        return rc;
    }
    *comm_out = static_cast<Transport *>(c);
    return DOPE_OK;
}

int dope_comm_loopback(int32_t world, void **comm_out) {
    if (world < 1 || !comm_out) return DOPE_E_ARGS;
    LoopbackTransport *c = new LoopbackTransport();
    c->world = world;
    *comm_out = static_cast<Transport *>(c);
    return DOPE_OK;
}

int dope_comm_loopback_peer(int32_t world, const dope_lattice *const *S, void **comm_out, void **peers_out) {
    if (world < 1 || world > DOPE_MAX_SHARDS || !S || !comm_out || !peers_out) return DOPE_E_ARGS;
    std::vector<uint8_t *> halo(world);
    std::vector<int64_t *> agg(world);
    for (int r = 0; r < world; ++r) {
        if (!S[r] || !S[r]->halo || !S[r]->agg || S[r]->shard_index != r || S[r]->shard_count != world)
            return DOPE_E_ARGS;
        halo[r] = static_cast<uint8_t *>(S[r]->halo);
        agg[r] = S[r]->agg;
    }
    LoopbackTransport *c = new LoopbackTransport();
    c->world = world;
    c->peer = true;
    for (int r = 0; r < world; ++r) {
        int rc = upload_peers(*c, peers_of(r, world, halo, agg, unit_bytes(S[r])), &peers_out[r]);
        if (rc) {
            delete c;
            return rc;
        }
    }
    *comm_out = static_cast<Transport *>(c);
    return DOPE_OK;
}

int dope_peer_alloc(int64_t bytes, void **ptr) {
    if (bytes <= 0 || !ptr) return DOPE_E_ARGS;
    if (cudaMalloc(ptr, (size_t)bytes) != cudaSuccess) return DOPE_E_CUDA;
    return cudaMemset(*ptr, 0, (size_t)bytes) == cudaSuccess ? DOPE_OK : DOPE_E_CUDA;
}

int dope_peer_free(void *ptr) { return cudaFree(ptr) == cudaSuccess ? DOPE_OK : DOPE_E_CUDA; }

int dope_peer_export(const dope_lattice *L, uint8_t *out128) {
    if (!L || !L->halo || !L->agg || !out128) return DOPE_E_ARGS;
    cudaIpcMemHandle_t h[2];
    if (cudaIpcGetMemHandle(&h[0], L->halo) != cudaSuccess) return DOPE_E_CUDA;
    if (cudaIpcGetMemHandle(&h[1], L->agg) != cudaSuccess) return DOPE_E_CUDA;
    static_assert(sizeof(cudaIpcMemHandle_t) == 64, "IPC handle size");
    memcpy(out128, h, 128);
    return DOPE_OK;
}

int dope_comm_peer_init(const dope_lattice *L, const uint8_t *all128, void **comm_out, void **peers_out) {
    if (!L || !all128 || !comm_out || !peers_out || !L->halo || !L->agg) return DOPE_E_ARGS;
    const int world = L->shard_count, rank = L->shard_index;
    if (world < 1 || world > DOPE_MAX_SHARDS || rank < 0 || rank >= world) return DOPE_E_ARGS;
    PeerTransport *c = new PeerTransport();
    c->world = world;
    c->rank = rank;
    c->peer = true;
    std::vector<uint8_t *> halo(world);
    std::vector<int64_t *> agg(world);
    for (int q = 0; q < world; ++q) {
        if (q == rank) {
            halo[q] = static_cast<uint8_t *>(L->halo);
            agg[q] = L->agg;
            continue;
        }
        cudaIpcMemHandle_t h[2];
        memcpy(h, all128 + (size_t)128 * q, 128);
        void *ph = nullptr, *pa = nullptr;
        if (cudaIpcOpenMemHandle(&ph, h[0], cudaIpcMemLazyEnablePeerAccess) != cudaSuccess ||
            cudaIpcOpenMemHandle(&pa, h[1], cudaIpcMemLazyEnablePeerAccess) != cudaSuccess) {
            if (ph) cudaIpcCloseMemHandle(ph);
            delete c;
            return DOPE_E_CUDA;
        }
        c->ipc_mem.push_back(ph);
        c->ipc_mem.push_back(pa);
        halo[q] = static_cast<uint8_t *>(ph);
        agg[q] = static_cast<int64_t *>(pa);
    }
    int rc = upload_peers(*c, peers_of(rank, world, halo, agg, unit_bytes(L)), peers_out);
    if (rc) {
        delete c;
        return rc;
    }
    *comm_out = static_cast<Transport *>(c);
    return DOPE_OK;
}

int dope_comm_destroy(void *comm) {
    if (!comm) return DOPE_OK;
    Transport *t = static_cast<Transport *>(comm);
    sharded_graphs().erase_owner(comm);   // graphs captured against this communicator
    int rc = DOPE_OK;
    if (NcclTransport *n = dynamic_cast<NcclTransport *>(t)) rc = nc(nccl().CommDestroy(n->comm));
    delete t;
    return rc;
}

int dope_sharded_run_group(const dope_lattice *const *S, int32_t nloc, void *comm, int32_t iters,
                           int32_t use_graph, void *stream) {
    if (!comm) return DOPE_E_ARGS;
    Transport &T = *static_cast<Transport *>(comm);
    cudaStream_t s = (cudaStream_t)stream;
    int rc = check_shards(S, nloc, T);
    if (rc) return rc;
    if (iters <= 0) return DOPE_OK;
    for (int r = 0; r < nloc; ++r)
        if ((rc = dope_rebuild_dirty_list(S[r], s))) return rc;
    if (!use_graph) {
        for (int i = 0; i < iters; ++i)
            if ((rc = one_iteration(S, nloc, T, s))) return rc;
        return DOPE_OK;
    }
    std::string key;
    for (int r = 0; r < nloc; ++r) key.append((const char *)S[r], sizeof(dope_lattice));
    key.append((const char *)&iters, sizeof(iters));
    key.append((const char *)&comm, sizeof(comm));
    cudaGraphExec_t exec = sharded_graphs().find(key);
    if (!exec) {
        // outside capture: kernel attributes, and NCCL peer connections (the
        // first send/recv / all-gather on a communicator sets them up).  The
        // warm-up moves the current halo slots and agg tables, which the
        // first iteration overwrites before reading.
        for (int r = 0; r < nloc; ++r)
            if ((rc = dope_prepare_kernels(S[r]))) return rc;
        if (!T.peer) {
            if ((rc = T.move_rows(S, nloc, s))) return rc;
            if ((rc = T.gather_agg(S, nloc, s))) return rc;
        }
        cudaStream_t cs;
        if ((rc = cu(cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking)))) return rc;
        cudaGraph_t graph;
        if ((rc = cu(cudaStreamBeginCapture(cs, cudaStreamCaptureModeThreadLocal)))) {
            cudaStreamDestroy(cs);
            return rc;
        }
        for (int i = 0; i < iters && !rc; ++i) rc = one_iteration(S, nloc, T, cs);
        cudaError_t e = cudaStreamEndCapture(cs, &graph);
        cudaStreamDestroy(cs);
        if (!rc && e != cudaSuccess) rc = DOPE_E_CUDA;
        if (!rc) {
            rc = cu(cudaGraphInstantiate(&exec, graph, 0));
        }
        if (e == cudaSuccess) cudaGraphDestroy(graph);
        if (rc) return rc;
        sharded_graphs().put(key, exec, comm);
    }
    return cu(cudaGraphLaunch(exec, s));
}

int dope_sharded_finish_group(const dope_lattice *const *S, int32_t nloc, void *comm, void *stream) {
    if (!comm) return DOPE_E_ARGS;
    Transport &T = *static_cast<Transport *>(comm);
    cudaStream_t s = (cudaStream_t)stream;
    int rc = check_shards(S, nloc, T);
    if (rc) return rc;
    for (int r = 0; r < nloc; ++r)
        if ((rc = dope_energy_local(S[r], s))) return rc;   // -> agg slot [5] (peer mode: pushed)
    if (!T.peer && (rc = T.gather_agg(S, nloc, s))) return rc;
    for (int r = 0; r < nloc; ++r)
        if ((rc = dope_finish_decide(S[r], s))) return rc;
    return DOPE_OK;
}

int dope_sharded_run(const dope_lattice *L, void *comm, int32_t iters, int32_t use_graph, void *stream) {
    return dope_sharded_run_group(&L, 1, comm, iters, use_graph, stream);
}

int dope_sharded_finish(const dope_lattice *L, void *comm, void *stream) {
    return dope_sharded_finish_group(&L, 1, comm, stream);
}

}  // extern "C"
