// dope_lattice.cu -- B200 (sm_100a) kernels for DOPE's ADMM hot path on
// integer lattice models, behind the C ABI of include/dope_b200.h.
//
//   K1 k_block_mincut   one CTA per sub-region.  Prologue computes the block
//                       objective (blockform.py:89-105 collapsed to the q==1
//                       stencil) straight from u, a, y and the y-halo; the
//                       block's residual graph lives in shared memory; exact
//                       integer push-relabel with a warp-level bit-parallel
//                       global relabel (ballot-built masks, shfl word shifts);
//                       labels = nodes that reach the sink in the final
//                       residual graph (= the reference's sink tree,
//                       _core.pyx:257-259; see DESIGN.md for the proof that
//                       this set is unique, hence bit-exact).
//   K2 k_consensus      one CTA per sub-region: solve_global + clamp
//                       (admm.py:136-180), update_multipliers (admm.py:183-190),
//                       block residual partials (admm.py:193-199), energy
//                       partials (energy.py:187-194), next-iteration dirty
//                       blocks, best-iterate copy.
//   K3 k_finalize       one CTA: deterministic reduction of the partials, trace
//                       record, best iterate (strict <), stop rule
//                       (admm.py:225-249).
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <map>
#include <mutex>
#include <string>

#include "dope_b200.h"
#include "common.cuh"
#include "graph_cache.cuh"


namespace dope {


static thread_local char g_last_err[256] = "";

static int cuda_check(cudaError_t e, const char *what) {
    if (e == cudaSuccess) return DOPE_OK;
    snprintf(g_last_err, sizeof(g_last_err), "%s: %s", what, cudaGetErrorString(e));
    return DOPE_E_CUDA;
}

struct Lat2 {
    Axis az, ay, ax;        // depth (3D only; trivial in 2D), rows, cols
    int32_t W;              // grid width (row stride)
    int32_t lamw, mu, q;    // q = lamw / mu
    int32_t cap;            // pair capacity per direction = 2*lamw
    int32_t warm, skip_clean, fuse;
    double eps;
    const int32_t *u;
    astore_t *a;            // multipliers, updated in place
    ystore_t *y2[3];       // rotating iterates: st.ycur (current), st.ybest (best)
    uint8_t *yhat, *resid;
    uint32_t *dirty;
    int64_t *pe, *pr, *pu;
    int32_t *pf;
    int64_t *pc;   // [0] E, [1] U, [2] M2 + 1 (max), [3] F (or), [4] sum ss, [5] sum rsq_excess,
                   // [6] count of the solved-block list (solved_list)
    dope_run_state *st;
    int64_t *tr_e;
    double *tr_rs, *tr_mr;
    int32_t *tr_cl;
    int64_t *timeline;
    int32_t max_iters;
    int32_t K;
    int32_t boxd, boxh, boxw;  // padded box used for the block layout
    int32_t vec4;           // all block columns start/end on 16-byte boundaries
    int32_t ndim;
    uint8_t *scratch;       // 3D: per-block node state (excess, heights)
    int32_t gup, gdn;       // 2D: a ghost row (neighbour shard) exists above / below
    int32_t gzu, gzd;       // 3D: a ghost plane (neighbour shard) exists before / after
    int32_t sharded;        // consensus writes local aggregates; dope_decide applies
    int64_t *agg;           // [E, R2 (double bits), max ss, clamped] of this shard
    int32_t pdl;            // launched with programmatic dependent launch (DOPE_PDL=1)
    int32_t nib3;           // 3D: shared-memory K1 with nibble residual planes (lattice3d_smem.cuh)
    int32_t q3;             // 3D: u / a / y rows can be read as quads (W % 4 == 0, aligned)
    int32_t slist;          // K1 lists its solved blocks for the TMA consensus pass (solved_list)
    uint64_t *trace_hash;   // audit mode: per-iteration state digests (may be null)
    int64_t hash_base;      // global index of the first pixel (shards)
    int32_t shard_index, shard_count;   // sharded: this shard's slot in the agg table
    astore_t *ga_up, *ga_dn;            // sharded: multipliers of the ghost rows / planes
    uint32_t *dlist;        // run loop: two dirty-block worklists (dirty_list), else null
    const dope_peers *peers;  // peer-memory exchange (sharded), else null
    uint32_t *pflags;       // peer mode: this shard's flags [row from above, row from below,
                            // K1 done-counter, pad, agg-slot flag per shard]
    int32_t ovl;            // run loop: the consensus pass overlaps K1 (k1_publish_done, PDL launch)
    uint32_t *kdone;        // overlap mode: iteration + 1 of each block's last FINISHED solve
    uint32_t *kq;           // TMA consensus pass: queue of tile-work blocks (4 words each, K
                            // entries) + [length, claims, CTAs done], or null
};

// ---------------------------------------------------------------------------
// K1 -> consensus overlap (run loop, TMA consensus pass): K1 CTAs write their
// block's dirty-flag clear, solve epoch and solved-list slot, fence, and only
// then trigger the dependent launch, so the consensus pass starts with the
// iteration's solved set fixed; each solving CTA publishes its labels with a
// release store of the block's done epoch, which the consensus producer
// acquires before it streams the block's (or a neighbour's) labels.
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint32_t ld_acquire_gpu(const uint32_t *p) {
    uint32_t v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_release_gpu(uint32_t *p, uint32_t v) {
    asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
// K1 epilogue: every thread's label / residual stores precede the flag (the
// barrier orders them before thread 0's cumulative release)
__device__ __forceinline__ void k1_publish_done(const Lat2 &L, int k) {
    __syncthreads();
    if (threadIdx.x == 0) st_release_gpu(L.kdone + k, (uint32_t)L.st->iteration + 1u);
}

// ---------------------------------------------------------------------------
// Peer-memory exchange (dope_peers): system-scope release / acquire flags.
// Epochs carry the run generation so flags left by an earlier run never match.
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint32_t ld_acquire_sys(const uint32_t *p) {
    uint32_t v;
    asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_release_sys(uint32_t *p, uint32_t v) {
    asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void wait_flag(const uint32_t *p, uint32_t v) {
    while (ld_acquire_sys(p) != v) __nanosleep(100);
}
__device__ __forceinline__ uint32_t peer_epoch(const dope_run_state *st, uint32_t step) {
    return ((uint32_t)st->generation << 16) + step;
}

// Dirty-block worklists of the run loop (dirty[9K, 11K + 2)): list p = [count,
// K entries]; the consensus pass of iteration t appends every block it marks
// dirty (first mark only) to list (t + 1) & 1, which K1 of iteration t + 1
// deals out first-come: CTA i solves entry i, so every block that needs a
// solve starts in the first wave instead of wherever its id puts it among the
// K mostly-clean CTAs.  K1 resets the other list for the next pass.
__device__ __forceinline__ uint32_t *dirty_list(const Lat2 &L, int parity) {
    return L.dlist + (size_t)(parity & 1) * (L.K + 1);
}

// Mark block k dirty for the next iteration (and list it, run loop).
__device__ __forceinline__ void mark_dirty(const Lat2 &L, int64_t k) {
    DOPE_ASSERT(k >= 0 && k < L.K);
    if (!L.dlist) {
        L.dirty[k] = 1u;
        return;
    }
    if (atomicExch(&L.dirty[k], 1u) == 0u) {
        uint32_t *lst = dirty_list(L, L.st->iteration + 1);
        const uint32_t slot = atomicAdd(lst, 1u);
        if (slot < (uint32_t)L.K) lst[1 + slot] = (uint32_t)k;
    }
}

// Sharded mode: the halo buffer's layout is in common.cuh (halo_bytes).


// agg table of the sharded run loop: AGG_SLOT int64 per shard, filled by each
// shard's consensus pass (and end-of-run energy), gathered across shards
// before dope_decide: [0] energy of y_{t-1}, [1] sum of block ss, [2] sum of
// the residual excesses (rsq_excess), [3] max block ss, [4] clamp flag,
// [5] end-of-run energy of the last iterate.
constexpr int AGG_SLOT = 8;

// Peer mode, every K1 CTA on its way out (CTA-uniform call): the last CTA of
// the grid pushes this shard's first / last row of labels into the
// neighbours' halo slots and raises their row flags (epoch = this iteration).
__device__ __noinline__ void k1_peer_exit_impl(uint32_t *pflags, const dope_peers *pr, const uint8_t *yhat,
                                               const dope_run_state *st, int64_t P, int64_t lastoff) {
    // (plain arguments: a `const Lat2 &` would force the caller's whole
    // parameter block into local memory)
    __shared__ int last;
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        last = atomicAdd(&pflags[2], 1u) == gridDim.x - 1;
    }
    __syncthreads();
    if (!last) return;
    __threadfence();
    uint8_t *up = pr->row_to_up, *dn = pr->row_to_dn;
    for (int64_t c = threadIdx.x; c < P; c += blockDim.x) {
        if (up) up[c] = yhat[c];
        if (dn) dn[c] = yhat[lastoff + c];
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence_system();
        const uint32_t ep = peer_epoch(st, (uint32_t)st->iteration + 1u);
        if (up) st_release_sys(pr->flag_to_up, ep);
        if (dn) st_release_sys(pr->flag_to_dn, ep);
        pflags[2] = 0u;
    }
}
__device__ __forceinline__ void k1_peer_exit(const Lat2 &L) {
    const int64_t P = L.ndim == 3 ? (int64_t)L.ay.dim * L.W : (int64_t)L.W;
    const int64_t lastoff = ((L.ndim == 3 ? (int64_t)L.az.dim : (int64_t)L.ay.dim) - 1) * P;
    k1_peer_exit_impl(L.pflags, L.peers, L.yhat, L.st, P, lastoff);
}

// Append block k to the solved-block list (see solved_list); dirty[8K + k] =
// 1 + the block's latest slot.
__device__ __forceinline__ void solved_append(const Lat2 &L, int k) {
    const uint32_t slot = (uint32_t)atomicAdd(reinterpret_cast<unsigned long long *>(&L.pc[6]), 1ull);
    if (slot < (uint32_t)L.K) {
        L.dirty[(size_t)7 * L.K + slot] = (uint32_t)k;
        L.dirty[(size_t)8 * L.K + k] = slot + 1u;
    }
}

// ---------------------------------------------------------------------------
// K1: block min-cut (2D, 4-connected)
// ---------------------------------------------------------------------------

// Warp-level compaction (K1 sweeps): the lanes whose bit is set in `word`
// (node v of lane i) join the warp's batch slots[0..cnt); every full batch of
// 32 runs work(node), one node per lane.  Returns the new batch fill.
__device__ __forceinline__ uint32_t lanemask_lt() {
    uint32_t m;
    asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
    return m;
}
template <class F>
__device__ __forceinline__ int warp_enqueue(uint16_t *slots, uint32_t word, int cnt, int lane, int v, F &&work) {
    while (word) {
        const bool mine = (word >> lane) & 1u;
        const int rank = __popc(word & lanemask_lt());
        const int room = 32 - cnt;
        if (mine && rank < room) slots[cnt + rank] = (uint16_t)v;
        const int n = __popc(word);
        word = __ballot_sync(FULLMASK, mine && rank >= room);
        if (n >= room) {
            __syncwarp();
            work((int)slots[lane]);
            __syncwarp();
            cnt = 0;
        } else {
            cnt += n;
        }
    }
    return cnt;
}

// 4 bytes -> 4 bits: bit j set iff byte j is nonzero
__device__ __forceinline__ uint32_t nz_bits4(uint32_t x) {
    const uint32_t t = (((x & 0x7F7F7F7Fu) + 0x7F7F7F7Fu) | x) & 0x80808080u;
    return ((t >> 7) * 0x00204081u) >> 21 & 0xFu;
}

template <int BH, int BW, int NT>
struct K1Cfg {
    static constexpr int M = BH * BW;
    static_assert(M % NT == 0, "nodes per thread");
    static_assert(M % 64 == 0, "bit words");
    static constexpr int NPT = M / NT;
    static constexpr int NW = M / 64;
    static constexpr size_t OFF_G = 0;                       // int32[M]
    static constexpr size_t OFF_R = OFF_G + 4 * (size_t)M;   // uint8[4][M]  (E,W,S,N)
    static constexpr size_t OFF_H = OFF_R + 4 * (size_t)M;   // uint16[M]
    static constexpr size_t OFF_MASK = OFF_H + 2 * (size_t)M;  // uint64[6][NW]
    static constexpr size_t OFF_REACH = OFF_MASK + 6 * 8 * (size_t)NW;
    static constexpr size_t OFF_MISC = OFF_REACH + 8 * (size_t)NW;
    static constexpr size_t SMEM = OFF_MISC + 64;
};

struct K1Tune {
    int32_t sweep_min, sweep_mul;   // sweeps per round = sweep_min + sweep_mul*levels
    int32_t max_rounds;
    int32_t dense_min, dense_mul;   // the same for dense rounds (most nodes active: cold solves)
};

// resident CTAs per SM the register allocation must allow for the 256-thread
// 64x64 kernel: 5 (= its shared-memory limit; 48 registers, measured on C3
// against 4 and unbounded)
#ifndef K1_MINB
#define K1_MINB 5
#endif
#ifndef K1_MINB128
#define K1_MINB128 1
#endif
#ifndef K1_MINB64
#define K1_MINB64 1
#endif
// 64x64 with 512 threads (the wide variant): 2 CTAs/SM (68 registers would
// leave one -- C5 b64 K1 18.9 vs 21.3 us)
#define K1_MINB_OF(bh, nt)                                                                                \
    ((bh) == 64 && (nt) == 512 ? 2                                                                        \
                               : ((nt) == 256 ? K1_MINB : ((nt) == 128 ? K1_MINB128 : ((nt) == 64 ? K1_MINB64 : 1))))
// One block's solve (K1 body): prologue, rounds of (BFS, sweeps), epilogue.
template <int BH, int BW, int NT>
__device__ __forceinline__ void k1_body(const Lat2 &L, const K1Tune &T, int k, int ycur, bool last,
                                        uint64_t t_begin) {
    using C = K1Cfg<BH, BW, NT>;
    constexpr int M = C::M, NPT = C::NPT, NW = C::NW;
    extern __shared__ __align__(16) uint8_t smem[];
    int32_t *g = reinterpret_cast<int32_t *>(smem + C::OFF_G);
    uint8_t *rr = smem + C::OFF_R;
    uint16_t *h = reinterpret_cast<uint16_t *>(smem + C::OFF_H);
    uint64_t *masks = reinterpret_cast<uint64_t *>(smem + C::OFF_MASK);
    uint64_t *reach = reinterpret_cast<uint64_t *>(smem + C::OFF_REACH);
    int *misc = reinterpret_cast<int *>(smem + C::OFF_MISC);
    uint32_t *masks32 = reinterpret_cast<uint32_t *>(masks);
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    __syncthreads();
    if (L.timeline && tid == 0) {
        L.timeline[8 * k + 0] = (int64_t)t_begin;
        L.timeline[8 * k + 1] = (int64_t)t_begin;
        L.timeline[8 * k + 2] = -1;
        L.timeline[8 * k + 3] = 0;
        L.timeline[8 * k + 4] = (int64_t)t_begin;
        L.timeline[8 * k + 5] = (int64_t)t_begin;
    }
    if (tid == 0) {
        L.dirty[k] = 0;
        const uint32_t ep = (uint32_t)L.st->iteration + 1u;
        L.dirty[L.K + k] = ep;   // solve epoch (consensus fast path)
        if (L.slist) solved_append(L, k);
        if (L.ovl && last) __threadfence();   // the consensus pass may start once every CTA triggered
    }
    // (a CTA triggers when all its threads did: thread 0 after its fence; a
    // worklist CTA at its last block)
    if (L.ovl && last) griddep_launch();

    const int by = k / L.ax.k, bx = k % L.ax.k;
    int32_t lo_r, hr, lo_c, wc;
    L.ay.range(by, lo_r, hr);
    L.ax.range(bx, lo_c, wc);
    const int32_t Wg = L.W;
    const int32_t cap = L.cap;
    const astore_t *__restrict__ a_cur = L.a;
    const ystore_t *__restrict__ y_cur = L.y2[ycur];
    // stored residual graph: E and S planes only (the W / N residual of an
    // arc pair is 2*cap minus the forward one: r(v->w) + r(w->v) = 2*cap)
    uint8_t *gres = L.resid + (size_t)k * 2 * M;

    // ---- prologue: 2*linear (blockform.py:103-104 on the q==1 stencil) ----
    // lin2 = 2u + lamw * sum_cross (y2_g - y2_j) + mu*(2a - y2_g) + mu
    if (L.warm) {
        // E and S residual planes (block-major, 2*M bytes): asynchronous
        // 16-byte copies into shared planes 0 (E) and 2 (S)
        for (int i = tid; i < M * 2 / 16; i += NT) {
            const int so = (i < M / 16) ? 16 * i : 2 * M + 16 * (i - M / 16);
            asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(
                             (uint32_t)__cvta_generic_to_shared(rr + so)),
                         "l"(gres + 16 * i)
                         : "memory");
        }
        asm volatile("cp.async.commit_group;" ::: "memory");
    }
    const bool has_up = lo_r > 0 || L.gup, has_dn = lo_r + hr < L.ay.dim || L.gdn, has_lf = lo_c > 0,
               has_rt = lo_c + wc < Wg;
    if (L.vec4) {
        // quads of 4 consecutive box nodes: int4 of u, 8 B of a, 4 B of y2
        // every quad of this thread in one batch of loads (one round trip)
        constexpr int NQ = M / 4;
        constexpr int QU = (NQ / NT) < 1 ? 1 : ((NQ / NT) > 4 ? 4 : (NQ / NT));
        for (int q0 = tid; q0 < NQ; q0 += QU * NT) {
            int4 uq[QU];
            uint2 aq[QU];
            uint32_t yq[QU], yu[QU], yd[QU];
            int yl[QU], yrr[QU];
            bool ok[QU];
#pragma unroll
            for (int j = 0; j < QU; ++j) {
                const int qd = q0 + j * NT;
                const int v0 = 4 * qd, r = v0 / BW, c0 = v0 % BW;
                ok[j] = qd < NQ && r < hr && c0 < wc;
                uq[j] = make_int4(0, 0, 0, 0);
                aq[j] = make_uint2(0, 0);
                yq[j] = yu[j] = yd[j] = 0;
                yl[j] = yrr[j] = 0;
                if (ok[j]) {
                    const int64_t G = (int64_t)(lo_r + r) * Wg + lo_c + c0;
                    DOPE_ASSERT(G >= 0 && G + 4 <= (int64_t)L.ay.dim * Wg);
                    uq[j] = __ldg(reinterpret_cast<const int4 *>(L.u + G));
                    aq[j] = *reinterpret_cast<const uint2 *>(a_cur + G);
                    yq[j] = *reinterpret_cast<const uint32_t *>(y_cur + G);
                    if (r == 0 && has_up) yu[j] = *reinterpret_cast<const uint32_t *>(y_cur + G - Wg);
                    if (r == hr - 1 && has_dn) yd[j] = *reinterpret_cast<const uint32_t *>(y_cur + G + Wg);
                    if (c0 == 0 && has_lf) yl[j] = y_cur[G - 1];
                    if (c0 + 4 == wc && has_rt) yrr[j] = y_cur[G + 4];
                }
            }
#pragma unroll
            for (int j = 0; j < QU; ++j) {
                const int qd = q0 + j * NT;
                if (qd >= NQ) continue;
                const int v0 = 4 * qd, r = v0 / BW, c0 = v0 % BW;
                int4 out = make_int4(0, 0, 0, 0);
                if (ok[j]) {
                    const bool top = r == 0 && has_up, bot = r == hr - 1 && has_dn;
                    const int uv[4] = {uq[j].x, uq[j].y, uq[j].z, uq[j].w};
                    int av[4];
                    unpack_a4(aq[j], av);
                    int lin[4];
#pragma unroll
                    for (int e = 0; e < 4; ++e) {
                        const int yv = byte_at(yq[j], e);
                        int sx = 0;
                        if (top) sx += yv - byte_at(yu[j], e);
                        if (bot) sx += yv - byte_at(yd[j], e);
                        if (e == 0 && c0 == 0 && has_lf) sx += yv - yl[j];
                        if (e == 3 && c0 + 4 == wc && has_rt) sx += yv - yrr[j];
                        lin[e] = 2 * uv[e] + L.lamw * sx + L.mu * (2 * av[e] - yv) + L.mu;
                    }
                    out = make_int4(lin[0], lin[1], lin[2], lin[3]);
                }
                *reinterpret_cast<int4 *>(g + v0) = out;
            }
        }
    } else {
        for (int i = 0; i < NPT; ++i) {
            const int v = tid + i * NT;
            const int r = v / BW, c = v % BW;
            int32_t lin2 = 0;
            if (r < hr && c < wc) {
                const int64_t G = (int64_t)(lo_r + r) * Wg + lo_c + c;
                const int32_t yg = y_cur[G];
                int32_t sx = 0;
                if (c == 0 && has_lf) sx += yg - (int32_t)y_cur[G - 1];
                if (c == wc - 1 && has_rt) sx += yg - (int32_t)y_cur[G + 1];
                if (r == 0 && has_up) sx += yg - (int32_t)y_cur[G - Wg];
                if (r == hr - 1 && has_dn) sx += yg - (int32_t)y_cur[G + Wg];
                lin2 = 2 * L.u[G] + L.lamw * sx + L.mu * (2 * (int32_t)a_cur[G] - yg) + L.mu;
            }
            g[v] = lin2;
        }
    }
    if (L.warm) asm volatile("cp.async.wait_all;" ::: "memory");
    __syncthreads();
    if (L.timeline && tid == 0) {   // diagnostics: prologue loads done
        uint64_t t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        L.timeline[8 * k + 7] = (int64_t)t;
    }
    // g = lin2 + net inflow of the stored flow (warm) / cold residual graph
    if (L.warm) {
        // quads of 4 nodes: W = 2cap - E(west), N = 2cap - S(north) bytewise
        // (no borrow: every residual is <= 2cap), node sums in 16-bit lanes
        const uint32_t CAP2 = 0x01010101u * (uint32_t)(2 * cap);
        for (int q = tid; q < M / 4; q += NT) {
            const int v0 = 4 * q, r = v0 / BW, c0 = v0 % BW;
            const int nv = r < hr ? wc - c0 : 0;                   // valid nodes in this quad
            const uint32_t vm = nv >= 4 ? 0xFFFFFFFFu : (nv <= 0 ? 0u : (0xFFFFFFFFu >> (8 * (4 - nv))));
            const uint32_t E = *reinterpret_cast<const uint32_t *>(rr + v0);
            const uint32_t S = *reinterpret_cast<const uint32_t *>(rr + 2 * M + v0);
            const uint32_t ep = c0 > 0 ? (uint32_t)rr[v0 - 1] : 0u;
            const uint32_t W = (CAP2 - ((E << 8) | ep)) & vm & (c0 == 0 ? 0xFFFFFF00u : 0xFFFFFFFFu);
            const uint32_t N = r > 0 ? (CAP2 - *reinterpret_cast<const uint32_t *>(rr + 2 * M + v0 - BW)) & vm : 0u;
            *reinterpret_cast<uint32_t *>(rr + 1 * M + v0) = W;
            *reinterpret_cast<uint32_t *>(rr + 3 * M + v0) = N;
            const uint32_t lo = (E & 0x00FF00FFu) + (W & 0x00FF00FFu) + (S & 0x00FF00FFu) + (N & 0x00FF00FFu);
            const uint32_t hi = ((E >> 8) & 0x00FF00FFu) + ((W >> 8) & 0x00FF00FFu) + ((S >> 8) & 0x00FF00FFu) +
                                ((N >> 8) & 0x00FF00FFu);
            const int vert = (r > 0) + (r + 1 < hr);
            int4 gv = *reinterpret_cast<const int4 *>(g + v0);
            // arcs per node: E if c+1 < wc, W if c > 0, plus the vertical ones
            auto deg = [&](int c) { return (c < wc) ? (vert + (c > 0) + (c + 1 < wc)) : 0; };
            gv.x += (int)(lo & 0xFFFFu) - cap * deg(c0);
            gv.y += (int)(hi & 0xFFFFu) - cap * deg(c0 + 1);
            gv.z += (int)(lo >> 16) - cap * deg(c0 + 2);
            gv.w += (int)(hi >> 16) - cap * deg(c0 + 3);
            if (nv > 0) *reinterpret_cast<int4 *>(g + v0) = gv;
        }
    } else
    for (int i = 0; i < NPT; ++i) {
        const int v = tid + i * NT;
        const int r = v / BW, c = v % BW;
        if (!(r < hr && c < wc)) {
            rr[0 * M + v] = 0;
            rr[1 * M + v] = 0;
            rr[2 * M + v] = 0;
            rr[3 * M + v] = 0;
            continue;
        }
        const bool hasE = c + 1 < wc, hasW = c > 0, hasS = r + 1 < hr, hasN = r > 0;
        if (L.warm) {
            const int32_t rE = hasE ? rr[0 * M + v] : cap, rS = hasS ? rr[2 * M + v] : cap;
            const int32_t rW = hasW ? 2 * cap - rr[0 * M + v - 1] : cap;
            const int32_t rN = hasN ? 2 * cap - rr[2 * M + v - BW] : cap;
            rr[1 * M + v] = hasW ? (uint8_t)rW : 0;
            rr[3 * M + v] = hasN ? (uint8_t)rN : 0;
            g[v] += (rE - cap) + (rW - cap) + (rS - cap) + (rN - cap);
        } else {
            rr[0 * M + v] = hasE ? cap : 0;
            rr[1 * M + v] = hasW ? cap : 0;
            rr[2 * M + v] = hasS ? cap : 0;
            rr[3 * M + v] = hasN ? cap : 0;
        }
    }
    __syncthreads();

    if (L.timeline && tid == 0) {
        uint64_t t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        L.timeline[8 * k + 4] = (int64_t)t;
    }
    // ---- solve: rounds of (global relabel BFS, push/relabel sweeps) ----
#ifdef K1_DIAG2
    __shared__ long long dclk[3][5];   // per sweep of round 1: start, push done, barrier, relabel done, end
    __shared__ int dnp[3];
    if (tid == 0)
        for (int i = 0; i < 15; ++i) dclk[i / 5][i % 5] = 0;
#endif
    uint64_t t_bfs = 0;   // diagnostics (timeline mode, thread 0): last BFS start and levels
    int lev_last = 0;
    int rounds = 0;
    long long sweeps_done = 0;
    for (;;) {
        if (L.timeline && tid == 0)   // diagnostics: this round's BFS start
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_bfs));
#ifdef K1_DIAG2
        long long c_r0 = clock64(), c_r1 = 0;
#endif
        // residual masks: one (direction, 32-node group) word per thread
        // step, from the group's 32 residual bytes (nonzero bytes -> bits)
        for (int p = tid; p < 4 * 2 * NW; p += NT) {
            const int d = p / (2 * NW), w = p - d * (2 * NW);
            const uint4 *src = reinterpret_cast<const uint4 *>(rr + d * M + 32 * w);
            const uint4 x0 = src[0], x1 = src[1];
            masks32[p] = nz_bits4(x0.x) | nz_bits4(x0.y) << 4 | nz_bits4(x0.z) << 8 | nz_bits4(x0.w) << 12 |
                         nz_bits4(x1.x) << 16 | nz_bits4(x1.y) << 20 | nz_bits4(x1.z) << 24 | nz_bits4(x1.w) << 28;
        }
        // sink / active masks (ballots: warp covers 32 consecutive nodes per step)
#pragma unroll 2
        for (int i = 0; i < NPT; ++i) {
            const int v = tid + i * NT;
            const int32_t gv = g[v];
            const uint32_t bK = __ballot_sync(FULLMASK, gv < 0);
            const uint32_t bA = __ballot_sync(FULLMASK, gv > 0);
            h[v] = gv < 0 ? 0 : HINF;          // sink set: level 0 (BFS skips them)
            if (lane == 0) {
                const int w32 = (i * NT + warp * 32) >> 5;
                masks32[4 * 2 * NW + w32] = bK;
                masks32[5 * 2 * NW + w32] = bA;
            }
        }
        __syncthreads();
#ifdef K1_DIAG2
        c_r1 = clock64();
#endif
        if (warp == 0) {
            int levels = 0;
            const int hit = bfs_relabel<NW, BW, 0>(masks, reach, h, lane, &levels);
            if (lane == 0) { misc[0] = hit; misc[1] = levels; }
        }
        __syncthreads();
        const int hit = misc[0];
        const int levels = misc[1];
#ifdef K1_DIAG2
        if (tid == 0) {   // [8K + 8k + 6 / 7]: first / last round's (mask build, BFS) cycles
            const long long c_r2 = clock64();
            const long long v = ((c_r1 - c_r0) & 0xFFFFF) | (((c_r2 - c_r1) & 0xFFFFF) << 20) | ((long long)levels << 40);
            if (L.timeline) L.timeline[8 * (size_t)L.K + 8 * k + (rounds == 0 ? 6 : 7)] = v;
        }
#endif
        if (L.timeline && tid == 0 && rounds == 0) {
            uint64_t t;
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
            L.timeline[8 * k + 5] = (int64_t)t;
            int nact = 0;   // active nodes at the first BFS
            for (int w = 0; w < 2 * NW; ++w) nact += __popc(masks32[5 * 2 * NW + w]);
            L.timeline[8 * k + 6] = levels | ((int64_t)nact << 16);
        }
        if (L.timeline && tid == 0) lev_last = levels;
        if (!hit) break;
        if (++rounds > T.max_rounds) {
            if (tid == 0) atomicCAS(&L.st->error, 0, k + 1);
            break;
        }
        int cap_sweeps = T.sweep_min + T.sweep_mul * levels;
        // The sweeps visit only candidate nodes, kept as bitmasks in the BFS
        // scratch (both rebuilt by the next BFS): C = nodes to push from
        // (initially the active nodes the BFS reached: reach & active), N =
        // nodes to relabel (pushers left with excess, nodes that received
        // some).  A warp owns the 32-node groups of its lanes (the BFS mask
        // layout: group i of warp w = 32-bit word i * NT / 32 + w); it reads
        // its group words in one load per lane and compacts the set bits
        // into batches of 32, one node per lane, in a slot row.  Warm solves
        // move little excess: a straggler's sweeps typically push from a
        // handful of nodes, where a scan of every node's g and h cost
        // ~1000-3000 cycles per phase (tools/mb_scan.cu, tools/k1_stragglers.py).
        uint32_t *candC = reinterpret_cast<uint32_t *>(reach);          // 2 * NW words
        uint32_t *candN = masks32;                                       // 2 * NW words
        uint16_t *slots = reinterpret_cast<uint16_t *>(masks32 + 2 * NW) + warp * 32;
        static_assert(8 * NW + (NT / 32) * 64 <= 6 * 8 * NW, "candidate masks and slots fit the BFS masks");
        // Dense rounds (cold solves: most nodes active) sweep every node as
        // plain loops -- the candidate bookkeeping would only add atomics.
        if (tid == 0) misc[2] = 0;
        __syncthreads();
        {
            int myc = 0;
            for (int w = tid; w < 2 * NW; w += NT) {   // reach & active
                const uint32_t c = candC[w] & masks32[5 * 2 * NW + w];
                candC[w] = c;
                myc += __popc(c);
            }
            if (myc) atomicAdd(&misc[2], myc);
        }
        __syncthreads();
        if (misc[2] > M / 16) {
            cap_sweeps = T.dense_min + T.dense_mul * levels;
            for (int sw = 0; sw < cap_sweeps; ++sw) {
                ++sweeps_done;
                // push phase: admissible arcs h(w) == h(v) - 1
#pragma unroll 2
                for (int i = 0; i < NPT; ++i) {
                    const int v = tid + i * NT;
                    const int32_t e = g[v];
                    if (e <= 0) continue;
                    const uint16_t hv = h[v];
                    if (hv == HINF || hv == 0) continue;
                    const uint16_t ht = hv - 1;
                    int32_t left = e;
#pragma unroll
                    for (int d = 0; d < 4; ++d) {
                        const int off = (d == 0) ? 1 : (d == 1) ? -1 : (d == 2) ? BW : -BW;
                        const int32_t rv = rr[d * M + v];
                        if (rv == 0) continue;
                        const int w = v + off;
                        if (h[w] != ht) continue;
                        const int32_t delta = left < rv ? left : rv;
                        DOPE_ASSERT(w >= 0 && w < M && delta > 0 && rv <= 2 * cap &&
                                    rr[(d ^ 1) * M + w] + delta <= 2 * cap);   // r + r' = 2 cap per arc pair
                        rr[d * M + v] = (uint8_t)(rv - delta);
                        rr[(d ^ 1) * M + w] = (uint8_t)(rr[(d ^ 1) * M + w] + delta);
                        atomicAdd(&g[w], delta);
                        left -= delta;
                        if (left == 0) break;
                    }
                    if (left != e) atomicSub(&g[v], e - left);
                }
                __syncthreads();
                // relabel phase: h(v) = 1 + min over residual arcs (monotone)
                int act = 0;
#pragma unroll 2
                for (int i = 0; i < NPT; ++i) {
                    const int v = tid + i * NT;
                    if (g[v] <= 0) continue;
                    const uint16_t hv = h[v];
                    if (hv == HINF) continue;
                    uint32_t mn = HINF;
#pragma unroll
                    for (int d = 0; d < 4; ++d) {
                        const int off = (d == 0) ? 1 : (d == 1) ? -1 : (d == 2) ? BW : -BW;
                        if (rr[d * M + v] == 0) continue;
                        const uint32_t hw = h[v + off];
                        mn = hw < mn ? hw : mn;
                    }
                    const uint32_t nh = (mn + 1 >= (uint32_t)M) ? HINF : mn + 1;
                    if (nh != hv) h[v] = (uint16_t)nh;
                    act |= (nh != HINF);
                }
                if (!__syncthreads_or(act)) break;
            }
            continue;   // next round: global relabel
        }
        for (int w = tid; w < 2 * NW; w += NT) candN[w] = 0u;
        __syncthreads();
        for (int sw = 0; sw < cap_sweeps; ++sw) {
            ++sweeps_done;
#ifdef K1_DIAG2
            int npush = 0;
            if (tid == 0 && rounds == 1 && sw < 3) dclk[sw][0] = clock64();
#endif
            int act = 0;
#pragma unroll 1
            for (int phase = 0; phase < 2; ++phase) {   // 0: push from C, 1: relabel N
                uint32_t *cand = phase == 0 ? candC : candN;
                // this warp's group words (lane j: group j), taken and cleared
                uint32_t gw = 0;
                if (lane < NPT) {
                    const int wi = lane * (NT / 32) + warp;
                    gw = cand[wi];
                    if (gw) cand[wi] = 0u;
                }
                uint32_t groups = __ballot_sync(FULLMASK, gw != 0u);
                int cnt = 0;
                while (groups || cnt) {
                    const int i = groups ? __ffs(groups) - 1 : 0;
                    uint32_t word = groups ? __shfl_sync(FULLMASK, gw, i) : 0u;
                    if (groups) groups &= groups - 1;
                    const int v = i * NT + warp * 32 + lane;
                    const bool tail = groups == 0u;
                    while (word || (tail && cnt)) {
                        const bool mine = (word >> lane) & 1u;
                        const int rank = __popc(word & lanemask_lt());
                        const int room = 32 - cnt;
                        if (mine && rank < room) slots[cnt + rank] = (uint16_t)v;
                        const int nw = __popc(word);
                        word = __ballot_sync(FULLMASK, mine && rank >= room);
                        const int fill = cnt + (nw < room ? nw : room);
                        if (fill < 32 && !(tail && word == 0u)) {
                            cnt = fill;
                            continue;
                        }
                        // a full batch (or the last one): one node per lane
                        __syncwarp();
                        if (lane < fill) {
                            const int u = slots[lane];
                            const int32_t e = g[u];
                            const uint16_t hu = h[u];
                            if (phase == 0) {
                                if (e > 0 && hu != HINF) {
#ifdef K1_DIAG2
                                    ++npush;
#endif
                                    int32_t left = e;
                                    if (hu != 0) {
                                        // push along the admissible arcs h(w) == h(u) - 1
                                        const uint16_t ht = hu - 1;
#pragma unroll
                                        for (int d = 0; d < 4; ++d) {
                                            const int off = (d == 0) ? 1 : (d == 1) ? -1 : (d == 2) ? BW : -BW;
                                            const int32_t rv = rr[d * M + u];
                                            if (rv == 0) continue;
                                            const int w = u + off;
                                            if (h[w] != ht) continue;
                                            const int32_t delta = left < rv ? left : rv;
                                            DOPE_ASSERT(w >= 0 && w < M && delta > 0 && rv <= 2 * cap &&
                                                        rr[(d ^ 1) * M + w] + delta <= 2 * cap);   // r + r' = 2 cap
                                            rr[d * M + u] = (uint8_t)(rv - delta);
                                            rr[(d ^ 1) * M + w] = (uint8_t)(rr[(d ^ 1) * M + w] + delta);
                                            atomicAdd(&g[w], delta);
                                            atomicOr(&candN[w >> 5], 1u << (w & 31));   // w may turn active
                                            left -= delta;
                                            if (left == 0) break;
                                        }
                                        if (left != e) atomicSub(&g[u], e - left);
                                    }
                                    if (left > 0) atomicOr(&candN[u >> 5], 1u << (u & 31));
                                }
                            } else if (e > 0 && hu != HINF) {
                                // h(u) = 1 + min over residual arcs (monotone)
                                uint32_t mn = HINF;
#pragma unroll
                                for (int d = 0; d < 4; ++d) {
                                    const int off = (d == 0) ? 1 : (d == 1) ? -1 : (d == 2) ? BW : -BW;
                                    if (rr[d * M + u] == 0) continue;
                                    const uint32_t hw = h[u + off];
                                    mn = hw < mn ? hw : mn;
                                }
                                const uint32_t nh = (mn + 1 >= (uint32_t)M) ? HINF : mn + 1;
                                if (nh != hu) h[u] = (uint16_t)nh;
                                if (nh != HINF) {   // pushes next sweep
                                    act = 1;
                                    atomicOr(&candC[u >> 5], 1u << (u & 31));
                                }
                            }
                        }
                        __syncwarp();
                        cnt = 0;
                    }
                }
#ifdef K1_DIAG2
                if (tid == 0 && rounds == 1 && sw < 3) dclk[sw][1 + 2 * phase] = clock64();
#endif
                if (phase == 0) {
                    __syncthreads();
#ifdef K1_DIAG2
                    if (tid == 0 && rounds == 1 && sw < 3) dclk[sw][2] = clock64();
                    {
                        const int np = __syncthreads_count(npush);
                        if (tid == 0 && rounds == 1 && sw < 3) dnp[sw] = np;
                    }
#endif
                }
            }
#ifdef K1_DIAG2
            if (tid == 0 && rounds == 1 && sw < 3) dclk[sw][4] = clock64();
#endif
            if (!__syncthreads_or(act)) break;
        }
    }

    // ---- epilogue: labels (sink side), residual graph, stats ----
    if (L.vec4) {   // 4 labels per 32-bit store (quads never straddle the block edge)
        for (int q = tid; q < M / 4; q += NT) {
            const int v0 = 4 * q, r = v0 / BW, c0 = v0 % BW;
            if (r < hr && c0 < wc) {
                const uint32_t b = (uint32_t)(reach[v0 >> 6] >> (v0 & 63)) & 0xFu;
                const int64_t G = (int64_t)(lo_r + r) * Wg + lo_c + c0;
                DOPE_ASSERT(G >= 0 && G + 4 <= (int64_t)L.ay.dim * Wg);
                *reinterpret_cast<uint32_t *>(L.yhat + G) = (b * 0x00204081u) & 0x01010101u;
            }
        }
    } else {
        for (int i = 0; i < NPT; ++i) {
            const int v = tid + i * NT;
            const int r = v / BW, c = v % BW;
            if (r < hr && c < wc) {
                const int64_t G = (int64_t)(lo_r + r) * Wg + lo_c + c;
                L.yhat[G] = (uint8_t)((reach[v >> 6] >> (v & 63)) & 1ull);
            }
        }
    }
    if (L.warm && sweeps_done > 0) {   // E and S planes back (unchanged when nothing was pushed)
        uint4 *dst = reinterpret_cast<uint4 *>(gres);
        for (int i = tid; i < M * 2 / 16; i += NT) {
            const int so = (i < M / 16) ? 16 * i : 2 * M + 16 * (i - M / 16);
            dst[i] = *reinterpret_cast<const uint4 *>(rr + so);
        }
    }
    if (tid == 0 && L.timeline) {
        uint64_t t_end;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_end));
        L.timeline[8 * k + 1] = (int64_t)t_end;
        // rounds | levels of the last BFS << 16; sweeps | (last BFS start - CTA start, ns) << 24
        L.timeline[8 * k + 2] = rounds | ((int64_t)lev_last << 16);
        L.timeline[8 * k + 3] = sweeps_done | ((int64_t)(t_bfs - t_begin) << 24);
    }
#ifdef K1_DIAG2
    // [8K + 8k + j]: sweep j < 3 of round 1: (push scan+work, barrier, relabel, end) cycles in 16-bit
    // fields, pushers in bits 48..63
    if (tid == 0 && L.timeline)
        for (int j = 0; j < 3; ++j) {
            const long long c0 = dclk[j][0];
            const auto f = [&](int i) { return (long long)((dclk[j][i] - dclk[j][i - 1]) & 0xFFFF); };
            L.timeline[8 * (size_t)L.K + 8 * k + j] =
                c0 ? (f(1) | f(2) << 16 | f(3) << 32 | (long long)(dnp[j] & 0x7FFF) << 48) : 0;
            L.timeline[8 * (size_t)L.K + 8 * k + 3 + j] = c0 ? (dclk[j][4] - dclk[j][3]) : 0;
        }
#endif
    if (tid == 0) {
        atomicAdd((unsigned long long *)&L.st->solves, 1ull);
        atomicAdd((unsigned long long *)&L.st->sweeps, (unsigned long long)sweeps_done);
        atomicMax(&L.st->max_rounds_seen, rounds);
    }
    if (L.ovl) k1_publish_done(L, k);
}


template <int BH, int BW, int NT>
__global__ void __launch_bounds__(NT, (K1_MINB_OF(BH, NT))) k_block_mincut(Lat2 L, K1Tune T) {
    using C = K1Cfg<BH, BW, NT>;
    constexpr int M = C::M, NPT = C::NPT, NW = C::NW;
    extern __shared__ __align__(16) uint8_t smem[];
    int32_t *g = reinterpret_cast<int32_t *>(smem + C::OFF_G);
    uint8_t *rr = smem + C::OFF_R;
    uint16_t *h = reinterpret_cast<uint16_t *>(smem + C::OFF_H);
    uint64_t *masks = reinterpret_cast<uint64_t *>(smem + C::OFF_MASK);
    uint64_t *reach = reinterpret_cast<uint64_t *>(smem + C::OFF_REACH);
    int *misc = reinterpret_cast<int *>(smem + C::OFF_MISC);
    uint32_t *masks32 = reinterpret_cast<uint32_t *>(masks);

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    int k = blockIdx.x;
    uint64_t t_begin = 0;   // diagnostics: CTA start (recorded once the block is known)
    if (L.timeline && tid == 0) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_begin));
    if (L.pdl) {
        griddep_wait();     // the previous consensus pass (PDL launch)
        griddep_launch();   // all K1 CTAs are resident: the consensus pass may launch
    }
#ifdef K1_DIAG2
    // per-SM count of resident K1 CTAs at [16K, 16K + 256) of the timeline
    uint32_t smid_;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(smid_));
    int *sm_cnt = L.timeline ? reinterpret_cast<int *>(L.timeline + 16 * (size_t)L.K) : nullptr;
    if (sm_cnt && tid == 0) atomicAdd(sm_cnt + smid_, 1);
    struct SmLeave {
        int *c; uint32_t s; int t;
        __device__ ~SmLeave() { if (c && t == 0) atomicSub(c + s, 1); }
    } sm_leave_{sm_cnt, smid_, tid};
#endif
    int ycur;
    if (L.dlist) {
        // run loop: CTA i takes entry i of this iteration's dirty-block list
        // (both lists' count and entry i are read with the run state, one
        // round trip: most CTAs find nothing to do and must leave fast)
        const int stop = L.st->stop;
        ycur = L.st->ycur;
        const int it = L.st->iteration;
        const uint32_t bi = blockIdx.x < (unsigned)L.K ? blockIdx.x : 0u;
        const uint32_t c0 = __ldcg(L.dlist), c1 = __ldcg(L.dlist + L.K + 1);
        const uint32_t e0 = __ldcg(L.dlist + 1 + bi), e1 = __ldcg(L.dlist + L.K + 2 + bi);
        if (blockIdx.x == 0 && tid == 0) {
            dirty_list(L, it + 1)[0] = 0u;   // the next pass fills it
            if (L.ovl) __threadfence();      // before this CTA's trigger (or exit)
        }
        const uint32_t cnt = (it & 1) ? c1 : c0, ent = (it & 1) ? e1 : e0;
        if (stop || blockIdx.x >= cnt) {
            if (L.peers && (L.gup | L.gdn | L.gzu | L.gzd)) k1_peer_exit(L);
            return;
        }
        k = (int)ent;
        DOPE_ASSERT(cnt <= (uint32_t)L.K && k >= 0 && k < L.K);
    } else {
        // the flags and the current buffer in one round trip: a clean CTA must
        // leave its slot fast (4096 CTAs churn through ~5 slots per SM), a
        // dirty one needs ycur before its first data load
        const int stop = L.st->stop;
        ycur = L.st->ycur;
        const uint32_t dk = L.skip_clean ? L.dirty[k] : 1u;
        if (stop || dk == 0) {
            if (L.peers && (L.gup | L.gdn | L.gzu | L.gzd)) k1_peer_exit(L);
            return;
        }
    }
    k1_body<BH, BW, NT>(L, T, k, ycur, true, t_begin);
    if (L.peers && (L.gup | L.gdn | L.gzu | L.gzd)) k1_peer_exit(L);
}

// K1, worklist mode (run loop with dirty-block worklists): one wave of
// resident CTAs walks the iteration's list -- CTA i takes entries i, i +
// grid, ... -- so clean blocks cost no CTA launches (a 4096-CTA grid of
// mostly-exiting CTAs finished dispatching ~15 us into the iteration, which
// is when the overlapped consensus pass could start).
#ifndef K1WL_MINB
#define K1WL_MINB 5
#endif
template <int BH, int BW, int NT>
__global__ void __launch_bounds__(NT, (BH == 64 && NT == 256 ? K1WL_MINB : K1_MINB_OF(BH, NT)))
    k_block_mincut_wl(const __grid_constant__ Lat2 L, const __grid_constant__ K1Tune T) {
    const int tid = threadIdx.x;
    uint64_t t_begin = 0;
    if (L.timeline && tid == 0) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_begin));
    const int stop = L.st->stop;
    const int ycur = L.st->ycur;
    const int it = L.st->iteration;
    const uint32_t bi = blockIdx.x < (unsigned)L.K ? blockIdx.x : 0u;
    const uint32_t c0 = __ldcg(L.dlist), c1 = __ldcg(L.dlist + L.K + 1);
    const uint32_t e0 = __ldcg(L.dlist + 1 + bi), e1 = __ldcg(L.dlist + L.K + 2 + bi);
    if (blockIdx.x == 0 && tid == 0) {
        dirty_list(L, it + 1)[0] = 0u;   // the next pass fills it
        if (L.ovl) __threadfence();      // before this CTA's trigger (or exit)
    }
    const uint32_t cnt = (it & 1) ? c1 : c0, ent = (it & 1) ? e1 : e0;
    if (!stop) {
        const uint32_t *lst = dirty_list(L, it);
        DOPE_ASSERT(cnt <= (uint32_t)L.K);
        for (uint32_t e = blockIdx.x; e < cnt; e += gridDim.x) {
            const int k = (int)(e == blockIdx.x ? ent : __ldcg(lst + 1 + e));
            DOPE_ASSERT(k >= 0 && k < L.K);
            k1_body<BH, BW, NT>(L, T, k, ycur, e + gridDim.x >= cnt, t_begin);
            __syncthreads();   // shared memory reused by the next block
            if (L.timeline && tid == 0) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_begin));
        }
    }
    if (L.peers && (L.gup | L.gdn | L.gzu | L.gzd)) k1_peer_exit(L);
}

// cold residual graphs for every block (warm-start initial state)
__global__ void k_init_resid(Lat2 L) {
    const int k = blockIdx.x;
    const int M = L.boxh * L.boxw;
    const int by = k / L.ax.k, bx = k % L.ax.k;
    int32_t lo_r, hr, lo_c, wc;
    L.ay.range(by, lo_r, hr);
    L.ax.range(bx, lo_c, wc);
    uint8_t *gres = L.resid + (size_t)k * 2 * M;   // E and S planes
    // 4 nodes per 32-bit store (box widths are multiples of 16)
    for (int q = threadIdx.x; q < M / 4; q += blockDim.x) {
        const int v0 = 4 * q, r = v0 / L.boxw, c0 = v0 % L.boxw;
        uint32_t e = 0, sv = 0;
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const int c = c0 + i;
            const bool valid = r < hr && c < wc;
            e |= (uint32_t)((valid && c + 1 < wc) ? L.cap : 0) << (8 * i);
            sv |= (uint32_t)((valid && r + 1 < hr) ? L.cap : 0) << (8 * i);
        }
        reinterpret_cast<uint32_t *>(gres)[q] = e;
        reinterpret_cast<uint32_t *>(gres + M)[q] = sv;
    }
}

__global__ void k_init_state(Lat2 L, int64_t n) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
        L.y2[0][i] = 1;              // y = 1/2 (admm.py:102-110); best_y = copy
        L.a[i] = 0;
        L.yhat[i] = 0;
    }
    if (blockIdx.x == 0 && L.pc)
        for (int i = threadIdx.x; i < DOPE_PART_CTA_LEN; i += blockDim.x) L.pc[i] = 0;
    if (L.ndim == 2) {   // ghost rows of the initial iterate: the neighbours' y = 1/2
        for (int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; c < L.W; c += stride) {
            L.y2[0][-L.W + c] = 1;
            L.y2[0][(int64_t)L.ay.dim * L.W + c] = 1;
            L.yhat[-L.W + c] = 0;
            L.yhat[(int64_t)L.ay.dim * L.W + c] = 0;
        }
    } else if (L.gzu || L.gzd) {   // 3D shards: ghost planes
        const int64_t HW = (int64_t)L.ay.dim * L.W, below = (int64_t)L.az.dim * HW;
        for (int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; c < HW; c += stride) {
            if (L.gzu) {
                L.y2[0][-HW + c] = 1;
                L.yhat[-HW + c] = 0;
            }
            if (L.gzd) {
                L.y2[0][below + c] = 1;
                L.yhat[below + c] = 0;
            }
        }
    }
    if (L.ga_up) {   // sharded: multipliers of the ghost rows / planes
        const int64_t U = L.ndim == 3 ? (int64_t)L.ay.dim * L.W : (int64_t)L.W;
        for (int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; c < U; c += stride) {
            L.ga_up[c] = 0;
            L.ga_dn[c] = 0;
            if (L.ndim == 2) {   // every rotating buffer's ghost rows start at y = 1/2
                for (int b = 1; b < 3; ++b) {
                    L.y2[b][-L.W + c] = 1;
                    L.y2[b][(int64_t)L.ay.dim * L.W + c] = 1;
                }
            }
        }
    }
    if (L.ndim == 3 && L.scratch) {   // slab accumulators of the 3D consensus pass (slab_acc3)
        const size_t M = (size_t)L.boxd * L.boxh * L.boxw;
        unsigned long long *acc = reinterpret_cast<unsigned long long *>(L.scratch + (size_t)L.K * (7 * M + 128));
        for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < 8 * (int64_t)L.K; i += stride) acc[i] = 0ull;
    }
    // solve epochs and the stamps of the clean-block consensus passes
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < 6 * (int64_t)L.K; i += stride)
            L.dirty[L.K + i] = 0u;
    // finished-solve epochs of the overlap mode (dirty[11K + 2, 12K + 2)) and
    // the consensus pass's tile-work queue (dirty[12K + 2, 16K + 8))
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < 5 * (int64_t)L.K + 6; i += stride)
        L.dirty[(size_t)11 * L.K + 2 + i] = 0u;
    if (L.dlist) {   // iteration 0 solves every block: list 0 = all, list 1 empty
        for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < L.K; i += stride)
            L.dlist[1 + i] = (uint32_t)i;
        if (blockIdx.x == 0 && threadIdx.x == 0) {
            L.dlist[0] = (uint32_t)L.K;
            L.dlist[L.K + 1] = 0u;
        }
    }
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < L.K; i += stride) {
        L.dirty[i] = 1u;
        L.pe[i] = 0;
        L.pr[i] = 0;
        L.pu[i] = 0;
        L.pf[i] = 0;
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        dope_run_state s;
        memset(&s, 0, sizeof(s));
        s.best_energy = INT64_MAX;
        s.generation = L.st->generation + 1;   // tags this run's peer-exchange epochs
        *L.st = s;
    }
}

// sum u * y2 of the initial iterate (y2 = 1): the running unary term starts at sum u
// Sum of a per-thread int64 partial over the CTA, one atomic per CTA
// (a per-warp atomic on one address serialises thousands of updates).
__device__ __forceinline__ void cta_atomic_add(int64_t v, int64_t *dst) {
    __shared__ int64_t red[32];
    v = warp_sum(v);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
    __syncthreads();
    if (lane == 0) red[warp] = v;
    __syncthreads();
    if (threadIdx.x == 0) {
        int64_t t = 0;
        for (int w = 0; w < nw; ++w) t += red[w];
        if (t) atomicAdd(reinterpret_cast<unsigned long long *>(dst), (unsigned long long)t);
    }
}

__global__ void k_init_unary(Lat2 L, int64_t n) {
    int64_t acc = 0;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    const int64_t t0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (((uintptr_t)L.u & 15) == 0) {   // 16-byte loads
        const int4 *u4 = reinterpret_cast<const int4 *>(L.u);
        for (int64_t i = t0; i < n / 4; i += stride) {
            const int4 v = __ldg(u4 + i);
            acc += (int64_t)v.x + v.y + v.z + v.w;
        }
        for (int64_t i = n / 4 * 4 + t0; i < n; i += stride) acc += L.u[i];
    } else {
        for (int64_t i = t0; i < n; i += stride) acc += L.u[i];
    }
    cta_atomic_add(acc, &L.st->unary2);
}

// ---------------------------------------------------------------------------
// K2: consensus update (2D, 4-connected), one CTA per block
// ---------------------------------------------------------------------------
//
// Iteration t's K2 reads y_{t-1} (buffer st.ycur), writes y_t into the one
// buffer that is neither ycur nor st.ybest, and -- because y_{t-1} and all of
// its neighbours are already in HBM -- produces the per-block pair-energy
// partials of E(y_{t-1}) (energy.py:187-194) for the previous iteration's
// trace entry.  The unary part u.y is kept incrementally in st.unary2
// (= sum u*y2): each pass adds u*(y2_t - y2_{t-1}) where y moved, so u is only
// read where the labeling changed.  The best iterate is tracked by buffer
// index: no copies (admm.py:242-245).  The last iterate's energy is taken by
// dope_finish_run.

__device__ __forceinline__ int other_buffer(int cur, int best) {
    // the y buffer that is neither the current nor the best iterate
    if (cur == best) return (cur + 1) % 3;
    return 3 - cur - best;
}

// Apply one iteration's global aggregates to the run state (admm.py:231-249):
// trace entry, best iterate by buffer index (strict <), parity, stop rule,
// y-buffer rotation.  E2 is the energy of the previous iterate (y_{t}),
// R2/M2/F2 the residual sum, max block residual^2 and clamp flag of this one.
// s0 is a snapshot of the run state taken by the caller (its fields are read
// in one go instead of one dependent round trip per field).
__device__ void apply_iteration(const Lat2 &L, const dope_run_state &s0, int64_t E2, double R2, int64_t M2,
                                int F2, int cur, int best_idx, int out) {
    dope_run_state *st = L.st;
    int bidx = best_idx;
    const int t = s0.iteration;         // iterations completed before this one
    if (t >= 1) {
        if (t - 1 < L.max_iters) L.tr_e[t - 1] = E2;
        if (E2 < s0.best_energy) {
            st->best_energy = E2;
            st->best_iteration = t;
            bidx = cur;
        }
    }
    const double maxres = M2 < 0 ? 0.0 : sqrt((double)M2);
    if (t < L.max_iters) {
        L.tr_rs[t] = R2;
        L.tr_mr[t] = maxres;
        L.tr_cl[t] = F2;
    }
    st->parity = s0.parity ^ 1;
    st->iteration = t + 1;
    int stop = 0;
    if (L.K == 0 || maxres <= L.eps) {
        st->converged = 1;
        stop = 1;
    }
    int err = s0.error;
    if (!err && s0.a_bound >= 32000) {   // int16 multipliers
        err = -1;
        st->error = -1;
    }
    if (err || stop) st->stop = 1;
    st->ybest = bidx;
    st->ycur = out;
}

// Residual sum of squares, admm.py:237: sum over blocks of fl(fl(sqrt(ss))^2).
// Each term is ss + e with e an exact multiple of 2^-53 (|e| <= 4 ulp(ss)), so
// the sum is kept exactly as two integers (sum ss, sum e * 2^53) and rounded
// once: deterministic whatever order the blocks are visited in.
__device__ __forceinline__ int64_t rsq_excess(int64_t ss) {
    const double r = sqrt((double)ss);
    const double t = __dmul_rn(r, r);                      // fl(r^2), no contraction
    return (int64_t)((t - (double)ss) * 9007199254740992.0);   // exact (Sterbenz), x 2^53
}
__device__ __forceinline__ double rsq_total(int64_t sum_ss, int64_t sum_excess) {
    return (double)sum_ss + (double)sum_excess * 0x1p-53;
}

// The agg table the sharded loop uses for iteration `it`: peer mode alternates
// two halves by parity (a shard can be one iteration ahead of another and
// already pushing its next slot), the gather modes use the first.
__device__ __forceinline__ int64_t *agg_table(const Lat2 &L, int it) {
    return L.agg + (L.peers ? (size_t)(it & 1) * AGG_SLOT * L.shard_count : 0);
}

// Peer mode: this shard's slot into every other shard's table (same half),
// then their flags for it.  One thread.
__device__ void push_agg_slot(const Lat2 &L, int it, const int64_t *slot, uint32_t ep) {
    const dope_peers *pr = L.peers;
    const size_t off = (size_t)(it & 1) * AGG_SLOT * L.shard_count + (size_t)AGG_SLOT * L.shard_index;
    for (int r = 0; r < L.shard_count; ++r) {
        if (r == L.shard_index) continue;
        int64_t *dst = pr->agg_of[r] + off;
        for (int i = 0; i < AGG_SLOT; ++i) dst[i] = slot[i];
    }
    __threadfence_system();
    for (int r = 0; r < L.shard_count; ++r)
        if (r != L.shard_index) st_release_sys(pr->aflag_of[r] + L.shard_index, ep);
}

// Peer mode: wait until every other shard's slot for this epoch has arrived.
__device__ void wait_agg_slots(const Lat2 &L, uint32_t ep) {
    for (int r = 0; r < L.shard_count; ++r)
        if (r != L.shard_index) wait_flag(L.pflags + 4 + r, ep);
}

// Apply one consensus pass's global aggregates (pair energy E of y_{t-1},
// unary change U, residual sum R2, max block residual^2 M2, clamp flag F):
// run-loop decision, or -- when sharded -- publish them for the cross-rank
// all-reduce and leave the decision to dope_decide.  Always advances the
// running unary term.  One thread.
__device__ void finalize_apply(const Lat2 &L, dope_run_state s0, int64_t E2, int64_t U2, int64_t S2,
                               int64_t X2, int64_t M2, int F2, int cur, int best_idx, int out) {
    dope_run_state *st = L.st;
    E2 += s0.unary2 / 2;             // E(y_{t-1}) = u.y_{t-1} + pair terms
    st->unary2 = s0.unary2 + U2;     // now sum u*y2_t
    if (L.fuse) st->a_bound = ++s0.a_bound;   // this pass updated the multipliers
    if (!L.fuse) {                   // step-level API: rotate only
        st->ybest = best_idx;
        st->ycur = out;
    } else if (L.sharded) {          // this shard's slot of the agg table; dope_decide reduces
        int64_t *slot = agg_table(L, s0.iteration) + (size_t)AGG_SLOT * L.shard_index;
        slot[0] = E2;
        slot[1] = S2;
        slot[2] = X2;
        slot[3] = M2;
        slot[4] = F2;
        if (L.peers) push_agg_slot(L, s0.iteration, slot, peer_epoch(L.st, (uint32_t)s0.iteration + 1u));
    } else {
        apply_iteration(L, s0, E2, rsq_total(S2, X2), M2, F2, cur, best_idx, out);
    }
}


// Sharded mode: reduce the gathered agg table in shard order -- exact
// integers throughout, so every shard (and the single-GPU run) reaches the
// same trace entry, best iterate and stop decision -- and apply it.
__device__ void decide_apply(const Lat2 &L) {
    dope_run_state *st = L.st;
    const int cur = st->ycur, best = st->ybest;
    const dope_run_state s0 = *st;
    if (L.peers) wait_agg_slots(L, peer_epoch(st, (uint32_t)s0.iteration + 1u));
    const int64_t *table = agg_table(L, s0.iteration);
    int64_t E = 0, S = 0, X = 0, M = -1;
    int F = 0;
    for (int r = 0; r < L.shard_count; ++r) {
        const int64_t *slot = table + (size_t)AGG_SLOT * r;
        E += slot[0];
        S += slot[1];
        X += slot[2];
        M = slot[3] > M ? slot[3] : M;
        F |= (int)slot[4];
    }
    apply_iteration(L, s0, E, rsq_total(S, X), M, F, cur, best, other_buffer(cur, best));
}

__global__ void k_decide(Lat2 L) {
    if (L.st->stop) return;
    decide_apply(L);
}

// Sharded mode: the new iterate and multipliers of the ghost rows (2D) /
// planes (3D) -- the neighbour shards' boundary pixels -- recomputed here
// instead of exchanged.  A ghost pixel's update (admm.py:136-151 on the q == 1
// stencil, like the consensus pass) needs its own label and multiplier, the
// labels of its cross-block neighbours: in-row (in-plane) ones across block
// seams, the facing local boundary pixel, and -- never, with blocks at least
// two rows / planes deep -- the pixel beyond; all are in hand after the label
// halo.  The ghost multipliers are kept redundantly (a += yhat - y, exactly
// the owner's update), so the values equal the owner's bit for bit.  Runs
// after the consensus pass and before dope_decide: writes y into the output
// buffer's ghost rows and marks the adjacent local block dirty where the
// ghost iterate moved (it enters that block's objective, blockform.py:103).
__device__ void ghost_pixels(const Lat2 &L, int cur, int out) {
    const ystore_t *__restrict__ y_in = L.y2[cur];
    ystore_t *__restrict__ y_out = L.y2[out];
    const bool is3 = L.ndim == 3;
    const int64_t P = is3 ? (int64_t)L.ay.dim * L.W : (int64_t)L.W;   // pixels per ghost unit
    const int64_t below = (is3 ? (int64_t)L.az.dim : (int64_t)L.ay.dim) * P;
    const bool has_up = is3 ? L.gzu : L.gup, has_dn = is3 ? L.gzd : L.gdn;
    if (!has_up && !has_dn) return;
    const int kplane = is3 ? L.ay.k * L.ax.k : L.ax.k;   // blocks per block row / plane
    for (int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; c < P; c += (int64_t)gridDim.x * blockDim.x) {
        const int32_t r = is3 ? (int32_t)(c / L.W) : 0, x = (int32_t)(c - (int64_t)r * L.W);
        const int bx = L.ax.owner(x), by = is3 ? L.ay.owner(r) : 0;
        const int kin = by * L.ax.k + bx;   // local block facing this column, within its block row / plane
        for (int side = 0; side < 2; ++side) {
            if (side == 0 ? !has_up : !has_dn) continue;
            const int64_t G = side == 0 ? c - P : below + c;          // ghost pixel
            const int64_t I = side == 0 ? c : below - P + c;          // facing local pixel
            DOPE_ASSERT(G >= -P && G < below + P && I >= 0 && I < below);
            const int32_t yh = L.yhat[G];
            int32_t s = yh - L.yhat[I];
            if (x > 0 && L.ax.owner(x - 1) != bx) s += yh - L.yhat[G - 1];
            if (x + 1 < L.W && L.ax.owner(x + 1) != bx) s += yh - L.yhat[G + 1];
            if (is3) {
                if (r > 0 && L.ay.owner(r - 1) != by) s += yh - L.yhat[G - L.W];
                if (r + 1 < L.ay.dim && L.ay.owner(r + 1) != by) s += yh - L.yhat[G + L.W];
            }
            astore_t *ga = side == 0 ? L.ga_up : L.ga_dn;
            const int32_t aold = ga[c];
            const int32_t ypre = yh + aold - L.q * s;
            const int32_t y = ypre < 0 ? 0 : (ypre > 1 ? 1 : ypre);
            ga[c] = (astore_t)(aold + yh - y);
            y_out[G] = (ystore_t)(2 * y);
            if (2 * y != (int32_t)y_in[G])
                mark_dirty(L, side == 0 ? kin : (size_t)(L.K - kplane) + kin);
        }
    }
}

__global__ void k_ghost_consensus(Lat2 L) {
    dope_run_state *st = L.st;
    if (st->stop) return;
    const int cur = st->ycur, best = st->ybest;
    ghost_pixels(L, cur, other_buffer(cur, best));
}

// The sharded loop's step after the agg gather, in one launch: the ghost rows'
// new iterate (every CTA, as k_ghost_consensus) and -- in the last CTA to
// finish, once every ghost pixel is in -- the decision (as k_decide).
__global__ void k_ghost_decide(Lat2 L) {
    dope_run_state *st = L.st;
    if (st->stop) return;   // read before any CTA can be last: uniform over the grid
    const int cur = st->ycur, best = st->ybest;
    if (L.ga_up) ghost_pixels(L, cur, other_buffer(cur, best));
    __shared__ int last;
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        last = atomicAdd(&st->done_ctas, 1) == (int)gridDim.x - 1;
    }
    __syncthreads();
    if (last && threadIdx.x == 0) {
        __threadfence();
        st->done_ctas = 0;
        decide_apply(L);
    }
}

// Run-loop entry: this iteration's dirty-block list from the flags (they may
// have been set by step-level calls or the host since the last pass), the
// other list emptied.  One CTA.
__global__ void k_rebuild_dlist(Lat2 L) {
    const int it = L.st->iteration;
    uint32_t *cur = dirty_list(L, it);
    if (threadIdx.x == 0) {
        cur[0] = 0u;
        dirty_list(L, it + 1)[0] = 0u;
    }
    __syncthreads();
    for (int k = threadIdx.x; k < L.K; k += blockDim.x)
        if (L.dirty[k]) cur[1 + atomicAdd(cur, 1u)] = (uint32_t)k;
}

// Peer mode, after K1: wait for the neighbours' boundary rows of this
// iteration (their K1's last CTA raised the flags) and install them in the
// ghost rows / planes.  One CTA.
__global__ void k_peer_install(Lat2 L) {
    dope_run_state *st = L.st;
    if (st->stop) return;
    const bool is3 = L.ndim == 3;
    const bool up = is3 ? L.gzu : L.gup, dn = is3 ? L.gzd : L.gdn;
    const int64_t P = is3 ? (int64_t)L.ay.dim * L.W : (int64_t)L.W;
    const int64_t below = (is3 ? (int64_t)L.az.dim : (int64_t)L.ay.dim) * P;
    if (threadIdx.x == 0) {
        const uint32_t ep = peer_epoch(st, (uint32_t)st->iteration + 1u);
        if (up) wait_flag(L.pflags + 0, ep);
        if (dn) wait_flag(L.pflags + 1, ep);
    }
    __syncthreads();
    // halo slots: [2U, 3U) from above, [3U, 4U) from below (dope_halo_bytes)
    const uint8_t *from_up = reinterpret_cast<const uint8_t *>(L.ga_up) - halo_ga_offset(P) + 2 * P;
    const uint8_t *from_dn = from_up + P;
    for (int64_t c = threadIdx.x; c < P; c += blockDim.x) {
        if (up) L.yhat[c - P] = from_up[c];
        if (dn) L.yhat[below + c] = from_dn[c];
    }
}

// The integer path's unary from the caller's float64 vector (the reference's
// EnergyModel.unary): exact integers within +-2^28, else *bad = 1.
__global__ void k_unary_i32(const double *__restrict__ u, int64_t n, int32_t *__restrict__ out, int32_t *bad) {
    int b = 0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const double v = u[i];
        const bool ok = v == rint(v) && fabs(v) <= 268435456.0;
        b |= !ok;
        out[i] = ok ? (int32_t)v : 0;
    }
    if (__syncthreads_or(b) && threadIdx.x == 0) atomicOr(bad, 1);
}

// Sharded mode, end of run: move this shard's energy of the last iterate into
// its agg slot (the cross-shard sum happens in k_finish_decide).
__global__ void k_publish_energy(Lat2 L) {
    dope_run_state *st = L.st;
    int64_t *slot = agg_table(L, st->iteration) + (size_t)AGG_SLOT * L.shard_index;
    slot[5] = st->energy_acc;
    st->energy_acc = 0;
    if (L.peers) push_agg_slot(L, st->iteration, slot, peer_epoch(st, 0x8000u + (uint32_t)st->iteration));
}

// Sharded mode: copy this shard's first and last local rows (labels or the
// current iterate, both bytes) into caller staging buffers for the halo exchange.
__global__ void k_pack_rows(Lat2 L, int which, void *first, void *last) {
    // the exchanged unit: a row (2D, slabs of block rows) or a plane (3D, slabs of block planes)
    const int64_t P = L.ndim == 3 ? (int64_t)L.ay.dim * L.W : (int64_t)L.W;
    const int64_t lastoff = ((L.ndim == 3 ? (int64_t)L.az.dim : (int64_t)L.ay.dim) - 1) * P;
    const uint8_t *src = which == 0 ? L.yhat : L.y2[L.st->ycur];
    for (int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; c < P; c += (int64_t)gridDim.x * blockDim.x) {
        if (first) static_cast<uint8_t *>(first)[c] = src[c];
        if (last) static_cast<uint8_t *>(last)[c] = src[lastoff + c];
    }
}

// Sharded mode: install the neighbour shards' boundary rows into the ghost
// rows.  which == 0: labels; which == 1: current iterate y2, marking the local
// boundary block row dirty where the neighbour's y changed (it enters this
// shard's block objectives, blockform.py:103).
__global__ void k_ghost_update(Lat2 L, int which, const void *up_new, const void *dn_new) {
    if (L.ndim == 3) {   // ghost planes; a changed ghost y marks the adjacent local block
        const int64_t HW = (int64_t)L.ay.dim * L.W, below = (int64_t)L.az.dim * HW;
        const uint8_t *up = static_cast<const uint8_t *>(up_new), *dn = static_cast<const uint8_t *>(dn_new);
        for (int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; c < HW; c += (int64_t)gridDim.x * blockDim.x) {
            if (which == 0) {
                if (L.gzu && up) L.yhat[-HW + c] = up[c];
                if (L.gzd && dn) L.yhat[below + c] = dn[c];
            } else {
                uint8_t *y = L.y2[L.st->ycur];
                const int r = (int)(c / L.W), col = (int)(c - (int64_t)r * L.W);
                const int kyx = L.ay.owner(r) * L.ax.k + L.ax.owner(col);
                if (L.gzu && up && y[-HW + c] != up[c]) {
                    mark_dirty(L, kyx);
                    y[-HW + c] = up[c];
                }
                if (L.gzd && dn && y[below + c] != dn[c]) {
                    mark_dirty(L, (L.az.k - 1) * L.ay.k * L.ax.k + kyx);
                    y[below + c] = dn[c];
                }
            }
        }
        return;
    }
    const int32_t W = L.W;
    const int64_t below = (int64_t)L.ay.dim * W;
    const uint8_t *up = static_cast<const uint8_t *>(up_new), *dn = static_cast<const uint8_t *>(dn_new);
    for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < W; c += gridDim.x * blockDim.x) {
        if (which == 0) {
            if (L.gup && up) L.yhat[-W + c] = up[c];
            if (L.gdn && dn) L.yhat[below + c] = dn[c];
        } else {
            uint8_t *y = L.y2[L.st->ycur];
            const int bx = L.ax.owner(c);
            if (L.gup && up && y[-W + c] != up[c]) {
                mark_dirty(L, bx);
                y[-W + c] = up[c];
            }
            if (L.gdn && dn && y[below + c] != dn[c]) {
                mark_dirty(L, (L.ay.k - 1) * L.ax.k + bx);
                y[below + c] = dn[c];
            }
        }
    }
}

// This CTA's exact pass aggregates (thread 0): pair energy, unary change,
// max block ss, clamp flag, sum ss, sum of residual excesses (rsq_excess).
struct CtaAgg {
    int64_t E = 0, U = 0, M = -1, S = 0, X = 0;
    int F = 0;
    __device__ void add_block(int64_t e, int64_t u, int64_t ss, int clamped) {
        E += e;
        U += u;
        M = ss > M ? ss : M;
        S += ss;
        X += rsq_excess(ss);
        F |= clamped;
    }
};

// One thread per CTA, after its last block: fold the CTA's aggregates into
// the pass-wide ones (order-free integer atomics); the last CTA to arrive
// applies the pass (trace, best iterate, stop rule, buffer rotation).
__device__ void pass_tail(const Lat2 &L, const CtaAgg &c, int cur, int best, int out) {
    if (c.E) atomicAdd(reinterpret_cast<unsigned long long *>(&L.pc[0]), (unsigned long long)c.E);
    if (c.U) atomicAdd(reinterpret_cast<unsigned long long *>(&L.pc[1]), (unsigned long long)c.U);
    if (c.M >= 0) atomicMax(reinterpret_cast<unsigned long long *>(&L.pc[2]), (unsigned long long)(c.M + 1));
    if (c.F) atomicOr(reinterpret_cast<unsigned long long *>(&L.pc[3]), 1ull);
    if (c.S) atomicAdd(reinterpret_cast<unsigned long long *>(&L.pc[4]), (unsigned long long)c.S);
    if (c.X) atomicAdd(reinterpret_cast<unsigned long long *>(&L.pc[5]), (unsigned long long)c.X);
    __threadfence();
    dope_run_state *st = L.st;
    if (atomicAdd(&st->done_ctas, 1) == (int)(gridDim.x * gridDim.y * gridDim.z) - 1) {
        __threadfence();
        // overlap mode: K1 (error flag, statistics) complete before the decision;
        // the grid cannot complete before K1 either
        if (L.ovl) griddep_wait();
        const dope_run_state s0 = *st;
        const int64_t E2 = __ldcg(&L.pc[0]), U2 = __ldcg(&L.pc[1]), M2 = __ldcg(&L.pc[2]) - 1;
        const int F2 = (int)__ldcg(&L.pc[3]);
        const int64_t S2 = __ldcg(&L.pc[4]), X2 = __ldcg(&L.pc[5]);
        for (int i = 0; i < 8; ++i) L.pc[i] = 0;   // incl. the solved-list count
        if (L.kq) {   // the tile-work queue's counters (its entries were cleared as taken)
            L.kq[4 * (size_t)L.K] = 0u;
            L.kq[4 * (size_t)L.K + 1] = 0u;
            L.kq[4 * (size_t)L.K + 2] = 0u;
        }
        finalize_apply(L, s0, E2, U2, S2, X2, M2, F2, cur, best, out);
        st->done_ctas = 0;
    }
}

// Per-block epilogue of the scalar / vector consensus kernels: reduce the
// thread partials; thread 0 publishes the block's partials and dirty marks
// and folds them into the CTA aggregates.  Ends with a barrier (the shared
// scratch is reused by the CTA's next block).
__device__ __forceinline__ void block_epilogue(const Lat2 &L, int k, int64_t e_acc, int64_t du, int64_t ss,
                                               int clamped, int chg_self, int chgL, int chgR, int chgU,
                                               int chgD, CtaAgg &agg) {
    __shared__ int64_t red_e[32], red_s[32], red_u[32];
    __shared__ int red_f[32];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    e_acc = warp_sum(e_acc);
    du = warp_sum(du);
    ss = warp_sum(ss);
    const unsigned fl = __ballot_sync(FULLMASK, clamped) ? 1u : 0u;
    const unsigned f0 = __ballot_sync(FULLMASK, chg_self) ? 2u : 0u;
    const unsigned f1 = __ballot_sync(FULLMASK, chgL) ? 4u : 0u;
    const unsigned f2 = __ballot_sync(FULLMASK, chgR) ? 8u : 0u;
    const unsigned f3 = __ballot_sync(FULLMASK, chgU) ? 16u : 0u;
    const unsigned f4 = __ballot_sync(FULLMASK, chgD) ? 32u : 0u;
    if (lane == 0) {
        red_e[warp] = e_acc;
        red_u[warp] = du;
        red_s[warp] = ss;
        red_f[warp] = (int)(fl | f0 | f1 | f2 | f3 | f4);
    }
    __syncthreads();
    if (tid == 0) {
        int64_t E = 0, S = 0, U = 0;
        int Fm = 0;
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) {
            E += red_e[w];
            U += red_u[w];
            S += red_s[w];
            Fm |= red_f[w];
        }
        L.pe[k] = E;
        L.pu[k] = U;
        L.pr[k] = S;
        L.pf[k] = Fm & 1;
        if (Fm & 2) mark_dirty(L, k);
        if (Fm & 4) mark_dirty(L, k - 1);
        if (Fm & 8) mark_dirty(L, k + 1);
        if ((Fm & 16) && k - L.ax.k >= 0) mark_dirty(L, k - L.ax.k);
        if ((Fm & 32) && k + L.ax.k < L.K) mark_dirty(L, k + L.ax.k);
        agg.add_block(E, U, S, Fm & 1);
    }
    __syncthreads();
}

// Multiplier range: |a| moves by at most 1 per pass (yhat, y in {0, 1}), so
// st.a_bound (passes so far) bounds it; the run loop stops at 32000 passes
// (apply_iteration) and the step-level pass checks each value.
__device__ __forceinline__ void check_a(const Lat2 &L, int a) {
    if (a > 32000 || a < -32000) atomicCAS(&L.st->error, 0, -1);
}

// Generic consensus (any tiling, incl. ragged): one CTA per block, scalar.
__global__ void __launch_bounds__(256) k_consensus(Lat2 L) {
    if (L.pdl) {
        griddep_wait();
        griddep_launch();
    }
    if (L.st->stop) return;
    const int tid = threadIdx.x;
    CtaAgg agg;
    const int cur = L.st->ycur, best = L.st->ybest, out = other_buffer(cur, best);
    for (int k = blockIdx.x; k < L.K; k += gridDim.x) {
    const int by = k / L.ax.k, bx = k % L.ax.k;
    int32_t lo_r, hr, lo_c, wc;
    L.ay.range(by, lo_r, hr);
    L.ax.range(bx, lo_c, wc);
    const int32_t W = L.W, H = L.ay.dim;
    const ystore_t *__restrict__ y_in = L.y2[cur];
    ystore_t *__restrict__ y_out = L.y2[out];
    // multipliers are updated in place (a_{t+1}[p] depends on a_t[p] only)
    const astore_t *a_in = L.a;
    astore_t *a_out = L.fuse ? L.a : nullptr;
    const bool want_e = L.fuse && L.st->iteration >= 1;
    const bool has_up = lo_r > 0 || L.gup, has_dn = lo_r + hr < H || L.gdn, has_lf = lo_c > 0,
               has_rt = lo_c + wc < W;

    int64_t e_acc = 0, du = 0, ss = 0;
    int clamped = 0, chg_self = 0, chgL = 0, chgR = 0, chgU = 0, chgD = 0;
    const int m = hr * wc;
    for (int v = tid; v < m; v += blockDim.x) {
        const int r = v / wc, c = v - r * wc;
        const int32_t R = lo_r + r, Cc = lo_c + c;
        const int64_t G = (int64_t)R * W + Cc;
        const int32_t yh = L.yhat[G];
        int32_t s = 0;
        if (c == 0 && has_lf) s += yh - L.yhat[G - 1];
        if (c == wc - 1 && has_rt) s += yh - L.yhat[G + 1];
        if (r == 0 && has_up) s += yh - L.yhat[G - W];
        if (r == hr - 1 && has_dn) s += yh - L.yhat[G + W];
        const int32_t aold = a_in[G];
        const int32_t ypre = yh + aold - L.q * s;
        const int32_t y = ypre < 0 ? 0 : (ypre > 1 ? 1 : ypre);
        const int32_t y2old = y_in[G];
        clamped |= (ypre < 0 || ypre > 1);
        if (a_out) a_out[G] = (astore_t)(aold + yh - y);
        y_out[G] = (ystore_t)(2 * y);
        ss += (yh - y) * (yh - y);
        if (2 * y != y2old) du += (int64_t)L.u[G] * (2 * y - y2old);
        if (want_e) {
            const int32_t o = y2old >> 1;
            int32_t qd = 0;
            if (Cc + 1 < W) qd += o ^ (y_in[G + 1] >> 1);
            if (R + 1 < H || L.gdn) qd += o ^ (y_in[G + W] >> 1);
            e_acc += (int64_t)L.lamw * qd;
        }
        const bool ychg = (2 * y != y2old);
        chg_self |= ychg || (yh != y);
        if (ychg) {
            chgL |= (c == 0 && has_lf);
            chgR |= (c == wc - 1 && has_rt);
            chgU |= (r == 0 && has_up);
            chgD |= (r == hr - 1 && has_dn);
        }
    }
    block_epilogue(L, k, e_acc, du, ss, clamped, chg_self, chgL, chgR, chgU, chgD, agg);
    }
    if (tid == 0) pass_tail(L, agg, cur, best, out);
}

// Vectorized consensus for uniform tilings whose block width is a power of
// two in [4, 128] and grid width a multiple of 4.  Thread t owns up to QPT
// quads (4 consecutive pixels of a block row); the quads of one block row sit
// in consecutive lanes of one warp.  All loads of a thread are issued before
// any is used; nothing goes through shared memory.
template <int NT>
__global__ void __launch_bounds__(NT) k_consensus_vec(Lat2 L, int lq) {
    constexpr int QPT = 4;
    if (L.pdl) {
        griddep_wait();
        griddep_launch();
    }
    if (L.st->stop) return;
    const int tid = threadIdx.x;
    CtaAgg agg;
    const int cur = L.st->ycur, best = L.st->ybest, out = other_buffer(cur, best);
    for (int k = blockIdx.x; k < L.K; k += gridDim.x) {
    const int by = k / L.ax.k, bx = k - by * L.ax.k;
    int32_t lo_r, hr, lo_c, wc;
    L.ay.range(by, lo_r, hr);
    L.ax.range(bx, lo_c, wc);
    const int32_t W = L.W, H = L.ay.dim;
    const int QR = 1 << lq;              // quads per block row
    const int nq = hr << lq;
    const ystore_t *__restrict__ y_in = L.y2[cur];
    ystore_t *__restrict__ y_out = L.y2[out];
    // multipliers are updated in place (a_{t+1}[p] depends on a_t[p] only)
    const astore_t *a_in = L.a;
    astore_t *a_out = L.fuse ? L.a : nullptr;
    const bool want_e = L.fuse && L.st->iteration >= 1;
    const int32_t q = L.q;
    const bool has_up = lo_r > 0 || L.gup, has_dn = lo_r + hr < H || L.gdn, has_lf = lo_c > 0,
               has_rt = lo_c + wc < W;

    // ---- issue every load of this thread's quads ----
    uint32_t yh4[QPT], up4[QPT], dn4[QPT], yo[QPT], yb[QPT];
    uint2 av[QPT];
    int lf[QPT], rt[QPT], yr[QPT];
#pragma unroll
    for (int j = 0; j < QPT; ++j) {
        const int t = tid + j * NT;
        yh4[j] = up4[j] = dn4[j] = yo[j] = yb[j] = 0;
        av[j] = make_uint2(0, 0);
        lf[j] = rt[j] = yr[j] = 0;
        if (t < nq) {
            const int r = t >> lq, c0 = (t & (QR - 1)) << 2;
            const int64_t G = (int64_t)(lo_r + r) * W + lo_c + c0;
            yh4[j] = __ldcs(reinterpret_cast<const unsigned int *>(L.yhat + G));
            av[j] = __ldcs(reinterpret_cast<const uint2 *>(a_in + G));
            yo[j] = __ldcg(reinterpret_cast<const unsigned int *>(y_in + G));
            if (want_e && (lo_r + r + 1 < H || L.gdn))
                yb[j] = __ldcg(reinterpret_cast<const unsigned int *>(y_in + G + W));
            if (r == 0 && has_up) up4[j] = *reinterpret_cast<const uint32_t *>(L.yhat + G - W);
            if (r == hr - 1 && has_dn) dn4[j] = *reinterpret_cast<const uint32_t *>(L.yhat + G + W);
            if (c0 == 0 && has_lf) lf[j] = L.yhat[G - 1];
            if (c0 + 4 == wc && has_rt) {
                rt[j] = L.yhat[G + 4];
                if (want_e) yr[j] = y_in[G + 4];
            }
        }
    }

    // ---- consensus update + pair energy of the previous iterate ----
    int64_t du = 0;
    int ss = 0, quad = 0;
    int clamped = 0, chg_self = 0, chgL = 0, chgR = 0, chgU = 0, chgD = 0;
#pragma unroll
    for (int j = 0; j < QPT; ++j) {
        const int t = tid + j * NT;
        const bool valid = t < nq;
        const int r = t >> lq, c0 = (t & (QR - 1)) << 2;
        // previous iterate as packed bits (y2 in {0,2} once t >= 1)
        const uint32_t ob = (uint32_t)((byte_at(yo[j], 0) >> 1) | ((byte_at(yo[j], 1) >> 1) << 1) |
                                       ((byte_at(yo[j], 2) >> 1) << 2) | ((byte_at(yo[j], 3) >> 1) << 3));
        const uint32_t nxt = __shfl_down_sync(FULLMASK, ob, 1);
        if (!valid) continue;
        const int64_t G = (int64_t)(lo_r + r) * W + lo_c + c0;
        const bool top = (r == 0 && has_up), bot = (r == hr - 1 && has_dn);
        const bool lft = (c0 == 0 && has_lf), rgt = (c0 + 4 == wc && has_rt);
        if (want_e) {
            const uint32_t bb = (uint32_t)((byte_at(yb[j], 0) >> 1) | ((byte_at(yb[j], 1) >> 1) << 1) |
                                           ((byte_at(yb[j], 2) >> 1) << 2) | ((byte_at(yb[j], 3) >> 1) << 3));
            quad += __popc((ob ^ (ob >> 1)) & 0x7u);            // pairs inside the quad
            if (c0 + 4 < wc) quad += (int)((ob >> 3) ^ (nxt & 1u));
            else if (rgt) quad += (int)((ob >> 3) ^ (uint32_t)(yr[j] >> 1));
            if (lo_r + r + 1 < H || L.gdn) quad += __popc(ob ^ bb);
        }
        int a4[4];
        unpack_a4(av[j], a4);
        int y[4], an[4];
        bool ychg_any = false;
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const int yh = byte_at(yh4[j], i);
            int sx = 0;
            if (top) sx += yh - byte_at(up4[j], i);
            if (bot) sx += yh - byte_at(dn4[j], i);
            if (i == 0 && lft) sx += yh - lf[j];
            if (i == 3 && rgt) sx += yh - rt[j];
            const int ypre = yh + a4[i] - q * sx;
            clamped |= (unsigned)ypre > 1u;
            y[i] = ypre < 0 ? 0 : (ypre > 1 ? 1 : ypre);
            an[i] = a4[i] + yh - y[i];
            ss += yh ^ y[i];
            const int yold = byte_at(yo[j], i);
            const bool ychg = (2 * y[i] != yold);
            if (ychg) du += (int64_t)__ldg(L.u + G + i) * (2 * y[i] - yold);
            ychg_any |= ychg;
            chg_self |= ychg | (yh != y[i]);
        }
        if (a_out) __stcs(reinterpret_cast<uint2 *>(a_out + G), pack_a4(an[0], an[1], an[2], an[3]));
        __stcg(reinterpret_cast<unsigned int *>(y_out + G), pack_y4(2 * y[0], 2 * y[1], 2 * y[2], 2 * y[3]));
        if (ychg_any) {
            chgU |= top;
            chgD |= bot;
            chgL |= (lft && (2 * y[0] != byte_at(yo[j], 0)));
            chgR |= (rgt && (2 * y[3] != byte_at(yo[j], 3)));
        }
    }
    const int64_t e64 = (int64_t)L.lamw * quad;
    block_epilogue(L, k, e64, du, (int64_t)ss, clamped, chg_self, chgL, chgR, chgU, chgD, agg);
    }
    if (tid == 0) pass_tail(L, agg, cur, best, out);
}

// Consensus for small blocks (<= 32 x 32, whole x quads): one WARP per block,
// WPC blocks per CTA in flight, no CTA barrier per block (the per-CTA barrier
// and the per-CTA aggregate atomics dominated k_consensus_vec on 16^2 / 32^2
// tilings: thousands of CTAs, each a few blocks).  Lane l owns quads
// l, l + 32, ...; a row is 1 << lq quads (<= 8), so the quad right of a
// quad is in the next lane unless the quad ends the row.  Same arithmetic as
// k_consensus_vec, plus the clean-block pass of k_consensus3d_vec (2D: the 4
// face neighbours; the iterate is copied into the output buffer).
template <int WPC, int QB, int MINB>   // QB: quads per lane per batch
__global__ void __launch_bounds__(WPC * 32, MINB) k_consensus_warp(Lat2 L, int lq) {
    if (L.pdl) {
        griddep_wait();
        griddep_launch();
    }
    if (L.st->stop) return;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int cur = L.st->ycur, best = L.st->ybest, out = other_buffer(cur, best);
    const ystore_t *__restrict__ y_in = L.y2[cur];
    ystore_t *__restrict__ y_out = L.y2[out];
    const astore_t *a_in = L.a;
    astore_t *a_out = L.fuse ? L.a : nullptr;
    const int it = L.st->iteration;
    const bool want_e = L.fuse && it >= 1;
    const bool clean_ok = L.fuse && L.skip_clean && it >= 2;
    const uint32_t ep = (uint32_t)it + 1u;
    const int32_t W = L.W, H = L.ay.dim, q = L.q;
    const int QR = 1 << lq;
    CtaAgg agg;   // this warp's blocks (lane 0)
    const int nwarps = gridDim.x * WPC;
    for (int k = blockIdx.x * WPC + warp; k < L.K; k += nwarps) {
        const int by = k / L.ax.k, bx = k - by * L.ax.k;
        int32_t lo_r, hr, lo_c, wc;
        L.ay.range(by, lo_r, hr);
        L.ax.range(bx, lo_c, wc);
        const bool has_up = lo_r > 0 || L.gup, has_dn = lo_r + hr < H || L.gdn, has_lf = lo_c > 0,
                   has_rt = lo_c + wc < W;
        const int nq = hr << lq;
        if (clean_ok) {
            const uint32_t *epo = L.dirty + L.K;
            bool fast = epo[k] != ep;
            fast = fast && !(has_lf && epo[k - 1] == ep) && !(has_rt && epo[k + 1] == ep);
            fast = fast && !(lo_r > 0 && epo[k - L.ax.k] == ep) && !(lo_r + hr < H && epo[k + L.ax.k] == ep);
            fast = fast && !(lo_r == 0 && L.gup) && !(lo_r + hr == H && L.gdn);
            if (fast) {   // fixed point: only the output buffer needs the iterate
                for (int t = lane; t < nq; t += 32) {
                    const int r = t >> lq, c0 = (t & (QR - 1)) << 2;
                    const int64_t G = (int64_t)(lo_r + r) * W + lo_c + c0;
                    *reinterpret_cast<unsigned int *>(y_out + G) = *reinterpret_cast<const unsigned int *>(y_in + G);
                }
                if (lane == 0) {
                    L.pu[k] = 0;
                    L.pr[k] = 0;
                    agg.add_block(L.pe[k], 0, 0, L.pf[k] & 1);
                }
                continue;
            }
        }
        int64_t du = 0;
        int ss = 0, quad = 0;
        int clamped = 0, chg_self = 0, chgL = 0, chgR = 0, chgU = 0, chgD = 0;
        for (int t0 = 0; t0 < nq; t0 += 32 * QB) {
            uint32_t yh4[QB], up4[QB], dn4[QB], yo[QB], yb[QB];
            uint2 av[QB];
            int lf[QB], rt[QB], yr[QB];
#pragma unroll
            for (int j = 0; j < QB; ++j) {
                const int t = t0 + lane + 32 * j;
                yh4[j] = up4[j] = dn4[j] = yo[j] = yb[j] = 0;
                av[j] = make_uint2(0, 0);
                lf[j] = rt[j] = yr[j] = 0;
                if (t < nq) {
                    const int r = t >> lq, c0 = (t & (QR - 1)) << 2;
                    const int64_t G = (int64_t)(lo_r + r) * W + lo_c + c0;
                    yh4[j] = __ldcs(reinterpret_cast<const unsigned int *>(L.yhat + G));
                    av[j] = __ldcs(reinterpret_cast<const uint2 *>(a_in + G));
                    yo[j] = __ldcg(reinterpret_cast<const unsigned int *>(y_in + G));
                    if (want_e && (lo_r + r + 1 < H || L.gdn))
                        yb[j] = __ldcg(reinterpret_cast<const unsigned int *>(y_in + G + W));
                    if (r == 0 && has_up) up4[j] = *reinterpret_cast<const uint32_t *>(L.yhat + G - W);
                    if (r == hr - 1 && has_dn) dn4[j] = *reinterpret_cast<const uint32_t *>(L.yhat + G + W);
                    if (c0 == 0 && has_lf) lf[j] = L.yhat[G - 1];
                    if (c0 + 4 == wc && has_rt) {
                        rt[j] = L.yhat[G + 4];
                        if (want_e) yr[j] = y_in[G + 4];
                    }
                }
            }
#pragma unroll
            for (int j = 0; j < QB; ++j) {
                const int t = t0 + lane + 32 * j;
                const int r = t >> lq, c0 = (t & (QR - 1)) << 2;
                const uint32_t ob = (uint32_t)((byte_at(yo[j], 0) >> 1) | ((byte_at(yo[j], 1) >> 1) << 1) |
                                               ((byte_at(yo[j], 2) >> 1) << 2) | ((byte_at(yo[j], 3) >> 1) << 3));
                const uint32_t nxt = __shfl_down_sync(FULLMASK, ob, 1);
                if (t >= nq) continue;
                const int64_t G = (int64_t)(lo_r + r) * W + lo_c + c0;
                const bool top = (r == 0 && has_up), bot = (r == hr - 1 && has_dn);
                const bool lft = (c0 == 0 && has_lf), rgt = (c0 + 4 == wc && has_rt);
                if (want_e) {
                    const uint32_t bb = (uint32_t)((byte_at(yb[j], 0) >> 1) | ((byte_at(yb[j], 1) >> 1) << 1) |
                                                   ((byte_at(yb[j], 2) >> 1) << 2) | ((byte_at(yb[j], 3) >> 1) << 3));
                    quad += __popc((ob ^ (ob >> 1)) & 0x7u);
                    if (c0 + 4 < wc) quad += (int)((ob >> 3) ^ (nxt & 1u));
                    else if (rgt) quad += (int)((ob >> 3) ^ (uint32_t)(yr[j] >> 1));
                    if (lo_r + r + 1 < H || L.gdn) quad += __popc(ob ^ bb);
                }
                int a4[4];
                unpack_a4(av[j], a4);
                int y[4], an[4];
                bool ychg_any = false;
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                    const int yh = byte_at(yh4[j], i);
                    int sx = 0;
                    if (top) sx += yh - byte_at(up4[j], i);
                    if (bot) sx += yh - byte_at(dn4[j], i);
                    if (i == 0 && lft) sx += yh - lf[j];
                    if (i == 3 && rgt) sx += yh - rt[j];
                    const int ypre = yh + a4[i] - q * sx;
                    clamped |= (unsigned)ypre > 1u;
                    y[i] = ypre < 0 ? 0 : (ypre > 1 ? 1 : ypre);
                    an[i] = a4[i] + yh - y[i];
                    ss += yh ^ y[i];
                    const int yold = byte_at(yo[j], i);
                    const bool ychg = (2 * y[i] != yold);
                    if (ychg) du += (int64_t)__ldg(L.u + G + i) * (2 * y[i] - yold);
                    ychg_any |= ychg;
                    chg_self |= ychg | (yh != y[i]);
                }
                if (a_out) __stcs(reinterpret_cast<uint2 *>(a_out + G), pack_a4(an[0], an[1], an[2], an[3]));
                __stcg(reinterpret_cast<unsigned int *>(y_out + G), pack_y4(2 * y[0], 2 * y[1], 2 * y[2], 2 * y[3]));
                if (ychg_any) {
                    chgU |= top;
                    chgD |= bot;
                    chgL |= (lft && (2 * y[0] != byte_at(yo[j], 0)));
                    chgR |= (rgt && (2 * y[3] != byte_at(yo[j], 3)));
                }
            }
        }
        // warp reduction; lane 0 publishes the block
        const int64_t E = (int64_t)L.lamw * (int64_t)__reduce_add_sync(FULLMASK, (unsigned)quad);
        const int64_t U = warp_sum(du);
        const int64_t S = (int64_t)__reduce_add_sync(FULLMASK, (unsigned)ss);
        const unsigned fm = __reduce_or_sync(FULLMASK, (clamped ? 1u : 0u) | (chg_self ? 2u : 0u) | (chgL ? 4u : 0u) |
                                                           (chgR ? 8u : 0u) | (chgU ? 16u : 0u) | (chgD ? 32u : 0u));
        if (lane == 0) {
            L.pe[k] = E;
            L.pu[k] = U;
            L.pr[k] = S;
            L.pf[k] = (int)(fm & 1u);
            if (fm & 2u) mark_dirty(L, k);
            if (fm & 4u) mark_dirty(L, k - 1);
            if (fm & 8u) mark_dirty(L, k + 1);
            if ((fm & 16u) && k - L.ax.k >= 0) mark_dirty(L, k - L.ax.k);
            if ((fm & 32u) && k + L.ax.k < L.K) mark_dirty(L, k + L.ax.k);
            agg.add_block(E, U, S, (int)(fm & 1u));
        }
    }
    // fold the warps' aggregates, then the CTA's
    __shared__ int64_t sE[WPC], sU[WPC], sM[WPC], sS[WPC], sX[WPC];
    __shared__ int sF[WPC];
    if (lane == 0) {
        sE[warp] = agg.E;
        sU[warp] = agg.U;
        sM[warp] = agg.M;
        sS[warp] = agg.S;
        sX[warp] = agg.X;
        sF[warp] = agg.F;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        CtaAgg c;
        for (int w = 0; w < WPC; ++w) {
            c.E += sE[w];
            c.U += sU[w];
            c.M = sM[w] > c.M ? sM[w] : c.M;
            c.S += sS[w];
            c.X += sX[w];
            c.F |= sF[w];
        }
        pass_tail(L, c, cur, best, out);
    }
}

// a += yhat - y for the step-level API (admm.py:183-190), in place.
__global__ void k_update_multipliers(Lat2 L, int64_t n) {
    astore_t *a = L.a;
    const ystore_t *y2 = L.y2[L.st->ycur];
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
        const int an = (int)a[i] + (int)L.yhat[i] - (y2[i] >> 1);
        check_a(L, an);
        a[i] = (astore_t)an;
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) L.st->a_bound += 1;
}

// E of the current iterate into st.energy_acc: pair terms here, plus the
// running unary term u.y = unary2 / 2 (exact integer sums: order-free).
__global__ void k_energy_current(Lat2 L, int64_t n) {
    const ystore_t *y2 = L.y2[L.st->ycur];
    int64_t acc = 0;
    const int64_t HW = (int64_t)L.ay.dim * L.W;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
        const int32_t c = (int32_t)(i % L.W);
        const int64_t r = (i / L.W) % L.ay.dim, z = i / HW;
        const int32_t yi = y2[i] >> 1;
        int32_t qd = 0;
        if (c + 1 < L.W) qd += yi ^ (y2[i + 1] >> 1);
        if (r + 1 < L.ay.dim || L.gdn) qd += yi ^ (y2[i + L.W] >> 1);
        if (z + 1 < L.az.dim || L.gzd) qd += yi ^ (y2[i + HW] >> 1);
        acc += (int64_t)L.lamw * qd;
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) acc += L.st->unary2 / 2;
    acc = warp_sum(acc);
    if ((threadIdx.x & 31) == 0)
        atomicAdd((unsigned long long *)&L.st->energy_acc, (unsigned long long)acc);
}

// Vector form of k_energy_current for grids whose width is a multiple of 4:
// one 4-byte word of y2 per step, pairs as XOR + popcount on the 0/2 bytes.
__global__ void k_energy_current_vec(Lat2 L, uint32_t nwords) {
    const ystore_t *y2 = L.y2[L.st->ycur];
    const uint32_t W4 = (uint32_t)L.W >> 2, H = (uint32_t)L.ay.dim, D = (uint32_t)L.az.dim;
    const int64_t HW = (int64_t)H * L.W;
    int64_t acc = 0;
    for (uint32_t w = blockIdx.x * blockDim.x + threadIdx.x; w < nwords; w += gridDim.x * blockDim.x) {
        const uint32_t row = w / W4, c4 = w - row * W4;
        const uint32_t r = row % H, z = row / H;
        const int64_t G = 4 * (int64_t)w;
        const uint32_t y = *reinterpret_cast<const uint32_t *>(y2 + G);
        const uint32_t nx = c4 + 1 < W4 ? *reinterpret_cast<const uint32_t *>(y2 + G + 4) : (y >> 24);
        int qd = __popc(y ^ __funnelshift_r(y, nx, 8));
        if (r + 1 < H || L.gdn) qd += __popc(y ^ *reinterpret_cast<const uint32_t *>(y2 + G + L.W));
        if (z + 1 < D || L.gzd) qd += __popc(y ^ *reinterpret_cast<const uint32_t *>(y2 + G + HW));
        acc += qd;
    }
    acc *= L.lamw;
    if (blockIdx.x == 0 && threadIdx.x == 0) acc += L.st->unary2 / 2;
    cta_atomic_add(acc, &L.st->energy_acc);
}

// End of run (admm.py:242-252): trace energy + best check of the last
// iterate, then state.y = best iterate unless converged.
__global__ void k_finish_decide(Lat2 L) {
    dope_run_state *st = L.st;
    const int T = st->iteration;
    if (T >= 1 && !st->error) {
        int64_t E = st->energy_acc;
        if (L.sharded) {   // the gathered end-of-run energies of every shard
            if (L.peers) wait_agg_slots(L, peer_epoch(st, 0x8000u + (uint32_t)T));
            const int64_t *table = agg_table(L, T);
            E = 0;
            for (int r = 0; r < L.shard_count; ++r) E += table[(size_t)AGG_SLOT * r + 5];
        }
        if (T - 1 < L.max_iters) L.tr_e[T - 1] = E;
        if (E < st->best_energy) {
            st->best_energy = E;
            st->best_iteration = T;
            st->ybest = st->ycur;
        }
    }
    st->energy_acc = 0;
    if (!st->converged) st->ycur = st->ybest;
    st->stop = 1;
}

// binarize (admm.py:202-204) of the current iterate: y >= 1/2 -> 1
__global__ void k_binarize(Lat2 L, int64_t n, uint8_t *out) {
    const ystore_t *y2 = L.y2[L.st->ycur];
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride)
        out[i] = (uint8_t)(y2[i] >= 1);
}

// 4*E of an arbitrary doubled labeling (y2 = 2y): 2*sum u*y2 + lamw*sum (y2_i-y2_j)^2
__global__ void k_energy4(Lat2 L, const int32_t *__restrict__ y2, int64_t n,
                          unsigned long long *out) {
    int64_t acc = 0;
    const int64_t HW = (int64_t)L.ay.dim * L.W;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
        const int32_t c = (int32_t)(i % L.W);
        const int64_t r = (i / L.W) % L.ay.dim, z = i / HW;
        const int32_t yi = y2[i];
        int64_t qd = 0;
        if (c + 1 < L.W) { const int64_t d = yi - y2[i + 1]; qd += d * d; }
        if (r + 1 < L.ay.dim) { const int64_t d = yi - y2[i + L.W]; qd += d * d; }
        if (z + 1 < L.az.dim) { const int64_t d = yi - y2[i + HW]; qd += d * d; }
        acc += 2 * (int64_t)L.u[i] * yi + (int64_t)L.lamw * qd;
    }
    acc = warp_sum(acc);
    if ((threadIdx.x & 31) == 0) atomicAdd(out, (unsigned long long)acc);
}

// ---------------------------------------------------------------------------
// Stamps of the clean-block consensus passes (dirty[2K, 7K), zeroed by
// init_state): [2K + b*K + k] = pass + 1 at which y buffer b last received
// block k's whole iterate, [5K + k] = pass + 1 of the last pass that changed
// block k's iterate, [6K + k] = pass + 1 of the last pass whose energy
// partial pe[k] holds E(y_{pass-1}) over block k's pairs (2D TMA pass).
__device__ __forceinline__ uint32_t *ybuf_stamp(const Lat2 &L, int b) { return L.dirty + (size_t)(2 + b) * L.K; }
__device__ __forceinline__ uint32_t *ychg_stamp(const Lat2 &L) { return L.dirty + (size_t)5 * L.K; }
__device__ __forceinline__ uint32_t *pe_stamp(const Lat2 &L) { return L.dirty + (size_t)6 * L.K; }

// Blocks solved since the last consensus pass, for the next pass to deal out
// evenly: dirty[7K, 8K) lists them, dirty[8K + k] = 1 + block k's latest
// slot, pc[6] = their count (zeroed by pass_tail and init).  Slot i holds a
// block for this pass iff i < count, list[i] = k, slot[k] = i + 1 and k's
// solve epoch is this iteration; the pass deals those out and handles every
// other solved block like any other block, so a stale list or count costs
// balance, never results.
__device__ __forceinline__ uint32_t *solved_list(const Lat2 &L) { return L.dirty + (size_t)7 * L.K; }
__device__ __forceinline__ uint32_t *solved_slot(const Lat2 &L) { return L.dirty + (size_t)8 * L.K; }
__device__ __forceinline__ int solved_count(const Lat2 &L) {
    const unsigned long long v = __ldcg(reinterpret_cast<const unsigned long long *>(&L.pc[6]));
    return v < (unsigned long long)L.K ? (int)v : L.K;
}

#include "consensus_tma.cuh"
#include "lattice3d.cuh"
#include "lattice3d_smem.cuh"

// ---------------------------------------------------------------------------
// Host side
// ---------------------------------------------------------------------------

struct Variant {
    int bh, bw, nt;
    size_t smem;
    void (*kernel)(Lat2, K1Tune);
    void (*kernel_wl)(Lat2, K1Tune);   // worklist mode (k_block_mincut_wl)
};

template <int BH, int BW, int NT>
static Variant make_variant() {
    return Variant{BH, BW, NT, K1Cfg<BH, BW, NT>::SMEM, &k_block_mincut<BH, BW, NT>, &k_block_mincut_wl<BH, BW, NT>};
}

static int sm_count();

static const Variant *pick_variant(int maxh, int maxw, int nblocks) {
    static const Variant table[] = {
        make_variant<16, 16, 64>(),
        make_variant<32, 32, 128>(),
        make_variant<64, 64, 256>(),
        make_variant<128, 128, 512>(),
    };
    // With few blocks per SM the K1 time is the slowest solve, not throughput:
    // twice the threads per block then pay (measured: C5 b64, K = 1024, K1
    // 23.0 -> 18.9 us; C3, K = 4096, 29.2 -> 31.0 us).  DOPE_K1_WIDE=0/1 forces.
    static const Variant wide64 = make_variant<64, 64, 512>();
    static const Variant wide128 = make_variant<128, 128, 1024>();
    static const int force = getenv("DOPE_K1_WIDE") ? atoi(getenv("DOPE_K1_WIDE")) : -1;
    const bool wide = force >= 0 ? force != 0 : nblocks <= 8 * sm_count();
    if (wide && maxh > 32 && maxw > 32 && maxh <= 64 && maxw <= 64) return &wide64;
    if (wide && maxh > 64 && maxw > 64 && maxh <= 128 && maxw <= 128) return &wide128;
    for (const Variant &v : table)
        if (maxh <= v.bh && maxw <= v.bw) return &v;
    return nullptr;
}

struct Variant3 {
    int bd, bh, bw, nt;
    size_t smem;
    void (*kernel)(Lat2, K1Tune);
};

template <int BD, int BH, int BW, int NT>
static Variant3 make_variant3() {
    return Variant3{BD, BH, BW, NT, K1Cfg3<BD, BH, BW, NT>::SMEM, &k_block_mincut3d<BD, BH, BW, NT>};
}

static const Variant3 *pick_variant3(int maxd, int maxh, int maxw) {
    static const Variant3 table[] = {
        make_variant3<16, 16, 16, 256>(),
        make_variant3<32, 32, 32, 512>(),
    };
    for (const Variant3 &v : table)
        if (maxd <= v.bd && maxh <= v.bh && maxw <= v.bw) return &v;
    return nullptr;
}

static int k2_tma_width(const Lat2 &o);
static int sm_count();
#ifndef K2T_CPS
#define K2T_CPS 4   // persistent TMA consensus CTAs per SM
#endif
constexpr int K2_CPS_FWD = K2T_CPS;

static int build_lat2(const dope_lattice *L, Lat2 &o, const Variant **var,
                      const Variant3 **var3 = nullptr) {
    if (!L || !L->u || !L->a || !L->y2[0] || !L->y2[1] || !L->y2[2] || !L->yhat || !L->resid ||
        !L->dirty || !L->part_energy || !L->part_unary || !L->part_ressq || !L->part_flags || !L->state ||
        (L->ndim == 2 && !L->part_cta))
        return DOPE_E_ARGS;
    const bool is3 = L->ndim == 3;
    if (!((L->ndim == 2 && L->conn == 4) || (is3 && L->conn == 6))) return DOPE_E_GEOMETRY;
    for (int a = 0; a < L->ndim; ++a) {
        if (L->dims[a] < 1 || L->kpa[a] < 1) return DOPE_E_ARGS;
        if (L->kpa[a] > L->dims[a]) return DOPE_E_ARGS;
    }
    const int64_t n = is3 ? L->dims[0] * L->dims[1] * L->dims[2] : L->dims[0] * L->dims[1];
    if (n > (int64_t)INT32_MAX) return DOPE_E_ARGS;
    if (L->mu <= 0 || L->lamw < 0 || (L->lamw % L->mu) != 0) return DOPE_E_ARGS;
    if (2 * (int64_t)L->lamw * 2 > 255) return DOPE_E_CAPACITY;   // r + r' = 2*cap <= 255
    if (is3 && !L->scratch) return DOPE_E_ARGS;
    memset(&o, 0, sizeof(o));
    o.ndim = L->ndim;
    if (is3) {
        o.az = make_axis(L->dims[0], L->kpa[0]);
        o.ay = make_axis(L->dims[1], L->kpa[1]);
        o.ax = make_axis(L->dims[2], L->kpa[2]);
        o.W = (int32_t)L->dims[2];
        o.K = L->kpa[0] * L->kpa[1] * L->kpa[2];
    } else {
        o.az = make_axis(1, 1);
        o.ay = make_axis(L->dims[0], L->kpa[0]);
        o.ax = make_axis(L->dims[1], L->kpa[1]);
        o.W = (int32_t)L->dims[1];
        o.K = L->kpa[0] * L->kpa[1];
    }
    o.lamw = L->lamw;
    o.mu = L->mu;
    o.q = L->lamw / L->mu;
    o.cap = 2 * L->lamw;
    o.warm = L->warm_start;
    o.skip_clean = L->skip_clean;
    o.fuse = L->fuse_multipliers;
    o.eps = L->eps;
    o.u = L->u;
    o.a = L->a;
    o.y2[0] = L->y2[0];
    o.y2[1] = L->y2[1];
    o.y2[2] = L->y2[2];
    o.yhat = L->yhat;
    o.resid = L->resid;
    o.scratch = L->scratch;
    o.dirty = L->dirty;
    o.pe = L->part_energy;
    o.pu = L->part_unary;
    o.pr = L->part_ressq;
    o.pf = L->part_flags;
    o.pc = L->part_cta;
    o.st = L->state;
    o.tr_e = L->trace_energy;
    o.tr_rs = L->trace_residual_sq;
    o.tr_mr = L->trace_max_residual;
    o.tr_cl = L->trace_clamped;
    o.timeline = L->timeline;
    o.max_iters = L->max_iters;
    o.gup = is3 ? 0 : L->ghost_up;
    o.gdn = is3 ? 0 : L->ghost_dn;
    o.gzu = is3 ? L->ghost_up : 0;
    o.gzd = is3 ? L->ghost_dn : 0;
    o.sharded = L->sharded;
    o.agg = L->agg;
    o.trace_hash = L->trace_hash;
    o.hash_base = L->hash_base;
    o.shard_index = L->sharded ? L->shard_index : 0;
    o.shard_count = L->sharded ? L->shard_count : 1;
    if (L->sharded && (L->shard_count < 1 || L->shard_index < 0 || L->shard_index >= L->shard_count))
        return DOPE_E_ARGS;
    // dirty-block worklists: run loop (fused pass, clean-block skipping) with a
    // K1 that deals them out (2D integer K1, shared-memory K1-3D)
    // (only with more blocks than the first K1 wave holds: with fewer, every
    // CTA starts at once and the list's extra round trip is pure cost -- C1)
    if (L->fuse_multipliers && L->skip_clean && !getenv("DOPE_NO_DLIST") && o.K > 2 * sm_count())
        o.dlist = L->dirty + (size_t)9 * o.K;
    if (L->sharded && L->halo) {
        const int64_t U = is3 ? L->dims[1] * L->dims[2] : L->dims[1];
        uint8_t *h = static_cast<uint8_t *>(L->halo);
        o.ga_up = reinterpret_cast<astore_t *>(h + halo_ga_offset(U));
        o.ga_dn = o.ga_up + U;
        o.pflags = reinterpret_cast<uint32_t *>(h + halo_flag_offset(U));
        if (L->peers) {
            if (L->shard_count > DOPE_MAX_SHARDS) return DOPE_E_ARGS;
            o.peers = L->peers;
        }
    }
    if (o.sharded && (!o.agg || (is3 ? o.az.rem != 0 : o.ay.rem != 0))) return DOPE_E_ARGS;
    const int maxd = o.az.base + (o.az.rem ? 1 : 0);
    const int maxh = o.ay.base + (o.ay.rem ? 1 : 0);
    const int maxw = o.ax.base + (o.ax.rem ? 1 : 0);
    if (is3) {
        const Variant3 *v3 = pick_variant3(maxd, maxh, maxw);
        if (!v3) return DOPE_E_GEOMETRY;
        o.boxd = v3->bd;
        o.boxh = v3->bh;
        o.boxw = v3->bw;
        if (var3) *var3 = v3;
        if (var) *var = nullptr;
    } else {
        const Variant *v = pick_variant(maxh, maxw, o.K);
        if (!v) return DOPE_E_GEOMETRY;
        o.boxd = 1;
        o.boxh = v->bh;
        o.boxw = v->bw;
        if (var) *var = v;
        if (var3) *var3 = nullptr;
    }
    // quad loads: 4 labels / 4 y2 bytes as one word, 4 multipliers as 8 bytes
    const uintptr_t al = (uintptr_t)o.y2[0] | (uintptr_t)o.y2[1] | (uintptr_t)o.y2[2] | (uintptr_t)o.yhat |
                         ((uintptr_t)o.a >> 1) | ((uintptr_t)o.u >> 2);
    o.pdl = getenv("DOPE_PDL") != nullptr;
    o.vec4 = !is3 && (o.W % 4 == 0) && (o.ax.rem == 0) && (o.ax.base % 4 == 0) && (al % 4 == 0);
    // the TMA consensus pass deals out the solved blocks when its CTAs hold
    // more than two blocks each
    o.slist = k2_tma_width(o) != 0 && o.K > 2 * K2_CPS_FWD * sm_count();
    // ... and shares phase B's tile-work blocks through a pass-wide queue
    if (o.slist && !getenv("DOPE_NO_K2Q")) o.kq = L->dirty + (size_t)12 * o.K + 2;
    o.q3 = is3 && (o.W % 4 == 0) && (al % 4 == 0);
    // 32^3 boxes with 2*cap <= 15 run the shared-memory K1 (nibble residuals);
    // DOPE_K1_3D=l2 forces the HBM-scratch kernel (diagnostics)
    static const bool k1_3d_l2 = [] {
        const char *e = getenv("DOPE_K1_3D");
        return e && strcmp(e, "l2") == 0;
    }();
    o.nib3 = is3 && !k1_3d_l2 && o.boxd == 32 && o.boxh == 32 && o.boxw == 32 && 2 * o.cap <= 15;
    if (is3 && !o.nib3) o.dlist = nullptr;   // the HBM-scratch K1-3D scans the flags
    return DOPE_OK;
}

// K1-3D (shared-memory kernel): a global relabel every 3 sweeps measured best
// on C4 (9.2 ms of K1 per 60-iteration run vs 15.5 ms at 1 + levels sweeps):
// in a 32^3 block excess that lost its path keeps sloshing until the next
// relabel marks it dead, and the all-warp BFS costs only ~0.4 us per level.
static K1Tune tune_3d() {
    static K1Tune t = [] {
        K1Tune x;
        x.sweep_min = 3;
        x.sweep_mul = 0;
        x.max_rounds = 1 << 16;
        if (const char *e = getenv("DOPE_SWEEP3_MIN")) x.sweep_min = atoi(e);
        if (const char *e = getenv("DOPE_SWEEP3_MUL")) x.sweep_mul = atoi(e);
        x.dense_min = x.sweep_min;
        x.dense_mul = x.sweep_mul;
        if (const char *e = getenv("DOPE_SWEEP3D_MIN")) x.dense_min = atoi(e);
        if (const char *e = getenv("DOPE_SWEEP3D_MUL")) x.dense_mul = atoi(e);
        return x;
    }();
    return t;
}

// 2D K1: a global relabel every 3 sweeps (measured over C1/C3/C5: C3 16.0k ->
// 17.5k it/s, C1 25k -> 41k, C5 +1-4 % vs 1 + levels sweeps per round).
static K1Tune default_tune() {
    static K1Tune t = [] {
        K1Tune x;
        x.sweep_min = 3;
        x.sweep_mul = 0;
        x.max_rounds = 1 << 16;
        if (const char *e = getenv("DOPE_SWEEP_MIN")) x.sweep_min = atoi(e);
        if (const char *e = getenv("DOPE_SWEEP_MUL")) x.sweep_mul = atoi(e);
        x.dense_min = x.sweep_min;
        x.dense_mul = x.sweep_mul;
        if (const char *e = getenv("DOPE_SWEEPD_MIN")) x.dense_min = atoi(e);
        if (const char *e = getenv("DOPE_SWEEPD_MUL")) x.dense_mul = atoi(e);
        return x;
    }();
    return t;
}

// Dense rounds (cold solves) with one block per SM at most: the solve's
// latency is K1's time and the one-warp BFS sits on the critical path, so
// a round sweeps 1 + levels times (C1, K = 16: 40.7k -> 48.2k it/s);
// with several waves of blocks, throughput counts and 3 sweeps per round
// stay best (C3 / C5 b32-b128, 1 / 2 / 6 / 12 / 24 / 1 + levels measured).
static K1Tune tune_2d(int nblocks) {
    K1Tune x = default_tune();
    if (!getenv("DOPE_SWEEPD_MIN") && !getenv("DOPE_SWEEPD_MUL") && nblocks <= sm_count()) {
        x.dense_min = 1;
        x.dense_mul = 1;
    }
    return x;
}

static int configure_k1(const Variant *v) {
    static std::mutex mu;
    static std::map<void *, bool> configured;
    std::lock_guard<std::mutex> lk(mu);
    if (!configured[(void *)v->kernel]) {
        int rc = cuda_check(cudaFuncSetAttribute(v->kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                 (int)v->smem), "cudaFuncSetAttribute(K1)");
        if (rc) return rc;
        rc = cuda_check(cudaFuncSetAttribute(v->kernel_wl, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             (int)v->smem), "cudaFuncSetAttribute(K1 worklist)");
        if (rc) return rc;
        configured[(void *)v->kernel] = true;
    }
    return DOPE_OK;
}

static int configure_k1_3d(const Variant3 *v) {
    static std::mutex mu;
    static std::map<void *, bool> configured;
    std::lock_guard<std::mutex> lk(mu);
    if (!configured[(void *)v->kernel]) {
        int rc = cuda_check(cudaFuncSetAttribute(v->kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                 (int)v->smem), "cudaFuncSetAttribute(K1-3D)");
        if (rc) return rc;
        if (v->bd == 32) {
            rc = cuda_check(cudaFuncSetAttribute(k_block_mincut3d_s, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                 (int)k1s::SMEM), "cudaFuncSetAttribute(K1-3D smem)");
            if (rc) return rc;
        }
        configured[(void *)v->kernel] = true;
    }
    return DOPE_OK;
}

struct Plan {
    Lat2 o;
    const Variant *v = nullptr;
    const Variant3 *v3 = nullptr;
    int64_t n = 0;
};

static int build_plan(const dope_lattice *L, Plan &P) {
    int rc = build_lat2(L, P.o, &P.v, &P.v3);
    if (rc) return rc;
    P.n = (int64_t)P.o.az.dim * P.o.ay.dim * P.o.W;
    return DOPE_OK;
}

static int configure_plan(const Plan &P) {
    return P.v3 ? configure_k1_3d(P.v3) : configure_k1(P.v);
}

// Launch with programmatic stream serialisation (PDL) when DOPE_PDL=1: the
// kernel may start while the previous one drains and orders itself with
// griddep_wait().  Off by default: measured neutral on C3 and 5-10 % slower on
// C5 (early-launched CTAs hold SM slots); same results either way.
template <typename... KArgs, typename... Args>
static cudaError_t launch_attr(bool pdl, void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                               Args... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = pdl ? 1 : 0;
    return cudaLaunchKernelEx(&cfg, kern, static_cast<KArgs>(args)...);
}

template <typename... KArgs, typename... Args>
static cudaError_t launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                              Args... args) {
    static const bool off = getenv("DOPE_PDL") == nullptr;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = off ? 0 : 1;
    return cudaLaunchKernelEx(&cfg, kern, static_cast<KArgs>(args)...);
}

// Audit mode: digest of (yhat, 2y, a) after the iteration (dope_lattice.trace_hash).
static int launch_digest(const Plan &P, cudaStream_t s) {
    if (!P.o.trace_hash) return DOPE_OK;
    const Lat2 &o = P.o;
    k_digest_begin<<<1, 1, 0, s>>>(o.st, o.trace_hash, o.max_iters);
    k_digest<dope_run_state, ystore_t, astore_t><<<2 * 148, 256, 0, s>>>(
        o.st, o.trace_hash, o.max_iters, P.n, o.hash_base, o.yhat, o.y2[0], o.y2[1], o.y2[2], o.a);
    return cuda_check(cudaGetLastError(), "state digest");
}

// resident CTAs of a 2D K1 worklist kernel per SM (its grid is one wave)
static int k1_wave(const Variant *v) {
    static std::mutex mu;
    static std::map<void *, int> occ;
    std::lock_guard<std::mutex> lk(mu);
    auto it = occ.find((void *)v->kernel_wl);
    if (it != occ.end()) return it->second;
    int n = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, v->kernel_wl, v->nt, v->smem) != cudaSuccess || n < 1) n = 1;
    occ[(void *)v->kernel_wl] = n;
    return n;
}

static int launch_k1(const Plan &P, cudaStream_t s) {
    int rc = configure_plan(P);
    if (rc) return rc;
    if (P.v3 && P.o.nib3) k_block_mincut3d_s<<<P.o.K, k1s::NT, k1s::SMEM, s>>>(P.o, tune_3d());
    else if (P.v3) P.v3->kernel<<<P.o.K, P.v3->nt, P.v3->smem, s>>>(P.o, default_tune());
    else {
        // worklist mode, DOPE_K1_WL=1: one wave walks the list (measured on C3:
        // the overlapped pass starts ~6 us earlier but ends no earlier, and the
        // cold iterations are slower); default: one CTA per block
        static const bool wl = getenv("DOPE_K1_WL") != nullptr;
        if (P.o.dlist && wl) {
            const int wave = k1_wave(P.v) * sm_count();
            return cuda_check(launch_pdl(P.v->kernel_wl, dim3(wave < P.o.K ? wave : P.o.K), dim3(P.v->nt),
                                         P.v->smem, s, P.o, tune_2d(P.o.K)),
                              "launch K1 (worklist)");
        }
        return cuda_check(launch_pdl(P.v->kernel, dim3(P.o.K), dim3(P.v->nt), P.v->smem, s, P.o, tune_2d(P.o.K)),
                          "launch K1");
    }
    return cuda_check(cudaGetLastError(), "launch K1");
}

static int k2_lq(const Lat2 &o) {
    // log2(quads per block row) when the vector kernel applies, else -1
    if (o.W % 4 != 0 || o.ax.rem != 0) return -1;
    for (int lq = 0; lq <= 5; ++lq)
        if (o.ax.base == (4 << lq)) return lq;
    return -1;
}

static PFN_cuTensorMapEncodeTiled_v12000 tmap_encoder() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        void *ptr = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(ptr);
    });
    return fn;
}

static bool make_map(CUtensorMap *m, CUtensorMapDataType dt, int esize, void *base, int64_t W,
                     int64_t H, int bw, int bh) {
    auto enc = tmap_encoder();
    if (!enc) return false;
    cuuint64_t dims[2] = {(cuuint64_t)W, (cuuint64_t)H};
    cuuint64_t strides[1] = {(cuuint64_t)(W * esize)};
    cuuint32_t box[2] = {(cuuint32_t)bw, (cuuint32_t)bh};
    cuuint32_t es[2] = {1, 1};
    return enc(m, dt, 2, base, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
               CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

static int sm_count() {
    static int n = 0;
    if (!n) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
        if (n <= 0) n = 148;
    }
    return n;
}

// persistent TMA consensus: run-loop mode, uniform tiling, 64/128-wide blocks
template <int TW, int TH, int NT, int ST>
static int k2_tma_attr() {
    return cuda_check(cudaFuncSetAttribute(k_consensus_tma<TW, TH, NT, ST>,
                                           cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           TmaCfg<TW, TH, NT, ST>::SMEM),
                      "attr K2");
}

template <int TW, int TH, int NT, int ST>
static int launch_k2_tma(const Lat2 &o, cudaStream_t s, int ctas_per_sm) {
    using C = TmaCfg<TW, TH, NT, ST>;
    if (o.ay.base % TH != 0) {
        snprintf(g_last_err, sizeof(g_last_err), "K2 tile height %d does not divide the block height", TH);
        return DOPE_E_GEOMETRY;
    }
    static std::once_flag once;
    std::call_once(once, [] { k2_tma_attr<TW, TH, NT, ST>(); });
    TmaMaps M;
    const int64_t W = o.W, H = o.ay.dim;
    bool ok = make_map(&M.a, CU_TENSOR_MAP_DATA_TYPE_UINT16, 2, o.a, W, H, TW, C::TH);
    // y2 and yhat carry one ghost row above and below the shard (caller-owned)
    for (int i = 0; i < 3 && ok; ++i) {
        ok = make_map(&M.y[i], CU_TENSOR_MAP_DATA_TYPE_UINT8, 1, o.y2[i] - W, W, H + 2, TW, C::TH + 1);
        ok = ok && make_map(&M.yr[i], CU_TENSOR_MAP_DATA_TYPE_UINT8, 1, o.y2[i] - W, W, H + 2, 16, C::TH);
        ok = ok && make_map(&M.yrow[i], CU_TENSOR_MAP_DATA_TYPE_UINT8, 1, o.y2[i] - W, W, H + 2, TW, 1);
    }
    ok = ok && make_map(&M.h16, CU_TENSOR_MAP_DATA_TYPE_UINT8, 1, o.yhat - W, W, H + 2, 16, 1);
    ok = ok && make_map(&M.yhat, CU_TENSOR_MAP_DATA_TYPE_UINT8, 1, o.yhat - W, W, H + 2, C::YHW, C::TH + 2);
    ok = ok && make_map(&M.hrow, CU_TENSOR_MAP_DATA_TYPE_UINT8, 1, o.yhat - W, W, H + 2, TW, 1);
    ok = ok && make_map(&M.hcol, CU_TENSOR_MAP_DATA_TYPE_UINT8, 1, o.yhat - W, W, H + 2, 16, C::TH);
    ok = ok && make_map(&M.arow, CU_TENSOR_MAP_DATA_TYPE_UINT16, 2, o.a, W, H, TW, 1);
    ok = ok && make_map(&M.acol, CU_TENSOR_MAP_DATA_TYPE_UINT16, 2, o.a, W, H, 8, C::TH);
    if (!ok) {
        snprintf(g_last_err, sizeof(g_last_err), "cuTensorMapEncodeTiled failed");
        return DOPE_E_CUDA;
    }
    // every CTA must be resident at once: with the tile-work queue a CTA
    // waits for all others to publish theirs (never more CTAs than fit)
    static int occ = -1;
    if (occ < 0 && cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_consensus_tma<TW, TH, NT, ST>, C::NT + 32,
                                                                  (size_t)C::SMEM) != cudaSuccess)
        occ = 1;
    static const int cps_env = getenv("DOPE_K2_CPS") ? atoi(getenv("DOPE_K2_CPS")) : 0;
    if (cps_env > 0) ctas_per_sm = cps_env;
    const int per_sm = ctas_per_sm < occ ? ctas_per_sm : (occ < 1 ? 1 : occ);
    int grid = per_sm * sm_count();
    grid = o.K < grid ? o.K : grid;
    const uint32_t magic = (uint32_t)(((1ull << 32) + o.ax.k - 1) / o.ax.k);
    // DOPE_K2_SETTLE=0: no ring-only / settled clean blocks (A/B diagnostics)
    static const int settle = getenv("DOPE_K2_SETTLE") ? atoi(getenv("DOPE_K2_SETTLE")) : 1;
    // (measured: with at most two blocks per CTA the settled / ring-only
    // modes do not pay for their metadata -- C5 b64 / b128)
    const int st_mode = settle && o.K > 2 * grid ? 1 : 0;
    if (o.ovl)   // overlap mode: a programmatic dependent of K1 (see k1_publish_done)
        return cuda_check(launch_attr(true, k_consensus_tma<TW, TH, NT, ST>, dim3(grid), dim3(C::NT + 32),
                                      (size_t)C::SMEM, s, o, M, magic, st_mode),
                          "launch K2 (tma, overlapped)");
    return cuda_check(launch_pdl(k_consensus_tma<TW, TH, NT, ST>, dim3(grid), dim3(C::NT + 32), (size_t)C::SMEM, s,
                                 o, M, magic, st_mode),
                      "launch K2 (tma)");
}

// measured on C3 (tools/k2_variants.sh)
constexpr int K2_TH = 64, K2_NT = 128, K2_STAGES = 2, K2_CPS = K2_CPS_FWD;

static int k2_tma_width(const Lat2 &o) {
    // eligible: run-loop mode, uniform tiling, 64/128-wide blocks, TMA-friendly strides
    if (!o.fuse || o.ax.rem != 0 || o.ay.rem != 0 || (o.W % 16) != 0 || o.ndim != 2) return 0;
    // TMA global addresses must be 16-byte aligned (y2 / yhat maps start one row up)
    const uintptr_t al = (uintptr_t)(o.y2[0] - o.W) | (uintptr_t)(o.y2[1] - o.W) | (uintptr_t)(o.y2[2] - o.W) |
                         (uintptr_t)(o.yhat - o.W) | (uintptr_t)o.a;
    if (al % 16 != 0 || !o.vec4) return 0;
    if (o.ax.base == 64 && o.ay.base % K2_TH == 0) return 64;
    if (o.ax.base == 128 && o.ay.base % (K2_TH / 2) == 0) return 128;
    return 0;
}

static int launch_k2(const Lat2 &o, cudaStream_t s) {
    if (o.ndim == 3) {
        // vector path: whole x quads per block row, 4-byte aligned rows
        const uintptr_t al = (uintptr_t)o.y2[0] | (uintptr_t)o.y2[1] | (uintptr_t)o.y2[2] | (uintptr_t)o.yhat |
                             ((uintptr_t)o.a >> 1);
        int lq = -1;
        for (int l = 0; l <= 5; ++l)
            if (o.ax.base == (4 << l)) lq = l;
        if (!getenv("DOPE_NO_VEC3") && !getenv("DOPE_NO_PLANE3") && lq == 3 && o.ax.rem == 0 &&
            o.ay.base == 32 && o.ay.rem == 0 && o.W % 4 == 0 && al % 8 == 0) {
            const int sms = sm_count();
            const int units = o.K * ((o.az.base + K2P_SLAB - 1) / K2P_SLAB);   // (block, slab) work units
            return cuda_check(launch_pdl(k_consensus3d_plane, dim3(units < 4 * sms ? units : 4 * sms), dim3(256), 0, s,
                                         o),
                              "launch K2-3D (plane)");
        }
        if (!getenv("DOPE_NO_VEC3") && lq >= 0 && o.ax.rem == 0 && o.W % 4 == 0 && al % 4 == 0) {
            const int sms = sm_count();
            const int v3 = getenv("DOPE_VEC3_NT") ? atoi(getenv("DOPE_VEC3_NT")) : 256;
            if (v3 == 512)
                return cuda_check(launch_pdl(k_consensus3d_vec<512>, dim3(o.K < 4 * sms ? o.K : 4 * sms), dim3(512),
                                             0, s, o, lq),
                                  "launch K2-3D (vec)");
            return cuda_check(launch_pdl(k_consensus3d_vec<256>, dim3(o.K < 4 * sms ? o.K : 4 * sms), dim3(256), 0,
                                         s, o, lq),
                              "launch K2-3D (vec)");
        }
        k_consensus3d<<<o.K, 512, 0, s>>>(o);
        return cuda_check(cudaGetLastError(), "launch K2-3D");
    }
    const int tw = k2_tma_width(o);
    static const int variant = getenv("DOPE_K2_VARIANT") ? atoi(getenv("DOPE_K2_VARIANT")) : 0;
    if (tw && !getenv("DOPE_NO_TMA")) {
        if (tw == 64) {
            switch (variant) {
                case 1: return launch_k2_tma<64, 16, 128, 6>(o, s, 4);
                case 2: return launch_k2_tma<64, 32, 128, 4>(o, s, 4);
                case 3: return launch_k2_tma<64, 16, 64, 8>(o, s, 6);
                case 4: return launch_k2_tma<64, 16, 128, 10>(o, s, 4);
                case 5: return launch_k2_tma<64, 32, 128, 3>(o, s, 4);
                case 6: return launch_k2_tma<64, 16, 128, 8>(o, s, 4);
                case 7: return launch_k2_tma<64, 16, 256, 8>(o, s, 2);
                default: return launch_k2_tma<64, K2_TH, K2_NT, K2_STAGES>(o, s, K2_CPS);
            }
        }
        return launch_k2_tma<128, K2_TH / 2, K2_NT, K2_STAGES>(o, s, K2_CPS);
    }
    const int lq = k2_lq(o);
    if (lq >= 0) {
        const int64_t quads = (int64_t)(o.ay.base + (o.ay.rem ? 1 : 0)) << lq;
        // persistent grids (a few thousand threads per SM): the last-CTA
        // counter and the aggregate atomics scale with CTAs, not blocks
        const int sms = sm_count();
        auto grid = [&](int per_sm) { return o.K < per_sm * sms ? o.K : per_sm * sms; };
        cudaError_t e;
        static const bool no_warp = getenv("DOPE_NO_K2_WARP") != nullptr;
        if (!no_warp && lq <= 3 && quads <= 256)   // blocks <= 32 x 32: a warp per block
        {
            static const int wv = getenv("DOPE_K2W_VAR") ? atoi(getenv("DOPE_K2W_VAR")) : -1;
            const int var = wv >= 0 ? wv : 0;   // 2 quads per batch at 4 CTAs/SM measured best (C5 b16, b32)
            if (var == 0) e = launch_pdl(k_consensus_warp<8, 2, 4>, dim3(grid(4)), dim3(256), 0, s, o, lq);
            else if (var == 1) e = launch_pdl(k_consensus_warp<8, 4, 3>, dim3(grid(3)), dim3(256), 0, s, o, lq);
            else e = launch_pdl(k_consensus_warp<8, 8, 2>, dim3(grid(2)), dim3(256), 0, s, o, lq);
        }
        else if (quads <= 4 * 32) e = launch_pdl(k_consensus_vec<32>, dim3(grid(32)), dim3(32), 0, s, o, lq);
        else if (quads <= 4 * 64) e = launch_pdl(k_consensus_vec<64>, dim3(grid(24)), dim3(64), 0, s, o, lq);
        else if (quads <= 4 * 256) e = launch_pdl(k_consensus_vec<256>, dim3(grid(8)), dim3(256), 0, s, o, lq);
        else if (quads <= 4 * 1024) e = launch_pdl(k_consensus_vec<1024>, dim3(grid(2)), dim3(1024), 0, s, o, lq);
        else e = launch_pdl(k_consensus, dim3(grid(8)), dim3(256), 0, s, o);
        return cuda_check(e, "launch K2");
    } else {
        const int sms = sm_count();
        return cuda_check(launch_pdl(k_consensus, dim3(o.K < 8 * sms ? o.K : 8 * sms), dim3(256), 0, s, o),
                          "launch K2");
    }
    return cuda_check(cudaGetLastError(), "launch K2");
}

static int grid_for(int64_t n) {
    int64_t b = (n + 255) / 256;
    if (b > 148 * 16) b = 148 * 16;
    return (int)(b < 1 ? 1 : b);
}

}  // namespace dope

using namespace dope;

extern "C" {

const char *dope_backend_name(void) { return "b200-sm100a"; }
int dope_abi_version(void) { return DOPE_ABI_VERSION; }
const char *dope_last_cuda_error(void) { return g_last_err; }

int64_t dope_resid_stride(const dope_lattice *L) {
    if (!L) return 0;
    if (L->ndim == 3) {
        for (int a = 0; a < 3; ++a)
            if (L->kpa[a] < 1 || L->dims[a] < 1) return 0;
        Axis az = make_axis(L->dims[0], L->kpa[0]), ay = make_axis(L->dims[1], L->kpa[1]),
             ax = make_axis(L->dims[2], L->kpa[2]);
        const Variant3 *v = pick_variant3(az.base + (az.rem ? 1 : 0), ay.base + (ay.rem ? 1 : 0),
                                          ax.base + (ax.rem ? 1 : 0));
        return v ? (int64_t)6 * v->bd * v->bh * v->bw : 0;
    }
    if (L->ndim != 2 || L->kpa[0] < 1 || L->kpa[1] < 1) return 0;
    Axis ay = make_axis(L->dims[0], L->kpa[0]), ax = make_axis(L->dims[1], L->kpa[1]);
    const Variant *v = pick_variant(ay.base + (ay.rem ? 1 : 0), ax.base + (ax.rem ? 1 : 0), 0);
    if (!v) return 0;
    return (int64_t)2 * v->bh * v->bw;   // E and S residual planes
}

int64_t dope_scratch_stride(const dope_lattice *L) {
    // 3D: excess (int32) + heights (uint16) per box node, 6 bytes (the
    // residual planes' 6 bytes give the same figure), then the int8 u brick
    // of the shared-memory K1 (box + 128-byte header) and 64 bytes of slab
    // accumulators for the 3D consensus pass; 2D keeps them in SMEM
    if (!L || L->ndim != 3) return 0;
    const int64_t six = dope_resid_stride(L);
    return six + six / 6 + 128 + 64;   // + the consensus pass's slab accumulators
}

int dope_lattice_check(const dope_lattice *L) {
    Plan P;
    return build_plan(L, P);
}

int dope_prepare_kernels(const dope_lattice *L) {
    // kernel attributes (dynamic shared memory) must be set outside stream capture
    Plan P;
    int rc = build_plan(L, P);
    if (rc) return rc;
    if ((rc = configure_plan(P))) return rc;
    if (P.o.ndim == 2 && P.o.fuse) {
        const int tw = k2_tma_width(P.o);
        if (tw == 64) return k2_tma_attr<64, K2_TH, K2_NT, K2_STAGES>();
        if (tw == 128) return k2_tma_attr<128, K2_TH / 2, K2_NT, K2_STAGES>();
    }
    return DOPE_OK;
}

int dope_admm_init(const dope_lattice *L, void *stream) {
    Plan P;
    int rc = build_plan(L, P);
    if (rc) return rc;
    cudaStream_t s = (cudaStream_t)stream;
    k_init_state<<<grid_for(P.n), 256, 0, s>>>(P.o, P.n);
    rc = cuda_check(cudaGetLastError(), "init_state");
    if (rc) return rc;
    k_init_unary<<<grid_for(P.n), 256, 0, s>>>(P.o, P.n);
    rc = cuda_check(cudaGetLastError(), "init_unary");
    if (rc) return rc;
    if (P.v3 && P.o.nib3) {
        k_init_ubrick<<<P.o.K, 256, 0, s>>>(P.o);
        rc = cuda_check(cudaGetLastError(), "init_ubrick");
        if (rc) return rc;
    }
    if (P.v3 && P.o.nib3) k_init_resid3d_nib<<<P.o.K, 256, 0, s>>>(P.o);
    else if (P.v3) k_init_resid3d<<<P.o.K, 256, 0, s>>>(P.o, P.o.boxd, P.o.boxh, P.o.boxw);
    else k_init_resid<<<P.o.K, 256, 0, s>>>(P.o);
    return cuda_check(cudaGetLastError(), "init_resid");
}

int dope_update_blocks(const dope_lattice *L, void *stream) {
    Plan P;
    int rc = build_plan(L, P);
    if (rc) return rc;
    return launch_k1(P, (cudaStream_t)stream);
}

int dope_update_global(const dope_lattice *L, void *stream) {
    Plan P;
    int rc = build_plan(L, P);
    if (rc) return rc;
    return launch_k2(P.o, (cudaStream_t)stream);
}

int dope_update_multipliers(const dope_lattice *L, void *stream) {
    Plan P;
    int rc = build_plan(L, P);
    if (rc) return rc;
    k_update_multipliers<<<grid_for(P.n), 256, 0, (cudaStream_t)stream>>>(P.o, P.n);
    return cuda_check(cudaGetLastError(), "update_multipliers");
}

// Overlap mode (run loop only: K1 and the consensus pass are adjacent in the
// stream): 2D integer K1 + the TMA consensus pass on one GPU.
static void enable_overlap(Plan &P) {
    static const bool off = getenv("DOPE_NO_OVL") != nullptr || getenv("DOPE_NO_TMA") != nullptr ||
                            getenv("DOPE_K2_VARIANT") != nullptr;
    if (off || !P.v || P.v3 || P.o.sharded || !P.o.skip_clean || !P.o.fuse || !k2_tma_width(P.o)) return;
    P.o.ovl = 1;
    P.o.pdl = 0;   // K1 itself is an ordinary launch (the previous pass complete)
    P.o.kdone = P.o.dirty + (size_t)11 * P.o.K + 2;
}

int dope_admm_run(const dope_lattice *L, int32_t iters, int32_t use_graph, void *stream) {
    Plan P;
    int rc = build_plan(L, P);
    if (rc) return rc;
    enable_overlap(P);
    cudaStream_t s = (cudaStream_t)stream;
    if (iters <= 0) return DOPE_OK;
    if ((rc = dope_rebuild_dirty_list(L, stream))) return rc;
    if (!use_graph) {
        for (int i = 0; i < iters; ++i) {
            if ((rc = launch_k1(P, s))) return rc;
            if ((rc = launch_k2(P.o, s))) return rc;
            if ((rc = launch_digest(P, s))) return rc;
        }
        return DOPE_OK;
    }
    // CUDA graph of `iters` iterations, cached by the lattice description
    static GraphCache cache;
    std::string key((const char *)L, sizeof(*L));
    key.append((const char *)&iters, sizeof(iters));
    cudaGraphExec_t exec = cache.find(key);
    if (!exec) {
        // kernel attributes must be set outside stream capture
        if ((rc = dope_prepare_kernels(L))) return rc;
        cudaStream_t cs;
        if ((rc = cuda_check(cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking), "stream"))) return rc;
        cudaGraph_t graph;
        if ((rc = cuda_check(cudaStreamBeginCapture(cs, cudaStreamCaptureModeThreadLocal), "capture"))) return rc;
        for (int i = 0; i < iters && !rc; ++i) {
            rc = launch_k1(P, cs);
            if (!rc) rc = launch_k2(P.o, cs);
            if (!rc) rc = launch_digest(P, cs);
        }
        cudaError_t e = cudaStreamEndCapture(cs, &graph);
        if (rc) return rc;
        if ((rc = cuda_check(e, "end capture"))) return rc;
        rc = cuda_check(cudaGraphInstantiate(&exec, graph, 0), "instantiate");
        cudaGraphDestroy(graph);
        cudaStreamDestroy(cs);
        if (rc) return rc;
        cache.put(key, exec);
    }
    return cuda_check(cudaGraphLaunch(exec, s), "graph launch");
}

int64_t dope_graph_cache_entries(void) { return graph_cache_entries_all(); }

void dope_graph_cache_clear(void) { graph_cache_clear_all(); }

static int launch_energy_current(const Lat2 &o, int64_t n, cudaStream_t s) {
    const uintptr_t al = (uintptr_t)o.y2[0] | (uintptr_t)o.y2[1] | (uintptr_t)o.y2[2];
    if (o.W % 4 == 0 && al % 4 == 0 && n / 4 < (int64_t)UINT32_MAX)
        k_energy_current_vec<<<grid_for(n / 4), 256, 0, s>>>(o, (uint32_t)(n / 4));
    else
        k_energy_current<<<grid_for(n), 256, 0, s>>>(o, n);
    return cuda_check(cudaGetLastError(), "energy_current");
}

int dope_finish_run(const dope_lattice *L, void *stream) {
    Plan P;
    int rc = build_plan(L, P);
    if (rc) return rc;
    cudaStream_t s = (cudaStream_t)stream;
    if ((rc = launch_energy_current(P.o, P.n, s))) return rc;
    k_finish_decide<<<1, 1, 0, s>>>(P.o);
    return cuda_check(cudaGetLastError(), "finish_decide");
}

int dope_decide(const dope_lattice *L, void *stream) {
    Plan P;
    int rc = build_plan(L, P);
    if (rc) return rc;
    if (!P.o.sharded) return DOPE_E_ARGS;
    k_decide<<<1, 1, 0, (cudaStream_t)stream>>>(P.o);
    return cuda_check(cudaGetLastError(), "decide");
}

int dope_ghost_update(const dope_lattice *L, int32_t which, const void *up_row, const void *dn_row,
                      void *stream) {
    Plan P;
    int rc = build_plan(L, P);
    if (rc) return rc;
    if (which != 0 && which != 1) return DOPE_E_ARGS;
    const int64_t unit = P.o.ndim == 3 ? (int64_t)P.o.ay.dim * P.o.W : (int64_t)P.o.W;
    k_ghost_update<<<grid_for(unit), 256, 0, (cudaStream_t)stream>>>(P.o, which, up_row, dn_row);
    return cuda_check(cudaGetLastError(), "ghost_update");
}

int dope_pack_rows(const dope_lattice *L, int32_t which, void *first_row, void *last_row,
                   void *stream) {
    Plan P;
    int rc = build_plan(L, P);
    if (rc) return rc;
    if (which != 0 && which != 1) return DOPE_E_ARGS;
    const int64_t unit = P.o.ndim == 3 ? (int64_t)P.o.ay.dim * P.o.W : (int64_t)P.o.W;
    k_pack_rows<<<grid_for(unit), 256, 0, (cudaStream_t)stream>>>(P.o, which, first_row, last_row);
    return cuda_check(cudaGetLastError(), "pack_rows");
}

int dope_energy_local(const dope_lattice *L, void *stream) {
    Plan P;
    int rc = build_plan(L, P);
    if (rc) return rc;
    if ((rc = launch_energy_current(P.o, P.n, (cudaStream_t)stream))) return rc;
    if (!P.o.sharded) return DOPE_OK;
    k_publish_energy<<<1, 1, 0, (cudaStream_t)stream>>>(P.o);
    return cuda_check(cudaGetLastError(), "publish_energy");
}

int64_t dope_halo_bytes(const dope_lattice *L) {
    if (!L || (L->ndim != 2 && L->ndim != 3)) return 0;
    return halo_bytes(L->ndim == 3 ? L->dims[1] * L->dims[2] : L->dims[1], L->shard_count);
}

int dope_ghost_consensus(const dope_lattice *L, void *stream) {
    Plan P;
    int rc = build_plan(L, P);
    if (rc) return rc;
    if (!P.o.sharded || !P.o.ga_up) return DOPE_E_ARGS;
    // the ghost unit's far-side neighbour must lie in its own block (blocks at
    // least two rows / planes deep along the sharded axis)
    if ((L->ghost_up || L->ghost_dn) && (P.o.ndim == 3 ? P.o.az.base : P.o.ay.base) < 2) return DOPE_E_GEOMETRY;
    const int64_t unit = P.o.ndim == 3 ? (int64_t)P.o.ay.dim * P.o.W : (int64_t)P.o.W;
    k_ghost_consensus<<<grid_for(unit), 256, 0, (cudaStream_t)stream>>>(P.o);
    return cuda_check(cudaGetLastError(), "ghost_consensus");
}

int dope_rebuild_dirty_list(const dope_lattice *L, void *stream) {
    Plan P;
    int rc = build_plan(L, P);
    if (rc) return rc;
    if (!P.o.dlist) return DOPE_OK;
    k_rebuild_dlist<<<1, 1024, 0, (cudaStream_t)stream>>>(P.o);
    return cuda_check(cudaGetLastError(), "rebuild_dlist");
}

int dope_unary_i32(const double *u, int64_t n, int32_t *out, int32_t *bad, void *stream) {
    if (n < 0 || (n && (!u || !out || !bad))) return DOPE_E_ARGS;
    if (n == 0) return DOPE_OK;
    k_unary_i32<<<grid_for(n), 256, 0, (cudaStream_t)stream>>>(u, n, out, bad);
    return cuda_check(cudaGetLastError(), "unary_i32");
}

int dope_host_register(void *ptr, int64_t bytes) {
    if (!ptr || bytes <= 0) return DOPE_E_ARGS;
    const cudaError_t e = cudaHostRegister(ptr, (size_t)bytes, cudaHostRegisterDefault);
    if (e != cudaSuccess) {
        (void)cudaGetLastError();   // not sticky: the caller falls back to staging
        return DOPE_E_CUDA;
    }
    return DOPE_OK;
}

int dope_host_unregister(void *ptr) {
    if (!ptr) return DOPE_E_ARGS;
    const cudaError_t e = cudaHostUnregister(ptr);
    if (e != cudaSuccess) {
        (void)cudaGetLastError();
        return DOPE_E_CUDA;
    }
    return DOPE_OK;
}

int dope_ghost_decide(const dope_lattice *L, void *stream) {
    Plan P;
    int rc = build_plan(L, P);
    if (rc) return rc;
    if (!P.o.sharded) return DOPE_E_ARGS;
    const bool ghosts = P.o.ga_up && (L->ghost_up || L->ghost_dn);
    if (ghosts && (P.o.ndim == 3 ? P.o.az.base : P.o.ay.base) < 2) return DOPE_E_GEOMETRY;
    const int64_t unit = P.o.ndim == 3 ? (int64_t)P.o.ay.dim * P.o.W : (int64_t)P.o.W;
    k_ghost_decide<<<ghosts ? grid_for(unit) : 1, 256, 0, (cudaStream_t)stream>>>(P.o);
    return cuda_check(cudaGetLastError(), "ghost_decide");
}

int dope_peer_install(const dope_lattice *L, void *stream) {
    Plan P;
    int rc = build_plan(L, P);
    if (rc) return rc;
    if (!P.o.peers || !P.o.ga_up) return DOPE_E_ARGS;
    k_peer_install<<<1, 256, 0, (cudaStream_t)stream>>>(P.o);
    return cuda_check(cudaGetLastError(), "peer_install");
}

int dope_trace_digest(const dope_lattice *L, void *stream) {
    Plan P;
    int rc = build_plan(L, P);
    if (rc) return rc;
    return launch_digest(P, (cudaStream_t)stream);
}

int dope_finish_decide(const dope_lattice *L, void *stream) {
    Plan P;
    int rc = build_plan(L, P);
    if (rc) return rc;
    k_finish_decide<<<1, 1, 0, (cudaStream_t)stream>>>(P.o);
    return cuda_check(cudaGetLastError(), "finish_decide");
}

int dope_binarize(const dope_lattice *L, uint8_t *out, void *stream) {
    Plan P;
    int rc = build_plan(L, P);
    if (rc) return rc;
    if (!out) return DOPE_E_ARGS;
    k_binarize<<<grid_for(P.n), 256, 0, (cudaStream_t)stream>>>(P.o, P.n, out);
    return cuda_check(cudaGetLastError(), "binarize");
}

int dope_energy4(const dope_lattice *L, const int32_t *y2, int64_t *out, void *stream) {
    Plan P;
    int rc = build_plan(L, P);
    if (rc) return rc;
    if (!y2 || !out) return DOPE_E_ARGS;
    cudaStream_t s = (cudaStream_t)stream;
    if ((rc = cuda_check(cudaMemsetAsync(out, 0, sizeof(int64_t), s), "memset"))) return rc;
    k_energy4<<<grid_for(P.n), 256, 0, s>>>(P.o, y2, P.n, (unsigned long long *)out);
    return cuda_check(cudaGetLastError(), "energy4");
}

}  // extern "C"
