// mincut_core.cuh -- the block min-cut solve shared by the float-weight and
// the general (overlapping) lattice paths: quantised int32 capacities staged
// in shared memory, rounds of (warp-ballot masks, one-warp bit-parallel
// global-relabel BFS from the sink set, push/relabel sweeps); labels = the
// BFS's sink-reachable set left in `reach`.
#pragma once
#include "common.cuh"

namespace dope_f {
using namespace dope;

template <int BH, int BW, int NT, int NDIR>
struct K1FCfg {
    static constexpr int M = BH * BW;
    static constexpr int NPT = M / NT;
    static constexpr int NW = M / 64;
    static constexpr size_t OFF_G = 0;
    static constexpr size_t OFF_R = OFF_G + 4 * (size_t)M;
    static constexpr size_t OFF_H = OFF_R + 4 * (size_t)NDIR * M;
    static constexpr size_t OFF_MASK = OFF_H + 2 * (size_t)M;
    // BFS masks; during the sweeps the relabel candidates + one 32-slot row per warp
    static constexpr size_t MASKB = 8 * (size_t)(NDIR + 2) * NW > 8 * (size_t)NW + (NT / 32) * 64
                                        ? 8 * (size_t)(NDIR + 2) * NW
                                        : 8 * (size_t)NW + (NT / 32) * 64;
    static constexpr size_t OFF_REACH = OFF_MASK + MASKB;
    static constexpr size_t OFF_MISC = OFF_REACH + 8 * (size_t)NW;
    static constexpr size_t SMEM = OFF_MISC + 64;
};

// Solve the staged block: g = signed terminal excess (int32, >0 source side),
// rr[d*M + v] = residual of arc v -> v + off(d) (directions E W S N SE NW SW NE,
// opposite = d ^ 1).  Leaves the sink-reachable set in reach[].  Returns the
// number of global-relabel rounds, or -1 past the round limit.
// ---- bulk (TMA) copies of a block's residual planes, one issuing thread ----
__device__ __forceinline__ uint32_t mc_smem(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mc_bar_init(uint64_t *bar) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(mc_smem(bar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mc_bar_expect(uint64_t *bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(mc_smem(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mc_bar_wait(uint64_t *bar, uint32_t parity) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "MCWAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, %2;\n"
        "@!p bra MCWAIT_%=;\n"
        "}\n" ::"r"(mc_smem(bar)), "r"(parity), "r"(0x989680) : "memory");
}
__device__ __forceinline__ void mc_bulk_load(void *dst, const void *src, uint32_t bytes, uint64_t *bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 ::"r"(mc_smem(dst)), "l"(src), "r"(bytes), "r"(mc_smem(bar)) : "memory");
}
__device__ __forceinline__ void mc_bulk_store(void *dst, const void *src, uint32_t bytes) {
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;"
                 ::"l"(dst), "r"(mc_smem(src)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mc_bulk_store_wait() {
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

#ifdef K1F_DIAG
static __device__ long long g_k1f_diag[16 * 4096];
__device__ __forceinline__ long long k1f_now() {
    long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
#define K1F_D(slot, expr) do { if (threadIdx.x == 0 && blockIdx.x < 4096) g_k1f_diag[16 * blockIdx.x + (slot)] expr; } while (0)
#else
#define K1F_D(slot, expr) do { } while (0)
#endif

// Work for the warps that wait while warp 0 runs a global-relabel BFS alone:
// idle(i) is called by every thread of warps 1 .. NT/32 - 1 during the i-th BFS
// of the solve (i = 0, 1, ...; the same count on every thread).
struct NoIdle {
    __device__ __forceinline__ void operator()(int) const {}
};

template <int BH, int BW, int NT, int NDIR, class Idle = NoIdle>
__device__ int mincut_solve(int32_t *g, int32_t *rr, uint16_t *h, uint64_t *masks, uint64_t *reach, int *misc,
                            int sweep_min, int sweep_mul, Idle idle = Idle()) {
    using Cf = K1FCfg<BH, BW, NT, NDIR>;
    constexpr int M = Cf::M, NPT = Cf::NPT, NW = Cf::NW;
    uint32_t *masks32 = reinterpret_cast<uint32_t *>(masks);
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    constexpr int OFFS[8] = {1, -1, BW, -BW, BW + 1, -BW - 1, BW - 1, -BW + 1};
    int rounds = 0;
    for (;;) {
        for (int i = 0; i < NPT; ++i) {
            const int v = tid + i * NT;
            const int32_t gvv = g[v];
            uint32_t b[NDIR];
#pragma unroll
            for (int d = 0; d < NDIR; ++d) b[d] = __ballot_sync(FULLMASK, rr[d * M + v] != 0);
            const uint32_t bK = __ballot_sync(FULLMASK, gvv < 0);
            const uint32_t bA = __ballot_sync(FULLMASK, gvv > 0);
            if (lane == 0) {
                const int w32 = (i * NT + warp * 32) >> 5;
#pragma unroll
                for (int d = 0; d < NDIR; ++d) masks32[d * 2 * NW + w32] = b[d];
                masks32[NDIR * 2 * NW + w32] = bK;
                masks32[(NDIR + 1) * 2 * NW + w32] = bA;
            }
        }
        // level planes of the BFS live in the height array until they are decoded
        uint64_t *planes = reinterpret_cast<uint64_t *>(h);
        for (int w = tid; w < M / 4; w += NT) planes[w] = 0ull;
        __syncthreads();
        if (warp == 0) {
            int levels = 0;
            const int hit = bfs_relabel_planes<NW, BW, 0, NDIR == 8>(masks, reach, planes, lane, &levels);
            if (lane == 0) { misc[0] = hit; misc[1] = levels; }
        } else {
            idle(rounds);
        }
        __syncthreads();
        const int hit = misc[0], levels = misc[1];
        K1F_D(4, += levels);
        K1F_D(8, = rounds == 0 ? k1f_now() : g_k1f_diag[16 * blockIdx.x + 8]);
        if (!hit) break;
        if (++rounds > (1 << 16)) return -1;
        levels_to_heights<M, NT>(planes, reach, h, levels);   // published by the barriers below
        // sweeps per relabel: min + mul * levels; dense rounds (cold solves) may
        // carry their own pair in the high halves of the two arguments
        const int cap_sweeps = (sweep_min & 0xFFFF) + (sweep_mul & 0xFFFF) * levels;
        const int cap_dense = (sweep_min >> 16) ? (sweep_min >> 16) + (sweep_mul >> 16) * levels : cap_sweeps;
        // Sweeps over candidate bitmasks, as in the integer K1
        // (dope_lattice.cu): C = nodes to push from (reach & active after the
        // BFS), N = nodes to relabel; each warp compacts the set bits of its
        // 32-node groups into batches of 32, one node per lane.
        uint32_t *candC = reinterpret_cast<uint32_t *>(reach);
        uint32_t *candN = masks32;
        uint16_t *slots = reinterpret_cast<uint16_t *>(masks32 + 2 * NW) + warp * 32;
        static_assert(8 * NW + (NT / 32) * 64 <= Cf::MASKB, "candidate masks and slots fit");
        static_assert(NPT <= 32, "one group word per lane");
        // dense rounds (most nodes active) sweep every node as plain loops
        if (tid == 0) misc[2] = 0;
        __syncthreads();
        {
            int myc = 0;
            for (int w = tid; w < 2 * NW; w += NT) {
                const uint32_t c = candC[w] & masks32[(NDIR + 1) * 2 * NW + w];
                candC[w] = c;
                myc += __popc(c);
            }
            if (myc) atomicAdd(&misc[2], myc);
        }
        __syncthreads();
        K1F_D(9, += misc[2]);
        if (misc[2] > M / 16) {
            K1F_D(6, += 1);
            for (int sw = 0; sw < cap_dense; ++sw) {
                K1F_D(5, += 1);
                for (int i = 0; i < NPT; ++i) {
                    const int v = tid + i * NT;
                    const int32_t e = g[v];
                    if (e <= 0) continue;
                    const uint16_t hv = h[v];
                    if (hv == HINF || hv == 0) continue;
                    const uint16_t ht = hv - 1;
                    int32_t left = e;
#pragma unroll
                    for (int d = 0; d < NDIR; ++d) {
                        const int32_t rv = rr[d * M + v];
                        if (rv == 0) continue;
                        const int w = v + OFFS[d];
                        if (h[w] != ht) continue;
                        const int32_t delta = left < rv ? left : rv;
                        rr[d * M + v] = rv - delta;
                        rr[(d ^ 1) * M + w] += delta;
                        atomicAdd(&g[w], delta);
                        left -= delta;
                        if (left == 0) break;
                    }
                    if (left != e) atomicSub(&g[v], e - left);
                }
                __syncthreads();
                int act = 0;
                for (int i = 0; i < NPT; ++i) {
                    const int v = tid + i * NT;
                    if (g[v] <= 0) continue;
                    const uint16_t hv = h[v];
                    if (hv == HINF) continue;
                    uint32_t mn = HINF;
#pragma unroll
                    for (int d = 0; d < NDIR; ++d) {
                        if (rr[d * M + v] == 0) continue;
                        const uint32_t hw = h[v + OFFS[d]];
                        mn = hw < mn ? hw : mn;
                    }
                    const uint32_t nh = (mn + 1 >= (uint32_t)M) ? HINF : mn + 1;
                    if (nh != hv) h[v] = (uint16_t)nh;
                    act |= (nh != HINF);
                }
                if (!__syncthreads_or(act)) break;
            }
            continue;
        }
        for (int w = tid; w < 2 * NW; w += NT) candN[w] = 0u;
        __syncthreads();
        for (int sw = 0; sw < cap_sweeps; ++sw) {
            int act = 0;
            K1F_D(5, += 1);
#pragma unroll 1
            for (int phase = 0; phase < 2; ++phase) {   // 0: push from C, 1: relabel N
                uint32_t *cand = phase == 0 ? candC : candN;
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
                        uint32_t lt;
                        asm("mov.u32 %0, %%lanemask_lt;" : "=r"(lt));
                        const int rank = __popc(word & lt);
                        const int room = 32 - cnt;
                        if (mine && rank < room) slots[cnt + rank] = (uint16_t)v;
                        const int nw = __popc(word);
                        word = __ballot_sync(FULLMASK, mine && rank >= room);
                        const int fill = cnt + (nw < room ? nw : room);
                        if (fill < 32 && !(tail && word == 0u)) {
                            cnt = fill;
                            continue;
                        }
                        __syncwarp();
                        if (lane < fill) {
                            const int u = slots[lane];
                            const int32_t e = g[u];
                            const uint16_t hu = h[u];
                            if (phase == 0) {
                                if (e > 0 && hu != HINF) {
                                    int32_t left = e;
                                    if (hu != 0) {
                                        const uint16_t ht = hu - 1;
                                        // every arc's residual and head height first (independent
                                        // loads), then the sequential split of the excess
                                        int32_t rvs[NDIR];
                                        uint16_t hws[NDIR];
#pragma unroll
                                        for (int d = 0; d < NDIR; ++d) {
                                            rvs[d] = rr[d * M + u];
                                            const int w = u + OFFS[d];
                                            hws[d] = h[w < 0 ? 0 : (w >= M ? M - 1 : w)];
                                        }
#pragma unroll
                                        for (int d = 0; d < NDIR; ++d) {
                                            const int32_t rv = rvs[d];
                                            if (rv == 0) continue;
                                            const int w = u + OFFS[d];
                                            if (hws[d] != ht) continue;
                                            const int32_t delta = left < rv ? left : rv;
                                            DOPE_ASSERT(w >= 0 && w < M && delta > 0 && h[w] == ht &&
                                                        rr[d * M + u] == rv);
                                            rr[d * M + u] = rv - delta;
                                            rr[(d ^ 1) * M + w] += delta;
                                            atomicAdd(&g[w], delta);
                                            atomicOr(&candN[w >> 5], 1u << (w & 31));
                                            left -= delta;
                                            if (left == 0) break;
                                        }
                                        if (left != e) atomicSub(&g[u], e - left);
                                    }
                                    if (left > 0) atomicOr(&candN[u >> 5], 1u << (u & 31));
                                }
                            } else if (e > 0 && hu != HINF) {
                                uint32_t mn = HINF;
#pragma unroll
                                for (int d = 0; d < NDIR; ++d) {   // independent loads (clamped index)
                                    const int w = u + OFFS[d];
                                    const uint32_t hw = h[w < 0 ? 0 : (w >= M ? M - 1 : w)];
                                    const uint32_t cand = rr[d * M + u] != 0 ? hw : (uint32_t)HINF;
                                    mn = cand < mn ? cand : mn;
                                }
                                const uint32_t nh = (mn + 1 >= (uint32_t)M) ? HINF : mn + 1;
                                if (nh != hu) h[u] = (uint16_t)nh;
                                if (nh != HINF) {
                                    act = 1;
                                    atomicOr(&candC[u >> 5], 1u << (u & 31));
                                }
                            }
                        }
                        __syncwarp();
                        cnt = 0;
                    }
                }
                if (phase == 0) __syncthreads();
            }
            if (!__syncthreads_or(act)) break;
        }
    }
    return rounds;
}

}  // namespace dope_f
