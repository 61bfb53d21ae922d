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
    static constexpr size_t OFF_REACH = OFF_MASK + 8 * (size_t)(NDIR + 2) * NW;
    static constexpr size_t OFF_MISC = OFF_REACH + 8 * (size_t)NW;
    static constexpr size_t SMEM = OFF_MISC + 64;
};

// Solve the staged block: g = signed terminal excess (int32, >0 source side),
// rr[d*M + v] = residual of arc v -> v + off(d) (directions E W S N SE NW SW NE,
// opposite = d ^ 1).  Leaves the sink-reachable set in reach[].  Returns the
// number of global-relabel rounds, or -1 past the round limit.
template <int BH, int BW, int NT, int NDIR>
__device__ int mincut_solve(int32_t *g, int32_t *rr, uint16_t *h, uint64_t *masks, uint64_t *reach, int *misc,
                            int sweep_min, int sweep_mul) {
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
            h[v] = gvv < 0 ? 0 : HINF;
            if (lane == 0) {
                const int w32 = (i * NT + warp * 32) >> 5;
#pragma unroll
                for (int d = 0; d < NDIR; ++d) masks32[d * 2 * NW + w32] = b[d];
                masks32[NDIR * 2 * NW + w32] = bK;
                masks32[(NDIR + 1) * 2 * NW + w32] = bA;
            }
        }
        __syncthreads();
        if (warp == 0) {
            int levels = 0;
            const int hit = bfs_relabel<NW, BW, 0, NDIR == 8>(masks, reach, h, lane, &levels);
            if (lane == 0) { misc[0] = hit; misc[1] = levels; }
        }
        __syncthreads();
        const int hit = misc[0], levels = misc[1];
        if (!hit) break;
        if (++rounds > (1 << 16)) return -1;
        const int cap_sweeps = sweep_min + sweep_mul * levels;
        for (int sw = 0; sw < cap_sweeps; ++sw) {
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
    }
    return rounds;
}

}  // namespace dope_f
