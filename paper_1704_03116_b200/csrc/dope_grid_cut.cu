// dope_grid_cut.cu -- whole-grid serial graph cut on the GPU (SURVEY.md §8(f)
// row 2: cli.run_serial -> maxflow.solve_binary on the full image, the
// baseline of the compare mode, cli.py:95-100).
//
// One cooperative kernel over the whole 2D lattice (4- or 8-connected):
// capacities quantised once to int32 at scale qscale (1 for integer models:
// exact), excess in int64; rounds of
//   * global relabel: level-synchronous BFS from the deficit (sink-side)
//     nodes through residual arcs, grid-wide syncs between levels;
//   * push / relabel sweeps (push on admissible arcs h(w) = h(v) - 1 with
//     atomics on the excess, then monotone relabel);
// until no node with excess reaches a deficit.  Labels = nodes that reach a
// deficit in the final residual graph -- the minimal minimiser, the same set
// BK's sink tree yields (maxflow.py:100-108).
#include <cooperative_groups.h>
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>
#include <stdio.h>

#include "common.cuh"
#include "dope_b200.h"

namespace cg = cooperative_groups;

namespace dope_gc {
using namespace dope;

static thread_local char g_err[256] = "";
static int cuda_check(cudaError_t e, const char *what) {
    if (e == cudaSuccess) return DOPE_OK;
    snprintf(g_err, sizeof(g_err), "%s: %s", what, cudaGetErrorString(e));
    return DOPE_E_CUDA;
}

constexpr int32_t GINF = 0x3FFFFFFF;

struct GridCut {
    int32_t H, W, ndir;
    const double *tcap;          // n: signed terminal capacity (+ source / - sink)
    const double *w[4];          // E S SE SW pair weights (pair stored at the lower pixel)
    double lam, qs;
    int64_t *e;                  // n: excess (signed; < 0: remaining sink capacity)
    int32_t *rc;                 // ndir * n residuals, directions E W S N SE NW SW NE
    int32_t *h;                  // n
    int32_t *flags;              // 4 ints of grid-wide flags
    uint8_t *labels;             // n
    int64_t *stats;              // [rounds, sweeps, flow_q]
};

__device__ __forceinline__ int dy_of(int d) { return (d == 2 || d == 4 || d == 6) ? 1 : (d == 3 || d == 5 || d == 7) ? -1 : 0; }
__device__ __forceinline__ int dx_of(int d) { return (d == 0 || d == 4 || d == 7) ? 1 : (d == 1 || d == 5 || d == 6) ? -1 : 0; }

__device__ __forceinline__ double wpair(const GridCut &g, int R, int Cc, int d) {
    const int rn = R + dy_of(d), cn = Cc + dx_of(d);
    if (rn < 0 || rn >= g.H || cn < 0 || cn >= g.W) return 0.0;
    const int64_t W = g.W, G = (int64_t)R * W + Cc;
    switch (d) {
        case 0: return g.w[0][G];
        case 1: return g.w[0][G - 1];
        case 2: return g.w[1][G];
        case 3: return g.w[1][G - W];
        case 4: return g.w[2][G];
        case 5: return g.w[2][G - W - 1];
        case 6: return g.w[3][G];
        default: return g.w[3][G - W + 1];
    }
}

__device__ __forceinline__ int64_t nbr(const GridCut &g, int64_t v, int d) {
    return v + (int64_t)dy_of(d) * g.W + dx_of(d);
}

__global__ void k_gc_init(GridCut g) {
    const int64_t n = (int64_t)g.H * g.W;
    for (int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; v < n; v += (int64_t)gridDim.x * blockDim.x) {
        const int R = (int)(v / g.W), Cc = (int)(v - (int64_t)R * g.W);
        g.e[v] = (int64_t)llrint(g.tcap[v] * g.qs);
        for (int d = 0; d < g.ndir; ++d) {
            const double w = wpair(g, R, Cc, d);
            g.rc[(int64_t)d * n + v] = w > 0 ? (int32_t)llrint(g.lam * w * g.qs) : 0;
        }
    }
    if (blockIdx.x == 0 && threadIdx.x < 4) g.flags[threadIdx.x] = 0;
}

__global__ void __launch_bounds__(256) k_gc_solve(GridCut g, int sweep_min, int sweep_mul, int max_rounds) {
    cg::grid_group grid = cg::this_grid();
    const int64_t n = (int64_t)g.H * g.W;
    const int64_t t0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    int rounds = 0;
    int64_t sweeps = 0;
    for (;;) {
        // ---- global relabel: exact distances to the deficit set ----
        for (int64_t v = t0; v < n; v += stride) g.h[v] = g.e[v] < 0 ? 0 : GINF;
        if (t0 == 0) g.flags[0] = g.flags[1] = 0;
        grid.sync();
        for (int L = 0;; ++L) {
            int changed = 0;
            for (int64_t v = t0; v < n; v += stride) {
                if (g.h[v] != GINF) continue;
                const int R = (int)(v / g.W), Cc = (int)(v - (int64_t)R * g.W);
                for (int d = 0; d < g.ndir; ++d) {
                    if (g.rc[(int64_t)d * n + v] == 0) continue;
                    const int rn = R + dy_of(d), cn = Cc + dx_of(d);
                    if (rn < 0 || rn >= g.H || cn < 0 || cn >= g.W) continue;
                    if (g.h[nbr(g, v, d)] == L) {
                        g.h[v] = L + 1;
                        changed = 1;
                        break;
                    }
                }
            }
            if (__syncthreads_or(changed) && threadIdx.x == 0) atomicOr(&g.flags[L & 1], 1);
            grid.sync();
            const int any = g.flags[L & 1];
            grid.sync();   // everyone has read the flag before it is reused
            if (t0 == 0) g.flags[L & 1] = 0;
            if (!any) break;
        }
        // any excess that still reaches a deficit?
        int hit = 0;
        for (int64_t v = t0; v < n; v += stride) hit |= (g.e[v] > 0 && g.h[v] != GINF);
        if (__syncthreads_or(hit) && threadIdx.x == 0) atomicOr(&g.flags[2], 1);
        grid.sync();
        const int go = g.flags[2];
        grid.sync();
        if (t0 == 0) g.flags[2] = 0;
        if (!go) break;
        if (++rounds > max_rounds) {
            if (t0 == 0) g.stats[0] = -1;
            break;
        }
        // ---- push / relabel sweeps ----
        const int cap_sweeps = sweep_min + sweep_mul * 4;
        for (int sw = 0; sw < cap_sweeps; ++sw) {
            ++sweeps;
            for (int64_t v = t0; v < n; v += stride) {
                const int64_t ex = g.e[v];
                if (ex <= 0) continue;
                const int32_t hv = g.h[v];
                if (hv == GINF || hv == 0) continue;
                const int R = (int)(v / g.W), Cc = (int)(v - (int64_t)R * g.W);
                int64_t left = ex;
                for (int d = 0; d < g.ndir && left > 0; ++d) {
                    const int64_t ri = (int64_t)d * n + v;
                    const int32_t rv = g.rc[ri];
                    if (rv == 0) continue;
                    const int rn = R + dy_of(d), cn = Cc + dx_of(d);
                    if (rn < 0 || rn >= g.H || cn < 0 || cn >= g.W) continue;
                    const int64_t w = nbr(g, v, d);
                    if (g.h[w] != hv - 1) continue;
                    const int32_t delta = left < rv ? (int32_t)left : rv;
                    g.rc[ri] = rv - delta;
                    g.rc[(int64_t)(d ^ 1) * n + w] += delta;   // only this push touches the arc pair now
                    atomicAdd(reinterpret_cast<unsigned long long *>(&g.e[w]), (unsigned long long)(int64_t)delta);
                    left -= delta;
                }
                if (left != ex)
                    atomicAdd(reinterpret_cast<unsigned long long *>(&g.e[v]), (unsigned long long)(left - ex));
            }
            grid.sync();
            int act = 0;
            for (int64_t v = t0; v < n; v += stride) {
                if (g.e[v] <= 0) continue;
                const int32_t hv = g.h[v];
                if (hv == GINF) continue;
                const int R = (int)(v / g.W), Cc = (int)(v - (int64_t)R * g.W);
                int32_t mn = GINF;
                for (int d = 0; d < g.ndir; ++d) {
                    if (g.rc[(int64_t)d * n + v] == 0) continue;
                    const int rn = R + dy_of(d), cn = Cc + dx_of(d);
                    if (rn < 0 || rn >= g.H || cn < 0 || cn >= g.W) continue;
                    const int32_t hw = g.h[nbr(g, v, d)];
                    mn = hw < mn ? hw : mn;
                }
                const int32_t nh = mn >= GINF - 1 ? GINF : mn + 1;
                if (nh != hv) g.h[v] = nh;
                act |= nh != GINF;
            }
            if (__syncthreads_or(act) && threadIdx.x == 0) atomicOr(&g.flags[3], 1);
            grid.sync();
            const int more = g.flags[3];
            grid.sync();
            if (t0 == 0) g.flags[3] = 0;
            if (!more) break;
        }
    }
    // labels: the deficit-reachable set of the last relabel
    for (int64_t v = t0; v < n; v += stride) g.labels[v] = g.h[v] != GINF ? 1 : 0;
    if (t0 == 0) {
        if (g.stats[0] >= 0) g.stats[0] = rounds;
        g.stats[1] = sweeps;
    }
}

}  // namespace dope_gc

using namespace dope_gc;

extern "C" {

const char *dope_gc_last_error(void) { return g_err; }

int64_t dope_gc_workspace_bytes(int64_t H, int64_t W, int32_t conn) {
    if (H < 1 || W < 1 || (conn != 4 && conn != 8)) return -1;
    const int64_t n = H * W;
    return n * 8 + (int64_t)conn * n * 4 + n * 4 + 64;
}

int dope_gc_mincut(int64_t H, int64_t W, int32_t conn, const double *tcap, const double *const *w, double lam,
                   double qscale, uint8_t *labels, int64_t *stats, void *workspace, int64_t ws_bytes, void *stream) {
    if (H < 1 || W < 1 || H * W > INT32_MAX || (conn != 4 && conn != 8) || !tcap || !w || !labels || !stats ||
        !workspace || !(qscale > 0) || lam < 0)
        return DOPE_E_ARGS;
    if (ws_bytes < dope_gc_workspace_bytes(H, W, conn)) return DOPE_E_ARGS;
    GridCut g;
    g.H = (int32_t)H;
    g.W = (int32_t)W;
    g.ndir = conn;
    g.tcap = tcap;
    for (int i = 0; i < 4; ++i) g.w[i] = (i < (conn == 8 ? 4 : 2)) ? w[i] : nullptr;
    g.lam = lam;
    g.qs = qscale;
    const int64_t n = H * W;
    uint8_t *p = static_cast<uint8_t *>(workspace);
    g.e = reinterpret_cast<int64_t *>(p);
    g.rc = reinterpret_cast<int32_t *>(p + n * 8);
    g.h = reinterpret_cast<int32_t *>(p + n * 8 + (int64_t)conn * n * 4);
    g.flags = reinterpret_cast<int32_t *>(p + n * 8 + (int64_t)conn * n * 4 + n * 4);
    g.labels = labels;
    g.stats = stats;
    cudaStream_t s = (cudaStream_t)stream;
    int rc = cuda_check(cudaMemsetAsync(stats, 0, 3 * sizeof(int64_t), s), "memset");
    if (rc) return rc;
    k_gc_init<<<1184, 256, 0, s>>>(g);
    if ((rc = cuda_check(cudaGetLastError(), "gc init"))) return rc;
    int dev = 0, sms = 0, per = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if ((rc = cuda_check(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_gc_solve, 256, 0), "occupancy")))
        return rc;
    int grid = per * sms;
    const int64_t need = (n + 255) / 256;
    if (need < grid) grid = (int)need;
    int smin = 1, smul = 1, mr = 1 << 20;
    void *args[] = {&g, &smin, &smul, &mr};
    return cuda_check(cudaLaunchCooperativeKernel((void *)k_gc_solve, dim3(grid), dim3(256), args, 0, s),
                      "gc solve");
}

}  // extern "C"
