// dope_graph.cu -- seam 1 of include/dope_b200.h: min cut of one general
// two-terminal graph given as pair arcs, the contract of the reference's
// kernel backend bk_maxflow (/root/reference/pkg/src/dope/_core.pyx:263-333,
// _core_py.py:25-35).
//
// One CTA solves one graph with push-relabel in float64:
//   * arcs 2p: i->j (cap_ij[p]) and 2p+1: j->i (cap_ji[p]) (_core.pyx:293-297),
//     tail-grouped adjacency in pair order (_core.pyx:298-310);
//   * residuals <= EPS (1e-12) count as saturated, |tcap| <= EPS as no
//     terminal arc (_core.pyx:13, 41-58);
//   * excess is accumulated by PULLING each phase's per-arc pushes in
//     adjacency order, so the arithmetic (hence flow and labels) is
//     deterministic run to run;
//   * global relabel = level-synchronous BFS from the sink set over reverse
//     residual arcs; the final complete BFS gives labels = sink-reachable
//     nodes, which for a maximum preflow is the unique minimal sink side of
//     the minimum cut -- the set the reference's BK sink tree equals.
#include <cuda_runtime.h>
#include <stdint.h>

#include "common.cuh"
#include "dope_b200.h"

namespace dope_graph {

constexpr double EPS = 1e-12;
constexpr int HINF = 0x3fffffff;
constexpr int NT = 1024;

struct Ws {
    double *g, *rc, *fl;
    int *h, *off, *adj, *head, *fill, *q0, *q1;
    int *misc;
};

__host__ __device__ inline size_t align8(size_t x) { return (x + 7) & ~(size_t)7; }

__host__ __device__ inline size_t ws_layout(int32_t m, int64_t P, Ws *w, char *base) {
    size_t o = 0;
    auto take = [&](size_t bytes) { size_t at = o; o = align8(o + bytes); return at; };
    size_t og = take(sizeof(double) * (m > 0 ? m : 1));
    size_t orc = take(sizeof(double) * (2 * P > 0 ? 2 * P : 1));
    size_t ofl = take(sizeof(double) * (2 * P > 0 ? 2 * P : 1));
    size_t oh = take(sizeof(int) * (m > 0 ? m : 1));
    size_t ooff = take(sizeof(int) * (m + 1));
    size_t oadj = take(sizeof(int) * (2 * P > 0 ? 2 * P : 1));
    size_t ohead = take(sizeof(int) * (2 * P > 0 ? 2 * P : 1));
    size_t ofill = take(sizeof(int) * (m > 0 ? m : 1));
    size_t oq0 = take(sizeof(int) * (m > 0 ? m : 1));
    size_t oq1 = take(sizeof(int) * (m > 0 ? m : 1));
    size_t omisc = take(sizeof(int) * 16);
    if (w && base) {
        w->g = (double *)(base + og);
        w->rc = (double *)(base + orc);
        w->fl = (double *)(base + ofl);
        w->h = (int *)(base + oh);
        w->off = (int *)(base + ooff);
        w->adj = (int *)(base + oadj);
        w->head = (int *)(base + ohead);
        w->fill = (int *)(base + ofill);
        w->q0 = (int *)(base + oq0);
        w->q1 = (int *)(base + oq1);
        w->misc = (int *)(base + omisc);
    }
    return o;
}

__device__ void bfs_from_sink(const Ws &w, int m, int tid) {
    // h = 0 on the sink set (g < -EPS), BFS over arcs u->v with rc > EPS
    __shared__ int qlen, nlen;
    for (int i = tid; i < m; i += NT) w.h[i] = HINF;
    if (tid == 0) qlen = 0;
    __syncthreads();
    for (int i = tid; i < m; i += NT) {
        if (w.g[i] < -EPS) {
            w.h[i] = 0;
            w.q0[atomicAdd(&qlen, 1)] = i;
        }
    }
    __syncthreads();
    int *cur = w.q0, *nxt = w.q1;
    int level = 0;
    while (qlen > 0) {
        if (tid == 0) nlen = 0;
        __syncthreads();
        for (int t = tid; t < qlen; t += NT) {
            const int v = cur[t];
            for (int ai = w.off[v]; ai < w.off[v + 1]; ++ai) {
                const int a = w.adj[ai];          // v -> x ; reverse arc a^1 : x -> v
                const int x = w.head[a];
                if (w.rc[a ^ 1] > EPS && atomicCAS(&w.h[x], HINF, level + 1) == HINF)
                    nxt[atomicAdd(&nlen, 1)] = x;
            }
        }
        __syncthreads();
        if (tid == 0) qlen = nlen;
        int *t2 = cur; cur = nxt; nxt = t2;
        ++level;
        __syncthreads();
    }
}

// pre_off / pre_adj (optional): the graph's tail-grouped adjacency, built once
// by the caller (the batched step-level solves reuse one structure per block
// every iteration instead of a serial per-solve build).
__device__ void solve_graph(int32_t m, const double *__restrict__ tcap, int64_t P, const int32_t *__restrict__ pi,
                            const int32_t *__restrict__ pj, const double *__restrict__ cij,
                            const double *__restrict__ cji, uint8_t *__restrict__ labels,
                            double *__restrict__ flow, char *wsbase, const int32_t *pre_off = nullptr,
                            const int32_t *pre_adj = nullptr) {
    Ws w;
    ws_layout(m, P, &w, wsbase);
    const int tid = threadIdx.x;
    __shared__ int s_any;
    for (int i = tid; i < m; i += NT) w.g[i] = tcap[i];
    for (int64_t p = tid; p < P; p += NT) {
        DOPE_ASSERT(pi[p] >= 0 && pi[p] < m && pj[p] >= 0 && pj[p] < m);
        w.rc[2 * p] = cij[p];
        w.rc[2 * p + 1] = cji[p];
        w.head[2 * p] = pj[p];
        w.head[2 * p + 1] = pi[p];
    }
    if (pre_off) {
        for (int i = tid; i <= m; i += NT) w.off[i] = pre_off[i];
        for (int64_t a = tid; a < 2 * P; a += NT) w.adj[a] = pre_adj[a];
    } else if (tid == 0) {
        // tail-grouped adjacency in pair order (deterministic, serial)
        for (int i = 0; i <= m; ++i) w.off[i] = 0;
        for (int64_t p = 0; p < P; ++p) { w.off[pi[p] + 1] += 1; w.off[pj[p] + 1] += 1; }
        for (int i = 0; i < m; ++i) w.off[i + 1] += w.off[i];
        for (int i = 0; i < m; ++i) w.fill[i] = w.off[i];
        for (int64_t p = 0; p < P; ++p) {
            w.adj[w.fill[pi[p]]++] = (int)(2 * p);
            w.adj[w.fill[pj[p]]++] = (int)(2 * p + 1);
        }
    }
    for (int64_t a = tid; a < 2 * P; a += NT) w.fl[a] = 0.0;
    __syncthreads();

    for (int round = 0; round < (1 << 20); ++round) {
        bfs_from_sink(w, m, tid);
        if (tid == 0) s_any = 0;
        __syncthreads();
        int any = 0;
        for (int i = tid; i < m; i += NT) any |= (w.g[i] > EPS && w.h[i] != HINF);
        if (any) s_any = 1;
        __syncthreads();
        if (!s_any) break;
        for (int sweep = 0; sweep < 4 * m + 8; ++sweep) {
            // push: record per-arc flow, update the tail's own residuals/excess
            for (int u = tid; u < m; u += NT) {
                double e = w.g[u];
                const int hu = w.h[u];
                if (!(e > EPS) || hu == HINF || hu == 0) continue;
                for (int ai = w.off[u]; ai < w.off[u + 1] && e > EPS; ++ai) {
                    const int a = w.adj[ai];
                    const double r = w.rc[a];
                    if (!(r > EPS) || w.h[w.head[a]] != hu - 1) continue;
                    const double d = e < r ? e : r;
                    w.rc[a] = r - d;
                    w.rc[a ^ 1] += d;
                    w.fl[a] = d;
                    e -= d;
                }
                w.g[u] = e;
            }
            __syncthreads();
            // pull: excess += sum of flows pushed into u, in adjacency order
            for (int u = tid; u < m; u += NT) {
                double add = 0.0;
                for (int ai = w.off[u]; ai < w.off[u + 1]; ++ai) {
                    const int b = w.adj[ai] ^ 1;     // arc x -> u
                    const double f = w.fl[b];
                    if (f != 0.0) { add += f; w.fl[b] = 0.0; }
                }
                if (add != 0.0) w.g[u] += add;
            }
            __syncthreads();
            // relabel
            int act = 0;
            for (int u = tid; u < m; u += NT) {
                if (!(w.g[u] > EPS)) continue;
                const int hu = w.h[u];
                if (hu == HINF) continue;
                int mn = HINF;
                for (int ai = w.off[u]; ai < w.off[u + 1]; ++ai) {
                    const int a = w.adj[ai];
                    if (w.rc[a] > EPS) {
                        const int hx = w.h[w.head[a]];
                        mn = hx < mn ? hx : mn;
                    }
                }
                const int nh = (mn >= m) ? HINF : mn + 1;
                if (nh > hu) w.h[u] = nh;
                act |= (nh != HINF);
            }
            if (!__syncthreads_or(act)) break;
        }
    }
    // labels: final complete BFS; flow = absorbed sink capacity
    __shared__ double red[NT / 32];
    double fsum = 0.0;
    for (int i = tid; i < m; i += NT) {
        labels[i] = (uint8_t)(w.h[i] != HINF);
        const double t0 = tcap[i] < 0.0 ? -tcap[i] : 0.0;
        const double t1 = w.g[i] < 0.0 ? -w.g[i] : 0.0;
        fsum += t0 - t1;
    }
    for (int o = 16; o > 0; o >>= 1) fsum += __shfl_xor_sync(0xffffffffu, fsum, o);
    if ((tid & 31) == 0) red[tid >> 5] = fsum;
    __syncthreads();
    if (tid == 0) {
        double s = 0.0;
        for (int i = 0; i < NT / 32; ++i) s += red[i];
        flow[0] = s;
    }
}

__global__ void __launch_bounds__(NT) k_graph_maxflow(int32_t m, const double *__restrict__ tcap,
                                                      int64_t P, const int32_t *__restrict__ pi,
                                                      const int32_t *__restrict__ pj,
                                                      const double *__restrict__ cij,
                                                      const double *__restrict__ cji,
                                                      uint8_t *__restrict__ labels,
                                                      double *__restrict__ flow, char *wsbase) {
    solve_graph(m, tcap, P, pi, pj, cij, cji, labels, flow, wsbase);
}

// A batch of independent graphs, one CTA each (the step-level update_blocks of
// the general graph path): graph b has nodes [node_off[b], node_off[b+1]) and
// pairs [pair_off[b], pair_off[b+1]) of the concatenated arrays (pair ends are
// graph-local) and the workspace at ws_off[b].
__global__ void __launch_bounds__(NT) k_graph_maxflow_batch(const int64_t *node_off, const int64_t *pair_off,
                                                            const int64_t *ws_off, const double *tcap,
                                                            const int32_t *pi, const int32_t *pj, const double *cij,
                                                            const double *cji, uint8_t *labels, double *flow,
                                                            char *wsbase, const int32_t *adj_off,
                                                            const int32_t *adj) {
    const int b = blockIdx.x;
    const int64_t n0 = node_off[b], p0 = pair_off[b];
    const int32_t m = (int32_t)(node_off[b + 1] - n0);
    const int64_t P = pair_off[b + 1] - p0;
    if (m == 0) {
        if (threadIdx.x == 0) flow[b] = 0.0;
        return;
    }
    solve_graph(m, tcap + n0, P, pi + p0, pj + p0, cij + p0, cji + p0, labels + n0, flow + b, wsbase + ws_off[b],
                adj_off ? adj_off + n0 + b : nullptr, adj ? adj + 2 * p0 : nullptr);
}

}  // namespace dope_graph

extern "C" {

int64_t dope_bk_workspace_bytes(int32_t m, int64_t npairs) {
    if (m < 0 || npairs < 0) return -1;
    return (int64_t)dope_graph::ws_layout(m, npairs, nullptr, nullptr);
}

int dope_bk_maxflow(int32_t m, const double *tcap, int64_t npairs, const int32_t *pair_i,
                    const int32_t *pair_j, const double *cap_ij, const double *cap_ji,
                    uint8_t *labels, double *flow, void *workspace, int64_t workspace_bytes,
                    void *stream) {
    if (m < 0 || npairs < 0 || !flow) return DOPE_E_ARGS;
    if (npairs > (1ll << 30)) return DOPE_E_ARGS;
    cudaStream_t s = (cudaStream_t)stream;
    if (m == 0) {
        return cudaMemsetAsync(flow, 0, sizeof(double), s) == cudaSuccess ? DOPE_OK : DOPE_E_CUDA;
    }
    if (!tcap || !labels || !workspace) return DOPE_E_ARGS;
    if (npairs && (!pair_i || !pair_j || !cap_ij || !cap_ji)) return DOPE_E_ARGS;
    if (workspace_bytes < dope_bk_workspace_bytes(m, npairs)) return DOPE_E_ARGS;
    dope_graph::k_graph_maxflow<<<1, dope_graph::NT, 0, s>>>(m, tcap, npairs, pair_i, pair_j,
                                                             cap_ij, cap_ji, labels, flow,
                                                             (char *)workspace);
    return cudaGetLastError() == cudaSuccess ? DOPE_OK : DOPE_E_CUDA;
}

int dope_bk_maxflow_batch(int32_t B, const int64_t *node_off, const int64_t *pair_off, const int64_t *ws_off,
                          const double *tcap, const int32_t *pair_i, const int32_t *pair_j, const double *cap_ij,
                          const double *cap_ji, uint8_t *labels, double *flows, void *workspace,
                          const int32_t *adj_off, const int32_t *adj, void *stream) {
    if (B < 0 || (B && (!node_off || !pair_off || !ws_off || !flows || !workspace))) return DOPE_E_ARGS;
    if (B == 0) return DOPE_OK;
    dope_graph::k_graph_maxflow_batch<<<B, dope_graph::NT, 0, (cudaStream_t)stream>>>(
        node_off, pair_off, ws_off, tcap, pair_i, pair_j, cap_ij, cap_ji, labels, flows, (char *)workspace, adj_off,
        adj);
    return cudaGetLastError() == cudaSuccess ? DOPE_OK : DOPE_E_CUDA;
}

}  // extern "C"
