// dope_float.cu -- float-weight 2D lattices (BASELINE C2: 1024^2, 8-connected
// contrast-sensitive Potts, lambda = 2, rho = 0.5), behind dope_lattice_f.
//
// Exactness strategy:
//   * the block objective is evaluated in float64 in the reference's
//     operation order (blockform.py:103-104; cross terms in ascending global
//     index, r = d - dhat precomputed on the host as blockform.py:75 does);
//   * capacities are quantised once to int32 at scale S (default 2^16):
//     terminal rint(linear*S), pair rint(lam*w*S) -- the block min cut is then
//     solved EXACTLY (integer push-relabel, labels = sink-reachable set) for
//     the quantised energy; the survey's probe found identical traces to the
//     reference at S >= 2^16 on a C2-like instance;
//   * the consensus update replays solve_global's float64 accumulation order
//     (admm.py:145-151: own-block term and per-neighbour-block coupling sums in
//     block-id order).
// Parity bar (BASELINE): final energy within 1e-5 relative, <= 0.01 % labels.
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <stdio.h>
#include <string.h>

#include <map>
#include <mutex>
#include <string>

#include "common.cuh"
#include "graph_cache.cuh"
#include "dope_b200.h"
#include "mincut_core.cuh"

namespace dope_f {
using namespace dope;

static thread_local char g_err[256] = "";
static int cuda_check(cudaError_t e, const char *what) {
    if (e == cudaSuccess) return DOPE_OK;
    snprintf(g_err, sizeof(g_err), "%s: %s", what, cudaGetErrorString(e));
    return DOPE_E_CUDA;
}

struct LatF {
    Axis ay, ax;
    int32_t W, conn, ndir;
    double lam, mu, eps, qs;
    double inv_mu;                // 1/mu when mu is a power of two (x/mu == x*inv_mu exactly), else 0
    int32_t warm, skip_clean, fuse, max_iters, K, boxh, boxw;
    int32_t epre;                 // dope_lattice_f.energy_prepass
    const double *u, *rdiag;
    const double *w[4];          // E S SE SW, weight of pair (i, i+off) at i
    const int32_t *cq[4];        // quantised lam*w*S, same layout
    double *a0, *a1;
    double *y[3];
    uint8_t *yhat;
    int32_t *resid;
    uint32_t *dirty;
    double *pe, *pr;
    int32_t *pf;
    dope_run_state *st;
    double *tr_e, *tr_rs, *tr_mr;
    int32_t *tr_cl;
    uint64_t *trace_hash;        // audit mode: per-iteration label digests (may be null)
};

// neighbour directions: E W S N SE NW SW NE (opposites d ^ 1)
__device__ __forceinline__ int dy_of(int d) { return (d == 2 || d == 4 || d == 6) ? 1 : (d == 3 || d == 5 || d == 7) ? -1 : 0; }
__device__ __forceinline__ int dx_of(int d) { return (d == 0 || d == 4 || d == 7) ? 1 : (d == 1 || d == 5 || d == 6) ? -1 : 0; }

// weight / quantised capacity of the pair (g, g + off_d)
__device__ __forceinline__ int64_t pair_low(const LatF &L, int64_t G, int d, int &plane) {
    // forward planes: E(0) S(1) SE(2) SW(3); the pair is stored at its lower pixel
    const int64_t W = L.W;
    switch (d) {
        case 0: plane = 0; return G;
        case 1: plane = 0; return G - 1;
        case 2: plane = 1; return G;
        case 3: plane = 1; return G - W;
        case 4: plane = 2; return G;
        case 5: plane = 2; return G - W - 1;
        case 6: plane = 3; return G;
        default: plane = 3; return G - W + 1;
    }
}

// Energy of the current iterate over a re-solved block's interior pixels (the
// term the consensus pass needs of its "previous" iterate, energy.py:187-194):
// computed inside K1f by the warps that would otherwise wait for warp 0's BFS,
// a chunk of (NT - 32) pixels per BFS, the rest after the solve (under the
// residual planes' bulk stores).  Partial
// sums live in shared memory (no register is held across the solve).
template <int NT>
struct EnergyIdle {
    const LatF &L;
    double *eacc;          // [NT] per-thread partial sums (shared)
    const double *y;       // the current iterate
    int32_t lo_r, lo_c, iw, mi;
    static constexpr int CH = NT - 32;
    __device__ __forceinline__ double pixel(int p) const {
        const int r = p / iw + 1, c = p - (r - 1) * iw + 1;
        const int64_t W = L.W;
        const int64_t G = (int64_t)(lo_r + r) * W + lo_c + c;
        // interior pixels: every forward pair exists (E S [SE SW])
        const double yo = y[G];
        const double d0 = yo - y[G + 1], d1 = yo - y[G + W];
        double q = L.w[0][G] * (d0 * d0);
        q += L.w[1][G] * (d1 * d1);
        if (L.ndir == 8) {
            const double d2 = yo - y[G + W + 1], d3 = yo - y[G + W - 1];
            q += L.w[2][G] * (d2 * d2);
            q += L.w[3][G] * (d3 * d3);
        }
        return L.u[G] * yo + L.lam * q;
    }
    // chunks per BFS (1 and 2 measured alike on C2; with 2 a solve with two
    // BFS runs leaves nothing for the tail)
    #ifndef K1F_EPRE_PER_CALL
#define K1F_EPRE_PER_CALL 2
#endif
    static constexpr int PER_CALL = K1F_EPRE_PER_CALL;
    __device__ __forceinline__ void operator()(int call) const {
        const int t = (int)threadIdx.x - 32;
        double e = 0.0;
#pragma unroll
        for (int j = 0; j < PER_CALL; ++j) {
            const int p = (PER_CALL * call + j) * CH + t;
            if (p < mi) e += pixel(p);
        }
        eacc[threadIdx.x] += e;
    }
};

// ---------------------------------------------------------------------------
// K1f: block min cut, quantised float capacities, 4/8 directions
// ---------------------------------------------------------------------------
template <int BH, int BW, int NT, int NDIR>
__global__ void __launch_bounds__(NT) k_block_mincut_f(LatF L, int sweep_min, int sweep_mul) {
    using Cf = K1FCfg<BH, BW, NT, NDIR>;
    constexpr int M = Cf::M, NPT = Cf::NPT;
    extern __shared__ __align__(16) uint8_t smem[];
    int32_t *g = reinterpret_cast<int32_t *>(smem + Cf::OFF_G);
    int32_t *rr = reinterpret_cast<int32_t *>(smem + Cf::OFF_R);
    uint16_t *h = reinterpret_cast<uint16_t *>(smem + Cf::OFF_H);
    uint64_t *masks = reinterpret_cast<uint64_t *>(smem + Cf::OFF_MASK);
    uint64_t *reach = reinterpret_cast<uint64_t *>(smem + Cf::OFF_REACH);
    int *misc = reinterpret_cast<int *>(smem + Cf::OFF_MISC);
    double *eacc = reinterpret_cast<double *>(smem + Cf::SMEM);   // [NT], after the core's layout
    const int tid = threadIdx.x;
    const int k = blockIdx.x;
    const int it0 = L.st->iteration;   // with the stop flag: one round trip
    if (L.st->stop) return;
    if (L.skip_clean && L.dirty[k] == 0) return;
    uint64_t *bar = reinterpret_cast<uint64_t *>(misc + 8);
    if (tid == 0) mc_bar_init(bar);
    __syncthreads();
    if (tid == 0) {
        L.dirty[k] = 0;
        L.dirty[L.K + k] = (uint32_t)it0 + 1u;   // solve epoch (K2f's clean-block pass)
    }
    const int by = k / L.ax.k, bx = k - by * L.ax.k;
    int32_t lo_r, hr, lo_c, wc;
    L.ay.range(by, lo_r, hr);
    L.ax.range(bx, lo_c, wc);
#ifdef K1F_DIAG
    if (tid == 0 && k < 4096) {
        for (int i = 0; i < 16; ++i) g_k1f_diag[16 * k + i] = 0;
        g_k1f_diag[16 * k + 0] = k1f_now();
    }
#endif
    const int32_t Wg = L.W, H = L.ay.dim;
    const double *__restrict__ a_cur = L.st->parity ? L.a1 : L.a0;
    const double *__restrict__ y_cur = L.y[L.st->ycur];
    int32_t *gres = L.resid + (size_t)k * NDIR * M;

    // ---- prologue: linear in float64 (blockform.py:103-104), quantised ----
    // Warm start: the kept residual planes stream into shared memory first
    // (all 16-byte loads in flight); the stored flow is then read back from
    // them through the arc-pair invariant r(v->w) + r(w->v) = 2 cap(v,w), so
    // no capacity plane is re-read: net inflow on arc d = (r_d(v) - r_d'(w)) / 2.
    if (L.warm && tid == 0) {
        // one bulk copy per plane (16-byte loads by the threads took 8 dependent
        // round trips: 9 us of prologue per solve)
        DOPE_ASSERT((reinterpret_cast<uintptr_t>(gres) & 15) == 0);
        mc_bar_expect(bar, NDIR * M * 4);
#pragma unroll
        for (int d = 0; d < NDIR; ++d) mc_bulk_load(rr + d * M, gres + d * M, M * 4, bar);
    }
    // (a) the ring of border nodes, one per thread (its cross-block sum needs
    //     up to 2 * NDIR more operands: all loads of a node in flight together,
    //     and no interior warp diverges into it); (b) the interior nodes, the
    //     four operands of a batch of nodes in flight together.
    {
        const int nring = (hr <= 2 || wc <= 2) ? hr * wc : 2 * wc + 2 * (hr - 2);
        for (int t = tid; t < nring; t += NT) {
            int r, c;
            if (hr <= 2 || wc <= 2) { r = t / wc; c = t - r * wc; }
            else if (t < wc) { r = 0; c = t; }
            else if (t < 2 * wc) { r = hr - 1; c = t - wc; }
            else { const int q = t - 2 * wc; r = 1 + (q >> 1); c = (q & 1) ? wc - 1 : 0; }
            const int32_t R = lo_r + r, Cc = lo_c + c;
            const int64_t G = (int64_t)R * Wg + Cc;
            // cross-block neighbours in ascending global index: NW N NE W E SW S SE
            constexpr int ORD8[8] = {5, 3, 7, 1, 0, 6, 2, 4};
            constexpr int ORD4[4] = {3, 1, 0, 2};
            double tw[NDIR], ty[NDIR];
#pragma unroll
            for (int t2 = 0; t2 < NDIR; ++t2) {
                const int d = NDIR == 8 ? ORD8[t2] : ORD4[t2];
                const int rn = R + dy_of(d), cn = Cc + dx_of(d);
                const bool cross = !(rn < 0 || rn >= H || cn < 0 || cn >= Wg) &&
                                   !(rn >= lo_r && rn < lo_r + hr && cn >= lo_c && cn < lo_c + wc);
                int pl;
                const int64_t low = pair_low(L, G, d, pl);
                tw[t2] = cross ? L.w[pl][low] : 0.0;
                ty[t2] = cross ? y_cur[(int64_t)rn * Wg + cn] : 0.0;
            }
            const double sy = y_cur[G], uu = L.u[G], rd = L.rdiag[G], av = a_cur[G];
            double cy = 0.0;
#pragma unroll
            for (int t2 = 0; t2 < NDIR; ++t2) {
                const int d = NDIR == 8 ? ORD8[t2] : ORD4[t2];
                const int rn = R + dy_of(d), cn = Cc + dx_of(d);
                if (rn < 0 || rn >= H || cn < 0 || cn >= Wg) continue;
                if (rn >= lo_r && rn < lo_r + hr && cn >= lo_c && cn < lo_c + wc) continue;
                cy += (-tw[t2]) * ty[t2];
            }
            const double lin = uu + L.lam * (cy + rd * sy) + L.mu * ((av - sy) + 0.5);
            const double qv = rint(lin * L.qs);
            g[r * BW + c] = (int32_t)fmax(fmin(qv, 1.0e9), -1.0e9);
        }
    }
    constexpr int GRP = NPT < 4 ? NPT : 4;   // nodes per batch of loads (register budget)
#pragma unroll 1
    for (int i0 = 0; i0 < NPT; i0 += GRP) {
        double p_u[GRP], p_y[GRP], p_rd[GRP], p_a[GRP];
#pragma unroll
        for (int i = 0; i < GRP; ++i) {
            const int v = tid + (i0 + i) * NT;
            const int r = v / BW, c = v % BW;
            const bool inner = r > 0 && c > 0 && r < hr - 1 && c < wc - 1;
            const int64_t G = (int64_t)(lo_r + r) * Wg + lo_c + c;
            p_u[i] = inner ? L.u[G] : 0.0;
            p_y[i] = inner ? y_cur[G] : 0.0;
            p_rd[i] = inner ? L.rdiag[G] : 0.0;
            p_a[i] = inner ? a_cur[G] : 0.0;
        }
#pragma unroll
        for (int i = 0; i < GRP; ++i) {
            const int v = tid + (i0 + i) * NT;
            const int r = v / BW, c = v % BW;
            const bool valid = r < hr && c < wc;
            const bool inner = r > 0 && c > 0 && r < hr - 1 && c < wc - 1;
            if (inner) {
                const double sy = p_y[i];
                const double lin = p_u[i] + L.lam * (0.0 + p_rd[i] * sy) + L.mu * ((p_a[i] - sy) + 0.5);
                const double qv = rint(lin * L.qs);
                g[v] = (int32_t)fmax(fmin(qv, 1.0e9), -1.0e9);
            } else if (!valid) {
                g[v] = 0;
            }
            if (!L.warm) {
                const int64_t G = (int64_t)(lo_r + r) * Wg + lo_c + c;
#pragma unroll
                for (int d = 0; d < NDIR; ++d) {
                    const int rb = r + dy_of(d), cb = c + dx_of(d);
                    const bool has = valid && rb >= 0 && rb < hr && cb >= 0 && cb < wc;
                    int pl;
                    const int64_t low = pair_low(L, G, d, pl);
                    rr[d * M + v] = has ? L.cq[pl][low] : 0;
                }
            }
        }
    }
    K1F_D(10, = k1f_now());
    if (L.warm) mc_bar_wait(bar, 0);
    K1F_D(11, = k1f_now());
    __syncthreads();
    K1F_D(12, = k1f_now());
    if (L.warm) {
        for (int i = 0; i < NPT; ++i) {
            const int v = tid + i * NT;
            const int r = v / BW, c = v % BW;
            if (!(r < hr && c < wc)) continue;
            int32_t f2 = 0;
#pragma unroll
            for (int d = 0; d < NDIR; ++d) {
                const int rb = r + dy_of(d), cb = c + dx_of(d);
                if (rb >= 0 && rb < hr && cb >= 0 && cb < wc)
                    f2 += rr[d * M + v] - rr[(d ^ 1) * M + rb * BW + cb];
            }
            g[v] += f2 / 2;
        }
        __syncthreads();
    }

    K1F_D(1, = k1f_now());
    // interior energy of the current iterate for the consensus pass (run loop,
    // from the second iteration on): see EnergyIdle
    const int e_iw = wc - 2, e_ih = hr - 2;
    const bool e_on = L.fuse && L.epre && it0 >= 1 && e_iw > 0 && e_ih > 0;
    const EnergyIdle<NT> eidle{L, eacc, y_cur, lo_r, lo_c, e_iw, e_on ? e_iw * e_ih : 0};
    eacc[tid] = 0.0;
    int rounds_;
    {
        rounds_ = mincut_solve<BH, BW, NT, NDIR>(g, rr, h, masks, reach, misc, sweep_min, sweep_mul, eidle);
        if (rounds_ < 0 && tid == 0) atomicCAS(&L.st->error, 0, k + 1);
        K1F_D(3, = rounds_);
        K1F_D(2, = k1f_now());
    }
    if (L.warm) {
        // the residual planes go back by bulk stores while the labels are written
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncthreads();
        if (tid == 0) {
#pragma unroll
            for (int d = 0; d < NDIR; ++d) mc_bulk_store(gres + d * M, rr + d * M, M * 4);
        }
    }
    for (int i = 0; i < NPT; ++i) {
        const int v = tid + i * NT;
        const int r = v / BW, c = v % BW;
        if (r < hr && c < wc)
            L.yhat[(int64_t)(lo_r + r) * Wg + lo_c + c] = (uint8_t)((reach[v >> 6] >> (v & 63)) & 1ull);
    }
    // the interior energy's tail and block sum overlap the bulk stores
    if (e_on && rounds_ >= 0) {
        // chunks the BFS waits did not reach (rounds_ + 1 BFS runs)
        const int done = EnergyIdle<NT>::PER_CALL * (rounds_ + 1) * EnergyIdle<NT>::CH;
        double e = 0.0;
#pragma unroll 4
        for (int p = done + tid; p < eidle.mi; p += NT) e += eidle.pixel(p);   // loads of all chunks in flight
        e += eacc[tid];
        // per-warp sums (32 slots per block; absent warps hold 0): the consensus
        // pass folds them in a fixed order -- no CTA barrier on K1f's tail
        e = warp_sum(e);
        if ((tid & 31) == 0) L.pe[L.K + 32 * (size_t)k + (tid >> 5)] = e;
        if (NT < 1024 && tid < 32 && tid >= NT / 32) L.pe[L.K + 32 * (size_t)k + tid] = 0.0;
        if (tid == 0) L.dirty[6 * L.K + k] = (uint32_t)it0 + 1u;   // ... of this pass
    }
    if (L.warm && tid == 0) mc_bulk_store_wait();
    if (tid == 0) atomicAdd((unsigned long long *)&L.st->solves, 1ull);
    __syncthreads();
    K1F_D(7, = k1f_now());
}

// cold residual planes (quantised capacities of in-block arcs)
__global__ void k_init_resid_f(LatF L, int M, int bw) {
    const int k = blockIdx.x;
    const int by = k / L.ax.k, bx = k - by * L.ax.k;
    int32_t lo_r, hr, lo_c, wc;
    L.ay.range(by, lo_r, hr);
    L.ax.range(bx, lo_c, wc);
    int32_t *gres = L.resid + (size_t)k * L.ndir * M;
    for (int v = threadIdx.x; v < M; v += blockDim.x) {
        const int r = v / bw, c = v % bw;
        const bool valid = r < hr && c < wc;
        const int64_t G = (int64_t)(lo_r + r) * L.W + lo_c + c;
        for (int d = 0; d < L.ndir; ++d) {
            const int rb = r + dy_of(d), cb = c + dx_of(d);
            const bool has = valid && rb >= 0 && rb < hr && cb >= 0 && cb < wc;
            int pl;
            const int64_t low = pair_low(L, G, d, pl);
            gres[d * M + v] = has ? L.cq[pl][low] : 0;
        }
    }
}

__global__ void k_init_state_f(LatF L, int64_t n) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
        L.y[0][i] = 0.5;             // admm.py:102-110; best_y = copy
        L.a0[i] = 0.0;
        L.a1[i] = 0.0;
        L.yhat[i] = 0;
    }
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < L.K; i += stride) {
        L.dirty[i] = 1u;
        L.dirty[L.K + i] = 0u;                 // solve epochs
        L.dirty[2 * L.K + i] = 0u;             // y buffer 0 holds the initial iterate ...
        L.dirty[3 * L.K + i] = 0xFFFFFFFFu;    // ... buffers 1, 2 nothing yet
        L.dirty[4 * L.K + i] = 0xFFFFFFFFu;
        L.dirty[5 * L.K + i] = 0u;             // pass of the last change of the block's iterate
        if (L.epre) L.dirty[6 * L.K + i] = 0u; // pass of K1f's interior energy sum
        L.pe[i] = 0.0;
        L.pr[i] = 0.0;
        L.pf[i] = 0;
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        dope_run_state s;
        memset(&s, 0, sizeof(s));
        s.best_energy = __double_as_longlong(INFINITY);
        *L.st = s;
    }
}

__device__ __forceinline__ int other_buffer_f(int cur, int best) {
    if (cur == best) return (cur + 1) % 3;
    return 3 - cur - best;
}

// ---------------------------------------------------------------------------
// K2f: consensus (solve_global admm.py:136-151 float order, clamp, multipliers,
// residual and energy partials, dirty marks), one CTA per block; the last CTA
// finalizes the iteration (admm.py:231-249).
// ---------------------------------------------------------------------------
__device__ void apply_f(const LatF &L, double E2, double R2, double M2, int F2, int cur, int best,
                        int out) {
    dope_run_state *st = L.st;
    int bidx = best;
    const int t = st->iteration;
    if (t >= 1) {
        if (t - 1 < L.max_iters) L.tr_e[t - 1] = E2;
        if (E2 < __longlong_as_double(st->best_energy)) {
            st->best_energy = __double_as_longlong(E2);
            st->best_iteration = t;
            bidx = cur;
        }
    }
    const double maxres = M2 < 0 ? 0.0 : sqrt(M2);
    if (t < L.max_iters) {
        L.tr_rs[t] = R2;
        L.tr_mr[t] = maxres;
        L.tr_cl[t] = F2;
    }
    st->iteration = t + 1;
    if (L.K == 0 || maxres <= L.eps) {
        st->converged = 1;
        st->stop = 1;
    }
    if (st->error) st->stop = 1;
    st->ybest = bidx;
    st->ycur = out;
}

// K2f threads per CTA: 512 (8 pixels each) keeps two CTAs per SM, so C2's 256
// blocks run in one wave (1024 threads: 45 us per pass, 512: 38 us)
#ifndef K2F_THREADS
#define K2F_THREADS 512
#endif
constexpr int K2F_NT = K2F_THREADS;

// The last consensus CTA of a pass: fold every block's partials (fixed order)
// and apply the iteration (admm.py:226-249), or -- step-level API -- rotate.
__device__ __forceinline__ void k2f_finalize(const LatF &L, int cur, int best, int out) {
    constexpr int NWARP = K2F_NT / 32;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    __threadfence();
    __shared__ double sE[NWARP], sR[NWARP], sM[NWARP];
    __shared__ int sF[NWARP];
    if (!L.fuse) {
        if (tid == 0) {
            L.st->ybest = best;
            L.st->ycur = out;
            L.st->done_ctas = 0;
        }
        return;
    }
    double E = 0.0, R2 = 0.0, M2 = -1.0;
    int F = 0;
    for (int b = tid; b < L.K; b += blockDim.x) {
        E += __ldcg(&L.pe[b]);
        const double sq = __ldcg(&L.pr[b]);
        const double rr = sqrt(sq);
        R2 += rr * rr;
        M2 = sq > M2 ? sq : M2;
        F |= __ldcg(&L.pf[b]) & 1;
    }
    E = warp_sum(E);
    R2 = warp_sum(R2);
    for (int o = 16; o > 0; o >>= 1) {
        const double t = __shfl_xor_sync(FULLMASK, M2, o);
        M2 = t > M2 ? t : M2;
    }
    F = __any_sync(FULLMASK, F);
    if (lane == 0) { sE[warp] = E; sR[warp] = R2; sM[warp] = M2; sF[warp] = F; }
    __syncthreads();
    if (tid == 0) {
        double E2 = 0.0, RR = 0.0, MM = -1.0;
        int FF = 0;
        for (int w = 0; w < NWARP; ++w) {
            E2 += sE[w]; RR += sR[w]; MM = sM[w] > MM ? sM[w] : MM; FF |= sF[w];
        }
        apply_f(L, E2, RR, MM, FF, cur, best, out);
        L.st->done_ctas = 0;
    }
}

#ifdef K1F_DIAG
static __device__ long long g_k2f_diag[16 * 4096];
#define K2F_D(slot) do { if (threadIdx.x == 0 && blockIdx.x < 4096) g_k2f_diag[16 * blockIdx.x + (slot)] = k1f_now(); } while (0)
#else
#define K2F_D(slot) do { } while (0)
#endif
__global__ void __launch_bounds__(K2F_NT, 2) k_consensus_f(LatF L) {
    K2F_D(0);
    if (L.st->stop) return;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int k = blockIdx.x;
    const int by = k / L.ax.k, bx = k - by * L.ax.k;
    int32_t lo_r, hr, lo_c, wc;
    L.ay.range(by, lo_r, hr);
    L.ax.range(bx, lo_c, wc);
    const int32_t W = L.W, H = L.ay.dim;
    const int cur = L.st->ycur, best = L.st->ybest, out = other_buffer_f(cur, best);
    const double *__restrict__ y_in = L.y[cur];
    double *__restrict__ y_out = L.y[out];
    const int p = L.st->parity;
    // multipliers in place: a_{t+1}[g] depends on a_t[g] only
    const double *a_in = p ? L.a1 : L.a0;
    double *a_out = L.fuse ? (p ? L.a1 : L.a0) : nullptr;
    const int iteration = L.st->iteration;
    const bool want_e = L.fuse && iteration >= 1;
    const int32_t pass = iteration + 1;    // this pass (= this iteration's K1 solve epoch)
    int32_t *ybuf = reinterpret_cast<int32_t *>(L.dirty + 2 * L.K);    // [3][K] buffer stamps
    int32_t *lastchg = reinterpret_cast<int32_t *>(L.dirty + 5 * L.K);
    __shared__ unsigned nbmark;            // bit (dy+1)*3 + (dx+1): neighbour block dirty
    // 0 full update; clean block (not re-solved now, unmoved in the last pass):
    // 1 fixed point, nothing to do; 2 fixed point, copy y into the output
    // buffer; 3 ring only (a neighbour was re-solved), 4 ring only + copy
    __shared__ int mode;
    __shared__ int last;
    __shared__ int epre;                   // K1f summed this block's interior energy in this pass
    if (tid == 0) {
        nbmark = 0;
        epre = L.epre && L.dirty[6 * L.K + k] == (uint32_t)(iteration + 1);
        // Clean-block fixed point: a block K1 did not re-solve
        // had y and a unmoved (so y == yhat) in the previous pass, and no
        // border pixel next to it moved either; if none of its 8 neighbours
        // was re-solved now, every input of this pass equals the last one's,
        // so y, a, the residual (0), the clamp flags and the energy partial of
        // the unmoved iterate are all the previous pass's -- bit for bit.
        // With a re-solved neighbour only the ring pixels (those with a
        // cross-block neighbour) see new inputs: the interior (r = 0 there:
        // y = clamp(yhat + a)) is still a fixed point, its clamp flags are the
        // memo in part_flags bit 1.
        int m = 0;
        if (L.skip_clean && L.fuse && iteration >= 2 && L.dirty[L.K + k] != (uint32_t)pass) {
            bool nb = false;
            for (int dy = -1; dy <= 1; ++dy)
                for (int dx = -1; dx <= 1; ++dx) {
                    const int nby = by + dy, nbx = bx + dx;
                    if ((dy || dx) && nby >= 0 && nby < L.ay.k && nbx >= 0 && nbx < L.ax.k &&
                        L.dirty[L.K + nby * L.ax.k + nbx] == (uint32_t)pass)
                        nb = true;
                }
            const bool stale = ybuf[out * L.K + k] < lastchg[k];
            m = nb ? (stale ? 4 : 3) : (stale ? 2 : 1);
        }
        mode = m;
    }
    __syncthreads();
    K2F_D(1);
#ifdef K1F_DIAG
    if (threadIdx.x == 0) g_k2f_diag[16 * blockIdx.x + 15] = mode;
#endif
    if (mode == 2 || mode == 4) {   // the output buffer holds an older iterate of this block: copy
        for (int v = tid; v < hr * wc; v += K2F_NT) {
            const int r = v / wc, c = v - r * wc;
            const int64_t G = (int64_t)(lo_r + r) * W + lo_c + c;
            y_out[G] = y_in[G];   // ring pixels are rewritten below in mode 4
        }
        if (mode == 4) __syncthreads();
    }
    if (mode == 1 || mode == 2) {
        __syncthreads();
        if (tid == 0) {
            if (mode == 2) ybuf[out * L.K + k] = pass;
            __threadfence();
            last = (atomicAdd(&L.st->done_ctas, 1) == L.K - 1);
        }
        __syncthreads();
        if (last) k2f_finalize(L, cur, best, out);
        return;
    }

    // read-only planes through restrict-qualified pointers: the loads of
    // the next pixels may be issued ahead of this pixel's stores
    const double *__restrict__ uu = L.u;
    const double *__restrict__ rdg = L.rdiag;
    const double *__restrict__ w0 = L.w[0];
    const double *__restrict__ w1 = L.w[1];
    const double *__restrict__ w2 = L.w[2];
    const double *__restrict__ w3 = L.w[3];
    const uint8_t *__restrict__ yhp = L.yhat;
    double e_acc = 0.0, ss = 0.0;
    int clamped = 0;
    unsigned marks = 0;
    // One pixel of solve_global (admm.py:145-151) + clamp, multipliers,
    // residual, energy of the previous iterate and dirty marks.  Block-border
    // pixels sum their cross-block terms in block-id order; they are handled
    // by a second pass so that no warp of the interior pass diverges into it.
    auto pixel = [&](int r, int c, bool border) {
        const int32_t R = lo_r + r, Cc = lo_c + c;
        const int64_t G = (int64_t)R * W + Cc;
        const double yh = (double)yhp[G];
        const double av = a_in[G];
        const double yold = y_in[G];
        // ring pixels: the energy term of the previous iterate first, so that its
        // loads travel with the pixel's other operands (one round trip less)
        double e_term = 0.0;
        if (want_e && mode == 0 && border) {
            double q = 0.0;
            // pairs owned by this pixel: E S SE SW (forward planes)
            if (Cc + 1 < W) { const double d = yold - y_in[G + 1]; q += w0[G] * (d * d); }
            if (R + 1 < H) {
                const double d = yold - y_in[G + W];
                q += w1[G] * (d * d);
                if (L.ndir == 8) {
                    if (Cc + 1 < W) { const double d2 = yold - y_in[G + W + 1]; q += w2[G] * (d2 * d2); }
                    if (Cc > 0) { const double d3 = yold - y_in[G + W - 1]; q += w3[G] * (d3 * d3); }
                }
            }
            e_term = uu[G] * yold + L.lam * q;
        }
        // own-block term and cross-block coupling sums, in block-id order
        const double own = L.mu * (yh + av) - L.lam * (rdg[G] * yh);
        double acc = 0.0;
        if (border) {
            int nb_blk[8];
            double nb_term[8];
            int64_t nb_idx[8];
            int nn = 0;
            // every cross-block neighbour's weight and label first (independent
            // loads), then the block-id ordering on registers
            double p_w[8];
            uint8_t p_yh[8];
#pragma unroll
            for (int d = 0; d < 8; ++d) {
                const int rn = R + dy_of(d), cn = Cc + dx_of(d);
                const bool in = d < L.ndir && !(rn < 0 || rn >= H || cn < 0 || cn >= W);
                const bool cross = in && !(rn >= lo_r && rn < lo_r + hr && cn >= lo_c && cn < lo_c + wc);
                int pl;
                const int64_t low = pair_low(L, G, d, pl);
                p_w[d] = cross ? L.w[pl][low] : 0.0;
                p_yh[d] = cross ? L.yhat[(int64_t)rn * W + cn] : (uint8_t)0;
            }
#pragma unroll
            for (int d = 0; d < 8; ++d) {
                if (d >= L.ndir) break;
                const int rn = R + dy_of(d), cn = Cc + dx_of(d);
                if (rn < 0 || rn >= H || cn < 0 || cn >= W) continue;
                // neighbour at distance 1: its block is this one or the adjacent one
                const int br = by + (rn < lo_r ? -1 : (rn >= lo_r + hr ? 1 : 0));
                const int bc = bx + (cn < lo_c ? -1 : (cn >= lo_c + wc ? 1 : 0));
                if (br == by && bc == bx) continue;
                const int64_t J = (int64_t)rn * W + cn;
                int q = nn++;
                const int bid = br * L.ax.k + bc;
                while (q > 0 && (nb_blk[q - 1] > bid || (nb_blk[q - 1] == bid && nb_idx[q - 1] > J))) {
                    nb_blk[q] = nb_blk[q - 1]; nb_idx[q] = nb_idx[q - 1]; nb_term[q] = nb_term[q - 1];
                    --q;
                }
                nb_blk[q] = bid;
                nb_idx[q] = J;
                nb_term[q] = (-p_w[d]) * (double)p_yh[d];
            }
            bool own_done = false;
            int t2 = 0;
            while (t2 < nn || !own_done) {
                if (!own_done && (t2 >= nn || nb_blk[t2] > k)) {
                    acc += own;
                    own_done = true;
                    continue;
                }
                const int b = nb_blk[t2];
                double sb = 0.0;
                while (t2 < nn && nb_blk[t2] == b) sb += nb_term[t2++];
                acc -= L.lam * sb;
            }
        } else {
            acc = 0.0 + own;
        }
        const double yp = L.inv_mu != 0.0 ? acc * L.inv_mu : acc / (L.mu * 1.0);
        clamped |= (yp < 0.0 || yp > 1.0);
        const double y = yp < 0.0 ? 0.0 : (yp > 1.0 ? 1.0 : yp);
        if (a_out) a_out[G] = av + (yh - y);
        y_out[G] = y;
        const double dlt = yh - y;
        ss += dlt * dlt;
        if (want_e && mode == 0 && border) e_acc += e_term;
        const bool ychg = (y != yold);
        if (ychg || (av + (yh - y)) != av) marks |= 1u;
        if (ychg) marks |= 1u << 10;
        if (ychg && border) {
            for (int d = 0; d < L.ndir; ++d) {
                const int rn = R + dy_of(d), cn = Cc + dx_of(d);
                if (rn < 0 || rn >= H || cn < 0 || cn >= W) continue;
                const int br = rn < lo_r ? -1 : (rn >= lo_r + hr ? 1 : 0);
                const int bc = cn < lo_c ? -1 : (cn >= lo_c + wc ? 1 : 0);
                if (br || bc) marks |= 1u << (1 + (br + 1) * 3 + (bc + 1));
            }
        }
    };
    // interior pixels (a fixed point in the ring-only modes)
    const int iw = wc - 2, ih = hr - 2;
    const int mi = (iw > 0 && ih > 0 && mode == 0) ? iw * ih : 0;
    // The energy of the previous iterate reads only planes nothing writes in
    // this pass: its own loop, so the loads of several pixels are in flight
    // together (inside pixel() every pixel's loads waited behind the previous
    // pixel's in-place multiplier store).  Same per-thread summation order.
    __shared__ double epre_sum;
    if (want_e && epre && warp == 1) {   // K1f's 32 per-warp interior sums, fixed order
        double v = L.pe[L.K + 32 * (size_t)k + lane];
        v = warp_sum(v);
        if (lane == 0) epre_sum = v;
    }
    if (want_e && !epre) {
#pragma unroll 4
        for (int v = tid; v < mi; v += K2F_NT) {
            const int r = v / iw + 1, c = v % iw + 1;
            const int32_t R = lo_r + r, Cc = lo_c + c;
            const int64_t G = (int64_t)R * W + Cc;
            const double yold = y_in[G];
            double q = 0.0;
            if (Cc + 1 < W) { const double d = yold - y_in[G + 1]; q += w0[G] * (d * d); }
            if (R + 1 < H) {
                const double d = yold - y_in[G + W];
                q += w1[G] * (d * d);
                if (L.ndir == 8) {
                    if (Cc + 1 < W) { const double d2 = yold - y_in[G + W + 1]; q += w2[G] * (d2 * d2); }
                    if (Cc > 0) { const double d3 = yold - y_in[G + W - 1]; q += w3[G] * (d3 * d3); }
                }
            }
            e_acc += uu[G] * yold + L.lam * q;
        }
    }
    K2F_D(2);
    // interior update (no cross-block term): the operands of a batch of pixels
    // first, then the in-place stores
    constexpr int KB = 4;
    for (int v0 = tid; v0 < mi; v0 += KB * K2F_NT) {
        double b_a[KB], b_rd[KB], b_yo[KB], b_yh[KB];
        int64_t b_G[KB];
#pragma unroll
        for (int j = 0; j < KB; ++j) {
            const int v = v0 + j * K2F_NT;
            const bool ok = v < mi;
            const int r = ok ? v / iw + 1 : 1, c = ok ? v % iw + 1 : 1;
            const int64_t G = (int64_t)(lo_r + r) * W + lo_c + c;
            b_G[j] = ok ? G : -1;
            b_yh[j] = (double)yhp[G];
            b_a[j] = a_in[G];
            b_rd[j] = rdg[G];
            b_yo[j] = y_in[G];
        }
#pragma unroll
        for (int j = 0; j < KB; ++j) {
            const int64_t G = b_G[j];
            if (G < 0) continue;
            const double yh = b_yh[j], av = b_a[j];
            const double own = L.mu * (yh + av) - L.lam * (b_rd[j] * yh);
            const double acc = 0.0 + own;
            const double yp = L.inv_mu != 0.0 ? acc * L.inv_mu : acc / (L.mu * 1.0);
            clamped |= (yp < 0.0 || yp > 1.0);
            const double y = yp < 0.0 ? 0.0 : (yp > 1.0 ? 1.0 : yp);
            const double yold = b_yo[j];
            if (a_out) a_out[G] = av + (yh - y);
            y_out[G] = y;
            const double dlt = yh - y;
            ss += dlt * dlt;
            const bool ychg = (y != yold);
            if (ychg || (av + (yh - y)) != av) marks |= 1u;
            if (ychg) marks |= 1u << 10;
        }
    }
    K2F_D(3);
    const int clamped_int = clamped;
    // the ring of border pixels: top row, bottom row, then left / right columns
    const int nring = (hr <= 2 || wc <= 2) ? hr * wc : 2 * wc + 2 * (hr - 2);
    for (int t = tid; t < nring; t += K2F_NT) {
        int r, c;
        if (hr <= 2 || wc <= 2) { r = t / wc; c = t - r * wc; }
        else if (t < wc) { r = 0; c = t; }
        else if (t < 2 * wc) { r = hr - 1; c = t - wc; }
        else { const int u = t - 2 * wc; r = 1 + (u >> 1); c = (u & 1) ? wc - 1 : 0; }
        pixel(r, c, true);
    }
    K2F_D(4);
    constexpr int NWARP = K2F_NT / 32;
    __shared__ double red_e[NWARP], red_s[NWARP];
    __shared__ int red_f[NWARP];
    e_acc = warp_sum(e_acc);
    ss = warp_sum(ss);
    for (int o = 16; o > 0; o >>= 1) marks |= __shfl_xor_sync(FULLMASK, marks, o);
    const int fl = (__any_sync(FULLMASK, clamped) ? 1 : 0) | (__any_sync(FULLMASK, clamped_int) ? 2 : 0);
    if (lane == 0) {
        red_e[warp] = e_acc;
        red_s[warp] = ss;
        red_f[warp] = fl;
        atomicOr(&nbmark, marks);
    }
    __syncthreads();
    K2F_D(5);
    if (tid == 0) {
        double E = 0.0, S = 0.0;
        int F = 0;
        for (int w = 0; w < NWARP; ++w) { E += red_e[w]; S += red_s[w]; F |= red_f[w]; }
        if (mode == 0) {
            if (want_e && epre) E += epre_sum;   // interior part from K1f
            L.pe[k] = E;
            L.pf[k] = F;   // bit 0 any pixel clamped, bit 1 an interior pixel clamped
        } else {           // ring only: the energy partial and the interior clamp memo hold
            const int memo = L.pf[k] & 2;
            L.pf[k] = memo | ((F & 1) | (memo >> 1));
        }
        L.pr[k] = S;
        const unsigned mk = nbmark;
        if (mk & 1u) L.dirty[k] = 1u;
        ybuf[out * L.K + k] = pass;             // the output buffer holds the new iterate
        if (mk & (1u << 10)) lastchg[k] = pass;
        for (int dy = -1; dy <= 1; ++dy)
            for (int dx = -1; dx <= 1; ++dx)
                if ((dy || dx) && (mk & (1u << (1 + (dy + 1) * 3 + (dx + 1)))))
                    L.dirty[(by + dy) * L.ax.k + bx + dx] = 1u;
        __threadfence();
        last = (atomicAdd(&L.st->done_ctas, 1) == L.K - 1);
    }
    __syncthreads();
    K2F_D(6);
    if (last) k2f_finalize(L, cur, best, out);
    K2F_D(7);
}

__global__ void k_update_multipliers_f(LatF L, int64_t n) {
    double *a = L.st->parity ? L.a1 : L.a0;
    const double *y = L.y[L.st->ycur];
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride)
        a[i] = a[i] + ((double)L.yhat[i] - y[i]);
}

// energy of the current iterate, one CTA per block -> pe[], then one CTA
// reduces in a fixed order (deterministic float sums)
__global__ void __launch_bounds__(256) k_energy_blocks_f(LatF L) {
    const int k = blockIdx.x, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int by = k / L.ax.k, bx = k - by * L.ax.k;
    int32_t lo_r, hr, lo_c, wc;
    L.ay.range(by, lo_r, hr);
    L.ax.range(bx, lo_c, wc);
    const int32_t W = L.W, H = L.ay.dim;
    const double *y = L.y[L.st->ycur];
    double e = 0.0;
    for (int v = tid; v < hr * wc; v += blockDim.x) {
        const int r = v / wc, c = v - r * wc;
        const int32_t R = lo_r + r, Cc = lo_c + c;
        const int64_t G = (int64_t)R * W + Cc;
        const double yg = y[G];
        double q = 0.0;
        if (Cc + 1 < W) { const double d = yg - y[G + 1]; q += L.w[0][G] * (d * d); }
        if (R + 1 < H) {
            const double d = yg - y[G + W];
            q += L.w[1][G] * (d * d);
            if (L.ndir == 8) {
                if (Cc + 1 < W) { const double d2 = yg - y[G + W + 1]; q += L.w[2][G] * (d2 * d2); }
                if (Cc > 0) { const double d3 = yg - y[G + W - 1]; q += L.w[3][G] * (d3 * d3); }
            }
        }
        e += L.u[G] * yg + L.lam * q;
    }
    __shared__ double red[8];
    e = warp_sum(e);
    if (lane == 0) red[warp] = e;
    __syncthreads();
    if (tid == 0) {
        double E = 0.0;
        for (int w = 0; w < 8; ++w) E += red[w];
        L.pe[k] = E;
    }
}

__global__ void k_finish_f(LatF L) {
    dope_run_state *st = L.st;
    __shared__ double red[32];
    double E = 0.0;
    for (int b = threadIdx.x; b < L.K; b += blockDim.x) E += L.pe[b];
    E = warp_sum(E);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = E;
    __syncthreads();
    if (threadIdx.x == 0) {
        double T = 0.0;
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) T += red[w];
        for (int b = 0; b < L.K; ++b) L.pe[b] = 0.0;
        const int it = st->iteration;
        if (it >= 1 && !st->error) {
            if (it - 1 < L.max_iters) L.tr_e[it - 1] = T;
            if (T < __longlong_as_double(st->best_energy)) {
                st->best_energy = __double_as_longlong(T);
                st->best_iteration = it;
                st->ybest = st->ycur;
            }
        }
        if (!st->converged) st->ycur = st->ybest;
        st->stop = 1;
    }
}

__global__ void k_binarize_f(LatF L, int64_t n, uint8_t *out) {
    const double *y = L.y[L.st->ycur];
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride)
        out[i] = (uint8_t)(y[i] >= 0.5);
}

// ---------------------------------------------------------------------------
// host
// ---------------------------------------------------------------------------
struct VarF {
    int bh, bw, nt, ndir;
    size_t smem;
    void (*kernel)(LatF, int, int);
};

template <int BH, int BW, int NT, int ND>
static VarF make_varf() {
    return VarF{BH, BW, NT, ND, K1FCfg<BH, BW, NT, ND>::SMEM + 8 * (size_t)NT, &k_block_mincut_f<BH, BW, NT, ND>};
}

static const VarF *pick_varf(int conn, int maxh, int maxw, int nblocks) {
    static const VarF table[] = {
        make_varf<32, 32, 256, 4>(), make_varf<64, 64, 512, 4>(),
        make_varf<32, 32, 256, 8>(), make_varf<64, 64, 512, 8>(),
    };
    // few blocks per SM: the slowest solve sets K1, twice the threads pay
    // (as in the integer path); DOPE_K1_WIDE=0/1 forces
    static const VarF wide[] = {make_varf<64, 64, 1024, 4>(), make_varf<64, 64, 1024, 8>()};
    static const int force = getenv("DOPE_K1_WIDE") ? atoi(getenv("DOPE_K1_WIDE")) : -1;
    static const int sms = [] {
        int dev = 0, n = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
        return n > 0 ? n : 148;
    }();
    if ((force >= 0 ? force != 0 : (nblocks > 0 && nblocks <= 8 * sms)) && maxh > 32 && maxw > 32 && maxh <= 64 &&
        maxw <= 64)
        return &wide[conn == 8 ? 1 : 0];
    for (const VarF &v : table)
        if (v.ndir == conn && maxh <= v.bh && maxw <= v.bw) return &v;
    return nullptr;
}

static int build(const dope_lattice_f *L, LatF &o, const VarF **var) {
    if (!L || !L->u || !L->rdiag || !L->a[0] || !L->a[1] || !L->y[0] || !L->y[1] || !L->y[2] ||
        !L->yhat || !L->resid || !L->dirty || !L->part_energy || !L->part_ressq || !L->part_flags ||
        !L->state)
        return DOPE_E_ARGS;
    if (L->conn != 4 && L->conn != 8) return DOPE_E_GEOMETRY;
    const int np = L->conn == 8 ? 4 : 2;
    for (int i = 0; i < np; ++i)
        if (!L->w[i] || !L->capq[i]) return DOPE_E_ARGS;
    if (L->dims[0] < 1 || L->dims[1] < 1 || L->kpa[0] < 1 || L->kpa[1] < 1 ||
        L->kpa[0] > L->dims[0] || L->kpa[1] > L->dims[1])
        return DOPE_E_ARGS;
    if (!(L->mu > 0) || L->lam < 0 || !(L->qscale > 0)) return DOPE_E_ARGS;
    memset(&o, 0, sizeof(o));
    o.ay = make_axis(L->dims[0], L->kpa[0]);
    o.ax = make_axis(L->dims[1], L->kpa[1]);
    o.W = (int32_t)L->dims[1];
    o.conn = L->conn;
    o.ndir = L->conn;
    o.lam = L->lam;
    o.mu = L->mu;
    {
        int ex;
        o.inv_mu = (L->mu > 0 && frexp(L->mu, &ex) == 0.5) ? 1.0 / L->mu : 0.0;
    }
    o.eps = L->eps;
    o.qs = L->qscale;
    o.warm = L->warm_start;
    o.skip_clean = L->skip_clean;
    o.fuse = L->fuse_multipliers;
    o.epre = L->energy_prepass;
    o.max_iters = L->max_iters;
    o.K = L->kpa[0] * L->kpa[1];
    o.u = L->u;
    o.rdiag = L->rdiag;
    for (int i = 0; i < 4; ++i) {
        o.w[i] = L->w[i];
        o.cq[i] = L->capq[i];
    }
    o.a0 = L->a[0];
    o.a1 = L->a[1];
    for (int i = 0; i < 3; ++i) o.y[i] = L->y[i];
    o.yhat = L->yhat;
    o.resid = L->resid;
    o.dirty = L->dirty;
    o.pe = L->part_energy;
    o.pr = L->part_ressq;
    o.pf = L->part_flags;
    o.st = L->state;
    o.trace_hash = L->trace_hash;
    o.tr_e = L->trace_energy;
    o.tr_rs = L->trace_residual_sq;
    o.tr_mr = L->trace_max_residual;
    o.tr_cl = L->trace_clamped;
    const VarF *v = pick_varf(L->conn, o.ay.base + (o.ay.rem ? 1 : 0), o.ax.base + (o.ax.rem ? 1 : 0), L->kpa[0] * L->kpa[1]);
    if (!v) return DOPE_E_GEOMETRY;
    o.boxh = v->bh;
    o.boxw = v->bw;
    if (var) *var = v;
    return DOPE_OK;
}

static int grid_for(int64_t n) {
    int64_t b = (n + 255) / 256;
    if (b > 148 * 16) b = 148 * 16;
    return (int)(b < 1 ? 1 : b);
}

static int configure(const VarF *v) {
    static std::mutex mu;
    static std::map<void *, bool> done;
    std::lock_guard<std::mutex> lk(mu);
    if (!done[(void *)v->kernel]) {
        int rc = cuda_check(cudaFuncSetAttribute(v->kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                 (int)v->smem), "attr K1f");
        if (rc) return rc;
        done[(void *)v->kernel] = true;
    }
    return DOPE_OK;
}

static int launch_k1(const LatF &o, const VarF *v, cudaStream_t s) {
    int rc = configure(v);
    if (rc) return rc;
    // sweeps per global relabel = sweep_min + sweep_mul * levels (DOPE_SWEEPF_MIN / _MUL);
    // 6 fixed sweeps measured best on C2 (K1 10.4 -> 7.8 ms per run vs 1 + levels)
    static const int smin = getenv("DOPE_SWEEPF_MIN") ? atoi(getenv("DOPE_SWEEPF_MIN")) : 6;
    static const int smul = getenv("DOPE_SWEEPF_MUL") ? atoi(getenv("DOPE_SWEEPF_MUL")) : 0;
    // dense rounds (DOPE_SWEEPF_DMIN / _DMUL; 0 / unset: as the sparse rounds)
    static const int dmin = getenv("DOPE_SWEEPF_DMIN") ? atoi(getenv("DOPE_SWEEPF_DMIN")) : 0;
    static const int dmul = getenv("DOPE_SWEEPF_DMUL") ? atoi(getenv("DOPE_SWEEPF_DMUL")) : 0;
    v->kernel<<<o.K, v->nt, v->smem, s>>>(o, smin | (dmin << 16), smul | (dmul << 16));
    return cuda_check(cudaGetLastError(), "launch K1f");
}

static int launch_k2(const LatF &o, cudaStream_t s) {
    k_consensus_f<<<o.K, K2F_NT, 0, s>>>(o);
    return cuda_check(cudaGetLastError(), "launch K2f");
}

}  // namespace dope_f

using namespace dope_f;

extern "C" {

const char *dope_f_last_error(void) { return g_err; }

int64_t dope_f_resid_stride(const dope_lattice_f *L) {
    if (!L || (L->conn != 4 && L->conn != 8) || L->kpa[0] < 1 || L->kpa[1] < 1) return 0;
    Axis ay = make_axis(L->dims[0], L->kpa[0]), ax = make_axis(L->dims[1], L->kpa[1]);
    const VarF *v = pick_varf(L->conn, ay.base + (ay.rem ? 1 : 0), ax.base + (ax.rem ? 1 : 0), 0);
    return v ? (int64_t)4 * v->ndir * v->bh * v->bw : 0;
}

int dope_f_check(const dope_lattice_f *L) {
    LatF o;
    return build(L, o, nullptr);
}

int dope_f_admm_init(const dope_lattice_f *L, void *stream) {
    LatF o;
    const VarF *v;
    int rc = build(L, o, &v);
    if (rc) return rc;
    cudaStream_t s = (cudaStream_t)stream;
    const int64_t n = L->dims[0] * L->dims[1];
    k_init_state_f<<<grid_for(n), 256, 0, s>>>(o, n);
    if ((rc = cuda_check(cudaGetLastError(), "init_state_f"))) return rc;
    k_init_resid_f<<<o.K, 256, 0, s>>>(o, v->bh * v->bw, v->bw);
    return cuda_check(cudaGetLastError(), "init_resid_f");
}

int dope_f_update_blocks(const dope_lattice_f *L, void *stream) {
    LatF o;
    const VarF *v;
    int rc = build(L, o, &v);
    if (rc) return rc;
    return launch_k1(o, v, (cudaStream_t)stream);
}

int dope_f_update_global(const dope_lattice_f *L, void *stream) {
    LatF o;
    int rc = build(L, o, nullptr);
    if (rc) return rc;
    return launch_k2(o, (cudaStream_t)stream);
}

int dope_f_update_multipliers(const dope_lattice_f *L, void *stream) {
    LatF o;
    int rc = build(L, o, nullptr);
    if (rc) return rc;
    const int64_t n = L->dims[0] * L->dims[1];
    k_update_multipliers_f<<<grid_for(n), 256, 0, (cudaStream_t)stream>>>(o, n);
    return cuda_check(cudaGetLastError(), "update_multipliers_f");
}

// Audit mode: digest of the iteration's labels (y and a are not integers here).
#ifdef K1F_DIAG
extern "C" int dope_f_diag_read(long long *host, int n) {
    return (int)cudaMemcpyFromSymbol(host, dope_f::g_k1f_diag, sizeof(long long) * n);
}
extern "C" int dope_f_diag_read_k2(long long *host, int n) {
    return (int)cudaMemcpyFromSymbol(host, dope_f::g_k2f_diag, sizeof(long long) * n);
}
#endif
static int launch_digest_f(const LatF &o, cudaStream_t s) {
    if (!o.trace_hash) return DOPE_OK;
    k_digest_begin<<<1, 1, 0, s>>>(o.st, o.trace_hash, o.max_iters);
    k_digest<dope_run_state, uint8_t, int16_t><<<2 * 148, 256, 0, s>>>(
        o.st, o.trace_hash, o.max_iters, (int64_t)o.ay.dim * o.W, 0, o.yhat, nullptr, nullptr, nullptr, nullptr);
    return cuda_check(cudaGetLastError(), "state digest");
}

int dope_f_admm_run(const dope_lattice_f *L, int32_t iters, int32_t use_graph, void *stream) {
    LatF o;
    const VarF *v;
    int rc = build(L, o, &v);
    if (rc) return rc;
    cudaStream_t s = (cudaStream_t)stream;
    if (iters <= 0) return DOPE_OK;
    if (!use_graph) {
        for (int i = 0; i < iters; ++i) {
            if ((rc = launch_k1(o, v, s))) return rc;
            if ((rc = launch_k2(o, s))) return rc;
            if ((rc = launch_digest_f(o, s))) return rc;
        }
        return DOPE_OK;
    }
    static GraphCache cache;
    std::string key((const char *)L, sizeof(*L));
    key.append((const char *)&iters, sizeof(iters));
    cudaGraphExec_t exec = cache.find(key);
    if (!exec) {
        if ((rc = configure(v))) return rc;
        cudaStream_t cs;
        if ((rc = cuda_check(cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking), "stream"))) return rc;
        cudaGraph_t graph;
        if ((rc = cuda_check(cudaStreamBeginCapture(cs, cudaStreamCaptureModeThreadLocal), "capture"))) return rc;
        for (int i = 0; i < iters && !rc; ++i) {
            rc = launch_k1(o, v, cs);
            if (!rc) rc = launch_k2(o, cs);
            if (!rc) rc = launch_digest_f(o, cs);
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

int dope_f_finish_run(const dope_lattice_f *L, void *stream) {
    LatF o;
    int rc = build(L, o, nullptr);
    if (rc) return rc;
    cudaStream_t s = (cudaStream_t)stream;
    k_energy_blocks_f<<<o.K, 256, 0, s>>>(o);
    if ((rc = cuda_check(cudaGetLastError(), "energy_f"))) return rc;
    k_finish_f<<<1, 1024, 0, s>>>(o);
    return cuda_check(cudaGetLastError(), "finish_f");
}

int dope_f_binarize(const dope_lattice_f *L, uint8_t *out, void *stream) {
    LatF o;
    int rc = build(L, o, nullptr);
    if (rc) return rc;
    if (!out) return DOPE_E_ARGS;
    const int64_t n = L->dims[0] * L->dims[1];
    k_binarize_f<<<grid_for(n), 256, 0, (cudaStream_t)stream>>>(o, n, out);
    return cuda_check(cudaGetLastError(), "binarize_f");
}

}  // extern "C"
