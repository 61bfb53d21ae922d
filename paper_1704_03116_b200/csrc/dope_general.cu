// dope_general.cu -- the general lattice path behind dope_general
// (SURVEY.md §8(f) row 1 and the reference's default schedule):
//   * box partitions with overlap (make_partition overlap_pct 10 / 25,
//     partition.py:62-108): pixel block counts q in {1, 2, 4}; every block
//     owns a COPY of its pixels' labels and multipliers;
//   * float64 lattice weights, 4- or 8-connected;
//   * mu schedule mu_t = mu0 * mu_fact^t (admm.py:189) and the eps stop rule.
//
// Per block copy the block objective is blockform.py:48-105 on the stencil:
//   u_hat = u / q,  w_hat_ij = w_ij / (q_i q_j)  (pairs inside the box),
//   r_i = d_i / q_i^2 - sum_{j in box} w_hat_ij,
//   (C y)_i = (d_i / q_i)(1 - 1/q_i) y_i - sum_{j~i in box} (w_ij / q_i)(1 - 1/q_j) y_j
//             - sum_{j~i outside} (w_ij / q_i) y_j,
//   linear_i = u_hat_i + lam ((C y)_i + r_i y_i) + mu (a_i - y_i + 1/2).
// The global step is solve_global (admm.py:136-151) gathered per pixel over
// the (at most 3 x 3) blocks whose box or its one-pixel ring holds it, in
// block order; the multiplier update and block residuals are fused per block
// copy.  Capacities are quantised once per solve (scale qscale) and the block
// min cut is solved exactly on them (mincut_core.cuh), as on the float path;
// the parity bar is the float one: final energy within 1e-5 relative,
// <= 0.01 % labels.
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

#include <type_traits>
#include <stdlib.h>
#include <stdio.h>
#include <string.h>

#include <map>
#include <mutex>
#include <string>

#include "common.cuh"
#include "dope_b200.h"
#include "graph_cache.cuh"
#include "mincut_core.cuh"

namespace dope_g {
using namespace dope;
using dope_f::K1FCfg;
using dope_f::mincut_solve;

static thread_local char g_err[256] = "";
static int cuda_check(cudaError_t e, const char *what) {
    if (e == cudaSuccess) return DOPE_OK;
    snprintf(g_err, sizeof(g_err), "%s: %s", what, cudaGetErrorString(e));
    return DOPE_E_CUDA;
}

struct LatG {
    int32_t H, W, KY, KX, K, ndir, boxh, boxw, max_iters, warm, npe;
    const int32_t *rg;           // [KY lo][KY len][KX lo][KX len]
    double lam, mu0, mu_fact, eps, qs;
    const double *u;
    const double *w[4];          // E S SE SW, weight of pair (i, i + off) stored at i
    const uint8_t *q;
    double *a;                   // K * box, per copy
    uint8_t *yhat;               // K * box, per copy
    int32_t *resid;              // K * ndir * box
    double *y[3];
    double *pe;                  // npe energy partials
    double *pr;                  // K: ||yhat_k - S_k y||^2
    int32_t *pcl;                // npe clamp flags of the global step
    double *scal;                // [0] current mu
    dope_run_state *st;
    double *tr_e, *tr_rs, *tr_mr, *tr_mu;
    int32_t *tr_cl;
};

// neighbour directions: E W S N SE NW SW NE (opposite d ^ 1)
__device__ __forceinline__ int dy_of(int d) { return (d == 2 || d == 4 || d == 6) ? 1 : (d == 3 || d == 5 || d == 7) ? -1 : 0; }
__device__ __forceinline__ int dx_of(int d) { return (d == 0 || d == 4 || d == 7) ? 1 : (d == 1 || d == 5 || d == 6) ? -1 : 0; }

// x / q for a copy count (or a product of two); q = 2^k -- every box
// partition of a 2D grid has q in {1, 2, 4} -- is an exact multiplication by
// 2^-k, so the result is bit-identical to the division at a fraction of its cost
__device__ __forceinline__ double qdiv(double x, int q) {
    if ((q & (q - 1)) == 0) return x * __longlong_as_double((long long)(1023 - (31 - __clz(q))) << 52);
    return x / (double)q;
}

// weight of the pair (G, G + off_d); 0 outside the grid
__device__ __forceinline__ double wpair(const LatG &L, int R, int Cc, int d) {
    const int rn = R + dy_of(d), cn = Cc + dx_of(d);
    if (rn < 0 || rn >= L.H || cn < 0 || cn >= L.W) return 0.0;
    const int64_t W = L.W, G = (int64_t)R * W + Cc;
    switch (d) {
        case 0: return L.w[0][G];
        case 1: return L.w[0][G - 1];
        case 2: return L.w[1][G];
        case 3: return L.w[1][G - W];
        case 4: return L.w[2][G];
        case 5: return L.w[2][G - W - 1];
        case 6: return L.w[3][G];
        default: return L.w[3][G - W + 1];
    }
}

struct Box {
    int lo_r, hr, lo_c, wc;
    __device__ bool holds(int R, int Cc) const {
        return R >= lo_r && R < lo_r + hr && Cc >= lo_c && Cc < lo_c + wc;
    }
};

__device__ __forceinline__ Box box_of(const LatG &L, int k) {
    const int by = k / L.KX, bx = k - by * L.KX;
    return Box{L.rg[by], L.rg[L.KY + by], L.rg[2 * L.KY + bx], L.rg[2 * L.KY + L.KX + bx]};
}

// Per-copy stencil coefficients of pixel (R, C) inside box b:
//   d = full degree, dhat = in-box scaled degree
__device__ __forceinline__ void degrees(const LatG &L, const Box &b, int R, int Cc, int qi, double &d,
                                        double &dhat) {
    d = 0.0;
    dhat = 0.0;
    for (int dd = 0; dd < L.ndir; ++dd) {
        const double w = wpair(L, R, Cc, dd);
        if (w == 0.0) continue;
        d += w;
        const int rn = R + dy_of(dd), cn = Cc + dx_of(dd);
        if (b.holds(rn, cn)) dhat += qdiv(w, qi * (int)L.q[(int64_t)rn * L.W + cn]);
    }
}

// ---------------------------------------------------------------------------
// K1g: block min cut per copy (blockform.py:89-105 + solvers.solve_block)
// ---------------------------------------------------------------------------
template <int BH, int BW, int NT, int NDIR>
__global__ void __launch_bounds__(NT) k_block_mincut_g(LatG L, int sweep_min, int sweep_mul) {
    using Cf = K1FCfg<BH, BW, NT, NDIR>;
    constexpr int M = Cf::M, NPT = Cf::NPT;
    extern __shared__ __align__(16) uint8_t smem[];
    int32_t *g = reinterpret_cast<int32_t *>(smem + Cf::OFF_G);
    int32_t *rr = reinterpret_cast<int32_t *>(smem + Cf::OFF_R);
    uint16_t *h = reinterpret_cast<uint16_t *>(smem + Cf::OFF_H);
    uint64_t *masks = reinterpret_cast<uint64_t *>(smem + Cf::OFF_MASK);
    uint64_t *reach = reinterpret_cast<uint64_t *>(smem + Cf::OFF_REACH);
    int *misc = reinterpret_cast<int *>(smem + Cf::OFF_MISC);
    const int tid = threadIdx.x;
    const int k = blockIdx.x;
    if (L.st->stop) return;
    const Box b = box_of(L, k);
    const double mu = L.scal[0];
    const double *__restrict__ y = L.y[L.st->ycur];
    const double *__restrict__ ak = L.a + (size_t)k * M;
    int32_t *gres = L.resid + (size_t)k * NDIR * M;
    const int64_t Wg = L.W;

    // warm start: the copy's residual planes stream into shared memory first;
    // the stored flow is read back through r(v->w) + r(w->v) = 2 cap(v,w)
    if (L.warm) {
        const int4 *src = reinterpret_cast<const int4 *>(gres);
        int4 *dst = reinterpret_cast<int4 *>(rr);
#pragma unroll 4
        for (int i = tid; i < NDIR * M / 4; i += NT) dst[i] = src[i];
    }
    for (int i = 0; i < NPT; ++i) {
        const int v = tid + i * NT;
        const int r = v / BW, c = v % BW;
        int32_t gv = 0;
        if (r < b.hr && c < b.wc) {
            const int R = b.lo_r + r, Cc = b.lo_c + c;
            const int64_t G = (int64_t)R * Wg + Cc;
            const int qi = L.q[G];
            const double yi = y[G];
            // one pass over the stencil: weights and counts loaded once
            double wv[NDIR];
            int qv[NDIR];
            double d = 0.0, dhat = 0.0;
#pragma unroll
            for (int dd = 0; dd < NDIR; ++dd) {
                wv[dd] = wpair(L, R, Cc, dd);
                qv[dd] = wv[dd] != 0.0 ? (int)L.q[(int64_t)(R + dy_of(dd)) * Wg + Cc + dx_of(dd)] : 1;
            }
            // degrees() in the same order: d over the stencil, dhat over the in-box part
#pragma unroll
            for (int dd = 0; dd < NDIR; ++dd) {
                if (wv[dd] == 0.0) continue;
                d += wv[dd];
                if (b.holds(R + dy_of(dd), Cc + dx_of(dd))) dhat += qdiv(wv[dd], qi * qv[dd]);
            }
            double cy = qdiv(d, qi) * (1.0 - qdiv(1.0, qi)) * yi;
#pragma unroll
            for (int dd = 0; dd < NDIR; ++dd) {
                const double w = wv[dd];
                const int rn = R + dy_of(dd), cn = Cc + dx_of(dd);
                const bool inb = w != 0.0 && b.holds(rn, cn);
                int32_t capd = 0;
                if (w != 0.0) {
                    const int64_t Gn = (int64_t)rn * Wg + cn;
                    const int qj = qv[dd];
                    if (inb) {
                        cy += qdiv(-w, qi) * (1.0 - qdiv(1.0, qj)) * y[Gn];
                        if (!L.warm) capd = (int32_t)rint(L.lam * qdiv(w, qi * qj) * L.qs);
                    } else {
                        cy += qdiv(-w, qi) * y[Gn];
                    }
                }
                if (!L.warm) rr[dd * M + v] = capd;
            }
            const double rdiag = qdiv(d, qi * qi) - dhat;
            const double lin = qdiv(L.u[G], qi) + L.lam * (cy + rdiag * yi) + mu * ((ak[v] - yi) + 0.5);
            gv = (int32_t)fmax(fmin(rint(lin * L.qs), 1.0e9), -1.0e9);
        } else if (!L.warm) {
#pragma unroll
            for (int dd = 0; dd < NDIR; ++dd) rr[dd * M + v] = 0;
        }
        g[v] = gv;
    }
    __syncthreads();
    if (L.warm) {
        // arcs outside the copy's box (or of zero weight) hold 0 in both planes
        for (int i = 0; i < NPT; ++i) {
            const int v = tid + i * NT;
            const int r = v / BW, c = v % BW;
            if (!(r < b.hr && c < b.wc)) continue;
            int32_t f2 = 0;
#pragma unroll
            for (int dd = 0; dd < NDIR; ++dd) {
                const int rb = r + dy_of(dd), cb = c + dx_of(dd);
                if (rb >= 0 && rb < b.hr && cb >= 0 && cb < b.wc)
                    f2 += rr[dd * M + v] - rr[(dd ^ 1) * M + rb * BW + cb];
            }
            g[v] += f2 / 2;
        }
        __syncthreads();
    }
    if (mincut_solve<BH, BW, NT, NDIR>(g, rr, h, masks, reach, misc, sweep_min, sweep_mul) < 0 && tid == 0)
        atomicCAS(&L.st->error, 0, k + 1);
    uint8_t *yk = L.yhat + (size_t)k * M;
    for (int i = 0; i < NPT; ++i) {
        const int v = tid + i * NT;
        const int r = v / BW, c = v % BW;
        yk[v] = (r < b.hr && c < b.wc) ? (uint8_t)((reach[v >> 6] >> (v & 63)) & 1ull) : 0;
    }
    if (L.warm) {
        int4 *dst = reinterpret_cast<int4 *>(gres);
        const int4 *src = reinterpret_cast<const int4 *>(rr);
        for (int i = tid; i < NDIR * M / 4; i += NT) dst[i] = src[i];
    }
    if (tid == 0) atomicAdd((unsigned long long *)&L.st->solves, 1ull);
}

// cold residual planes per copy
__global__ void k_init_resid_g(LatG L, int M, int bw) {
    const int k = blockIdx.x;
    const Box b = box_of(L, k);
    int32_t *gres = L.resid + (size_t)k * L.ndir * M;
    for (int v = threadIdx.x; v < M; v += blockDim.x) {
        const int r = v / bw, c = v % bw;
        const bool valid = r < b.hr && c < b.wc;
        const int R = b.lo_r + r, Cc = b.lo_c + c;
        for (int d = 0; d < L.ndir; ++d) {
            int32_t cap = 0;
            if (valid) {
                const double w = wpair(L, R, Cc, d);
                const int rn = R + dy_of(d), cn = Cc + dx_of(d);
                if (w != 0.0 && b.holds(rn, cn)) {
                    const double qi = L.q[(int64_t)R * L.W + Cc], qj = L.q[(int64_t)rn * L.W + cn];
                    cap = (int32_t)rint(L.lam * (w / (qi * qj)) * L.qs);
                }
            }
            gres[d * M + v] = cap;
        }
    }
}

__global__ void k_init_state_g(LatG L, int64_t n, int64_t ncopy) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    const int64_t i0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    for (int64_t i = i0; i < n; i += stride) L.y[0][i] = 0.5;   // admm.py:102-110
    for (int64_t i = i0; i < ncopy; i += stride) {
        L.a[i] = 0.0;
        L.yhat[i] = 0;
    }
    if (i0 == 0) {
        dope_run_state s;
        memset(&s, 0, sizeof(s));
        s.best_energy = __double_as_longlong(INFINITY);
        *L.st = s;
        L.scal[0] = L.mu0;
    }
}

// ---------------------------------------------------------------------------
// K2g: global step (admm.py:136-151, 172-180), one thread per pixel
// ---------------------------------------------------------------------------
#ifndef KG_MINB
#define KG_MINB 4
#endif
__global__ void __launch_bounds__(256, KG_MINB) k_global_g(LatG L, int boxw, int M) {
    const dope_run_state *st = L.st;
    if (st->stop) return;
    const int cur = st->ycur, best = st->ybest;
    const int out = (cur == best) ? (cur + 1) % 3 : 3 - cur - best;
    double *__restrict__ yo = L.y[out];
    const double mu = L.scal[0];
    const int64_t n = (int64_t)L.H * L.W;
    const int baseY = L.H / L.KY, baseX = L.W / L.KX;
    int clamped = 0;
    for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < n; p += (int64_t)gridDim.x * blockDim.x) {
        const int R = (int)(p / L.W), Cc = (int)(p - (int64_t)R * L.W);
        const int qp = L.q[p];
        // the pixel's stencil, loaded once: weights and neighbour block counts
        double wd[8];
        int qd[8];
        double d = 0.0;
        bool pow2 = (qp & (qp - 1)) == 0;
        // the neighbours' counts are loaded with the weights, not after them
        // (clamped into the grid; a pair outside has weight 0 and count 1)
        int qraw[8];
#pragma unroll
        for (int dd = 0; dd < 8; ++dd) {
            int rn = R + dy_of(dd), cn = Cc + dx_of(dd);
            rn = rn < 0 ? 0 : (rn >= L.H ? L.H - 1 : rn);
            cn = cn < 0 ? 0 : (cn >= L.W ? L.W - 1 : cn);
            qraw[dd] = dd < L.ndir ? (int)L.q[(int64_t)rn * L.W + cn] : 1;
            wd[dd] = dd < L.ndir ? wpair(L, R, Cc, dd) : 0.0;
        }
#pragma unroll
        for (int dd = 0; dd < 8; ++dd) {
            qd[dd] = wd[dd] != 0.0 ? qraw[dd] : 1;
            pow2 &= (qd[dd] & (qd[dd] - 1)) == 0;
            d += wd[dd];
        }
        // candidate blocks: the base-range owner +-1 on each axis (boxes grow
        // by less than a block length, so nothing further holds the pixel or
        // its ring), in block order
        int by0 = R / (baseY > 0 ? baseY : 1), bx0 = Cc / (baseX > 0 ? baseX : 1);
        by0 = by0 >= L.KY ? L.KY - 1 : by0;
        bx0 = bx0 >= L.KX ? L.KX - 1 : bx0;
        double acc = 0.0;
        // P2: every count here is a power of two -- the divisions become exact
        // multiplications by per-pixel reciprocals (2^-k, exact in float too)
        auto candidates = [&](auto P2) {
            constexpr bool p2 = decltype(P2)::value;
            float iq[8];
            float iqp = 1.0f;
            if (p2) {
                iqp = 1.0f / (float)qp;
#pragma unroll
                for (int dd = 0; dd < 8; ++dd) iq[dd] = 1.0f / (float)qd[dd];
            }
            const double inq = p2 ? 1.0 - (double)iqp : 1.0 - qdiv(1.0, qp);
            for (int by = by0 - 1; by <= by0 + 1; ++by) {
                if (by < 0 || by >= L.KY) continue;
                const int lr = L.rg[by], hr = L.rg[L.KY + by];
                if (R < lr - 1 || R > lr + hr) continue;
                for (int bx = bx0 - 1; bx <= bx0 + 1; ++bx) {
                    if (bx < 0 || bx >= L.KX) continue;
                    const int lc = L.rg[2 * L.KY + bx], wc = L.rg[2 * L.KY + L.KX + bx];
                    if (Cc < lc - 1 || Cc > lc + wc) continue;
                    const int k = by * L.KX + bx;
                    const Box b{lr, hr, lc, wc};
                    const uint8_t *yk = L.yhat + (size_t)k * M;
                    const bool inb = b.holds(R, Cc);
                    double ct = 0.0, dhat = 0.0;
#pragma unroll
                    for (int dd = 0; dd < 8; ++dd) {
                        if (wd[dd] == 0.0) continue;
                        const int rn = R + dy_of(dd), cn = Cc + dx_of(dd);
                        if (!b.holds(rn, cn)) continue;
                        const double yi = yk[(rn - lr) * boxw + (cn - lc)];
                        const double wq = p2 ? -wd[dd] * (double)iq[dd] : qdiv(-wd[dd], qd[dd]);
                        ct += inb ? wq * inq * yi : wq * yi;
                        dhat += p2 ? wd[dd] * (double)(iqp * iq[dd]) : qdiv(wd[dd], qp * qd[dd]);
                    }
                    if (inb) {
                        const int v = (R - lr) * boxw + (Cc - lc);
                        const double yh = yk[v];
                        const double rdiag = (p2 ? d * (double)(iqp * iqp) : qdiv(d, qp * qp)) - dhat;
                        acc += mu * (yh + L.a[(size_t)k * M + v]) - L.lam * (rdiag * yh);
                        ct += (p2 ? d * (double)iqp : qdiv(d, qp)) * inq * yh;
                    }
                    acc -= L.lam * ct;
                }
            }
        };
        if (pow2) candidates(std::true_type{});
        else candidates(std::false_type{});
        double yv = acc / (mu * (double)qp);
        clamped |= (yv < 0.0 || yv > 1.0);
        yv = yv < 0.0 ? 0.0 : (yv > 1.0 ? 1.0 : yv);
        yo[p] = yv;
    }
    clamped = __syncthreads_or(clamped);
    if (threadIdx.x == 0 && clamped) L.pcl[blockIdx.x % L.npe] = 1;
}

// ---------------------------------------------------------------------------
// K3g: block residuals + multiplier update per copy (admm.py:183-199)
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256) k_residual_g(LatG L, int boxw, int M) {
    const dope_run_state *st = L.st;
    if (st->stop) return;
    const int cur = st->ycur, best = st->ybest;
    const int out = (cur == best) ? (cur + 1) % 3 : 3 - cur - best;
    const double *__restrict__ y = L.y[out];
    const int k = blockIdx.x;
    const Box b = box_of(L, k);
    double ss = 0.0;
    const int m = b.hr * b.wc;
    for (int i = threadIdx.x; i < m; i += blockDim.x) {
        const int r = i / b.wc, c = i - r * b.wc;
        const int v = r * boxw + c;
        const double diff = (double)L.yhat[(size_t)k * M + v] - y[(int64_t)(b.lo_r + r) * L.W + b.lo_c + c];
        ss += diff * diff;
        L.a[(size_t)k * M + v] += diff;
    }
    __shared__ double red[8];
    for (int o = 16; o > 0; o >>= 1) ss += __shfl_xor_sync(FULLMASK, ss, o);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = ss;
    __syncthreads();
    if (threadIdx.x == 0) {
        double t = 0.0;
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += red[w];
        L.pr[k] = t;
    }
}

// ---------------------------------------------------------------------------
// K4g: energy of the new iterate (energy.py:187-194), fixed-order partials
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256) k_energy_g(LatG L) {
    const dope_run_state *st = L.st;
    if (st->stop) return;
    const int cur = st->ycur, best = st->ybest;
    const int out = (cur == best) ? (cur + 1) % 3 : 3 - cur - best;
    const double *__restrict__ y = L.y[out];
    const int64_t n = (int64_t)L.H * L.W;
    double e = 0.0;
    for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < n; p += (int64_t)gridDim.x * blockDim.x) {
        const int R = (int)(p / L.W), Cc = (int)(p - (int64_t)R * L.W);
        const double yp = y[p];
        double pair = 0.0;
        // forward pairs E S SE SW, each stored at its lower pixel
        const int fwd[4] = {0, 2, 4, 6};
        for (int t = 0; t < (L.ndir == 8 ? 4 : 2); ++t) {
            const int d = fwd[t];
            const double w = wpair(L, R, Cc, d);
            if (w == 0.0) continue;
            const double df = yp - y[(int64_t)(R + dy_of(d)) * L.W + Cc + dx_of(d)];
            pair += w * df * df;
        }
        e += L.u[p] * yp + L.lam * pair;
    }
    __shared__ double red[8];
    for (int o = 16; o > 0; o >>= 1) e += __shfl_xor_sync(FULLMASK, e, o);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = e;
    __syncthreads();
    if (threadIdx.x == 0) {
        double t = 0.0;
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += red[w];
        L.pe[blockIdx.x] = t;
    }
}

// ---------------------------------------------------------------------------
// finalize: trace, best iterate (strict <), mu *= mu_fact, stop rule
// (admm.py:228-249); one thread, fixed summation order
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(1024) k_finalize_g(LatG L) {
    dope_run_state *st = L.st;
    if (st->stop) return;
    // fixed-order reduction over the partials: thread-strided, then a fixed
    // shuffle tree and warp order (deterministic)
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    double E = 0.0, R2 = 0.0, mx = 0.0;
    int cl = 0;
    for (int i = tid; i < L.npe; i += blockDim.x) {
        E += L.pe[i];
        cl |= L.pcl[i];
        L.pcl[i] = 0;
    }
    for (int k = tid; k < L.K; k += blockDim.x) {
        const double r = sqrt(L.pr[k]);
        R2 += r * r;
        mx = r > mx ? r : mx;
    }
    for (int o = 16; o > 0; o >>= 1) {
        E += __shfl_xor_sync(FULLMASK, E, o);
        R2 += __shfl_xor_sync(FULLMASK, R2, o);
        const double m2 = __shfl_xor_sync(FULLMASK, mx, o);
        mx = m2 > mx ? m2 : mx;
    }
    cl = __any_sync(FULLMASK, cl);
    __shared__ double sE[32], sR[32], sM[32];
    __shared__ int sC[32];
    if (lane == 0) { sE[warp] = E; sR[warp] = R2; sM[warp] = mx; sC[warp] = cl; }
    __syncthreads();
    if (tid != 0) return;
    E = 0.0;
    R2 = 0.0;
    mx = 0.0;
    cl = 0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) {
        E += sE[w];
        R2 += sR[w];
        mx = sM[w] > mx ? sM[w] : mx;
        cl |= sC[w];
    }
    const int t = st->iteration;
    const double mu = L.scal[0];
    if (t < L.max_iters) {
        L.tr_e[t] = E;
        L.tr_rs[t] = R2;
        L.tr_mr[t] = mx;
        L.tr_mu[t] = mu;
        L.tr_cl[t] = cl;
    }
    const int cur = st->ycur, best = st->ybest;
    const int out = (cur == best) ? (cur + 1) % 3 : 3 - cur - best;
    if (E < __longlong_as_double(st->best_energy)) {
        st->best_energy = __double_as_longlong(E);
        st->best_iteration = t + 1;
        st->ybest = out;
    }
    st->ycur = out;
    st->iteration = t + 1;
    L.scal[0] = mu * L.mu_fact;
    if (L.K == 0 || mx <= L.eps) {
        st->converged = 1;
        st->stop = 1;
    }
    if (st->error) st->stop = 1;
}

// state.y := best unless converged (admm.py:250-251): point ycur at it
__global__ void k_finish_g(LatG L) {
    dope_run_state *st = L.st;
    if (!st->converged && st->iteration > 0) st->ycur = st->ybest;
}

__global__ void k_binarize_g(LatG L, int64_t n, uint8_t *out) {
    const double *y = L.y[L.st->ycur];
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        out[i] = y[i] >= 0.5 ? 1 : 0;
}

// ---------------------------------------------------------------------------
// host side
// ---------------------------------------------------------------------------
struct VarG {
    int bh, bw, nt, ndir;
    size_t smem;
    void (*kernel)(LatG, int, int);
};

template <int BH, int BW, int NT, int ND>
static VarG make_varg() {
    return VarG{BH, BW, NT, ND, K1FCfg<BH, BW, NT, ND>::SMEM, &k_block_mincut_g<BH, BW, NT, ND>};
}

static const VarG *pick_varg(int conn, int maxh, int maxw, int ncopies) {
    static const VarG table[] = {
        // 40 x 48: the 32-blocks of a 25 %-overlap partition (boxes <= 40 x 40)
        // without padding them to 64 x 64 (1920 nodes: 30 BFS words)
        make_varg<32, 32, 256, 4>(), make_varg<40, 48, 384, 4>(), make_varg<64, 64, 512, 4>(),
        make_varg<32, 32, 256, 8>(), make_varg<40, 48, 384, 8>(), make_varg<64, 64, 512, 8>(),
    };
    // few block copies per SM: the slowest solve sets K1g, more threads per
    // copy pay (as in the integer and float paths); DOPE_K1_WIDE=0/1 forces
    static const VarG wide[] = {
        make_varg<32, 32, 512, 4>(), make_varg<40, 48, 960, 4>(), make_varg<64, 64, 1024, 4>(),
        make_varg<32, 32, 512, 8>(), make_varg<40, 48, 960, 8>(), make_varg<64, 64, 1024, 8>(),
    };
    static const int force = getenv("DOPE_K1_WIDE") ? atoi(getenv("DOPE_K1_WIDE")) : -1;
    static const int sms = [] {
        int dev = 0, n = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
        return n > 0 ? n : 148;
    }();
    const bool use_wide = force >= 0 ? force != 0 : (ncopies > 0 && ncopies <= 8 * sms);
    for (const VarG &v : (use_wide ? wide : table))
        if (v.ndir == conn && maxh <= v.bh && maxw <= v.bw) return &v;
    return nullptr;
}

static int npe_for(int64_t n) {
    int64_t b = (n + 255) / 256;
    if (b > 148 * 8) b = 148 * 8;
    return (int)(b < 1 ? 1 : b);
}

static int build(const dope_general *L, LatG &o, const VarG **var) {
    if (!L || !L->u || !L->q || !L->ranges || !L->a || !L->yhat || !L->resid || !L->y[0] || !L->y[1] ||
        !L->y[2] || !L->part_energy || !L->part_ressq || !L->part_flags || !L->scal || !L->state)
        return DOPE_E_ARGS;
    if (L->conn != 4 && L->conn != 8) return DOPE_E_GEOMETRY;
    for (int i = 0; i < (L->conn == 8 ? 4 : 2); ++i)
        if (!L->w[i]) return DOPE_E_ARGS;
    if (L->dims[0] < 1 || L->dims[1] < 1 || L->kpa[0] < 1 || L->kpa[1] < 1 || L->kpa[0] > L->dims[0] ||
        L->kpa[1] > L->dims[1] || L->dims[0] * L->dims[1] > INT32_MAX)
        return DOPE_E_ARGS;
    if (!(L->mu0 > 0) || L->lam < 0 || !(L->qscale > 0) || L->mu_fact < 1.0 || L->eps < 0) return DOPE_E_ARGS;
    if (L->box[0] < 1 || L->box[1] < 1) return DOPE_E_ARGS;
    memset(&o, 0, sizeof(o));
    o.H = (int32_t)L->dims[0];
    o.W = (int32_t)L->dims[1];
    o.KY = L->kpa[0];
    o.KX = L->kpa[1];
    o.K = o.KY * o.KX;
    o.ndir = L->conn;
    o.max_iters = L->max_iters;
    o.warm = L->warm_start;
    o.rg = L->ranges;
    o.lam = L->lam;
    o.mu0 = L->mu0;
    o.mu_fact = L->mu_fact;
    o.eps = L->eps;
    o.qs = L->qscale;
    o.u = L->u;
    for (int i = 0; i < 4; ++i) o.w[i] = L->w[i];
    o.q = L->q;
    o.a = L->a;
    o.yhat = L->yhat;
    o.resid = L->resid;
    for (int i = 0; i < 3; ++i) o.y[i] = L->y[i];
    o.pe = L->part_energy;
    o.pr = L->part_ressq;
    o.pcl = L->part_flags;
    o.scal = L->scal;
    o.st = L->state;
    o.tr_e = L->trace_energy;
    o.tr_rs = L->trace_residual_sq;
    o.tr_mr = L->trace_max_residual;
    o.tr_mu = L->trace_mu;
    o.tr_cl = L->trace_clamped;
    o.npe = npe_for((int64_t)o.H * o.W);
    const VarG *v = pick_varg(L->conn, L->box[0], L->box[1], o.K);
    if (!v) return DOPE_E_GEOMETRY;
    o.boxh = v->bh;
    o.boxw = v->bw;
    if (var) *var = v;
    return DOPE_OK;
}

static int configure(const VarG *v) {
    static std::mutex mu;
    static std::map<const VarG *, bool> done;
    std::lock_guard<std::mutex> lk(mu);
    if (done[v]) return DOPE_OK;
    int rc = cuda_check(cudaFuncSetAttribute(v->kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)v->smem),
                        "attr K1g");
    if (!rc) done[v] = true;
    return rc;
}

static int blocks_pass(const LatG &o, const VarG *v, cudaStream_t s) {
    static const int smin = getenv("DOPE_SWEEPG_MIN") ? atoi(getenv("DOPE_SWEEPG_MIN")) : 1;
    static const int smul = getenv("DOPE_SWEEPG_MUL") ? atoi(getenv("DOPE_SWEEPG_MUL")) : 1;
    v->kernel<<<o.K, v->nt, v->smem, s>>>(o, smin, smul);
    return cuda_check(cudaGetLastError(), "general K1");
}

static int global_pass(const LatG &o, cudaStream_t s) {
    const int M = o.boxh * o.boxw;
    k_global_g<<<o.npe, 256, 0, s>>>(o, o.boxw, M);
    k_residual_g<<<o.K, 256, 0, s>>>(o, o.boxw, M);
    k_energy_g<<<o.npe, 256, 0, s>>>(o);
    k_finalize_g<<<1, 1024, 0, s>>>(o);
    return cuda_check(cudaGetLastError(), "general global step");
}

static int one_iteration(const LatG &o, const VarG *v, cudaStream_t s) {
    int rc = blocks_pass(o, v, s);
    return rc ? rc : global_pass(o, s);
}

}  // namespace dope_g

using namespace dope_g;

extern "C" {

const char *dope_g_last_error(void) { return g_err; }

int64_t dope_g_copy_stride(const dope_general *L) {
    if (!L) return 0;
    const VarG *v = pick_varg(L->conn, L->box[0], L->box[1], 0);
    return v ? (int64_t)v->bh * v->bw : 0;
}

int64_t dope_g_box_width(const dope_general *L) {
    if (!L) return 0;
    const VarG *v = pick_varg(L->conn, L->box[0], L->box[1], 0);
    return v ? (int64_t)v->bw : 0;
}

int64_t dope_g_partials(const dope_general *L) {
    if (!L || L->dims[0] < 1 || L->dims[1] < 1) return 0;
    return npe_for(L->dims[0] * L->dims[1]);
}

int dope_g_check(const dope_general *L) {
    LatG o;
    return build(L, o, nullptr);
}

int dope_g_admm_init(const dope_general *L, void *stream) {
    LatG o;
    const VarG *v;
    int rc = build(L, o, &v);
    if (rc) return rc;
    if ((rc = configure(v))) return rc;
    cudaStream_t s = (cudaStream_t)stream;
    const int M = o.boxh * o.boxw;
    const int64_t n = (int64_t)o.H * o.W, ncopy = (int64_t)o.K * M;
    k_init_state_g<<<148 * 4, 256, 0, s>>>(o, n, ncopy);
    k_init_resid_g<<<o.K, 256, 0, s>>>(o, M, o.boxw);
    cudaMemsetAsync(o.pcl, 0, sizeof(int32_t) * o.npe, s);
    return cuda_check(cudaGetLastError(), "general init");
}

int dope_g_admm_run(const dope_general *L, int32_t iters, int32_t use_graph, void *stream) {
    LatG o;
    const VarG *v;
    int rc = build(L, o, &v);
    if (rc) return rc;
    if ((rc = configure(v))) return rc;
    cudaStream_t s = (cudaStream_t)stream;
    if (iters <= 0) return DOPE_OK;
    if (!use_graph) {
        for (int i = 0; i < iters; ++i)
            if ((rc = one_iteration(o, v, s))) return rc;
        return DOPE_OK;
    }
    static GraphCache cache;
    std::string key((const char *)L, sizeof(*L));
    key.append((const char *)&iters, sizeof(iters));
    cudaGraphExec_t exec = cache.find(key);
    if (!exec) {
        cudaStream_t cs;
        if (cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking) != cudaSuccess) return DOPE_E_CUDA;
        cudaGraph_t graph;
        if (cudaStreamBeginCapture(cs, cudaStreamCaptureModeThreadLocal) != cudaSuccess) return DOPE_E_CUDA;
        for (int i = 0; i < iters && !rc; ++i) rc = one_iteration(o, v, cs);
        cudaError_t e = cudaStreamEndCapture(cs, &graph);
        if (rc) return rc;
        if (e != cudaSuccess) return cuda_check(e, "capture");
        if (cudaGraphInstantiate(&exec, graph, 0) != cudaSuccess) return DOPE_E_CUDA;
        cudaGraphDestroy(graph);
        cudaStreamDestroy(cs);
        cache.put(key, exec);
    }
    return cuda_check(cudaGraphLaunch(exec, s), "graph launch");
}

int dope_g_update_blocks(const dope_general *L, void *stream) {
    LatG o;
    const VarG *v;
    int rc = build(L, o, &v);
    if (rc) return rc;
    if ((rc = configure(v))) return rc;
    return blocks_pass(o, v, (cudaStream_t)stream);
}

int dope_g_update_global(const dope_general *L, void *stream) {
    LatG o;
    int rc = build(L, o, nullptr);
    if (rc) return rc;
    return global_pass(o, (cudaStream_t)stream);
}

int dope_g_finish_run(const dope_general *L, void *stream) {
    LatG o;
    int rc = build(L, o, nullptr);
    if (rc) return rc;
    k_finish_g<<<1, 1, 0, (cudaStream_t)stream>>>(o);
    return cuda_check(cudaGetLastError(), "general finish");
}

int dope_g_binarize(const dope_general *L, uint8_t *out, void *stream) {
    LatG o;
    int rc = build(L, o, nullptr);
    if (rc) return rc;
    if (!out) return DOPE_E_ARGS;
    const int64_t n = (int64_t)o.H * o.W;
    k_binarize_g<<<npe_for(n), 256, 0, (cudaStream_t)stream>>>(o, n, out);
    return cuda_check(cudaGetLastError(), "general binarize");
}

}  // extern "C"
