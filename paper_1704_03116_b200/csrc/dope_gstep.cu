// dope_gstep.cu -- the consensus ADMM step functions for ANY pairwise model on
// ANY box partition (general graph path), float64, on the device.
//
// The lattice kernels (dope_lattice.cu, dope_float.cu, dope_general.cu) hold
// the benchmarked configurations; this file covers everything else the
// reference's API accepts -- arbitrary SparseWeights pair sets (e.g. the
// kernel-3/5/7 windows of build_potts_weights, random graphs), overlapping
// 2D and 3D partitions, any mu schedule -- and backs the step-level API
// (update_blocks / solve_global / update_global / block_residuals /
// update_multipliers / consensus_objective, admm.py:113-199) and
// evaluate_energy (energy.py:187-194) for them.
//
// Layout: the symmetric CSR of W (columns ascending, both triangles), row
// sums d, counts q; every block's pixels are "entries" e = blk_ptr[k] + i
// (i = block-local index, pixels ascending, partition.py:52-59); each pixel
// lists the entries holding it (blocks ascending).  Block-local state (labels,
// multipliers, linear terms, the remainder r) is entry-indexed.
//
// The block operators of blockform.py:48-105 are evaluated on the fly:
//   C_k[i, j] = (L[g, j] / q_g) * m_j,  m_j = 1 - 1/q_j if j in block k else 1
//   r_k[i]    = d_g / q_g^2 - dhat_i,   dhat_i = sum_{j ~ g, j in k} w_gj / (q_g q_j)
// (g = global pixel of entry i, L = D - W).  With q a power of two and
// integer u / w / mu the arithmetic is exact.
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>
#include <stdio.h>

#include "common.cuh"
#include "dope_b200.h"

namespace dope_gs {

static thread_local char g_err[256] = "";

static int cuda_check(cudaError_t e, const char *what) {
    if (e == cudaSuccess) return DOPE_OK;
    snprintf(g_err, sizeof(g_err), "%s: %s", what, cudaGetErrorString(e));
    return DOPE_E_CUDA;
}

static int grid_for(int64_t n, int nt = 256) {
    int64_t b = (n + nt - 1) / nt;
    if (b > 148 * 16) b = 148 * 16;
    return (int)(b < 1 ? 1 : b);
}

// entry of block k holding pixel j, or -1
__device__ __forceinline__ int64_t entry_of(const dope_gstep &G, int64_t j, int32_t k) {
    DOPE_ASSERT(j >= 0 && j < G.n && k >= 0 && k < G.K);
    for (int64_t t = G.mem_ptr[j]; t < G.mem_ptr[j + 1]; ++t) {
        const int64_t e = G.mem_ent[t];
        if (G.ent_blk[e] == k) return e;
    }
    return -1;
}

// (C_k y)_i for entry e (pixel g of block k): CSR row of L scaled by 1/q_g and
// masked, summed in ascending column order (the diagonal in its place)
__device__ double coupling_row(const dope_gstep &G, int64_t e, const double *__restrict__ y) {
    const int64_t g = G.ent_pix[e];
    const int32_t k = G.ent_blk[e];
    const double qi = 1.0 / G.q[g];
    double s = 0.0;
    bool diag = false;
    for (int64_t t = G.adj_ptr[g]; t < G.adj_ptr[g + 1]; ++t) {
        const int64_t j = G.adj_idx[t];
        if (!diag && j > g) {
            s += ((qi * G.deg[g]) * (1.0 - qi)) * y[g];
            diag = true;
        }
        const double m = entry_of(G, j, k) >= 0 ? 1.0 - 1.0 / G.q[j] : 1.0;
        s += ((qi * -G.adj_w[t]) * m) * y[j];
    }
    if (!diag) s += ((qi * G.deg[g]) * (1.0 - qi)) * y[g];
    return s;
}

// r = d / q^2 - dhat per entry (once per model / partition)
__global__ void k_prepare(dope_gstep G, double *r) {
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < G.M; e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t g = G.ent_pix[e];
        const int32_t k = G.ent_blk[e];
        const double qi = 1.0 / G.q[g];
        double dh = 0.0;
        for (int64_t t = G.adj_ptr[g]; t < G.adj_ptr[g + 1]; ++t) {
            const int64_t j = G.adj_idx[t];
            if (entry_of(G, j, k) >= 0) dh += G.adj_w[t] * qi * (1.0 / G.q[j]);
        }
        r[e] = G.deg[g] * (qi * qi) - dh;
    }
}

// block_objective (blockform.py:89-105) for every entry of blocks [k0, k1):
// linear = uhat + lam * (C y + r * S y) + mu * ((a - S y) + 1/2)
__global__ void k_objective(dope_gstep G, int64_t e0, int64_t e1, const double *__restrict__ y,
                            const double *__restrict__ a, double mu, double lam, double *__restrict__ lin) {
    for (int64_t e = e0 + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < e1; e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t g = G.ent_pix[e];
        const double sy = y[g];
        const double uh = G.u[g] * (1.0 / G.q[g]);
        lin[e] = uh + lam * (coupling_row(G, e, y) + G.r[e] * sy) + mu * ((a[e] - sy) + 0.5);
    }
}

// solve_global (admm.py:136-151): per pixel, sum over the blocks holding it or
// a neighbour of S_k'(mu (yhat + a) - lam r yhat) - lam C_k' yhat, / (mu q);
// update_global's clamp (admm.py:172-180) when clamp != 0
__global__ void k_global(dope_gstep G, const uint8_t *__restrict__ yhat, const double *__restrict__ a, double mu,
                         double lam, double *__restrict__ y, int clamp, int *clamped) {
    int cl = 0;
    for (int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; g < G.n; g += (int64_t)gridDim.x * blockDim.x) {
        const double qg = G.q[g], qi = 1.0 / qg;
        double acc = 0.0;
        for (int64_t t = G.mem_ptr[g]; t < G.mem_ptr[g + 1]; ++t) {   // blocks holding g
            const int64_t e = G.mem_ent[t];
            const double yh = (double)yhat[e];
            acc += mu * (yh + a[e]) - lam * (G.r[e] * yh);
            acc -= lam * (((qi * G.deg[g]) * (1.0 - qi)) * yh);      // diagonal of C_k
        }
        for (int64_t s = G.adj_ptr[g]; s < G.adj_ptr[g + 1]; ++s) {  // C_k[i_j, g] for neighbours j
            const int64_t j = G.adj_idx[s];
            const double cj = (1.0 / G.q[j]) * -G.adj_w[s];
            for (int64_t t = G.mem_ptr[j]; t < G.mem_ptr[j + 1]; ++t) {
                const int64_t e = G.mem_ent[t];
                const double m = entry_of(G, g, G.ent_blk[e]) >= 0 ? 1.0 - qi : 1.0;
                acc -= lam * ((cj * m) * (double)yhat[e]);
            }
        }
        double v = acc / (mu * qg);
        if (clamp) {
            if (v < 0.0 || v > 1.0) cl = 1;
            v = v < 0.0 ? 0.0 : (v > 1.0 ? 1.0 : v);
        }
        y[g] = v;
    }
    if (clamp && __syncthreads_or(cl) && threadIdx.x == 0) atomicOr(clamped, 1);
}

// fixed-order CTA sum (deterministic: the same tree every run)
template <int NT>
__device__ double cta_sum(double v, double *sh) {
    sh[threadIdx.x] = v;
    __syncthreads();
    for (int o = NT / 2; o > 0; o >>= 1) {
        if ((int)threadIdx.x < o) sh[threadIdx.x] += sh[threadIdx.x + o];
        __syncthreads();
    }
    const double r = sh[0];
    __syncthreads();
    return r;
}

constexpr int RNT = 256;

// per block: ||yhat_k - S_k y||^2 (block_residuals, admm.py:193-199) -> ss[k]
__global__ void __launch_bounds__(RNT) k_residuals(dope_gstep G, const uint8_t *__restrict__ yhat,
                                                   const double *__restrict__ y, double *ss) {
    __shared__ double sh[RNT];
    const int32_t k = blockIdx.x;
    double acc = 0.0;
    for (int64_t e = G.blk_ptr[k] + threadIdx.x; e < G.blk_ptr[k + 1]; e += RNT) {
        const double d = (double)yhat[e] - y[G.ent_pix[e]];
        acc += d * d;
    }
    acc = cta_sum<RNT>(acc, sh);
    if (threadIdx.x == 0) ss[k] = acc;
}

// a_k += yhat_k - S_k y (update_multipliers, admm.py:183-190)
__global__ void k_multipliers(dope_gstep G, const uint8_t *__restrict__ yhat, const double *__restrict__ y,
                              double *a) {
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < G.M; e += (int64_t)gridDim.x * blockDim.x)
        a[e] = a[e] + ((double)yhat[e] - y[G.ent_pix[e]]);
}

// consensus_objective (admm.py:154-169) per block: out[2k] = yhat . (C y + r S y),
// out[2k + 1] = ||S y - (yhat + a)||^2
__global__ void __launch_bounds__(RNT) k_consensus_obj(dope_gstep G, const uint8_t *__restrict__ yhat,
                                                       const double *__restrict__ a, const double *__restrict__ y,
                                                       double *out) {
    __shared__ double sh[RNT];
    const int32_t k = blockIdx.x;
    double c = 0.0, p = 0.0;
    for (int64_t e = G.blk_ptr[k] + threadIdx.x; e < G.blk_ptr[k + 1]; e += RNT) {
        const int64_t g = G.ent_pix[e];
        const double yh = (double)yhat[e];
        c += yh * (coupling_row(G, e, y) + G.r[e] * y[g]);
        const double d = y[g] - (yh + a[e]);
        p += d * d;
    }
    c = cta_sum<RNT>(c, sh);
    p = cta_sum<RNT>(p, sh);
    if (threadIdx.x == 0) {
        out[2 * k] = c;
        out[2 * k + 1] = p;
    }
}

// evaluate_energy (energy.py:187-194): per-CTA partials of sum w (y_i - y_j)^2
// over the pair list and of sum u y, then one CTA folds them in CTA order
constexpr int ENT = 256;
constexpr int ECTAS = 592;   // 4 x 148

__global__ void __launch_bounds__(ENT) k_energy_parts(int64_t n, const double *__restrict__ u, int64_t P,
                                                      const int32_t *__restrict__ pi, const int32_t *__restrict__ pj,
                                                      const double *__restrict__ w, const double *__restrict__ y,
                                                      double *parts) {
    __shared__ double sh[ENT];
    double q = 0.0, l = 0.0;
    const int64_t stride = (int64_t)gridDim.x * ENT;
    for (int64_t p = blockIdx.x * (int64_t)ENT + threadIdx.x; p < P; p += stride) {
        const double d = y[pi[p]] - y[pj[p]];
        q += w[p] * (d * d);
    }
    for (int64_t g = blockIdx.x * (int64_t)ENT + threadIdx.x; g < n; g += stride) l += u[g] * y[g];
    q = cta_sum<ENT>(q, sh);
    l = cta_sum<ENT>(l, sh);
    if (threadIdx.x == 0) {
        parts[2 * blockIdx.x] = q;
        parts[2 * blockIdx.x + 1] = l;
    }
}

__global__ void k_energy_fold(const double *parts, int nparts, double lam, double *out) {
    double q = 0.0, l = 0.0;
    for (int i = 0; i < nparts; ++i) {
        q += parts[2 * i];
        l += parts[2 * i + 1];
    }
    out[0] = l + lam * q;
    out[1] = q;
    out[2] = l;
}

// Exhaustive minimiser (solvers.py:53-82) of every block in a batch, m <= 24:
// codes scanned with variable 0 as the most significant bit; the lowest energy
// wins, ties to the smallest code.  One CTA per block.
constexpr int XNT = 256;
__global__ void __launch_bounds__(XNT) k_exhaustive(const int64_t *node_off, const int64_t *pair_off,
                                                    const double *__restrict__ lin, const int32_t *__restrict__ pi,
                                                    const int32_t *__restrict__ pj, const double *__restrict__ w,
                                                    double lam, uint8_t *labels, double *energy) {
    __shared__ double se[XNT];
    __shared__ int64_t sc[XNT];
    const int b = blockIdx.x;
    const int64_t n0 = node_off[b], m = node_off[b + 1] - n0;
    const int64_t p0 = pair_off[b], P = pair_off[b + 1] - p0;
    double best = INFINITY;
    int64_t bcode = INT64_MAX;
    const int64_t ncodes = m > 0 ? (int64_t)1 << m : 0;
    for (int64_t c = threadIdx.x; c < ncodes; c += XNT) {
        double e = 0.0;
        for (int64_t i = 0; i < m; ++i)
            if ((c >> (m - 1 - i)) & 1) e += lin[n0 + i];
        double qd = 0.0;
        for (int64_t p = 0; p < P; ++p) {
            const int bi = (int)((c >> (m - 1 - pi[p0 + p])) & 1), bj = (int)((c >> (m - 1 - pj[p0 + p])) & 1);
            if (bi != bj) qd += w[p0 + p];
        }
        e += lam * qd;
        if (e < best) {   // ascending codes per thread: strict < keeps the smallest
            best = e;
            bcode = c;
        }
    }
    se[threadIdx.x] = best;
    sc[threadIdx.x] = bcode;
    __syncthreads();
    for (int o = XNT / 2; o > 0; o >>= 1) {
        if ((int)threadIdx.x < o) {
            const double e2 = se[threadIdx.x + o];
            const int64_t c2 = sc[threadIdx.x + o];
            if (e2 < se[threadIdx.x] || (e2 == se[threadIdx.x] && c2 < sc[threadIdx.x])) {
                se[threadIdx.x] = e2;
                sc[threadIdx.x] = c2;
            }
        }
        __syncthreads();
    }
    const int64_t code = m > 0 ? sc[0] : 0;
    for (int64_t i = threadIdx.x; i < m; i += XNT) labels[n0 + i] = (uint8_t)((code >> (m - 1 - i)) & 1);
    if (threadIdx.x == 0) energy[b] = m > 0 ? se[0] : 0.0;
}

// the partition layout (entries, memberships, counts)
static bool valid_layout(const dope_gstep *G) {
    return G && G->n >= 0 && G->K >= 0 && G->M >= 0 && G->blk_ptr && G->q && G->mem_ptr &&
           (G->M == 0 || (G->ent_pix && G->ent_blk && G->mem_ent));
}
// ... and the model (CSR of W, degrees, unary)
static bool valid(const dope_gstep *G) {
    return valid_layout(G) && G->adj_ptr && G->deg && G->u && (G->n == 0 || (G->adj_idx || G->adj_ptr));
}

}  // namespace dope_gs

using namespace dope_gs;

extern "C" {

const char *dope_gs_last_error(void) { return g_err; }

int dope_gs_prepare(const dope_gstep *G, double *r, void *stream) {
    if (!valid(G) || (G->M && !r)) return DOPE_E_ARGS;
    if (G->M == 0) return DOPE_OK;
    k_prepare<<<grid_for(G->M), 256, 0, (cudaStream_t)stream>>>(*G, r);
    return cuda_check(cudaGetLastError(), "gs_prepare");
}

int dope_gs_objective(const dope_gstep *G, int64_t e0, int64_t e1, const double *y, const double *a, double mu,
                      double lam, double *linear, void *stream) {
    if (!valid(G) || !G->r || !y || !a || !linear || e0 < 0 || e1 > G->M || e0 > e1) return DOPE_E_ARGS;
    if (e0 == e1) return DOPE_OK;
    k_objective<<<grid_for(e1 - e0), 256, 0, (cudaStream_t)stream>>>(*G, e0, e1, y, a, mu, lam, linear);
    return cuda_check(cudaGetLastError(), "gs_objective");
}

int dope_gs_solve_global(const dope_gstep *G, const uint8_t *yhat, const double *a, double mu, double lam,
                         double *y, int32_t clamp, int32_t *clamped, void *stream) {
    if (!valid(G) || !G->r || !y || (G->M && (!yhat || !a)) || (clamp && !clamped)) return DOPE_E_ARGS;
    if (!(mu > 0)) return DOPE_E_ARGS;   // admm.py:143-144
    if (G->n == 0) return DOPE_OK;
    k_global<<<grid_for(G->n), 256, 0, (cudaStream_t)stream>>>(*G, yhat, a, mu, lam, y, clamp, clamped);
    return cuda_check(cudaGetLastError(), "gs_global");
}

int dope_gs_residuals(const dope_gstep *G, const uint8_t *yhat, const double *y, double *ss, void *stream) {
    if (!valid_layout(G) || !y || !ss || (G->M && !yhat)) return DOPE_E_ARGS;
    if (G->K == 0) return DOPE_OK;
    k_residuals<<<G->K, RNT, 0, (cudaStream_t)stream>>>(*G, yhat, y, ss);
    return cuda_check(cudaGetLastError(), "gs_residuals");
}

int dope_gs_update_multipliers(const dope_gstep *G, const uint8_t *yhat, const double *y, double *a,
                               void *stream) {
    if (!valid_layout(G) || !y || (G->M && (!yhat || !a))) return DOPE_E_ARGS;
    if (G->M == 0) return DOPE_OK;
    k_multipliers<<<grid_for(G->M), 256, 0, (cudaStream_t)stream>>>(*G, yhat, y, a);
    return cuda_check(cudaGetLastError(), "gs_multipliers");
}

int dope_gs_consensus_objective(const dope_gstep *G, const uint8_t *yhat, const double *a, const double *y,
                                double *out2k, void *stream) {
    if (!valid(G) || !G->r || !y || !out2k || (G->M && (!yhat || !a))) return DOPE_E_ARGS;
    if (G->K == 0) return DOPE_OK;
    k_consensus_obj<<<G->K, RNT, 0, (cudaStream_t)stream>>>(*G, yhat, a, y, out2k);
    return cuda_check(cudaGetLastError(), "gs_consensus_objective");
}

int64_t dope_gs_energy_scratch(void) { return 2 * ECTAS; }

int dope_gs_energy(int64_t n, const double *u, int64_t npairs, const int32_t *pair_i, const int32_t *pair_j,
                   const double *w, double lam, const double *y, double *scratch, double *out3, void *stream) {
    if (n < 0 || npairs < 0 || !scratch || !out3 || (n && (!u || !y)) || (npairs && (!pair_i || !pair_j || !w)))
        return DOPE_E_ARGS;
    cudaStream_t s = (cudaStream_t)stream;
    k_energy_parts<<<ECTAS, ENT, 0, s>>>(n, u, npairs, pair_i, pair_j, w, y, scratch);
    int rc = cuda_check(cudaGetLastError(), "gs_energy");
    if (rc) return rc;
    k_energy_fold<<<1, 1, 0, s>>>(scratch, ECTAS, lam, out3);
    return cuda_check(cudaGetLastError(), "gs_energy_fold");
}

int dope_exhaustive_batch(int32_t B, const int64_t *node_off, const int64_t *pair_off, const double *linear,
                          const int32_t *pair_i, const int32_t *pair_j, const double *w, double lam,
                          uint8_t *labels, double *energy, void *stream) {
    if (B < 0 || (B && (!node_off || !pair_off || !labels || !energy))) return DOPE_E_ARGS;
    if (B == 0) return DOPE_OK;
    k_exhaustive<<<B, XNT, 0, (cudaStream_t)stream>>>(node_off, pair_off, linear, pair_i, pair_j, w, lam, labels,
                                                      energy);
    return cuda_check(cudaGetLastError(), "exhaustive");
}

}  // extern "C"
