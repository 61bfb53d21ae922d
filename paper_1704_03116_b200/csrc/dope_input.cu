// dope_input.cu -- model construction on the GPU:
//   * contrast-sensitive Potts weights over a lattice window
//     (energy.py:124-162 build_potts_weights): pairs enumerated per half-kernel
//     offset, source region row-major, w = exp(-|x_i - x_j|^2 / (2 sigma^2));
//   * the RMS neighbour difference that picks sigma (energy.py:165-184);
//   * colour-model unaries (energy.py:298-323 compute_unaries): per pixel the
//     log-posterior ratio of two k-means mixtures (log-sum-exp), seeds pinned
//     to -/+ 1e6 * (1 + max |u| over unseeded pixels).
// All of it is element-wise / reduction work over HBM-resident images.
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>
#include <stdio.h>

#include "common.cuh"
#include "dope_b200.h"

namespace dope_in {
using namespace dope;

static thread_local char g_err[256] = "";
static int cuda_check(cudaError_t e, const char *what) {
    if (e == cudaSuccess) return DOPE_OK;
    snprintf(g_err, sizeof(g_err), "%s: %s", what, cudaGetErrorString(e));
    return DOPE_E_CUDA;
}

// lattice window (passed by value: <= 32 KB of kernel parameters)
constexpr int MAXOFF = 240;   // half window of a 3D kernel-9 ball is the largest
struct Win {
    int ndim;
    int64_t dims[3], strides[3];
    int noff;
    int32_t off[MAXOFF][3];
    int32_t lo[MAXOFF][3], ext[MAXOFF][3];   // source region per offset
    int64_t start[MAXOFF + 1];                // prefix of pair counts per offset
};

// pair p -> (i, j) of the reference's enumeration order
__device__ __forceinline__ void pair_of(const Win &w, int64_t p, int &o, int64_t &i, int64_t &j) {
    // offset of pair p: binary search over the prefix counts
    int lo = 0, hi = w.noff - 1;
    while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (p >= w.start[mid]) lo = mid;
        else hi = mid - 1;
    }
    o = lo;
    int64_t q = p - w.start[o];
    int64_t idx = 0, jdx = 0;
    for (int a = w.ndim - 1; a >= 0; --a) {
        const int64_t e = w.ext[o][a];
        const int64_t c = q % e;
        q /= e;
        const int64_t x = w.lo[o][a] + c;
        idx += x * w.strides[a];
        jdx += (x + w.off[o][a]) * w.strides[a];
    }
    i = idx;
    j = jdx;
}

__global__ void k_potts_weights(Win w, int channels, const double *__restrict__ data, double inv2s2, int contrast,
                                int64_t *__restrict__ rows, int64_t *__restrict__ cols, double *__restrict__ vals) {
    const int64_t total = w.start[w.noff];
    for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < total;
         p += (int64_t)gridDim.x * blockDim.x) {
        int o;
        int64_t i, j;
        pair_of(w, p, o, i, j);
        double v = 1.0;
        if (contrast) {
            double d2 = 0.0;
            for (int c = 0; c < channels; ++c) {
                const double d = data[i * channels + c] - data[j * channels + c];
                d2 += d * d;
            }
            v = exp(-d2 * inv2s2);
        }
        rows[p] = i;
        cols[p] = j;
        vals[p] = v;
    }
}

// sum over pairs of |x_i - x_j|^2: per-CTA partials in fixed order
__global__ void __launch_bounds__(256) k_sq_diff(Win w, int channels, const double *__restrict__ data,
                                                 double *__restrict__ part) {
    const int64_t total = w.start[w.noff];
    double acc = 0.0;
    for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < total;
         p += (int64_t)gridDim.x * blockDim.x) {
        int o;
        int64_t i, j;
        pair_of(w, p, o, i, j);
        for (int c = 0; c < channels; ++c) {
            const double d = data[i * channels + c] - data[j * channels + c];
            acc += d * d;
        }
    }
    __shared__ double red[8];
    for (int s = 16; s > 0; s >>= 1) acc += __shfl_xor_sync(FULLMASK, acc, s);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
    __syncthreads();
    if (threadIdx.x == 0) {
        double t = 0.0;
        for (int k = 0; k < 8; ++k) t += red[k];
        part[blockIdx.x] = t;
    }
}

// log sum_c w_c exp(-|x - c|^2 / (2 sigma^2)) (energy.py:290-296)
__device__ __forceinline__ double mixture_ll(const double *x, int channels, const double *cent, const double *wt,
                                             int ncl, double inv2s2) {
    double z[16];
    double zmax = -INFINITY;
    for (int k = 0; k < ncl; ++k) {
        double d2 = 0.0;
        for (int c = 0; c < channels; ++c) {
            const double d = x[c] - cent[k * channels + c];
            d2 += d * d;
        }
        const double lw = wt[k] > 0 ? log(fmax(wt[k], 1e-300)) : -INFINITY;
        z[k] = lw - d2 * inv2s2;
        zmax = z[k] > zmax ? z[k] : zmax;
    }
    double s = 0.0;
    for (int k = 0; k < ncl; ++k) s += exp(z[k] - zmax);
    return zmax + log(s);
}

__global__ void __launch_bounds__(256) k_unaries(int64_t n, int channels, const double *__restrict__ data,
                                                 const int8_t *__restrict__ seeds, const double *__restrict__ fgc,
                                                 const double *__restrict__ bgc, const double *__restrict__ fgw,
                                                 const double *__restrict__ bgw, int ncl, double inv2s2,
                                                 double *__restrict__ u, double *__restrict__ part) {
    double mx = 0.0;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const double *x = data + i * channels;
        const double v = mixture_ll(x, channels, bgc, bgw, ncl, inv2s2) - mixture_ll(x, channels, fgc, fgw, ncl, inv2s2);
        u[i] = v;
        if (!seeds || seeds[i] == 0) mx = fabs(v) > mx ? fabs(v) : mx;
    }
    __shared__ double red[8];
    for (int s = 16; s > 0; s >>= 1) {
        const double t = __shfl_xor_sync(FULLMASK, mx, s);
        mx = t > mx ? t : mx;
    }
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = mx;
    __syncthreads();
    if (threadIdx.x == 0) {
        double t = 0.0;
        for (int k = 0; k < 8; ++k) t = red[k] > t ? red[k] : t;
        part[blockIdx.x] = t;
    }
}

// seeded pixels pinned to -/+ u_max (energy.py:319-322); u_max from the partials
__global__ void k_pin_seeds(int64_t n, const int8_t *__restrict__ seeds, int npart, const double *__restrict__ part,
                            double *__restrict__ u) {
    __shared__ double umax;
    if (threadIdx.x == 0) {
        double b = 0.0;
        for (int k = 0; k < npart; ++k) b = part[k] > b ? part[k] : b;
        umax = 1e6 * (1.0 + b);
    }
    __syncthreads();
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        if (seeds[i] == 2) u[i] = -umax;       // SEED_FG
        else if (seeds[i] == 1) u[i] = umax;   // SEED_BG
    }
}

static int build_win(int ndim, const int64_t *dims, int noff, const int32_t *offs, Win &w) {
    if (ndim < 2 || ndim > 3 || noff < 1 || noff > MAXOFF || !dims || !offs) return DOPE_E_ARGS;
    w.ndim = ndim;
    w.noff = noff;
    int64_t s = 1;
    for (int a = ndim - 1; a >= 0; --a) {
        if (dims[a] < 1) return DOPE_E_ARGS;
        w.dims[a] = dims[a];
        w.strides[a] = s;
        s *= dims[a];
    }
    w.start[0] = 0;
    for (int o = 0; o < noff; ++o) {
        int64_t cnt = 1;
        for (int a = 0; a < ndim; ++a) {
            const int32_t d = offs[o * ndim + a];
            w.off[o][a] = d;
            if (dims[a] > INT32_MAX) return DOPE_E_ARGS;
            const int64_t lo = d < 0 ? -d : 0, hi = dims[a] - (d > 0 ? d : 0);
            w.lo[o][a] = (int32_t)lo;
            w.ext[o][a] = (int32_t)(hi > lo ? hi - lo : 0);
            cnt *= w.ext[o][a];
        }
        w.start[o + 1] = w.start[o] + cnt;
    }
    return DOPE_OK;
}

static int grid_for(int64_t n) {
    int64_t b = (n + 255) / 256;
    if (b > 148 * 8) b = 148 * 8;
    return (int)(b < 1 ? 1 : b);
}

}  // namespace dope_in

using namespace dope_in;

extern "C" {

const char *dope_in_last_error(void) { return g_err; }

int64_t dope_in_pair_count(int32_t ndim, const int64_t *dims, int32_t noff, const int32_t *offs) {
    Win w;
    return build_win(ndim, dims, noff, offs, w) ? -1 : w.start[noff];
}

int dope_in_potts_weights(int32_t ndim, const int64_t *dims, int32_t channels, const double *data, int32_t noff,
                          const int32_t *offs, double sigma, int32_t contrast, int64_t *rows, int64_t *cols,
                          double *vals, void *stream) {
    Win w;
    int rc = build_win(ndim, dims, noff, offs, w);
    if (rc) return rc;
    if (!(sigma > 0) || channels < 1 || (contrast && !data)) return DOPE_E_ARGS;
    const int64_t total = w.start[noff];
    if (total == 0) return DOPE_OK;
    if (!rows || !cols || !vals) return DOPE_E_ARGS;
    k_potts_weights<<<grid_for(total), 256, 0, (cudaStream_t)stream>>>(w, channels, data, 1.0 / (2.0 * sigma * sigma),
                                                                       contrast, rows, cols, vals);
    return cuda_check(cudaGetLastError(), "potts weights");
}

int64_t dope_in_partials(int64_t n) { return grid_for(n); }

int dope_in_sq_diff(int32_t ndim, const int64_t *dims, int32_t channels, const double *data, int32_t noff,
                    const int32_t *offs, double *partials, void *stream) {
    Win w;
    int rc = build_win(ndim, dims, noff, offs, w);
    if (rc) return rc;
    if (!data || !partials || channels < 1) return DOPE_E_ARGS;
    const int64_t total = w.start[noff];
    k_sq_diff<<<grid_for(total), 256, 0, (cudaStream_t)stream>>>(w, channels, data, partials);
    return cuda_check(cudaGetLastError(), "sq diff");
}

int dope_in_unaries(int64_t n, int32_t channels, const double *data, const int8_t *seeds, const double *fg_centroids,
                    const double *bg_centroids, const double *fg_weights, const double *bg_weights,
                    int32_t nclusters, double bandwidth, double *u, double *partials, void *stream) {
    if (n < 1 || channels < 1 || !data || !fg_centroids || !bg_centroids || !fg_weights || !bg_weights || !u ||
        !partials || nclusters < 1 || nclusters > 16 || !(bandwidth > 0))
        return DOPE_E_ARGS;
    cudaStream_t s = (cudaStream_t)stream;
    const int g = grid_for(n);
    k_unaries<<<g, 256, 0, s>>>(n, channels, data, seeds, fg_centroids, bg_centroids, fg_weights, bg_weights,
                                nclusters, 1.0 / (2.0 * bandwidth * bandwidth), u, partials);
    int rc = cuda_check(cudaGetLastError(), "unaries");
    if (rc || !seeds) return rc;
    k_pin_seeds<<<g, 256, 0, s>>>(n, seeds, g, partials, u);
    return cuda_check(cudaGetLastError(), "pin seeds");
}

}  // extern "C"
