/*
 * dope_oracle.c -- CPU ORACLE.  TEST INFRASTRUCTURE ONLY.
 *
 * This file is the checker, never the product.  Only tests/, the smoke()
 * check in __graft_entry__.py and bench.py's cpu_baseline / --impl reference
 * leg may load it.  The product path (paper_1704_03116_b200) never links or
 * calls anything here and fails loudly when its CUDA library is missing.
 *
 * It restates, in plain C, the reference algorithm on the DOPE hot path:
 *
 *  1. oracle_bk_maxflow: the two-tree augmenting-path max-flow of
 *     /root/reference/pkg/src/dope/_core.pyx:28-260 (readable twin
 *     _core_py.py:25-288), with the same arc numbering (_core.pyx:293-297),
 *     the same tail-grouped adjacency in pair order (_core.pyx:298-310), the
 *     same FIFO active/orphan queues and the same tie-breaks, so labels AND
 *     the flow value are bit-identical to the reference on identical inputs.
 *     Labels: 1 iff the node ends in the sink tree (_core.pyx:257-259).
 *
 *  2. The consensus (ADMM) loop of admm.py:207-252 for a lattice stencil
 *     model on a NON-OVERLAPPING box partition (q == 1 everywhere), where the
 *     coupling operators of blockform.py:48-86 collapse to a one-pixel
 *     cross-block stencil:
 *       block_objective (blockform.py:89-105):
 *         linear_g = u_g + lam*(sum_{j~g, out} -w_gj y_j + r_g y_g)
 *                        + mu*((a_g - y_g) + 0.5),  r_g = sum_{j~g,out} w_gj
 *       solve_global (admm.py:136-151) + clamp (admm.py:172-180):
 *         acc_g = mu*(yh_g + a_g) - lam*(r_g*yh_g);  then per neighbouring
 *         block in id order acc_g -= lam*(sum_i -w_ig yh_i);  y = acc/mu
 *       block_residuals (admm.py:193-199), evaluate_energy (energy.py:187-194),
 *       update_multipliers (admm.py:183-190), best-iterate / stop rule
 *       (admm.py:242-252).
 *     Floating-point order follows SURVEY.md Appendix C where it matters.
 *
 * Block solves may run on several host threads (the reference's
 * ThreadPoolExecutor over blocks, admm.py:128-132); results do not depend on
 * the thread count.
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define BK_EPS 1e-12
#define TREE_FREE 0
#define TREE_SRC 1
#define TREE_SINK 2
#define PAR_NONE (-1LL)
#define PAR_TERMINAL (-2LL)
#define PAR_ORPHAN (-3LL)
#define DIST_INF (1LL << 62)

/* ------------------------------------------------------------------------ */
/* 1. BK max-flow                                                            */
/* ------------------------------------------------------------------------ */

typedef struct {
    int64_t cap_nodes, cap_arcs;
    int32_t *head, *adj, *queue, *orphans;
    double *rcap, *tcap;
    int64_t *off, *fill, *parent, *ts, *dist;
    int8_t *tree;
    uint8_t *active;
} bk_ws;

static void bk_ws_free(bk_ws *w) {
    free(w->head); free(w->adj); free(w->queue); free(w->orphans);
    free(w->rcap); free(w->tcap); free(w->off); free(w->fill);
    free(w->parent); free(w->ts); free(w->dist); free(w->tree); free(w->active);
    memset(w, 0, sizeof(*w));
}

static int bk_ws_reserve(bk_ws *w, int64_t m, int64_t narcs) {
    if (m <= w->cap_nodes && narcs <= w->cap_arcs) return 0;
    bk_ws_free(w);
    int64_t a = narcs > 0 ? narcs : 1;
    w->cap_nodes = m; w->cap_arcs = narcs;
    w->head = malloc(sizeof(int32_t) * a);
    w->adj = malloc(sizeof(int32_t) * a);
    w->rcap = malloc(sizeof(double) * a);
    w->queue = malloc(sizeof(int32_t) * (m + 1));
    w->orphans = malloc(sizeof(int32_t) * (m + 1));
    w->tcap = malloc(sizeof(double) * m);
    w->off = malloc(sizeof(int64_t) * (m + 1));
    w->fill = malloc(sizeof(int64_t) * (m + 1));
    w->parent = malloc(sizeof(int64_t) * m);
    w->ts = malloc(sizeof(int64_t) * m);
    w->dist = malloc(sizeof(int64_t) * m);
    w->tree = malloc(m);
    w->active = malloc(m);
    if (!w->head || !w->adj || !w->rcap || !w->queue || !w->orphans || !w->tcap ||
        !w->off || !w->fill || !w->parent || !w->ts || !w->dist || !w->tree || !w->active)
        return -1;
    return 0;
}

/* Follows _core.pyx:28-260 step for step. */
static double bk_core(bk_ws *w, int32_t m, uint8_t *labels) {
    double *tcap = w->tcap, *rcap = w->rcap;
    int32_t *head = w->head, *adj = w->adj, *queue = w->queue, *orphans = w->orphans;
    int64_t *off = w->off, *parent = w->parent, *ts = w->ts, *dist = w->dist;
    int8_t *tree = w->tree;
    uint8_t *active = w->active;
    const int32_t qcap = m + 1;
    int32_t qhead = 0, qtail = 0, ohead = 0, otail = 0;
    int64_t tick = 0;
    int32_t cur = -1;
    double flow = 0.0;

    for (int32_t i = 0; i < m; i++) {
        tree[i] = TREE_FREE; parent[i] = PAR_NONE; ts[i] = 0; dist[i] = 0; active[i] = 0;
    }
#define BK_ACTIVATE(x)                         \
    do {                                       \
        if (!active[x]) {                      \
            active[x] = 1;                     \
            queue[qtail] = (x);                \
            qtail = (qtail + 1) % qcap;        \
        }                                      \
    } while (0)
#define BK_ORPHAN(x)                           \
    do {                                       \
        parent[x] = PAR_ORPHAN;                \
        orphans[otail] = (x);                  \
        otail = (otail + 1) % qcap;            \
    } while (0)

    for (int32_t i = 0; i < m; i++) {
        if (tcap[i] > BK_EPS) {
            tree[i] = TREE_SRC; parent[i] = PAR_TERMINAL; dist[i] = 1; BK_ACTIVATE(i);
        } else if (tcap[i] < -BK_EPS) {
            tree[i] = TREE_SINK; parent[i] = PAR_TERMINAL; dist[i] = 1; BK_ACTIVATE(i);
        }
    }

    for (;;) {
        if (cur >= 0 && parent[cur] == PAR_NONE) cur = -1;
        if (cur < 0) {
            while (qhead != qtail) {
                int32_t i = queue[qhead];
                qhead = (qhead + 1) % qcap;
                active[i] = 0;
                if (parent[i] != PAR_NONE) { cur = i; break; }
            }
            if (cur < 0) break;
        }
        int32_t i = cur;
        int64_t mid = -1;
        if (tree[i] == TREE_SRC) {
            for (int64_t ai = off[i]; ai < off[i + 1]; ai++) {
                int32_t a = adj[ai];
                if (rcap[a] > BK_EPS) {
                    int32_t j = head[a];
                    if (parent[j] == PAR_NONE) {
                        tree[j] = TREE_SRC; parent[j] = a ^ 1; ts[j] = ts[i]; dist[j] = dist[i] + 1;
                        BK_ACTIVATE(j);
                    } else if (tree[j] == TREE_SINK) {
                        mid = a; break;
                    } else if (ts[j] <= ts[i] && dist[j] > dist[i]) {
                        parent[j] = a ^ 1; ts[j] = ts[i]; dist[j] = dist[i] + 1;
                    }
                }
            }
        } else {
            for (int64_t ai = off[i]; ai < off[i + 1]; ai++) {
                int32_t a = adj[ai];
                if (rcap[a ^ 1] > BK_EPS) {
                    int32_t j = head[a];
                    if (parent[j] == PAR_NONE) {
                        tree[j] = TREE_SINK; parent[j] = a ^ 1; ts[j] = ts[i]; dist[j] = dist[i] + 1;
                        BK_ACTIVATE(j);
                    } else if (tree[j] == TREE_SRC) {
                        mid = a ^ 1; break;
                    } else if (ts[j] <= ts[i] && dist[j] > dist[i]) {
                        parent[j] = a ^ 1; ts[j] = ts[i]; dist[j] = dist[i] + 1;
                    }
                }
            }
        }
        tick += 1;
        if (mid < 0) { cur = -1; continue; }

        /* bottleneck along source path, middle arc, sink path (_core.pyx:129-147) */
        double b = rcap[mid];
        int32_t x = head[mid ^ 1];
        while (parent[x] != PAR_TERMINAL) {
            int64_t pa = parent[x];
            if (rcap[pa ^ 1] < b) b = rcap[pa ^ 1];
            x = head[pa];
        }
        if (tcap[x] < b) b = tcap[x];
        x = head[mid];
        while (parent[x] != PAR_TERMINAL) {
            int64_t pa = parent[x];
            if (rcap[pa] < b) b = rcap[pa];
            x = head[pa];
        }
        if (-tcap[x] < b) b = -tcap[x];

        /* push and orphan saturated tree arcs (_core.pyx:149-181) */
        rcap[mid] -= b;
        rcap[mid ^ 1] += b;
        x = head[mid ^ 1];
        while (parent[x] != PAR_TERMINAL) {
            int64_t pa = parent[x];
            rcap[pa] += b;
            rcap[pa ^ 1] -= b;
            if (rcap[pa ^ 1] <= BK_EPS) BK_ORPHAN(x);
            x = head[pa];
        }
        tcap[x] -= b;
        if (tcap[x] <= BK_EPS) BK_ORPHAN(x);
        x = head[mid];
        while (parent[x] != PAR_TERMINAL) {
            int64_t pa = parent[x];
            rcap[pa] -= b;
            rcap[pa ^ 1] += b;
            if (rcap[pa] <= BK_EPS) BK_ORPHAN(x);
            x = head[pa];
        }
        tcap[x] += b;
        if (tcap[x] >= -BK_EPS) BK_ORPHAN(x);
        flow += b;

        /* adopt orphans, FIFO (_core.pyx:183-254) */
        while (ohead != otail) {
            int32_t o = orphans[ohead];
            ohead = (ohead + 1) % qcap;
            int8_t t = tree[o];
            int64_t min_d = DIST_INF;
            int64_t best = -1;
            for (int64_t ai = off[o]; ai < off[o + 1]; ai++) {
                int32_t a = adj[ai];
                double ra = (t == TREE_SRC) ? rcap[a ^ 1] : rcap[a];
                if (!(ra > BK_EPS)) continue;
                int32_t j = head[a];
                if (tree[j] != t || parent[j] == PAR_NONE) continue;
                int64_t d = 0;
                int32_t jj = j;
                for (;;) {
                    if (ts[jj] == tick) { d += dist[jj]; break; }
                    int64_t pa = parent[jj];
                    d += 1;
                    if (pa == PAR_TERMINAL) { ts[jj] = tick; dist[jj] = 1; break; }
                    if (pa == PAR_ORPHAN || pa == PAR_NONE) { d = DIST_INF; break; }
                    jj = head[pa];
                }
                if (d < DIST_INF) {
                    if (d < min_d) { min_d = d; best = a; }
                    jj = j;
                    int64_t dd = d;
                    while (ts[jj] != tick) {
                        ts[jj] = tick; dist[jj] = dd; dd -= 1; jj = head[parent[jj]];
                    }
                }
            }
            if (best >= 0) {
                parent[o] = best; ts[o] = tick; dist[o] = min_d + 1;
            } else {
                for (int64_t ai = off[o]; ai < off[o + 1]; ai++) {
                    int32_t a = adj[ai];
                    int32_t j = head[a];
                    if (tree[j] != t || parent[j] == PAR_NONE) continue;
                    double ra = (t == TREE_SRC) ? rcap[a ^ 1] : rcap[a];
                    if (ra > BK_EPS) BK_ACTIVATE(j);
                    int64_t pa = parent[j];
                    if (pa >= 0 && head[pa] == o) BK_ORPHAN(j);
                }
                tree[o] = TREE_FREE;
                parent[o] = PAR_NONE;
            }
        }
    }
#undef BK_ACTIVATE
#undef BK_ORPHAN
    for (int32_t i = 0; i < m; i++) labels[i] = (tree[i] == TREE_SINK) ? 1 : 0;
    return flow;
}

/* Arc/adjacency build of _core.pyx:282-310, then the core. */
static int bk_solve(bk_ws *w, int32_t m, const double *tcap, int64_t npairs,
                    const int32_t *pi, const int32_t *pj, const double *cij,
                    const double *cji, uint8_t *labels, double *flow) {
    if (m < 0 || npairs < 0) return -1;
    if (m == 0) { *flow = 0.0; return 0; }
    int64_t narcs = 2 * npairs;
    if (bk_ws_reserve(w, m, narcs)) return -2;
    memcpy(w->tcap, tcap, sizeof(double) * m);
    for (int64_t p = 0; p < npairs; p++) {
        if (pi[p] < 0 || pi[p] >= m || pj[p] < 0 || pj[p] >= m) return -1;
        w->head[2 * p] = pj[p];
        w->head[2 * p + 1] = pi[p];
        w->rcap[2 * p] = cij[p];
        w->rcap[2 * p + 1] = cji[p];
    }
    memset(w->off, 0, sizeof(int64_t) * (m + 1));
    for (int64_t p = 0; p < npairs; p++) { w->off[pi[p] + 1] += 1; w->off[pj[p] + 1] += 1; }
    for (int32_t i = 0; i < m; i++) w->off[i + 1] += w->off[i];
    memcpy(w->fill, w->off, sizeof(int64_t) * m);
    for (int64_t p = 0; p < npairs; p++) {
        w->adj[w->fill[pi[p]]++] = (int32_t)(2 * p);
        w->adj[w->fill[pj[p]]++] = (int32_t)(2 * p + 1);
    }
    memset(labels, 0, m);
    *flow = bk_core(w, m, labels);
    return 0;
}

/* Public: _core.bk_maxflow contract (_core.pyx:263-333; _core_py.py:25-35).
 * Inputs are not modified.  Returns 0 on success. */
int oracle_bk_maxflow(int32_t m, const double *tcap, int64_t npairs,
                      const int32_t *pi, const int32_t *pj, const double *cij,
                      const double *cji, uint8_t *labels, double *flow) {
    bk_ws w;
    memset(&w, 0, sizeof(w));
    int rc = bk_solve(&w, m, tcap, npairs, pi, pj, cij, cji, labels, flow);
    bk_ws_free(&w);
    return rc;
}

/* ------------------------------------------------------------------------ */
/* 2. Lattice model + non-overlapping box partition                           */
/* ------------------------------------------------------------------------ */

#define MAX_DIRS 13

typedef struct {
    int32_t ndim;               /* 2 or 3 */
    int64_t dims[3];            /* row-major axes, e.g. (H, W) or (D, H, W) */
    int64_t kpa[3];             /* blocks per axis (make_partition k_per_axis) */
    int32_t ndirs;              /* forward stencil offsets, i<j canonical */
    int32_t off[MAX_DIRS][3];   /* per-axis offset of each direction */
    const double *w[MAX_DIRS];  /* per-direction weight plane (indexed by the
                                   lower pixel i of the pair), or NULL */
    double wconst[MAX_DIRS];    /* used when w[d] == NULL */
    const double *u;            /* unary, n */
    double lam;
} oracle_lattice;

typedef struct {
    const oracle_lattice *L;
    int64_t n, K;
    int64_t strides[3];
    int64_t *lo[3], *hi[3];     /* per-axis block ranges (partition.py:62-77, overlap 0) */
    int64_t *blk_of_axis[3];    /* per-axis coordinate -> range index */
} lattice_ctx;

static void axis_ranges(int64_t dim, int64_t k, int64_t *lo, int64_t *hi, int64_t *owner) {
    int64_t base = dim / k, rem = dim % k, x = 0;
    for (int64_t r = 0; r < k; r++) {
        int64_t len = base + (r < rem ? 1 : 0);
        lo[r] = x; hi[r] = x + len;
        for (int64_t c = x; c < x + len; c++) owner[c] = r;
        x += len;
    }
}

static int ctx_init(lattice_ctx *c, const oracle_lattice *L) {
    memset(c, 0, sizeof(*c));
    c->L = L;
    c->n = 1; c->K = 1;
    for (int a = 0; a < L->ndim; a++) {
        if (L->kpa[a] < 1 || L->kpa[a] > L->dims[a]) return -1;
        c->n *= L->dims[a]; c->K *= L->kpa[a];
    }
    c->strides[L->ndim - 1] = 1;
    for (int a = L->ndim - 2; a >= 0; a--) c->strides[a] = c->strides[a + 1] * L->dims[a + 1];
    for (int a = 0; a < L->ndim; a++) {
        c->lo[a] = malloc(sizeof(int64_t) * L->kpa[a]);
        c->hi[a] = malloc(sizeof(int64_t) * L->kpa[a]);
        c->blk_of_axis[a] = malloc(sizeof(int64_t) * L->dims[a]);
        axis_ranges(L->dims[a], L->kpa[a], c->lo[a], c->hi[a], c->blk_of_axis[a]);
    }
    return 0;
}

static void ctx_free(lattice_ctx *c) {
    for (int a = 0; a < 3; a++) { free(c->lo[a]); free(c->hi[a]); free(c->blk_of_axis[a]); }
}

static inline void coords_of(const lattice_ctx *c, int64_t g, int64_t *x) {
    for (int a = 0; a < c->L->ndim; a++) { x[a] = g / c->strides[a]; g %= c->strides[a]; }
}

static inline int64_t block_of(const lattice_ctx *c, const int64_t *x) {
    int64_t b = 0;
    for (int a = 0; a < c->L->ndim; a++) b = b * c->L->kpa[a] + c->blk_of_axis[a][x[a]];
    return b;
}

/* Neighbour of pixel g (coords x) through direction d with sign s (+1: the
 * forward partner j = g + off, -1: the backward partner).  Returns -1 when
 * outside the grid.  *wout receives the pair weight. */
static inline int64_t neighbour(const lattice_ctx *c, int64_t g, const int64_t *x, int d,
                                int s, double *wout) {
    const oracle_lattice *L = c->L;
    int64_t lin = 0;
    for (int a = 0; a < L->ndim; a++) {
        int64_t y = x[a] + s * L->off[d][a];
        if (y < 0 || y >= L->dims[a]) return -1;
        lin += y * c->strides[a];
    }
    int64_t low = s > 0 ? g : lin;
    *wout = L->w[d] ? L->w[d][low] : L->wconst[d];
    return lin;
}

static inline int inside_ext(const lattice_ctx *c, int64_t j, const int64_t *ext) {
    int64_t xj[3];
    coords_of(c, j, xj);
    for (int a = 0; a < c->L->ndim; a++)
        if (xj[a] < ext[2 * a] || xj[a] >= ext[2 * a + 1]) return 0;
    return 1;
}

/* r_diag = d/q^2 - dhat with q == 1 (blockform.py:58, 75): d is the row
 * sum of the symmetric weight matrix built from (rows,cols)+(cols,rows)
 * (energy.py:71-76), i.e. forward partners in direction order then backward
 * partners in direction order; dhat accumulates the in-block pairs with
 * np.add.at, first where g is the lower index, then where it is the higher
 * one (energy.py:64-69), each ascending. */
static double r_diag(const lattice_ctx *c, int64_t g, const int64_t *x, const int64_t *ext) {
    const oracle_lattice *L = c->L;
    double dsum = 0.0;
    int64_t fi[MAX_DIRS], bi[MAX_DIRS];
    double fw[MAX_DIRS], bw[MAX_DIRS];
    int nf = 0, nb = 0;
    for (int s = 1; s >= -1; s -= 2)
        for (int d = 0; d < L->ndirs; d++) {
            double wv;
            int64_t j = neighbour(c, g, x, d, s, &wv);
            if (j < 0) continue;
            dsum += wv;
            if (inside_ext(c, j, ext) && wv != 0.0) {
                if (s > 0) { fi[nf] = j; fw[nf] = wv; nf++; }
                else { bi[nb] = j; bw[nb] = wv; nb++; }
            }
        }
    for (int p = 1; p < nf; p++) {
        int64_t ki = fi[p]; double kw = fw[p]; int q = p - 1;
        while (q >= 0 && fi[q] > ki) { fi[q + 1] = fi[q]; fw[q + 1] = fw[q]; q--; }
        fi[q + 1] = ki; fw[q + 1] = kw;
    }
    for (int p = 1; p < nb; p++) {
        int64_t ki = bi[p]; double kw = bw[p]; int q = p - 1;
        while (q >= 0 && bi[q] > ki) { bi[q + 1] = bi[q]; bw[q + 1] = bw[q]; q--; }
        bi[q + 1] = ki; bw[q + 1] = kw;
    }
    double dhat = 0.0;
    for (int p = 0; p < nf; p++) dhat += fw[p];
    for (int p = 0; p < nb; p++) dhat += bw[p];
    return dsum - dhat;
}

/* Block k's pixel list in row-major box order (partition.py:52-59). */
static int64_t block_pixels(const lattice_ctx *c, int64_t k, int64_t *pix, int64_t *ext) {
    const oracle_lattice *L = c->L;
    int64_t bi[3] = {0, 0, 0}, kk = k;
    for (int a = L->ndim - 1; a >= 0; a--) { bi[a] = kk % L->kpa[a]; kk /= L->kpa[a]; }
    int64_t lo[3] = {0, 0, 0}, len[3] = {1, 1, 1};
    int64_t m = 1;
    for (int a = 0; a < L->ndim; a++) {
        lo[a] = c->lo[a][bi[a]]; len[a] = c->hi[a][bi[a]] - lo[a]; m *= len[a];
        if (ext) { ext[2 * a] = lo[a]; ext[2 * a + 1] = lo[a] + len[a]; }
    }
    if (pix) {
        int64_t idx = 0;
        if (L->ndim == 2) {
            for (int64_t r = 0; r < len[0]; r++)
                for (int64_t q = 0; q < len[1]; q++)
                    pix[idx++] = (lo[0] + r) * c->strides[0] + lo[1] + q;
        } else {
            for (int64_t z = 0; z < len[0]; z++)
                for (int64_t r = 0; r < len[1]; r++)
                    for (int64_t q = 0; q < len[2]; q++)
                        pix[idx++] = (lo[0] + z) * c->strides[0] + (lo[1] + r) * c->strides[1] + lo[2] + q;
        }
    }
    return m;
}

/* --------------------------- block solves -------------------------------- */

typedef struct {
    const lattice_ctx *c;
    const double *y, *a;
    double mu;
    uint8_t *yhat;
    int64_t next_block;
    pthread_mutex_t lock;
    int error;            /* 0 or 1+block id of the first failure */
} blocks_job;

typedef struct {
    int64_t *pix, *local;    /* pixel list; global->local map is done by search */
    double *lin, *cij, *cji;
    int32_t *pi, *pj;
    uint8_t *lab;
    int64_t cap_m, cap_p;
    bk_ws ws;
} block_scratch;

static int scratch_reserve(block_scratch *s, int64_t m, int64_t p) {
    if (m > s->cap_m) {
        free(s->pix); free(s->lin); free(s->lab);
        s->pix = malloc(sizeof(int64_t) * m);
        s->lin = malloc(sizeof(double) * m);
        s->lab = malloc(m);
        s->cap_m = m;
    }
    if (p > s->cap_p) {
        free(s->pi); free(s->pj); free(s->cij); free(s->cji);
        s->pi = malloc(sizeof(int32_t) * (p ? p : 1));
        s->pj = malloc(sizeof(int32_t) * (p ? p : 1));
        s->cij = malloc(sizeof(double) * (p ? p : 1));
        s->cji = malloc(sizeof(double) * (p ? p : 1));
        s->cap_p = p;
    }
    return (s->pix && s->lin && s->lab && s->pi && s->pj && s->cij && s->cji) ? 0 : -1;
}

static void scratch_free(block_scratch *s) {
    free(s->pix); free(s->lin); free(s->lab); free(s->pi); free(s->pj); free(s->cij); free(s->cji);
    bk_ws_free(&s->ws);
}

/* Solve one block: block_objective (blockform.py:89-105) + solve_binary
 * (maxflow.py:73-113).  Pairs are listed in CSR order of the block-local
 * weight matrix (row ascending, then column ascending), as the reference's
 * w_scaled[p][:, p].tocoo() row<col selection yields (blockform.py:64-67). */
static int solve_one_block(const lattice_ctx *c, int64_t k, const double *y, const double *a,
                           double mu, uint8_t *yhat, block_scratch *s) {
    const oracle_lattice *L = c->L;
    int64_t ext[6];
    int64_t m = block_pixels(c, k, NULL, ext);
    if (scratch_reserve(s, m, m * L->ndirs)) return -1;
    block_pixels(c, k, s->pix, ext);
    int64_t len[3] = {1, 1, 1}, lstr[3] = {0, 0, 0};
    for (int a2 = 0; a2 < L->ndim; a2++) len[a2] = ext[2 * a2 + 1] - ext[2 * a2];
    lstr[L->ndim - 1] = 1;
    for (int a2 = L->ndim - 2; a2 >= 0; a2--) lstr[a2] = lstr[a2 + 1] * len[a2 + 1];

    int64_t np = 0;
    for (int64_t i = 0; i < m; i++) {
        int64_t g = s->pix[i], x[3];
        coords_of(c, g, x);
        /* linear term */
        double cy = 0.0, r = 0.0;
        /* c_rows @ y: CSR row sum over global columns ascending (blockform.py:103).
         * Cross-block neighbours: backward partners have lower index than
         * forward ones; within each group directions are visited so that
         * indices ascend. */
        int64_t nb_idx[2 * MAX_DIRS];
        double nb_w[2 * MAX_DIRS];
        int nn = 0;
        for (int s2 = -1; s2 <= 1; s2 += 2) {
            for (int d = 0; d < L->ndirs; d++) {
                double wv;
                int64_t j = neighbour(c, g, x, d, s2, &wv);
                if (j < 0) continue;
                int64_t xj[3];
                coords_of(c, j, xj);
                int inside = 1;
                for (int a2 = 0; a2 < L->ndim; a2++)
                    if (xj[a2] < ext[2 * a2] || xj[a2] >= ext[2 * a2 + 1]) inside = 0;
                if (inside) continue;
                nb_idx[nn] = j; nb_w[nn] = wv; nn++;
            }
        }
        /* sort cross neighbours by global index (insertion sort, nn <= 26) */
        for (int p2 = 1; p2 < nn; p2++) {
            int64_t ki = nb_idx[p2]; double kw = nb_w[p2]; int q = p2 - 1;
            while (q >= 0 && nb_idx[q] > ki) { nb_idx[q + 1] = nb_idx[q]; nb_w[q + 1] = nb_w[q]; q--; }
            nb_idx[q + 1] = ki; nb_w[q + 1] = kw;
        }
        for (int p2 = 0; p2 < nn; p2++) { cy += (-nb_w[p2]) * y[nb_idx[p2]]; }
        r = r_diag(c, g, x, ext);
        double sy = y[g];
        s->lin[i] = L->u[g] + L->lam * (cy + r * sy) + mu * ((a[g] - sy) + 0.5);
        /* in-block forward pairs, CSR order (i ascending; j ascending) */
        int64_t cand[MAX_DIRS];
        double cw[MAX_DIRS];
        int nc = 0;
        for (int d = 0; d < L->ndirs; d++) {
            int64_t lj = 0;
            int ok = 1;
            for (int a2 = 0; a2 < L->ndim; a2++) {
                int64_t li = (x[a2] - ext[2 * a2]) + L->off[d][a2];
                if (li < 0 || li >= len[a2]) { ok = 0; break; }
                lj += li * lstr[a2];
            }
            if (!ok) continue;
            cand[nc] = lj;
            cw[nc] = L->w[d] ? L->w[d][g] : L->wconst[d];
            nc++;
        }
        for (int p2 = 1; p2 < nc; p2++) {
            int64_t ki = cand[p2]; double kw = cw[p2]; int q = p2 - 1;
            while (q >= 0 && cand[q] > ki) { cand[q + 1] = cand[q]; cw[q + 1] = cw[q]; q--; }
            cand[q + 1] = ki; cw[q + 1] = kw;
        }
        for (int p2 = 0; p2 < nc; p2++) {
            if (cw[p2] == 0.0) continue;    /* structural zeros are not stored */
            if (cw[p2] < 0.0) return -3;     /* NonSubmodularError (maxflow.py:86-89) */
            s->pi[np] = (int32_t)i;
            s->pj[np] = (int32_t)cand[p2];
            s->cij[np] = L->lam * cw[p2];
            s->cji[np] = L->lam * cw[p2];
            np++;
        }
    }
    double flow;
    int rc = bk_solve(&s->ws, (int32_t)m, s->lin, np, s->pi, s->pj, s->cij, s->cji, s->lab, &flow);
    if (rc) return rc;
    for (int64_t i = 0; i < m; i++) yhat[s->pix[i]] = s->lab[i];
    return 0;
}

static void *blocks_worker(void *arg) {
    blocks_job *job = (blocks_job *)arg;
    block_scratch s;
    memset(&s, 0, sizeof(s));
    for (;;) {
        pthread_mutex_lock(&job->lock);
        int64_t k = job->next_block++;
        int stop = job->error != 0;
        pthread_mutex_unlock(&job->lock);
        if (stop || k >= job->c->K) break;
        int rc = solve_one_block(job->c, k, job->y, job->a, job->mu, job->yhat, &s);
        if (rc) {
            pthread_mutex_lock(&job->lock);
            if (!job->error || (int64_t)job->error > k + 1) job->error = (int)(k + 1);
            pthread_mutex_unlock(&job->lock);
        }
    }
    scratch_free(&s);
    return NULL;
}

static int update_blocks(const lattice_ctx *c, const double *y, const double *a, double mu,
                         uint8_t *yhat, int threads) {
    blocks_job job;
    memset(&job, 0, sizeof(job));
    job.c = c; job.y = y; job.a = a; job.mu = mu; job.yhat = yhat;
    pthread_mutex_init(&job.lock, NULL);
    if (threads < 1) threads = 1;
    if (threads > 256) threads = 256;
    if (threads == 1) {
        blocks_worker(&job);
    } else {
        pthread_t th[256];
        for (int t = 0; t < threads; t++) pthread_create(&th[t], NULL, blocks_worker, &job);
        for (int t = 0; t < threads; t++) pthread_join(th[t], NULL);
    }
    pthread_mutex_destroy(&job.lock);
    return job.error;   /* 0, or 1 + first failing block id */
}

/* --------------------------- global update -------------------------------- */

/* solve_global (admm.py:136-151) + clamp (admm.py:172-180), q == 1. */
static int update_global(const lattice_ctx *c, const uint8_t *yhat, const double *a, double mu,
                         double *y, int *clamped) {
    const oracle_lattice *L = c->L;
    if (!(mu > 0)) return -1;
    int cl = 0;
    for (int64_t g = 0; g < c->n; g++) {
        int64_t x[3];
        coords_of(c, g, x);
        int64_t bg = block_of(c, x);
        /* cross neighbours grouped per owning block; blocks visited in id
         * order, within a block contributions in block-local (= global for
         * row-major boxes) ascending order */
        int64_t nb_idx[2 * MAX_DIRS], nb_blk[2 * MAX_DIRS];
        double nb_w[2 * MAX_DIRS];
        int nn = 0;
        double r = 0.0;
        for (int s2 = -1; s2 <= 1; s2 += 2)
            for (int d = 0; d < L->ndirs; d++) {
                double wv;
                int64_t j = neighbour(c, g, x, d, s2, &wv);
                if (j < 0) continue;
                int64_t xj[3];
                coords_of(c, j, xj);
                int64_t bj = block_of(c, xj);
                if (bj == bg) continue;
                nb_idx[nn] = j; nb_blk[nn] = bj; nb_w[nn] = wv; nn++;
            }
        for (int p2 = 1; p2 < nn; p2++) {
            int64_t ki = nb_idx[p2], kb = nb_blk[p2]; double kw = nb_w[p2]; int q = p2 - 1;
            while (q >= 0 && (nb_blk[q] > kb || (nb_blk[q] == kb && nb_idx[q] > ki))) {
                nb_idx[q + 1] = nb_idx[q]; nb_blk[q + 1] = nb_blk[q]; nb_w[q + 1] = nb_w[q]; q--;
            }
            nb_idx[q + 1] = ki; nb_blk[q + 1] = kb; nb_w[q + 1] = kw;
        }
        {
            int64_t gext[6];
            int64_t bi[3] = {0, 0, 0};
            for (int a2 = 0; a2 < L->ndim; a2++) {
                bi[a2] = c->blk_of_axis[a2][x[a2]];
                gext[2 * a2] = c->lo[a2][bi[a2]];
                gext[2 * a2 + 1] = c->hi[a2][bi[a2]];
            }
            r = r_diag(c, g, x, gext);
        }
        double yh = (double)yhat[g];
        double acc = 0.0;
        int own_done = 0;
        int p2 = 0;
        while (p2 < nn || !own_done) {
            if (!own_done && (p2 >= nn || nb_blk[p2] > bg)) {
                acc += mu * (yh + a[g]) - L->lam * (r * yh);
                own_done = 1;
                continue;
            }
            int64_t kb = nb_blk[p2];
            double s = 0.0;
            while (p2 < nn && nb_blk[p2] == kb) { s += (-nb_w[p2]) * (double)yhat[nb_idx[p2]]; p2++; }
            acc -= L->lam * s;
        }
        double v = acc / (mu * 1.0);
        if (v < 0.0 || v > 1.0) cl = 1;
        y[g] = v < 0.0 ? 0.0 : (v > 1.0 ? 1.0 : v);
    }
    *clamped = cl;
    return 0;
}

static void block_residuals(const lattice_ctx *c, const uint8_t *yhat, const double *y,
                            double *res, double *ss_scratch) {
    for (int64_t k = 0; k < c->K; k++) ss_scratch[k] = 0.0;
    /* per block, pixels in block order */
    int64_t *pix = malloc(sizeof(int64_t) * 1);
    int64_t cap = 1;
    for (int64_t k = 0; k < c->K; k++) {
        int64_t m = block_pixels(c, k, NULL, NULL);
        if (m > cap) { free(pix); pix = malloc(sizeof(int64_t) * m); cap = m; }
        block_pixels(c, k, pix, NULL);
        double s = 0.0;
        for (int64_t i = 0; i < m; i++) {
            double d = (double)yhat[pix[i]] - y[pix[i]];
            s += d * d;
        }
        res[k] = sqrt(s);
    }
    free(pix);
}

/* evaluate_energy (energy.py:187-194): u.y + lam * sum_pairs w (y_i - y_j)^2,
 * pairs enumerated direction by direction, each in row-major order of i. */
static double energy(const lattice_ctx *c, const double *y) {
    const oracle_lattice *L = c->L;
    double quad = 0.0, lin = 0.0;
    for (int d = 0; d < L->ndirs; d++) {
        for (int64_t g = 0; g < c->n; g++) {
            int64_t x[3];
            coords_of(c, g, x);
            double wv;
            int64_t j = neighbour(c, g, x, d, +1, &wv);
            if (j < 0) continue;
            double df = y[g] - y[j];
            quad += wv * (df * df);
        }
    }
    for (int64_t g = 0; g < c->n; g++) lin += L->u[g] * y[g];
    return lin + L->lam * quad;
}

/* ------------------------------------------------------------------------ */
/* Public step API (mirrors admm.py's step functions)                         */
/* ------------------------------------------------------------------------ */

int oracle_num_blocks(const oracle_lattice *L, int64_t *K) {
    lattice_ctx c;
    if (ctx_init(&c, L)) { ctx_free(&c); return -1; }
    *K = c.K;
    ctx_free(&c);
    return 0;
}

int oracle_update_blocks(const oracle_lattice *L, const double *y, const double *a, double mu,
                         uint8_t *yhat, int threads) {
    lattice_ctx c;
    if (ctx_init(&c, L)) { ctx_free(&c); return -1; }
    int rc = update_blocks(&c, y, a, mu, yhat, threads);
    ctx_free(&c);
    return rc;
}

int oracle_update_global(const oracle_lattice *L, const uint8_t *yhat, const double *a, double mu,
                         double *y, int *clamped) {
    lattice_ctx c;
    if (ctx_init(&c, L)) { ctx_free(&c); return -1; }
    int rc = update_global(&c, yhat, a, mu, y, clamped);
    ctx_free(&c);
    return rc;
}

int oracle_block_residuals(const oracle_lattice *L, const uint8_t *yhat, const double *y,
                           double *res) {
    lattice_ctx c;
    if (ctx_init(&c, L)) { ctx_free(&c); return -1; }
    double *tmp = malloc(sizeof(double) * c.K);
    block_residuals(&c, yhat, y, res, tmp);
    free(tmp);
    ctx_free(&c);
    return 0;
}

double oracle_energy(const oracle_lattice *L, const double *y) {
    lattice_ctx c;
    if (ctx_init(&c, L)) { ctx_free(&c); return NAN; }
    double e = energy(&c, y);
    ctx_free(&c);
    return e;
}

typedef struct {
    int32_t iterations, converged, best_iteration;
    double mu_final;
} oracle_run_info;

/* Per-iteration state digest (test fixtures only; no reference counterpart).
 * H_k = sum over pixels g of v_k(g) * mix64(3 g + k) mod 2^64 for
 * v_0 = yhat, v_1 = 2 y (an integer on the q == 1 integer configs), v_2 = a
 * (integer there): an order-independent position-weighted sum, so a GPU
 * reduction in any order -- or per-shard partial sums with a global index
 * base -- gives the same three words.  mix64 = the splitmix64 finaliser. */
static inline uint64_t mix64(uint64_t x) {
    x += 0x9E3779B97F4A7C15ull;
    x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
    x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
    return x ^ (x >> 31);
}

static void state_digest(int64_t n, const uint8_t *yhat, const double *y, const double *a,
                         uint64_t *out3) {
    uint64_t h0 = 0, h1 = 0, h2 = 0;
    for (int64_t g = 0; g < n; g++) {
        const uint64_t b = 3 * (uint64_t)g;
        h0 += (uint64_t)yhat[g] * mix64(b);
        h1 += (uint64_t)(int64_t)llround(2.0 * y[g]) * mix64(b + 1);
        h2 += (uint64_t)(int64_t)llround(a[g]) * mix64(b + 2);
    }
    out3[0] = h0; out3[1] = h1; out3[2] = h2;
}

int oracle_state_digest(int64_t n, const uint8_t *yhat, const double *y, const double *a,
                        uint64_t *out3) {
    state_digest(n, yhat, y, a, out3);
    return 0;
}

/* run (admm.py:207-252) with the trace of admm.py:233-241.
 * trace_* arrays have max_iters entries; yhat_hist (optional) max_iters*n;
 * digests (optional) 3*max_iters words of state_digest per iteration.
 * y (in: ignored, out: state.y after run, i.e. best iterate when not
 * converged), a (out: final multipliers, global layout), yhat (out: final
 * block labels, global layout), labels (out: binarize(state.y)). */
int oracle_run(const oracle_lattice *L, double mu0, double mu_fact, double eps, int32_t max_iters,
               int threads, double *y, double *a, uint8_t *yhat, int8_t *labels,
               double *tr_mu, double *tr_energy, double *tr_ressq, double *tr_maxres,
               int32_t *tr_clamped, uint8_t *yhat_hist, uint64_t *digests, oracle_run_info *info) {
    lattice_ctx c;
    if (ctx_init(&c, L)) { ctx_free(&c); return -1; }
    int64_t n = c.n, K = c.K;
    double *best_y = malloc(sizeof(double) * n);
    double *res = malloc(sizeof(double) * K);
    double *tmp = malloc(sizeof(double) * K);
    for (int64_t g = 0; g < n; g++) { y[g] = 0.5; a[g] = 0.0; yhat[g] = 0; best_y[g] = 0.5; }
    double mu = mu0, best_e = INFINITY;
    int rc = 0;
    info->converged = 0; info->best_iteration = 0; info->iterations = 0;
    for (int32_t it = 1; it <= max_iters; it++) {
        info->iterations = it;
        double mu_at_solve = mu;
        rc = update_blocks(&c, y, a, mu, yhat, threads);
        if (rc) { rc = rc > 0 ? rc : -2; break; }
        int clamped = 0;
        if (update_global(&c, yhat, a, mu, y, &clamped)) { rc = -1; break; }
        block_residuals(&c, yhat, y, res, tmp);
        double e = energy(&c, y);
        double ressq = 0.0, maxres = 0.0;
        for (int64_t k = 0; k < K; k++) { ressq += res[k] * res[k]; if (k == 0 || res[k] > maxres) maxres = res[k]; }
        tr_mu[it - 1] = mu_at_solve; tr_energy[it - 1] = e; tr_ressq[it - 1] = ressq;
        tr_maxres[it - 1] = maxres; tr_clamped[it - 1] = clamped;
        if (yhat_hist) memcpy(yhat_hist + (int64_t)(it - 1) * n, yhat, n);
        if (e < best_e) { best_e = e; memcpy(best_y, y, sizeof(double) * n); info->best_iteration = it; }
        for (int64_t g = 0; g < n; g++) a[g] = a[g] + ((double)yhat[g] - y[g]);
        mu *= mu_fact;
        /* digest of (yhat_t, y_t, a_t) after the multiplier update -- what the
         * device state holds at the end of iteration t */
        if (digests) state_digest(n, yhat, y, a, digests + 3 * (int64_t)(it - 1));
        if (K == 0 || maxres <= eps) { info->converged = 1; break; }
    }
    if (!rc && !info->converged) memcpy(y, best_y, sizeof(double) * n);
    for (int64_t g = 0; g < n; g++) labels[g] = y[g] >= 0.5 ? 1 : 0;
    info->mu_final = mu;
    free(best_y); free(res); free(tmp);
    ctx_free(&c);
    return rc;
}
