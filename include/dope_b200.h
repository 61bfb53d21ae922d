/*
 * dope_b200.h -- C ABI of the B200-native DOPE hot path.
 *
 * Drop-in boundary for the reference's two seams:
 *
 *   Seam 1 (per graph) replaces the kernel-backend function
 *     bk_maxflow(tcap, pair_i, pair_j, cap_ij, cap_ji) -> (labels, flow)
 *     /root/reference/pkg/src/dope/_core.pyx:263-333 (contract
 *     _core_py.py:25-35; bound by name at maxflow.py:14 via _kernels.py:19-21)
 *     -> dope_bk_maxflow().
 *
 *   Seam 2 (batched, one CTA per sub-region) replaces the per-iteration step
 *   functions of admm.py:
 *     update_blocks      admm.py:113-133  (+ blockform.block_objective
 *                        blockform.py:89-105, maxflow.solve_binary
 *                        maxflow.py:111-113)            -> dope_update_blocks()
 *     update_global      admm.py:172-180  (solve_global admm.py:136-151)
 *     update_multipliers admm.py:183-190
 *     block_residuals    admm.py:193-199
 *     evaluate_energy    energy.py:187-194              -> dope_update_global()
 *     run bookkeeping    admm.py:225-252 (trace, best, stop) -> last CTA of
 *                                                          dope_update_global
 *     run                admm.py:207-252                -> dope_admm_run(),
 *                                                          dope_finish_run()
 *     binarize           admm.py:202-204                -> dope_binarize()
 *
 * Conventions
 *   - Plain pointers and sizes; no framework types.  Device pointers are
 *     caller-owned (the Python host allocates them with torch); the library
 *     allocates nothing persistent.  `stream` is a cudaStream_t passed as
 *     void*; every call is asynchronous on it.
 *   - Return codes: 0 ok; < 0 invalid arguments / unsupported geometry
 *     (see DOPE_E_*); > 0 never returned by launch calls -- solver failures
 *     are reported on the device in dope_run_state.error as 1 + block id
 *     (the reference's BlockSolveError(block_id), admm.py:27-32).
 *   - Integer lattice path: grid coordinates row-major (GridShape.strides,
 *     grid.py:46-52), block ids row-major over the block lattice
 *     (partition.py:103), non-overlapping near-equal box tiling
 *     (partition.py:62-77 with overlap 0).  All per-pixel arrays are global
 *     row-major so they compare elementwise with the reference's vectors.
 */
#ifndef DOPE_B200_H
#define DOPE_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define DOPE_ABI_VERSION 1

#define DOPE_OK 0
#define DOPE_E_ARGS (-1)        /* null pointer / bad size */
#define DOPE_E_GEOMETRY (-2)    /* no kernel variant for this block box */
#define DOPE_E_CAPACITY (-3)    /* capacities exceed the int8 residual range */
#define DOPE_E_CUDA (-4)        /* a CUDA launch failed (see dope_last_cuda_error) */
#define DOPE_E_NONSUBMODULAR (-5)

/* Device-resident run bookkeeping (one per run; caller allocates
 * sizeof(dope_run_state) bytes of device memory, 8-byte aligned). */
typedef struct dope_run_state {
    int64_t best_energy;        /* energy of the best iterate so far           */
    int32_t iteration;          /* iterations completed                        */
    int32_t best_iteration;     /* admm.py:242-245 (strict <)                  */
    int32_t converged;          /* admm.py:247-249                             */
    int32_t stop;               /* converged, error or finished: later
                                   iteration launches are no-ops               */
    int32_t ycur;               /* y buffer (0..2) holding the current iterate */
    int32_t ybest;              /* y buffer holding the best iterate           */
    int32_t parity;             /* which multiplier buffer is current          */
    int32_t error;              /* 0, 1 + first failing block id, or -1 when
                                   the multipliers would leave int16          */
    int32_t max_rounds_seen;    /* diagnostics: max global-relabel rounds      */
    int32_t done_ctas;          /* last-CTA-done counter of the consensus pass */
    int64_t solves;             /* diagnostics: block solves performed         */
    int64_t sweeps;             /* diagnostics: push/relabel sweeps            */
    int64_t energy_acc;         /* scratch of the end-of-run energy pass       */
    int64_t unary2;             /* sum u * y2 of the current iterate (kept
                                   incrementally: u is read only where y moved) */
    int32_t a_bound;            /* multiplier passes so far: an upper bound on
                                   |a| (int16 storage; the run loop stops with
                                   error -1 at 32000)                          */
    int32_t generation;         /* runs begun on this state (dope_admm_init): the
                                   peer-exchange epochs are generation-tagged */
} dope_run_state;

/* Length (int64 elements) of dope_lattice.part_cta. */
#define DOPE_PART_CTA_LEN 8

/* Integer lattice problem (C1, C3, C4, C5 of BASELINE.json).
 * Scaling: all quantities that are half-integers in the reference are held
 * doubled: y2 = 2*y (y = 1/2 at init, {0,1} afterwards), block terminal
 * capacity 2*linear, pair capacity 2*lambda*w.  Energies are exact integers.
 * Storage: y2 as uint8 (values 0, 1, 2), multipliers as int16 (|a| grows by
 * at most 1 per iteration; runs are limited to 32000 iterations), u int32. */
typedef struct dope_lattice {
    int32_t ndim;               /* 2 or 3                                     */
    int32_t conn;               /* 4 (2D) or 6 (3D)                           */
    int64_t dims[3];            /* row-major grid extents (unused axes = 1)   */
    int32_t kpa[3];             /* blocks per axis (make_partition)           */
    int32_t lamw;               /* lambda * w, integer, constant over pairs   */
    int32_t mu;                 /* ADMM penalty, integer; lamw % mu == 0      */
    double eps;                 /* stop when max block residual <= eps        */
    int32_t max_iters;          /* trace capacity                             */
    int32_t warm_start;         /* 1: reuse each block's residual graph       */
    int32_t skip_clean;         /* 1: re-solve only blocks whose linear term
                                   may have changed (exact)    */
    int32_t fuse_multipliers;   /* 1: dope_update_global also does
                                   update_multipliers (the run loop)          */
    /* caller-owned device buffers */
    const int32_t *u;           /* n   unary                                  */
    int16_t *a;                 /* n   multipliers, updated in place          */
    uint8_t *y2[3];             /* n   2*y; three rotating iterate buffers:
                                   current, best, and the next output         */
    uint8_t *yhat;              /* n   block labels (global layout)           */
    uint8_t *resid;             /* K * resid_stride bytes: residual graphs    */
    uint32_t *dirty;            /* 16K + 8: [0, K) block needs a re-solve
                                   (init 1); [K, 2K) iteration + 1 of the
                                   block's last solve; [2K, 5K) pass + 1 at
                                   which y buffer b last received block k's
                                   iterate, [5K, 6K) pass + 1 of the last
                                   change of block k's iterate, [6K, 7K) pass
                                   + 1 whose energy partial of block k is
                                   current (clean-block consensus passes);
                                   [7K, 8K) the blocks solved this iteration,
                                   [8K, 9K) 1 + block k's slot in that list,
                                   [9K, 11K + 2) the run loop's two dirty-block
                                   worklists [count, K entries], [11K + 2,
                                   12K + 2) iteration + 1 of the block's last
                                   finished solve (K1 / consensus overlap),
                                   [12K + 2, 16K + 8) the consensus pass's
                                   tile-work queue (4 words per entry, then
                                   length, claims, CTAs done): 16K + 8 in all */
    int64_t *part_energy;       /* K   per-block pair-energy partials          */
    int64_t *part_unary;        /* K   per-block change of sum u*y2           */
    int64_t *part_ressq;        /* K   per-block sum (yhat - y)^2             */
    int32_t *part_flags;        /* K   bit0: clamped                          */
    int64_t *part_cta;          /* DOPE_PART_CTA_LEN: pass-wide aggregates and
                                   the count of the iteration's solved-block
                                   list (2D); zeroed by
                                   dope_admm_init                              */
    dope_run_state *state;      /* 1                                          */
    int64_t *trace_energy;      /* max_iters                                  */
    double *trace_residual_sq;  /* max_iters                                  */
    double *trace_max_residual; /* max_iters                                  */
    int32_t *trace_clamped;     /* max_iters                                  */
    int64_t *timeline;          /* optional (may be NULL): 8 int64 per block of
                                   the last K1 launch (2D): globaltimer stamps,
                                   rounds, sweeps (diagnostics only)          */
    uint8_t *scratch;           /* 3D only: K * dope_scratch_stride bytes of
                                   per-sub-region node state and the int8 u
                                   bricks dope_admm_init fills (may be NULL in
                                   2D)                                          */
    /* Sharding: this lattice is a slab of whole block rows (2D) or whole
     * block planes (3D, along the depth axis) of a larger grid.  y2[i] and
     * yhat must then point one row (2D) / one plane (3D) INTO allocations
     * that carry a ghost row / plane on each side (2D allocations always do;
     * 3D ones only need them on a side whose ghost flag is set). */
    int32_t ghost_up;           /* a neighbour shard exists above / before     */
    int32_t ghost_dn;           /* a neighbour shard exists below / after      */
    int32_t sharded;            /* run-loop consensus publishes its slot of
                                   agg[] instead of deciding; dope_decide
                                   reduces the gathered table                  */
    int64_t *agg;               /* sharded: 8 * shard_count int64, one slot per
                                   shard: [energy of y_{t-1}, sum of block
                                   ||yhat - y||^2, sum of their rounding
                                   excesses x 2^53, max block ||.||^2, clamped,
                                   end-of-run energy, 0, 0] -- exact integers,
                                   reduced in shard order by dope_decide      */
    void *halo;                 /* sharded: dope_halo_bytes(L) bytes: boundary
                                   rows out / in (U bytes each, U = W in 2D,
                                   dims[1] * dims[2] in 3D) and the int16
                                   multipliers of the two ghost rows / planes */
    /* Audit mode (optional, NULL = off): after every iteration of the run
     * loop the device adds the iteration's state digest -- position-weighted
     * sums of yhat, 2y and a, oracle/dope_oracle.c state_digest -- into
     * trace_hash[3 (t - 1) .. 3 (t - 1) + 2]; the buffer holds 3 * max_iters
     * + 2 words and must be zeroed before the run.  hash_base = global index
     * of this lattice's first pixel (a shard of a larger grid), else 0.     */
    uint64_t *trace_hash;
    int64_t hash_base;
    int32_t shard_index;        /* sharded: this shard's slot in agg[]          */
    int32_t shard_count;        /* sharded: number of shards (slots in agg[])   */
    const struct dope_peers *peers; /* peer-memory exchange (device pointer to a
                                   dope_peers, see below), or NULL            */
} dope_lattice;

/* Peer-memory exchange of the sharded loop (no NCCL inside the run loop):
 * the kernel that produces a halo row or an agg slot stores it straight into
 * the neighbour / peer shards' memory (NVLink P2P stores across GPUs, plain
 * stores between loopback shards) and raises an epoch flag there; the
 * consumer waits on the flag.  K1's last CTA pushes the shard's boundary label
 * rows, the consensus pass's last CTA pushes the agg slot (table halves
 * alternate by iteration parity), dope_peer_install / dope_ghost_decide wait.
 * Layout in each shard's halo buffer after the ghost multipliers: uint32
 * flags [row from above, row from below, K1 done-counter, pad, agg-slot flag
 * of every shard] (dope_halo_bytes counts them); agg[] holds 2 x 8 x
 * shard_count int64 in peer mode. */
#define DOPE_MAX_SHARDS 64
typedef struct dope_peers {
    uint8_t *row_to_up;         /* upper neighbour's "from below" halo slot, or NULL */
    uint8_t *row_to_dn;         /* lower neighbour's "from above" halo slot, or NULL */
    uint32_t *flag_to_up;       /* its row flag for that slot                  */
    uint32_t *flag_to_dn;
    int64_t *agg_of[DOPE_MAX_SHARDS];    /* every shard's agg table            */
    uint32_t *aflag_of[DOPE_MAX_SHARDS]; /* every shard's agg-slot flags       */
} dope_peers;

/* Library / ABI identification; "b200-sm100a". */
const char *dope_backend_name(void);
int dope_abi_version(void);
const char *dope_last_cuda_error(void);

/* Bytes of residual state per block for this geometry (0 if unsupported). */
int64_t dope_resid_stride(const dope_lattice *L);
/* Bytes of per-block scratch (3D node state; 0 in 2D). */
int64_t dope_scratch_stride(const dope_lattice *L);
/* Validate geometry / capacities; 0 or DOPE_E_*. */
int dope_lattice_check(const dope_lattice *L);
/* Set kernel attributes ahead of CUDA-graph capture (called internally). */
int dope_prepare_kernels(const dope_lattice *L);

/* init_state (admm.py:102-110): y = 1/2, a = 0, yhat = 0, every block dirty,
 * cold residual graphs, run state reset. */
int dope_admm_init(const dope_lattice *L, void *stream);
/* update_blocks: one CTA per sub-region computes 2*linear from (u, a, y,
 * y-halo) and solves the block min cut on the GPU; yhat = sink side. */
int dope_update_blocks(const dope_lattice *L, void *stream);
/* update_global + block_residuals (+ update_multipliers when
 * fuse_multipliers); marks next iteration's dirty blocks.  In run-loop mode
 * (fuse_multipliers) the last CTA also finalizes the iteration: trace entry,
 * best iterate (its energy is that of the previous iterate, whose
 * neighbours are all in HBM already), stop rule. */
int dope_update_global(const dope_lattice *L, void *stream);
/* update_multipliers alone (a += yhat - y) for the step-level API. */
int dope_update_multipliers(const dope_lattice *L, void *stream);
/* `iters` iterations of blocks -> global -> reduce (no host sync); launches
 * become no-ops once converged.  use_graph: capture one iteration in a CUDA
 * graph and replay it. */
int dope_admm_run(const dope_lattice *L, int32_t iters, int32_t use_graph, void *stream);
/* Run-loop entry (dope_admm_run / dope_sharded_run call it): the current
 * iteration's dirty-block worklist rebuilt from the re-solve flags. */
int dope_rebuild_dirty_list(const dope_lattice *L, void *stream);
/* End of run (admm.py:242-252): energy + best check of the last iterate;
 * the current iterate becomes the best one unless converged. */
int dope_finish_run(const dope_lattice *L, void *stream);
/* Sharded run loop: reduce the gathered agg[] table in shard order and apply
 * it (trace, best, stop) -- identical on every shard. */
int dope_decide(const dope_lattice *L, void *stream);
/* Sharded run loop, after the consensus pass (before dope_decide): new
 * iterate and multipliers of the ghost rows / planes computed locally from
 * the exchanged labels (replaces a y-halo exchange); marks the adjacent local
 * blocks dirty where the ghost iterate moved.  Blocks must be >= 2 rows /
 * planes deep along the sharded axis (else DOPE_E_GEOMETRY). */
int dope_ghost_consensus(const dope_lattice *L, void *stream);
/* dope_ghost_consensus and dope_decide in one launch (the last CTA decides
 * once every ghost pixel is in): the run loop's step after the agg gather. */
int dope_ghost_decide(const dope_lattice *L, void *stream);
/* Bytes of the sharded halo buffer (L->halo) for this geometry. */
int64_t dope_halo_bytes(const dope_lattice *L);
/* Audit mode: add this iteration's state digest into L->trace_hash (no-op
 * when trace_hash is NULL or the iteration was already digested). */
int dope_trace_digest(const dope_lattice *L, void *stream);
/* Sharded run loop: install the neighbour shards' boundary rows (2D) /
 * planes (3D) into the ghost rows / planes; which = 0: labels (uint8[U]),
 * 1: current y2 (uint8[U], marks the adjacent local blocks dirty where it
 * changed). */
int dope_ghost_update(const dope_lattice *L, int32_t which, const void *up_row,
                      const void *dn_row, void *stream);
/* Sharded run loop: copy the first / last local row (2D) / plane (3D) of the
 * labels (which=0) or of the current iterate y2 (which=1) into staging
 * buffers (either may be NULL) for the halo exchange (U bytes each). */
int dope_pack_rows(const dope_lattice *L, int32_t which, void *first_row, void *last_row,
                   void *stream);
/* dope_finish_run in two halves for sharded runs: the local energy of the
 * current iterate into this shard's agg slot (gather the table across
 * shards), then the final decision on the summed energy. */
int dope_energy_local(const dope_lattice *L, void *stream);
int dope_finish_decide(const dope_lattice *L, void *stream);
/* Multi-GPU (NCCL over NVLink / NVSwitch), one rank per GPU, 2D and 3D
 * lattices (slabs of block rows / block planes).  Per iteration: K1, ONE
 * grouped send/recv of the boundary label rows, the consensus pass, ONE
 * all-gather of the 64-byte agg slots, dope_ghost_decide (at world size 1:
 * K1, the consensus pass, dope_ghost_decide -- nothing to exchange).
 * dope_comm_unique_id on rank 0, broadcast the 128 bytes, dope_comm_init on
 * every rank.  dope_sharded_run runs `iters` iterations of that loop --
 * captured in one CUDA graph when use_graph; dope_sharded_finish ends the
 * run (energy of the last iterate gathered, final decision). */
int dope_comm_unique_id(uint8_t *out128);
int dope_comm_init(int32_t rank, int32_t world, const uint8_t *id128, void **comm_out);
/* Loopback communicator: all `world` shards of one grid held by THIS process
 * on one device -- the single-GPU stand-in for `world` ranks.  It runs the
 * same iteration (and graph capture) as the NCCL communicator: each boundary
 * row travels by one cudaMemcpyAsync into the receiver's halo slot, each agg
 * slot by one copy into every peer's table; no kernel waits on another. */
int dope_comm_loopback(int32_t world, void **comm_out);
/* Loopback shards with the peer-memory exchange: builds each shard's
 * dope_peers (device memory owned by the communicator) from the shards'
 * halo / agg buffers and returns their device pointers in peers_out[world]
 * (set shards[r]->peers = peers_out[r] before running). */
int dope_comm_loopback_peer(int32_t world, const dope_lattice *const *shards, void **comm_out,
                            void **peers_out);
/* Multi-GPU peer-memory exchange over CUDA IPC: each rank allocates its halo
 * and agg buffers with dope_peer_alloc (IPC needs allocation bases), exports
 * their handles (dope_peer_export, 128 bytes), all-gathers them out of band
 * (e.g. torch.distributed), and opens the others' (dope_comm_peer_init). */
int dope_peer_alloc(int64_t bytes, void **ptr);
int dope_peer_free(void *ptr);
int dope_peer_export(const dope_lattice *L, uint8_t *out128);
int dope_comm_peer_init(const dope_lattice *L, const uint8_t *all128, void **comm_out, void **peers_out);
/* Peer mode, after K1: wait for the neighbours' boundary rows, install them
 * in the ghost rows. */
int dope_peer_install(const dope_lattice *L, void *stream);
int dope_comm_destroy(void *comm);
/* One shard (NCCL communicator: this rank's slab). */
int dope_sharded_run(const dope_lattice *L, void *comm, int32_t iters, int32_t use_graph,
                     void *stream);
int dope_sharded_finish(const dope_lattice *L, void *comm, void *stream);
/* All shards a communicator holds in this process: 1 for NCCL, `world` for
 * loopback (shards[r].shard_index == r). */
int dope_sharded_run_group(const dope_lattice *const *shards, int32_t nshards, void *comm,
                           int32_t iters, int32_t use_graph, void *stream);
int dope_sharded_finish_group(const dope_lattice *const *shards, int32_t nshards, void *comm,
                              void *stream);
/* Instantiated run-loop graphs held by the library (bounded LRU per loop
 * kind, DOPE_GRAPH_CACHE entries each) and a way to drop them all. */
int64_t dope_graph_cache_entries(void);
void dope_graph_cache_clear(void);
/* The integer path's unary from a float64 vector (EnergyModel.unary): out[i]
 * = u[i] when every u[i] is an integer within +-2^28, else *bad |= 1 (zero
 * it first) -- the device side of re-running a lowered model on new unaries. */
int dope_unary_i32(const double *u, int64_t n, int32_t *out, int32_t *bad, void *stream);
/* Page-lock / release a caller's host buffer in place (cudaHostRegister),
 * so the unary of run()'s serving loop is DMA'd without a staging copy.
 * Returns DOPE_OK, or DOPE_E_CUDA with the runtime error cleared. */
int dope_host_register(void *ptr, int64_t bytes);
int dope_host_unregister(void *ptr);
/* binarize (admm.py:202-204) of the current iterate into out[n] (0/1). */
int dope_binarize(const dope_lattice *L, uint8_t *out, void *stream);
/* evaluate_energy of an arbitrary doubled labeling y2 (int path):
 * out[0] = sum u*y2 * 2 + lamw * sum (y2_i - y2_j)^2, i.e. 4*E (exact). */
int dope_energy4(const dope_lattice *L, const int32_t *y2, int64_t *out, void *stream);

/* Seam 1: general two-terminal graph, float64 capacities with the
 * reference's EPS = 1e-12 saturation rule (_core.pyx:13).  Device pointers;
 * m nodes, npairs pairs (arc 2p: i->j with cap_ij[p], arc 2p+1: j->i with
 * cap_ji[p], _core.pyx:293-297).  labels[i] = 1 iff node i reaches the sink
 * in the final residual graph (== the reference's sink tree); flow[0]
 * receives the max-flow value.  Inputs are not modified (_core.pyx:269).
 * `workspace` must hold dope_bk_workspace_bytes(m, npairs) bytes. */
int dope_bk_maxflow(int32_t m, const double *tcap, int64_t npairs, const int32_t *pair_i,
                    const int32_t *pair_j, const double *cap_ij, const double *cap_ji,
                    uint8_t *labels, double *flow, void *workspace, int64_t workspace_bytes,
                    void *stream);
int64_t dope_bk_workspace_bytes(int32_t m, int64_t npairs);

/* ------------------------------------------------------------------------
 * Float-weight 2D lattices (BASELINE C2: 8-connected contrast weights).
 * The block objective is evaluated in float64 in the reference's order and
 * quantised once: terminal rint(linear*qscale), pair rint(lam*w*qscale); the
 * block min cut of the quantised energy is solved exactly.  y and a are
 * float64; state.best_energy holds the best energy's double bits.
 * ------------------------------------------------------------------------ */
typedef struct dope_lattice_f {
    int32_t conn;               /* 4 or 8                                      */
    int64_t dims[2];            /* H, W                                        */
    int32_t kpa[2];
    double lam;                 /* lambda                                      */
    double mu;                  /* ADMM penalty (mu_fact = 1)                  */
    double eps;
    double qscale;              /* capacity quantisation scale (2^16)          */
    int32_t max_iters, warm_start, skip_clean, fuse_multipliers;
    const double *u;            /* n                                           */
    const double *w[4];         /* E S SE SW weight planes: w of pair (i, i+off)
                                   stored at i (SE/SW only when conn == 8)     */
    const double *rdiag;        /* n: r = d - dhat (blockform.py:75)      */
    const int32_t *capq[4];     /* rint(lam * w * qscale), same layout          */
    double *a[2];               /* n; a[0] updated in place (a[1] unused by the
                                   run loop, kept for the ABI)                 */
    double *y[3];               /* n, rotating iterates                        */
    uint8_t *yhat;              /* n                                           */
    int32_t *resid;             /* K * dope_f_resid_stride bytes               */
    uint32_t *dirty;            /* 6K: [0, K) re-solve flags, [K, 2K) solve
                                   epochs, [2K, 5K) y-buffer stamps, [5K, 6K)
                                   last change of each block's iterate (the
                                   clean-block consensus pass)                 */
    double *part_energy;        /* K                                           */
    double *part_ressq;         /* K                                           */
    int32_t *part_flags;        /* K                                           */
    dope_run_state *state;
    double *trace_energy, *trace_residual_sq, *trace_max_residual;
    int32_t *trace_clamped;
    uint64_t *trace_hash;       /* optional audit digests (labels only), as in
                                   dope_lattice                                */
    int32_t energy_prepass;     /* 1: the block min-cut kernel also sums the
                                   energy of the current iterate over the
                                   interior of every block it re-solves (in
                                   the warps that wait for a relabel BFS), so
                                   the consensus pass skips that loop.  Needs
                                   dirty = 7K words ([6K, 7K): pass of each
                                   block's interior energy) and part_energy =
                                   33K doubles ([K, 33K): 32 per-warp sums per
                                   block).  0: the 6K / K layouts              */
} dope_lattice_f;

int64_t dope_f_resid_stride(const dope_lattice_f *L);
int dope_f_check(const dope_lattice_f *L);
const char *dope_f_last_error(void);
int dope_f_admm_init(const dope_lattice_f *L, void *stream);
int dope_f_update_blocks(const dope_lattice_f *L, void *stream);
int dope_f_update_global(const dope_lattice_f *L, void *stream);
int dope_f_update_multipliers(const dope_lattice_f *L, void *stream);
int dope_f_admm_run(const dope_lattice_f *L, int32_t iters, int32_t use_graph, void *stream);
int dope_f_finish_run(const dope_lattice_f *L, void *stream);
int dope_f_binarize(const dope_lattice_f *L, uint8_t *out, void *stream);

/* ---------------------------------------------------------------------------
 * General lattice path: box partitions WITH overlap
 * (make_partition overlap_pct 10 / 25: pixel block counts q in {1, 2, 4}, every
 * block owns a copy of its pixels' labels and multipliers), float64 4- or
 * 8-connected weights, mu schedule mu_t = mu0 * mu_fact^t and the eps stop
 * rule -- the reference's default AdmmConfig.  Replaces admm.run /
 * update_blocks / update_global / update_multipliers (admm.py:113-252) with
 * blockform.py:48-105 evaluated per copy on the lattice stencil.  Float
 * parity bar (final energy within 1e-5 relative, <= 0.01 % labels).
 * ------------------------------------------------------------------------- */
typedef struct dope_general {
    int32_t conn;               /* 4 or 8                                      */
    int64_t dims[2];            /* H, W                                        */
    int32_t kpa[2];             /* blocks per axis                             */
    int32_t box[2];             /* largest block extent per axis               */
    double lam, mu0, mu_fact, eps;
    double qscale;              /* capacity quantisation scale (2^16)          */
    int32_t max_iters, warm_start;
    const double *u;            /* n                                           */
    const double *w[4];         /* E S SE SW weight planes (pair stored at its
                                   lower pixel; SE/SW only when conn == 8)     */
    const uint8_t *q;           /* n: blocks holding each pixel                */
    const int32_t *ranges;      /* 2*KY + 2*KX: row lo[KY], row len[KY],
                                   col lo[KX], col len[KX] (partition.py:62-77) */
    double *a;                  /* K * dope_g_copy_stride: per-copy multipliers */
    uint8_t *yhat;              /* K * dope_g_copy_stride: per-copy labels     */
    int32_t *resid;             /* K * conn * dope_g_copy_stride: residuals    */
    double *y[3];               /* n: rotating iterates (current, best, next)  */
    double *part_energy;        /* dope_g_partials(): energy partials          */
    double *part_ressq;         /* K: ||yhat_k - S_k y||^2                     */
    int32_t *part_flags;        /* dope_g_partials(): clamp flags (zeroed)     */
    double *scal;               /* 1: current mu                               */
    dope_run_state *state;
    double *trace_energy, *trace_residual_sq, *trace_max_residual, *trace_mu;
    int32_t *trace_clamped;     /* max_iters each                              */
} dope_general;

int64_t dope_g_copy_stride(const dope_general *L);
/* Row length of the padded per-copy box (copy_stride = rows * this). */
int64_t dope_g_box_width(const dope_general *L);
int64_t dope_g_partials(const dope_general *L);
int dope_g_check(const dope_general *L);
const char *dope_g_last_error(void);
int dope_g_admm_init(const dope_general *L, void *stream);
int dope_g_admm_run(const dope_general *L, int32_t iters, int32_t use_graph, void *stream);
int dope_g_update_blocks(const dope_general *L, void *stream);   /* one K1 pass   */
int dope_g_update_global(const dope_general *L, void *stream);   /* global step,
                           residuals + multipliers, energy, trace / stop    */
int dope_g_finish_run(const dope_general *L, void *stream);
int dope_g_binarize(const dope_general *L, uint8_t *out, void *stream);

/* ---------------------------------------------------------------------------
 * Model construction on the GPU.  `dims` and `offs`
 * (the half window, grid.py:80-116, offsets row-major) are HOST arrays; all
 * other pointers are device buffers.
 * ------------------------------------------------------------------------- */
const char *dope_in_last_error(void);
/* number of pairs of the half window over the grid (-1: bad arguments)     */
int64_t dope_in_pair_count(int32_t ndim, const int64_t *dims, int32_t noff, const int32_t *offs);
/* length of the partial-sum arrays the reductions below write              */
int64_t dope_in_partials(int64_t n);
/* build_potts_weights (energy.py:124-162): rows/cols/vals of every pair in
 * the reference's order; vals = exp(-|x_i - x_j|^2 / (2 sigma^2)) or 1     */
int dope_in_potts_weights(int32_t ndim, const int64_t *dims, int32_t channels, const double *data,
                          int32_t noff, const int32_t *offs, double sigma, int32_t contrast,
                          int64_t *rows, int64_t *cols, double *vals, void *stream);
/* estimate_sigma (energy.py:165-184): per-CTA partial sums of |x_i - x_j|^2 */
int dope_in_sq_diff(int32_t ndim, const int64_t *dims, int32_t channels, const double *data,
                    int32_t noff, const int32_t *offs, double *partials, void *stream);
/* compute_unaries (energy.py:298-323); seeds may be NULL                    */
int dope_in_unaries(int64_t n, int32_t channels, const double *data, const int8_t *seeds,
                    const double *fg_centroids, const double *bg_centroids, const double *fg_weights,
                    const double *bg_weights, int32_t nclusters, double bandwidth, double *u,
                    double *partials, void *stream);

/* ---------------------------------------------------------------------------
 * Whole-grid serial graph cut (cli.run_serial ->
 * maxflow.solve_binary on the full image).  2D lattice, 4- or 8-connected:
 * tcap = signed terminal capacity (maxflow.py:73-97), w[0..3] = E S SE SW pair
 * weights (device, pair stored at its lower pixel), capacities lam * w.  One
 * cooperative kernel; labels = nodes reaching the sink side (ties -> 0).
 * stats (device, 3 int64): global-relabel rounds (-1: round limit), sweeps.
 * ------------------------------------------------------------------------- */
const char *dope_gc_last_error(void);
int64_t dope_gc_workspace_bytes(int64_t H, int64_t W, int32_t conn);
int dope_gc_mincut(int64_t H, int64_t W, int32_t conn, const double *tcap, const double *const *w,
                   double lam, double qscale, uint8_t *labels, int64_t *stats, void *workspace,
                   int64_t ws_bytes, void *stream);

/* ---------------------------------------------------------------------------
 * General graph path (dope_gstep.cu): the step functions of admm.py:113-199 and
 * evaluate_energy (energy.py:187-194) for ANY SparseWeights pair set on ANY
 * box partition (2D / 3D, overlap 0 / 10 / 25), float64 -- what the lattice
 * kernels above do not cover.  Block-local data are "entries": block k's
 * pixels (ascending, partition.py:52-59) at [blk_ptr[k], blk_ptr[k + 1]).
 * The block operators of blockform.py:48-105 are evaluated on the fly from
 * the symmetric CSR of W.  All pointers are device pointers.
 * ------------------------------------------------------------------------- */
typedef struct dope_gstep {
    int64_t n;                  /* pixels                                      */
    int32_t K;                  /* blocks                                      */
    int64_t M;                  /* entries: sum of block sizes                 */
    const int64_t *adj_ptr;     /* n + 1: symmetric CSR of W (both triangles,
                                   columns ascending)                          */
    const int32_t *adj_idx;
    const double *adj_w;
    const double *deg;          /* n: row sums d of W                          */
    const double *u;            /* n: unary                                    */
    const double *q;            /* n: block counts (partition.counts)          */
    const int64_t *blk_ptr;     /* K + 1                                       */
    const int32_t *ent_pix;     /* M: global pixel of each entry               */
    const int32_t *ent_blk;     /* M: block of each entry                      */
    const int64_t *mem_ptr;     /* n + 1: entries holding each pixel           */
    const int64_t *mem_ent;     /* sum q: those entries, blocks ascending      */
    const double *r;            /* M: remainder d/q^2 - dhat (dope_gs_prepare) */
} dope_gstep;

const char *dope_gs_last_error(void);
/* r[e] = d_g / q_g^2 - dhat_e (blockform.py:75) for every entry. */
int dope_gs_prepare(const dope_gstep *G, double *r, void *stream);
/* block_objective (blockform.py:89-105) of entries [e0, e1):
 * linear = u/q + lam (C y + r S y) + mu ((a - S y) + 1/2). */
int dope_gs_objective(const dope_gstep *G, int64_t e0, int64_t e1, const double *y, const double *a,
                      double mu, double lam, double *linear, void *stream);
/* solve_global (admm.py:136-151) -> y; clamp != 0: update_global's clip to
 * [0, 1] and *clamped |= any value outside (admm.py:172-180; zero it first).
 * mu <= 0 -> DOPE_E_ARGS (the reference's ValueError). */
int dope_gs_solve_global(const dope_gstep *G, const uint8_t *yhat, const double *a, double mu, double lam,
                         double *y, int32_t clamp, int32_t *clamped, void *stream);
/* ss[k] = ||yhat_k - S_k y||^2 (block_residuals, admm.py:193-199). */
int dope_gs_residuals(const dope_gstep *G, const uint8_t *yhat, const double *y, double *ss, void *stream);
/* a += yhat - S y per entry (update_multipliers, admm.py:183-190). */
int dope_gs_update_multipliers(const dope_gstep *G, const uint8_t *yhat, const double *y, double *a,
                               void *stream);
/* consensus_objective (admm.py:154-169) per block: out[2k] = yhat_k . (C_k y +
 * r_k S_k y), out[2k + 1] = ||S_k y - (yhat_k + a_k)||^2. */
int dope_gs_consensus_objective(const dope_gstep *G, const uint8_t *yhat, const double *a, const double *y,
                                double *out2k, void *stream);
/* evaluate_energy (energy.py:187-194) over a pair list: out3 = [u.y + lam q,
 * q = sum w (y_i - y_j)^2, u.y]; deterministic (fixed-order reduction);
 * scratch holds dope_gs_energy_scratch() doubles. */
int64_t dope_gs_energy_scratch(void);
int dope_gs_energy(int64_t n, const double *u, int64_t npairs, const int32_t *pair_i, const int32_t *pair_j,
                   const double *w, double lam, const double *y, double *scratch, double *out3, void *stream);
/* A batch of B graphs, one CTA each, with seam 1's semantics (labels = nodes
 * reaching the sink; flows[b]); graph b: nodes [node_off[b], node_off[b+1]),
 * pairs [pair_off[b], pair_off[b+1]) with graph-local ends, workspace at
 * ws_off[b] (dope_bk_workspace_bytes of that graph).  Offsets are device
 * arrays.  adj_off / adj (optional, NULL: built per solve): each graph's
 * tail-grouped arc lists in pair order (arc 2p: i->j, 2p+1: j->i), graph b's
 * m_b + 1 offsets at adj_off + node_off[b] + b, its 2 P_b arcs at
 * adj + 2 pair_off[b]. */
int dope_bk_maxflow_batch(int32_t B, const int64_t *node_off, const int64_t *pair_off, const int64_t *ws_off,
                          const double *tcap, const int32_t *pair_i, const int32_t *pair_j, const double *cap_ij,
                          const double *cap_ji, uint8_t *labels, double *flows, void *workspace,
                          const int32_t *adj_off, const int32_t *adj, void *stream);
/* exhaustive_minimize (solvers.py:53-82) of a batch of graphs of <= 24 nodes:
 * variable 0 is the most significant bit, ties to the smallest code. */
int dope_exhaustive_batch(int32_t B, const int64_t *node_off, const int64_t *pair_off, const double *linear,
                          const int32_t *pair_i, const int32_t *pair_j, const double *w, double lam,
                          uint8_t *labels, double *energy, void *stream);

#ifdef __cplusplus
}
#endif
#endif /* DOPE_B200_H */
