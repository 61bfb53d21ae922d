"""ctypes binding of include/dope_b200.h (the C ABI of libdope_b200.so).

The library is REQUIRED: there is no CPU fallback.  Loading fails loudly when
the .so is missing or was built against a different ABI version.
"""
from __future__ import annotations

import ctypes as C
from pathlib import Path

import os

# DOPE_LIB: load another build of the library (e.g. the bounds-checked
# libdope_b200_checked.so of `python -m paper_1704_03116_b200.build --checked`)
LIB_PATH = Path(os.environ.get("DOPE_LIB") or Path(__file__).resolve().parent / "libdope_b200.so")
ABI_VERSION = 1

DOPE_OK = 0
DOPE_E_ARGS = -1
DOPE_E_GEOMETRY = -2
DOPE_E_CAPACITY = -3
DOPE_E_CUDA = -4
DOPE_E_NONSUBMODULAR = -5


PART_CTA_LEN = 8   # DOPE_PART_CTA_LEN


class RunState(C.Structure):
    """Mirror of dope_run_state."""
    _fields_ = [
        ("best_energy", C.c_int64),
        ("iteration", C.c_int32),
        ("best_iteration", C.c_int32),
        ("converged", C.c_int32),
        ("stop", C.c_int32),
        ("ycur", C.c_int32),
        ("ybest", C.c_int32),
        ("parity", C.c_int32),
        ("error", C.c_int32),
        ("max_rounds_seen", C.c_int32),
        ("done_ctas", C.c_int32),
        ("solves", C.c_int64),
        ("sweeps", C.c_int64),
        ("energy_acc", C.c_int64),
        ("unary2", C.c_int64),
        ("a_bound", C.c_int32),
        ("generation", C.c_int32),
    ]


class Lattice(C.Structure):
    """Mirror of dope_lattice."""
    _fields_ = [
        ("ndim", C.c_int32),
        ("conn", C.c_int32),
        ("dims", C.c_int64 * 3),
        ("kpa", C.c_int32 * 3),
        ("lamw", C.c_int32),
        ("mu", C.c_int32),
        ("eps", C.c_double),
        ("max_iters", C.c_int32),
        ("warm_start", C.c_int32),
        ("skip_clean", C.c_int32),
        ("fuse_multipliers", C.c_int32),
        ("u", C.c_void_p),
        ("a", C.c_void_p),
        ("y2", C.c_void_p * 3),
        ("yhat", C.c_void_p),
        ("resid", C.c_void_p),
        ("dirty", C.c_void_p),
        ("part_energy", C.c_void_p),
        ("part_unary", C.c_void_p),
        ("part_ressq", C.c_void_p),
        ("part_flags", C.c_void_p),
        ("part_cta", C.c_void_p),
        ("state", C.c_void_p),
        ("trace_energy", C.c_void_p),
        ("trace_residual_sq", C.c_void_p),
        ("trace_max_residual", C.c_void_p),
        ("trace_clamped", C.c_void_p),
        ("timeline", C.c_void_p),
        ("scratch", C.c_void_p),
        ("ghost_up", C.c_int32),
        ("ghost_dn", C.c_int32),
        ("sharded", C.c_int32),
        ("agg", C.c_void_p),
        ("halo", C.c_void_p),
        ("trace_hash", C.c_void_p),
        ("hash_base", C.c_int64),
        ("shard_index", C.c_int32),
        ("shard_count", C.c_int32),
        ("peers", C.c_void_p),
    ]


class LatticeF(C.Structure):
    """Mirror of dope_lattice_f (float-weight 2D lattices)."""
    _fields_ = [
        ("conn", C.c_int32),
        ("dims", C.c_int64 * 2),
        ("kpa", C.c_int32 * 2),
        ("lam", C.c_double),
        ("mu", C.c_double),
        ("eps", C.c_double),
        ("qscale", C.c_double),
        ("max_iters", C.c_int32),
        ("warm_start", C.c_int32),
        ("skip_clean", C.c_int32),
        ("fuse_multipliers", C.c_int32),
        ("u", C.c_void_p),
        ("w", C.c_void_p * 4),
        ("rdiag", C.c_void_p),
        ("capq", C.c_void_p * 4),
        ("a", C.c_void_p * 2),
        ("y", C.c_void_p * 3),
        ("yhat", C.c_void_p),
        ("resid", C.c_void_p),
        ("dirty", C.c_void_p),
        ("part_energy", C.c_void_p),
        ("part_ressq", C.c_void_p),
        ("part_flags", C.c_void_p),
        ("state", C.c_void_p),
        ("trace_energy", C.c_void_p),
        ("trace_residual_sq", C.c_void_p),
        ("trace_max_residual", C.c_void_p),
        ("trace_clamped", C.c_void_p),
        ("trace_hash", C.c_void_p),
        ("energy_prepass", C.c_int32),
    ]


class General(C.Structure):
    """Mirror of dope_general (overlapping partitions, mu schedule)."""
    _fields_ = [
        ("conn", C.c_int32),
        ("dims", C.c_int64 * 2),
        ("kpa", C.c_int32 * 2),
        ("box", C.c_int32 * 2),
        ("lam", C.c_double),
        ("mu0", C.c_double),
        ("mu_fact", C.c_double),
        ("eps", C.c_double),
        ("qscale", C.c_double),
        ("max_iters", C.c_int32),
        ("warm_start", C.c_int32),
        ("u", C.c_void_p),
        ("w", C.c_void_p * 4),
        ("q", C.c_void_p),
        ("ranges", C.c_void_p),
        ("a", C.c_void_p),
        ("yhat", C.c_void_p),
        ("resid", C.c_void_p),
        ("y", C.c_void_p * 3),
        ("part_energy", C.c_void_p),
        ("part_ressq", C.c_void_p),
        ("part_flags", C.c_void_p),
        ("scal", C.c_void_p),
        ("state", C.c_void_p),
        ("trace_energy", C.c_void_p),
        ("trace_residual_sq", C.c_void_p),
        ("trace_max_residual", C.c_void_p),
        ("trace_mu", C.c_void_p),
        ("trace_clamped", C.c_void_p),
    ]


class GStep(C.Structure):
    """Mirror of dope_gstep (general graph path)."""
    _fields_ = [
        ("n", C.c_int64),
        ("K", C.c_int32),
        ("M", C.c_int64),
        ("adj_ptr", C.c_void_p),
        ("adj_idx", C.c_void_p),
        ("adj_w", C.c_void_p),
        ("deg", C.c_void_p),
        ("u", C.c_void_p),
        ("q", C.c_void_p),
        ("blk_ptr", C.c_void_p),
        ("ent_pix", C.c_void_p),
        ("ent_blk", C.c_void_p),
        ("mem_ptr", C.c_void_p),
        ("mem_ent", C.c_void_p),
        ("r", C.c_void_p),
    ]


class DopeError(RuntimeError):
    pass


_lib = None


def lib():
    """Load libdope_b200.so (raises if absent -- no fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    if not LIB_PATH.exists():
        raise DopeError(
            f"{LIB_PATH} is missing: build it with `python -m paper_1704_03116_b200.build` "
            "(the DOPE B200 path has no CPU fallback)")
    lb = C.CDLL(str(LIB_PATH))
    lb.dope_backend_name.restype = C.c_char_p
    lb.dope_abi_version.restype = C.c_int
    lb.dope_last_cuda_error.restype = C.c_char_p
    P = C.POINTER(Lattice)
    lb.dope_resid_stride.restype = C.c_int64
    lb.dope_resid_stride.argtypes = [P]
    lb.dope_scratch_stride.restype = C.c_int64
    lb.dope_scratch_stride.argtypes = [P]
    lb.dope_lattice_check.restype = C.c_int
    lb.dope_lattice_check.argtypes = [P]
    for name in ("dope_admm_init", "dope_update_blocks", "dope_update_global",
                 "dope_update_multipliers", "dope_finish_run", "dope_energy_local",
                 "dope_finish_decide", "dope_ghost_consensus", "dope_trace_digest", "dope_ghost_decide",
                 "dope_rebuild_dirty_list"):
        f = getattr(lb, name)
        f.restype = C.c_int
        f.argtypes = [P, C.c_void_p]
    lb.dope_admm_run.restype = C.c_int
    lb.dope_admm_run.argtypes = [P, C.c_int32, C.c_int32, C.c_void_p]
    lb.dope_prepare_kernels.restype = C.c_int
    lb.dope_prepare_kernels.argtypes = [P]
    lb.dope_comm_unique_id.restype = C.c_int
    lb.dope_comm_unique_id.argtypes = [C.c_void_p]
    lb.dope_comm_init.restype = C.c_int
    lb.dope_comm_init.argtypes = [C.c_int32, C.c_int32, C.c_void_p, C.POINTER(C.c_void_p)]
    lb.dope_comm_destroy.restype = C.c_int
    lb.dope_comm_destroy.argtypes = [C.c_void_p]
    lb.dope_sharded_run.restype = C.c_int
    lb.dope_sharded_run.argtypes = [P, C.c_void_p, C.c_int32, C.c_int32, C.c_void_p]
    lb.dope_sharded_finish.restype = C.c_int
    lb.dope_sharded_finish.argtypes = [P, C.c_void_p, C.c_void_p]
    lb.dope_comm_loopback.restype = C.c_int
    lb.dope_comm_loopback.argtypes = [C.c_int32, C.POINTER(C.c_void_p)]
    PP = C.POINTER(P)
    lb.dope_sharded_run_group.restype = C.c_int
    lb.dope_sharded_run_group.argtypes = [PP, C.c_int32, C.c_void_p, C.c_int32, C.c_int32, C.c_void_p]
    lb.dope_sharded_finish_group.restype = C.c_int
    lb.dope_sharded_finish_group.argtypes = [PP, C.c_int32, C.c_void_p, C.c_void_p]
    lb.dope_comm_loopback_peer.restype = C.c_int
    lb.dope_comm_loopback_peer.argtypes = [C.c_int32, PP, C.POINTER(C.c_void_p), C.POINTER(C.c_void_p)]
    lb.dope_peer_install.restype = C.c_int
    lb.dope_peer_install.argtypes = [P, C.c_void_p]
    lb.dope_peer_alloc.restype = C.c_int
    lb.dope_peer_alloc.argtypes = [C.c_int64, C.POINTER(C.c_void_p)]
    lb.dope_peer_free.restype = C.c_int
    lb.dope_peer_free.argtypes = [C.c_void_p]
    lb.dope_peer_export.restype = C.c_int
    lb.dope_peer_export.argtypes = [P, C.c_void_p]
    lb.dope_comm_peer_init.restype = C.c_int
    lb.dope_comm_peer_init.argtypes = [P, C.c_void_p, C.POINTER(C.c_void_p), C.POINTER(C.c_void_p)]
    lb.dope_halo_bytes.restype = C.c_int64
    lb.dope_halo_bytes.argtypes = [P]
    lb.dope_graph_cache_entries.restype = C.c_int64
    lb.dope_graph_cache_entries.argtypes = []
    lb.dope_graph_cache_clear.restype = None
    lb.dope_graph_cache_clear.argtypes = []
    lb.dope_pack_rows.restype = C.c_int
    lb.dope_pack_rows.argtypes = [P, C.c_int32, C.c_void_p, C.c_void_p, C.c_void_p]
    lb.dope_decide.restype = C.c_int
    lb.dope_decide.argtypes = [P, C.c_void_p]
    lb.dope_ghost_update.restype = C.c_int
    lb.dope_ghost_update.argtypes = [P, C.c_int32, C.c_void_p, C.c_void_p, C.c_void_p]
    lb.dope_binarize.restype = C.c_int
    lb.dope_binarize.argtypes = [P, C.c_void_p, C.c_void_p]
    lb.dope_energy4.restype = C.c_int
    lb.dope_energy4.argtypes = [P, C.c_void_p, C.c_void_p, C.c_void_p]
    lb.dope_bk_maxflow.restype = C.c_int
    lb.dope_bk_maxflow.argtypes = [C.c_int32, C.c_void_p, C.c_int64, C.c_void_p, C.c_void_p,
                                   C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                                   C.c_int64, C.c_void_p]
    lb.dope_bk_workspace_bytes.restype = C.c_int64
    lb.dope_bk_workspace_bytes.argtypes = [C.c_int32, C.c_int64]
    PF = C.POINTER(LatticeF)
    lb.dope_f_resid_stride.restype = C.c_int64
    lb.dope_f_resid_stride.argtypes = [PF]
    lb.dope_f_check.restype = C.c_int
    lb.dope_f_check.argtypes = [PF]
    lb.dope_f_last_error.restype = C.c_char_p
    for name in ("dope_f_admm_init", "dope_f_update_blocks", "dope_f_update_global",
                 "dope_f_update_multipliers", "dope_f_finish_run"):
        f = getattr(lb, name)
        f.restype = C.c_int
        f.argtypes = [PF, C.c_void_p]
    lb.dope_f_admm_run.restype = C.c_int
    lb.dope_f_admm_run.argtypes = [PF, C.c_int32, C.c_int32, C.c_void_p]
    lb.dope_f_binarize.restype = C.c_int
    lb.dope_f_binarize.argtypes = [PF, C.c_void_p, C.c_void_p]
    lb.dope_in_last_error.restype = C.c_char_p
    lb.dope_in_pair_count.restype = C.c_int64
    lb.dope_in_pair_count.argtypes = [C.c_int32, C.c_void_p, C.c_int32, C.c_void_p]
    lb.dope_in_partials.restype = C.c_int64
    lb.dope_in_partials.argtypes = [C.c_int64]
    lb.dope_in_potts_weights.restype = C.c_int
    lb.dope_in_potts_weights.argtypes = [C.c_int32, C.c_void_p, C.c_int32, C.c_void_p, C.c_int32, C.c_void_p,
                                         C.c_double, C.c_int32, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]
    lb.dope_in_sq_diff.restype = C.c_int
    lb.dope_in_sq_diff.argtypes = [C.c_int32, C.c_void_p, C.c_int32, C.c_void_p, C.c_int32, C.c_void_p,
                                   C.c_void_p, C.c_void_p]
    lb.dope_in_unaries.restype = C.c_int
    lb.dope_in_unaries.argtypes = [C.c_int64, C.c_int32, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                                   C.c_void_p, C.c_void_p, C.c_int32, C.c_double, C.c_void_p, C.c_void_p,
                                   C.c_void_p]
    lb.dope_gc_last_error.restype = C.c_char_p
    lb.dope_gc_workspace_bytes.restype = C.c_int64
    lb.dope_gc_workspace_bytes.argtypes = [C.c_int64, C.c_int64, C.c_int32]
    lb.dope_gc_mincut.restype = C.c_int
    lb.dope_gc_mincut.argtypes = [C.c_int64, C.c_int64, C.c_int32, C.c_void_p, C.c_void_p, C.c_double,
                                  C.c_double, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p]
    PG = C.POINTER(General)
    for name in ("dope_g_copy_stride", "dope_g_box_width", "dope_g_partials"):
        f = getattr(lb, name)
        f.restype = C.c_int64
        f.argtypes = [PG]
    lb.dope_g_check.restype = C.c_int
    lb.dope_g_check.argtypes = [PG]
    lb.dope_g_last_error.restype = C.c_char_p
    for name in ("dope_g_admm_init", "dope_g_finish_run", "dope_g_update_blocks", "dope_g_update_global"):
        f = getattr(lb, name)
        f.restype = C.c_int
        f.argtypes = [PG, C.c_void_p]
    lb.dope_g_admm_run.restype = C.c_int
    lb.dope_g_admm_run.argtypes = [PG, C.c_int32, C.c_int32, C.c_void_p]
    lb.dope_g_binarize.restype = C.c_int
    lb.dope_g_binarize.argtypes = [PG, C.c_void_p, C.c_void_p]
    PS = C.POINTER(GStep)
    V = C.c_void_p
    lb.dope_gs_last_error.restype = C.c_char_p
    lb.dope_gs_prepare.restype = C.c_int
    lb.dope_gs_prepare.argtypes = [PS, V, V]
    lb.dope_gs_objective.restype = C.c_int
    lb.dope_gs_objective.argtypes = [PS, C.c_int64, C.c_int64, V, V, C.c_double, C.c_double, V, V]
    lb.dope_gs_solve_global.restype = C.c_int
    lb.dope_gs_solve_global.argtypes = [PS, V, V, C.c_double, C.c_double, V, C.c_int32, V, V]
    lb.dope_gs_residuals.restype = C.c_int
    lb.dope_gs_residuals.argtypes = [PS, V, V, V, V]
    lb.dope_gs_update_multipliers.restype = C.c_int
    lb.dope_gs_update_multipliers.argtypes = [PS, V, V, V, V]
    lb.dope_gs_consensus_objective.restype = C.c_int
    lb.dope_gs_consensus_objective.argtypes = [PS, V, V, V, V, V]
    lb.dope_gs_energy_scratch.restype = C.c_int64
    lb.dope_gs_energy_scratch.argtypes = []
    lb.dope_gs_energy.restype = C.c_int
    lb.dope_gs_energy.argtypes = [C.c_int64, V, C.c_int64, V, V, V, C.c_double, V, V, V, V]
    lb.dope_bk_maxflow_batch.restype = C.c_int
    lb.dope_bk_maxflow_batch.argtypes = [C.c_int32, V, V, V, V, V, V, V, V, V, V, V, V, V, V]
    lb.dope_exhaustive_batch.restype = C.c_int
    lb.dope_exhaustive_batch.argtypes = [C.c_int32, V, V, V, V, V, V, C.c_double, V, V, V]
    lb.dope_trace_digest.restype = C.c_int
    lb.dope_host_register.restype = C.c_int
    lb.dope_host_register.argtypes = [V, C.c_int64]
    lb.dope_host_unregister.restype = C.c_int
    lb.dope_host_unregister.argtypes = [V]
    lb.dope_unary_i32.restype = C.c_int
    lb.dope_unary_i32.argtypes = [V, C.c_int64, V, V, V]
    if lb.dope_abi_version() != ABI_VERSION:
        raise DopeError(f"libdope_b200 ABI {lb.dope_abi_version()} != {ABI_VERSION}")
    _lib = lb
    return lb


def check(rc: int, what: str) -> None:
    if rc == DOPE_OK:
        return
    msg = {DOPE_E_ARGS: "invalid arguments", DOPE_E_GEOMETRY: "unsupported block geometry",
           DOPE_E_CAPACITY: "capacities exceed the int8 residual range",
           DOPE_E_NONSUBMODULAR: "negative pairwise weights"}.get(rc)
    if rc == DOPE_E_CUDA:
        lb = lib()
        msg = "CUDA error: " + (lb.dope_last_cuda_error().decode() or lb.dope_f_last_error().decode()
                                or lb.dope_gs_last_error().decode())
    raise DopeError(f"{what} failed ({rc}): {msg}")
