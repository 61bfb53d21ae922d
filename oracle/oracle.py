"""ctypes front of the CPU oracle (TEST INFRASTRUCTURE ONLY).

Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline leg import
this module, and only as the checker.  The product package
(paper_1704_03116_b200) never imports it.

Functions restate the reference hot path (see dope_oracle.c for file:line
citations):
  bk_maxflow      -- _core.bk_maxflow contract (_core.pyx:263-333)
  run             -- admm.run (admm.py:207-252) on a q == 1 lattice partition
  update_blocks / update_global / block_residuals / energy -- step functions
  reference_core() -- the reference's own compiled _core (oracle/_ref), if built
"""
from __future__ import annotations

import ctypes as C
import glob
import importlib.util
import os
from dataclasses import dataclass
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
MAX_DIRS = 13


class _Lattice(C.Structure):
    _fields_ = [
        ("ndim", C.c_int32),
        ("dims", C.c_int64 * 3),
        ("kpa", C.c_int64 * 3),
        ("ndirs", C.c_int32),
        ("off", (C.c_int32 * 3) * MAX_DIRS),
        ("w", C.c_void_p * MAX_DIRS),
        ("wconst", C.c_double * MAX_DIRS),
        ("u", C.c_void_p),
        ("lam", C.c_double),
    ]


class _RunInfo(C.Structure):
    _fields_ = [("iterations", C.c_int32), ("converged", C.c_int32),
                ("best_iteration", C.c_int32), ("mu_final", C.c_double)]


_lib = None


def lib():
    global _lib
    if _lib is None:
        path = HERE / "liboracle.so"
        if not path.exists() or path.stat().st_mtime < (HERE / "dope_oracle.c").stat().st_mtime:
            from build_oracle import build_oracle  # type: ignore
            build_oracle()
        _lib = C.CDLL(str(path))
        _lib.oracle_bk_maxflow.restype = C.c_int
        _lib.oracle_bk_maxflow.argtypes = [C.c_int32, C.c_void_p, C.c_int64, C.c_void_p, C.c_void_p,
                                           C.c_void_p, C.c_void_p, C.c_void_p,
                                           C.POINTER(C.c_double)]
        _lib.oracle_run.restype = C.c_int
        _lib.oracle_run.argtypes = [C.POINTER(_Lattice), C.c_double, C.c_double, C.c_double,
                                    C.c_int32, C.c_int] + [C.c_void_p] * 11 + [C.POINTER(_RunInfo)]
        _lib.oracle_state_digest.restype = C.c_int
        _lib.oracle_state_digest.argtypes = [C.c_int64, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]
        _lib.oracle_update_blocks.restype = C.c_int
        _lib.oracle_update_blocks.argtypes = [C.POINTER(_Lattice), C.c_void_p, C.c_void_p,
                                              C.c_double, C.c_void_p, C.c_int]
        _lib.oracle_update_global.restype = C.c_int
        _lib.oracle_update_global.argtypes = [C.POINTER(_Lattice), C.c_void_p, C.c_void_p,
                                              C.c_double, C.c_void_p, C.POINTER(C.c_int)]
        _lib.oracle_block_residuals.restype = C.c_int
        _lib.oracle_block_residuals.argtypes = [C.POINTER(_Lattice), C.c_void_p, C.c_void_p,
                                                C.c_void_p]
        _lib.oracle_energy.restype = C.c_double
        _lib.oracle_energy.argtypes = [C.POINTER(_Lattice), C.c_void_p]
        _lib.oracle_num_blocks.restype = C.c_int
        _lib.oracle_num_blocks.argtypes = [C.POINTER(_Lattice), C.POINTER(C.c_int64)]
    return _lib


def _ptr(a: np.ndarray) -> int:
    return a.ctypes.data


def bk_maxflow(tcap, pair_i, pair_j, cap_ij, cap_ji):
    """Oracle restatement of _core.bk_maxflow: (labels uint8[m], flow)."""
    tcap = np.ascontiguousarray(tcap, dtype=np.float64)
    pi = np.ascontiguousarray(pair_i, dtype=np.int32)
    pj = np.ascontiguousarray(pair_j, dtype=np.int32)
    cij = np.ascontiguousarray(cap_ij, dtype=np.float64)
    cji = np.ascontiguousarray(cap_ji, dtype=np.float64)
    m = tcap.size
    labels = np.zeros(m, dtype=np.uint8)
    flow = C.c_double(0.0)
    rc = lib().oracle_bk_maxflow(m, _ptr(tcap), pi.size, _ptr(pi), _ptr(pj), _ptr(cij),
                                 _ptr(cji), _ptr(labels), C.byref(flow))
    if rc:
        raise ValueError(f"oracle_bk_maxflow failed ({rc})")
    return labels, float(flow.value)


@dataclass
class LatticeSpec:
    """A lattice-stencil energy on a non-overlapping box partition.

    dims: row-major grid dims; kpa: blocks per axis (make_partition's
    k_per_axis, overlap 0); offsets: forward stencil offsets (i<j pairs);
    weights: per-direction weight planes indexed by the lower pixel of each
    pair (np.ndarray of n) or scalars; u: unary (n); lam: lambda.
    """
    dims: tuple
    kpa: tuple
    offsets: list
    weights: list
    u: np.ndarray
    lam: float

    def _struct(self):
        s = _Lattice()
        s.ndim = len(self.dims)
        for a, d in enumerate(self.dims):
            s.dims[a] = int(d)
            s.kpa[a] = int(self.kpa[a])
        s.ndirs = len(self.offsets)
        keep = []
        for d, (off, w) in enumerate(zip(self.offsets, self.weights)):
            for a in range(len(self.dims)):
                s.off[d][a] = int(off[a])
            if np.isscalar(w):
                s.w[d] = None
                s.wconst[d] = float(w)
            else:
                arr = np.ascontiguousarray(w, dtype=np.float64).ravel()
                keep.append(arr)
                s.w[d] = _ptr(arr)
        u = np.ascontiguousarray(self.u, dtype=np.float64).ravel()
        keep.append(u)
        s.u = _ptr(u)
        s.lam = float(self.lam)
        return s, keep

    @property
    def n(self) -> int:
        return int(np.prod(self.dims))

    def num_blocks(self) -> int:
        s, keep = self._struct()
        k = C.c_int64(0)
        if lib().oracle_num_blocks(C.byref(s), C.byref(k)):
            raise ValueError("bad partition")
        return int(k.value)


def run(spec: LatticeSpec, mu0: float, mu_fact: float, eps: float, max_iters: int,
        threads: int = 1, keep_history: bool = False, digests: bool = False) -> dict:
    s, keep = spec._struct()
    n = spec.n
    y = np.empty(n)
    a = np.empty(n)
    yhat = np.empty(n, dtype=np.uint8)
    labels = np.empty(n, dtype=np.int8)
    tr = {k: np.zeros(max_iters) for k in ("mu", "energy", "residual_sq", "max_block_residual")}
    clamped = np.zeros(max_iters, dtype=np.int32)
    hist = np.zeros((max_iters, n), dtype=np.uint8) if keep_history else None
    dig = np.zeros((max_iters, 3), dtype=np.uint64) if digests else None
    info = _RunInfo()
    rc = lib().oracle_run(C.byref(s), mu0, mu_fact, eps, max_iters, threads, _ptr(y), _ptr(a),
                          _ptr(yhat), _ptr(labels), _ptr(tr["mu"]), _ptr(tr["energy"]),
                          _ptr(tr["residual_sq"]), _ptr(tr["max_block_residual"]), _ptr(clamped),
                          _ptr(hist) if hist is not None else None,
                          _ptr(dig) if dig is not None else None, C.byref(info))
    if rc:
        raise RuntimeError(f"oracle_run failed ({rc})")
    it = info.iterations
    out = {k: v[:it].copy() for k, v in tr.items()}
    out.update(clamped=clamped[:it].astype(bool), y=y, a=a, yhat=yhat, labels=labels,
               iterations=it, converged=bool(info.converged),
               best_iteration=int(info.best_iteration), mu_final=info.mu_final)
    if hist is not None:
        out["yhat_history"] = hist[:it].copy()
    if dig is not None:
        out["digests"] = dig[:it].copy()
    return out


def state_digest(yhat, y, a) -> np.ndarray:
    """(yhat, 2y, a) position-weighted digest of one state (dope_oracle.c state_digest)."""
    yhat = np.ascontiguousarray(yhat, dtype=np.uint8)
    y = np.ascontiguousarray(y, dtype=np.float64)
    a = np.ascontiguousarray(a, dtype=np.float64)
    out = np.zeros(3, dtype=np.uint64)
    lib().oracle_state_digest(yhat.size, _ptr(yhat), _ptr(y), _ptr(a), _ptr(out))
    return out


def update_blocks(spec: LatticeSpec, y, a, mu, threads: int = 1) -> np.ndarray:
    s, keep = spec._struct()
    y = np.ascontiguousarray(y, dtype=np.float64)
    a = np.ascontiguousarray(a, dtype=np.float64)
    yhat = np.zeros(spec.n, dtype=np.uint8)
    rc = lib().oracle_update_blocks(C.byref(s), _ptr(y), _ptr(a), float(mu), _ptr(yhat), threads)
    if rc:
        raise RuntimeError(f"oracle_update_blocks failed ({rc})")
    return yhat


def update_global(spec: LatticeSpec, yhat, a, mu):
    s, keep = spec._struct()
    yhat = np.ascontiguousarray(yhat, dtype=np.uint8)
    a = np.ascontiguousarray(a, dtype=np.float64)
    y = np.zeros(spec.n)
    cl = C.c_int(0)
    rc = lib().oracle_update_global(C.byref(s), _ptr(yhat), _ptr(a), float(mu), _ptr(y),
                                    C.byref(cl))
    if rc:
        raise ValueError("oracle_update_global failed")
    return y, bool(cl.value)


def block_residuals(spec: LatticeSpec, yhat, y) -> np.ndarray:
    s, keep = spec._struct()
    yhat = np.ascontiguousarray(yhat, dtype=np.uint8)
    y = np.ascontiguousarray(y, dtype=np.float64)
    res = np.zeros(spec.num_blocks())
    lib().oracle_block_residuals(C.byref(s), _ptr(yhat), _ptr(y), _ptr(res))
    return res


def energy(spec: LatticeSpec, y) -> float:
    s, keep = spec._struct()
    y = np.ascontiguousarray(y, dtype=np.float64)
    return float(lib().oracle_energy(C.byref(s), _ptr(y)))


def reference_core():
    """The reference's own compiled max-flow core (oracle/_ref), or None."""
    paths = glob.glob(str(HERE / "_ref" / "_core*.so"))
    if not paths:
        return None
    spec = importlib.util.spec_from_file_location("_core", paths[0])
    mod = importlib.util.module_from_spec(spec)
    try:
        spec.loader.exec_module(mod)
    except ImportError:
        return None
    return mod
