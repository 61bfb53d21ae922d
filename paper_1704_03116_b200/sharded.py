"""Multi-GPU sharding of the ADMM loop: slabs of block rows (2D) or block
planes (3D, along the depth axis), halo exchange.

The reference parallelises `update_blocks` over sub-regions with a thread
pool (admm.py:186-190) and keeps everything else global.  Here the
sub-regions are sharded across GPUs as contiguous slabs of block rows.  Within
an iteration the only cross-shard data are one-pixel halos:

  1. K1 on every shard (the block objective reads y of the row / plane
     above and below the slab from the ghost rows / planes);
  2. exchange of the label (yhat) boundary rows -> ghost rows;
  3. consensus pass on every shard -> local aggregates
     [energy of y_{t-1}, sum of block residuals^2, max block residual^2, clamp];
  4. all-reduce of the aggregates (sum, sum, max, max);
  5. `dope_decide` applies the identical trace / best-iterate / stop rule on
     every shard;
  6. exchange of the new y boundary rows -> ghost rows (a changed ghost marks
     the adjacent local block row dirty).

Integer energies, max residuals and labels are therefore bit-identical to the
single-GPU run; the float trace field residual_sq is summed per shard first
(rtol 1e-12).  Communicators: `VirtualComm` runs G shards inside one process
(single-GPU emulation used by the tests), `DistComm` uses torch.distributed
(NCCL on B200s, gloo on CPU) with one shard per rank.
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import _lib
from .admm import AdmmConfig, TraceRecord, _DeviceState, _device
from .energy import EnergyModel
from .lowering import LatticeLowering, lower_lattice
from .partition import Partition


def shard_block_rows(ky: int, world: int) -> list:
    """Contiguous near-equal slabs of block rows, one per rank."""
    if world < 1 or world > ky:
        raise ValueError(f"cannot shard {ky} block rows over {world} ranks")
    base, rem = divmod(ky, world)
    out, lo = [], 0
    for r in range(world):
        n = base + (1 if r < rem else 0)
        out.append((lo, lo + n))
        lo += n
    return out


class _Problems:
    """Minimal stand-in for BlockProblems of one slab (device unary + lowering)."""

    def __init__(self, lowering: LatticeLowering, device):
        import torch
        self.lowering = lowering
        self.device = device
        self.u = torch.as_tensor(lowering.u, device=device)

    @property
    def lam(self) -> float:
        return self.lowering.lam


class GpuShard:
    """One slab of whole block rows (2D) / block planes (3D) on the current
    CUDA device (product executor)."""

    def __init__(self, full: LatticeLowering, kb0: int, kb1: int, mu: int, eps: float,
                 max_iters: int, warm_start: bool = True, skip_clean: bool = True):
        import torch
        dims, kpa = tuple(full.dims), tuple(full.kpa)
        n0, k0 = dims[0], kpa[0]   # the sharded axis: rows (2D) / planes (3D)
        if n0 % k0:
            raise NotImplementedError("sharding needs a uniform tiling along the sharded axis")
        bh = n0 // k0
        self.kb0, self.kb1, self.bh = kb0, kb1, bh
        self.r0, self.r1 = kb0 * bh, kb1 * bh
        u = full.u.reshape(dims)[self.r0:self.r1].ravel()
        low = LatticeLowering((self.r1 - self.r0,) + dims[1:], (kb1 - kb0,) + kpa[1:], full.conn,
                              full.lamw, np.ascontiguousarray(u), full.lam)
        dev = _device()
        self.problems = _Problems(low, dev)
        self.dev = _DeviceState(self.problems, mu, eps, max_iters, warm_start, skip_clean)
        L = self.dev.L
        L.ghost_up = int(kb0 > 0)
        L.ghost_dn = int(kb1 < k0)
        L.sharded = 1
        L.fuse_multipliers = 1
        _lib.check(_lib.lib().dope_lattice_check(C.byref(L)), "dope_lattice_check (shard)")
        self.W = int(np.prod(dims[1:]))   # exchanged unit: one row (2D) / plane (3D), bytes
        self.rows_u8 = [torch.zeros(self.W, dtype=torch.uint8, device=dev) for _ in range(4)]

    # -- kernels ------------------------------------------------------------
    def call(self, name, *args):
        self.dev.call(name, *args)

    def init(self):
        self.call("dope_admm_init")

    def update_blocks(self):
        self.call("dope_update_blocks")

    def update_global(self):
        self.call("dope_update_global")

    def decide(self):
        self.call("dope_decide")

    def energy_local(self):
        self.call("dope_energy_local")

    def finish_decide(self):
        self.call("dope_finish_decide")

    def staging(self, which):
        """(send_first, send_last, recv_up, recv_dn) buffers for labels / y."""
        return self.rows_u8   # labels and y2 are both one byte per pixel

    def pack_rows(self, which):
        first, last, _, _ = self.staging(which)
        lb = _lib.lib()
        _lib.check(lb.dope_pack_rows(C.byref(self.dev.L), which, first.data_ptr(), last.data_ptr(),
                                     self.dev.stream()), "dope_pack_rows")
        return first, last

    def ghost_update(self, which, up, dn):
        lb = _lib.lib()
        _lib.check(lb.dope_ghost_update(C.byref(self.dev.L), which,
                                        up.data_ptr() if up is not None else None,
                                        dn.data_ptr() if dn is not None else None,
                                        self.dev.stream()), "dope_ghost_update")

    # -- aggregates ---------------------------------------------------------
    @property
    def agg(self):
        return self.dev.agg

    @property
    def energy_acc(self):
        import torch
        return self.dev.state.view(torch.int64)[8:9]     # dope_run_state.energy_acc

    def labels(self):
        return self.dev.binarize()


class VirtualComm:
    """All shards in this process (single-GPU emulation of G ranks)."""

    def exchange(self, shards, which):
        packed = [s.pack_rows(which) for s in shards]
        for i, s in enumerate(shards):
            up = packed[i - 1][1] if i > 0 else None
            dn = packed[i + 1][0] if i + 1 < len(shards) else None
            s.ghost_update(which, up, dn)

    def allreduce_agg(self, shards):
        import torch
        a = torch.stack([s.agg for s in shards])
        r2 = a[:, 1].contiguous().view(torch.float64)
        out = torch.stack([a[:, 0].sum(), r2.sum().view(torch.int64), a[:, 2].max(), a[:, 3].max()])
        for s in shards:
            s.agg.copy_(out)

    def allreduce_energy(self, shards):
        import torch
        tot = torch.stack([s.energy_acc for s in shards]).sum(dim=0)
        for s in shards:
            s.energy_acc.copy_(tot)


class DistComm:
    """One shard per rank over torch.distributed (NCCL on GPUs, gloo on CPU)."""

    def __init__(self, group=None):
        import torch.distributed as dist
        self.dist = dist
        self.group = group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)

    def exchange(self, shards, which):
        (s,) = shards
        first, last = s.pack_rows(which)
        _, _, recv_up, recv_dn = s.staging(which)
        dist = self.dist
        ops = []
        if self.rank > 0:
            ops.append(dist.P2POp(dist.isend, first, self.rank - 1, self.group))
            ops.append(dist.P2POp(dist.irecv, recv_up, self.rank - 1, self.group))
        if self.rank + 1 < self.world:
            ops.append(dist.P2POp(dist.isend, last, self.rank + 1, self.group))
            ops.append(dist.P2POp(dist.irecv, recv_dn, self.rank + 1, self.group))
        if ops:
            for req in dist.batch_isend_irecv(ops):
                req.wait()
        s.ghost_update(which, recv_up if self.rank > 0 else None,
                       recv_dn if self.rank + 1 < self.world else None)

    def allreduce_agg(self, shards):
        import torch
        (s,) = shards
        a = s.agg
        dist = self.dist
        dist.all_reduce(a[0:1], op=dist.ReduceOp.SUM, group=self.group)
        r2 = a[1:2].view(torch.float64)
        dist.all_reduce(r2, op=dist.ReduceOp.SUM, group=self.group)
        dist.all_reduce(a[2:4], op=dist.ReduceOp.MAX, group=self.group)

    def allreduce_energy(self, shards):
        (s,) = shards
        self.dist.all_reduce(s.energy_acc, op=self.dist.ReduceOp.SUM, group=self.group)


def run_shards(shards, comm, max_iters: int):
    """The sharded run loop (admm.py:283-310 distributed by slabs)."""
    for s in shards:
        s.init()
    for _ in range(max_iters):
        for s in shards:
            s.update_blocks()
        comm.exchange(shards, 0)
        for s in shards:
            s.update_global()
        comm.allreduce_agg(shards)
        for s in shards:
            s.decide()
        comm.exchange(shards, 1)
    for s in shards:
        s.energy_local()
    comm.allreduce_energy(shards)
    for s in shards:
        s.finish_decide()


def run_virtual(model: EnergyModel, partition: Partition, config: AdmmConfig, shards: int):
    """`run` with the sub-regions sharded over `shards` virtual ranks on this GPU.

    Returns (labels, trace, state_fields) assembled from the shards."""
    full = lower_lattice(model, partition)
    if config.mu_fact != 1.0:
        raise NotImplementedError("the integer lattice path keeps mu fixed (mu_fact == 1)")
    mu0 = config.resolved_mu0(len(full.dims))
    eps = config.resolved_eps(partition)
    slabs = shard_block_rows(full.kpa[0], shards)
    sh = [GpuShard(full, a, b, int(mu0), eps, config.max_iters, config.warm_start,
                   config.skip_clean) for a, b in slabs]
    run_shards(sh, VirtualComm(), config.max_iters)
    return collect(sh, mu0, config)


def collect(shards, mu0, config):
    """Labels / trace / state of a sharded run (all shards hold the same decisions)."""
    import torch
    labels = torch.cat([s.labels() for s in shards]).to(torch.int8).cpu().numpy()
    s0 = shards[0].dev
    rs = s0.raise_on_error()
    it = rs.iteration
    e = s0.tr_e[:it].cpu().numpy()
    r2 = s0.tr_rs[:it].cpu().numpy()
    mr = s0.tr_mr[:it].cpu().numpy()
    cl = s0.tr_cl[:it].cpu().numpy()
    trace = [TraceRecord(t + 1, mu0, float(e[t]), float(r2[t]), float(mr[t]), 0.0, bool(cl[t]))
             for t in range(it)]
    y = torch.cat([s.dev.y2_current() for s in shards]).double().div_(2.0).cpu().numpy()
    yhat = torch.cat([s.dev.yhat for s in shards]).cpu().numpy()
    return labels, trace, {"iterations": it, "converged": bool(rs.converged),
                           "best_iteration": int(rs.best_iteration), "y": y, "yhat": yhat}


class NcclComm:
    """NCCL communicator owned by libdope_b200 (one rank per GPU).

    The 128-byte unique id is created on rank 0 and broadcast with
    torch.distributed (any backend); the halo exchanges and all-reduces then
    run inside dope_sharded_run's CUDA graph."""

    def __init__(self, rank: int, world: int, group=None):
        import torch
        import torch.distributed as dist
        lb = _lib.lib()
        uid = torch.zeros(128, dtype=torch.uint8)
        if rank == 0:
            buf = (C.c_uint8 * 128)()
            _lib.check(lb.dope_comm_unique_id(buf), "dope_comm_unique_id")
            uid.copy_(torch.tensor(list(buf), dtype=torch.uint8))
        if world > 1:
            obj = [uid]
            dist.broadcast_object_list(obj, src=0, group=group)
            uid = obj[0]
        raw = (C.c_uint8 * 128)(*uid.tolist())
        self.handle = C.c_void_p()
        _lib.check(lb.dope_comm_init(rank, world, raw, C.byref(self.handle)), "dope_comm_init")
        self.rank, self.world = rank, world

    def close(self):
        if self.handle:
            _lib.lib().dope_comm_destroy(self.handle)
            self.handle = C.c_void_p()


class NcclShard(GpuShard):
    """A GpuShard whose whole run loop (NCCL halos included) is one CUDA graph."""

    def __init__(self, *args, **kw):
        import torch
        super().__init__(*args, **kw)
        self.halo = torch.zeros(16 * self.W, dtype=torch.uint8, device=self.problems.device)
        self.dev.L.halo = self.halo.data_ptr()

    def run(self, comm: NcclComm, iters: int, use_graph: bool = True):
        lb = _lib.lib()
        self.init()
        _lib.check(lb.dope_sharded_run(C.byref(self.dev.L), comm.handle, iters, int(use_graph),
                                       self.dev.stream()), "dope_sharded_run")
        _lib.check(lb.dope_sharded_finish(C.byref(self.dev.L), comm.handle, self.dev.stream()),
                   "dope_sharded_finish")


def shard_for_rank(model: EnergyModel, partition: Partition, config: AdmmConfig, rank: int,
                   world: int, cls=NcclShard):
    full = lower_lattice(model, partition)
    mu0 = config.resolved_mu0(len(full.dims))
    kb0, kb1 = shard_block_rows(full.kpa[0], world)[rank]
    return cls(full, kb0, kb1, int(mu0), config.resolved_eps(partition), config.max_iters,
               config.warm_start, config.skip_clean)
