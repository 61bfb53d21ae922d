"""Sharding of the ADMM loop over GPUs: slabs of block rows (2D) or block
planes (3D, along the depth axis) with one ghost row / plane on each side.

The reference parallelises `update_blocks` over sub-regions with a thread
pool inside one process (admm.py:128-132) and keeps everything else global.
Here the sub-regions are sharded across GPUs as contiguous slabs; within an
iteration the only cross-shard data are:

  1. K1 on every shard (the block objective reads y of the row / plane above
     and below the slab from the ghost rows / planes);
  2. the label (yhat) boundary rows -> the neighbours' ghost rows;
  3. the consensus pass on every shard -> this shard's slot of the agg table
     [energy of y_{t-1}, sum ss, sum of rounding excesses, max ss, clamp] --
     exact integers;
  4. `dope_ghost_consensus`: the ghost rows' new y and multipliers recomputed
     locally from the labels of step 2 (no y halo: the values equal the
     owner's bit for bit);
  5. one all-gather of the agg slots;
  6. `dope_decide`: the table reduced in shard order -> the same trace,
     best iterate and stop rule on every shard.

Every trace field, label and iterate is therefore bit-identical to the
single-GPU run (and the reference).  Communicators (csrc/dope_comm.cu): NCCL,
one shard per rank (`NcclComm`, `NcclShard`), and loopback, all shards in one
process on one GPU (`LoopbackGroup`, the single-GPU stand-in for G ranks that
drives the same C++ iteration and graph capture).  `run_shards` + `DistComm`
restate the protocol step by step over torch.distributed for executors that
implement the shard interface (the gloo CPU protocol test).
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import _lib
from .admm import AdmmConfig, TraceRecord, _DeviceState, _device
from .energy import EnergyModel
from .lowering import LatticeLowering, lower_lattice
from .partition import Partition

AGG_SLOT = 8   # int64 per shard in the agg table (dope_b200.h)


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


def _check_config(full: LatticeLowering, config: AdmmConfig) -> int:
    """The integer sharded path's limits (the same as admm._bind): a fixed,
    integer mu dividing lambda*w.  Raises instead of truncating."""
    if config.mu_fact != 1.0:
        raise NotImplementedError("the sharded integer path keeps mu fixed (mu_fact == 1)")
    mu0 = config.resolved_mu0(len(full.dims))
    if mu0 != round(mu0) or mu0 <= 0:
        raise NotImplementedError("the sharded integer path needs an integer mu0")
    if full.lamw % int(round(mu0)) != 0:
        raise NotImplementedError("the sharded integer path needs lambda*w divisible by mu0")
    return int(round(mu0))


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
                 max_iters: int, warm_start: bool = True, skip_clean: bool = True,
                 index: int = 0, count: int = 1, digests: bool = False, ipc: bool = False):
        import torch
        dims, kpa = tuple(full.dims), tuple(full.kpa)
        n0, k0 = dims[0], kpa[0]   # the sharded axis: rows (2D) / planes (3D)
        if n0 % k0:
            raise NotImplementedError("sharding needs a uniform tiling along the sharded axis")
        bh = n0 // k0
        if count > 1 and bh < 2:
            raise NotImplementedError("sharding needs blocks at least two rows / planes deep")
        self.kb0, self.kb1, self.bh = kb0, kb1, bh
        self.r0, self.r1 = kb0 * bh, kb1 * bh
        self.index, self.count = index, count
        u = full.u.reshape(dims)[self.r0:self.r1].ravel()
        low = LatticeLowering((self.r1 - self.r0,) + dims[1:], (kb1 - kb0,) + kpa[1:], full.conn,
                              full.lamw, np.ascontiguousarray(u), full.lam)
        dev = _device()
        self.problems = _Problems(low, dev)
        self.dev = _DeviceState(self.problems, mu, eps, max_iters, warm_start, skip_clean,
                                digests=digests)
        L = self.dev.L
        L.ghost_up = int(kb0 > 0)
        L.ghost_dn = int(kb1 < k0)
        L.sharded = 1
        L.fuse_multipliers = 1
        L.shard_index, L.shard_count = index, count
        self.unit = int(np.prod(dims[1:]))   # pixels per row (2D) / plane (3D)
        L.hash_base = self.r0 * self.unit
        lb = _lib.lib()
        halo_bytes = int(lb.dope_halo_bytes(C.byref(L)))
        agg_bytes = 2 * AGG_SLOT * count * 8     # two parity halves (peer mode alternates them)
        self._raw = []
        if ipc:   # CUDA IPC needs allocation bases: the library allocates them
            self.halo = self.agg = None
            for nbytes, field in ((halo_bytes, "halo"), (agg_bytes, "agg")):
                ptr = C.c_void_p()
                _lib.check(lb.dope_peer_alloc(nbytes, C.byref(ptr)), "dope_peer_alloc")
                self._raw.append(ptr)
                setattr(L, field, ptr.value)
        else:
            self.agg = torch.zeros(2 * AGG_SLOT * count, dtype=torch.int64, device=dev)
            L.agg = self.agg.data_ptr()
            self.halo = torch.zeros(halo_bytes, dtype=torch.uint8, device=dev)
            L.halo = self.halo.data_ptr()
        _lib.check(lb.dope_lattice_check(C.byref(L)), "dope_lattice_check (shard)")

    # -- step interface (run_shards) -----------------------------------------
    def call(self, name, *args):
        self.dev.call(name, *args)

    def init(self):
        self.call("dope_admm_init")

    def update_blocks(self):
        self.call("dope_update_blocks")

    def update_global(self):
        self.call("dope_update_global")

    def ghost_consensus(self):
        self.call("dope_ghost_consensus")

    def decide(self):
        self.call("dope_decide")

    def energy_local(self):
        self.call("dope_energy_local")

    def finish_decide(self):
        self.call("dope_finish_decide")

    def halo_slots(self):
        """(first row out, last row out, from above, from below) views of the halo buffer."""
        U = self.unit
        return tuple(self.halo[i * U:(i + 1) * U] for i in range(4))

    def pack_rows(self):
        first, last, _, _ = self.halo_slots()
        _lib.check(_lib.lib().dope_pack_rows(C.byref(self.dev.L), 0, first.data_ptr(), last.data_ptr(),
                                             self.dev.stream()), "dope_pack_rows")

    def install_rows(self):
        _, _, up, dn = self.halo_slots()
        L = self.dev.L
        _lib.check(_lib.lib().dope_ghost_update(C.byref(L), 0, up.data_ptr() if L.ghost_up else None,
                                                dn.data_ptr() if L.ghost_dn else None,
                                                self.dev.stream()), "dope_ghost_update")

    def labels(self):
        return self.dev.binarize()

    def __del__(self):
        for ptr in getattr(self, "_raw", []):
            _lib.lib().dope_peer_free(ptr)

    def digests(self):
        """Per-iteration (yhat, 2y, a) digests of this slab (global index base)."""
        it = self.dev.run_state().iteration
        return self.dev.trace_hash[:3 * it].cpu().numpy().view(np.uint64).reshape(it, 3)


class DistComm:
    """One shard per rank over torch.distributed (NCCL on GPUs, gloo on CPU)."""

    def __init__(self, group=None):
        import torch.distributed as dist
        self.dist = dist
        self.group = group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)

    def move_rows(self, shards):
        (s,) = shards
        first, last, up, dn = s.halo_slots()
        dist = self.dist
        ops = []
        if self.rank > 0:
            ops.append(dist.P2POp(dist.isend, first, self.rank - 1, self.group))
            ops.append(dist.P2POp(dist.irecv, up, self.rank - 1, self.group))
        if self.rank + 1 < self.world:
            ops.append(dist.P2POp(dist.isend, last, self.rank + 1, self.group))
            ops.append(dist.P2POp(dist.irecv, dn, self.rank + 1, self.group))
        if ops:
            for req in dist.batch_isend_irecv(ops):
                req.wait()

    def gather_agg(self, shards):
        import torch
        (s,) = shards
        table = s.agg[:AGG_SLOT * self.world].view(self.world, AGG_SLOT)   # the first half
        mine = table[self.rank].clone()
        parts = [torch.empty_like(mine) for _ in range(self.world)]
        self.dist.all_gather(parts, mine, group=self.group)
        table.copy_(torch.stack(parts))


def run_shards(shards, comm, max_iters: int):
    """The sharded run loop step by step (csrc/dope_comm.cu one_iteration)."""
    for s in shards:
        s.init()
    for _ in range(max_iters):
        for s in shards:
            s.update_blocks()
        for s in shards:
            s.pack_rows()
        comm.move_rows(shards)
        for s in shards:
            s.install_rows()
        for s in shards:
            s.update_global()
        for s in shards:
            s.ghost_consensus()
        comm.gather_agg(shards)
        for s in shards:
            s.decide()
    for s in shards:
        s.energy_local()
    comm.gather_agg(shards)
    for s in shards:
        s.finish_decide()


class LoopbackGroup:
    """All G shards of one grid in this process, on this GPU, run by the C++
    loopback communicator: the same iteration and graph capture as NCCL, each
    halo row moved by one cudaMemcpyAsync, each agg slot copied into every
    peer table -- or, with peer=True, the peer-memory exchange: the kernels
    store the rows and slots into the other shards' buffers themselves and
    wait on epoch flags (the multi-GPU IPC design, on one device)."""

    def __init__(self, shards, peer: bool = False):
        self.shards = list(shards)
        self.handle = C.c_void_p()
        self._arr = (C.POINTER(_lib.Lattice) * len(self.shards))(
            *[C.pointer(s.dev.L) for s in self.shards])
        if peer:
            peers = (C.c_void_p * len(self.shards))()
            _lib.check(_lib.lib().dope_comm_loopback_peer(len(self.shards), self._arr, C.byref(self.handle),
                                                          peers), "dope_comm_loopback_peer")
            for s, p in zip(self.shards, peers):
                s.dev.L.peers = p
        else:
            _lib.check(_lib.lib().dope_comm_loopback(len(self.shards), C.byref(self.handle)),
                       "dope_comm_loopback")

    def run(self, iters: int, use_graph: bool = True):
        lb = _lib.lib()
        for s in self.shards:
            s.init()
        st = self.shards[0].dev.stream()
        _lib.check(lb.dope_sharded_run_group(self._arr, len(self.shards), self.handle, iters,
                                             int(use_graph), st), "dope_sharded_run_group")
        _lib.check(lb.dope_sharded_finish_group(self._arr, len(self.shards), self.handle, st),
                   "dope_sharded_finish_group")

    def close(self):
        if self.handle:
            _lib.lib().dope_comm_destroy(self.handle)
            self.handle = C.c_void_p()


def _make_shards(model: EnergyModel, partition: Partition, config: AdmmConfig, world: int,
                 ranks, digests: bool = False):
    full = lower_lattice(model, partition)
    mu = _check_config(full, config)
    eps = config.resolved_eps(partition)
    slabs = shard_block_rows(full.kpa[0], world)
    return [GpuShard(full, slabs[r][0], slabs[r][1], mu, eps, config.max_iters, config.warm_start,
                     config.skip_clean, index=r, count=world, digests=digests) for r in ranks]


def run_virtual(model: EnergyModel, partition: Partition, config: AdmmConfig, shards: int,
                use_graph: bool = True, digests: bool = False, peer: bool = False):
    """`run` with the sub-regions sharded over `shards` loopback ranks on this GPU
    (peer: the peer-memory exchange instead of copies between kernels).

    Returns (labels, trace, state_fields) assembled from the shards."""
    sh = _make_shards(model, partition, config, shards, range(shards), digests)
    group = LoopbackGroup(sh, peer=peer)
    try:
        group.run(config.max_iters, use_graph)
        out = collect(sh, config.resolved_mu0(partition.shape.ndim), config)
    finally:
        group.close()
    if digests:
        tot = sh[0].digests().copy()
        for s in sh[1:]:
            tot += s.digests()
        out[2]["digests"] = tot
    return out


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
    a = torch.cat([s.dev.a for s in shards]).double().cpu().numpy()
    return labels, trace, {"iterations": it, "converged": bool(rs.converged),
                           "best_iteration": int(rs.best_iteration), "y": y, "yhat": yhat, "a": a}


class NcclComm:
    """NCCL communicator owned by libdope_b200 (one rank per GPU).

    The 128-byte unique id is created on rank 0 and broadcast with
    torch.distributed (any backend); the halo exchange and the agg all-gather
    then run inside dope_sharded_run's CUDA graph."""

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


class IpcPeerComm:
    """Peer-memory exchange across GPUs (one shard per rank): the shard's halo
    and agg buffers come from dope_peer_alloc, their CUDA IPC handles are
    all-gathered over torch.distributed, every rank opens the others' and the
    run loop's kernels store halo rows / agg slots into peer memory directly
    (DESIGN.md §7).  Use with shard_for_rank(..., cls=NcclShard, ipc=True)."""

    def __init__(self, shard: "GpuShard", group=None):
        import torch.distributed as dist
        lb = _lib.lib()
        L = shard.dev.L
        mine = (C.c_uint8 * 128)()
        _lib.check(lb.dope_peer_export(C.byref(L), mine), "dope_peer_export")
        world = L.shard_count
        allh = [bytes(mine)]
        if world > 1:
            allh = [None] * world
            dist.all_gather_object(allh, bytes(mine), group=group)
        buf = (C.c_uint8 * (128 * world))(*b"".join(allh))
        self.handle = C.c_void_p()
        peers = C.c_void_p()
        _lib.check(lb.dope_comm_peer_init(C.byref(L), buf, C.byref(self.handle), C.byref(peers)),
                   "dope_comm_peer_init")
        L.peers = peers.value

    def close(self):
        if self.handle:
            _lib.lib().dope_comm_destroy(self.handle)
            self.handle = C.c_void_p()


class NcclShard(GpuShard):
    """A GpuShard whose whole run loop (NCCL halo and gather included) is one CUDA graph."""

    def run(self, comm: NcclComm, iters: int, use_graph: bool = True):
        lb = _lib.lib()
        self.init()
        _lib.check(lb.dope_sharded_run(C.byref(self.dev.L), comm.handle, iters, int(use_graph),
                                       self.dev.stream()), "dope_sharded_run")
        _lib.check(lb.dope_sharded_finish(C.byref(self.dev.L), comm.handle, self.dev.stream()),
                   "dope_sharded_finish")


def shard_for_rank(model: EnergyModel, partition: Partition, config: AdmmConfig, rank: int,
                   world: int, cls=NcclShard, ipc: bool = False):
    full = lower_lattice(model, partition)
    mu = _check_config(full, config)
    kb0, kb1 = shard_block_rows(full.kpa[0], world)[rank]
    return cls(full, kb0, kb1, mu, config.resolved_eps(partition), config.max_iters,
               config.warm_start, config.skip_clean, index=rank, count=world, ipc=ipc)
