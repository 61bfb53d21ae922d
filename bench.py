#!/usr/bin/env python
"""Benchmark of the DOPE hot path on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C3] [--impl b200|reference]

A "step" is one complete ADMM run of the workload from init_state (C3: the
4096^2 4-connected grid, 4096 sub-regions of 64^2, 100 iterations -- the grid
BASELINE.json's north star targets), inputs resident in HBM.  value =
ADMM iterations/s over the whole job; pixel-edges/s = E * iterations/s.
Prints ONE JSON line on rank 0.

--impl reference times the reference algorithm's CPU implementation (the
oracle's C port of the reference loop, all host threads) on a bounded sample
of the same workload -- the reference's own Python loop cannot leave the build
container (it is reported in DESIGN.md instead).
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

BYTES_PER_PIXEL_ITER = 21      # read u,a,y (int32), write a,y, yhat (1 B)


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=10)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--impl", default="b200", choices=["b200", "reference"])
    p.add_argument("--config", default="C3")
    p.add_argument("--iters", type=int, default=None, help="override ADMM iterations per run")
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--cpu-sample-iters", type=int, default=2)
    p.add_argument("--no-graph", action="store_true")
    p.add_argument("--sharded", action="store_true",
                   help="use the NCCL-sharded run loop even on one GPU (path check)")
    p.add_argument("--peer", action="store_true",
                   help="sharded loop with the peer-memory exchange (CUDA IPC) instead of NCCL")
    return p.parse_args()


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def measured_peaks():
    f = ROOT / "MEASURED_PEAKS.json"
    if f.exists():
        d = json.loads(f.read_text())
        return float(d["hbm_gbs"]), "measured"
    return 6650.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks / throttle reasons during the timed region."""

    def __init__(self, index: int):
        self.index = index
        self.rows = []
        self._stop = threading.Event()
        self._proc = None

    def start(self):
        q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        try:
            self._proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={q}", "--format=csv,noheader,nounits",
                 "-lms", "20"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self._proc = None
            return
        threading.Thread(target=self._read, daemon=True).start()

    def _read(self):
        for line in self._proc.stdout:
            if self._stop.is_set():
                break
            self.rows.append([x.strip() for x in line.split(",")])

    def stop(self):
        self._stop.set()
        if self._proc:
            self._proc.terminate()
            try:
                self._proc.wait(timeout=2)
            except Exception:
                self._proc.kill()

    def summary(self):
        sm = [float(r[0]) for r in self.rows if len(r) >= 7 and r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if len(r) >= 7 and r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = set()
        for r in self.rows:
            if len(r) >= 7:
                for nm, v in zip(names, r[3:7]):
                    if v.strip().lower() in ("active", "1"):
                        reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": sorted(reasons),
                "samples": len(self.rows)}


def kernel_bytes(wl, n, k_local, solves_per_iter, is_float):
    """Algorithmic bytes per launch of each kernel (DESIGN.md §4 states them).

    K1, per solved block (int): read u (4 B/px), multipliers (2), iterate (1)
    and the stored E/S residual planes (2); write labels (1) and the planes (2)
    = 12 B/px.  K2 (int): every pixel reads and writes its 1-byte iterate into
    the rotating buffer (2 B/px); a re-solved block additionally reads and
    writes its int16 multipliers and reads its labels (+5 B/px); the generic
    (non-TMA) consensus moves the full 7 B/px everywhere.  Float path (C2):
    f64 state, K1 = 44 B/px per solved block, K2 = 81 B/px.
    """
    bpx = n / max(k_local, 1)
    if is_float:
        return {"K1_block_mincut": 44.0 * bpx * solves_per_iter, "K2_consensus": 81.0 * n}
    bh, bw = wl.block[-2], wl.block[-1]
    tma = len(wl.block) == 2 and bw in (64, 128) and wl.dims[-1] % bw == 0 and wl.dims[0] % bh == 0
    k2 = 2.0 * n + 5.0 * bpx * solves_per_iter if tma else 7.0 * n
    return {"K1_block_mincut": 12.0 * bpx * solves_per_iter, "K2_consensus": k2}


def build_problem(wl, device, lower=True):
    """Lower the workload (validation happens once, outside timing)."""
    import paper_1704_03116_b200 as dope
    rows, cols, vals = wl.pair_arrays()
    model = dope.EnergyModel(wl.u.astype(np.float64), dope.SparseWeights(wl.n, rows, cols, vals),
                             wl.lam)
    del rows, cols, vals
    part = dope.make_partition(dope.GridShape(wl.dims), wl.kpa, 0, materialize=False)
    problems = dope.assemble_block_problems(model, part) if lower else None
    return model, part, problems


def cpu_model() -> str:
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def cpu_baseline(wl, iters: int, extras: bool = True):
    """Oracle C port of the reference loop on the host cores (bounded sample):
    `iters` iterations from init_state on all host threads; with extras, one
    iteration on ONE thread and the block solves of the first iteration alone
    (threads = 1 vs nproc, block-solve-only rate)."""
    sys.path.insert(0, str(ROOT / "oracle"))
    import oracle as orc
    threads = os.cpu_count() or 1
    spec = orc.LatticeSpec(wl.dims, wl.kpa, wl.offsets, wl.weights, wl.u.astype(np.float64), wl.lam)
    t0 = time.perf_counter()
    out = orc.run(spec, wl.rho, 1.0, 0.0, iters, threads=threads)
    dt = time.perf_counter() - t0
    res = {"value": out["iterations"] / dt, "unit": "iterations/s", "cores": threads,
           "kind": "port", "cpu_model": cpu_model(),
           "sample": f"{wl.name}: first {out['iterations']} ADMM iterations from init_state "
                     f"(oracle C port of admm.run + BK, {threads} threads), {dt:.1f} s"}
    if extras:
        t0 = time.perf_counter()
        one = orc.run(spec, wl.rho, 1.0, 0.0, 1, threads=1)
        res["threads_1"] = {"value": one["iterations"] / (time.perf_counter() - t0), "unit": "iterations/s",
                            "sample": "first ADMM iteration, 1 thread"}
        y = np.full(wl.n, 0.5)
        a = np.zeros(wl.n)
        t0 = time.perf_counter()
        orc.update_blocks(spec, y, a, wl.rho, threads=threads)
        res["block_solves_only"] = {"value": 1.0 / (time.perf_counter() - t0), "unit": "update_blocks/s",
                                    "sample": f"first iteration's {wl.num_blocks} block solves, {threads} threads"}
    return res


def is_general(wl) -> bool:
    return bool(wl.meta) and "overlap" in wl.meta


def general_model(wl):
    import paper_1704_03116_b200 as dope
    rows, cols, vals = wl.pair_arrays()
    model = dope.EnergyModel(np.asarray(wl.u, dtype=np.float64), dope.SparseWeights(wl.n, rows, cols, vals),
                             wl.lam)
    part = dope.make_partition(dope.GridShape(wl.dims), wl.kpa, int(wl.meta["overlap"]))
    return model, part


def cpu_baseline_general(wl, iters: int):
    """General-path oracle (numpy + the oracle's BK, one host thread) on a
    bounded sample: the first `iters` iterations of the same workload."""
    sys.path.insert(0, str(ROOT / "oracle"))
    import general as og
    from paper_1704_03116_b200.lowering import lattice_planes
    model, _ = general_model(wl)
    planes, conn = lattice_planes(model, wl.dims)
    spec = og.GeneralSpec(wl.dims, conn, wl.u, planes, wl.lam, wl.kpa, int(wl.meta["overlap"]))
    t0 = time.perf_counter()
    out = og.run(spec, wl.meta["mu0"], wl.meta["mu_fact"], 0.0, iters)
    dt = time.perf_counter() - t0
    return {"value": out["iterations"] / dt, "unit": "iterations/s", "cores": 1, "kind": "port",
            "sample": f"{wl.name}: first {out['iterations']} ADMM iterations from init_state "
                      f"(general-path oracle: numpy stencil + BK restatement, 1 thread), {dt:.1f} s"}


def run_general_bench(args, wl):
    """One GPU, general path (overlap + growing mu): same contract fields."""
    import torch
    from paper_1704_03116_b200.general import GeneralDevice, lower_general
    iters = args.iters or wl.iters
    model, part = general_model(wl)
    low = lower_general(model, part)
    gd = GeneralDevice(low, wl.meta["mu0"], wl.meta["mu_fact"], 0.0, iters)
    use_graph = not args.no_graph

    def step():
        gd.init()
        gd.run(iters, use_graph)
        gd.finish()

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    rs = gd.run_state()
    iters_done = int(rs.iteration)
    sampler = ClockSampler(0)
    sampler.start()
    t_wait = time.time()
    while not sampler.rows and time.time() - t_wait < 5.0:
        step()
        torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(args.steps):
        step()
    e1.record()
    torch.cuda.synchronize()
    sampler.stop()
    ms = e0.elapsed_time(e1)
    value = iters_done * args.steps / (ms / 1e3)
    # per-kernel timing (eager launches on the stream)
    gd.init()
    kt = {"K1_block_mincut": [], "K2_consensus": []}
    stream = torch.cuda.current_stream()
    for _ in range(iters_done):
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
        ev[0].record(stream)
        gd.step_blocks()
        ev[1].record(stream)
        gd.step_global()
        ev[2].record(stream)
        kt["K1_block_mincut"].append(ev)
    torch.cuda.synchronize()
    k1 = [e[0].elapsed_time(e[1]) for e in kt["K1_block_mincut"]]
    k2 = [e[1].elapsed_time(e[2]) for e in kt["K1_block_mincut"]]
    ncopy = sum(b.size for b in part.blocks)
    n = low.n
    nd = low.conn
    # algorithmic bytes (general path): K1 per copy pixel: u, y, a
    # (f64) + q + weights (8 B per direction pair, 2 directions per pair) +
    # residual planes r/w (4 B x conn x 2) + label; global step per pixel: the
    # copies' labels and multipliers (q x 9 B), weights, u, q, y out, and per
    # copy the multiplier update (r/w 16 B) + residual, energy pass (y, u, w)
    k1b = ncopy * (8 + 8 + 8 + 1 + 4 * nd + 8 * nd + 1)
    k2b = ncopy * (9 + 16 + 1) + n * (8 + 1 + 4 * nd + 8 + 8 + 8 + 4 * nd)
    kstat = {}
    for name, v, b in (("K1_block_mincut", k1, k1b), ("K2_consensus", k2, k2b)):
        kstat[name] = {"total_ms": sum(v), "avg_ms": sum(v) / len(v), "launches": len(v),
                       "median_ms": statistics.median(v), "algorithmic_bytes_per_launch": b,
                       "achieved_GBps": b / (sum(v) / len(v) / 1e3) / 1e9}
    dom = max(kstat, key=lambda k: kstat[k]["total_ms"])
    peak, peak_kind = measured_peaks()
    roof = {"bound": "hbm", "achieved": kstat[dom]["achieved_GBps"], "peak": peak, "unit": "GB/s",
            "frac": kstat[dom]["achieved_GBps"] / peak, "traffic": None, "kernel": dom,
            "peak_source": f"MEASURED_PEAKS.json hbm_gbs ({peak_kind})",
            "algorithmic_bytes_per_launch": kstat[dom]["algorithmic_bytes_per_launch"]}
    # e2e: unaries and weights from pinned host memory, labels + trace back
    e2e = None
    if not args.no_e2e:
        u_host = gd.u.cpu().pin_memory()
        w_host = [w.cpu().pin_memory() for w in gd.w]
        lab = torch.empty(n, dtype=torch.uint8).pin_memory()
        trh = torch.empty(iters, dtype=torch.float64).pin_memory()
        hb = u_host.numel() * 8 + sum(w.numel() * 8 for w in w_host)
        for s in range(args.warmup + args.steps):
            if s == args.warmup:
                torch.cuda.synchronize()
                f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                f0.record()
            gd.u.copy_(u_host, non_blocking=True)
            for wd, wh in zip(gd.w, w_host):
                wd.copy_(wh, non_blocking=True)
            step()
            lab.copy_(gd.binarize(), non_blocking=True)
            trh.copy_(gd.tr["e"], non_blocking=True)
        f1.record()
        torch.cuda.synchronize()
        e2e = {"value": iters_done * args.steps / (f0.elapsed_time(f1) / 1e3), "unit": "iterations/s",
               "h2d_bytes_per_step": hb, "d2h_bytes_per_step": n + 8 * iters}
    line = {"metric": "ADMM iterations/s", "value": value, "unit": "iterations/s", "n_gpus": 1,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic",
            "config": {"workload": f"{wl.name}: {wl.dims[0]}x{wl.dims[1]} {nd}-connected contrast-weighted "
                                   f"Potts, {part.k} sub-regions of {wl.block[0]}x{wl.block[1]} grown by "
                                   f"{wl.meta['overlap']} % (q in {{1,2,4}}), mu0 {wl.meta['mu0']}, "
                                   f"mu_fact {wl.meta['mu_fact']}, {iters_done} ADMM iterations per step",
                       "pixel_edges_per_s": value * wl.num_pairs, "path": "general (overlap, growing mu)",
                       "l2": "state fits in the 126 MB L2 (no flush between steps)",
                       "parallelism": "1 GPU", "kernels": kstat},
            "roofline": roof, "clocks": sampler.summary(),
            "gpu_launches": (5 * iters_done + 4) * args.steps}
    if e2e:
        line["e2e"] = e2e
    if not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline_general(wl, args.cpu_sample_iters)
    print(json.dumps(line), flush=True)


def run_reference(args):
    ws, rank, _ = dist_env()
    if rank != 0:
        return
    from paper_1704_03116_b200 import workloads as W
    wl = W.by_name(args.config)
    iters = max(1, args.cpu_sample_iters)
    vals = []
    for s in range(args.warmup + args.steps):
        r = cpu_baseline_general(wl, iters) if is_general(wl) else cpu_baseline(wl, iters, extras=False)
        if s >= args.warmup:
            vals.append(r["value"])
    v = statistics.mean(vals)
    line = {"metric": "ADMM iterations/s", "value": v, "unit": "iterations/s", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * iters / v,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "impl": "reference",
            "config": {"workload": f"{wl.name} {wl.dims[0]}x{wl.dims[1]} {wl.conn}-conn, "
                                   f"{wl.num_blocks} sub-regions of {wl.block[0]}x{wl.block[1]}; "
                                   f"each step = first {iters} iterations",
                       "pixel_edges_per_s": v * wl.num_pairs},
            "cpu_baseline": {**r, "value": v},
            "e2e": {"value": v, "unit": "iterations/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)
    import torch
    import torch.distributed as dist
    ws, rank, local = dist_env()
    torch.cuda.set_device(local)
    if ws > 1:
        dist.init_process_group("nccl", init_method="env://")
    from paper_1704_03116_b200 import workloads as W
    from paper_1704_03116_b200.admm import make_device_state
    wl = W.by_name(args.config)
    if is_general(wl):
        if ws > 1:
            raise SystemExit("the general-path bench runs on one GPU")
        return run_general_bench(args, wl)
    iters = args.iters or wl.iters
    use_graph = int(not args.no_graph)
    if args.peer:
        args.sharded = True
    if ws == 1 and not args.sharded:
        model, part, problems = build_problem(wl, torch.device("cuda", local))
        dev = make_device_state(problems, wl.rho, 0.0, iters, True, True)

        def step():
            dev.call("dope_admm_init")
            dev.call("dope_admm_run", iters, use_graph, fuse=1)
            dev.call("dope_finish_run")
    else:
        # strong scaling: ONE grid, its block rows sharded over the ranks; halos and
        # the 4-scalar all-reduce run over NCCL inside one CUDA graph per run
        import paper_1704_03116_b200 as dope
        from paper_1704_03116_b200 import sharded
        model, part, _ = build_problem(wl, torch.device("cuda", local), lower=False)
        cfg = dope.AdmmConfig(mu0=wl.rho, mu_fact=1.0, eps=0.0, max_iters=iters)
        if ws == 1 and not dist.is_initialized():
            os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
            os.environ.setdefault("MASTER_PORT", "29533")
            dist.init_process_group("nccl", rank=0, world_size=1)
        if args.peer:
            shard = sharded.shard_for_rank(model, part, cfg, rank, ws, ipc=True)
            comm = sharded.IpcPeerComm(shard)
        else:
            comm = sharded.NcclComm(rank, ws)
            shard = sharded.shard_for_rank(model, part, cfg, rank, ws)
        dev = shard.dev
        problems = shard.problems

        def step():
            shard.run(comm, iters, bool(use_graph))

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    rs = dev.raise_on_error()
    iters_done = rs.iteration

    sampler = ClockSampler(local)
    sampler.start()
    t_wait = time.time()
    while not sampler.rows and time.time() - t_wait < 5.0:   # sampler running before timing
        step()
        torch.cuda.synchronize()
    if ws > 1:
        dist.barrier()
    torch.cuda.synchronize()
    t_start = torch.cuda.Event(enable_timing=True)
    t_end = torch.cuda.Event(enable_timing=True)
    t_start.record()
    for _ in range(args.steps):
        step()
    t_end.record()
    torch.cuda.synchronize()
    if ws > 1:
        dist.barrier()
    sampler.stop()
    ms = t_start.elapsed_time(t_end)
    rs = dev.raise_on_error()
    assert rs.iteration == iters_done
    if ws > 1:
        t = torch.tensor([ms], device="cuda", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    # one grid (sharded over the ranks when ws > 1): iterations of that grid per second
    total_iters = iters_done * args.steps
    value = total_iters / (ms / 1e3)
    n_local = problems.lowering.n
    solves_per_run = rs.solves
    sweeps_per_run = rs.sweeps

    # ---- per-kernel timing pass (CUDA events on the launching stream) ----
    evs = {"K1_block_mincut": [], "K2_consensus": []}
    shard_mode = ws > 1 or args.sharded
    if shard_mode:
        dev.L.sharded = 0            # kernel timing on this rank's slab alone (no halos)
    dev.call("dope_admm_init")
    stream = torch.cuda.current_stream()
    for it in range(iters_done):
        e = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
        e[0].record(stream)
        dev.call("dope_update_blocks")
        e[1].record(stream)
        dev.call("dope_update_global", fuse=1)      # + fused finalize (last CTA)
        e[2].record(stream)
        evs["K1_block_mincut"].append((e[0], e[1]))
        evs["K2_consensus"].append((e[1], e[2]))
    torch.cuda.synchronize()
    kern = {k: [a.elapsed_time(b) for a, b in v] for k, v in evs.items()}
    if shard_mode:
        dev.L.sharded = 1
    kstat = {k: {"total_ms": sum(v), "avg_ms": sum(v) / len(v), "launches": len(v),
                 "first3_ms": v[:3], "median_ms": statistics.median(v)}
             for k, v in kern.items()}
    dom = max(kstat, key=lambda k: kstat[k]["total_ms"])
    peak, peak_kind = measured_peaks()
    n = n_local
    k_local = problems.lowering.K
    is_float = getattr(problems, "kind", "int") == "float"
    alg = kernel_bytes(wl, n, k_local, solves_per_run / max(iters_done, 1), is_float)
    for kname, st_ in kstat.items():   # per-kernel roofline beside the timings
        st_["algorithmic_bytes_per_launch"] = alg[kname]
        st_["achieved_GBps"] = alg[kname] / (st_["avg_ms"] / 1e3) / 1e9
    alg_bytes = alg[dom]
    achieved = alg_bytes / (kstat[dom]["avg_ms"] / 1e3) / 1e9
    traffic = None
    tfile = ROOT / "profiles" / "ncu_traffic.json"
    if tfile.exists():
        tj = json.loads(tfile.read_text())
        key = f"{wl.name}:{dom}"
        if key in tj:
            traffic = tj[key]["traffic_bytes"]
    roof = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
            "frac": achieved / peak, "traffic": traffic,
            "traffic_source": "profiles/ncu_traffic.json (ncu --set full, one launch)" if traffic else None,
            "kernel": dom,
            "peak_source": f"MEASURED_PEAKS.json hbm_gbs ({peak_kind})",
            "algorithmic_bytes_per_launch": alg_bytes}
    # 21 B/pixel (+ 4 B per stored non-constant-weight pair on float configs)
    iter_bytes = BYTES_PER_PIXEL_ITER * n + (4 * wl.num_pairs * n // wl.n if is_float else 0)
    iter_roof = {"bytes_per_iteration_per_gpu": iter_bytes,
                 "achieved_GBps_per_gpu": iter_bytes * value / 1e9,
                 "frac_of_measured_hbm": iter_bytes * value / 1e9 / peak,
                 "formula": "(21 B/pixel + 4 B/float-weight pair)/iteration (SURVEY 8(d)) x "
                            "pixels per GPU x iterations/s"}

    # ---- e2e through the C ABI with host buffers ----
    e2e = None
    if not args.no_e2e and ws == 1 and not args.sharded:
        # production pipelining: every step copies its unaries from pinned
        # host memory and reads its labels + trace back, but the copies run
        # on a second stream behind / ahead of the previous / next step's
        # solve (double-buffered device inputs and outputs)
        import ctypes as C
        from paper_1704_03116_b200 import _lib
        u_host = problems.u.cpu().pin_memory()
        u_bytes = u_host.numel() * u_host.element_size()
        U = [problems.u, torch.empty_like(problems.u)]
        lab_dev = [torch.empty(n, dtype=torch.uint8, device=problems.u.device) for _ in range(2)]
        tr_dev = [torch.empty_like(dev.tr_e) for _ in range(2)]
        lab_host = [torch.empty(n, dtype=torch.uint8).pin_memory() for _ in range(2)]
        tr_host = [torch.empty(dev.tr_e.numel(), dtype=dev.tr_e.dtype).pin_memory() for _ in range(2)]
        # both on non-default streams: the legacy default stream would
        # serialise with the copy stream
        comp = torch.cuda.Stream()
        cs = torch.cuda.Stream()        # host -> device
        co = torch.cuda.Stream()        # device -> host (its own queue: a D2H waiting
        comp.wait_stream(torch.cuda.current_stream())   # for a solve must not hold up the next H2D)
        used = [torch.cuda.Event() for _ in range(2)]     # compute on buffer i finished
        ready = [torch.cuda.Event() for _ in range(2)]    # input copy into buffer i finished
        fetched = [torch.cuda.Event() for _ in range(2)]  # results of buffer i are on the host
        lb = _lib.lib()
        binarize = lb.dope_f_binarize if is_float else lb.dope_binarize
        total = args.warmup + args.steps

        def h2d(i, first):
            with torch.cuda.stream(cs):
                if not first:
                    cs.wait_event(used[i])
                U[i].copy_(u_host, non_blocking=True)
                ready[i].record(cs)

        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        h2d(0, True)
        for s in range(total):
            i = s % 2
            if s == args.warmup:
                torch.cuda.synchronize()
                e0.record(comp)
                h2d(i, True)            # this step's copy inside the timed region
            comp.wait_event(ready[i])
            if s >= 2:
                comp.wait_event(fetched[i])   # output buffers i are free again
            dev.L.u = U[i].data_ptr()
            with torch.cuda.stream(comp):
                step()
                _lib.check(binarize(C.byref(dev.L), lab_dev[i].data_ptr(), C.c_void_p(comp.cuda_stream)),
                           "binarize")
                tr_dev[i].copy_(dev.tr_e)
            used[i].record(comp)
            with torch.cuda.stream(co):
                co.wait_event(used[i])
                lab_host[i].copy_(lab_dev[i], non_blocking=True)
                tr_host[i].copy_(tr_dev[i], non_blocking=True)
                fetched[i].record(co)
            if s + 1 < total and s + 1 != args.warmup:
                h2d((s + 1) % 2, False)   # next step's input overlaps this solve
        comp.wait_stream(cs)
        comp.wait_stream(co)
        e1.record(comp)
        torch.cuda.synchronize()
        torch.cuda.current_stream().wait_stream(comp)
        dev.L.u = problems.u.data_ptr()
        ms_e2e = e0.elapsed_time(e1)
        e2e = {"value": iters_done * args.steps / (ms_e2e / 1e3), "unit": "iterations/s",
               "h2d_bytes_per_step": u_bytes, "d2h_bytes_per_step": n + 8 * iters,
               "pipelining": "double-buffered: step s+1's H2D and step s's D2H on copy streams "
                             "overlap the solves"}
    elif not args.no_e2e:
        u_host = problems.u.cpu().pin_memory()
        u_bytes = u_host.numel() * u_host.element_size()
        lab_host = torch.empty(n, dtype=torch.int8).pin_memory()
        tr_host = torch.empty(iters, dtype=torch.int64).pin_memory()
        for s in range(args.warmup + args.steps):
            if s == args.warmup:
                torch.cuda.synchronize()
                if ws > 1:
                    dist.barrier()
                e0 = torch.cuda.Event(enable_timing=True)
                e1 = torch.cuda.Event(enable_timing=True)
                e0.record()
            problems.u.copy_(u_host, non_blocking=True)
            step()
            lab_host.copy_(dev.binarize().view(torch.int8), non_blocking=True)
            tr_host.copy_(dev.tr_e, non_blocking=True)
        e1.record()
        torch.cuda.synchronize()
        ms_e2e = e0.elapsed_time(e1)
        if ws > 1:
            t = torch.tensor([ms_e2e], device="cuda", dtype=torch.float64)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ms_e2e = float(t.item())
        e2e = {"value": iters_done * args.steps / (ms_e2e / 1e3), "unit": "iterations/s",
               "h2d_bytes_per_step": u_bytes, "d2h_bytes_per_step": n + 8 * iters}

    # ---- e2e through the reference-named public API: run(model, part, cfg) ----
    # host numpy float64 unary in, numpy labels + trace out, every step; the
    # weights / partition objects repeat, so run() reuses the lowering and the
    # device buffers and only uploads (and checks, on the device) the unary
    e2e_public = None
    if not args.no_e2e and ws == 1 and not args.sharded:
        import paper_1704_03116_b200 as dope
        cfgp = dope.AdmmConfig(mu0=wl.rho, mu_fact=1.0, eps=0.0, max_iters=iters,
                               use_graph=bool(use_graph))
        u_np = np.ascontiguousarray(wl.u, dtype=np.float64)

        def pstep():
            return dope.run(dope.EnergyModel(u_np, model.weights, wl.lam), part, cfgp)

        # the first calls lower the model, capture the graph and register the
        # host buffers (C5-b16: 1548, 22, 11 ms, then 4.6 ms per call)
        for _ in range(max(4, args.warmup + 1)):
            pstep()
        torch.cuda.synchronize()
        p0, p1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        p0.record()
        for _ in range(args.steps):
            lab_p, st_p = pstep()
        p1.record()
        torch.cuda.synchronize()
        assert st_p.iteration == iters_done
        e2e_public = {"value": iters_done * args.steps / (p0.elapsed_time(p1) / 1e3), "unit": "iterations/s",
                      "h2d_bytes_per_step": u_np.nbytes, "d2h_bytes_per_step": n + 4 * 8 * iters,
                      "call": "paper_1704_03116_b200.run(EnergyModel(u_host_f64, weights, lam), partition, "
                              "AdmmConfig(...)) -> (labels numpy, AdmmState with trace), synchronous"}

    # quality of the answer (BASELINE configs[4]: final energy vs block size):
    # the returned labeling's energy (best iterate) against the whole-grid
    # serial min cut of compare mode (cli.py:95-100), both on the device
    quality = None
    if rank == 0 and ws == 1 and not args.sharded and len(wl.dims) == 2 and wl.integer:
        import paper_1704_03116_b200 as dope
        from paper_1704_03116_b200 import compare
        e_best = float(rs.best_energy)
        _, e_serial, _ = compare.run_serial(model, dope.GridShape(wl.dims))
        quality = {"energy_returned": e_best, "best_iteration": int(rs.best_iteration),
                   "serial_cut_energy": e_serial,
                   "relative_energy_diff_pct": compare.relative_energy_diff(e_serial, e_best)}

    cpu = None
    if rank == 0 and ws == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline(wl, args.cpu_sample_iters)

    if rank == 0:
        line = {
            "metric": "ADMM iterations/s", "value": value, "unit": "iterations/s",
            "n_gpus": ws, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": ms / args.steps, "higher_is_better": True,
            "scaling": "strong" if ws > 1 else "weak",
            "vs_baseline": None, "dtype": "f64" if is_float else "int32", "data": "synthetic",
            "config": {"workload": f"{wl.name}: {'x'.join(map(str, wl.dims))} {wl.conn}-connected "
                                   f"{'contrast-weighted' if is_float else 'constant-weight'} Potts, "
                                   f"{wl.num_blocks} sub-regions of {'x'.join(map(str, wl.block))}, "
                                   f"{iters_done} ADMM iterations per step (full run from init)",
                       "pixel_edges_per_s": value * wl.num_pairs,
                       "l2": ("inputs larger than L2 (state > 126 MB)" if wl.n * 21 > 126e6 else
                              "state fits in the 126 MB L2 (small config; no flush between steps)"),
                       "parallelism": (f"{ws} GPU(s): block {'planes' if len(wl.dims) == 3 else 'rows'} "
                                       f"sharded in slabs; per iteration one label-halo exchange and one "
                                       f"64-byte agg gather "
                                       + ("by peer-memory stores inside the kernels (CUDA IPC)" if args.peer
                                          else "over NCCL") + ", captured in one CUDA graph"
                                       if (ws > 1 or args.sharded) else "1 GPU"),
                       "block_solves_per_run": solves_per_run,
                       "push_relabel_sweeps_per_run": sweeps_per_run,
                       "kernels": kstat},
            "roofline": roof, "iteration_roofline": iter_roof,
            "clocks": sampler.summary(), "gpu_launches": ((2 * iters_done + 3) if ws == 1 else (8 * iters_done + 6)) * args.steps,
        }
        if e2e:
            line["e2e"] = e2e
        if e2e_public:
            line["e2e_public_api"] = e2e_public
        if quality:
            line["config"]["quality"] = quality
        if cpu:
            line["cpu_baseline"] = cpu
        print(json.dumps(line), flush=True)
    if dist.is_initialized():
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
