"""Summarise ncu captures into profiles/ (run here, on the CPU box).

    python tools/ncu_summary.py <tag> <launches.csv> <full1.ncu-rep> [<full2.ncu-rep> ...]

Writes profiles/<tag>_ncu.md (launch-list shares + per-kernel full-set
metrics) and profiles/ncu_traffic.json (DRAM bytes per launch of each profiled
kernel, read by bench.py for roofline.traffic).
"""
import collections
import csv
import json
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
WANT = ["Duration", "DRAM Throughput", "Memory Throughput", "Executed Ipc Active",
        "Issue Slots Busy", "Achieved Occupancy", "Theoretical Occupancy", "Registers Per Thread",
        "Block Size", "Grid Size", "Dynamic Shared Memory Per Block",
        "Warp Cycles Per Issued Instruction", "Executed Instructions", "L2 Hit Rate"]
RAW = ["dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__time_duration.sum",
       "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
       "smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio",
       "smsp__average_warps_issue_stalled_wait_per_issue_active.ratio",
       "smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio",
       "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum"]


def ncu_csv(rep, page):
    out = subprocess.run(["ncu", "-i", str(rep), "--page", page, "--csv"], capture_output=True,
                         text=True, check=True).stdout
    return list(csv.reader(out.splitlines()))


def launches(path):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    hdr, data = rows[hi], rows[hi + 1:]
    ki, mi, vi, ii = (hdr.index(x) for x in ("Kernel Name", "Metric Name", "Metric Value", "ID"))
    per = collections.defaultdict(dict)
    for r in data:
        if len(r) <= vi:
            continue
        per[int(r[ii])][r[mi]] = float(r[vi].replace(",", ""))
        per[int(r[ii])]["name"] = r[ki]
    agg = collections.defaultdict(lambda: [0, 0.0, 0.0])
    for d in per.values():
        n = d["name"].split("(")[0].replace("void ", "")
        a = agg[n]
        a[0] += 1
        a[1] += d.get("gpu__time_duration.sum", 0.0)
        a[2] += d.get("dram__bytes_read.sum", 0.0) + d.get("dram__bytes_write.sum", 0.0)
    return agg


def main():
    tag, lcsv, reps = sys.argv[1], sys.argv[2], sys.argv[3:]
    workload = tag.split("_")[-1] if "_" in tag else "C3"   # e.g. r1_C3
    lines = [f"# ncu summary `{tag}`", "",
             "Captured on one B200 with `ncu --clock-control none` (launch list: "
             "`--metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum`; "
             f"per-kernel: `--set full --import-source on`), driver `tools/profile_round.sh` (launch list: the bench command itself; full sets: `tools/prof_run.py {workload} 20`, launch 8) "
             "(prof_run launches one kernel at a time, no CUDA graph).  "
             "ncu serialises launches and flushes caches, so compare SHARES, not absolutes.", "",
             "## Launch list", "", "| kernel | launches | total us | share | avg us | DRAM MB/launch |",
             "|---|---|---|---|---|---|"]
    agg = launches(lcsv)
    tot = sum(a[1] for a in agg.values())
    for n, a in sorted(agg.items(), key=lambda t: -t[1][1]):
        lines.append(f"| `{n}` | {a[0]} | {a[1] / 1e3:.1f} | {100 * a[1] / tot:.1f}% | "
                     f"{a[1] / a[0] / 1e3:.1f} | {a[2] / a[0] / 1e6:.1f} |")
    traffic = {}
    for rep in reps:
        det = ncu_csv(rep, "details")
        hdr = det[0]
        kname = None
        vals = {}
        for row in det[1:]:
            d = dict(zip(hdr, row))
            kname = d.get("Kernel Name", kname)
            if d.get("Metric Name") in WANT:
                vals[d["Metric Name"]] = f"{d['Metric Value']} {d['Metric Unit']}".strip()
        raw = ncu_csv(rep, "raw")
        h, un, v = raw[0], raw[1], raw[2]
        rv = {k: x for k, x in zip(h, v) if k in RAW}
        units = {k: x for k, x in zip(h, un) if k in RAW}
        lines += ["", f"## `{Path(rep).name}` -- {kname}", "", "| metric | value |", "|---|---|"]
        for k in WANT:
            if k in vals:
                lines.append(f"| {k} | {vals[k]} |")
        for k in RAW:
            if k in rv:
                lines.append(f"| `{k}` | {rv[k]} {units.get(k, '')} |")
        try:
            rd = float(rv["dram__bytes_read.sum"])
            wr = float(rv["dram__bytes_write.sum"])
            scale = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
            rd *= scale[units["dram__bytes_read.sum"]]
            wr *= scale[units["dram__bytes_write.sum"]]
            unit_scale = 1.0
            key = "K2_consensus" if "consensus" in (kname or "") else (
                "K1_block_mincut" if "mincut" in (kname or "") else kname)
            traffic[f"{workload}:{key}"] = {"dram_read_bytes": rd * unit_scale, "dram_write_bytes": wr * unit_scale,
                            "traffic_bytes": (rd + wr) * unit_scale, "source": f"profiles/{tag}_ncu.md",
                            "kernel": kname}
        except (KeyError, ValueError):
            pass
    out = ROOT / "profiles" / f"{tag}_ncu.md"
    out.write_text("\n".join(lines) + "\n")
    tj = ROOT / "profiles" / "ncu_traffic.json"
    old = json.loads(tj.read_text()) if tj.exists() else {}
    old.update(traffic)
    tj.write_text(json.dumps(old, indent=1) + "\n")
    print(out, tj)


if __name__ == "__main__":
    main()
