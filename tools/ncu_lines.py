"""Per-source-line totals (instructions executed, stall samples) from an ncu
report captured with -lineinfo / --import-source (cuda,sass source view)."""
import csv
import collections
import subprocess
import sys


def main():
    rep = sys.argv[1]
    top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    agg = collections.defaultdict(lambda: [0.0, 0.0, ""])
    fname = ""
    hdr = None
    cur_line = None
    for r in rows:
        if len(r) >= 2 and r[0] == "File Path":
            fname = r[1].split("/")[-1]
            continue
        if r and r[0] == "Line No":
            hdr = r
            continue
        if hdr is None or len(r) < len(hdr):
            continue
        if r[0]:
            cur_line = (fname, int(r[0]), r[1])
        if cur_line is None or not r[2]:
            continue
        try:
            samples = float(r[hdr.index("Warp Stall Sampling (All Samples)")] or 0)
            inst = float(r[hdr.index("Instructions Executed")] or 0)
        except ValueError:
            continue
        a = agg[cur_line[:2]]
        a[0] += samples
        a[1] += inst
        a[2] = cur_line[2]
    tot_s = sum(v[0] for v in agg.values()) or 1
    tot_i = sum(v[1] for v in agg.values()) or 1
    print(f"total samples {tot_s:.0f}, instructions {tot_i:.3g}")
    for (f, ln), (s, i, src) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
        print(f"{100*s/tot_s:5.1f}% smp {100*i/tot_i:5.1f}% ins  {f}:{ln}  {src.strip()[:90]}")


if __name__ == "__main__":
    main()
