"""Markdown results table (README / DESIGN §10) from a bench_all.jsonl."""
import json
import sys


def main(path):
    print("| config | ADMM it/s | pixel-edges/s | e2e it/s (C ABI) | e2e it/s (public `run`) | "
          "dominant kernel, roofline frac | iteration roofline | CPU port it/s (16 thr) |")
    print("|---|---|---|---|---|---|---|---|")
    for line in open(path):
        if not line.startswith("{"):
            continue
        d = json.loads(line)
        name = d["config"]["workload"].split(":")[0]
        pub = d.get("e2e_public_api", {}).get("value")
        it = d.get("iteration_roofline", {}).get("frac_of_measured_hbm")
        r = d["roofline"]
        print(f"| {name} | {d['value']:,.0f} | {d['config']['pixel_edges_per_s']:.2g} | "
              f"{d['e2e']['value']:,.0f} | {'--' if pub is None else f'{pub:,.0f}'} | "
              f"{r.get('kernel', 'K1')} {r['frac']:.3f} | {'--' if it is None else f'{it:.2f}'} | "
              f"{d['cpu_baseline']['value']:.3g} |")


if __name__ == "__main__":
    main(sys.argv[1])
