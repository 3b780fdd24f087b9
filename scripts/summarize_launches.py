"""Summarise an ncu launch list (CSV from --metrics ... --csv --log-file) per kernel.

usage: python scripts/summarize_launches.py launches.csv [n d m]
With n d m, prints algorithmic bytes / time per kernel (DESIGN.md §4 formulas).
"""
import collections
import csv
import sys


def main():
    path = sys.argv[1]
    nd = None
    if len(sys.argv) >= 5:
        n, d, m = map(int, sys.argv[2:5])
        nd = n * d
        alg = {"k_grid_pcg_spmv": 32 * nd + 8 * m + 16 * n, "k_pcg_spmv": 32 * nd + 8 * m + 16 * n,
               "k_pcg_update": 48 * nd + 8 * n, "k_grid_pcg_init": 32 * nd + 8 * m + 16 * n,
               "k_pcg_init": 32 * nd + 8 * m + 16 * n, "k_grid_sb_pass": 16 * m * d + 24 * nd + 8 * m,
               "k_sb_pass": 16 * m * d + 24 * nd + 8 * m}
    rows = list(csv.reader(open(path)))
    hdr, data = None, []
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            data.append(dict(zip(hdr, r)))
    agg = collections.defaultdict(lambda: collections.defaultdict(list))
    for d in data:
        name = d["Kernel Name"].split("(")[0].split("<")[0].replace("void ", "").replace("pfe_dev::", "").strip()
        agg[name][d["Metric Name"]].append(float(d["Metric Value"]))
    tot = sum(sum(v["gpu__time_duration.sum"]) for v in agg.values()) or 1.0
    print(f"{'kernel':24s} {'launches':>8s} {'avg_us':>9s} {'share':>6s} {'dram_MB':>9s} {'dram_GB/s':>9s} {'alg_GB/s':>9s}")
    for k, v in sorted(agg.items(), key=lambda x: -sum(x[1]["gpu__time_duration.sum"])):
        t = v["gpu__time_duration.sum"]
        avg = sum(t) / len(t)
        line = f"{k:24s} {len(t):8d} {avg / 1e3:9.2f} {sum(t) / tot:6.3f}"
        if v.get("dram__bytes_read.sum"):
            b = (sum(v["dram__bytes_read.sum"]) + sum(v["dram__bytes_write.sum"])) / len(t)
            line += f" {b / 1e6:9.1f} {b / avg:9.0f}"
        else:
            line += f" {'':9s} {'':9s}"
        if nd and k in alg:
            line += f" {alg[k] / avg:9.0f}"
        print(line)


if __name__ == "__main__":
    main()
