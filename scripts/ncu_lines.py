"""Aggregates an ncu source page (--page source --csv --print-source cuda,sass)
per CUDA source line: warp-stall samples and the top stall reasons.

usage: ncu -i rep --page source --csv --print-source cuda,sass > x.csv
       python scripts/ncu_lines.py x.csv [top]
"""
import csv
import sys


def main():
    path = sys.argv[1]
    top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
    rows, fname, header = [], None, None
    with open(path) as f:
        for rec in csv.reader(f):
            if not rec:
                continue
            if rec[0] == "File Path":
                fname = rec[1].rsplit("/", 1)[-1]
                header = None
                continue
            if rec[0] == "Function Name":
                continue
            if rec[0] == "Line No":
                header = rec
                continue
            if header is None or rec[1:3] == ["-", "-"] and False:
                continue
            if rec[2] != "-":  # sass rows carry an address; cuda rows have "-"
                continue
            d = dict(zip(header, rec))
            try:
                samples = int(d.get("Warp Stall Sampling (All Samples)", "0") or 0)
            except ValueError:
                continue
            stalls = {k: int(v) for k, v in zip(header, rec) if k.startswith("stall_") and v.isdigit() and int(v)}
            rows.append((samples, fname, rec[0], rec[1][:90], stalls))
    total = sum(r[0] for r in rows) or 1
    rows.sort(key=lambda r: -r[0])
    agg = {}
    for r in rows:
        for k, v in r[4].items():
            agg[k] = agg.get(k, 0) + v
    print("total samples", total)
    print("stalls:", ", ".join(f"{k}={v / total:.1%}" for k, v in sorted(agg.items(), key=lambda kv: -kv[1])[:8]))
    for s, fn, ln, src, st in rows[:top]:
        reasons = ", ".join(f"{k[6:]}={v}" for k, v in sorted(st.items(), key=lambda kv: -kv[1])[:3])
        print(f"{s / total:6.1%} {fn}:{ln:>4} {src:90s} {reasons}")


if __name__ == "__main__":
    main()
