"""Writes a profiles/ summary of one ncu capture: key raw metrics per launch
plus the per-line warp-stall table (scripts/ncu_lines.py output).

usage: python scripts/ncu_summary.py raw.csv lines.txt out.txt "header line" ["header line" ...]
"""
import csv
import sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed", "launch__block_size", "launch__grid_size",
        "launch__registers_per_thread", "launch__shared_mem_per_block_dynamic", "lts__t_sector_hit_rate.pct",
        "l1tex__t_sector_hit_rate.pct", "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed", "smsp__inst_executed.sum"]


def main():
    raw, lines, out = sys.argv[1:4]
    rows = list(csv.reader(open(raw)))
    hdr, units = rows[0], rows[1]
    with open(out, "w") as f:
        for h in sys.argv[4:]:
            f.write(f"# {h}\n")
        for r in rows[2:]:
            f.write(f"\n{r[hdr.index('Kernel Name')]}\n")
            for k in KEYS:
                if k in hdr:
                    i = hdr.index(k)
                    f.write(f"{k:<80s} {r[i]:>16s} {units[i]}\n")
        f.write("\n# warp-stall samples per CUDA source line (scripts/ncu_lines.py)\n")
        f.write(open(lines).read())


if __name__ == "__main__":
    main()
