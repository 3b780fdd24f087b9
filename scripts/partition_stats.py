"""Per-PCG-iteration exchange volume of the multi-GPU partitions.

C5 (general 16-NN graph, vertex ranges in BFS storage order): owned / ghost /
sent rows per rank from the library's own partitioner
(pfe_range_partition_stats).  C3 / C4 (pixel grids, row bands): R halo rows
per band boundary.  Bytes per exchange = rows x d x 8.
usage: python scripts/partition_stats.py [c5 c4 c3] > gpurun_out/partition_stats.json
"""
import json
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_1612_06496_b200 import api  # noqa: E402
from paper_1612_06496_b200.inputs import make_config  # noqa: E402

out = {}
for name in (sys.argv[1:] or ["c5", "c4", "c3"]):
    cfg = make_config(name)
    g, d = cfg.graph, cfg.params.dim
    rec = {"n": g.n, "m": g.m, "d": d}
    for P in (2, 4, 8):
        if g.grid:
            h, w, r = g.grid
            rows = np.full(P, 2 * r * w)
            rows[0] = rows[-1] = r * w
            rec[f"P{P}"] = {"halo_rows_per_rank": rows.tolist(), "owned_rows": [g.n // P] * P,
                            "ghost_fraction_max": float(rows.max() / (g.n / P)),
                            "bytes_per_exchange_max": int(rows.max() * d * 8)}
        else:
            st = api.range_partition_stats(g, P)
            gf = st["ghosts"] / st["owned"]
            rec[f"P{P}"] = {"owned": st["owned"].tolist(), "ghosts": st["ghosts"].tolist(),
                            "sends": st["sends"].tolist(), "ghost_fraction": gf.round(4).tolist(),
                            "ghost_fraction_max": float(gf.max()),
                            "bytes_per_exchange_max": int(max(st["ghosts"].max(), st["sends"].max()) * d * 8)}
    out[name] = rec
    print(json.dumps({name: rec}), file=sys.stderr, flush=True)
print(json.dumps(out, indent=1))
