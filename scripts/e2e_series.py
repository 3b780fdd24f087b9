"""Per-call wall time of the one-call pfe_solve, repeated (drift check)."""
import sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_1612_06496_b200 import api
from paper_1612_06496_b200.inputs import make_config
name = sys.argv[1] if len(sys.argv) > 1 else "c1"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 30
cfg = make_config(name)
g, prm = cfg.graph, cfg.params
y0 = api.random_embedding(g.n, prm.dim, cfg.y0_seed, g.degree)
ts = []
for i in range(reps):
    t0 = time.perf_counter()
    api.soc(g, prm, y0)
    ts.append(1e3 * (time.perf_counter() - t0))
print(name, "ms per call:", " ".join(f"{t:.1f}" for t in ts))
