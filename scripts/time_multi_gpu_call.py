"""Wall time of the one-call multi-GPU entry point (pfe_solve_multi_gpu) on the
visible GPUs against the one-call single-GPU pfe_solve, same configuration."""
import sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
from paper_1612_06496_b200 import api
from paper_1612_06496_b200.inputs import make_config
name = sys.argv[1] if len(sys.argv) > 1 else "c4"
cfg = make_config(name)
g, prm = cfg.graph, cfg.params
y0 = api.random_embedding(g.n, prm.dim, cfg.y0_seed, g.degree)
devs = list(range(torch.cuda.device_count()))
for rep in range(2):
    t0 = time.perf_counter(); y, ms = api.soc_multi_gpu(g, prm, y0, devs, return_ms=True); t1 = time.perf_counter()
    print(f"{name} pfe_solve_multi_gpu on {len(devs)} GPU(s): wall {t1 - t0:.2f} s, device {ms / 1e3:.2f} s", flush=True)
    t0 = time.perf_counter(); y1 = api.soc(g, prm, y0); t1 = time.perf_counter()
    print(f"{name} pfe_solve (single GPU, persistent): wall {t1 - t0:.2f} s", flush=True)
