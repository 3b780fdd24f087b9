"""Device time of the projection (k_tsqr_local + k_tsqr_final + k_project_apply)
per outer iteration on a configuration (CUDA events, profile mode)."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_1612_06496_b200 import api, _native as N
from paper_1612_06496_b200.inputs import make_config
for name in sys.argv[1:] or ["c4"]:
    cfg = make_config(name)
    g, prm = cfg.graph, cfg.params
    y0 = api.random_embedding(g.n, prm.dim, cfg.y0_seed, g.degree)
    s = api.PfeSolver(g, prm, use_graphs=False, warn=False, profile=True, persistent=True)
    st = s.make_state(y0)
    s.run_soc(st, 2, 2)
    s.kernel_times(reset=True)
    s.run_soc(st, 2, 2)
    kt = s.kernel_times()
    print(name, {k: (round(v[0] / max(v[1], 1), 3), v[1]) for k, v in kt.items() if v[1]}, flush=True)
    st.close(); s.close()
