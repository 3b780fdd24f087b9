"""Small driver for ncu captures: builds a config, warms up, runs N solves.

usage: python scripts/prof_run.py [config] [solves] [--host]
"""
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

from paper_1612_06496_b200 import api  # noqa: E402
from paper_1612_06496_b200.inputs import make_config  # noqa: E402


def main():
    args = [a for a in sys.argv[1:] if not a.startswith("--")]
    name = args[0] if args else "c2"
    solves = int(args[1]) if len(args) > 1 else 1
    host = "--host" in sys.argv
    cfg = make_config(name)
    g, prm = cfg.graph, cfg.params
    y0 = api.random_embedding(g.n, prm.dim, cfg.y0_seed, g.degree)
    s = api.PfeSolver(g, prm, use_graphs=not host, warn=False)
    st = s.make_state(y0)
    for _ in range(solves):
        st.reset()
        s.run_soc(st, prm.soc_max, prm.sb_max_stage1)
    print(name, "ms", s.last_ms(), s.report())


if __name__ == "__main__":
    main()
