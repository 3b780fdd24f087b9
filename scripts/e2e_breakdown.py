"""Breakdown of the end-to-end call (solver create, state upload, solve,
download, destroy) for a config, repeated; prints mean milliseconds per stage.

usage: python scripts/e2e_breakdown.py [config] [reps]
"""
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "c2"
    reps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
    from paper_1612_06496_b200 import api
    from paper_1612_06496_b200.inputs import make_config

    cfg = make_config(name)
    g, prm = cfg.graph, cfg.params
    y0 = api.random_embedding(g.n, prm.dim, cfg.y0_seed, g.degree)
    api.soc(g, prm, y0)  # context + module load
    acc = {}
    for i in range(reps):
        t = [time.perf_counter()]
        s = api.PfeSolver(g, prm, warn=False)
        t.append(time.perf_counter())
        st = s.make_state(y0)
        t.append(time.perf_counter())
        s.run_soc(st, prm.soc_max, prm.sb_max_stage1)
        t.append(time.perf_counter())
        y = st.y
        t.append(time.perf_counter())
        del st, s
        t.append(time.perf_counter())
        for k, (a, b) in zip(["create", "state", "solve", "download", "destroy"], zip(t, t[1:])):
            acc.setdefault(k, []).append(1e3 * (b - a))
    for k, v in acc.items():
        print(f"{k:9s} {sum(v[1:]) / max(1, len(v) - 1):9.2f} ms (first {v[0]:.2f})")
    t0 = time.perf_counter()
    for _ in range(reps):
        api.soc(g, prm, y0)
    print(f"api.soc   {1e3 * (time.perf_counter() - t0) / reps:9.2f} ms")


if __name__ == "__main__":
    main()
