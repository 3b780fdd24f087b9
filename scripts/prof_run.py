"""Small driver for ncu captures and phase traces: builds a config, runs N solves.

usage: python scripts/prof_run.py [config] [solves] [--host] [--multi] [--trace]
  --host   host-driven multi-kernel path (ncu can profile each kernel)
  --multi  one kernel per phase (CUDA graph) instead of the persistent kernel
  --trace  per-phase time breakdown of the last persistent launch (PFE_TRACE)
"""
import ctypes as C
import os
import sys
from collections import defaultdict
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

PHASES = {1: "init", 3: "spmv", 5: "update", 6: "finalize", 8: "sb_pass",
          # fine-grained points of the resident kernel (end of each sub-step)
          10: "beta_red", 11: "p_dir", 12: "q_Ap", 13: "x_r_upd", 14: "alpha_red"}


def main():
    args = [a for a in sys.argv[1:] if not a.startswith("--")]
    name = args[0] if args else "c2"
    solves = int(args[1]) if len(args) > 1 else 1
    host = "--host" in sys.argv
    multi = "--multi" in sys.argv or host
    if "--trace" in sys.argv:
        os.environ["PFE_TRACE"] = "1"
    from paper_1612_06496_b200 import _native as N
    from paper_1612_06496_b200 import api
    from paper_1612_06496_b200.inputs import make_config

    cfg = make_config(name)
    g, prm = cfg.graph, cfg.params
    y0 = api.random_embedding(g.n, prm.dim, cfg.y0_seed, g.degree)
    s = api.PfeSolver(g, prm, use_graphs=not host, warn=False, persistent=not multi)
    st = s.make_state(y0)
    for _ in range(solves):
        st.reset()
        s.run_soc(st, prm.soc_max, prm.sb_max_stage1)
    print(name, "ms", s.last_ms(), s.report())
    if "--trace" in sys.argv:
        buf = (C.c_uint64 * (1 << 16))()
        cnt = N.load().pfe_solver_trace(s._h, buf, 1 << 16)
        ev = [(int(v) >> 56, int(v) & ((1 << 56) - 1)) for v in buf[:cnt]]
        ev = [e for e in ev if e[1] != 0]
        agg = defaultdict(lambda: [0, 0.0])
        for (c0, t0), (c1, t1) in zip(ev, ev[1:]):
            if t1 < t0:
                break
            agg[c1][0] += 1
            agg[c1][1] += (t1 - t0) / 1e3
        total = sum(v[1] for v in agg.values())
        print(f"phase trace of the last persistent launch ({len(ev)} events, {total:.1f} us):")
        for c, (k, us) in sorted(agg.items()):
            print(f"  {PHASES.get(c, c):10s} n={k:4d} avg={us / k:8.2f} us total={us:9.1f} us share={us / total:.3f}")


if __name__ == "__main__":
    main()
