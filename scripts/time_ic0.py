"""Times one outer iteration (20 inner) of C2 with the IC(0) preconditioner
on the GPU and on the CPU oracle (1 core), lambda = r = 1, tol 1e-6, and the
same with Jacobi on the GPU.

usage: python scripts/time_ic0.py
"""
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))


def main():
    import oracle as O
    from paper_1612_06496_b200 import api
    from paper_1612_06496_b200.inputs import make_config

    cfg = make_config("c2")
    g = cfg.graph
    y0 = api.random_embedding(g.n, 4, 0, g.degree)
    for prec in (api.Preconditioner.Ic0, api.Preconditioner.Jacobi):
        prm = api.PfeParams(dim=4, lambda_=1.0, r=1.0, soc_max=1, sb_max_stage1=20, sb_max_stage2=0, conv_tol=0.0,
                            pcg=api.PcgConfig(1e-6, 50, prec))
        s = api.PfeSolver(g, prm, warn=False)
        st = s.make_state(y0)
        t0 = time.perf_counter()
        s.run_soc(st, 1, 20)
        dt = time.perf_counter() - t0
        print(f"GPU {prec.name}: 20 inner iterations {dt * 1e3:.1f} ms, pcg iterations {s.report()['pcg_iterations']}")
        if prec == api.Preconditioner.Ic0:
            t0 = time.perf_counter()
            res = O.solve(g, prm, y0, mode=0, log_cap=100)
            dc = time.perf_counter() - t0
            print(f"CPU oracle Ic0 (1 core): {dc * 1e3:.1f} ms, pcg iterations {int(res['pcg_log'].sum())}")


if __name__ == "__main__":
    main()
