"""Small invocations of every kernel family, run under compute-sanitizer
(scripts/gpu_sanitize.sh: memcheck, racecheck, synccheck, initcheck).

Each case is a tiny solve so the instrumented run stays short:
  resident   k_sb_resident (shared-memory resident persistent kernel, 8-nbr grid)
  tiled8     k_sb_persistent, 8-neighbour grid (cp.async tiles)
  tiled24    k_sb_persistent, 5x5 grid (TMA tiles)
  multi      one kernel per phase (grid stencil kernels + CUDA graph WHILE loop)
  csr        general-graph kernels (k-NN graph built on the GPU), d = 16
  ic0        IC(0) level-scheduled triangular solves
  bands      emulated row bands and vertex ranges
  extras     k-means, GMM init, projection, objective on the GPU
  tiled8tma  (not in the default list) k_sb_persistent on an 8-neighbour grid
             with TMA staging forced on (PFE_TMA=1): the known-fault path
usage: python scripts/sanitize_cases.py [case ...]   (default: all)
"""
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

from paper_1612_06496_b200 import api  # noqa: E402
from paper_1612_06496_b200.inputs import grid_graph, voronoi_image  # noqa: E402


def prm(d, soc=2, sb=3, pc=api.Preconditioner.Jacobi, lam=1.0, maxit=50):
    return api.PfeParams(dim=d, lambda_=lam, r=1.0, soc_max=soc, sb_max_stage1=sb, sb_max_stage2=0, conv_tol=0.0,
                         pcg=api.PcgConfig(1e-6, maxit, pc))


def image(h, w, radius, seed=1):
    rng = np.random.Generator(np.random.PCG64(seed))
    img, _ = voronoi_image(h, w, 5, 0.05, rng)
    return grid_graph(img, 0.1, radius, 2.0 if radius == 2 else None), img


def run(g, p, persistent, use_graphs=True):
    y0 = api.random_embedding(g.n, p.dim, 0, g.degree)
    s = api.PfeSolver(g, p, persistent=persistent, use_graphs=use_graphs, warn=False)
    st = s.make_state(y0)
    s.run_soc(st, p.soc_max, p.sb_max_stage1)
    y = st.y
    kind = s.report()["persistent_kind"]
    st.close()
    s.close()
    return y, kind


def main():
    cases = sys.argv[1:] or ["resident", "tiled8", "tiled24", "multi", "csr", "ic0", "bands", "extras"]
    for c in cases:
        if c == "resident":
            g, _ = image(40, 56, 1)
            _, kind = run(g, prm(4), 1)
            assert kind == 2, kind
        elif c == "tiled8":
            g, _ = image(37, 70, 1)
            _, kind = run(g, prm(8), 2)
            assert kind == 1, kind
        elif c == "tiled8tma":
            import os

            os.environ["PFE_TMA"] = os.environ.get("PFE_TMA_MASK", "1")
            g, _ = image(37, 70, 1)
            _, kind = run(g, prm(int(os.environ.get("PFE_SAN_D", "8"))), 2)
            os.environ.pop("PFE_TMA")
        elif c == "tiled24":
            g, _ = image(33, 64, 2)
            _, kind = run(g, prm(8), 2)
            assert kind == 1, kind
        elif c == "multi":
            g, _ = image(30, 45, 1)
            run(g, prm(4), 0, use_graphs=True)
            run(g, prm(3), 0, use_graphs=False)
        elif c == "csr":
            rng = np.random.Generator(np.random.PCG64(3))
            pts = rng.normal(size=(600, 16))
            gk = api.knn_graph_gpu(pts, 8)
            run(gk, prm(16), 0, use_graphs=True)
        elif c == "ic0":
            g, _ = image(12, 16, 1)
            run(g, prm(3, soc=1, sb=2, pc=api.Preconditioner.Ic0, lam=100.0, maxit=200), 0, use_graphs=False)
        elif c == "bands":
            g, _ = image(24, 30, 1)
            p = prm(4)
            y0 = api.random_embedding(g.n, 4, 0, g.degree)
            api.soc_banded(g, p, y0, 3)
            rng = np.random.Generator(np.random.PCG64(4))
            gk = api.knn_graph_gpu(rng.uniform(-1, 1, size=(300, 3)), 6)
            api.soc_banded(gk, prm(4), api.random_embedding(gk.n, 4, 0, gk.degree), 2)
        elif c == "extras":
            g, img = image(24, 32, 1)
            y = api.random_embedding(g.n, 4, 0, g.degree)
            api.kmeans(y, 4, 0, device=0)
            api.gmm_init_embedding(img.reshape(-1, 3), 3, 0, g.degree)
            api.project_orthogonal(y)
            api.objective(g, y)
        else:
            raise SystemExit(f"unknown case {c}")
        print(f"case {c}: ok", flush=True)


if __name__ == "__main__":
    main()
