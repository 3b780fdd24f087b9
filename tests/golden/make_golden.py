"""Generates the committed golden fixtures in tests/golden/*.npz — TEST INFRASTRUCTURE.

Each fixture is one small, seeded instance of the hot path (graph + PfeParams +
Y0) together with what the CPU oracle (oracle/, the Eigen-free restatement of
proj/core/src/{sparse,pcg,solver,cluster}.cpp, pinned to the recorded reference
run proj/test_output.txt:29-30) returns for it: the embedding Y after the
`soc` / `pfe_two_stage` loop (solver.cpp:110-136, 184-193), the objective
(solver.cpp:14-17), the per-inner-iteration PCG iteration log and the k-means
labels (cluster.cpp:54-124).

The fixtures freeze those outputs so the GPU tests compare against fixed
numbers, and tests/test_golden.py re-derives them from the oracle on every CPU
run (a change in the oracle or the input generators shows up as a diff).

usage: python tests/golden/make_golden.py        (rewrites every fixture)
"""
from __future__ import annotations

import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
ROOT = HERE.parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))

import oracle as O  # noqa: E402
from paper_1612_06496_b200 import api  # noqa: E402
from paper_1612_06496_b200.inputs import grid_graph, knn_graph, voronoi_image  # noqa: E402


def _params(d, soc, sb, tol=1e-6, maxit=50, lam=1.0, r=1.0, stage2=0, conv=0.0):
    return api.PfeParams(dim=d, lambda_=lam, r=r, soc_max=soc, sb_max_stage1=sb, sb_max_stage2=stage2,
                         conv_tol=conv, pcg=api.PcgConfig(tol, maxit, api.Preconditioner.Jacobi))


def _gmm_points(rng, n, dim, comps, lo, hi, std_lo, std_hi):
    means = rng.uniform(lo, hi, size=(comps, dim))
    stds = rng.uniform(std_lo, std_hi, size=comps)
    comp = rng.integers(0, comps, size=n)
    return means[comp] + rng.normal(size=(n, dim)) * stds[comp, None]


def cases():
    """name -> (graph, params, y0_seed, mode, k). mode 0 = soc, 1 = two_stage."""
    out = {}
    rng = np.random.Generator(np.random.PCG64(101))
    img, _ = voronoi_image(24, 32, 5, 0.05, rng)
    out["grid8_c2like"] = (grid_graph(img, 0.1, 1), _params(4, 3, 5), 0, 0, 5)
    rng = np.random.Generator(np.random.PCG64(102))
    img, _ = voronoi_image(20, 26, 6, 0.03, rng, gradient=1.0 / 64.0)
    out["grid5x5_c3like"] = (grid_graph(img, 0.1, 2, sigma_xy=2.0), _params(8, 2, 4, tol=1e-7), 0, 0, 6)
    rng = np.random.Generator(np.random.PCG64(103))
    img, _ = voronoi_image(16, 40, 4, 0.05, rng)
    out["grid8_two_stage"] = (grid_graph(img, 0.1, 1), _params(3, 2, 3, stage2=4, conv=1e-9), 1, 1, 4)
    rng = np.random.Generator(np.random.PCG64(104))
    pts = _gmm_points(rng, 300, 2, 4, -5.0, 5.0, 0.3, 0.3)
    out["knn10_c1like"] = (knn_graph(pts, 10), _params(3, 3, 5), 0, 0, 4)
    rng = np.random.Generator(np.random.PCG64(105))
    pts = _gmm_points(rng, 500, 16, 6, -10.0, 10.0, 0.5, 1.5)
    out["knn16_c5like"] = (knn_graph(pts, 16), _params(16, 2, 4), 0, 0, 6)
    # default lambda = 100 (solver.hpp:18): PCG hits the iteration cap
    rng = np.random.Generator(np.random.PCG64(106))
    img, _ = voronoi_image(12, 14, 3, 0.05, rng)
    out["grid8_lambda100_capped"] = (grid_graph(img, 0.1, 1), _params(5, 2, 3, lam=100.0, maxit=20), 0, 0, 3)
    return out


def oracle_outputs(g, prm, y0_seed, mode, k):
    y0 = api.random_embedding(g.n, prm.dim, y0_seed, g.degree)
    res = O.solve(g, prm, y0, mode=mode, log_cap=10000)
    y = res["y"]
    return {
        "y0": y0,
        "y": y,
        "objective": np.float64(O.objective(g, y)),
        "objective0": np.float64(O.objective(g, y0)),
        "pcg_log": np.asarray(res["pcg_log"], np.int32),
        "labels": np.asarray(O.kmeans(y, k, 0), np.int32),
    }


def pack(name, g, prm, y0_seed, mode, k):
    d = oracle_outputs(g, prm, y0_seed, mode, k)
    grid = np.asarray(g.grid if g.grid else (0, 0, 0), np.int32)
    p = np.array([prm.dim, prm.soc_max, prm.sb_max_stage1, prm.sb_max_stage2, prm.pcg.max_iter,
                  int(prm.pcg.preconditioner), mode, k, y0_seed], np.int64)
    f = np.array([prm.lambda_, prm.r, prm.conv_tol, prm.pcg.rel_tol], np.float64)
    return dict(n=np.int64(g.n), ei=g.ei, ej=g.ej, w=g.w, degree=g.degree, grid=grid, iparams=p, fparams=f, **d)


def load(path):
    """fixture -> (graph, params, mode, k, arrays)."""
    z = dict(np.load(path))
    h, w_, r = (int(v) for v in z["grid"])
    g = api.WeightedGraph(int(z["n"]), z["ei"], z["ej"], z["w"], z["degree"], grid=(h, w_, r) if h else None)
    d, soc, sb, st2, maxit, prec, mode, k, _ = (int(v) for v in z["iparams"])
    lam, r_, conv, tol = (float(v) for v in z["fparams"])
    prm = api.PfeParams(dim=d, lambda_=lam, r=r_, soc_max=soc, sb_max_stage1=sb, sb_max_stage2=st2,
                        conv_tol=conv, pcg=api.PcgConfig(tol, maxit, api.Preconditioner(prec)))
    return g, prm, mode, k, z


def main():
    for name, (g, prm, seed, mode, k) in cases().items():
        arrs = pack(name, g, prm, seed, mode, k)
        np.savez_compressed(HERE / f"{name}.npz", **arrs)
        print(f"{name}: n={g.n} m={g.m} d={prm.dim} objective {arrs['objective0']:.6f} -> "
              f"{arrs['objective']:.6f} pcg={int(arrs['pcg_log'].sum())}")


if __name__ == "__main__":
    main()
