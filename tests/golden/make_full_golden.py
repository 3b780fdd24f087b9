"""Full-size goldens for BASELINE.json configs C3, C4 and C5 — TEST INFRASTRUCTURE.

The CPU oracle (oracle/, the Eigen-free restatement of
proj/core/src/{sparse,pcg,solver,cluster}.cpp pinned to the recorded reference
run proj/test_output.txt:29-30) runs the configuration's complete ``soc`` loop
(solver.cpp:110-126, 184-189) at full size and full iteration counts, with
its column loop on several threads (columns are independent, so the result is
bitwise the single-thread one).  A full Y does not fit in git
(C4: 1.07 GB), so the fixture freezes size-independent evidence of it:

* ``graph_sha`` / ``y0_sha``: the exact inputs (the GPU test rebuilds the graph
  and Y0 and refuses to compare if either differs);
* ``rows`` + ``y_rows``: every ``stride``-th row of Y (>= 16k rows);
* ``block_sums``: per-column sums of Y over consecutive 4096-row blocks (a
  checksum of every row), ``col_norms``, ``fro``, ``gram`` = YᵀY;
* ``objective`` (solver.cpp:14-17) of Y and ``objective0`` of Y0;
* ``pcg_log``: PCG iterations per inner iteration (max over columns);
* ``labels``: ``kmeans(Y, k, seed 0)`` (cluster.cpp:54-124), uint8/uint16;
* ``times``: oracle set-up / inner-loop / projection seconds and threads.

C3 and C4 build their graphs with numpy (inputs.grid_graph).  C5's 16-NN
graph over 10^6 points in R^16 is built on the GPU (``pfe_knn_graph``), so its
golden is generated on the GPU box (scripts/gpu_golden_c5.sh); the oracle
still does all of the solving and clustering on the host.

usage: python tests/golden/make_full_golden.py c3 [c4 c5] [--threads T]
"""
from __future__ import annotations

import argparse
import hashlib
import os
import sys
import time
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
ROOT = HERE.parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))

import oracle as O  # noqa: E402

BLOCK = 4096
SAMPLE_ROWS = 16384


def graph_sha(g) -> str:
    h = hashlib.sha256()
    for a in (np.int64(g.n), np.ascontiguousarray(g.ei, np.int32), np.ascontiguousarray(g.ej, np.int32),
              np.ascontiguousarray(g.w, np.float64), np.ascontiguousarray(g.degree, np.float64)):
        h.update(np.asarray(a).tobytes())
    return h.hexdigest()


def array_sha(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a, np.float64).tobytes()).hexdigest()


def sample_rows(n):
    stride = max(1, n // SAMPLE_ROWS)
    return np.arange(0, n, stride, dtype=np.int64), stride


def block_sums(y):
    n, d = y.shape
    nb = (n + BLOCK - 1) // BLOCK
    pad = np.zeros((nb * BLOCK, d))
    pad[:n] = y
    return pad.reshape(nb, BLOCK, d).sum(axis=1)


def evidence(y):
    """The size-independent summaries both sides compute from a full Y."""
    rows, stride = sample_rows(y.shape[0])
    return {"rows": rows, "stride": np.int64(stride), "y_rows": np.ascontiguousarray(y[rows]),
            "block_sums": block_sums(y), "col_norms": np.linalg.norm(y, axis=0), "fro": np.float64(np.linalg.norm(y)),
            "gram": y.T @ y}


def make(name, threads, scale=None, out_dir=HERE):
    from paper_1612_06496_b200.inputs import make_config

    t0 = time.time()
    cfg = make_config(name, seed=0, scale=scale)
    g, prm = cfg.graph, cfg.params
    t_graph = time.time() - t0
    y0 = O.random_embedding(g.n, prm.dim, cfg.y0_seed, g.degree)  # == pfe_random_embedding bitwise
    O.set_threads(threads)
    t0 = time.time()
    res = O.solve_timed(g, prm, y0)
    t_solve = time.time() - t0
    y = res["y"]
    t0 = time.time()
    labels = O.kmeans(y, cfg.k, 0)
    t_km = time.time() - t0
    obj = O.objective(g, y)
    obj0 = O.objective(g, y0)
    O.set_threads(1)
    ldt = np.uint8 if cfg.k <= 256 else np.uint16
    out = dict(
        name=np.str_(name), n=np.int64(g.n), m=np.int64(g.m), d=np.int64(prm.dim), k=np.int64(cfg.k),
        soc_max=np.int64(prm.soc_max), sb_max=np.int64(prm.sb_max_stage1), pcg_tol=np.float64(prm.pcg.rel_tol),
        graph_sha=np.str_(graph_sha(g)), y0_sha=np.str_(array_sha(np.asfortranarray(y0))),
        objective=np.float64(obj), objective0=np.float64(obj0), pcg_log=np.asarray(res["pcg_log"], np.int32),
        labels=np.asarray(labels, ldt),
        times=np.array([res["t_setup"], res["t_inner"], res["t_outer"], t_km, t_graph, t_solve, threads]),
        **evidence(y))
    path = Path(out_dir) / f"full_{name}.npz"
    np.savez_compressed(path, **out)
    print(f"{name}: n={g.n} m={g.m} d={prm.dim} objective {obj0:.9g} -> {obj:.12g}; "
          f"pcg iterations {int(out['pcg_log'].sum())} over {res['inner']} inner; oracle set-up {res['t_setup']:.1f} s, "
          f"inner {res['t_inner']:.1f} s, projections {res['t_outer']:.1f} s, k-means {t_km:.1f} s on {threads} "
          f"threads; wrote {path.name} ({path.stat().st_size / 1e6:.2f} MB)", flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("configs", nargs="+")
    ap.add_argument("--threads", type=int, default=os.cpu_count() or 1)
    ap.add_argument("--scale", type=int, nargs="+", help="scaled-down run (script check only)")
    ap.add_argument("--out", default=str(HERE))
    a = ap.parse_args()
    for name in a.configs:
        make(name.lower(), a.threads, tuple(a.scale) if a.scale else None, a.out)


if __name__ == "__main__":
    main()
