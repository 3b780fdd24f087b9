"""north_star parity at FULL size and full iteration counts: C3, C4, C5.

The complete ``soc`` loop of each configuration (solver.cpp:110-126,
184-189; C3 10x30 on the 1024^2 5x5 grid, C4 5x20 on the 4096^2 8-neighbour
grid, C5 10x20 on the 10^6-point 16-NN graph) runs on the GPU and is compared
with the frozen output of the CPU oracle on the same inputs
(tests/golden/full_<cfg>.npz, made by tests/golden/make_full_golden.py with
the column-parallel oracle).  Gates (BASELINE.json north_star):

* relative Frobenius error of Y <= 1e-6 up to column sign, on the frozen row
  sample, on the 4096-row block sums (every row enters one), on the column
  norms and on the Gram matrix YᵀY;
* objective (solver.cpp:14-17) within 1e-6 relative;
* >= 99.9 % agreement of kmeans(Y, k, seed 0) labels (cluster.cpp:54-124),
  ids matched through the contingency table;
* the per-inner-iteration PCG iteration counts (pcg.cpp:68-89, max over the
  d columns) equal to the oracle's.

Every case prints and records (gpurun_out/full_parity_<cfg>.json) its
measured errors so the margin to each gate is visible.
"""
import json
import time
from pathlib import Path

import numpy as np
import pytest

from golden.make_full_golden import array_sha, block_sums, graph_sha
from paper_1612_06496_b200 import api
from paper_1612_06496_b200.inputs import make_config

pytestmark = [pytest.mark.gpu, pytest.mark.slow]

ROOT = Path(__file__).resolve().parents[1]
GOLDEN = ROOT / "tests" / "golden"


def labels_agree(a, b):
    from scipy.optimize import linear_sum_assignment

    a = np.asarray(a, np.int64)
    b = np.asarray(b, np.int64)
    t = np.zeros((a.max() + 1, b.max() + 1), np.int64)
    np.add.at(t, (a, b), 1)
    r, c = linear_sum_assignment(-t)
    return t[r, c].sum() / a.size


def rel(a, b):
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


@pytest.mark.parametrize("name", ["c3", "c4", "c5"])
def test_full_size_parity(name):
    path = GOLDEN / f"full_{name}.npz"
    assert path.exists(), f"missing golden {path.name}: run tests/golden/make_full_golden.py {name}"
    z = np.load(path)
    t0 = time.time()
    cfg = make_config(name, seed=0)
    g, prm = cfg.graph, cfg.params
    t_graph = time.time() - t0
    assert (g.n, g.m, prm.dim) == (int(z["n"]), int(z["m"]), int(z["d"]))
    assert graph_sha(g) == str(z["graph_sha"]), "graph differs from the one the golden was made from"
    y0 = api.random_embedding(g.n, prm.dim, cfg.y0_seed, g.degree)
    assert array_sha(np.asfortranarray(y0)) == str(z["y0_sha"])

    s = api.PfeSolver(g, prm, warn=False)
    st = s.make_state(y0)
    t0 = time.time()
    s.run_soc(st, int(z["soc_max"]), int(z["sb_max"]))
    t_solve = time.time() - t0
    y = st.y
    its, _, _ = s.pcg_log()
    kind = s.report()["persistent_kind"]
    st.close()
    s.close()

    rows = z["rows"]
    exp_rows = z["y_rows"]
    got_rows = y[rows]
    sign = np.sign(np.sum(got_rows * exp_rows, axis=0))
    sign[sign == 0] = 1.0
    ys = y * sign
    err = {
        "rows": rel(ys[rows], exp_rows),
        "block_sums": rel(block_sums(ys), z["block_sums"]),
        "col_norms": rel(np.linalg.norm(y, axis=0), z["col_norms"]),
        "fro": abs(float(np.linalg.norm(y)) - float(z["fro"])) / float(z["fro"]),
        "gram": rel(ys.T @ ys, z["gram"]),
    }
    obj = api.objective(g, y)
    err["objective"] = abs(obj - float(z["objective"])) / abs(float(z["objective"]))
    labels = api.kmeans(y, cfg.k, 0, device=0)
    agree = labels_agree(labels, z["labels"])
    k_gpu = its.max(axis=1)[-len(z["pcg_log"]):]
    pcg_mismatch = int(np.sum(k_gpu != z["pcg_log"]))
    rec = {"config": name, "n": g.n, "m": g.m, "d": prm.dim, "inner": int(len(k_gpu)),
           "rel_err": err, "objective_gpu": obj, "objective_oracle": float(z["objective"]),
           "label_agreement": agree, "pcg_log_mismatches": pcg_mismatch,
           "pcg_iterations_gpu": int(k_gpu.sum()), "pcg_iterations_oracle": int(z["pcg_log"].sum()),
           "persistent_kind": int(kind), "graph_build_s": t_graph, "gpu_solve_s": t_solve,
           "oracle_times_s": {"setup": float(z["times"][0]), "inner": float(z["times"][1]),
                              "projection": float(z["times"][2]), "threads": int(z["times"][6])}}
    print(json.dumps(rec))
    out = ROOT / "gpurun_out"
    out.mkdir(exist_ok=True)
    (out / f"full_parity_{name}.json").write_text(json.dumps(rec, indent=1))
    for k, v in err.items():
        assert v <= 1e-6, f"{name}: {k} relative error {v:.3g} > 1e-6"
    assert agree >= 0.999, f"{name}: label agreement {agree:.5f}"
    assert pcg_mismatch == 0, f"{name}: PCG log differs in {pcg_mismatch} inner iterations"
