"""IC(0)-preconditioned PCG on the GPU (the reference
default preconditioner, pcg.hpp:18 / solver.hpp:24): the reference's factor
(sparse.cpp:124-203) applied by level-scheduled device triangular solves
(sparse.cpp:205-238).  Checked against the CPU oracle's IC(0) path, and the
whole recorded reference run (acceptance.cpp:310-335 -> proj/test_output.txt:
29-30) is reproduced on the GPU: GMM init, default PfeParams (lambda = 100,
IC(0), 10 x 5 + 100 split-Bregman, conv_tol 1e-4), k-means labels."""
import numpy as np
import pytest

import oracle as O
from conftest import random_graph
from paper_1612_06496_b200 import api
from paper_1612_06496_b200.inputs import grid_graph, voronoi_image

pytestmark = pytest.mark.gpu


def ic0(d, lam=1.0, soc=2, sb=4, tol=1e-6, maxit=200, stage2=0, conv=0.0):
    return api.PfeParams(dim=d, lambda_=lam, r=1.0, soc_max=soc, sb_max_stage1=sb, sb_max_stage2=stage2,
                         conv_tol=conv, pcg=api.PcgConfig(tol, maxit, api.Preconditioner.Ic0))


def rel_signed(a, b):
    s = np.sign(np.sum(a * b, axis=0))
    s[s == 0] = 1.0
    return np.linalg.norm(a * s - b) / np.linalg.norm(b)


@pytest.mark.parametrize("kind,d,lam", [("random", 3, 1.0), ("grid", 4, 100.0), ("grid5", 2, 10.0)])
def test_ic0_soc_matches_oracle(kind, d, lam):
    rng = np.random.Generator(np.random.PCG64(31))
    if kind == "random":
        g = random_graph(60, 200, rng)
    else:
        img, _ = voronoi_image(24, 30, 4, 0.05, rng)
        g = grid_graph(img, 0.1, 1 if kind == "grid" else 2, 2.0 if kind == "grid5" else None)
    prm = ic0(d, lam=lam)
    y0 = api.random_embedding(g.n, d, 3, g.degree)
    s = api.PfeSolver(g, prm, warn=False)
    st = s.make_state(y0)
    s.run_soc(st, prm.soc_max, prm.sb_max_stage1)
    rep = s.report()
    assert rep["jacobi_fallback"] == 0
    its, _, _ = s.pcg_log()
    exp = O.solve(g, prm, y0, mode=0, log_cap=1000)
    assert rel_signed(st.y, exp["y"]) <= 1e-9
    # same PCG iteration counts as the reference's IC(0) path
    assert list(its.max(axis=1)) == list(exp["pcg_log"])


def test_ic0_converges_faster_than_jacobi():
    rng = np.random.Generator(np.random.PCG64(5))
    img, _ = voronoi_image(40, 50, 5, 0.05, rng)
    g = grid_graph(img, 0.1, 1)
    y0 = api.random_embedding(g.n, 4, 0, g.degree)
    out = {}
    for prec in (api.Preconditioner.Ic0, api.Preconditioner.Jacobi):
        prm = api.PfeParams(dim=4, lambda_=100.0, r=1.0, soc_max=1, sb_max_stage1=3, sb_max_stage2=0,
                            conv_tol=0.0, pcg=api.PcgConfig(1e-6, 1000, prec))
        s = api.PfeSolver(g, prm, warn=False)
        st = s.make_state(y0)
        s.run_soc(st, 1, 3)
        out[prec] = s.report()["pcg_iterations"]
    assert out[api.Preconditioner.Ic0] < out[api.Preconditioner.Jacobi]


def test_recorded_reference_run_on_gpu():
    """acceptance.cpp:310-335 with the reference defaults: the printed
    objective 26.055418 -> 0.001466 and covering 1.000000."""
    size = 64
    rgb = O.quadrant_rgb(size)
    ei, ej, w, deg, _ = O.build_image_graph(rgb)
    g = api.WeightedGraph(size * size, ei, ej, w, deg)
    prm = api.PfeParams()  # d=5, lambda=100, r=1, 10x5 + 100, conv_tol 1e-4, IC(0) tol 1e-6
    y0 = api.gmm_init_embedding(rgb.reshape(-1, 3), prm.dim, 0, deg)
    s = api.PfeSolver(g, prm, warn=False)
    st = s.two_stage(y0)
    assert s.report()["jacobi_fallback"] == 0
    y = st.y
    obj0, obj1 = api.objective(g, y0), api.objective(g, y)
    assert f"{obj0:.6f}" == "26.055418"
    assert f"{obj1:.6f}" == "0.001466"
    seg = api.kmeans(y, 4, 0)
    truth = np.array([(r >= size // 2) * 2 + (c >= size // 2) for r in range(size) for c in range(size)], np.int32)
    assert O.covering(seg, truth) == pytest.approx(1.0, abs=5e-7)


def test_ic0_standalone_split_bregman_matches_oracle():
    """The free split_bregman (solver.cpp:138-182) builds its own PcgOperator
    with the caller's config: IC(0) there too."""
    rng = np.random.Generator(np.random.PCG64(12))
    g = random_graph(50, 120, rng)
    p, b = rng.uniform(-1, 1, (50, 3)), rng.uniform(-1, 1, (50, 3))
    y_init = rng.uniform(-1, 1, (50, 3))
    prm = ic0(3, lam=5.0, tol=1e-10, maxit=500)
    traj = []
    got = api.split_bregman(g, g.degree, p, b, prm, y_init, 6, on_iterate=lambda it, y: traj.append(y))
    exp, exp_traj = O.split_bregman(g, g.degree, p, b, prm, y_init, 6, want_traj=True)
    assert len(traj) == len(exp_traj) == 6
    for a, c in zip(traj, exp_traj):
        assert np.abs(a - c).max() <= 1e-10
    assert np.abs(got - exp).max() <= 1e-10


def test_ic0_breakdown_falls_back_to_jacobi_like_the_reference():
    """A matrix without a stored diagonal entry in one row: IC(0) breaks
    down for every shift, PcgOperator falls back to Jacobi and says so
    (pcg.cpp:22-28) -- same iterations and result as the oracle."""
    n = 6
    rows, cols, vals = [], [], []
    for i in range(n):
        for j in (i - 1, i, i + 1):
            if 0 <= j < n and not (i == 3 and j == 3):
                rows.append(i)
                cols.append(j)
                vals.append(4.0 if i == j else -1.0)
    ptr = np.zeros(n + 1, np.int32)
    np.add.at(ptr, np.array(rows) + 1, 1)
    ptr = np.cumsum(ptr).astype(np.int32)
    a = (ptr, np.array(cols, np.int32), np.array(vals))
    rng = np.random.Generator(np.random.PCG64(4))
    b, x0 = rng.normal(size=(n, 2)), np.zeros((n, 2))
    x, reps = api.pcg_solve_multi(a, b, x0, api.PcgConfig(1e-8, 100, api.Preconditioner.Ic0))
    xo, its, conv, _ = O.pcg_solve_multi(a, b, x0, 1e-8, 100, int(api.Preconditioner.Ic0))
    assert all(r.jacobi_fallback for r in reps)
    assert [r.iterations for r in reps] == list(its)
    assert np.abs(x - xo).max() <= 1e-12 * max(1.0, np.abs(xo).max())


def test_ic0_disconnected_graph_and_stage2():
    """Two components, Stage II with conv_tol: the IC(0) path matches the
    oracle's two_stage."""
    rng = np.random.Generator(np.random.PCG64(8))
    g1 = random_graph(30, 60, rng)
    g2 = random_graph(25, 40, rng)
    ei = np.concatenate([g1.ei, g2.ei + 30])
    ej = np.concatenate([g1.ej, g2.ej + 30])
    w = np.concatenate([g1.w, g2.w])
    g = api.WeightedGraph(55, ei, ej, w, api.degree_vector(ei, ej, w, 55))
    prm = ic0(3, lam=20.0, soc=2, sb=3, stage2=4, conv=1e-9)
    y0 = api.random_embedding(g.n, 3, 1, g.degree)
    s = api.PfeSolver(g, prm, warn=False)
    got = s.two_stage(y0).y
    exp = O.solve(g, prm, y0, mode=1)
    assert rel_signed(got, exp) <= 1e-9
