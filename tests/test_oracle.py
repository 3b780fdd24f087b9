"""CPU oracle pinning (no GPU): the restatement against the reference's own
recorded run, known-answer tests and brute-force oracles."""
import numpy as np
import pytest

import oracle as O
from conftest import random_graph
from dense_oracles import KroneckerSolver, diff_matrix_dense, polar_factor
from paper_1612_06496_b200.api import PcgConfig, PfeParams, Preconditioner


def tight(d, lam, r):
    # test_solver.cpp:17-26
    return PfeParams(dim=d, lambda_=lam, r=r, conv_tol=0.0, pcg=PcgConfig(1e-13, 2000, Preconditioner.Ic0))


def test_golden_quadrant_run_matches_recorded_reference():
    """proj/test_output.txt:29-30 — criterion 7 covering 1.000000, criterion 8
    objective 26.055418 -> 0.001466 (printed with 6 decimals)."""
    r = O.golden_quadrant(64)
    assert f"{r['covering']:.6f}" == "1.000000"
    assert f"{r['obj0']:.6f}" == "26.055418"
    assert f"{r['obj1']:.6f}" == "0.001466"


def test_shrink_known_answers():
    # test_solver.cpp:30-35
    assert O.shrink([2.5], 1.0)[0] == 1.5
    assert O.shrink([-0.5], 1.0)[0] == 0.0
    v = np.random.default_rng(0).normal(size=50)
    assert np.array_equal(O.shrink(v, 0.0), v)


def test_objective_known_answers(rng):
    from paper_1612_06496_b200.api import WeightedGraph

    g = WeightedGraph(2, [0], [1], [2.0], [2.0, 2.0])
    assert O.objective(g, np.array([[0.0], [1.0]])) == 2.0  # test_solver.cpp:98-106
    g = random_graph(8, 6, rng)
    y = np.tile([1.0, -2.0, 0.5], (8, 1))
    assert O.objective(g, y) == 0.0


def test_normal_matrix_matches_dense_formula(rng):
    # test_sparse.cpp:110-125
    g = random_graph(10, 12, rng)
    ptr, idx, val = O.normal_matrix(g, 3.0, 0.7)
    a = np.zeros((10, 10))
    for r in range(10):
        for k in range(ptr[r], ptr[r + 1]):
            a[r, idx[k]] += val[k]
    m = diff_matrix_dense(g)
    ref = 1.5 * m.T @ m + 0.35 * np.diag(g.degree)
    assert np.abs(a - ref).max() < 1e-12
    assert np.all(np.linalg.eigvalsh(a) > 0)


def test_oracle_trajectory_matches_kronecker():
    """Acceptance criterion 1 (acceptance.cpp:43-92) on the oracle."""
    rng = np.random.Generator(np.random.PCG64(101))
    worst = 0.0
    for _ in range(25):
        n, d = int(rng.integers(3, 7)), int(rng.integers(1, 4))
        g = random_graph(n, 2, rng)
        y0, p, b = rng.normal(size=(n, d)), rng.normal(size=(n, d)), 0.2 * rng.normal(size=(n, d))
        prm = PfeParams(dim=d, lambda_=50.0, r=1.5, conv_tol=0.0, pcg=PcgConfig(1e-13, 10000, Preconditioner.Ic0))
        _, traj = O.split_bregman(g, g.degree, p, b, prm, y0, 8, want_traj=True)
        lit = []
        KroneckerSolver(diff_matrix_dense(g), g.degree, d, 50.0, 1.5).split_bregman(p, b, y0, 8, lit)
        assert len(traj) == len(lit) == 8
        worst = max(worst, max(np.abs(a - c).max() for a, c in zip(traj, lit)))
    assert worst <= 1e-8


@pytest.mark.parametrize("prec", [0, 1, 2])
def test_oracle_pcg_matches_dense(prec):
    """Acceptance criterion 3 (acceptance.cpp:127-155) for each preconditioner."""
    rng = np.random.Generator(np.random.PCG64(303))
    for _ in range(10):
        g = random_graph(50, 40, rng)
        a = O.normal_matrix(g, 50.0, 1.0)
        dense = np.zeros((50, 50))
        for r in range(50):
            dense[r, a[1][a[0][r]:a[0][r + 1]]] = a[2][a[0][r]:a[0][r + 1]]
        b = rng.normal(size=(50, 1))
        x, its, conv, _ = O.pcg_solve_multi(a, b, np.zeros((50, 1)), 1e-12, 1000, prec)
        ref = np.linalg.solve(dense, b)
        assert conv[0] == 1
        assert np.linalg.norm(x - ref) / np.linalg.norm(ref) <= 1e-8


def test_oracle_projection_matches_polar():
    """Acceptance criterion 4 (acceptance.cpp:159-184)."""
    rng = np.random.Generator(np.random.PCG64(404))
    for _ in range(100):
        d = int(rng.integers(1, 9))
        n = int(rng.integers(d + 1, 65))
        a = rng.normal(size=(n, d))
        p = O.project_orthogonal(a)
        assert np.abs(p.T @ p - np.eye(d)).max() <= 1e-8
        assert np.abs(p - polar_factor(a)).max() <= 1e-8


def test_oracle_projection_rank_deficiency():
    a = np.ones((4, 2))
    a[:, 1] = 2.0
    with pytest.raises(O.OracleError) as e:
        O.project_orthogonal(a)
    assert e.value.code == 2 and "rank-deficient in 1 column" in str(e.value)


def test_oracle_soc_matches_literal_outer_loop():
    """test_solver.cpp:252-271 on the oracle."""
    rng = np.random.Generator(np.random.PCG64(31))
    for trial in range(5):
        g = random_graph(6, 4, rng)
        y0 = O.random_embedding(6, 2, trial, g.degree)
        exp = KroneckerSolver(diff_matrix_dense(g), g.degree, 2, 10.0, 1.0).soc(y0, 3, 4)
        prm = tight(2, 10.0, 1.0)
        prm.soc_max, prm.sb_max_stage1 = 3, 4
        got = O.solve(g, prm, y0, mode=0)
        assert np.abs(got - exp).max() < 1e-7


def test_oracle_column_threads_bitwise(rng):
    """solve_multi columns are independent: threads change nothing."""
    g = random_graph(40, 60, rng)
    prm = PfeParams(dim=3, lambda_=1.0, r=1.0, soc_max=2, sb_max_stage1=3, sb_max_stage2=0, conv_tol=0.0,
                    pcg=PcgConfig(1e-6, 50, Preconditioner.Jacobi))
    y0 = O.random_embedding(40, 3, 5, g.degree)
    O.set_threads(1)
    a = O.solve(g, prm, y0)
    O.set_threads(3)
    b = O.solve(g, prm, y0)
    O.set_threads(1)
    assert np.array_equal(a, b)
