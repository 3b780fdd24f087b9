"""GPU parity of the building blocks through the C ABI: shrink, objective,
projection, PCG (test_solver.cpp:30-128, test_pcg.cpp, acceptance 3-5)."""
import numpy as np
import pytest

import oracle as O
from conftest import random_graph
from dense_oracles import polar_factor
from paper_1612_06496_b200 import api

pytestmark = pytest.mark.gpu


def test_shrink_bitwise_and_contracts():
    rng = np.random.Generator(np.random.PCG64(505))
    v = rng.normal(0, 2.0, size=100_003)
    for gamma in [0.0, 0.3, 1.0, 2.5]:
        assert np.array_equal(api.shrink(v, gamma), O.shrink(v, gamma))
    assert api.shrink([2.5], 1.0)[0] == 1.5
    assert api.shrink([-0.5], 1.0)[0] == 0.0
    with pytest.raises(api.ConfigError):
        api.shrink(v, -1.0)


def test_objective_matches_oracle(rng):
    from paper_1612_06496_b200.api import WeightedGraph

    g = WeightedGraph(2, [0], [1], [2.0], [2.0, 2.0])
    assert api.objective(g, np.array([[0.0], [1.0]])) == 2.0
    for _ in range(5):
        g = random_graph(40, 60, rng)
        y = rng.normal(size=(40, 3))
        assert api.objective(g, y) == pytest.approx(O.objective(g, y), rel=1e-12)
        assert api.objective(g, y + np.array([3.7, -1.2, 0.1])) == pytest.approx(api.objective(g, y), rel=1e-10)


@pytest.mark.parametrize("n,d", [(8, 3), (64, 8), (5000, 16), (300_000, 4)])
def test_projection_matches_polar_oracle(n, d):
    rng = np.random.Generator(np.random.PCG64(404 + n))
    a = rng.normal(size=(n, d))
    p = api.project_orthogonal(a)
    assert np.abs(p.T @ p - np.eye(d)).max() <= 1e-12
    assert np.abs(p - polar_factor(a)).max() <= 1e-10
    if n <= 5000:
        assert np.abs(p - O.project_orthogonal(a)).max() <= 1e-12


def test_projection_idempotent_scale_and_rank():
    rng = np.random.Generator(np.random.PCG64(5))
    q, _ = np.linalg.qr(rng.normal(size=(8, 3)))
    assert np.abs(api.project_orthogonal(q) - q).max() < 1e-12
    a = np.zeros((6, 3))
    a[:3] = 2 * np.eye(3)
    exp = np.zeros((6, 3))
    exp[:3] = np.eye(3)
    assert np.abs(api.project_orthogonal(a) - exp).max() < 1e-12
    a = np.ones((4, 2))
    a[:, 1] = 2.0
    with pytest.raises(api.NumericalError, match="rank-deficient in 1 column"):
        api.project_orthogonal(a)
    with pytest.raises(api.ConfigError):
        api.project_orthogonal(np.ones((2, 3)))


@pytest.mark.parametrize("prec", [api.Preconditioner.Jacobi, api.Preconditioner.NONE, api.Preconditioner.Ic0])
def test_pcg_solve_multi_matches_oracle_per_column(prec):
    """Equal per-column iteration counts and x to 1e-12."""
    rng = np.random.Generator(np.random.PCG64(23))
    for n, d in [(30, 4), (200, 3), (1000, 8)]:
        g = random_graph(n, 2 * n, rng)
        a = O.normal_matrix(g, 2.0, 1.0)
        b = rng.normal(size=(n, d))
        x0 = rng.normal(size=(n, d))
        cfg = api.PcgConfig(1e-10, 500, prec)
        x, reps = api.pcg_solve_multi(a, b, x0, cfg)
        xo, its, conv, res = O.pcg_solve_multi(a, b, x0, 1e-10, 500, int(prec))
        assert [r.iterations for r in reps] == list(its)
        assert all(r.converged for r in reps)
        assert not any(r.jacobi_fallback for r in reps)
        assert np.abs(x - xo).max() <= 1e-12 * max(1.0, np.abs(xo).max())


def test_pcg_trivial_cases():
    eye = (np.arange(4, dtype=np.int32), np.arange(3, dtype=np.int32), np.ones(3))
    b = np.array([0.3, -1.0, 2.0])
    x, rep = api.pcg_solve(eye, b, np.zeros(3), api.PcgConfig(preconditioner=api.Preconditioner.Jacobi))
    assert rep.converged and rep.iterations <= 1 and np.abs(x - b).max() < 1e-12
    rng = np.random.Generator(np.random.PCG64(1))
    g = random_graph(10, 20, rng)
    a = O.normal_matrix(g, 2.0, 1.0)
    x, rep = api.pcg_solve(a, np.zeros(10), rng.normal(size=10), api.PcgConfig(preconditioner=1))
    assert rep.converged and rep.iterations == 0 and np.all(x == 0.0)
    # identical columns give identical solutions (test_pcg.cpp:134-140)
    bb = np.repeat(rng.normal(size=(10, 1)), 2, axis=1)
    xx, _ = api.pcg_solve_multi(a, bb, np.zeros((10, 2)), api.PcgConfig(1e-10, 100, 1))
    assert np.array_equal(xx[:, 0], xx[:, 1])
    with pytest.raises(api.ConfigError):
        api.pcg_solve(eye, b, np.zeros(3), api.PcgConfig(rel_tol=0.0))


def test_pcg_maxiter_reports_unconverged():
    rng = np.random.Generator(np.random.PCG64(2))
    g = random_graph(200, 400, rng)
    a = O.normal_matrix(g, 100.0, 1.0)
    b = rng.normal(size=(200, 2))
    x, reps = api.pcg_solve_multi(a, b, np.zeros((200, 2)), api.PcgConfig(1e-14, 3, api.Preconditioner.Jacobi))
    xo, its, conv, res = O.pcg_solve_multi(a, b, np.zeros((200, 2)), 1e-14, 3, 1)
    assert [r.iterations for r in reps] == [3, 3] == list(its)
    assert not any(r.converged for r in reps)
    assert np.allclose([r.final_rel_residual for r in reps], res, rtol=1e-10)
    assert np.abs(x - xo).max() <= 1e-12
