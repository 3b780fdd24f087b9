"""BASELINE.json configurations C3, C4 and C5 on the GPU.

* Scaled-down images / point sets with the configs' full iteration counts,
  tolerances, radii and dimensions: Y (per-column sign), objective and
  k-means labels against the oracle (north_star parity gates).
* Full size, bounded iteration counts: the first inner iteration of C3 against
  the oracle, and size-independent properties at C4 / C5 scale (persistent vs
  one-kernel-per-phase agreement, orthonormal P, bitwise repeatability).
"""
import numpy as np
import pytest

import oracle as O
from paper_1612_06496_b200 import api
from paper_1612_06496_b200.inputs import make_config

pytestmark = pytest.mark.gpu


def rel(a, b):
    s = np.sign(np.sum(a * b, axis=0))
    s[s == 0] = 1.0
    return np.linalg.norm(a * s - b) / np.linalg.norm(b)


def labels_agree(a, b):
    from scipy.optimize import linear_sum_assignment

    t = np.zeros((a.max() + 1, b.max() + 1), np.int64)
    np.add.at(t, (a, b), 1)
    r, c = linear_sum_assignment(-t)
    return t[r, c].sum() / a.size


def gates(cfg, got, exp):
    g = cfg.graph
    assert rel(got, exp) <= 1e-6
    oo = O.objective(g, exp)
    assert abs(api.objective(g, got) - oo) <= 1e-6 * abs(oo)
    assert labels_agree(api.kmeans(got, cfg.k, 0), O.kmeans(exp, cfg.k, 0)) >= 0.999


def run_oracle(g, prm, y0, threads):
    O.set_threads(threads)
    try:
        return O.solve(g, prm, y0, mode=0)
    finally:
        O.set_threads(1)


@pytest.mark.parametrize("name,scale", [("c3", (160, 160)), ("c4", (256, 256)), ("c5", (20000,))])
def test_scaled_config_parity(name, scale):
    cfg = make_config(name, scale=scale)
    g, prm = cfg.graph, cfg.params
    y0 = api.random_embedding(g.n, prm.dim, cfg.y0_seed, g.degree)
    got = api.soc(g, prm, y0)
    exp = run_oracle(g, prm, y0, prm.dim)
    gates(cfg, got, exp)
    assert rel(got, exp) <= 1e-9  # in practice only the reduction order differs


@pytest.mark.slow
def test_c3_full_size_first_inner_iteration():
    """C3 at full size (1024^2, radius 2, d = 8): one inner iteration and one
    projection against the oracle."""
    cfg = make_config("c3")
    g, prm = cfg.graph, cfg.params
    prm.soc_max, prm.sb_max_stage1 = 1, 1
    y0 = api.random_embedding(g.n, prm.dim, cfg.y0_seed, g.degree)
    got = api.soc(g, prm, y0)
    exp = run_oracle(g, prm, y0, prm.dim)
    assert rel(got, exp) <= 1e-9


@pytest.mark.slow
def test_c4_full_size_properties():
    """C4 at full size (4096^2, d = 8), 1 outer x 2 inner iterations: the
    persistent kernel and the one-kernel-per-phase path agree, P is
    orthonormal, and runs repeat bitwise."""
    cfg = make_config("c4")
    g, prm = cfg.graph, cfg.params
    prm.soc_max, prm.sb_max_stage1 = 1, 2
    y0 = api.random_embedding(g.n, prm.dim, cfg.y0_seed, g.degree)
    s = api.PfeSolver(g, prm, warn=False)
    st = s.make_state(y0)
    s.run_soc(st, 1, 2)
    a = st.y
    p = st.p
    assert s.report()["persistent_kind"] == 1
    st.reset()
    s.run_soc(st, 1, 2)
    assert np.array_equal(st.y, a)
    del st
    s.close()
    b = api.soc(g, prm, y0, persistent=False)
    assert rel(a, b) <= 1e-12
    assert np.abs(p.T @ p - np.eye(prm.dim)).max() <= 1e-10


@pytest.mark.slow
def test_c5_full_size_properties():
    """C5 at full size (10^6 points, GPU-built 16-NN graph, d = 16), 1 outer x
    1 inner: graph-captured and host-driven loops agree bitwise, P orthonormal."""
    cfg = make_config("c5")
    g, prm = cfg.graph, cfg.params
    assert 12.0 < g.m / g.n < 13.5
    prm.soc_max, prm.sb_max_stage1 = 1, 1
    y0 = api.random_embedding(g.n, prm.dim, cfg.y0_seed, g.degree)
    a = api.soc(g, prm, y0, use_graphs=True)
    b = api.soc(g, prm, y0, use_graphs=False)
    assert np.array_equal(a, b)
    s = api.PfeSolver(g, prm, warn=False)
    st = s.make_state(y0)
    s.run_soc(st, 1, 1)
    p = st.p
    assert np.abs(p.T @ p - np.eye(prm.dim)).max() <= 1e-10
