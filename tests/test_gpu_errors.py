"""The reference's error and warning semantics on every execution path.

* solver.cpp:94: a NaN in the embedding after the inner solve raises
  NumericalError("split_bregman: NaN in embedding").  The persistent kernels
  stop the launch at the inner iteration that produced it.
* solver.cpp:87-92: a column whose PCG stopped unconverged prints
  "pfe: inner solve column <j> stopped at rel residual <r>" on stderr, also
  when the inner loop ran inside one persistent launch or a CUDA graph.
"""
import numpy as np
import pytest

from paper_1612_06496_b200 import api
from paper_1612_06496_b200.inputs import grid_graph, knn_graph, voronoi_image

pytestmark = pytest.mark.gpu

PATHS = [dict(persistent=True), dict(persistent="tiled"), dict(persistent=False, use_graphs=True),
         dict(persistent=False, use_graphs=False)]
IDS = ["resident", "tiled", "graph", "host"]


def grid(h=24, w=30, seed=5):
    rng = np.random.Generator(np.random.PCG64(seed))
    img, _ = voronoi_image(h, w, 4, 0.05, rng)
    return grid_graph(img, 0.1, 1)


def params(d=4, lam=1.0, maxit=50, soc=2, sb=4):
    return api.PfeParams(dim=d, lambda_=lam, r=1.0, soc_max=soc, sb_max_stage1=sb, sb_max_stage2=0, conv_tol=0.0,
                         pcg=api.PcgConfig(1e-6, maxit, api.Preconditioner.Jacobi))


@pytest.mark.parametrize("kw", PATHS, ids=IDS)
def test_nan_in_embedding_raises_numerical_error(kw):
    g = grid()
    prm = params()
    y0 = api.random_embedding(g.n, prm.dim, 0, g.degree)
    y0[7, 1] = np.nan
    s = api.PfeSolver(g, prm, warn=False, **kw)
    st = s.make_state(y0)
    with pytest.raises(api.NumericalError, match="split_bregman: NaN in embedding"):
        s.run_soc(st, prm.soc_max, prm.sb_max_stage1)
    # the flag is cleared with the error: a clean state solves normally afterwards
    st2 = s.make_state(api.random_embedding(g.n, prm.dim, 0, g.degree))
    s.run_soc(st2, 1, 2)
    assert np.isfinite(st2.y).all()


def test_nan_in_embedding_general_graph():
    rng = np.random.Generator(np.random.PCG64(2))
    g = knn_graph(rng.normal(size=(300, 3)), 6)
    prm = params(d=3)
    y0 = api.random_embedding(g.n, prm.dim, 0, g.degree)
    y0[11, 0] = np.inf
    with pytest.raises(api.NumericalError, match="split_bregman: NaN in embedding"):
        api.soc(g, prm, y0)


@pytest.mark.parametrize("kw", PATHS, ids=IDS)
def test_nonconverged_columns_warn_on_stderr(kw, capfd):
    """lambda = 100 with a 3-iteration PCG cap: every column stops unconverged."""
    g = grid()
    prm = params(lam=100.0, maxit=3, soc=1, sb=2)
    y0 = api.random_embedding(g.n, prm.dim, 0, g.degree)
    s = api.PfeSolver(g, prm, warn=True, **kw)
    st = s.make_state(y0)
    s.run_soc(st, 1, 2)
    err = capfd.readouterr().err
    lines = [ln for ln in err.splitlines() if ln.startswith("pfe: inner solve column")]
    assert len(lines) == 2 * prm.dim, err  # 2 inner iterations x d columns
    assert "stopped at rel residual" in lines[0]


@pytest.mark.gpu
def test_block_cache_reuses_and_releases_device_memory():
    """Destroyed solvers park their large device arrays for exact-size reuse
    (the one-call pfe_solve path); pfe_release_cached_memory hands them back."""
    from paper_1612_06496_b200 import _native as N

    lib = N.load()
    lib.pfe_release_cached_memory(0)
    rng = np.random.Generator(np.random.PCG64(3))
    img, _ = voronoi_image(512, 640, 6, 0.05, rng)  # n*d*8 = 10.5 MB per state array: above the 8 MB cache floor
    g = grid_graph(img, 0.1, 1)
    prm = api.PfeParams(dim=4, lambda_=1.0, r=1.0, soc_max=1, sb_max_stage1=2, sb_max_stage2=0, conv_tol=0.0,
                        pcg=api.PcgConfig(1e-6, 50, api.Preconditioner.Jacobi))
    y0 = api.random_embedding(g.n, 4, 0, g.degree)
    ya = api.soc(g, prm, y0)
    yb = api.soc(g, prm, y0)  # runs on recycled (uncleared) blocks: must not depend on their contents
    assert np.array_equal(ya, yb)
    freed = lib.pfe_release_cached_memory(0)
    assert freed >= 10 * g.n * 4 * 8
    assert lib.pfe_release_cached_memory(0) == 0
    assert np.array_equal(api.soc(g, prm, y0), ya)
    assert lib.pfe_release_cached_memory(99) == 0
