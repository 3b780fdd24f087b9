"""GPU GMM initial embedding (init.cpp:45-170, the CLI's
image init path main.cpp:109-110) against the CPU oracle's gmm_fit +
init_embedding on the same features, degrees and seed."""
import numpy as np
import pytest

import oracle as O
from paper_1612_06496_b200 import api
from paper_1612_06496_b200.inputs import grid_graph, voronoi_image

pytestmark = pytest.mark.gpu


def rel(a, b):
    return np.linalg.norm(a - b) / np.linalg.norm(b)


def test_gmm_init_quadrant_matches_oracle():
    """The 64x64 quadrant image of the recorded reference run
    (acceptance.cpp:310-335): d = k = 5, seed 0, reference image graph."""
    rgb = O.quadrant_rgb(64)
    ei, ej, w, deg, _ = O.build_image_graph(rgb)
    f = rgb.reshape(-1, 3)
    y, means, var, wts = api.gmm_init_embedding(f, 5, 0, deg, model=True)
    exp = O.gmm_init_embedding(f, 5, 0, deg)
    assert y.shape == (64 * 64, 5)
    assert rel(y, exp) <= 1e-8
    # the embedding is D-orthonormal: Y^T D Y = I
    g = y.T @ (deg[:, None] * y)
    assert np.abs(g - np.eye(5)).max() <= 1e-10
    assert abs(wts.sum() - 1.0) <= 1e-12 and (var >= 1e-6).all()


@pytest.mark.parametrize("h,w,regions,k,seed", [(60, 80, 6, 4, 0), (33, 47, 3, 8, 3), (120, 90, 8, 16, 1)])
def test_gmm_init_voronoi_matches_oracle(h, w, regions, k, seed):
    rng = np.random.Generator(np.random.PCG64(h * w))
    img, _ = voronoi_image(h, w, regions, 0.05, rng)
    g = grid_graph(img, 0.1, 1)
    f = img.reshape(-1, 3)
    y = api.gmm_init_embedding(f, k, seed, g.degree)
    exp = O.gmm_init_embedding(f, k, seed, g.degree)
    # EM sums associate differently (block partials) and exp/log are CUDA's:
    # agreement to rounding, amplified by the EM fixed point
    assert rel(y, exp) <= 1e-7


def test_gmm_init_then_pfe_matches_oracle_pipeline():
    """GMM init -> soc on the GPU vs the same pipeline on the CPU oracle."""
    rng = np.random.Generator(np.random.PCG64(77))
    img, _ = voronoi_image(40, 56, 5, 0.05, rng)
    g = grid_graph(img, 0.1, 1)
    f = img.reshape(-1, 3)
    prm = api.PfeParams(dim=4, lambda_=1.0, r=1.0, soc_max=3, sb_max_stage1=5, sb_max_stage2=0, conv_tol=0.0,
                        pcg=api.PcgConfig(1e-6, 50, api.Preconditioner.Jacobi))
    y0 = api.gmm_init_embedding(f, 4, 0, g.degree)
    got = api.soc(g, prm, y0)
    exp = O.solve(g, prm, O.gmm_init_embedding(f, 4, 0, g.degree), mode=0)
    s = np.sign(np.sum(got * exp, axis=0))
    assert np.linalg.norm(got * s - exp) / np.linalg.norm(exp) <= 1e-6


def test_gmm_init_config_errors():
    f = np.random.default_rng(0).uniform(size=(10, 3))
    deg = np.ones(10)
    for k in (0, 17, 11):
        with pytest.raises(api.ConfigError):
            api.gmm_init_embedding(f, k, 0, deg)
    bad = f.copy()
    bad[3, 1] = np.nan
    with pytest.raises(api.ConfigError):
        api.gmm_init_embedding(bad, 2, 0, deg)
