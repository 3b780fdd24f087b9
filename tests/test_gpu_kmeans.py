"""k-means "labels out" on the GPU (pfe_kmeans_device) against the host
implementation and the oracle (cluster.cpp:15-124): same seeding stream,
tie-breaks, empty-cluster split and stop rule."""
import time

import numpy as np
import pytest

import oracle as O
from paper_1612_06496_b200 import api
from paper_1612_06496_b200.inputs import make_config

pytestmark = pytest.mark.gpu


def agreement(a, b):
    from scipy.optimize import linear_sum_assignment

    t = np.zeros((a.max() + 1, b.max() + 1), np.int64)
    np.add.at(t, (a, b), 1)
    r, c = linear_sum_assignment(-t)
    return t[r, c].sum() / a.size


@pytest.mark.parametrize("n,d,k,seed", [(2000, 2, 4, 0), (5000, 8, 16, 3), (20000, 16, 32, 5), (777, 3, 9, 1)])
def test_device_kmeans_matches_host_and_oracle(n, d, k, seed):
    rng = np.random.Generator(np.random.PCG64(seed))
    centres = rng.uniform(-5, 5, size=(k, d))
    pts = centres[rng.integers(0, k, size=n)] + rng.normal(0, 0.4, size=(n, d))
    dev = api.kmeans(pts, k, seed, device=0)
    host = api.kmeans(pts, k, seed)
    orc = O.kmeans(pts, k, seed)
    assert agreement(dev, orc) >= 0.999
    assert np.mean(dev == host) >= 0.999  # same label ids, not just the same partition


def test_device_kmeans_empty_cluster_split():
    """Duplicated points force empty clusters (cluster.cpp:96-115)."""
    pts = np.repeat(np.array([[0.0, 0.0], [1.0, 1.0], [5.0, 5.0]]), [50, 3, 1], axis=0)
    pts = np.concatenate([pts, np.array([[0.0, 0.0]] * 10)])
    dev = api.kmeans(pts, 5, 2, device=0)
    assert np.array_equal(dev, api.kmeans(pts, 5, 2))
    assert np.array_equal(dev, O.kmeans(pts, 5, 2))


def test_device_kmeans_on_c2_embedding():
    """Labels out of the C2 solve: GPU k-means agrees with the oracle's."""
    cfg = make_config("c2", scale=(96, 144))
    g, prm = cfg.graph, cfg.params
    y0 = api.random_embedding(g.n, prm.dim, cfg.y0_seed, g.degree)
    y = api.soc(g, prm, y0)
    t0 = time.perf_counter()
    dev = api.kmeans(y, cfg.k, 0, device=0)
    assert time.perf_counter() - t0 < 5.0
    assert agreement(dev, O.kmeans(y, cfg.k, 0)) >= 0.999
