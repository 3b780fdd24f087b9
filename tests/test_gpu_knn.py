"""GPU k-NN graph builder (pfe_knn_graph) against the host builder
(inputs.knn_graph) on the same seeded point sets: identical edge lists,
sigma and weights (up to the last ulp of exp), degrees in edge order."""
import numpy as np
import pytest

from paper_1612_06496_b200 import api
from paper_1612_06496_b200.inputs import knn_graph, make_config

pytestmark = pytest.mark.gpu


def box_points(n, dim, seed):
    """Uniform points in a box (no outliers: the median-sigma heat kernel
    would isolate far outliers, which both builders reject)."""
    rng = np.random.Generator(np.random.PCG64(seed))
    return rng.uniform(-1.0, 1.0, size=(n, dim)) * rng.uniform(0.5, 2.0, size=dim)


@pytest.mark.parametrize("n,dim,k", [(2000, 2, 10), (5000, 16, 16), (3001, 3, 7), (1500, 9, 20), (700, 1, 5)])
def test_gpu_knn_matches_host_builder(n, dim, k):
    pts = box_points(n, dim, n + dim)
    host = knn_graph(pts, k)
    dev = api.knn_graph_gpu(pts, k)
    assert dev.n == host.n
    assert np.array_equal(dev.ei, host.ei) and np.array_equal(dev.ej, host.ej)
    assert dev.sigma == host.sigma
    np.testing.assert_allclose(dev.w, host.w, rtol=4e-16, atol=0)
    np.testing.assert_allclose(dev.degree, host.degree, rtol=1e-14, atol=0)


def test_gpu_knn_c1_config_graph():
    """C1's graph from the GPU builder equals the host-built one."""
    cfg = make_config("c1")
    rng = np.random.Generator(np.random.PCG64(0))
    centres = rng.uniform(-5.0, 5.0, size=(4, 2))
    comp = rng.integers(0, 4, size=2000)
    pts = centres[comp] + rng.normal(0.0, 0.3, size=(2000, 2))
    dev = api.knn_graph_gpu(pts, 10)
    assert np.array_equal(dev.ei, cfg.graph.ei) and np.array_equal(dev.ej, cfg.graph.ej)
    np.testing.assert_allclose(dev.w, cfg.graph.w, rtol=4e-16, atol=0)


def test_gpu_knn_rejects_bad_k():
    pts = box_points(10, 2, 1)
    with pytest.raises(api.ConfigError):
        api.knn_graph_gpu(pts, 10)
