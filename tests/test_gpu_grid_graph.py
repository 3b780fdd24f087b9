"""GPU pixel-grid graph builder (pfe_grid_graph) against
the host builder inputs.grid_graph (graph.cpp:105-159 semantics: heat kernel,
1e-12 drop, isolated-pixel repair, lexicographic edges, edge-order degree).

The edge lists must be identical; weights agree up to the last ulp of exp
(CUDA's exp vs the host libm's), and the measured mismatch is printed."""
import time

import numpy as np
import pytest

from paper_1612_06496_b200 import api
from paper_1612_06496_b200.inputs import grid_graph, make_config, voronoi_image

pytestmark = pytest.mark.gpu


def ulps(a, b):
    ia = np.asarray(a, np.float64).view(np.int64)
    ib = np.asarray(b, np.float64).view(np.int64)
    return np.abs(ia - ib)


def compare(host, dev, label):
    assert dev.n == host.n and dev.grid == host.grid
    assert dev.m == host.m, f"{label}: {dev.m} vs {host.m} edges"
    assert np.array_equal(dev.ei, host.ei) and np.array_equal(dev.ej, host.ej)
    u = ulps(dev.w, host.w)
    rel_deg = np.max(np.abs(dev.degree - host.degree) / host.degree)
    print(f"{label}: n={host.n} m={host.m} weights differing {np.count_nonzero(u)} "
          f"(max {u.max() if u.size else 0} ulp), degree max rel diff {rel_deg:.2e}")
    assert u.max() <= 1
    assert rel_deg <= 1e-15


@pytest.mark.parametrize("h,w,radius,sxy", [(37, 53, 1, None), (40, 41, 2, 2.0), (1, 9, 1, None), (9, 1, 2, None),
                                             (64, 96, 2, None)])
def test_grid_builder_matches_host(h, w, radius, sxy):
    rng = np.random.Generator(np.random.PCG64(h * 100 + w))
    img, _ = voronoi_image(h, w, 5, 0.05, rng)
    compare(grid_graph(img, 0.1, radius, sxy), api.grid_graph_gpu(img, 0.1, radius, sxy), f"{h}x{w} r={radius}")


def test_grid_builder_isolated_pixel_repair():
    """Pixels whose every candidate weight is below 1e-12 keep their strongest
    candidate, floored at 1e-12 (graph.cpp:135-142); adjacent isolated pixels
    that pick the same edge add it once."""
    img = np.zeros((12, 15, 3))
    img[3, 4] = 1.0            # one isolated pixel
    img[8, 8] = img[8, 9] = 1.0  # a pair: joined to each other, not isolated
    img[10, 2] = [1.0, 0.0, 0.0]
    img[10, 3] = [0.0, 1.0, 0.0]  # two adjacent pixels, isolated from everything
    img[0, 14] = 1.0           # a corner
    for radius in (1, 2):
        host = grid_graph(img, 0.1, radius)
        dev = api.grid_graph_gpu(img, 0.1, radius)
        compare(host, dev, f"isolated r={radius}")
        assert np.all(dev.degree > 0)


@pytest.mark.slow
@pytest.mark.parametrize("name", ["c2", "c3", "c4"])
def test_grid_builder_full_configs(name):
    """The configs' graphs (C4: 16.8 M pixels, 67 M edges) built on the GPU,
    timed beside the host builder."""
    cfg = make_config(name, seed=0)
    host = cfg.graph
    img = cfg.image
    h, w, radius = host.grid
    sxy = 2.0 if name == "c3" else None
    api.grid_graph_gpu(img[:8, :8], 0.1, radius, sxy)  # warm-up (context, module load)
    t0 = time.time()
    dev = api.grid_graph_gpu(img, 0.1, radius, sxy)
    t_gpu = time.time() - t0
    t0 = time.time()
    grid_graph(img, 0.1, radius, sxy)
    t_host = time.time() - t0
    print(f"{name}: GPU builder {t_gpu:.3f} s (incl. host<->device copies), numpy builder {t_host:.2f} s")
    compare(host, dev, name)
