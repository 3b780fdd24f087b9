import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))
if str(ROOT / "tests") not in sys.path:
    sys.path.insert(0, str(ROOT / "tests"))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) GPU and the built libpfe_b200.so")
    config.addinivalue_line("markers", "slow: long-running parity case")


def random_graph(n, extra_edges, rng):
    """Restates oracles.hpp:40-69: a shuffled chain covering every vertex plus
    extra random edges, weights U(0.1, 2), lexicographic, degree in edge order."""
    from paper_1612_06496_b200.api import WeightedGraph

    order = rng.permutation(n)
    edges = {}
    for t in range(n - 1):
        a, b = int(min(order[t], order[t + 1])), int(max(order[t], order[t + 1]))
        edges[(a, b)] = rng.uniform(0.1, 2.0)
    for _ in range(extra_edges):
        a, b = int(rng.integers(0, n)), int(rng.integers(0, n))
        if a == b:
            continue
        edges[(min(a, b), max(a, b))] = rng.uniform(0.1, 2.0)
    keys = sorted(edges)
    ei = np.array([k[0] for k in keys], np.int32)
    ej = np.array([k[1] for k in keys], np.int32)
    w = np.array([edges[k] for k in keys])
    deg = np.zeros(n)
    for i, j, x in zip(ei, ej, w):
        deg[i] += x
        deg[j] += x
    return WeightedGraph(n, ei, ej, w, deg)


@pytest.fixture
def rng():
    return np.random.Generator(np.random.PCG64(12345))
