"""General-graph solver topology built on the GPU (csrc/pfe_csrbuild.cu)
against the host builder (pfe_runtime.cu build_topology): the two must give
bit-identical solves, split states included, on k-NN graphs, graphs with
duplicate and unordered edges and graphs with several components."""
import os

import numpy as np
import pytest

import oracle as O
from conftest import random_graph
from paper_1612_06496_b200 import api
from paper_1612_06496_b200.inputs import knn_graph

pytestmark = pytest.mark.gpu


class builder:
    def __init__(self, device: bool):
        self.env = {"PFE_DEVICE_CSR": "1" if device else "0", "PFE_HOST_TOPOLOGY": "0" if device else "1"}

    def __enter__(self):
        self.old = {k: os.environ.get(k) for k in self.env}
        os.environ.update(self.env)

    def __exit__(self, *a):
        for k, v in self.old.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v


def params(d, soc=2, sb=4, stage2=0):
    return api.PfeParams(dim=d, lambda_=1.0, r=1.0, soc_max=soc, sb_max_stage1=sb, sb_max_stage2=stage2,
                         conv_tol=0.0, pcg=api.PcgConfig(1e-6, 50, api.Preconditioner.Jacobi))


def run(g, prm, y0, device):
    with builder(device):
        s = api.PfeSolver(g, prm)
        st = s.make_state(y0)
        s.run_soc(st, prm.soc_max, prm.sb_max_stage1)
        out = (st.y.copy(), st.split_b.copy(), st.split_s.copy(), s.pcg_log()[0].copy(), s.report()["setup_seconds"])
        st.close()
        s.close()
    return out


def same(a, b):
    for x, y in zip(a[:4], b[:4]):
        assert np.array_equal(x, y)


@pytest.mark.parametrize("n,k,d", [(1500, 8, 4), (3000, 5, 16), (700, 12, 3)])
def test_knn_graph_device_build_bitwise(n, k, d):
    rng = np.random.Generator(np.random.PCG64(n + k))
    g = knn_graph(rng.uniform(-1.0, 1.0, size=(n, 3)), k)
    prm = params(d)
    y0 = api.random_embedding(g.n, d, 1, g.degree)
    dev, host = run(g, prm, y0, True), run(g, prm, y0, False)
    same(dev, host)
    exp = O.solve(g, prm, y0, mode=0)
    sgn = np.sign((dev[0] * exp).sum(0))
    assert np.linalg.norm(dev[0] * sgn - exp) / np.linalg.norm(exp) <= 1e-10


def test_duplicate_unordered_edges_and_components_device_build_bitwise():
    """Three components of different sizes, edge list shuffled, some edges
    repeated (duplicate columns are summed in edge order), one weight pair
    cancelling is not possible for w > 0, so also a zero-weight edge (its
    off-diagonal entry is an exact zero and is dropped from A)."""
    rng = np.random.Generator(np.random.PCG64(11))
    parts = [random_graph(90, 200, rng), random_graph(40, 60, rng), random_graph(7, 5, rng)]
    off, ei, ej, w = 0, [], [], []
    for p in parts:
        ei.append(p.ei + off)
        ej.append(p.ej + off)
        w.append(p.w)
        off += p.n
    ei, ej, w = np.concatenate(ei), np.concatenate(ej), np.concatenate(w)
    dup = rng.integers(0, ei.size, size=40)
    ei, ej, w = np.r_[ei, ei[dup]], np.r_[ej, ej[dup]], np.r_[w, rng.uniform(0.1, 2.0, size=40)]
    w[5] = 0.0
    sh = rng.permutation(ei.size)
    ei, ej, w = ei[sh].astype(np.int32), ej[sh].astype(np.int32), w[sh]
    deg = np.zeros(off)
    for i, j, x in zip(ei, ej, w):
        deg[i] += x
        deg[j] += x
    g = api.WeightedGraph(off, ei, ej, w, deg)
    prm = params(5, soc=2, sb=3)
    y0 = api.random_embedding(g.n, 5, 2, g.degree)
    dev, host = run(g, prm, y0, True), run(g, prm, y0, False)
    same(dev, host)
    exp = O.solve(g, prm, y0, mode=0)
    sgn = np.sign((dev[0] * exp).sum(0))
    assert np.linalg.norm(dev[0] * sgn - exp) / np.linalg.norm(exp) <= 1e-10


def test_many_components_fall_back_to_host_builder():
    """More components than the device breadth-first search accepts: the
    solver is built on the host and still solves."""
    n = 2 * 5000
    ei = np.arange(0, n, 2, dtype=np.int32)
    ej = ei + 1
    w = np.full(ei.size, 0.5)
    g = api.WeightedGraph(n, ei, ej, w, np.full(n, 0.5))
    prm = params(2, soc=1, sb=2)
    y0 = api.random_embedding(g.n, 2, 3, g.degree)
    dev, host = run(g, prm, y0, True), run(g, prm, y0, False)
    same(dev, host)


def test_chain_like_graph_falls_back_to_host_builder():
    """A path graph has n breadth-first levels: the level-synchronous device
    search gives up after 16384 levels and the host builder takes over (the
    default builder choice: m >= 2^17 edges selects the device path)."""
    n = (1 << 17) + 50
    ei = np.arange(0, n - 1, dtype=np.int32)
    ej = ei + 1
    w = np.full(ei.size, 0.7)
    deg = np.full(n, 1.4)
    deg[0] = deg[-1] = 0.7
    g = api.WeightedGraph(n, ei, ej, w, deg)
    prm = params(2, soc=1, sb=2)
    y0 = api.random_embedding(g.n, 2, 3, g.degree)
    s = api.PfeSolver(g, prm)  # default switches
    st = s.make_state(y0)
    s.run_soc(st, 1, 2)
    y_default = st.y.copy()
    setup = s.report()["setup_seconds"]
    st.close()
    s.close()
    host = run(g, prm, y0, False)
    assert np.array_equal(y_default, host[0])
    assert setup < 20.0
