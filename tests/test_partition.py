"""Vertex-range partition of general graphs (pfe_band.cuh):
host-only statistics against an independent numpy/scipy restatement (BFS in
vertex order over components, neighbours ascending = incidence order of
lexicographic edge lists; contiguous ranges n*q/P)."""
import numpy as np
import pytest
from scipy.sparse import csr_matrix
from scipy.sparse.csgraph import breadth_first_order

from paper_1612_06496_b200 import api
from paper_1612_06496_b200.inputs import knn_graph


def bfs_positions(g):
    a = csr_matrix((np.ones(2 * g.m), (np.r_[g.ei, g.ej], np.r_[g.ej, g.ei])), shape=(g.n, g.n))
    a.sort_indices()
    pos = np.full(g.n, -1)
    nxt = 0
    for s in range(g.n):
        if pos[s] >= 0:
            continue
        order = breadth_first_order(a, s, directed=False, return_predecessors=False)
        pos[order] = np.arange(nxt, nxt + len(order))
        nxt += len(order)
    return pos


@pytest.mark.parametrize("parts", [2, 3, 5])
def test_range_partition_stats_match_restatement(parts):
    rng = np.random.Generator(np.random.PCG64(4))
    pts = np.concatenate([rng.normal(size=(300, 4)), rng.normal(size=(200, 4)) + 8.0])  # two components
    g = knn_graph(pts, 6)
    st = api.range_partition_stats(g, parts)
    pos = bfs_positions(g)
    start = (g.n * np.arange(parts + 1)) // parts
    owner = np.searchsorted(start, pos, side="right") - 1
    for r in range(parts):
        gh, snd = set(), set()
        for i, j in zip(g.ei, g.ej):
            for a, b in ((i, j), (j, i)):
                if owner[a] == r and owner[b] != r:
                    gh.add(pos[b])
                    snd.add((owner[b], a))
        assert st["owned"][r] == start[r + 1] - start[r]
        assert st["ghosts"][r] == len(gh)
        assert st["sends"][r] == len(snd)
    assert st["owned"].sum() == g.n

