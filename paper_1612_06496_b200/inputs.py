"""Seeded synthetic inputs for the five BASELINE.json configurations.

These stand in for the reference's data (BSDS500 images, are
not in this image): same shapes, sizes and value distributions as
BASELINE.json states, generated from a fixed numpy PCG64 seed.  The graph
builders generalise build_image_graph (graph.cpp:105-159) to the 8-neighbour
and 5x5 neighbourhoods the configs need: heat-kernel weights, weights below
1e-12 dropped, an isolated vertex keeps its strongest incident edge (weight
floored at 1e-12), edges sorted lexicographically (i < j), degree summed in
edge order (graph.cpp:15-22).  Under-specified parameters are fixed as
SURVEY.md Appendix A recommends and recorded in DESIGN.md §7.
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import Optional, Tuple

import numpy as np

from .api import PcgConfig, PfeParams, Preconditioner, WeightedGraph

WEIGHT_FLOOR = 1e-12

# forward stencil offsets (dy, dx) in lexicographic edge order
OFFSETS = {
    1: [(0, 1), (1, -1), (1, 0), (1, 1)],
    2: [(0, 1), (0, 2), (1, -2), (1, -1), (1, 0), (1, 1), (1, 2), (2, -2), (2, -1), (2, 0), (2, 1), (2, 2)],
}


def _degree(n, ei, ej, w):
    # For lexicographic (i < j) edge lists every vertex sees all its "j"
    # contributions before its "i" contributions, so two ordered passes
    # reproduce degrees_from_edges' per-vertex summation order.
    d = np.zeros(n)
    np.add.at(d, ej, w)
    np.add.at(d, ei, w)
    return d


def grid_graph(rgb: np.ndarray, sigma_rgb: float, radius: int = 1, sigma_xy: Optional[float] = None) -> WeightedGraph:
    """Heat-kernel pixel graph on an (H, W, 3) image over the (2r+1)^2-1 neighbourhood.

    w = exp(-|drgb|^2 / (2 sigma_rgb^2) - |dxy|^2 / (2 sigma_xy^2)) (xy term only if sigma_xy).
    """
    h, wd, _ = rgb.shape
    n = h * wd
    feats = rgb.reshape(n, 3)
    offs = OFFSETS[radius]
    S = len(offs)
    inv_rgb = 1.0 / (2.0 * sigma_rgb * sigma_rgb)
    inv_xy = 0.0 if sigma_xy is None else 1.0 / (2.0 * sigma_xy * sigma_xy)
    yy, xx = np.divmod(np.arange(n, dtype=np.int64), wd)
    W = np.full((n, S), -1.0)  # candidate weights; -1 = no neighbour
    J = np.full((n, S), -1, dtype=np.int64)
    for s, (dy, dx) in enumerate(offs):
        ok = (yy + dy < h) & (xx + dx >= 0) & (xx + dx < wd)
        i = np.nonzero(ok)[0]
        j = i + dy * wd + dx
        d2 = ((feats[i] - feats[j]) ** 2).sum(axis=1)
        e = d2 * inv_rgb
        if sigma_xy is not None:
            e = e + float(dy * dy + dx * dx) * inv_xy
        W[i, s] = np.exp(-e)
        J[i, s] = j
    cand = J >= 0
    keep = cand & (W >= WEIGHT_FLOOR)
    I = np.broadcast_to(np.arange(n)[:, None], (n, S))
    ei, ej, ew = I[keep], J[keep], W[keep]
    has = np.zeros(n, bool)
    has[ei] = True
    has[ej] = True
    iso = np.nonzero(~has)[0]
    if iso.size:
        # strongest incident candidate, first in edge order on ties (graph.cpp:357-364)
        ci, cj, cw = I[cand], J[cand], W[cand]
        extra = {}
        for v in iso:
            sel = np.nonzero((ci == v) | (cj == v))[0]
            k = sel[np.argmax(cw[sel])]
            extra[(int(ci[k]), int(cj[k]))] = max(float(cw[k]), WEIGHT_FLOOR)
        ei = np.concatenate([ei, np.array([a for a, _ in extra], dtype=np.int64)])
        ej = np.concatenate([ej, np.array([b for _, b in extra], dtype=np.int64)])
        ew = np.concatenate([ew, np.array(list(extra.values()))])
        order = np.lexsort((ej, ei))
        ei, ej, ew = ei[order], ej[order], ew[order]
        dup = np.concatenate([[False], (ei[1:] == ei[:-1]) & (ej[1:] == ej[:-1])])
        ei, ej, ew = ei[~dup], ej[~dup], ew[~dup]
    deg = _degree(n, ei, ej, ew)
    return WeightedGraph(n, ei.astype(np.int32), ej.astype(np.int32), ew, deg, sigma_rgb, grid=(h, wd, radius))


def knn_graph(points: np.ndarray, k: int, gpu: bool = False) -> WeightedGraph:
    """Union-symmetrised k-NN graph, heat kernel with sigma = median directed k-NN distance.

    w_ij = exp(-|x_i - x_j|^2 / (2 sigma^2)) once per unordered pair (not summed).
    Brute force on the host (the small C1 configuration and tests), or on the
    GPU with ``gpu=True`` (pfe_knn_graph; C5).
    """
    if gpu:
        from .api import knn_graph_gpu

        return knn_graph_gpu(points, k)
    n = points.shape[0]
    sq = (points ** 2).sum(1)
    nbr = np.empty((n, k), dtype=np.int64)
    dist = np.empty((n, k))
    step = max(1, 4096 * 64 // max(n, 1))
    for lo in range(0, n, step):
        hi = min(n, lo + step)
        d2 = sq[lo:hi, None] + sq[None, :] - 2.0 * points[lo:hi] @ points.T
        # exact distances for the candidates
        d2[np.arange(hi - lo), np.arange(lo, hi)] = np.inf
        idx = np.argpartition(d2, k, axis=1)[:, :k]
        exact = ((points[lo:hi, None, :] - points[idx]) ** 2).sum(-1)
        o = np.lexsort((idx, exact), axis=1)
        nbr[lo:hi] = np.take_along_axis(idx, o, 1)
        dist[lo:hi] = np.sqrt(np.take_along_axis(exact, o, 1))
    sigma = float(np.median(dist))
    a = np.repeat(np.arange(n), k)
    b = nbr.reshape(-1)
    i, j = np.minimum(a, b), np.maximum(a, b)
    key = np.unique(i * n + j)
    ei, ej = key // n, key % n
    d2 = ((points[ei] - points[ej]) ** 2).sum(1)
    w = np.exp(-d2 / (2.0 * sigma * sigma))
    keep = w >= WEIGHT_FLOOR
    ei, ej, w = ei[keep], ej[keep], w[keep]
    deg = _degree(n, ei, ej, w)
    if np.any(deg <= 0):
        raise ValueError("knn_graph: isolated vertex")
    return WeightedGraph(n, ei.astype(np.int32), ej.astype(np.int32), w, deg, sigma)


def voronoi_labels(h: int, w: int, sites: np.ndarray) -> np.ndarray:
    """Nearest-site label per pixel (ties to the lowest site index)."""
    from scipy.spatial import cKDTree

    yy, xx = np.mgrid[0:h, 0:w]
    pix = np.stack([yy.ravel() + 0.5, xx.ravel() + 0.5], 1)
    _, lab = cKDTree(sites).query(pix, k=1)
    return lab.reshape(h, w)


@dataclass
class Config:
    name: str
    graph: WeightedGraph
    params: PfeParams
    k: int            # k-means clusters for "labels out"
    y0_seed: int
    truth: Optional[np.ndarray] = None
    description: str = ""
    image: Optional[np.ndarray] = None  # (H, W, 3) RGB of the image configs


def _params(d, soc, sb, tol):
    # lambda = r = 1, Jacobi-PCG max 50, fixed counts (conv_tol 0), no Stage II
    #
    return PfeParams(dim=d, lambda_=1.0, r=1.0, soc_max=soc, sb_max_stage1=sb, sb_max_stage2=0, conv_tol=0.0,
                     pcg=PcgConfig(rel_tol=tol, max_iter=50, preconditioner=Preconditioner.Jacobi))


def voronoi_image(h, w, regions, noise, rng, gradient=0.0):
    sites = rng.uniform([0, 0], [h, w], size=(regions, 2))
    lab = voronoi_labels(h, w, sites)
    cols = rng.uniform(0.0, 1.0, size=(regions, 3))
    img = cols[lab]
    if gradient:
        G = rng.normal(0.0, gradient, size=(regions, 3, 2))
        yy, xx = np.mgrid[0:h, 0:w]
        dy = yy + 0.5 - sites[lab, 0]
        dx = xx + 0.5 - sites[lab, 1]
        img = img + G[lab, :, 0] * dy[..., None] + G[lab, :, 1] * dx[..., None]
    img = img + rng.normal(0.0, noise, size=img.shape)
    return np.clip(img, 0.0, 1.0), lab


def make_config(name: str, seed: int = 0, scale: Optional[Tuple[int, int]] = None) -> Config:
    """Builds configuration C1..C5 of BASELINE.json (``scale`` shrinks image configs for tests)."""
    rng = np.random.Generator(np.random.PCG64(seed))
    name = name.lower()
    if name == "c1":
        centres = rng.uniform(-5.0, 5.0, size=(4, 2))
        comp = rng.integers(0, 4, size=2000)
        pts = centres[comp] + rng.normal(0.0, 0.3, size=(2000, 2))
        g = knn_graph(pts, 10)
        return Config("c1", g, _params(3, 10, 20, 1e-6), 4, seed, comp,
                      "2000 points in R^2, 4 Gaussians, sym. 10-NN, d=3, 10x20")
    if name == "c2":
        h, w = scale or (321, 481)
        img, lab = voronoi_image(h, w, 8, 0.05, rng)
        g = grid_graph(img, 0.1, 1)
        return Config("c2", g, _params(4, 10, 20, 1e-6), 8, seed, lab.ravel(),
                      f"{w}x{h} Voronoi RGB (8 regions, noise 0.05), 8-nbr grid, d=4, 10x20", img)
    if name == "c3":
        h, w = scale or (1024, 1024)
        img, lab = voronoi_image(h, w, 32, 0.03, rng, gradient=1.0 / 512.0)
        g = grid_graph(img, 0.1, 2, sigma_xy=2.0)
        return Config("c3", g, _params(8, 10, 30, 1e-7), 32, seed, lab.ravel(),
                      f"{w}x{h} Voronoi RGB with gradients (32 regions), 5x5 grid RGB+xy, d=8, 10x30", img)
    if name == "c4":
        h, w = scale or (4096, 4096)
        img, lab = voronoi_image(h, w, 256, 0.05, rng)
        g = grid_graph(img, 0.1, 1)
        return Config("c4", g, _params(8, 5, 20, 1e-6), 256, seed, lab.ravel(),
                      f"{w}x{h} Voronoi RGB (256 regions), 8-nbr grid, d=8, 5x20", img)
    if name == "c5":
        n = scale[0] if scale else 1_000_000
        means = rng.uniform(-10.0, 10.0, size=(32, 16))
        stds = rng.uniform(0.5, 1.5, size=32)
        wts = rng.exponential(1.0, size=32)
        wts /= wts.sum()
        comp = rng.choice(32, size=n, p=wts)
        pts = means[comp] + rng.normal(size=(n, 16)) * stds[comp, None]
        g = knn_graph(pts, 16, gpu=True)  # 10^6 points: built once on the GPU (timed separately)
        return Config("c5", g, _params(16, 10, 20, 1e-6), 32, seed, comp,
                      f"{n} points in R^16, 32-component GMM, sym. 16-NN, d=16, 10x20")
    raise ValueError(f"unknown config {name}")
