"""Host-side logic of the multi-GPU row-band path, on CPU with torch.distributed
(gloo, world_size 2): the band plan of the library (pfe_band_plan), the halo
schedule (p' after SpMV, r after update, p' recomputed on the halo) and the
rank-ordered reduction of gathered per-band totals, replayed in numpy.  The
banded Jacobi-PCG must equal the single-domain one to rounding."""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1612_06496_b200 import api
from paper_1612_06496_b200.inputs import grid_graph, voronoi_image


def test_band_plan_partitions_rows():
    for H, P, R in [(321, 4, 1), (1024, 8, 2), (17, 2, 1), (10, 3, 2)]:
        owned = []
        for p in range(P):
            r0, r1, lo, hi = api.band_plan(H, P, R, p)
            owned.append((r0, r1))
            assert lo == (max(0, r0 - R) if p > 0 else r0)
            assert hi == (min(H, r1 + R) if p < P - 1 else r1)
            assert r1 - r0 >= H // P
        assert owned[0][0] == 0 and owned[-1][1] == H
        assert all(owned[i][1] == owned[i + 1][0] for i in range(P - 1))


def operator(g, lam=1.0, r=1.0):
    """Dense-ish A = (lam/2) M^T M + (r/2) D as a scipy CSR (reference order irrelevant here)."""
    import scipy.sparse as sp

    hl = 0.5 * lam
    a = sp.coo_matrix((np.r_[-hl * g.w * g.w, -hl * g.w * g.w], (np.r_[g.ei, g.ej], np.r_[g.ej, g.ei])),
                      shape=(g.n, g.n)).tocsr()
    diag = np.zeros(g.n)
    np.add.at(diag, g.ei, hl * g.w * g.w)
    np.add.at(diag, g.ej, hl * g.w * g.w)
    diag += 0.5 * r * g.degree
    return (a + sp.diags(diag)).tocsr(), diag


def banded_pcg(rank, P, g, W, R, b_glob, x0_glob, iters, comm):
    """Jacobi-PCG on band `rank` with the library's exchange schedule; fixed iterations."""
    A, diag = operator(g)
    r0, r1, lo, hi = api.band_plan(g.grid[0], P, R, rank)
    own = slice((r0 - lo) * W, (r1 - lo) * W)  # owned rows in local indexing
    loc = slice(lo * W, hi * W)
    A_own = A[r0 * W:r1 * W, lo * W:hi * W]
    invd = 1.0 / diag[loc]

    def halo(vec):  # refresh the R halo rows of a local vector from the neighbours
        if comm is None:
            return
        blk = R * W
        reqs = []
        import torch

        t = torch.from_numpy(vec)
        if rank > 0:
            reqs.append(dist.isend(t[(r0 - lo) * W:(r0 - lo) * W + blk].clone(), rank - 1))
            top = torch.empty(blk, dtype=torch.float64)
            reqs.append(dist.irecv(top, rank - 1))
        if rank < P - 1:
            reqs.append(dist.isend(t[(r1 - lo) * W - blk:(r1 - lo) * W].clone(), rank + 1))
            bot = torch.empty(blk, dtype=torch.float64)
            reqs.append(dist.irecv(bot, rank + 1))
        for q in reqs:
            q.wait()
        if rank > 0:
            vec[:blk] = top.numpy()
        if rank < P - 1:
            vec[(r1 - lo) * W:] = bot.numpy()

    def total(*vals):  # gather per-band totals, sum in rank order (identical on all bands)
        import torch

        mine = torch.tensor(vals, dtype=torch.float64)
        if comm is None:
            return list(mine.numpy())
        allv = [torch.empty_like(mine) for _ in range(P)]
        dist.all_gather(allv, mine)
        s = np.zeros(len(vals))
        for v in allv:
            s = s + v.numpy()
        return list(s)

    x = x0_glob[loc].copy()
    b = b_glob[loc]
    r = np.zeros_like(x)
    r[own] = b[own] - A_own @ x
    p = np.zeros_like(x)
    p[own] = invd[own] * r[own]
    bb, rr, rz = total(b[own] @ b[own], r[own] @ r[own], r[own] @ p[own])
    halo(p)
    beta = 0.0
    for k in range(1, iters + 1):
        if k > 1:
            p = invd * r + beta * p  # recomputed on owned + halo rows from exchanged r, p
        q = A_own @ p
        (pq,) = total(p[own] @ q)
        halo(p)
        alpha = rz / pq
        x[own] = x[own] + alpha * p[own]
        r[own] = r[own] - alpha * q
        rr, rz_new = total(r[own] @ r[own], r[own] @ (invd[own] * r[own]))
        halo(r)
        beta = rz_new / rz
        rz = rz_new
    return x[own], (r0, r1)


def _worker(rank, P, port, res_path):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=P)
    g, W, R, b, x0 = problem()
    xs, (r0, r1) = banded_pcg(rank, P, g, W, R, b, x0, 12, True)
    np.save(f"{res_path}_{rank}.npy", np.r_[r0, r1, xs])
    dist.destroy_process_group()


def problem():
    rng = np.random.Generator(np.random.PCG64(3))
    img, _ = voronoi_image(14, 11, 4, 0.05, rng)
    g = grid_graph(img, 0.1, 1)
    b = rng.normal(size=g.n)
    x0 = rng.normal(size=g.n)
    return g, 11, 1, b, x0


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def test_banded_pcg_two_ranks_gloo(tmp_path):
    P = 2
    res = str(tmp_path / "x")
    mp.spawn(_worker, args=(P, free_port(), res), nprocs=P, join=True)
    g, W, R, b, x0 = problem()
    full, _ = banded_pcg(0, 1, g, W, R, b, x0, 12, None)
    got = np.zeros(g.n)
    for rank in range(P):
        arr = np.load(f"{res}_{rank}.npy")
        r0, r1 = int(arr[0]), int(arr[1])
        got[r0 * W:r1 * W] = arr[2:]
    assert np.abs(got - full).max() <= 1e-12 * np.abs(full).max()


# ------------------------------------------------ IC(0) on row bands --------
def ic0_lower(A):
    """Row-oriented IC(0) of an SPD matrix on its own lower pattern (the
    sweep of sparse.cpp:124-203 without the shift retries: A here is strictly
    diagonally dominant)."""
    import scipy.sparse as sp

    n = A.shape[0]
    L = sp.tril(A).tolil()
    rows = [dict(zip(L.rows[i], L.data[i])) for i in range(n)]
    for i in range(n):
        for j in sorted(c for c in rows[i] if c < i):
            s = rows[i][j]
            for k, lik in rows[i].items():
                if k < j and k in rows[j]:
                    s -= lik * rows[j][k]
            rows[i][j] = s / rows[j][j]
        d = rows[i][i] - sum(v * v for c, v in rows[i].items() if c < i)
        assert d > 0.0
        rows[i][i] = np.sqrt(d)
    out = sp.lil_matrix((n, n))
    for i in range(n):
        for c, v in rows[i].items():
            out[i, c] = v
    return out.tocsr()


def banded_ic_pcg(rank, P, g, W, R, b_glob, x0_glob, iters, comm):
    """IC(0)-PCG on band `rank` with the library's schedule for partitioned
    solvers (pfe_band.cuh setup_team_ic / team_pcg): every rank holds the
    factor of the GLOBAL matrix, the owned rows of r are all-gathered into a
    global residual after the init and after every update, every rank applies
    the factor to it and takes z for its rows and its halo rows from the
    global z (no r halo exchange); r.z is computed on the global vectors."""
    import torch
    from scipy.sparse.linalg import spsolve_triangular

    A, _ = operator(g)
    L = ic0_lower(A)
    Lt = L.T.tocsr()
    r0, r1, lo, hi = api.band_plan(g.grid[0], P, R, rank)
    own = slice((r0 - lo) * W, (r1 - lo) * W)
    loc = slice(lo * W, hi * W)
    A_own = A[r0 * W:r1 * W, lo * W:hi * W]
    plans = [api.band_plan(g.grid[0], P, R, q) for q in range(P)]
    slot = max(q[1] - q[0] for q in plans) * W

    def gather_rows(vec_own):  # owned rows of every band -> the global vector
        if comm is None:
            return vec_own.copy()
        mine = torch.zeros(slot, dtype=torch.float64)
        mine[:vec_own.size] = torch.from_numpy(vec_own)
        allv = [torch.empty_like(mine) for _ in range(P)]
        dist.all_gather(allv, mine)
        full = np.zeros(g.n)
        for q, (q0, q1, _, _) in enumerate(plans):
            full[q0 * W:q1 * W] = allv[q].numpy()[:(q1 - q0) * W]
        return full

    def total(*vals):
        mine = torch.tensor(vals, dtype=torch.float64)
        if comm is None:
            return list(mine.numpy())
        allv = [torch.empty_like(mine) for _ in range(P)]
        dist.all_gather(allv, mine)
        s = np.zeros(len(vals))
        for v in allv:
            s = s + v.numpy()
        return list(s)

    def halo(vec):
        if comm is None:
            return
        blk = R * W
        t = torch.from_numpy(vec)
        reqs = []
        if rank > 0:
            reqs.append(dist.isend(t[(r0 - lo) * W:(r0 - lo) * W + blk].clone(), rank - 1))
            top = torch.empty(blk, dtype=torch.float64)
            reqs.append(dist.irecv(top, rank - 1))
        if rank < P - 1:
            reqs.append(dist.isend(t[(r1 - lo) * W - blk:(r1 - lo) * W].clone(), rank + 1))
            bot = torch.empty(blk, dtype=torch.float64)
            reqs.append(dist.irecv(bot, rank + 1))
        for q in reqs:
            q.wait()
        if rank > 0:
            vec[:blk] = top.numpy()
        if rank < P - 1:
            vec[(r1 - lo) * W:] = bot.numpy()

    def precondition(r_own):  # replicated: the same z and r.z on every rank
        r_full = gather_rows(r_own)
        z_full = spsolve_triangular(Lt, spsolve_triangular(L, r_full, lower=True), lower=False)
        return z_full, float(r_full @ z_full)

    x = x0_glob[loc].copy()
    b = b_glob[loc]
    r = np.zeros_like(x)
    r[own] = b[own] - A_own @ x
    z_full, rz = precondition(r[own])
    p = np.zeros_like(x)
    p[own] = z_full[r0 * W:r1 * W]
    halo(p)  # first iteration: p = z, halo rows exchanged like the library does
    beta = 0.0
    for k in range(1, iters + 1):
        if k > 1:
            p = z_full[loc] + beta * p  # owned + halo rows straight from the global z
        q = A_own @ p
        (pq,) = total(p[own] @ q)
        alpha = rz / pq
        x[own] = x[own] + alpha * p[own]
        r[own] = r[own] - alpha * q
        z_full, rz_new = precondition(r[own])
        beta = rz_new / rz
        rz = rz_new
    return x[own], (r0, r1)


def _ic_worker(rank, P, port, res_path):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=P)
    g, W, R, b, x0 = problem()
    xs, (r0, r1) = banded_ic_pcg(rank, P, g, W, R, b, x0, 8, True)
    np.save(f"{res_path}_{rank}.npy", np.r_[r0, r1, xs])
    dist.destroy_process_group()


def test_banded_ic0_pcg_two_ranks_gloo(tmp_path):
    """The IC(0) schedule of the partitioned solvers over two gloo ranks equals
    the single-domain IC(0)-PCG, and really preconditions (it converges faster
    than Jacobi on the same system)."""
    P = 2
    res = str(tmp_path / "xic")
    mp.spawn(_ic_worker, args=(P, free_port(), res), nprocs=P, join=True)
    g, W, R, b, x0 = problem()
    full, _ = banded_ic_pcg(0, 1, g, W, R, b, x0, 8, None)
    got = np.zeros(g.n)
    for rank in range(P):
        arr = np.load(f"{res}_{rank}.npy")
        r0, r1 = int(arr[0]), int(arr[1])
        got[r0 * W:r1 * W] = arr[2:]
    assert np.abs(got - full).max() <= 1e-12 * np.abs(full).max()
    A, _ = operator(g)
    jac, _ = banded_pcg(0, 1, g, W, R, b, x0, 8, None)
    res_ic = np.linalg.norm(b - A @ full)
    res_jac = np.linalg.norm(b - A @ jac)
    assert res_ic < 0.2 * res_jac


# ------------------------------------------------------------ vertex ranges --
def bfs_order(n, nbrs):
    """Storage order of the library's general-graph path (bfs_storage_order)."""
    pos = -np.ones(n, np.int64)
    nxt = 0
    queue = []
    for s0 in range(n):
        if pos[s0] >= 0:
            continue
        pos[s0] = nxt
        nxt += 1
        queue.append(s0)
        while queue:
            v = queue.pop(0)
            for u in nbrs[v]:
                if pos[u] < 0:
                    pos[u] = nxt
                    nxt += 1
                    queue.append(u)
    return pos


def range_problem():
    from conftest import random_graph

    rng = np.random.Generator(np.random.PCG64(9))
    g = random_graph(90, 200, rng)
    b = rng.normal(size=g.n)
    x0 = rng.normal(size=g.n)
    return g, b, x0


def ranged_pcg(rank, P, g, b_glob, x0_glob, iters, comm):
    """Jacobi-PCG on vertex range `rank` with the library's ghost schedule:
    owned vertices first, ghosts grouped by owner in storage order; p' is
    formed on owned rows and its ghosts exchanged before each SpMV."""
    A, diag = operator(g)
    nbrs = [[] for _ in range(g.n)]
    for i, j in zip(g.ei, g.ej):  # incidence in edge order
        nbrs[i].append(j)
        nbrs[j].append(i)
    pos = bfs_order(g.n, nbrs)
    vat = np.argsort(pos)
    starts = [g.n * q // P for q in range(P + 1)]
    owner = lambda ps: int(np.searchsorted(starts, ps, side="right") - 1)
    s0, s1 = starts[rank], starts[rank + 1]
    own = vat[s0:s1]
    ghost_pos = sorted({int(pos[u]) for v in own for u in nbrs[v] if not (s0 <= pos[u] < s1)})
    local = np.concatenate([own, vat[ghost_pos]]).astype(np.int64) if ghost_pos else own
    nown = len(own)
    A_loc = A[own][:, local]
    invd = 1.0 / diag[local]
    # exchange lists (rank -> peer): owned local rows adjacent to the peer's vertices
    send = {q: sorted({l for l, v in enumerate(own) for u in nbrs[v] if owner(pos[u]) == q})
            for q in range(P) if q != rank}
    recv = {q: [k + nown for k, ps in enumerate(ghost_pos) if owner(ps) == q] for q in range(P) if q != rank}

    def ghosts(vec):
        if comm is None:
            return
        import torch

        reqs, bufs = [], {}
        for q in send:
            if send[q]:
                reqs.append(dist.isend(torch.from_numpy(vec[send[q]].copy()), q))
            if recv[q]:
                bufs[q] = torch.empty(len(recv[q]), dtype=torch.float64)
                reqs.append(dist.irecv(bufs[q], q))
        for r in reqs:
            r.wait()
        for q, t in bufs.items():
            vec[recv[q]] = t.numpy()

    def total(*vals):
        import torch

        mine = torch.tensor(vals, dtype=torch.float64)
        if comm is None:
            return list(mine.numpy())
        allv = [torch.empty_like(mine) for _ in range(P)]
        dist.all_gather(allv, mine)
        s = np.zeros(len(vals))
        for v in allv:
            s = s + v.numpy()
        return list(s)

    o = slice(0, nown)
    x = x0_glob[local].copy()
    bb = b_glob[local]
    r = np.zeros_like(x)
    r[o] = bb[o] - A_loc @ x
    p = np.zeros_like(x)
    p[o] = invd[o] * r[o]
    _, _, rz = total(bb[o] @ bb[o], r[o] @ r[o], r[o] @ p[o])
    ghosts(p)
    beta = 0.0
    for k in range(1, iters + 1):
        if k > 1:
            p[o] = invd[o] * r[o] + beta * p[o]
            ghosts(p)
        q = A_loc @ p
        (pq,) = total(p[o] @ q)
        alpha = rz / pq
        x[o] = x[o] + alpha * p[o]
        r[o] = r[o] - alpha * q
        _, rz_new = total(r[o] @ r[o], r[o] @ (invd[o] * r[o]))
        beta = rz_new / rz
        rz = rz_new
    return x[o], own


def _range_worker(rank, P, port, res_path):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=P)
    g, b, x0 = range_problem()
    xs, own = ranged_pcg(rank, P, g, b, x0, 10, True)
    np.save(f"{res_path}_{rank}.npy", np.stack([own.astype(np.float64), xs]))
    dist.destroy_process_group()


def test_vertex_range_pcg_two_ranks_gloo(tmp_path):
    P = 2
    res = str(tmp_path / "v")
    mp.spawn(_range_worker, args=(P, free_port(), res), nprocs=P, join=True)
    g, b, x0 = range_problem()
    full, own = ranged_pcg(0, 1, g, b, x0, 10, None)
    ref = np.zeros(g.n)
    ref[own] = full
    got = np.zeros(g.n)
    for rank in range(P):
        arr = np.load(f"{res}_{rank}.npy")
        got[arr[0].astype(np.int64)] = arr[1]
    assert np.abs(got - ref).max() <= 1e-12 * np.abs(ref).max()
