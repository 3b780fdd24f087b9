"""Kernel lab driver (NOT product code): times the SpMV variants of
scripts/spmv_lab.cu on C5's operator A = (lambda/2) M^T M + (r/2) D in a
breadth-first storage order (like the library's), checks that every variant
gives the same bits as variant 0.

usage: python scripts/spmv_lab.py [variants...]
"""
import ctypes as C
import os
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))


def bfs_perm(n, indptr, indices):
    from scipy.sparse.csgraph import breadth_first_order, connected_components
    import scipy.sparse as sp

    g = sp.csr_matrix((np.ones(len(indices)), indices, indptr), shape=(n, n))
    ncomp, lab = connected_components(g, directed=False)
    order = []
    seen = np.zeros(n, bool)
    firsts = np.full(ncomp, -1)
    for v in range(n):  # components in order of their smallest vertex
        if firsts[lab[v]] < 0:
            firsts[lab[v]] = v
    for c in np.argsort(firsts):
        o = breadth_first_order(g, firsts[c], directed=False, return_predecessors=False)
        order.append(o)
    order = np.concatenate(order)
    perm = np.empty(n, np.int64)
    perm[order] = np.arange(n)
    return perm, ncomp


def main():
    import scipy.sparse as sp
    import torch

    from paper_1612_06496_b200.inputs import make_config

    t0 = time.time()
    cfg = make_config("c5")
    g, prm = cfg.graph, cfg.params
    n, d = g.n, prm.dim
    hl, dt = 0.5 * prm.lambda_, 0.5 * prm.r
    off = -((hl * g.w) * g.w)
    rows = np.concatenate([g.ei, g.ej])
    cols = np.concatenate([g.ej, g.ei])
    vals = np.concatenate([off, off])
    diag = np.zeros(n)
    np.add.at(diag, g.ei, (hl * g.w) * g.w)
    np.add.at(diag, g.ej, (hl * g.w) * g.w)
    diag = diag + dt * g.degree
    a = sp.csr_matrix((np.concatenate([vals, diag]), (np.concatenate([rows, np.arange(n)]),
                                                       np.concatenate([cols, np.arange(n)]))), shape=(n, n))
    lib = C.CDLL(str(ROOT / "scripts" / "libspmv_lab.so"))
    order = os.environ.get("LAB_ORDER", "bfs")
    if order.startswith("cluster"):
        csz = int(order[7:] or 64)
        perm = np.empty(n, np.int32)
        ip = a.indptr.astype(np.int32)
        ix = a.indices.astype(np.int32)
        lib.lab_cluster_order(n, ip.ctypes.data_as(C.c_void_p), ix.ctypes.data_as(C.c_void_p), csz,
                              perm.ctypes.data_as(C.c_void_p))
        ncomp = -1
    else:
        perm, ncomp = bfs_perm(n, a.indptr, a.indices)
    inv = np.argsort(perm)
    ap = a[inv][:, inv].tocsr()
    ap.sort_indices()
    print(f"order {order}", flush=True)
    print(f"C5 A: n={n} nnz={ap.nnz} components={ncomp} max row={np.diff(ap.indptr).max()} "
          f"build {time.time() - t0:.1f} s", flush=True)
    dev = torch.device("cuda:0")
    aptr = torch.tensor(ap.indptr.astype(np.int32), device=dev)
    acol = torch.tensor(ap.indices.astype(np.int32), device=dev)
    aval = torch.tensor(ap.data, device=dev)
    rng = np.random.default_rng(0)
    p = torch.tensor(rng.standard_normal((n, d)), device=dev)
    lib.lab_spmv.restype = C.c_int
    variants = [int(x) for x in sys.argv[1:]] or [0, 5, 20, 21, 22, 23, 24, 9]
    ref = None
    alg = 16 * n * d + 24 * (ap.nnz - n) // 2 + 12 * n
    for var in variants:
        q = torch.zeros((n, d), dtype=torch.float64, device=dev)
        ms = C.c_float(0)
        nb = lib.lab_spmv(var, n, C.c_void_p(aptr.data_ptr()), C.c_void_p(acol.data_ptr()),
                          C.c_void_p(aval.data_ptr()), C.c_void_p(p.data_ptr()), C.c_void_p(q.data_ptr()), int(os.environ.get("LAB_REPS", "20")),
                          C.byref(ms))
        torch.cuda.synchronize()
        if nb < 0:
            print(f"variant {var}: failed ({nb})", flush=True)
            continue
        qc = q.cpu().numpy()
        if var == 9:  # stream reference: not an SpMV
            if ms.value <= 0:
                continue
            print(f"variant  9 (stream reference): {ms.value * 1e3:8.1f} us  alg {alg / ms.value / 1e6:7.1f} GB/s",
                  flush=True)
            continue
        if ref is None:
            ref = qc
            ok = np.allclose(qc, (ap @ p.cpu().numpy()), rtol=1e-12, atol=1e-12)
        else:
            ok = np.array_equal(qc, ref)
        if ms.value <= 0:
            print(f"variant {var:2d}: launched once (LAB_REPS=0)", flush=True)
            continue
        print(f"variant {var:2d}: blocks/SM {nb} {ms.value * 1e3:8.1f} us  alg {alg / ms.value / 1e6:7.1f} GB/s "
              f"{'bitwise-equal' if ok else 'MISMATCH'}", flush=True)


if __name__ == "__main__":
    main()
