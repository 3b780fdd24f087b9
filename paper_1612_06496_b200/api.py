"""Python host mirror of the reference solver interface (namespace ``pfe`` in
/root/reference/proj/core/include/pfe/*.hpp), backed by the sm_100a library.

Same names, argument meaning and error behaviour as the reference:

=====================================  ==========================================
reference (C++)                        here
=====================================  ==========================================
``PfeParams`` (solver.hpp:16-25)        :class:`PfeParams`
``PcgConfig`` / ``Preconditioner``      :class:`PcgConfig` / :class:`Preconditioner`
``PcgReport`` (pcg.hpp:21-26)           :class:`PcgReport`
``WeightedGraph`` (graph.hpp:15-28)     :class:`WeightedGraph`
``SolverState`` (solver.hpp:28-34)      :class:`SolverState` (device resident)
``PfeSolver`` (solver.hpp:51-83)        :class:`PfeSolver`
``split_bregman`` free (solver.cpp:138) :func:`split_bregman`
``soc`` / ``pfe_two_stage``             :func:`soc` / :func:`pfe_two_stage`
``objective`` / ``shrink``              :func:`objective` / :func:`shrink`
``project_orthogonal``                  :func:`project_orthogonal`
``PcgOperator`` / ``pcg_solve_multi``   :class:`PcgOperator` / :func:`pcg_solve_multi`
``random_embedding`` / ``d_orthonormalize`` (init.cpp:140-181)
``kmeans`` (cluster.cpp:54-124)         :func:`kmeans` (labels out)
``IoError`` / ``NumericalError`` / ``ConfigError`` (errors.hpp:9-24)
=====================================  ==========================================

Matrices are numpy ``(rows, d)`` float64 arrays; they are handed to the C ABI
in column-major order (the reference's Eigen layout).
"""
from __future__ import annotations

import ctypes as C
import enum
from dataclasses import dataclass, field
from typing import Callable, List, Optional, Tuple

import numpy as np

from . import _native as N


class IoError(RuntimeError):
    pass


class NumericalError(RuntimeError):
    pass


class ConfigError(ValueError):
    pass


class CudaError(RuntimeError):
    pass


_EXC = {N.PFE_IO_ERROR: IoError, N.PFE_NUMERICAL_ERROR: NumericalError, N.PFE_CONFIG_ERROR: ConfigError,
        N.PFE_CUDA_ERROR: CudaError}


def _check(rc: int) -> None:
    if rc != N.PFE_OK:
        msg = N.load().pfe_last_error().decode(errors="replace")
        raise _EXC.get(rc, CudaError)(msg)


class Preconditioner(enum.IntEnum):
    Ic0 = 0
    Jacobi = 1
    NONE = 2


@dataclass
class PcgConfig:
    rel_tol: float = 1e-6
    max_iter: int = 1000
    preconditioner: Preconditioner = Preconditioner.Ic0


@dataclass
class PcgReport:
    iterations: int = 0
    final_rel_residual: float = 0.0
    converged: bool = False
    jacobi_fallback: bool = False


@dataclass
class PfeParams:
    dim: int = 5
    lambda_: float = 100.0
    r: float = 1.0
    soc_max: int = 10
    sb_max_stage1: int = 5
    sb_max_stage2: int = 100
    conv_tol: float = 1e-4
    pcg: PcgConfig = field(default_factory=PcgConfig)

    def to_c(self) -> N.pfe_params:
        return N.pfe_params(int(self.dim), float(self.lambda_), float(self.r), int(self.soc_max),
                            int(self.sb_max_stage1), int(self.sb_max_stage2), float(self.conv_tol),
                            float(self.pcg.rel_tol), int(self.pcg.max_iter), int(self.pcg.preconditioner))


@dataclass
class WeightedGraph:
    """Undirected graph, edges (i < j) in lexicographic order, degree used as given.

    ``grid`` = (height, width, radius) marks a pixel grid whose edges are
    stencil neighbours (radius 1: 8-neighbour, 2: 5x5); the solver then
    uses the stencil kernels.  Results do not depend on the hint.
    """
    n: int
    ei: np.ndarray
    ej: np.ndarray
    w: np.ndarray
    degree: np.ndarray
    sigma: float = 0.0
    grid: Optional[Tuple[int, int, int]] = None

    def __post_init__(self):
        self.ei = np.ascontiguousarray(self.ei, dtype=np.int32)
        self.ej = np.ascontiguousarray(self.ej, dtype=np.int32)
        self.w = np.ascontiguousarray(self.w, dtype=np.float64)
        self.degree = np.ascontiguousarray(self.degree, dtype=np.float64)

    @property
    def m(self) -> int:
        return int(self.w.shape[0])

    def edge_count(self) -> int:
        return self.m

    def to_c(self) -> N.pfe_graph:
        h, w, r = self.grid if self.grid else (0, 0, 0)
        return N.pfe_graph(int(self.n), int(self.m), N.iptr(self.ei), N.iptr(self.ej), N.dptr(self.w),
                           N.dptr(self.degree), int(h), int(w), int(r))


def degree_vector(ei, ej, w, n) -> np.ndarray:
    """graph.cpp:15-22: weighted degree, accumulated in edge order."""
    d = np.zeros(n)
    for i, j, x in zip(np.asarray(ei), np.asarray(ej), np.asarray(w)):
        d[i] += x
        d[j] += x
    return d


def _exec(device=0, use_graphs=True, warn=True, profile=False, persistent=True) -> N.pfe_exec:
    # persistent: True (shared-memory-resident kernel when the state fits),
    # "tiled" (persistent kernel streaming tiles from HBM/L2), False (one kernel per phase)
    mode = 2 if persistent == "tiled" else (persistent if type(persistent) is int else int(bool(persistent)))
    return N.pfe_exec(int(device), int(bool(use_graphs)), int(bool(warn)), int(bool(profile)), mode)


def _colmajor(a, rows=None, cols=None) -> np.ndarray:
    a = np.asarray(a, dtype=np.float64)
    if a.ndim == 1:
        a = a.reshape(-1, 1)
    if rows is not None and a.shape[0] != rows or cols is not None and a.shape[1] != cols:
        raise ConfigError("PfeSolver: initial embedding has wrong shape")
    return np.asfortranarray(a)


def _from_colmajor(buf: np.ndarray, rows: int, cols: int) -> np.ndarray:
    return np.array(buf.reshape(cols, rows).T, order="F")


_FIELDS = {"y": 0, "p": 1, "bregman": 2, "split_b": 3, "split_s": 4}


class SolverState:
    """Device-resident SolverState; fields download on access, upload on assignment."""

    def __init__(self, solver: "PfeSolver", handle: C.c_void_p):
        self._solver = solver
        self._h = handle

    def _rows(self, name):
        return self._solver.graph.m if name in ("split_b", "split_s") else self._solver.graph.n

    def _get(self, name):
        rows, d = self._rows(name), self._solver.params.dim
        buf = np.empty(rows * d)
        _check(N.load().pfe_state_get(self._h, _FIELDS[name], N.dptr(buf)))
        return _from_colmajor(buf, rows, d)

    def _set(self, name, value):
        arr = _colmajor(value, self._rows(name), self._solver.params.dim)
        _check(N.load().pfe_state_set(self._h, _FIELDS[name], N.dptr(arr)))

    y = property(lambda s: s._get("y"), lambda s, v: s._set("y", v))
    p = property(lambda s: s._get("p"), lambda s, v: s._set("p", v))
    bregman = property(lambda s: s._get("bregman"), lambda s, v: s._set("bregman", v))
    split_b = property(lambda s: s._get("split_b"), lambda s, v: s._set("split_b", v))
    split_s = property(lambda s: s._get("split_s"), lambda s, v: s._set("split_s", v))

    def reset(self) -> None:
        """Back to make_state(y0) without a host transfer."""
        _check(N.load().pfe_state_reset(self._h))

    def close(self) -> None:
        if self._h:
            N.load().pfe_state_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class PfeSolver:
    """PfeSolver (solver.hpp:51-83): operator, preconditioner and topology built once on the device."""

    def __init__(self, graph: WeightedGraph, params: PfeParams, device: int = 0, use_graphs: bool = True,
                 warn: bool = True, profile: bool = False, persistent: bool = True):
        lib = N.load()
        self.graph = graph
        self.params_ = params
        self._g = graph.to_c()
        self._p = params.to_c()
        self._x = _exec(device, use_graphs, warn, profile, persistent)
        h = C.c_void_p()
        _check(lib.pfe_solver_create(C.byref(self._g), C.byref(self._p), C.byref(self._x), C.byref(h)))
        self._h = h

    @property
    def params(self) -> PfeParams:
        return self.params_

    def diff_matrix(self) -> WeightedGraph:
        return self.graph

    def make_state(self, y0) -> SolverState:
        arr = _colmajor(y0, self.graph.n, self.params.dim)
        h = C.c_void_p()
        _check(N.load().pfe_state_create(self._h, N.dptr(arr), C.byref(h)))
        return SolverState(self, h)

    def split_bregman(self, state: SolverState, max_iter: int,
                      on_iterate: Optional[Callable[[int, np.ndarray], None]] = None) -> None:
        cb = N.ITERATE_FN()
        keep = None
        if on_iterate is not None:
            def _tramp(it, yp, n, d, _user):
                y = np.ctypeslib.as_array(yp, shape=(n * d,)).copy()
                on_iterate(int(it), _from_colmajor(y, n, d))
            keep = N.ITERATE_FN(_tramp)
            cb = keep
        _check(N.load().pfe_split_bregman(self._h, state._h, int(max_iter), cb, None))
        del keep

    def run_soc(self, state: SolverState, soc_max: int, sb_max: int) -> None:
        _check(N.load().pfe_run_soc(self._h, state._h, int(soc_max), int(sb_max)))

    def two_stage(self, y0) -> SolverState:
        st = self.make_state(y0)
        _check(N.load().pfe_two_stage(self._h, st._h))
        return st

    def objective(self, state: SolverState) -> float:
        out = C.c_double()
        _check(N.load().pfe_state_objective(self._h, state._h, C.byref(out)))
        return out.value

    def report(self) -> dict:
        r = N.pfe_report()
        _check(N.load().pfe_solver_report(self._h, C.byref(r)))
        return {k: getattr(r, k) for k, _ in N.pfe_report._fields_}

    def pcg_log(self):
        d = self.params.dim
        cap = 1 << 20
        n = self.report()["inner_iterations"]
        cap = max(1, n)
        it = np.zeros(cap * d, np.int32)
        st = np.zeros(cap * d, np.int32)
        rel = np.zeros(cap * d)
        cnt = N.load().pfe_solver_pcg_log(self._h, N.iptr(it), N.iptr(st), N.dptr(rel), cap)
        if cnt < 0:
            _check(int(-cnt))
        return it[:cnt * d].reshape(cnt, d), st[:cnt * d].reshape(cnt, d), rel[:cnt * d].reshape(cnt, d)

    def last_ms(self) -> float:
        """Device time (CUDA events on the solver stream) of the last solver call."""
        return float(N.load().pfe_solver_last_ms(self._h))

    def kernel_times(self, reset: bool = False) -> dict:
        t = N.pfe_kernel_times()
        _check(N.load().pfe_solver_kernel_times(self._h, C.byref(t), int(reset)))
        return {name: (t.ms[i], int(t.launches[i])) for i, name in enumerate(N.KERNEL_CLASSES)}

    def close(self) -> None:
        if getattr(self, "_h", None):
            N.load().pfe_solver_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def _solve(mode: int, g: WeightedGraph, params: PfeParams, y0, device=0, use_graphs=True, persistent=True):
    y0c = _colmajor(y0, g.n, params.dim)
    out = np.empty(g.n * params.dim)
    gc, pc, xc = g.to_c(), params.to_c(), _exec(device, use_graphs, persistent=persistent)
    rep = N.pfe_report()
    _check(N.load().pfe_solve(C.byref(gc), C.byref(pc), C.byref(xc), mode, N.dptr(y0c), N.dptr(out),
                              C.byref(rep)))
    return _from_colmajor(out, g.n, params.dim)


def soc(g: WeightedGraph, params: PfeParams, y0, **kw) -> np.ndarray:
    """soc(g, params, y0) (solver.cpp:184-189)."""
    return _solve(0, g, params, y0, **kw)


def pfe_two_stage(g: WeightedGraph, params: PfeParams, y0, **kw) -> np.ndarray:
    """pfe_two_stage(g, params, y0) (solver.cpp:191-193)."""
    return _solve(1, g, params, y0, **kw)


def split_bregman(g: WeightedGraph, d_vec, p, b, params: PfeParams, y_init, max_iter: int,
                  on_iterate: Optional[Callable[[int, np.ndarray], None]] = None, device: int = 0,
                  persistent=True) -> np.ndarray:
    """Standalone split_bregman with M = difference_matrix(g) (solver.cpp:138-182)."""
    y_init = np.asarray(y_init, dtype=np.float64)
    if y_init.ndim == 1:
        y_init = y_init.reshape(-1, 1)
    n, d = y_init.shape
    gg = WeightedGraph(g.n, g.ei, g.ej, g.w, np.asarray(d_vec, dtype=np.float64), grid=g.grid)
    gc = gg.to_c()
    pc = params.to_c()
    xc = _exec(device, True, False, persistent=persistent)
    pa, ba, ya = _colmajor(p, n, d), _colmajor(b, n, d), _colmajor(y_init, n, d)
    out = np.empty(n * d)
    cb = N.ITERATE_FN()
    keep = None
    if on_iterate is not None:
        def _tramp(it, yp, nn, dd, _user):
            on_iterate(int(it), _from_colmajor(np.ctypeslib.as_array(yp, shape=(nn * dd,)).copy(), nn, dd))
        keep = N.ITERATE_FN(_tramp)
        cb = keep
    _check(N.load().pfe_split_bregman_standalone(C.byref(gc), N.dptr(pa), N.dptr(ba), C.byref(pc), d, N.dptr(ya),
                                                 int(max_iter), C.byref(xc), N.dptr(out), cb, None))
    del keep
    return _from_colmajor(out, n, d)


def objective(g: WeightedGraph, y, device: int = 0) -> float:
    """objective(difference_matrix(g), Y) = sum_edges w |y_i - y_j|_1 (solver.cpp:14-17)."""
    y = np.asarray(y, dtype=np.float64)
    if y.ndim == 1:
        y = y.reshape(-1, 1)
    if y.shape[0] != g.n:
        raise ConfigError("objective: dimension mismatch")
    gc, xc = g.to_c(), _exec(device)
    ya = _colmajor(y)
    out = C.c_double()
    _check(N.load().pfe_objective(C.byref(gc), y.shape[1], N.dptr(ya), C.byref(xc), C.byref(out)))
    return out.value


def shrink(v, gamma: float, device: int = 0) -> np.ndarray:
    """shrink(V, gamma) = sign(v) max(|v| - gamma, 0) elementwise (solver.cpp:19-25)."""
    v = np.asarray(v, dtype=np.float64)
    flat = np.ascontiguousarray(v).reshape(-1)
    out = np.empty_like(flat)
    xc = _exec(device)
    _check(N.load().pfe_shrink(flat.size, N.dptr(flat), float(gamma), C.byref(xc), N.dptr(out)))
    return out.reshape(v.shape)


def project_orthogonal(a, device: int = 0) -> np.ndarray:
    """Frobenius-nearest matrix with orthonormal columns (solver.cpp:27-41)."""
    a = np.asarray(a, dtype=np.float64)
    if a.ndim == 1:
        a = a.reshape(-1, 1)
    n, d = a.shape
    if n < d:
        raise ConfigError("project_orthogonal: need rows >= cols")
    ac = _colmajor(a)
    out = np.empty(n * d)
    xc = _exec(device)
    _check(N.load().pfe_project_orthogonal(n, d, N.dptr(ac), C.byref(xc), N.dptr(out)))
    return _from_colmajor(out, n, d)


class PcgOperator:
    """PcgOperator(A, cfg) (pcg.hpp:31-54) over a CSR matrix (row_ptr, col_idx, values)."""

    def __init__(self, a, cfg: PcgConfig, device: int = 0):
        row_ptr, col_idx, values = a
        self.row_ptr = np.ascontiguousarray(row_ptr, dtype=np.int32)
        self.col_idx = np.ascontiguousarray(col_idx, dtype=np.int32)
        self.values = np.ascontiguousarray(values, dtype=np.float64)
        self.n = self.row_ptr.size - 1
        if cfg.rel_tol <= 0.0:
            raise ConfigError("PcgOperator: rel_tol must be > 0")
        if cfg.max_iter < 1:
            raise ConfigError("PcgOperator: max_iter must be >= 1")
        self.cfg = cfg
        self.device = device

    def solve_multi(self, b, x0) -> Tuple[np.ndarray, List[PcgReport]]:
        b = np.asarray(b, dtype=np.float64)
        x0 = np.asarray(x0, dtype=np.float64)
        if b.ndim == 1:
            b = b.reshape(-1, 1)
        if x0.ndim == 1:
            x0 = x0.reshape(-1, 1)
        if b.shape[0] != self.n or x0.shape[0] != self.n or b.shape[1] != x0.shape[1]:
            raise ConfigError("pcg_solve_multi: dimension mismatch")
        d = b.shape[1]
        bc, xc0 = _colmajor(b), _colmajor(x0)
        out = np.empty(self.n * d)
        its = np.zeros(d, np.int32)
        conv = np.zeros(d, np.int32)
        res = np.zeros(d)
        fb = np.zeros(d, np.int32)
        xc = _exec(self.device, True, False)
        _check(N.load().pfe_pcg_solve_multi(self.n, N.iptr(self.row_ptr), N.iptr(self.col_idx), N.dptr(self.values),
                                            d, N.dptr(bc), N.dptr(xc0), float(self.cfg.rel_tol),
                                            int(self.cfg.max_iter), int(self.cfg.preconditioner), C.byref(xc),
                                            N.dptr(out), N.iptr(its), N.iptr(conv), N.dptr(res), N.iptr(fb)))
        reps = [PcgReport(int(its[j]), float(res[j]), bool(conv[j]), bool(fb[j])) for j in range(d)]
        return _from_colmajor(out, self.n, d), reps

    def solve(self, b, x0) -> Tuple[np.ndarray, PcgReport]:
        x, reps = self.solve_multi(np.asarray(b).reshape(-1, 1), np.asarray(x0).reshape(-1, 1))
        return x[:, 0], reps[0]


def pcg_solve_multi(a, b, x0, cfg: PcgConfig, device: int = 0):
    """pcg_solve_multi (pcg.cpp:122-127)."""
    return PcgOperator(a, cfg, device).solve_multi(b, x0)


def pcg_solve(a, b, x0, cfg: PcgConfig, device: int = 0):
    """pcg_solve (pcg.cpp:116-120)."""
    return PcgOperator(a, cfg, device).solve(b, x0)


def random_embedding(n: int, d: int, seed: int, degree) -> np.ndarray:
    """random_embedding (init.cpp:172-181): mt19937_64 + libstdc++ normal, D-orthonormalized."""
    deg = np.ascontiguousarray(degree, dtype=np.float64)
    out = np.empty(n * d)
    _check(N.load().pfe_random_embedding(int(n), int(d), int(seed) & ((1 << 64) - 1), N.dptr(deg), N.dptr(out)))
    return _from_colmajor(out, n, d)


def d_orthonormalize(a, degree) -> np.ndarray:
    """d_orthonormalize (init.cpp:140-155)."""
    a = np.asarray(a, dtype=np.float64)
    n, d = a.shape
    deg = np.ascontiguousarray(degree, dtype=np.float64)
    ac = _colmajor(a)
    out = np.empty(n * d)
    _check(N.load().pfe_d_orthonormalize(n, d, N.dptr(ac), N.dptr(deg), N.dptr(out)))
    return _from_colmajor(out, n, d)


def kmeans(points, k: int, seed: int, max_iter: int = 100, device: Optional[int] = None) -> np.ndarray:
    """kmeans (cluster.cpp:54-124): k-means++ seeding + Lloyd; returns labels.

    ``device=None`` runs the host implementation (pfe_kmeans); a device
    ordinal runs the O(n k d) work on that GPU (pfe_kmeans_device) with the
    same random stream and rules."""
    pts = np.asarray(points, dtype=np.float64)
    if pts.ndim == 1:
        pts = pts.reshape(-1, 1)
    n, d = pts.shape
    pc = _colmajor(pts)
    lab = np.zeros(n, np.int32)
    if device is None:
        _check(N.load().pfe_kmeans(n, d, N.dptr(pc), int(k), int(seed), int(max_iter), N.iptr(lab)))
    else:
        _check(N.load().pfe_kmeans_device(n, d, N.dptr(pc), int(k), int(seed), int(max_iter), int(device),
                                          N.iptr(lab)))
    return lab


def gmm_init_embedding(features, k: int, seed: int, degree, device: int = 0, model: bool = False):
    """GMM initial embedding on the GPU (init.cpp:45-170: gmm_fit + init_embedding;
    pfe_gmm_init_device): k-means start, EM on the n x 3 features, then the
    responsibilities D-orthonormalised.  Returns Y0 (n x k), and with
    model=True also (means k x 3, variances k x 3, weights k)."""
    f = np.ascontiguousarray(features, dtype=np.float64).reshape(-1, 3)
    n = f.shape[0]
    deg = np.ascontiguousarray(degree, dtype=np.float64)
    if deg.shape != (n,):
        raise ConfigError("gmm_init_embedding: degree must have one entry per point")
    y = np.empty(n * int(k))
    means, var, wts = np.empty(3 * int(k)), np.empty(3 * int(k)), np.empty(int(k))
    _check(N.load().pfe_gmm_init_device(n, N.dptr(f), int(k), int(seed), N.dptr(deg), int(device), N.dptr(y),
                                        N.dptr(means), N.dptr(var), N.dptr(wts)))
    y0 = _from_colmajor(y, n, int(k))
    if model:
        return y0, means.reshape(-1, 3), var.reshape(-1, 3), wts
    return y0


def grid_graph_gpu(rgb, sigma_rgb: float, radius: int = 1, sigma_xy: Optional[float] = None,
                   device: int = 0) -> "WeightedGraph":
    """Heat-kernel pixel-grid graph built on the GPU (pfe_grid_graph); same
    definition as inputs.grid_graph (the host builder, graph.cpp:105-159
    semantics), with the grid hint set."""
    img = np.ascontiguousarray(rgb, dtype=np.float64)
    h, wd, _ = img.shape
    n = h * wd
    cap = n * (4 if radius == 1 else 12)
    ei, ej = np.empty(cap, np.int32), np.empty(cap, np.int32)
    w, deg = np.empty(cap), np.empty(n)
    m = C.c_int64()
    _check(N.load().pfe_grid_graph(h, wd, N.dptr(img), float(sigma_rgb), int(radius),
                                   float(sigma_xy) if sigma_xy is not None else 0.0, int(device), N.iptr(ei),
                                   N.iptr(ej), N.dptr(w), N.dptr(deg), C.byref(m)))
    mm = m.value
    return WeightedGraph(n, ei[:mm].copy(), ej[:mm].copy(), w[:mm].copy(), deg, float(sigma_rgb),
                         grid=(h, wd, int(radius)))


def knn_graph_gpu(points, k: int, device: int = 0) -> "WeightedGraph":
    """Union-symmetrised k-NN heat-kernel graph built on the GPU (pfe_knn_graph);
    same definition as inputs.knn_graph (the host builder)."""
    pts = np.ascontiguousarray(points, dtype=np.float64)
    if pts.ndim == 1:
        pts = pts.reshape(-1, 1)
    n, dim = pts.shape
    cap = n * int(k)
    ei, ej = np.empty(cap, np.int32), np.empty(cap, np.int32)
    w, deg = np.empty(cap), np.empty(n)
    m, sigma = C.c_int64(), C.c_double()
    _check(N.load().pfe_knn_graph(n, dim, N.dptr(pts), int(k), int(device), N.iptr(ei), N.iptr(ej), N.dptr(w),
                                  N.dptr(deg), C.byref(m), C.byref(sigma)))
    mm = m.value
    return WeightedGraph(n, ei[:mm].copy(), ej[:mm].copy(), w[:mm].copy(), deg, sigma.value)


# ------------------------------------------------------------ row bands ----
def band_plan(height: int, nranks: int, radius: int, rank: int) -> Tuple[int, int, int, int]:
    """Rows owned (r0, r1) and stored (lo, hi) by band `rank` (host only)."""
    out = np.zeros(4, np.int32)
    _check(N.load().pfe_band_plan(int(height), int(nranks), int(radius), int(rank), N.iptr(out)))
    return tuple(int(v) for v in out)


def soc_banded(g: WeightedGraph, params: PfeParams, y0, nbands: int, two_stage: bool = False,
               device: int = 0, return_report: bool = False):
    """The multi-GPU partitioned algorithm with `nbands` parts emulated on one
    device: row bands for pixel grids (grid hint), vertex ranges with ghost
    rows for general graphs."""
    y0c = _colmajor(y0, g.n, params.dim)
    out = np.empty(g.n * params.dim)
    gc, pc, xc = g.to_c(), params.to_c(), _exec(device, False, False, persistent=False)
    rep = N.pfe_report()
    _check(N.load().pfe_solve_banded(C.byref(gc), C.byref(pc), C.byref(xc), int(nbands), 1 if two_stage else 0,
                                     N.dptr(y0c), N.dptr(out), C.byref(rep)))
    y = _from_colmajor(out, g.n, params.dim)
    return (y, {k: getattr(rep, k) for k, _ in N.pfe_report._fields_}) if return_report else y


def soc_multi_gpu(g: WeightedGraph, params: PfeParams, y0, devices, two_stage: bool = False,
                  return_ms: bool = False, return_report: bool = False):
    """soc / pfe_two_stage of one graph over several GPUs from ONE call
    (pfe_solve_multi_gpu): row bands (pixel grids) or vertex ranges (general
    graphs), one band per listed device, NCCL communicators from
    ncclCommInitAll.  With return_ms, also the device time (max over GPUs)."""
    y0c = _colmajor(y0, g.n, params.dim)
    out = np.empty(g.n * params.dim)
    devs = np.ascontiguousarray(devices, np.int32)
    gc, pc, xc = g.to_c(), params.to_c(), _exec(int(devs[0]), False, False, persistent=False)
    rep = N.pfe_report()
    ms = np.zeros(1)
    _check(N.load().pfe_solve_multi_gpu(C.byref(gc), C.byref(pc), C.byref(xc), int(devs.size), N.iptr(devs),
                                        1 if two_stage else 0, N.dptr(y0c), N.dptr(out), C.byref(rep), N.dptr(ms)))
    y = _from_colmajor(out, g.n, params.dim)
    if return_report:
        return y, {k: getattr(rep, k) for k, _ in N.pfe_report._fields_}
    return (y, float(ms[0])) if return_ms else y


def range_partition_stats(g: WeightedGraph, nranks: int) -> dict:
    """Owned / ghost / sent rows per rank of the vertex-range partition a
    BandSolver uses for a general graph (host only, no device)."""
    own, gh, snd = (np.zeros(nranks, np.int64) for _ in range(3))
    gc = g.to_c()
    p64 = C.POINTER(C.c_int64)
    _check(N.load().pfe_range_partition_stats(C.byref(gc), int(nranks), own.ctypes.data_as(p64),
                                              gh.ctypes.data_as(p64), snd.ctypes.data_as(p64)))
    return {"owned": own, "ghosts": gh, "sends": snd}


def nccl_unique_id() -> bytes:
    buf = (C.c_uint8 * 128)()
    _check(N.load().pfe_nccl_unique_id(buf))
    return bytes(buf)


class BandSolver(PfeSolver):
    """One row band (pixel grids) or vertex range (general graphs) of a
    multi-GPU solve (one process per GPU, NCCL between ranks).

    Every rank passes the same global graph and the same NCCL id; make_state
    takes the global y0 and ``state.y`` returns the global Y on every rank.
    """

    def __init__(self, graph: WeightedGraph, params: PfeParams, nccl_id: bytes, nranks: int, rank: int,
                 device: int = 0, warn: bool = True):
        lib = N.load()
        self.graph = graph
        self.params_ = params
        self._g = graph.to_c()
        self._p = params.to_c()
        self._x = _exec(device, False, warn, False, False)
        idbuf = (C.c_uint8 * 128).from_buffer_copy(nccl_id)
        h = C.c_void_p()
        _check(lib.pfe_solver_create_band(C.byref(self._g), C.byref(self._p), C.byref(self._x), idbuf, int(nranks),
                                          int(rank), C.byref(h)))
        self._h = h
