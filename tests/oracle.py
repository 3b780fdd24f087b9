"""ctypes binding of the CPU oracle (oracle/libpfe_oracle.so) — TEST INFRASTRUCTURE.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
reference leg use this module, and only as the checker.
"""
from __future__ import annotations

import ctypes as C
import subprocess
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
ORACLE_DIR = ROOT / "oracle"
LIB = ORACLE_DIR / "build" / "libpfe_oracle.so"

_D = C.POINTER(C.c_double)
_I = C.POINTER(C.c_int32)


class orc_params(C.Structure):
    _fields_ = [("dim", C.c_int), ("lambda_", C.c_double), ("r", C.c_double), ("soc_max", C.c_int),
                ("sb_max_stage1", C.c_int), ("sb_max_stage2", C.c_int), ("conv_tol", C.c_double),
                ("pcg_rel_tol", C.c_double), ("pcg_max_iter", C.c_int), ("preconditioner", C.c_int)]


_lib = None


def build() -> Path:
    if not LIB.exists() or any(p.stat().st_mtime > LIB.stat().st_mtime for p in ORACLE_DIR.glob("*.[ch]pp")):
        subprocess.run(["make", "-C", str(ORACLE_DIR), "-j4", "build/libpfe_oracle.so"], check=True,
                       capture_output=True)
    return LIB


def lib() -> C.CDLL:
    global _lib
    if _lib is None:
        build()
        _lib = C.CDLL(str(LIB))
        _lib.orc_last_error.restype = C.c_char_p
    return _lib


class OracleError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"[{code}] {msg}")
        self.code = code


def _ck(rc):
    if rc != 0:
        raise OracleError(rc, lib().orc_last_error().decode())


def dp(a):
    return a.ctypes.data_as(_D)


def ip(a):
    return a.ctypes.data_as(_I)


def _cm(a, rows=None, cols=None):
    a = np.asarray(a, dtype=np.float64)
    if a.ndim == 1:
        a = a.reshape(-1, 1)
    return np.asfortranarray(a)


def _un(buf, rows, cols):
    return np.array(buf.reshape(cols, rows).T, order="F")


def params(p) -> orc_params:
    """From an api.PfeParams."""
    return orc_params(p.dim, p.lambda_, p.r, p.soc_max, p.sb_max_stage1, p.sb_max_stage2, p.conv_tol,
                      p.pcg.rel_tol, p.pcg.max_iter, int(p.pcg.preconditioner))


def set_threads(t: int):
    lib().orc_set_threads(int(t))


def _g(g):
    return (g.n, g.m, ip(g.ei), ip(g.ej), dp(g.w))


def solve(g, p, y0, mode=0, full_state=False, log_cap=0):
    """mode 0: soc, mode 1: two_stage.  Returns y (and state / PCG log)."""
    n, d, m = g.n, p.dim, g.m
    y0c = _cm(y0)
    outs = [np.empty(n * d) for _ in range(3)] + [np.empty(m * d) for _ in range(2)]
    log = np.zeros(max(1, log_cap), np.int32)
    ninner = C.c_long()
    pp = params(p)
    ptrs = [dp(o) if (full_state or i == 0) else None for i, o in enumerate(outs)]
    _ck(lib().orc_solve(mode, *_g(g), dp(g.degree), C.byref(pp), dp(y0c), *ptrs,
                        ip(log) if log_cap else None, log_cap, C.byref(ninner)))
    y = _un(outs[0], n, d)
    if not full_state and not log_cap:
        return y
    res = {"y": y, "inner": ninner.value}
    if full_state:
        res.update(p=_un(outs[1], n, d), bregman=_un(outs[2], n, d), split_b=_un(outs[3], m, d),
                   split_s=_un(outs[4], m, d))
    if log_cap:
        res["pcg_log"] = log[:min(log_cap, ninner.value)].copy()
    return res


def solve_timed(g, p, y0, log_cap=100000):
    """soc (mode 0) with the PCG log and wall seconds {setup, inner, outer}."""
    n, d = g.n, p.dim
    y0c = _cm(y0)
    y = np.empty(n * d)
    log = np.zeros(max(1, log_cap), np.int32)
    ninner = C.c_long()
    times = np.zeros(3)
    pp = params(p)
    _ck(lib().orc_solve_timed(0, *_g(g), dp(g.degree), C.byref(pp), dp(y0c), dp(y), None, None, None, None,
                              ip(log), log_cap, C.byref(ninner), dp(times)))
    return {"y": _un(y, n, d), "inner": ninner.value, "pcg_log": log[:min(log_cap, ninner.value)].copy(),
            "t_setup": float(times[0]), "t_inner": float(times[1]), "t_outer": float(times[2])}


class Session:
    """A resident oracle solve (orc_session_*): built once, then stepped a few
    inner iterations at a time along the soc schedule (bench.py CPU legs)."""

    def __init__(self, g, p, y0):
        self._h = C.c_void_p()
        setup = C.c_double()
        pp = params(p)
        _ck(lib().orc_session_create(*_g(g), dp(g.degree), C.byref(pp), dp(_cm(y0)), C.byref(self._h),
                                     C.byref(setup)))
        self.setup_s = setup.value

    def step(self, inner=1):
        """-> (inner-iteration seconds, projection seconds, PCG iterations per inner iteration)."""
        t = np.zeros(2)
        k = np.zeros(max(1, inner), np.int32)
        _ck(lib().orc_session_step(self._h, int(inner), dp(t), ip(k)))
        return float(t[0]), float(t[1]), k[:inner].copy()

    def close(self):
        if self._h:
            lib().orc_session_destroy(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def state_split_bregman(g, p, max_iter, y, pp_, breg, sb, ss, want_traj=False):
    n, d, m = g.n, p.dim, g.m
    arrs = [_cm(y).copy(order="F"), _cm(pp_).copy(order="F"), _cm(breg).copy(order="F"), _cm(sb).copy(order="F"),
            _cm(ss).copy(order="F")]
    traj = np.empty(max(1, max_iter) * n * d) if want_traj else None
    nt = C.c_int()
    prm = params(p)
    _ck(lib().orc_state_split_bregman(*_g(g), dp(g.degree), C.byref(prm), int(max_iter),
                                      *[dp(a) for a in arrs], dp(traj) if want_traj else None, C.byref(nt)))
    out = {"y": arrs[0], "p": arrs[1], "bregman": arrs[2], "split_b": arrs[3], "split_s": arrs[4]}
    if want_traj:
        out["traj"] = [_un(traj[k * n * d:(k + 1) * n * d], n, d) for k in range(nt.value)]
    return out


def split_bregman(g, d_vec, p_, b_, prm, y_init, max_iter, want_traj=False):
    y_init = _cm(y_init)
    n, d = y_init.shape
    out = np.empty(n * d)
    traj = np.empty(max(1, max_iter) * n * d) if want_traj else None
    nt = C.c_int()
    cp = params(prm)
    dv = np.ascontiguousarray(d_vec, dtype=np.float64)
    _ck(lib().orc_split_bregman(*_g(g), dp(dv), dp(_cm(p_)), dp(_cm(b_)), C.byref(cp), d, dp(y_init),
                                int(max_iter), dp(out), dp(traj) if want_traj else None, C.byref(nt)))
    y = _un(out, n, d)
    if want_traj:
        return y, [_un(traj[k * n * d:(k + 1) * n * d], n, d) for k in range(nt.value)]
    return y


def normal_matrix(g, lam, r, degree=None):
    deg = np.ascontiguousarray(g.degree if degree is None else degree, dtype=np.float64)
    nnz = C.c_int()
    _ck(lib().orc_normal_matrix(*_g(g), dp(deg), C.c_double(lam), C.c_double(r), C.byref(nnz), None, None, None))
    ptr = np.zeros(g.n + 1, np.int32)
    idx = np.zeros(nnz.value, np.int32)
    val = np.zeros(nnz.value)
    _ck(lib().orc_normal_matrix(*_g(g), dp(deg), C.c_double(lam), C.c_double(r), C.byref(nnz), ip(ptr), ip(idx),
                                dp(val)))
    return ptr, idx, val


def pcg_solve_multi(a, b, x0, rel_tol, max_iter, prec):
    ptr, idx, val = (np.ascontiguousarray(a[0], np.int32), np.ascontiguousarray(a[1], np.int32),
                     np.ascontiguousarray(a[2], np.float64))
    b, x0 = _cm(b), _cm(x0)
    n, d = b.shape
    x = np.empty(n * d)
    its = np.zeros(d, np.int32)
    conv = np.zeros(d, np.int32)
    res = np.zeros(d)
    _ck(lib().orc_pcg_solve_multi(n, ip(ptr), ip(idx), dp(val), d, dp(b), dp(x0), C.c_double(rel_tol),
                                  int(max_iter), int(prec), dp(x), ip(its), ip(conv), dp(res)))
    return _un(x, n, d), its, conv, res


def project_orthogonal(a):
    a = _cm(a)
    n, d = a.shape
    out = np.empty(n * d)
    _ck(lib().orc_project_orthogonal(n, d, dp(a), dp(out)))
    return _un(out, n, d)


def shrink(v, gamma):
    v = np.ascontiguousarray(v, dtype=np.float64).reshape(-1)
    out = np.empty_like(v)
    _ck(lib().orc_shrink(C.c_long(v.size), dp(v), C.c_double(gamma), dp(out)))
    return out


def objective(g, y):
    y = _cm(y)
    out = C.c_double()
    _ck(lib().orc_objective(*_g(g), y.shape[1], dp(y), C.byref(out)))
    return out.value


def random_embedding(n, d, seed, degree):
    out = np.empty(n * d)
    deg = np.ascontiguousarray(degree, dtype=np.float64)
    _ck(lib().orc_random_embedding(n, d, C.c_ulonglong(seed), dp(deg), dp(out)))
    return _un(out, n, d)


def kmeans(pts, k, seed, max_iter=100):
    pts = _cm(pts)
    n, d = pts.shape
    lab = np.zeros(n, np.int32)
    _ck(lib().orc_kmeans(n, d, dp(pts), k, C.c_ulonglong(seed), max_iter, ip(lab)))
    return lab


def covering(pred, gt):
    pred = np.ascontiguousarray(pred, np.int32)
    gt = np.ascontiguousarray(gt, np.int32)
    out = C.c_double()
    _ck(lib().orc_covering(pred.size, ip(pred), ip(gt), C.byref(out)))
    return out.value


def build_image_graph(rgb, sigma=0.0):
    """4-neighbour reference image graph; rgb (H, W, 3)."""
    h, w, _ = rgb.shape
    f = np.ascontiguousarray(rgb, dtype=np.float64)
    m = C.c_int()
    so = C.c_double()
    _ck(lib().orc_build_image_graph(h, w, dp(f), C.c_double(sigma), C.byref(m), None, None, None, None,
                                    C.byref(so)))
    ei = np.zeros(m.value, np.int32)
    ej = np.zeros(m.value, np.int32)
    wt = np.zeros(m.value)
    deg = np.zeros(h * w)
    _ck(lib().orc_build_image_graph(h, w, dp(f), C.c_double(sigma), C.byref(m), ip(ei), ip(ej), dp(wt), dp(deg),
                                    C.byref(so)))
    return ei, ej, wt, deg, so.value


def gmm_init_embedding(rgb_flat, k, seed, degree):
    f = np.ascontiguousarray(rgb_flat, dtype=np.float64)
    n = f.shape[0]
    out = np.empty(n * k)
    deg = np.ascontiguousarray(degree, dtype=np.float64)
    _ck(lib().orc_gmm_init_embedding(n, dp(f), k, C.c_ulonglong(seed), dp(deg), dp(out)))
    return _un(out, n, k)


def quadrant_rgb(size, noise=0.02, seed=7):
    out = np.empty(size * size * 3)
    _ck(lib().orc_quadrant_rgb(size, C.c_double(noise), C.c_ulonglong(seed), dp(out)))
    return out.reshape(size, size, 3)


def golden_quadrant(size=64):
    out = np.zeros(5)
    _ck(lib().orc_golden_quadrant(size, dp(out)))
    return {"obj0": out[0], "obj1": out[1], "covering": out[2], "seconds": out[3], "inner": int(out[4])}
