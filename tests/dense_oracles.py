"""Dense brute-force oracles (numpy restatement of proj/tests/oracles.hpp:21-175).

TEST INFRASTRUCTURE: independent of both the CPU oracle and the GPU library.
"""
import numpy as np


def diff_matrix_dense(g):
    """difference_matrix (graph.cpp:161-170) as a dense |E| x n matrix."""
    m = np.zeros((g.m, g.n))
    for k, (i, j, w) in enumerate(zip(g.ei, g.ej, g.w)):
        m[k, i] += w
        m[k, j] -= w
    return m


def kron_identity(d, m):
    """oracles.hpp:71-77"""
    return np.kron(np.eye(d), m)


def vec(m):
    return np.asarray(m).reshape(-1, order="F")


def unvec(v, rows, cols):
    return np.asarray(v).reshape(cols, rows).T


def shrink_vec(v, gamma):
    mag = np.abs(v) - gamma
    return np.where(mag > 0.0, np.where(v > 0.0, mag, -mag), 0.0)


def polar_factor(a):
    """oracles.hpp:98-102: A (A^T A)^{-1/2}."""
    lam, v = np.linalg.eigh(a.T @ a)
    return a @ v @ np.diag(1.0 / np.sqrt(lam)) @ v.T


class KroneckerSolver:
    """oracles.hpp:106-175: the literal dn x dn system, solved densely."""

    def __init__(self, m_dense, degree, d, lam, r):
        self.m = m_dense
        self.degree = np.asarray(degree)
        self.n = m_dense.shape[1]
        self.d = d
        self.lam = lam
        self.r = r
        self.l = kron_identity(d, m_dense)
        self.dt = kron_identity(d, np.diag(self.degree))
        self.dt_sqrt = kron_identity(d, np.diag(np.sqrt(self.degree)))
        self.system = 0.5 * lam * self.l.T @ self.l + 0.5 * r * self.dt

    def split_bregman(self, p, big_b, y0, iterations, trajectory=None, conv_tol=0.0):
        yv, pv, bv = vec(y0), vec(p), vec(big_b)
        inner_b = np.zeros(self.l.shape[0])
        inner_d = np.zeros(self.l.shape[0])
        for _ in range(iterations):
            rhs = 0.5 * self.lam * self.l.T @ (inner_d - inner_b) + 0.5 * self.r * self.dt_sqrt @ (pv - bv)
            y_old = yv
            yv = np.linalg.solve(self.system, rhs)
            ly = self.l @ yv
            inner_d = shrink_vec(ly + inner_b, 1.0 / self.lam)
            inner_b = inner_b + ly - inner_d
            if trajectory is not None:
                trajectory.append(unvec(yv, self.n, self.d))
            den = np.linalg.norm(y_old)
            if conv_tol > 0 and den > 0 and np.linalg.norm(yv - y_old) / den <= conv_tol:
                break
        return unvec(yv, self.n, self.d)

    def soc(self, y0, soc_iters, sb_iters, conv_tol=0.0):
        y = np.array(y0, dtype=float)
        dsq = np.diag(np.sqrt(self.degree))
        p = dsq @ y
        big_b = np.zeros((self.n, self.d))
        for _ in range(soc_iters):
            y_old = y
            y = self.split_bregman(p, big_b, y, sb_iters, None, conv_tol)
            p = polar_factor(dsq @ y + big_b)
            big_b = big_b + dsq @ y - p
            den = np.linalg.norm(y_old)
            if conv_tol > 0 and den > 0 and np.linalg.norm(y - y_old) / den <= conv_tol:
                break
        return y
