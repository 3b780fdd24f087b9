// TEST INFRASTRUCTURE ONLY — see pfe_oracle.hpp for the contract.
// Restates /root/reference/proj/core/src/{sparse,pcg,solver,graph,init,cluster,metrics}.cpp.
#include "pfe_oracle.hpp"

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <limits>
#include <map>
#include <chrono>
#include <random>
#include <thread>
#include <unordered_map>

namespace orc {

namespace {
int g_threads = 1;

// Runs body(j) for j in [0, count) on up to g_threads threads (static split).
template <class F>
void for_columns(long count, F&& body) {
  int t = std::min<long>(g_threads, count);
  if (t <= 1) {
    for (long j = 0; j < count; ++j) body(j);
    return;
  }
  std::vector<std::thread> pool;
  for (int w = 0; w < t; ++w) {
    pool.emplace_back([&, w] {
      for (long j = w; j < count; j += t) body(j);
    });
  }
  for (auto& th : pool) th.join();
}

// Runs body(lo, hi) over [0, count) split into g_threads contiguous ranges.
// Used only for per-element work whose results do not depend on the split
// (k-means distances); every sum stays sequential.
template <class F>
void for_ranges(long count, F&& body) {
  int t = static_cast<int>(std::min<long>(g_threads, count / 4096 + 1));
  if (t <= 1) {
    body(0L, count);
    return;
  }
  std::vector<std::thread> pool;
  const long chunk = (count + t - 1) / t;
  for (int w = 0; w < t; ++w) {
    const long lo = w * chunk, hi = std::min(count, lo + chunk);
    if (lo < hi) pool.emplace_back([&, lo, hi] { body(lo, hi); });
  }
  for (auto& th : pool) th.join();
}

double seq_dot(const double* a, const double* b, long n) {
  double s = 0.0;
  for (long i = 0; i < n; ++i) s += a[i] * b[i];
  return s;
}
double seq_norm(const double* a, long n) { return std::sqrt(seq_dot(a, a, n)); }
double mat_norm(const Mat& m) { return seq_norm(m.a.data(), static_cast<long>(m.a.size())); }
bool all_finite(const double* a, long n) {
  for (long i = 0; i < n; ++i)
    if (!std::isfinite(a[i])) return false;
  return true;
}
}  // namespace

void set_threads(int t) { g_threads = std::max(1, t); }
int get_threads() { return g_threads; }

// ------------------------------------------------------------------ sparse --

// sparse.cpp:11-50 — stable sort by (row, col), sum runs of equal keys in
// input order, drop exact-zero sums.
Csr csr_from_triplets(int nrows, int ncols, const std::vector<Trip>& t) {
  if (nrows < 0 || ncols < 0) throw ConfigError("csr_from_triplets: negative dimensions");
  for (const Trip& e : t) {
    if (e.row < 0 || e.row >= nrows || e.col < 0 || e.col >= ncols)
      throw ConfigError("csr_from_triplets: entry outside matrix");
    if (!std::isfinite(e.val)) throw ConfigError("csr_from_triplets: non-finite value");
  }
  std::vector<Trip> s(t);
  std::stable_sort(s.begin(), s.end(), [](const Trip& x, const Trip& y) {
    return x.row != y.row ? x.row < y.row : x.col < y.col;
  });
  Csr c;
  c.nrows = nrows;
  c.ncols = ncols;
  c.ptr.assign(static_cast<size_t>(nrows) + 1, 0);
  size_t k = 0;
  for (int row = 0; row < nrows; ++row) {
    while (k < s.size() && s[k].row == row) {
      const int col = s[k].col;
      double acc = 0.0;
      for (; k < s.size() && s[k].row == row && s[k].col == col; ++k) acc += s[k].val;
      if (acc != 0.0) {
        c.idx.push_back(col);
        c.val.push_back(acc);
      }
    }
    c.ptr[static_cast<size_t>(row) + 1] = static_cast<int>(c.val.size());
  }
  return c;
}

// sparse.cpp:52-72 — counting-sort transpose; row v of the result lists the
// source rows in increasing order.
Csr transpose(const Csr& a) {
  Csr t;
  t.nrows = a.ncols;
  t.ncols = a.nrows;
  t.ptr.assign(static_cast<size_t>(a.ncols) + 1, 0);
  t.idx.resize(a.val.size());
  t.val.resize(a.val.size());
  for (int c : a.idx) ++t.ptr[static_cast<size_t>(c) + 1];
  for (int c = 0; c < a.ncols; ++c) t.ptr[c + 1] += t.ptr[c];
  std::vector<int> fill(t.ptr.begin(), t.ptr.end() - 1);
  for (int r = 0; r < a.nrows; ++r)
    for (int k = a.ptr[r]; k < a.ptr[r + 1]; ++k) {
      const int at = fill[a.idx[k]]++;
      t.idx[at] = r;
      t.val[at] = a.val[k];
    }
  return t;
}

// sparse.cpp:74-85 — each row accumulated left to right from 0.0.
void spmv_raw(const Csr& a, const double* x, double* y) {
  for (int r = 0; r < a.nrows; ++r) {
    double acc = 0.0;
    for (int k = a.ptr[r]; k < a.ptr[r + 1]; ++k) acc += a.val[k] * x[a.idx[k]];
    y[r] = acc;
  }
}
Vec spmv(const Csr& a, const Vec& x) {
  if (static_cast<int>(x.size()) != a.ncols) throw ConfigError("spmv: dimension mismatch");
  Vec y(static_cast<size_t>(a.nrows));
  spmv_raw(a, x.data(), y.data());
  return y;
}

// sparse.cpp:87-94 — column j is exactly spmv(a, x.col(j)).
Mat spmm_dense(const Csr& a, const Mat& x) {
  if (x.rows != a.ncols) throw ConfigError("spmm_dense: dimension mismatch");
  Mat y(a.nrows, x.cols);
  for_columns(x.cols, [&](long j) { spmv_raw(a, x.col(j), y.col(j)); });
  return y;
}

// sparse.cpp:96-122 — (lambda/2) M^T M + (r/2) diag(deg) via triplets: per M
// row all (p, q) products (hl * m_p) * m_q, then the n diagonal terms last.
Csr form_normal_matrix(const Csr& m, const Vec& deg, double lambda, double r) {
  if (static_cast<int>(deg.size()) != m.ncols)
    throw ConfigError("form_normal_matrix: degree size mismatch");
  if (lambda < 0.0) throw ConfigError("form_normal_matrix: lambda must be >= 0");
  if (r <= 0.0) throw ConfigError("form_normal_matrix: r must be > 0");
  for (size_t i = 0; i < deg.size(); ++i)
    if (deg[i] <= 0.0)
      throw ConfigError("form_normal_matrix: nonpositive degree at vertex " + std::to_string(i) +
                        " (isolated vertex)");
  std::vector<Trip> t;
  t.reserve(static_cast<size_t>(m.nnz()) * 2 + deg.size());
  const double hl = 0.5 * lambda;
  for (int row = 0; row < m.nrows; ++row)
    for (int p = m.ptr[row]; p < m.ptr[row + 1]; ++p)
      for (int q = m.ptr[row]; q < m.ptr[row + 1]; ++q)
        t.push_back({m.idx[p], m.idx[q], hl * m.val[p] * m.val[q]});
  for (int i = 0; i < m.ncols; ++i) t.push_back({i, i, 0.5 * r * deg[static_cast<size_t>(i)]});
  return csr_from_triplets(m.ncols, m.ncols, t);
}

namespace {
// sparse.cpp:128-143
Csr lower_part(const Csr& a, double shift) {
  Csr l;
  l.nrows = a.nrows;
  l.ncols = a.ncols;
  l.ptr.assign(static_cast<size_t>(a.nrows) + 1, 0);
  for (int r = 0; r < a.nrows; ++r) {
    for (int k = a.ptr[r]; k < a.ptr[r + 1]; ++k) {
      const int c = a.idx[k];
      if (c > r) continue;
      l.idx.push_back(c);
      l.val.push_back(c == r ? a.val[k] + shift : a.val[k]);
    }
    l.ptr[r + 1] = static_cast<int>(l.val.size());
  }
  return l;
}

// sparse.cpp:146-180 — row-oriented IC(0) sweep.
bool ic0_sweep(Csr& l) {
  for (int i = 0; i < l.nrows; ++i) {
    const int b = l.ptr[i], e = l.ptr[i + 1];
    if (b == e || l.idx[e - 1] != i) return false;
    for (int k = b; k < e; ++k) {
      const int j = l.idx[k];
      double acc = 0.0;
      int pi = b, pj = l.ptr[j];
      const int ej = l.ptr[j + 1];
      while (pi < k && pj < ej && l.idx[pj] < j) {
        if (l.idx[pi] == l.idx[pj]) {
          acc += l.val[pi] * l.val[pj];
          ++pi;
          ++pj;
        } else if (l.idx[pi] < l.idx[pj]) {
          ++pi;
        } else {
          ++pj;
        }
      }
      if (j == i) {
        const double piv = l.val[k] - acc;
        if (!(piv > 0.0)) return false;
        l.val[k] = std::sqrt(piv);
      } else {
        l.val[k] = (l.val[k] - acc) / l.val[l.ptr[j + 1] - 1];
      }
    }
  }
  return true;
}
}  // namespace

// sparse.cpp:184-203
IcFactor incomplete_cholesky(const Csr& a) {
  if (a.nrows != a.ncols) throw ConfigError("incomplete_cholesky: matrix not square");
  double dmax = 0.0;
  for (int r = 0; r < a.nrows; ++r)
    for (int k = a.ptr[r]; k < a.ptr[r + 1]; ++k)
      if (a.idx[k] == r) dmax = std::max(dmax, a.val[k]);
  double shift = 0.0;
  for (int attempt = 0; attempt <= 8; ++attempt) {
    Csr l = lower_part(a, shift);
    if (ic0_sweep(l)) return IcFactor{std::move(l), shift};
    shift = (shift == 0.0) ? 1e-3 * std::max(dmax, 1.0) : 2.0 * shift;
  }
  throw NumericalError("incomplete_cholesky: breakdown persists after 8 diagonal shifts");
}

// sparse.cpp:205-238 — forward: L x = b; backward: L^T x = b by column sweeps.
void triangular_solve(const IcFactor& f, double* x, bool forward) {
  const Csr& l = f.lower;
  if (forward) {
    for (int i = 0; i < l.nrows; ++i) {
      double acc = x[i], dg = 0.0;
      for (int k = l.ptr[i]; k < l.ptr[i + 1]; ++k) {
        if (l.idx[k] == i)
          dg = l.val[k];
        else
          acc -= l.val[k] * x[l.idx[k]];
      }
      if (dg == 0.0) throw NumericalError("triangular_solve: zero diagonal");
      x[i] = acc / dg;
    }
  } else {
    for (int i = l.nrows - 1; i >= 0; --i) {
      const int e = l.ptr[i + 1];
      const double dg = (e > l.ptr[i] && l.idx[e - 1] == i) ? l.val[e - 1] : 0.0;
      if (dg == 0.0) throw NumericalError("triangular_solve: zero diagonal");
      x[i] /= dg;
      for (int k = l.ptr[i]; k < e - 1; ++k) x[l.idx[k]] -= l.val[k] * x[i];
    }
  }
}

// --------------------------------------------------------------------- pcg --

// pcg.cpp:9-29
PcgOperator::PcgOperator(Csr a, PcgConfig cfg) : a_(std::move(a)), cfg_(cfg) {
  if (a_.nrows != a_.ncols) throw ConfigError("PcgOperator: matrix not square");
  if (cfg_.rel_tol <= 0.0) throw ConfigError("PcgOperator: rel_tol must be > 0");
  if (cfg_.max_iter < 1) throw ConfigError("PcgOperator: max_iter must be >= 1");
  if (cfg_.prec != kNone) {
    inv_diag_.assign(static_cast<size_t>(a_.nrows), 1.0);
    for (int r = 0; r < a_.nrows; ++r)
      for (int k = a_.ptr[r]; k < a_.ptr[r + 1]; ++k)
        if (a_.idx[k] == r && a_.val[k] > 0.0) inv_diag_[static_cast<size_t>(r)] = 1.0 / a_.val[k];
  }
  if (cfg_.prec == kIc0) {
    try {
      ic_ = incomplete_cholesky(a_);
      have_ic_ = true;
    } catch (const NumericalError&) {
      fallback_ = true;
    }
  }
}

// pcg.cpp:31-38
void PcgOperator::precondition(const double* r, double* z) const {
  const long n = a_.nrows;
  if (have_ic_) {
    std::copy(r, r + n, z);
    triangular_solve(ic_, z, true);
    triangular_solve(ic_, z, false);
    return;
  }
  if (cfg_.prec != kNone) {
    for (long i = 0; i < n; ++i) z[i] = inv_diag_[static_cast<size_t>(i)] * r[i];
    return;
  }
  std::copy(r, r + n, z);
}

// pcg.cpp:40-92
PcgReport PcgOperator::solve(const double* b, const double* x0, double* xout) const {
  const long n = a_.nrows;
  PcgReport rep;
  rep.jacobi_fallback = fallback_;
  const double bnorm = seq_norm(b, n);
  if (bnorm == 0.0) {
    rep.converged = true;
    std::fill(xout, xout + n, 0.0);
    return rep;
  }
  Vec x(x0, x0 + n), r(static_cast<size_t>(n)), z(static_cast<size_t>(n)), p, q(static_cast<size_t>(n));
  spmv_raw(a_, x.data(), q.data());
  for (long i = 0; i < n; ++i) r[i] = b[i] - q[i];
  double rel = seq_norm(r.data(), n) / bnorm;
  if (rel <= cfg_.rel_tol) {
    rep.converged = true;
    rep.final_rel_residual = rel;
    std::copy(x.begin(), x.end(), xout);
    return rep;
  }
  precondition(r.data(), z.data());
  p = z;
  double rz = seq_dot(r.data(), z.data(), n);
  for (int it = 1; it <= cfg_.max_iter; ++it) {
    spmv_raw(a_, p.data(), q.data());
    const double pq = seq_dot(p.data(), q.data(), n);
    if (!(pq > 0.0) || !std::isfinite(pq))
      throw NumericalError("pcg_solve: indefinite or NaN curvature encountered");
    const double alpha = rz / pq;
    for (long i = 0; i < n; ++i) x[i] += alpha * p[i];
    for (long i = 0; i < n; ++i) r[i] -= alpha * q[i];
    if (!all_finite(x.data(), n)) throw NumericalError("pcg_solve: NaN in iterates");
    rel = seq_norm(r.data(), n) / bnorm;
    rep.iterations = it;
    if (rel <= cfg_.rel_tol) {
      rep.converged = true;
      break;
    }
    precondition(r.data(), z.data());
    const double rz_next = seq_dot(r.data(), z.data(), n);
    const double beta = rz_next / rz;
    for (long i = 0; i < n; ++i) p[i] = z[i] + beta * p[i];
    rz = rz_next;
  }
  rep.final_rel_residual = rel;
  std::copy(x.begin(), x.end(), xout);
  return rep;
}

// pcg.cpp:94-114 — columns independent; a NumericalError in one column
// leaves that column at x0 with residual = inf.
std::vector<PcgReport> PcgOperator::solve_multi(const Mat& b, const Mat& x0, Mat& x) const {
  if (b.rows != a_.nrows || x0.rows != a_.nrows || b.cols != x0.cols)
    throw ConfigError("pcg_solve_multi: dimension mismatch");
  x = Mat(b.rows, b.cols);
  std::vector<PcgReport> reps(static_cast<size_t>(b.cols));
  for_columns(b.cols, [&](long j) {
    try {
      reps[static_cast<size_t>(j)] = solve(b.col(j), x0.col(j), x.col(j));
    } catch (const NumericalError&) {
      std::copy(x0.col(j), x0.col(j) + b.rows, x.col(j));
      reps[static_cast<size_t>(j)] = PcgReport{};
      reps[static_cast<size_t>(j)].converged = false;
      reps[static_cast<size_t>(j)].final_rel_residual = std::numeric_limits<double>::infinity();
    }
  });
  return reps;
}

// ------------------------------------------------------------------- graph --

// graph.cpp:161-170 — row k = [+w at i, -w at j].
Csr difference_matrix(const Graph& g) {
  std::vector<Trip> t;
  t.reserve(static_cast<size_t>(g.m()) * 2);
  for (int k = 0; k < g.m(); ++k) {
    t.push_back({k, g.ei[k], g.w[k]});
    t.push_back({k, g.ej[k], -g.w[k]});
  }
  return csr_from_triplets(g.m(), g.n, t);
}

// graph.cpp:15-22 / 172-174
Vec degree_vector(const Graph& g) {
  Vec d(static_cast<size_t>(g.n), 0.0);
  for (int k = 0; k < g.m(); ++k) {
    d[g.ei[k]] += g.w[k];
    d[g.ej[k]] += g.w[k];
  }
  return d;
}

namespace {
double rgb_dist2(const std::vector<double>& f, long a, long b) {
  const double d0 = f[3 * a] - f[3 * b], d1 = f[3 * a + 1] - f[3 * b + 1], d2 = f[3 * a + 2] - f[3 * b + 2];
  return d0 * d0 + d1 * d1 + d2 * d2;
}
}  // namespace

// graph.cpp:87-103
double median_neighbor_distance(int h, int w, const std::vector<double>& f) {
  std::vector<double> ds;
  for (int r = 0; r < h; ++r)
    for (int c = 0; c < w; ++c) {
      const long v = static_cast<long>(r) * w + c;
      if (c + 1 < w) ds.push_back(std::sqrt(rgb_dist2(f, v, v + 1)));
      if (r + 1 < h) ds.push_back(std::sqrt(rgb_dist2(f, v, v + w)));
    }
  if (ds.empty()) return 0.0;
  std::nth_element(ds.begin(), ds.begin() + static_cast<long>(ds.size() / 2), ds.end());
  return ds[ds.size() / 2];
}

// graph.cpp:105-159 — 4-neighbour heat-kernel graph, 1e-12 floor, isolated
// vertex repair with the strongest incident edge.
Graph build_image_graph(int h, int w, const std::vector<double>& f, double sigma) {
  if (sigma <= 0.0) throw ConfigError("build_image_graph: sigma must be > 0");
  const long n = static_cast<long>(h) * w;
  if (n < 2) throw ConfigError("build_image_graph: grid must have at least 2 pixels");
  const double floor_w = 1e-12;
  const double inv = 1.0 / (2.0 * sigma * sigma);
  struct E {
    int i, j;
    double w;
  };
  std::vector<E> kept;
  std::vector<E> best(static_cast<size_t>(n), E{-1, -1, -1.0});
  auto consider = [&](int a, int b) {
    const double wt = std::exp(-rgb_dist2(f, a, b) * inv);
    if (wt >= floor_w) kept.push_back({a, b, wt});
    for (int v : {a, b})
      if (wt > best[static_cast<size_t>(v)].w) best[static_cast<size_t>(v)] = {a, b, wt};
  };
  for (int r = 0; r < h; ++r)
    for (int c = 0; c < w; ++c) {
      const int v = r * w + c;
      if (c + 1 < w) consider(v, v + 1);
      if (r + 1 < h) consider(v, v + w);
    }
  Vec deg(static_cast<size_t>(n), 0.0);
  for (const E& e : kept) {
    deg[e.i] += e.w;
    deg[e.j] += e.w;
  }
  for (long v = 0; v < n; ++v) {
    if (deg[static_cast<size_t>(v)] > 0.0) continue;
    E e = best[static_cast<size_t>(v)];
    e.w = std::max(e.w, floor_w);
    kept.push_back(e);
    deg[e.i] += e.w;
    deg[e.j] += e.w;
  }
  std::sort(kept.begin(), kept.end(),
            [](const E& a, const E& b) { return a.i != b.i ? a.i < b.i : a.j < b.j; });
  kept.erase(std::unique(kept.begin(), kept.end(),
                         [](const E& a, const E& b) { return a.i == b.i && a.j == b.j; }),
             kept.end());
  Graph g;
  g.n = static_cast<int>(n);
  for (const E& e : kept) {
    g.ei.push_back(e.i);
    g.ej.push_back(e.j);
    g.w.push_back(e.w);
  }
  g.degree = degree_vector(g);
  g.sigma = sigma;
  return g;
}

// ------------------------------------------------------------------ solver --

// solver.cpp:14-17
double objective(const Csr& m, const Mat& y) {
  if (y.rows != m.ncols) throw ConfigError("objective: dimension mismatch");
  Mat my = spmm_dense(m, y);
  double s = 0.0;
  for (double v : my.a) s += std::abs(v);
  return s;
}

// solver.cpp:19-25
Mat shrink(const Mat& v, double gamma) {
  if (gamma < 0.0) throw ConfigError("shrink: gamma must be >= 0");
  Mat out(v.rows, v.cols);
  for_ranges(static_cast<long>(v.a.size()), [&](long lo, long hi) {
    for (long i = lo; i < hi; ++i) {
      const double x = v.a[i];
      const double mag = std::abs(x) - gamma;
      out.a[i] = mag > 0.0 ? (x > 0.0 ? mag : -mag) : 0.0;
    }
  });
  return out;
}

// solver.cpp:27-41 — thin SVD A = U S V^T, P = U V^T; singular values below
// 1e-12 * max(1, s_max) are rank deficiency.  The reference uses Eigen's
// JacobiSVD (QR preconditioner + Jacobi sweeps on R); this restatement uses
// Householder QR followed by one-sided Jacobi on the d x d factor R, which
// yields the same (unique, full-rank) polar factor.
Mat project_orthogonal(const Mat& a) {
  if (a.rows < a.cols) throw ConfigError("project_orthogonal: need rows >= cols");
  const long n = a.rows, d = a.cols;
  Mat qr = a;
  Vec tau(static_cast<size_t>(d), 0.0);
  // Householder QR, reflectors stored below the diagonal (v_k(k) = 1 implied).
  for (long k = 0; k < d; ++k) {
    double* c = qr.col(k);
    double nrm = 0.0;
    for (long i = k; i < n; ++i) nrm += c[i] * c[i];
    nrm = std::sqrt(nrm);
    if (nrm == 0.0) {
      tau[k] = 0.0;
      continue;
    }
    const double alpha = c[k] > 0.0 ? -nrm : nrm;
    const double v0 = c[k] - alpha;
    for (long i = k + 1; i < n; ++i) c[i] /= v0;
    tau[k] = -v0 / alpha;  // H = I - tau v v^T with v = [1, c[k+1..]]
    c[k] = alpha;
    for (long j = k + 1; j < d; ++j) {
      double* cj = qr.col(j);
      double s = cj[k];
      for (long i = k + 1; i < n; ++i) s += c[i] * cj[i];
      s *= tau[k];
      cj[k] -= s;
      for (long i = k + 1; i < n; ++i) cj[i] -= s * c[i];
    }
  }
  // R (d x d), one-sided Jacobi: R V = U S.
  Mat w(d, d), v(d, d);
  for (long j = 0; j < d; ++j) {
    for (long i = 0; i <= j; ++i) w(i, j) = qr(i, j);
    v(j, j) = 1.0;
  }
  for (int sweep = 0; sweep < 100; ++sweep) {
    double off = 0.0;
    for (long p = 0; p < d; ++p)
      for (long q = p + 1; q < d; ++q) {
        double al = 0.0, be = 0.0, ga = 0.0;
        for (long i = 0; i < d; ++i) {
          al += w(i, p) * w(i, p);
          be += w(i, q) * w(i, q);
          ga += w(i, p) * w(i, q);
        }
        if (ga == 0.0 || std::abs(ga) <= 1e-15 * std::sqrt(al * be)) continue;
        off = std::max(off, std::abs(ga) / std::sqrt(al * be));
        const double zeta = (be - al) / (2.0 * ga);
        const double t = (zeta >= 0.0 ? 1.0 : -1.0) / (std::abs(zeta) + std::sqrt(1.0 + zeta * zeta));
        const double cs = 1.0 / std::sqrt(1.0 + t * t), sn = cs * t;
        for (long i = 0; i < d; ++i) {
          const double x = w(i, p), y = w(i, q);
          w(i, p) = cs * x - sn * y;
          w(i, q) = sn * x + cs * y;
          const double vx = v(i, p), vy = v(i, q);
          v(i, p) = cs * vx - sn * vy;
          v(i, q) = sn * vx + cs * vy;
        }
      }
    if (off <= 1e-15) break;
  }
  Vec sv(static_cast<size_t>(d));
  double smax = 0.0;
  for (long j = 0; j < d; ++j) {
    double s = 0.0;
    for (long i = 0; i < d; ++i) s += w(i, j) * w(i, j);
    sv[j] = std::sqrt(s);
    smax = std::max(smax, sv[j]);
  }
  const double tol = 1e-12 * std::max(1.0, smax);
  int deficient = 0;
  for (long j = 0; j < d; ++j)
    if (sv[j] <= tol) ++deficient;
  if (deficient > 0)
    throw NumericalError("project_orthogonal: input rank-deficient in " + std::to_string(deficient) +
                         " column(s)");
  // P_R = U_R V^T (d x d), embedded as the top block of an n x d matrix, then Q applied.
  Mat p(n, d);
  for (long i = 0; i < d; ++i)
    for (long j = 0; j < d; ++j) {
      double s = 0.0;
      for (long k = 0; k < d; ++k) s += (w(i, k) / sv[k]) * v(j, k);
      p(i, j) = s;
    }
  for (long k = d - 1; k >= 0; --k) {
    if (tau[k] == 0.0) continue;
    const double* c = qr.col(k);
    for (long j = 0; j < d; ++j) {
      double* pj = p.col(j);
      double s = pj[k];
      for (long i = k + 1; i < n; ++i) s += c[i] * pj[i];
      s *= tau[k];
      pj[k] -= s;
      for (long i = k + 1; i < n; ++i) pj[i] -= s * c[i];
    }
  }
  return p;
}

// solver.cpp:43-58
PfeSolver::PfeSolver(const Graph& g, const Params& params)
    : params_(params), n_(g.n), m_(difference_matrix(g)), mt_(transpose(m_)), degree_(g.degree) {
  sqrt_degree_.resize(degree_.size());
  for (size_t i = 0; i < degree_.size(); ++i) sqrt_degree_[i] = std::sqrt(degree_[i]);
  op_ = PcgOperator(form_normal_matrix(m_, g.degree, params.lambda, params.r), params.pcg);
  if (params.dim < 1) throw ConfigError("PfeSolver: dim must be >= 1");
  if (params.lambda <= 0.0 || params.r <= 0.0) throw ConfigError("PfeSolver: lambda and r must be > 0");
  if (params.soc_max < 1 || params.sb_max_stage1 < 1)
    throw ConfigError("PfeSolver: iteration caps must be >= 1");
}

// solver.cpp:60-71
State PfeSolver::make_state(const Mat& y0) const {
  if (y0.rows != n_ || y0.cols != params_.dim)
    throw ConfigError("PfeSolver: initial embedding has wrong shape");
  State st;
  st.y = y0;
  st.p = Mat(n_, params_.dim);
  for (long j = 0; j < y0.cols; ++j)
    for (long i = 0; i < n_; ++i) st.p(i, j) = sqrt_degree_[i] * y0(i, j);
  st.bregman = Mat(n_, params_.dim);
  st.split_b = Mat(m_.nrows, params_.dim);
  st.split_s = Mat(m_.nrows, params_.dim);
  return st;
}

namespace {
// The body shared by PfeSolver::split_bregman (solver.cpp:73-108) and the
// standalone split_bregman (solver.cpp:138-182).
void sb_loop(State& st, int max_iter, const IterCb& cb, const Csr& m, const Csr& mt,
             const Vec& sqrt_deg, const PcgOperator& op, double lambda, double r, double conv_tol,
             bool warn, RunLog* log) {
  const double hl = 0.5 * lambda, hr = 0.5 * r;
  const long n = st.y.rows, d = st.y.cols, ne = st.split_b.rows;
  Mat rhs_quad(n, d);
  for (long j = 0; j < d; ++j)
    for (long i = 0; i < n; ++i) rhs_quad(i, j) = hr * (sqrt_deg[i] * (st.p(i, j) - st.bregman(i, j)));
  for (int it = 0; it < max_iter; ++it) {
    const auto t0 = std::chrono::steady_clock::now();
    Mat sb(ne, d);
    // elementwise loops may run on several threads (no reductions: bitwise
    // identical); every dot / norm stays sequential
    for_ranges(static_cast<long>(sb.a.size()), [&](long lo, long hi) {
      for (long k = lo; k < hi; ++k) sb.a[k] = st.split_s.a[k] - st.split_b.a[k];
    });
    Mat rhs = spmm_dense(mt, sb);
    for_ranges(static_cast<long>(rhs.a.size()), [&](long lo, long hi) {
      for (long k = lo; k < hi; ++k) rhs.a[k] = hl * rhs.a[k] + rhs_quad.a[k];
    });
    Mat y_old = st.y;
    Mat y_new;
    std::vector<PcgReport> reps = op.solve_multi(rhs, st.y, y_new);
    int kmax = 0;
    for (size_t j = 0; j < reps.size(); ++j) {
      kmax = std::max(kmax, reps[j].iterations);
      if (warn && !reps[j].converged)
        // stdio, not iostream: a ctypes-loaded oracle can share the process
        // with another libstdc++ whose locale facets crash num_put
        std::fprintf(stderr, "pfe: inner solve column %zu stopped at rel residual %g\n", j,
                     reps[j].final_rel_residual);
    }
    if (log) {
      log->pcg_iters.push_back(kmax);
      ++log->inner_iterations;
    }
    st.y = std::move(y_new);
    if (!all_finite(st.y.a.data(), static_cast<long>(st.y.a.size())))
      throw NumericalError("split_bregman: NaN in embedding");
    Mat my = spmm_dense(m, st.y);
    Mat t(ne, d);
    for_ranges(static_cast<long>(t.a.size()), [&](long lo, long hi) {
      for (long k = lo; k < hi; ++k) t.a[k] = my.a[k] + st.split_b.a[k];
    });
    st.split_s = shrink(t, 1.0 / lambda);
    for_ranges(static_cast<long>(t.a.size()), [&](long lo, long hi) {
      for (long k = lo; k < hi; ++k) st.split_b.a[k] += my.a[k] - st.split_s.a[k];
    });
    if (log) log->t_inner += std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    if (cb) cb(it, st.y);
    const double den = mat_norm(y_old);
    if (conv_tol > 0.0 && den > 0.0) {
      Mat df(n, d);
      for (size_t k = 0; k < df.a.size(); ++k) df.a[k] = st.y.a[k] - y_old.a[k];
      if (mat_norm(df) / den <= conv_tol) break;
    }
  }
}
}  // namespace

void PfeSolver::split_bregman(State& st, int max_iter, const IterCb& cb) const {
  sb_loop(st, max_iter, cb, m_, mt_, sqrt_degree_, op_, params_.lambda, params_.r, params_.conv_tol,
          true, log);
}

// solver.cpp:116-118: dy = sqrt(D) Y; P = project_orthogonal(dy + B); B += dy - P
void PfeSolver::outer_update(State& st) const {
  const auto t0 = std::chrono::steady_clock::now();
  const long n = st.y.rows, d = st.y.cols;
  Mat dy(n, d), a(n, d);
  for (long j = 0; j < d; ++j)
    for (long i = 0; i < n; ++i) {
      dy(i, j) = sqrt_degree_[i] * st.y(i, j);
      a(i, j) = dy(i, j) + st.bregman(i, j);
    }
  st.p = project_orthogonal(a);
  for (size_t q = 0; q < dy.a.size(); ++q) st.bregman.a[q] += dy.a[q] - st.p.a[q];
  if (log) log->t_outer += std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
}

// solver.cpp:110-126
void PfeSolver::run_soc(State& st, int soc_max, int sb_max) const {
  for (int k = 0; k < soc_max; ++k) {
    std::fill(st.split_b.a.begin(), st.split_b.a.end(), 0.0);
    std::fill(st.split_s.a.begin(), st.split_s.a.end(), 0.0);
    Mat y_old = st.y;
    split_bregman(st, sb_max);
    outer_update(st);
    const long n = st.y.rows, d = st.y.cols;
    const double den = mat_norm(y_old);
    if (params_.conv_tol > 0.0 && den > 0.0) {
      Mat df(n, d);
      for (size_t q = 0; q < df.a.size(); ++q) df.a[q] = st.y.a[q] - y_old.a[q];
      if (mat_norm(df) / den <= params_.conv_tol) break;
    }
  }
}

// solver.cpp:128-136
State PfeSolver::two_stage(const Mat& y0) const {
  State st = make_state(y0);
  run_soc(st, params_.soc_max, params_.sb_max_stage1);
  if (params_.sb_max_stage2 > 0) split_bregman(st, params_.sb_max_stage2);
  return st;
}

// solver.cpp:138-182
Mat split_bregman(const Csr& m, const Vec& d_vec, const Mat& p, const Mat& b, const Params& params,
                  const Mat& y_init, int max_iter, const IterCb& cb) {
  State st;
  st.y = y_init;
  st.p = p;
  st.bregman = b;
  st.split_b = Mat(m.nrows, y_init.cols);
  st.split_s = Mat(m.nrows, y_init.cols);
  PcgOperator op(form_normal_matrix(m, d_vec, params.lambda, params.r), params.pcg);
  Csr mt = transpose(m);
  Vec sq(d_vec.size());
  for (size_t i = 0; i < d_vec.size(); ++i) sq[i] = std::sqrt(d_vec[i]);
  sb_loop(st, max_iter, cb, m, mt, sq, op, params.lambda, params.r, params.conv_tol, false, nullptr);
  return st.y;
}

Mat soc(const Graph& g, const Params& params, const Mat& y0) {
  PfeSolver s(g, params);
  State st = s.make_state(y0);
  s.run_soc(st, params.soc_max, params.sb_max_stage1);
  return st.y;
}

Mat pfe_two_stage(const Graph& g, const Params& params, const Mat& y0) {
  return PfeSolver(g, params).two_stage(y0).y;
}

// -------------------------------------------------------------------- init --
namespace {
// init.cpp:19-27
double diag_loglik(const double* x, const Mat& means, const Mat& vars, int j) {
  double ll = -1.5 * std::log(2.0 * M_PI);
  for (int c = 0; c < 3; ++c) {
    const double df = x[c] - means(j, c);
    ll -= 0.5 * (std::log(vars(j, c)) + df * df / vars(j, c));
  }
  return ll;
}
// init.cpp:30-41
long farthest_point(const Mat& f, const Mat& means) {
  long best = 0;
  double best_d = -1.0;
  for (long i = 0; i < f.rows; ++i) {
    double dmin = std::numeric_limits<double>::infinity();
    for (long j = 0; j < means.rows; ++j) {
      double s = 0.0;
      for (long c = 0; c < f.cols; ++c) {
        const double df = means(j, c) - f(i, c);
        s += df * df;
      }
      dmin = std::min(dmin, s);
    }
    if (dmin > best_d) {
      best_d = dmin;
      best = i;
    }
  }
  return best;
}
}  // namespace

// init.cpp:45-121
Gmm gmm_fit(const Mat& f, int k, uint64_t seed) {
  const long n = f.rows;
  if (k < 1) throw ConfigError("gmm_fit: k must be >= 1");
  if (n < k) throw ConfigError("gmm_fit: fewer points than components");
  if (f.cols != 3) throw ConfigError("gmm_fit: features must be n x 3");
  if (!all_finite(f.a.data(), static_cast<long>(f.a.size()))) throw ConfigError("gmm_fit: non-finite features");
  Gmm g;
  g.k = k;
  g.means = Mat(k, 3);
  g.variances = Mat(k, 3, 1e-2);
  g.weights.assign(static_cast<size_t>(k), 1.0 / k);
  std::vector<int> lab = kmeans(f, k, seed, 20);
  Vec cnt(static_cast<size_t>(k), 0.0);
  for (long i = 0; i < n; ++i) {
    for (int c = 0; c < 3; ++c) g.means(lab[i], c) += f(i, c);
    cnt[lab[i]] += 1.0;
  }
  for (int j = 0; j < k; ++j)
    if (cnt[j] > 0.0)
      for (int c = 0; c < 3; ++c) g.means(j, c) /= cnt[j];

  Mat resp(n, k);
  double prev = -std::numeric_limits<double>::infinity();
  int repairs = 0;
  Vec lp(static_cast<size_t>(k)), ex(static_cast<size_t>(k));
  double x[3];
  for (int iter = 0; iter < 50; ++iter) {
    double loglik = 0.0;
    for (long i = 0; i < n; ++i) {
      for (int c = 0; c < 3; ++c) x[c] = f(i, c);
      for (int j = 0; j < k; ++j) lp[j] = std::log(g.weights[j]) + diag_loglik(x, g.means, g.variances, j);
      double mx = lp[0];
      for (int j = 1; j < k; ++j) mx = std::max(mx, lp[j]);
      double s = 0.0;
      for (int j = 0; j < k; ++j) {
        ex[j] = std::exp(lp[j] - mx);
        s += ex[j];
      }
      for (int j = 0; j < k; ++j) resp(i, j) = ex[j] / s;
      loglik += mx + std::log(s);
    }
    bool repaired = false;
    for (int j = 0; j < k; ++j) {
      double nj = 0.0;
      for (long i = 0; i < n; ++i) nj += resp(i, j);
      if (nj < 1e-8 && repairs < 5) {
        const long fi = farthest_point(f, g.means);
        for (int c = 0; c < 3; ++c) {
          g.means(j, c) = f(fi, c);
          g.variances(j, c) = 1e-2;
        }
        g.weights[j] = 1.0 / n;
        ++repairs;
        repaired = true;
        continue;
      }
      if (nj <= 0.0) continue;
      double mean[3] = {0, 0, 0}, var[3] = {0, 0, 0};
      for (int c = 0; c < 3; ++c) {
        double s = 0.0;
        for (long i = 0; i < n; ++i) s += resp(i, j) * f(i, c);
        mean[c] = s / nj;
      }
      for (long i = 0; i < n; ++i)
        for (int c = 0; c < 3; ++c) {
          const double df = f(i, c) - mean[c];
          var[c] += resp(i, j) * (df * df);
        }
      for (int c = 0; c < 3; ++c) {
        var[c] /= nj;
        g.means(j, c) = mean[c];
        g.variances(j, c) = std::max(var[c], 1e-6);
      }
      g.weights[j] = nj / n;
    }
    double ws = 0.0;
    for (int j = 0; j < k; ++j) ws += g.weights[j];
    for (int j = 0; j < k; ++j) g.weights[j] /= ws;
    if (!repaired && loglik - prev < 1e-7 && iter > 0) break;
    prev = loglik;
  }
  return g;
}

// init.cpp:123-138
Mat responsibilities(const Gmm& g, const Mat& f) {
  const long n = f.rows;
  Mat resp(n, g.k);
  Vec lp(static_cast<size_t>(g.k)), ex(static_cast<size_t>(g.k));
  double x[3];
  for (long i = 0; i < n; ++i) {
    for (int c = 0; c < 3; ++c) x[c] = f(i, c);
    for (int j = 0; j < g.k; ++j) lp[j] = std::log(g.weights[j]) + diag_loglik(x, g.means, g.variances, j);
    double mx = lp[0];
    for (int j = 1; j < g.k; ++j) mx = std::max(mx, lp[j]);
    double s = 0.0;
    for (int j = 0; j < g.k; ++j) {
      ex[j] = std::exp(lp[j] - mx);
      s += ex[j];
    }
    for (int j = 0; j < g.k; ++j) resp(i, j) = ex[j] / s;
  }
  return resp;
}

// init.cpp:140-155 — modified Gram-Schmidt in <u, v> = u^T diag(deg) v.
Mat d_orthonormalize(const Mat& a, const Vec& deg) {
  if (a.rows != static_cast<long>(deg.size())) throw ConfigError("d_orthonormalize: size mismatch");
  Mat q = a;
  const long n = q.rows;
  for (long j = 0; j < q.cols; ++j) {
    double* qj = q.col(j);
    for (long i = 0; i < j; ++i) {
      const double* qi = q.col(i);
      double proj = 0.0;
      for (long t = 0; t < n; ++t) proj += qj[t] * (deg[t] * qi[t]);
      for (long t = 0; t < n; ++t) qj[t] -= proj * qi[t];
    }
    double s = 0.0;
    for (long t = 0; t < n; ++t) s += qj[t] * (deg[t] * qj[t]);
    const double nrm = std::sqrt(s);
    if (nrm < 1e-10) throw NumericalError("d_orthonormalize: dependent column " + std::to_string(j));
    for (long t = 0; t < n; ++t) qj[t] /= nrm;
  }
  return q;
}

// init.cpp:157-170
Mat init_embedding(const Gmm& g, const Mat& f, const Vec& deg) {
  Mat resp = responsibilities(g, f);
  try {
    return d_orthonormalize(resp, deg);
  } catch (const NumericalError&) {
    std::mt19937_64 rng(0x9e3779b97f4a7c15ull);
    std::normal_distribution<double> dist(0.0, 1e-6);
    for (long i = 0; i < resp.rows; ++i)
      for (long j = 0; j < resp.cols; ++j) resp(i, j) += dist(rng);
    return d_orthonormalize(resp, deg);
  }
}

// init.cpp:172-181 — row-major draw order from mt19937_64 + libstdc++ normal.
Mat random_embedding(int n, int d, uint64_t seed, const Vec& deg) {
  std::mt19937_64 rng(seed);
  std::normal_distribution<double> dist(0.0, 1.0);
  Mat a(n, d);
  for (long i = 0; i < n; ++i)
    for (long j = 0; j < d; ++j) a(i, j) = dist(rng);
  return d_orthonormalize(a, deg);
}

// ----------------------------------------------------------------- cluster --
namespace {
double row_dist2(const Mat& p, long i, const Mat& c, long j) {
  double s = 0.0;
  for (long t = 0; t < p.cols; ++t) {
    const double df = p(i, t) - c(j, t);
    s += df * df;
  }
  return s;
}
// cluster.cpp:15-51 — k-means++ seeding.
Mat seed_centroids(const Mat& pts, int k, std::mt19937_64& rng) {
  const long n = pts.rows;
  Mat cen(k, pts.cols);
  std::uniform_int_distribution<long> first(0, n - 1);
  const long f0 = first(rng);
  for (long t = 0; t < pts.cols; ++t) cen(0, t) = pts(f0, t);
  Vec d2(static_cast<size_t>(n));
  for_ranges(n, [&](long lo, long hi) {
    for (long i = lo; i < hi; ++i) d2[i] = row_dist2(pts, i, cen, 0);
  });
  std::uniform_real_distribution<double> uni(0.0, 1.0);
  for (int c = 1; c < k; ++c) {
    double total = 0.0;
    for (long i = 0; i < n; ++i) total += d2[i];
    long chosen = 0;
    if (total > 0.0) {
      const double target = uni(rng) * total;
      double acc = 0.0;
      for (long i = 0; i < n; ++i) {
        acc += d2[i];
        if (acc >= target) {
          chosen = i;
          break;
        }
      }
    } else {
      chosen = first(rng);
    }
    for (long t = 0; t < pts.cols; ++t) cen(c, t) = pts(chosen, t);
    for_ranges(n, [&](long lo, long hi) {
      for (long i = lo; i < hi; ++i) d2[i] = std::min(d2[i], row_dist2(pts, i, cen, c));
    });
  }
  return cen;
}
}  // namespace

// cluster.cpp:54-124 — Lloyd with lowest-index ties and empty-cluster split.
std::vector<int> kmeans(const Mat& pts, int k, uint64_t seed, int max_iter) {
  const long n = pts.rows;
  if (k < 1) throw ConfigError("kmeans: k must be >= 1");
  if (k > n) throw ConfigError("kmeans: k exceeds point count");
  std::mt19937_64 rng(seed);
  Mat cen = seed_centroids(pts, k, rng);
  std::vector<int> lab(static_cast<size_t>(n), 0);
  Vec bdist(static_cast<size_t>(n));
  double prev = std::numeric_limits<double>::infinity();
  for (int iter = 0; iter < max_iter; ++iter) {
    double inertia = 0.0;
    for_ranges(n, [&](long lo, long hi) {
      for (long i = lo; i < hi; ++i) {
        int best = 0;
        double bd = row_dist2(pts, i, cen, 0);
        for (int c = 1; c < k; ++c) {
          const double dd = row_dist2(pts, i, cen, c);
          if (dd < bd) {
            bd = dd;
            best = c;
          }
        }
        lab[i] = best;
        bdist[i] = bd;
      }
    });
    for (long i = 0; i < n; ++i) inertia += bdist[i];  // point order, as cluster.cpp sums it
    Mat sums(k, pts.cols);
    std::vector<long> cnt(static_cast<size_t>(k), 0);
    for (long i = 0; i < n; ++i) {
      for (long t = 0; t < pts.cols; ++t) sums(lab[i], t) += pts(i, t);
      ++cnt[lab[i]];
    }
    for (int c = 0; c < k; ++c) {
      if (cnt[c] > 0) {
        for (long t = 0; t < pts.cols; ++t) cen(c, t) = sums(c, t) / static_cast<double>(cnt[c]);
        continue;
      }
      int largest = 0;
      for (int c2 = 1; c2 < k; ++c2)
        if (cnt[c2] > cnt[largest]) largest = c2;
      long far_i = -1;
      double far_d = -1.0;
      for (long i = 0; i < n; ++i) {
        if (lab[i] != largest) continue;
        const double dd = row_dist2(pts, i, cen, largest);
        if (dd > far_d) {
          far_d = dd;
          far_i = i;
        }
      }
      for (long t = 0; t < pts.cols; ++t) cen(c, t) = pts(far_i, t);
      lab[far_i] = c;
      cnt[c] = 1;
      cnt[largest]--;
    }
    if (prev - inertia <= 1e-6 * std::max(prev, 1e-300) && inertia <= prev) break;
    prev = inertia;
  }
  return lab;
}

// metrics.cpp:57-72 (with the contingency table of metrics.cpp:15-51).
double covering(const std::vector<int>& pred, const std::vector<int>& gt) {
  if (pred.size() != gt.size()) throw ConfigError("metrics: segmentations have different sizes");
  if (pred.empty()) throw ConfigError("metrics: empty segmentation");
  auto compact = [](const std::vector<int>& l, int& k) {
    std::unordered_map<int, int> remap;
    std::vector<int> out(l.size());
    for (size_t i = 0; i < l.size(); ++i) {
      auto it = remap.try_emplace(l[i], static_cast<int>(remap.size())).first;
      out[i] = it->second;
    }
    k = static_cast<int>(remap.size());
    return out;
  };
  int ka = 0, kb = 0;
  std::vector<int> la = compact(gt, ka), lb = compact(pred, kb);
  std::map<std::pair<int, int>, long long> joint;
  std::vector<long long> row(static_cast<size_t>(ka), 0), col(static_cast<size_t>(kb), 0);
  for (size_t i = 0; i < la.size(); ++i) {
    joint[{la[i], lb[i]}]++;
    row[la[i]]++;
    col[lb[i]]++;
  }
  double acc = 0.0;
  for (int g = 0; g < ka; ++g) {
    double best = 0.0;
    for (int p = 0; p < kb; ++p) {
      auto it = joint.find({g, p});
      if (it == joint.end()) continue;
      const double inter = static_cast<double>(it->second);
      const double uni = static_cast<double>(row[g] + col[p]) - inter;
      best = std::max(best, inter / uni);
    }
    acc += static_cast<double>(row[g]) * best;
  }
  return acc / static_cast<double>(la.size());
}

}  // namespace orc
