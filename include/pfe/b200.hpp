// C++ drop-in facade over the B200 C ABI (pfe_b200.h), mirroring the
// reference library interface in /root/reference/proj/core/include/pfe:
//
//   pfe::PfeParams, PcgConfig, Preconditioner, PcgReport  (solver.hpp:16-25, pcg.hpp:13-26)
//   pfe::WeightedGraph                                     (graph.hpp:15-28)
//   pfe::CsrMatrix, difference_matrix, degree_vector       (sparse.hpp:17-25, graph.cpp:161-174)
//   pfe::SolverState, IterateCallback                      (solver.hpp:28-36)
//   pfe::PfeSolver {make_state, split_bregman, run_soc, two_stage, diff_matrix, params}
//   pfe::objective / shrink / project_orthogonal / split_bregman / soc / pfe_two_stage
//   pfe::PcgOperator / pcg_solve / pcg_solve_multi         (pcg.hpp:31-63)
//   pfe::random_embedding / d_orthonormalize / kmeans      (init.hpp, cluster.hpp)
//   pfe::IoError / NumericalError / ConfigError            (errors.hpp:9-24)
//
// Header-only; link with libpfe_b200.so.  Matrices are the reference's
// column-major n x d layout: Eigen::MatrixXd when Eigen is available,
// otherwise the minimal pfe::Matrix below with the same element layout and
// accessors (rows(), cols(), data(), operator()(i, j)).
#pragma once

#include <algorithm>
#include <cstdint>
#include <functional>
#include <memory>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "pfe_b200.h"

#if defined(PFE_B200_USE_EIGEN) || (defined(__has_include) && __has_include(<Eigen/Dense>))
#include <Eigen/Dense>
#define PFE_B200_HAVE_EIGEN 1
#endif

namespace pfe {

// ---------------------------------------------------------------- errors --
class IoError : public std::runtime_error {
 public:
  explicit IoError(const std::string& m) : std::runtime_error(m) {}
};
class NumericalError : public std::runtime_error {
 public:
  explicit NumericalError(const std::string& m) : std::runtime_error(m) {}
};
class ConfigError : public std::invalid_argument {
 public:
  explicit ConfigError(const std::string& m) : std::invalid_argument(m) {}
};
class DeviceError : public std::runtime_error {
 public:
  explicit DeviceError(const std::string& m) : std::runtime_error(m) {}
};

namespace detail {
inline void check(int rc) {
  if (rc == PFE_OK) return;
  const std::string msg = pfe_last_error();
  switch (rc) {
    case PFE_IO_ERROR:
      throw IoError(msg);
    case PFE_NUMERICAL_ERROR:
      throw NumericalError(msg);
    case PFE_CONFIG_ERROR:
      throw ConfigError(msg);
    default:
      throw DeviceError(msg);
  }
}
}  // namespace detail

// -------------------------------------------------------------- matrices --
#ifdef PFE_B200_HAVE_EIGEN
using Matrix = Eigen::MatrixXd;
using Vector = Eigen::VectorXd;
#else
class Matrix {
 public:
  Matrix() = default;
  Matrix(long r, long c) : r_(r), c_(c), a_(static_cast<size_t>(r * c), 0.0) {}
  static Matrix Zero(long r, long c) { return Matrix(r, c); }
  long rows() const { return r_; }
  long cols() const { return c_; }
  long size() const { return r_ * c_; }
  double* data() { return a_.data(); }
  const double* data() const { return a_.data(); }
  double& operator()(long i, long j) { return a_[static_cast<size_t>(i + j * r_)]; }
  double operator()(long i, long j) const { return a_[static_cast<size_t>(i + j * r_)]; }
  void resize(long r, long c) {
    r_ = r;
    c_ = c;
    a_.assign(static_cast<size_t>(r * c), 0.0);
  }
  bool operator==(const Matrix& o) const { return r_ == o.r_ && c_ == o.c_ && a_ == o.a_; }

 private:
  long r_ = 0, c_ = 0;
  std::vector<double> a_;
};
class Vector {
 public:
  Vector() = default;
  explicit Vector(long n) : a_(static_cast<size_t>(n), 0.0) {}
  Vector(std::initializer_list<double> v) : a_(v) {}
  long size() const { return static_cast<long>(a_.size()); }
  double* data() { return a_.data(); }
  const double* data() const { return a_.data(); }
  double& operator[](long i) { return a_[static_cast<size_t>(i)]; }
  double operator[](long i) const { return a_[static_cast<size_t>(i)]; }
  double& operator()(long i) { return a_[static_cast<size_t>(i)]; }
  double operator()(long i) const { return a_[static_cast<size_t>(i)]; }
  void resize(long n) { a_.assign(static_cast<size_t>(n), 0.0); }

 private:
  std::vector<double> a_;
};
#endif

using Embedding = Matrix;  // n x d, column-major (solver.hpp:14)

// ------------------------------------------------------------ parameters --
enum class Preconditioner { Ic0 = PFE_PRECOND_IC0, Jacobi = PFE_PRECOND_JACOBI, None = PFE_PRECOND_NONE };

struct PcgConfig {
  double rel_tol = 1e-6;
  int max_iter = 1000;
  Preconditioner preconditioner = Preconditioner::Ic0;
};

struct PcgReport {
  int iterations = 0;
  double final_rel_residual = 0.0;
  bool converged = false;
  bool jacobi_fallback = false;
};

struct PfeParams {
  int dim = 5;
  double lambda = 100.0;
  double r = 1.0;
  int soc_max = 10;
  int sb_max_stage1 = 5;
  int sb_max_stage2 = 100;
  double conv_tol = 1e-4;
  PcgConfig pcg{1e-6, 1000, Preconditioner::Ic0};
};

/// Execution options of the B200 backend (no reference counterpart).
struct ExecOptions {
  int device = 0;
  bool use_graphs = true;
  bool warn = true;
  bool profile = false;
  bool persistent = true;
};

// ----------------------------------------------------------------- graph --
struct WeightedGraph {
  struct Edge {
    int i;
    int j;
    double w;
  };
  int n = 0;
  std::vector<Edge> edges;
  Vector degree;
  double sigma = 0.0;
  // B200 extension: pixel-grid hint (height, width, radius) enabling the
  // stencil kernels; results do not depend on it.
  int grid_h = 0, grid_w = 0, grid_radius = 0;

  int edge_count() const { return static_cast<int>(edges.size()); }
};

struct CsrMatrix {
  int nrows = 0;
  int ncols = 0;
  std::vector<int> row_ptr;
  std::vector<int> col_idx;
  std::vector<double> values;
  int nnz() const { return static_cast<int>(values.size()); }
};

/// |E| x n matrix, row k = +w at i, -w at j (graph.cpp:161-170).
inline CsrMatrix difference_matrix(const WeightedGraph& g) {
  CsrMatrix m;
  m.nrows = g.edge_count();
  m.ncols = g.n;
  m.row_ptr.assign(static_cast<size_t>(m.nrows) + 1, 0);
  for (int k = 0; k < m.nrows; ++k) {
    const auto& e = g.edges[static_cast<size_t>(k)];
    const bool fwd = e.i < e.j;
    m.col_idx.push_back(fwd ? e.i : e.j);
    m.values.push_back(fwd ? e.w : -e.w);
    m.col_idx.push_back(fwd ? e.j : e.i);
    m.values.push_back(fwd ? -e.w : e.w);
    m.row_ptr[static_cast<size_t>(k) + 1] = 2 * (k + 1);
  }
  return m;
}

inline Vector degree_vector(const WeightedGraph& g) {
  Vector d(g.n);
  for (int t = 0; t < g.n; ++t) d[t] = 0.0;
  for (const auto& e : g.edges) {
    d[e.i] += e.w;
    d[e.j] += e.w;
  }
  return d;
}

namespace detail {
struct FlatGraph {
  std::vector<int32_t> ei, ej;
  std::vector<double> w, deg;
  pfe_graph view{};
};

inline std::shared_ptr<FlatGraph> flatten(const WeightedGraph& g, const Vector* deg_override = nullptr) {
  auto f = std::make_shared<FlatGraph>();
  f->ei.reserve(g.edges.size());
  f->ej.reserve(g.edges.size());
  f->w.reserve(g.edges.size());
  for (const auto& e : g.edges) {
    f->ei.push_back(e.i);
    f->ej.push_back(e.j);
    f->w.push_back(e.w);
  }
  const Vector& d = deg_override ? *deg_override : g.degree;
  if (d.size() != g.n) throw ConfigError("form_normal_matrix: degree size mismatch");
  f->deg.assign(d.data(), d.data() + d.size());
  f->view = pfe_graph{g.n, static_cast<int64_t>(f->w.size()), f->ei.data(), f->ej.data(), f->w.data(),
                      f->deg.data(), g.grid_h, g.grid_w, g.grid_radius};
  return f;
}

/// Recovers the edge list from an edge-incidence matrix (rows [+w, -w]).
inline WeightedGraph graph_from_difference(const CsrMatrix& m, const Vector& d_vec) {
  WeightedGraph g;
  g.n = m.ncols;
  g.degree = d_vec;
  for (int k = 0; k < m.nrows; ++k) {
    const int b = m.row_ptr[static_cast<size_t>(k)], e = m.row_ptr[static_cast<size_t>(k) + 1];
    if (e - b != 2 || m.values[static_cast<size_t>(b)] != -m.values[static_cast<size_t>(b) + 1])
      throw ConfigError("split_bregman: the B200 path needs an edge-incidence matrix (rows [+w, -w])");
    const int c0 = m.col_idx[static_cast<size_t>(b)], c1 = m.col_idx[static_cast<size_t>(b) + 1];
    const double v0 = m.values[static_cast<size_t>(b)];
    if (v0 > 0)
      g.edges.push_back({c0, c1, v0});
    else
      g.edges.push_back({c1, c0, -v0});
  }
  return g;
}

inline pfe_params to_c(const PfeParams& p) {
  return pfe_params{p.dim,          p.lambda,      p.r, p.soc_max, p.sb_max_stage1, p.sb_max_stage2, p.conv_tol,
                    p.pcg.rel_tol, p.pcg.max_iter, static_cast<int32_t>(p.pcg.preconditioner)};
}
inline pfe_exec to_c(const ExecOptions& x) {
  return pfe_exec{x.device, x.use_graphs ? 1 : 0, x.warn ? 1 : 0, x.profile ? 1 : 0, x.persistent ? 1 : 0};
}

template <class M>
M make_matrix(long r, long c) {
  M m(r, c);
  return m;
}
}  // namespace detail

struct SolverState {
  Matrix y;        // n x d embedding
  Matrix p;        // n x d orthogonality split variable
  Matrix bregman;  // n x d outer Bregman variable
  Matrix split_b;  // |E| x d inner Bregman variable
  Matrix split_s;  // |E| x d shrinkage variable
};

using IterateCallback = std::function<void(int iteration, const Matrix& y)>;

namespace detail {
struct CbCtx {
  const IterateCallback* cb;
};
inline void trampoline(int it, const double* y, int32_t n, int32_t d, void* user) {
  auto* c = static_cast<CbCtx*>(user);
  Matrix m = make_matrix<Matrix>(n, d);
  std::copy(y, y + static_cast<long>(n) * d, m.data());
  (*c->cb)(it, m);
}
}  // namespace detail

// ---------------------------------------------------------------- solver --
class PfeSolver {
 public:
  PfeSolver(const WeightedGraph& g, const PfeParams& params, const ExecOptions& exec = {})
      : params_(params), graph_(g), flat_(detail::flatten(g)) {
    const pfe_params pc = detail::to_c(params);
    const pfe_exec xc = detail::to_c(exec);
    pfe_solver* h = nullptr;
    detail::check(pfe_solver_create(&flat_->view, &pc, &xc, &h));
    h_.reset(h, pfe_solver_destroy);
  }

  SolverState make_state(const Embedding& y0) const {
    check_shape(y0);
    State st = device_state(y0);
    return download(st.get());
  }

  void split_bregman(SolverState& state, int max_iter, const IterateCallback& on_iterate = {}) const {
    check_shape(state.y);
    State st = upload(state);
    detail::CbCtx ctx{&on_iterate};
    detail::check(pfe_split_bregman(h_.get(), st.get(), max_iter, on_iterate ? &detail::trampoline : nullptr,
                                    on_iterate ? &ctx : nullptr));
    state = download(st.get());
  }

  void run_soc(SolverState& state, int soc_max, int sb_max) const {
    check_shape(state.y);
    State st = upload(state);
    detail::check(pfe_run_soc(h_.get(), st.get(), soc_max, sb_max));
    state = download(st.get());
  }

  SolverState two_stage(const Embedding& y0) const {
    check_shape(y0);
    State st = device_state(y0);
    detail::check(pfe_two_stage(h_.get(), st.get()));
    return download(st.get());
  }

  CsrMatrix diff_matrix() const { return difference_matrix(graph_); }
  const PfeParams& params() const { return params_; }

  pfe_report report() const {
    pfe_report r{};
    detail::check(pfe_solver_report(h_.get(), &r));
    return r;
  }

 private:
  using State = std::unique_ptr<pfe_state, void (*)(pfe_state*)>;

  void check_shape(const Matrix& y0) const {
    if (y0.rows() != graph_.n || y0.cols() != params_.dim)
      throw ConfigError("PfeSolver: initial embedding has wrong shape");
  }
  State device_state(const Matrix& y0) const {
    pfe_state* s = nullptr;
    detail::check(pfe_state_create(h_.get(), y0.data(), &s));
    return State(s, pfe_state_destroy);
  }
  State upload(const SolverState& v) const {
    State st = device_state(v.y);
    detail::check(pfe_state_set(st.get(), PFE_FIELD_P, v.p.data()));
    detail::check(pfe_state_set(st.get(), PFE_FIELD_BREGMAN, v.bregman.data()));
    detail::check(pfe_state_set(st.get(), PFE_FIELD_SPLIT_B, v.split_b.data()));
    detail::check(pfe_state_set(st.get(), PFE_FIELD_SPLIT_S, v.split_s.data()));
    return st;
  }
  SolverState download(pfe_state* st) const {
    const long n = graph_.n, m = graph_.edge_count(), d = params_.dim;
    SolverState v{detail::make_matrix<Matrix>(n, d), detail::make_matrix<Matrix>(n, d),
                  detail::make_matrix<Matrix>(n, d), detail::make_matrix<Matrix>(m, d),
                  detail::make_matrix<Matrix>(m, d)};
    detail::check(pfe_state_get(st, PFE_FIELD_Y, v.y.data()));
    detail::check(pfe_state_get(st, PFE_FIELD_P, v.p.data()));
    detail::check(pfe_state_get(st, PFE_FIELD_BREGMAN, v.bregman.data()));
    detail::check(pfe_state_get(st, PFE_FIELD_SPLIT_B, v.split_b.data()));
    detail::check(pfe_state_get(st, PFE_FIELD_SPLIT_S, v.split_s.data()));
    return v;
  }

  PfeParams params_;
  WeightedGraph graph_;
  std::shared_ptr<detail::FlatGraph> flat_;
  std::shared_ptr<pfe_solver> h_;
};

// ------------------------------------------------------------- free API --
inline double objective(const CsrMatrix& m, const Embedding& y, const ExecOptions& x = {}) {
  if (y.rows() != m.ncols) throw ConfigError("objective: dimension mismatch");
  Vector unit(m.ncols);
  for (int t = 0; t < m.ncols; ++t) unit[t] = 1.0;
  WeightedGraph g = detail::graph_from_difference(m, unit);
  auto f = detail::flatten(g);
  const pfe_exec xc = detail::to_c(x);
  double out = 0.0;
  detail::check(pfe_objective(&f->view, static_cast<int32_t>(y.cols()), y.data(), &xc, &out));
  return out;
}

inline Matrix shrink(const Matrix& v, double gamma, const ExecOptions& x = {}) {
  Matrix out = detail::make_matrix<Matrix>(v.rows(), v.cols());
  const pfe_exec xc = detail::to_c(x);
  detail::check(pfe_shrink(static_cast<int64_t>(v.size()), v.data(), gamma, &xc, out.data()));
  return out;
}

inline Matrix project_orthogonal(const Matrix& a, const ExecOptions& x = {}) {
  if (a.rows() < a.cols()) throw ConfigError("project_orthogonal: need rows >= cols");
  Matrix out = detail::make_matrix<Matrix>(a.rows(), a.cols());
  const pfe_exec xc = detail::to_c(x);
  detail::check(pfe_project_orthogonal(static_cast<int32_t>(a.rows()), static_cast<int32_t>(a.cols()), a.data(), &xc,
                                       out.data()));
  return out;
}

inline Embedding split_bregman(const CsrMatrix& m, const Vector& d_vec, const Matrix& p, const Matrix& b,
                               const PfeParams& params, const Embedding& y_init, int max_iter,
                               const IterateCallback& on_iterate = {}, const ExecOptions& x = {}) {
  WeightedGraph g = detail::graph_from_difference(m, d_vec);
  auto f = detail::flatten(g);
  const pfe_params pc = detail::to_c(params);
  const pfe_exec xc = detail::to_c(x);
  Embedding out = detail::make_matrix<Matrix>(y_init.rows(), y_init.cols());
  detail::CbCtx ctx{&on_iterate};
  detail::check(pfe_split_bregman_standalone(&f->view, p.data(), b.data(), &pc, static_cast<int32_t>(y_init.cols()),
                                             y_init.data(), max_iter, &xc, out.data(),
                                             on_iterate ? &detail::trampoline : nullptr,
                                             on_iterate ? &ctx : nullptr));
  return out;
}

inline Embedding soc(const WeightedGraph& g, const PfeParams& params, const Embedding& y0,
                     const ExecOptions& x = {}) {
  auto f = detail::flatten(g);
  const pfe_params pc = detail::to_c(params);
  const pfe_exec xc = detail::to_c(x);
  Embedding out = detail::make_matrix<Matrix>(g.n, params.dim);
  if (y0.rows() != g.n || y0.cols() != params.dim) throw ConfigError("PfeSolver: initial embedding has wrong shape");
  detail::check(pfe_solve(&f->view, &pc, &xc, 0, y0.data(), out.data(), nullptr));
  return out;
}

inline Embedding pfe_two_stage(const WeightedGraph& g, const PfeParams& params, const Embedding& y0,
                               const ExecOptions& x = {}) {
  auto f = detail::flatten(g);
  const pfe_params pc = detail::to_c(params);
  const pfe_exec xc = detail::to_c(x);
  Embedding out = detail::make_matrix<Matrix>(g.n, params.dim);
  if (y0.rows() != g.n || y0.cols() != params.dim) throw ConfigError("PfeSolver: initial embedding has wrong shape");
  detail::check(pfe_solve(&f->view, &pc, &xc, 1, y0.data(), out.data(), nullptr));
  return out;
}

// ------------------------------------------------------------------- pcg --
class PcgOperator {
 public:
  PcgOperator(CsrMatrix a, PcgConfig cfg, const ExecOptions& x = {}) : a_(std::move(a)), cfg_(cfg), x_(x) {
    if (a_.nrows != a_.ncols) throw ConfigError("PcgOperator: matrix not square");
    if (cfg_.rel_tol <= 0.0) throw ConfigError("PcgOperator: rel_tol must be > 0");
    if (cfg_.max_iter < 1) throw ConfigError("PcgOperator: max_iter must be >= 1");
    // the IC(0) breakdown test of the reference constructor (pcg.cpp:22-28),
    // so jacobi_fallback() is known before any solve
    if (cfg_.preconditioner == Preconditioner::Ic0) {
      int32_t fb = 0;
      detail::check(pfe_ic0_probe(a_.nrows, a_.row_ptr.data(), a_.col_idx.data(), a_.values.data(), &fb));
      fallback_ = fb != 0;
    }
  }

  // PcgOperator::solve (pcg.cpp:40-92): one right-hand side.
  std::pair<Vector, PcgReport> solve(const Vector& b, const Vector& x0) const {
    if (b.size() != a_.nrows || x0.size() != a_.nrows) throw ConfigError("pcg_solve: dimension mismatch");
    Matrix bm = detail::make_matrix<Matrix>(b.size(), 1), xm = detail::make_matrix<Matrix>(b.size(), 1);
    std::copy(b.data(), b.data() + b.size(), bm.data());
    std::copy(x0.data(), x0.data() + x0.size(), xm.data());
    auto res = solve_multi(bm, xm);
    Vector x(b.size());
    std::copy(res.first.data(), res.first.data() + b.size(), x.data());
    return {x, res.second[0]};
  }

  // pcg.hpp: true if IC(0) broke down and Jacobi is used instead.
  bool jacobi_fallback() const { return fallback_; }

  std::pair<Matrix, std::vector<PcgReport>> solve_multi(const Matrix& b, const Matrix& x0) const {
    if (b.rows() != a_.nrows || x0.rows() != a_.nrows || b.cols() != x0.cols())
      throw ConfigError("pcg_solve_multi: dimension mismatch");
    const int d = static_cast<int>(b.cols());
    Matrix x = detail::make_matrix<Matrix>(b.rows(), d);
    std::vector<int32_t> its(d), conv(d), fb(d);
    std::vector<double> res(d);
    const pfe_exec xc = detail::to_c(x_);
    detail::check(pfe_pcg_solve_multi(a_.nrows, a_.row_ptr.data(), a_.col_idx.data(), a_.values.data(), d, b.data(),
                                      x0.data(), cfg_.rel_tol, cfg_.max_iter,
                                      static_cast<int32_t>(cfg_.preconditioner), &xc, x.data(), its.data(),
                                      conv.data(), res.data(), fb.data()));
    std::vector<PcgReport> reps(static_cast<size_t>(d));
    for (int j = 0; j < d; ++j) reps[static_cast<size_t>(j)] = PcgReport{its[j], res[j], conv[j] != 0, fb[j] != 0};
    return {x, reps};
  }

  const CsrMatrix& matrix() const { return a_; }

 private:
  CsrMatrix a_;
  PcgConfig cfg_;
  ExecOptions x_;
  bool fallback_ = false;
};

// pcg_solve (pcg.cpp:116-121): an operator for this call, one right-hand side.
inline std::pair<Vector, PcgReport> pcg_solve(const CsrMatrix& a, const Vector& b, const Vector& x0,
                                              const PcgConfig& cfg) {
  return PcgOperator(a, cfg).solve(b, x0);
}

inline std::pair<Matrix, std::vector<PcgReport>> pcg_solve_multi(const CsrMatrix& a, const Matrix& b,
                                                                 const Matrix& x0, const PcgConfig& cfg) {
  return PcgOperator(a, cfg).solve_multi(b, x0);
}

// ------------------------------------------------ init / labels (host) ----
inline Matrix d_orthonormalize(const Matrix& a, const Vector& degrees) {
  if (a.rows() != degrees.size()) throw ConfigError("d_orthonormalize: size mismatch");
  Matrix out = detail::make_matrix<Matrix>(a.rows(), a.cols());
  detail::check(pfe_d_orthonormalize(static_cast<int32_t>(a.rows()), static_cast<int32_t>(a.cols()), a.data(),
                                     degrees.data(), out.data()));
  return out;
}

inline Matrix random_embedding(int n, int d, std::uint64_t seed, const Vector& degrees) {
  Matrix out = detail::make_matrix<Matrix>(n, d);
  detail::check(pfe_random_embedding(n, d, seed, degrees.data(), out.data()));
  return out;
}

// GMM initial embedding on the GPU (init.hpp: gmm_fit + init_embedding in
// one call; pfe_gmm_init_device).  features: n x 3 (column-major, as the
// reference's MatrixXd).  The fitted model is returned through `model`.
struct GmmModel {
  int k = 0;
  Matrix means;      // k x 3
  Matrix variances;  // k x 3, floored at 1e-6
  Vector weights;    // simplex, length k
};

inline Matrix gmm_init_embedding(const Matrix& features, int k, std::uint64_t seed, const Vector& degrees,
                                 GmmModel* model = nullptr, int device = 0) {
  const long n = features.rows();
  if (features.cols() != 3) throw ConfigError("gmm_fit: features must be n x 3");
  if (degrees.size() != n) throw ConfigError("init_embedding: degree size mismatch");
  std::vector<double> rgb(static_cast<size_t>(3 * n));
  for (long i = 0; i < n; ++i)
    for (int c = 0; c < 3; ++c) rgb[static_cast<size_t>(3 * i + c)] = features(i, c);
  Matrix out = detail::make_matrix<Matrix>(n, k > 0 ? k : 1);
  std::vector<double> means(static_cast<size_t>(3 * std::max(k, 1))), vars(means.size()),
      wts(static_cast<size_t>(std::max(k, 1)));
  detail::check(pfe_gmm_init_device(static_cast<int32_t>(n), rgb.data(), k, seed, degrees.data(), device, out.data(),
                                    means.data(), vars.data(), wts.data()));
  if (model) {
    model->k = k;
    model->means = detail::make_matrix<Matrix>(k, 3);
    model->variances = detail::make_matrix<Matrix>(k, 3);
    model->weights = Vector(static_cast<long>(k));
    for (int j = 0; j < k; ++j) {
      for (int c = 0; c < 3; ++c) {
        model->means(j, c) = means[static_cast<size_t>(3 * j + c)];
        model->variances(j, c) = vars[static_cast<size_t>(3 * j + c)];
      }
      model->weights[j] = wts[static_cast<size_t>(j)];
    }
  }
  return out;
}

struct Segmentation {
  std::vector<int> labels;
  int k = 0;
  int height = 0;
  int width = 0;
  int size() const { return static_cast<int>(labels.size()); }
};

inline Segmentation kmeans(const Matrix& points, int k, std::uint64_t seed, int max_iter = 100) {
  Segmentation s;
  s.k = k;
  std::vector<int32_t> lab(static_cast<size_t>(points.rows()));
  detail::check(pfe_kmeans(static_cast<int32_t>(points.rows()), static_cast<int32_t>(points.cols()), points.data(), k,
                           seed, max_iter, lab.data()));
  s.labels.assign(lab.begin(), lab.end());
  return s;
}

}  // namespace pfe
