// Link-level B200 backend for the reference library pfe::pfe_core.
//
// This translation unit defines, against the reference's OWN headers
// (proj/core/include/pfe/{solver,pcg,graph,sparse,errors}.hpp), every
// out-of-line function that proj/core/src/solver.cpp and pcg.cpp define.  A
// maintainer builds pfe_core with this file in place of those two sources
// and links libpfe_b200.so: tools/main.cpp, graph.cpp,
// sparse.cpp, init.cpp, cluster.cpp, imgio.cpp and metrics.cpp compile
// unchanged, and every solver call runs the sm_100a kernels behind the C ABI
// in include/pfe_b200.h.  There is no CPU fallback: without a usable device
// the calls throw pfe::ConfigError, as the C ABI returns status 3.
//
// Only this subset of Eigen is used, so the file also compiles against the
// minimal test stub in tests/cpp/eigen_stub: MatrixXd / VectorXd (Index)
// constructors, rows(), cols(), size(), data(), operator[], MatrixXd::Zero.
//
// Replaced definitions (reference file:line):
//   objective            solver.cpp:14-17     pfe_objective
//   shrink               solver.cpp:19-25     pfe_shrink
//   project_orthogonal   solver.cpp:27-41     pfe_project_orthogonal
//   PfeSolver::PfeSolver solver.cpp:43-58     validation here; device set-up per call
//   PfeSolver::make_state solver.cpp:60-71    host (value-semantics state)
//   PfeSolver::split_bregman solver.cpp:73-108 pfe_split_bregman
//   PfeSolver::run_soc   solver.cpp:110-126   pfe_run_soc
//   PfeSolver::two_stage solver.cpp:128-136   pfe_two_stage
//   split_bregman (free) solver.cpp:138-182   pfe_split_bregman_standalone
//   soc / pfe_two_stage  solver.cpp:184-193   pfe_solve (mode 0 / 1)
//   save_embedding / load_embedding solver.cpp:195-237 (host CSV I/O, kept semantics)
//   PcgOperator::PcgOperator pcg.cpp:9-29     validation + IC(0) breakdown probe (pfe_ic0_probe)
//   PcgOperator::solve / solve_multi pcg.cpp:40-114  pfe_pcg_solve_multi
//   pcg_solve / pcg_solve_multi pcg.cpp:116-127
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <limits>
#include <sstream>
#include <string>
#include <utility>
#include <vector>

#include "pfe/errors.hpp"
#include "pfe/graph.hpp"
#include "pfe/pcg.hpp"
#include "pfe/solver.hpp"
#include "pfe/sparse.hpp"
#include "pfe_b200.h"

namespace pfe {
namespace {

// ABI status -> the reference's exception types (main.cpp:431-446 mapping).
void check(int rc) {
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
      throw std::runtime_error("pfe (B200): " + msg);
  }
}

// Execution options of this backend: device 0, CUDA graphs / persistent
// kernels on, the reference's stderr warnings on.  PFE_B200_DEVICE selects
// another ordinal.
pfe_exec exec_options() {
  pfe_exec x = pfe_exec_default();
  if (const char* d = std::getenv("PFE_B200_DEVICE")) x.device = std::atoi(d);
  x.warn = 1;
  return x;
}

pfe_params to_c(const PfeParams& p) {
  pfe_params c{};
  c.dim = p.dim;
  c.lambda = p.lambda;
  c.r = p.r;
  c.soc_max = p.soc_max;
  c.sb_max_stage1 = p.sb_max_stage1;
  c.sb_max_stage2 = p.sb_max_stage2;
  c.conv_tol = p.conv_tol;
  c.pcg_rel_tol = p.pcg.rel_tol;
  c.pcg_max_iter = p.pcg.max_iter;
  c.preconditioner = static_cast<int32_t>(p.pcg.preconditioner);
  return c;
}

// The edge list behind an edge-incidence matrix M (graph.cpp:161-170): row
// k holds +w at column i and -w at column j (i < j; columns sorted).  Rows a
// zero weight emptied (csr_from_triplets drops exact zeros) are inert in the
// reference's iteration (their b, s stay 0), so they are left out of the
// device graph and re-inserted as zero rows on the way back.
struct EdgeList {
  int n = 0;
  long rows = 0;                  // |E| = M.nrows
  std::vector<int32_t> ei, ej;
  std::vector<double> w, degree;
  std::vector<long> row_of;       // device edge -> M row
  pfe_graph view{};
};

// A pixel grid recognised from the edge pattern (every edge a forward
// neighbour of radius 1 or 2 on some width): the stencil kernels then run
// instead of the general CSR ones.  Results are identical either way (the
// C ABI verifies the hint and otherwise ignores it).
void detect_grid(EdgeList& g) {
  long maxd = 0;
  for (size_t e = 0; e < g.ei.size(); ++e) maxd = std::max<long>(maxd, g.ej[e] - g.ei[e]);
  const long cands[][2] = {{1, maxd - 1}, {1, maxd}, {2, (maxd - 2) / 2}, {2, maxd / 2}};
  for (const auto& c : cands) {
    const long R = c[0], W = c[1];
    if (W < 2 || g.n % W != 0) continue;
    bool ok = !g.ei.empty();
    for (size_t e = 0; ok && e < g.ei.size(); ++e) {
      const long yi = g.ei[e] / W, xi = g.ei[e] % W, yj = g.ej[e] / W, xj = g.ej[e] % W;
      const long dy = yj - yi, dx = xj - xi;
      ok = dy >= 0 && dy <= R && dx >= -R && dx <= R && (dy > 0 || dx > 0);
    }
    if (ok) {
      g.view.grid_h = static_cast<int32_t>(g.n / W);
      g.view.grid_w = static_cast<int32_t>(W);
      g.view.grid_radius = static_cast<int32_t>(R);
      return;
    }
  }
}

EdgeList edges_from_difference(const CsrMatrix& m, const Eigen::VectorXd& degree, const char* who) {
  EdgeList g;
  g.n = m.ncols;
  g.rows = m.nrows;
  for (int k = 0; k < m.nrows; ++k) {
    const int b = m.row_ptr[static_cast<size_t>(k)], e = m.row_ptr[static_cast<size_t>(k) + 1];
    if (e == b) continue;  // a zero-weight edge
    if (e - b != 2 || m.values[static_cast<size_t>(b)] != -m.values[static_cast<size_t>(b) + 1])
      throw ConfigError(std::string(who) + ": the B200 backend needs an edge-incidence matrix (rows [+w, -w])");
    g.ei.push_back(m.col_idx[static_cast<size_t>(b)]);
    g.ej.push_back(m.col_idx[static_cast<size_t>(b) + 1]);
    g.w.push_back(m.values[static_cast<size_t>(b)]);
    g.row_of.push_back(k);
  }
  g.degree.assign(degree.data(), degree.data() + degree.size());
  g.view = pfe_graph{g.n, static_cast<int64_t>(g.w.size()), g.ei.data(), g.ej.data(), g.w.data(), g.degree.data(),
                     0, 0, 0};
  detect_grid(g);
  return g;
}

Eigen::MatrixXd zeros(long rows, long cols) { return Eigen::MatrixXd::Zero(rows, cols); }

// |E| x d column-major (M rows) <-> compacted device edge order
std::vector<double> compact_rows(const EdgeList& g, const Eigen::MatrixXd& a) {
  const long me = static_cast<long>(g.row_of.size()), d = a.cols();
  std::vector<double> out(static_cast<size_t>(me * d));
  for (long j = 0; j < d; ++j)
    for (long e = 0; e < me; ++e) out[static_cast<size_t>(e + j * me)] = a.data()[g.row_of[e] + j * g.rows];
  return out;
}
void expand_rows(const EdgeList& g, const std::vector<double>& c, Eigen::MatrixXd& a, long d) {
  const long me = static_cast<long>(g.row_of.size());
  a = zeros(g.rows, d);
  for (long j = 0; j < d; ++j)
    for (long e = 0; e < me; ++e) a.data()[g.row_of[e] + j * g.rows] = c[static_cast<size_t>(e + j * me)];
}

// RAII over the C handles.
struct Solver {
  pfe_solver* s = nullptr;
  ~Solver() { pfe_solver_destroy(s); }
};
struct State {
  pfe_state* s = nullptr;
  ~State() { pfe_state_destroy(s); }
};

struct CallbackCtx {
  const IterateCallback* cb;
};
void trampoline(int it, const double* y, int32_t n, int32_t d, void* user) {
  auto* ctx = static_cast<CallbackCtx*>(user);
  Eigen::MatrixXd yy = zeros(n, d);
  std::memcpy(yy.data(), y, sizeof(double) * static_cast<size_t>(n) * d);
  (*ctx->cb)(it, yy);
}

// Device solver + a device state loaded from a host SolverState.
void load_state(const EdgeList& g, pfe_solver* s, const SolverState& st, State& ds) {
  check(pfe_state_create(s, st.y.data(), &ds.s));
  check(pfe_state_set(ds.s, PFE_FIELD_P, st.p.data()));
  check(pfe_state_set(ds.s, PFE_FIELD_BREGMAN, st.bregman.data()));
  check(pfe_state_set(ds.s, PFE_FIELD_SPLIT_B, compact_rows(g, st.split_b).data()));
  check(pfe_state_set(ds.s, PFE_FIELD_SPLIT_S, compact_rows(g, st.split_s).data()));
}
void store_state(const EdgeList& g, const State& ds, SolverState& st, long d) {
  const long me = static_cast<long>(g.row_of.size());
  check(pfe_state_get(ds.s, PFE_FIELD_Y, st.y.data()));
  check(pfe_state_get(ds.s, PFE_FIELD_P, st.p.data()));
  check(pfe_state_get(ds.s, PFE_FIELD_BREGMAN, st.bregman.data()));
  std::vector<double> c(static_cast<size_t>(me * d));
  check(pfe_state_get(ds.s, PFE_FIELD_SPLIT_B, c.data()));
  expand_rows(g, c, st.split_b, d);
  check(pfe_state_get(ds.s, PFE_FIELD_SPLIT_S, c.data()));
  expand_rows(g, c, st.split_s, d);
}

void check_state_shape(const SolverState& st, long n, long e, long d) {
  if (st.y.rows() != n || st.y.cols() != d || st.p.rows() != n || st.p.cols() != d || st.bregman.rows() != n ||
      st.bregman.cols() != d || st.split_b.rows() != e || st.split_b.cols() != d || st.split_s.rows() != e ||
      st.split_s.cols() != d)
    throw ConfigError("PfeSolver: state has wrong shape");
}

// The checks form_normal_matrix makes on its inputs (sparse.cpp:96-106): the
// reference constructor reaches them before PcgOperator's and its own.
CsrMatrix normal_matrix_checks(const CsrMatrix& m, const Eigen::VectorXd& degrees, double lambda, double r) {
  if (degrees.size() != m.ncols) throw ConfigError("form_normal_matrix: degree size mismatch");
  if (lambda < 0.0) throw ConfigError("form_normal_matrix: lambda must be >= 0");
  if (r <= 0.0) throw ConfigError("form_normal_matrix: r must be > 0");
  for (long i = 0; i < degrees.size(); ++i)
    if (degrees[i] <= 0.0)
      throw ConfigError("form_normal_matrix: nonpositive degree at vertex " + std::to_string(i) +
                        " (isolated vertex)");
  CsrMatrix empty;  // A is formed on the device (pfe_solver_create)
  return empty;
}

}  // namespace

// ------------------------------------------------------------ solver.cpp --
double objective(const CsrMatrix& m, const Embedding& y) {
  if (y.rows() != m.ncols) throw ConfigError("objective: dimension mismatch");
  Eigen::VectorXd ones(m.ncols);
  for (long i = 0; i < ones.size(); ++i) ones[i] = 1.0;
  EdgeList g = edges_from_difference(m, ones, "objective");
  const pfe_exec x = exec_options();
  double out = 0.0;
  check(pfe_objective(&g.view, static_cast<int32_t>(y.cols()), y.data(), &x, &out));
  return out;
}

Eigen::MatrixXd shrink(const Eigen::MatrixXd& v, double gamma) {
  if (gamma < 0.0) throw ConfigError("shrink: gamma must be >= 0");
  Eigen::MatrixXd out = zeros(v.rows(), v.cols());
  const pfe_exec x = exec_options();
  check(pfe_shrink(static_cast<int64_t>(v.rows()) * v.cols(), v.data(), gamma, &x, out.data()));
  return out;
}

Eigen::MatrixXd project_orthogonal(const Eigen::MatrixXd& a) {
  if (a.rows() < a.cols()) throw ConfigError("project_orthogonal: need rows >= cols");
  Eigen::MatrixXd out = zeros(a.rows(), a.cols());
  const pfe_exec x = exec_options();
  check(pfe_project_orthogonal(static_cast<int32_t>(a.rows()), static_cast<int32_t>(a.cols()), a.data(), &x,
                               out.data()));
  return out;
}

// The solver keeps the reference's members and value semantics; M (m_) and
// the degrees are the graph the device solver is built from on each call
// (the class has no destructor hook to own a device handle).  mt_ is not
// needed on this path and stays empty.
PfeSolver::PfeSolver(const WeightedGraph& g, const PfeParams& params)
    : params_(params),
      n_(g.n),
      m_(difference_matrix(g)),
      mt_(),
      degree_(g.degree),
      sqrt_degree_(g.degree.size()),
      op_(normal_matrix_checks(m_, g.degree, params.lambda, params.r), params.pcg) {
  for (long i = 0; i < degree_.size(); ++i) sqrt_degree_[i] = std::sqrt(degree_[i]);
  if (params.dim < 1) throw ConfigError("PfeSolver: dim must be >= 1");
  if (params.lambda <= 0.0 || params.r <= 0.0) throw ConfigError("PfeSolver: lambda and r must be > 0");
  if (params.soc_max < 1 || params.sb_max_stage1 < 1) throw ConfigError("PfeSolver: iteration caps must be >= 1");
}

SolverState PfeSolver::make_state(const Embedding& y0) const {
  if (y0.rows() != n_ || y0.cols() != params_.dim) throw ConfigError("PfeSolver: initial embedding has wrong shape");
  const long n = n_, d = params_.dim;
  SolverState st;
  st.y = y0;
  st.p = zeros(n, d);
  for (long j = 0; j < d; ++j)
    for (long i = 0; i < n; ++i) st.p.data()[i + j * n] = sqrt_degree_[i] * y0.data()[i + j * n];
  st.bregman = zeros(n, d);
  st.split_b = zeros(m_.nrows, d);
  st.split_s = zeros(m_.nrows, d);
  return st;
}

void PfeSolver::split_bregman(SolverState& state, int max_iter, const IterateCallback& on_iterate) const {
  check_state_shape(state, n_, m_.nrows, params_.dim);
  EdgeList g = edges_from_difference(m_, degree_, "PfeSolver");
  const pfe_params pc = to_c(params_);
  const pfe_exec x = exec_options();
  Solver s;
  check(pfe_solver_create(&g.view, &pc, &x, &s.s));
  State ds;
  load_state(g, s.s, state, ds);
  CallbackCtx ctx{&on_iterate};
  check(pfe_split_bregman(s.s, ds.s, max_iter, on_iterate ? &trampoline : nullptr, on_iterate ? &ctx : nullptr));
  store_state(g, ds, state, params_.dim);
}

void PfeSolver::run_soc(SolverState& state, int soc_max, int sb_max) const {
  check_state_shape(state, n_, m_.nrows, params_.dim);
  EdgeList g = edges_from_difference(m_, degree_, "PfeSolver");
  const pfe_params pc = to_c(params_);
  const pfe_exec x = exec_options();
  Solver s;
  check(pfe_solver_create(&g.view, &pc, &x, &s.s));
  State ds;
  load_state(g, s.s, state, ds);
  check(pfe_run_soc(s.s, ds.s, soc_max, sb_max));
  store_state(g, ds, state, params_.dim);
}

SolverState PfeSolver::two_stage(const Embedding& y0) const {
  SolverState st = make_state(y0);
  EdgeList g = edges_from_difference(m_, degree_, "PfeSolver");
  const pfe_params pc = to_c(params_);
  const pfe_exec x = exec_options();
  Solver s;
  check(pfe_solver_create(&g.view, &pc, &x, &s.s));
  State ds;
  check(pfe_state_create(s.s, y0.data(), &ds.s));
  check(pfe_two_stage(s.s, ds.s));
  store_state(g, ds, st, params_.dim);
  return st;
}

Embedding split_bregman(const CsrMatrix& m, const Eigen::VectorXd& d_vec, const Eigen::MatrixXd& p,
                        const Eigen::MatrixXd& b, const PfeParams& params, const Embedding& y_init, int max_iter,
                        const IterateCallback& on_iterate) {
  EdgeList g = edges_from_difference(m, d_vec, "split_bregman");
  const pfe_params pc = to_c(params);
  const pfe_exec x = exec_options();
  const long n = y_init.rows(), d = y_init.cols();
  if (p.rows() != n || p.cols() != d || b.rows() != n || b.cols() != d || d_vec.size() != m.ncols ||
      n != m.ncols)
    throw ConfigError("split_bregman: dimension mismatch");
  Embedding out = zeros(n, d);
  CallbackCtx ctx{&on_iterate};
  check(pfe_split_bregman_standalone(&g.view, p.data(), b.data(), &pc, static_cast<int32_t>(d), y_init.data(),
                                     max_iter, &x, out.data(), on_iterate ? &trampoline : nullptr,
                                     on_iterate ? &ctx : nullptr));
  return out;
}

namespace {
Embedding solve_one_call(const WeightedGraph& wg, const PfeParams& params, const Embedding& y0, int mode) {
  PfeSolver check_args(wg, params);  // the reference's constructor checks, in its order
  if (y0.rows() != wg.n || y0.cols() != params.dim)
    throw ConfigError("PfeSolver: initial embedding has wrong shape");
  EdgeList g = edges_from_difference(check_args.diff_matrix(), wg.degree, "PfeSolver");
  const pfe_params pc = to_c(params);
  const pfe_exec x = exec_options();
  Embedding out = zeros(wg.n, params.dim);
  check(pfe_solve(&g.view, &pc, &x, mode, y0.data(), out.data(), nullptr));
  return out;
}
}  // namespace

Embedding soc(const WeightedGraph& g, const PfeParams& params, const Embedding& y0) {
  return solve_one_call(g, params, y0, 0);
}

Embedding pfe_two_stage(const WeightedGraph& g, const PfeParams& params, const Embedding& y0) {
  return solve_one_call(g, params, y0, 1);
}

// Embedding CSV (host file format; the semantics of solver.cpp:195-237).
void save_embedding(const Embedding& y, const std::string& path) {
  std::ofstream out(path);
  if (!out) throw IoError("save_embedding: cannot open " + path);
  out << y.rows() << " " << y.cols() << "\n";
  out.precision(17);
  for (long i = 0; i < y.rows(); ++i) {
    for (long j = 0; j < y.cols(); ++j) {
      if (j) out << ",";
      out << y.data()[i + j * y.rows()];
    }
    out << "\n";
  }
  if (!out) throw IoError("save_embedding: write failed for " + path);
}

Embedding load_embedding(const std::string& path) {
  std::ifstream in(path);
  if (!in) throw IoError("load_embedding: cannot open " + path);
  long n = 0, d = 0;
  if (!(in >> n >> d) || n < 1 || d < 1) throw IoError("load_embedding: bad header in " + path);
  Embedding y = zeros(n, d);
  std::string line;
  std::getline(in, line);
  for (long i = 0; i < n; ++i) {
    if (!std::getline(in, line)) throw IoError("load_embedding: truncated file " + path);
    std::istringstream is(line);
    std::string cell;
    for (long j = 0; j < d; ++j) {
      if (!std::getline(is, cell, ',')) throw IoError("load_embedding: short row " + std::to_string(i) + " in " + path);
      y.data()[i + j * n] = std::stod(cell);
    }
  }
  return y;
}

// --------------------------------------------------------------- pcg.cpp --
// The operator keeps the reference's members: A (solved on the device per
// call), the config, the Jacobi inverse diagonal and the IC(0) breakdown
// flag, probed at construction like the reference's factorization
// (pcg.cpp:22-28) so jacobi_fallback() is known before any solve.
PcgOperator::PcgOperator(CsrMatrix a, PcgConfig cfg) : a_(std::move(a)), cfg_(cfg) {
  if (a_.nrows != a_.ncols) throw ConfigError("PcgOperator: matrix not square");
  if (cfg_.rel_tol <= 0.0) throw ConfigError("PcgOperator: rel_tol must be > 0");
  if (cfg_.max_iter < 1) throw ConfigError("PcgOperator: max_iter must be >= 1");
  if (cfg_.preconditioner == Preconditioner::Ic0 && a_.nrows > 0) {
    int32_t fb = 0;
    check(pfe_ic0_probe(a_.nrows, a_.row_ptr.data(), a_.col_idx.data(), a_.values.data(), &fb));
    fallback_ = fb != 0;
  }
}

std::pair<Eigen::MatrixXd, std::vector<PcgReport>> PcgOperator::solve_multi(const Eigen::MatrixXd& b,
                                                                            const Eigen::MatrixXd& x0) const {
  if (b.rows() != a_.nrows || x0.rows() != a_.nrows || b.cols() != x0.cols())
    throw ConfigError("pcg_solve_multi: dimension mismatch");
  const int32_t d = static_cast<int32_t>(b.cols());
  Eigen::MatrixXd x = zeros(b.rows(), d);
  std::vector<PcgReport> reps(static_cast<size_t>(d));
  if (d == 0) return {x, reps};
  std::vector<int32_t> its(static_cast<size_t>(d)), conv(static_cast<size_t>(d)), fb(static_cast<size_t>(d));
  std::vector<double> res(static_cast<size_t>(d));
  const pfe_exec xo = exec_options();
  check(pfe_pcg_solve_multi(a_.nrows, a_.row_ptr.data(), a_.col_idx.data(), a_.values.data(), d, b.data(), x0.data(),
                            cfg_.rel_tol, cfg_.max_iter, static_cast<int32_t>(cfg_.preconditioner), &xo, x.data(),
                            its.data(), conv.data(), res.data(), fb.data()));
  for (int32_t j = 0; j < d; ++j) {
    PcgReport& r = reps[static_cast<size_t>(j)];
    r.iterations = its[static_cast<size_t>(j)];
    r.final_rel_residual = res[static_cast<size_t>(j)];
    r.converged = conv[static_cast<size_t>(j)] != 0;
    r.jacobi_fallback = fb[static_cast<size_t>(j)] != 0;
  }
  return {x, reps};
}

// solve (pcg.cpp:40-92) is solve_multi on one column; its NumericalError
// (curvature breakdown, NaN) is raised to the caller as the reference does,
// where solve_multi swallows it into the column's report (pcg.cpp:106-111).
std::pair<Eigen::VectorXd, PcgReport> PcgOperator::solve(const Eigen::VectorXd& b, const Eigen::VectorXd& x0) const {
  if (b.size() != a_.nrows || x0.size() != a_.nrows) throw ConfigError("pcg_solve: dimension mismatch");
  Eigen::MatrixXd bm = zeros(b.size(), 1), xm = zeros(b.size(), 1);
  std::memcpy(bm.data(), b.data(), sizeof(double) * static_cast<size_t>(b.size()));
  std::memcpy(xm.data(), x0.data(), sizeof(double) * static_cast<size_t>(b.size()));
  auto res = solve_multi(bm, xm);
  const PcgReport& rep = res.second[0];
  if (!rep.converged && std::isinf(rep.final_rel_residual))
    throw NumericalError("pcg_solve: breakdown (indefinite or NaN curvature, or NaN in iterates)");
  Eigen::VectorXd x(b.size());
  std::memcpy(x.data(), res.first.data(), sizeof(double) * static_cast<size_t>(b.size()));
  return {x, rep};
}

std::pair<Eigen::VectorXd, PcgReport> pcg_solve(const CsrMatrix& a, const Eigen::VectorXd& b,
                                                const Eigen::VectorXd& x0, const PcgConfig& cfg) {
  return PcgOperator(a, cfg).solve(b, x0);
}

std::pair<Eigen::MatrixXd, std::vector<PcgReport>> pcg_solve_multi(const CsrMatrix& a, const Eigen::MatrixXd& b,
                                                                   const Eigen::MatrixXd& x0,
                                                                   const PcgConfig& cfg) {
  return PcgOperator(a, cfg).solve_multi(b, x0);
}

}  // namespace pfe
