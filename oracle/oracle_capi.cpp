// TEST INFRASTRUCTURE ONLY — flat C entry points over the oracle so that
// tests/ and bench.py (cpu_baseline / --impl reference) can drive it through
// ctypes.  Status codes follow proj/tools/main.cpp:431-446:
// 0 ok, 1 IoError, 2 NumericalError, 3 ConfigError, 4 other.
// Dense matrices are column-major (the reference's Eigen layout).
#include <chrono>
#include <cstring>
#include <string>

#include "pfe_oracle.hpp"

using namespace orc;

namespace {
thread_local std::string g_err;

template <class F>
int guard(F&& f) {
  try {
    f();
    return 0;
  } catch (const IoError& e) {
    g_err = e.what();
    return 1;
  } catch (const NumericalError& e) {
    g_err = e.what();
    return 2;
  } catch (const ConfigError& e) {
    g_err = e.what();
    return 3;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 4;
  }
}

Graph make_graph(int n, int m, const int* ei, const int* ej, const double* w, const double* deg) {
  Graph g;
  g.n = n;
  g.ei.assign(ei, ei + m);
  g.ej.assign(ej, ej + m);
  g.w.assign(w, w + m);
  if (deg)
    g.degree.assign(deg, deg + n);
  else
    g.degree = degree_vector(g);
  return g;
}

Mat make_mat(long r, long c, const double* a) {
  Mat m(r, c);
  if (a) std::memcpy(m.a.data(), a, sizeof(double) * static_cast<size_t>(r * c));
  return m;
}

void put(const Mat& m, double* out) {
  if (out) std::memcpy(out, m.a.data(), sizeof(double) * m.a.size());
}
}  // namespace

extern "C" {

// Mirrors the field order of pfe_params in include/pfe_b200.h (its own copy:
// the oracle does not include product headers).
struct orc_params {
  int dim;
  double lambda;
  double r;
  int soc_max;
  int sb_max_stage1;
  int sb_max_stage2;
  double conv_tol;
  double pcg_rel_tol;
  int pcg_max_iter;
  int preconditioner;  // 0 Ic0, 1 Jacobi, 2 None
};

int orc_solve_timed(int mode, int n, int m, const int* ei, const int* ej, const double* w, const double* deg,
                    const orc_params* prm, const double* y0, double* y_out, double* p_out, double* breg_out,
                    double* sb_out, double* ss_out, int* pcg_log, int log_cap, long* n_inner, double* times);

static Params to_params(const orc_params* p) {
  Params q;
  q.dim = p->dim;
  q.lambda = p->lambda;
  q.r = p->r;
  q.soc_max = p->soc_max;
  q.sb_max_stage1 = p->sb_max_stage1;
  q.sb_max_stage2 = p->sb_max_stage2;
  q.conv_tol = p->conv_tol;
  q.pcg.rel_tol = p->pcg_rel_tol;
  q.pcg.max_iter = p->pcg_max_iter;
  q.pcg.prec = p->preconditioner;
  return q;
}

const char* orc_last_error(void) { return g_err.c_str(); }
void orc_set_threads(int t) { set_threads(t); }

int orc_random_embedding(int n, int d, unsigned long long seed, const double* deg, double* out) {
  return guard([&] { put(random_embedding(n, d, seed, Vec(deg, deg + n)), out); });
}

int orc_d_orthonormalize(int n, int d, const double* a, const double* deg, double* out) {
  return guard([&] { put(d_orthonormalize(make_mat(n, d, a), Vec(deg, deg + n)), out); });
}

// mode 0: soc (solver.cpp:184-189); mode 1: pfe_two_stage / two_stage
// (solver.cpp:128-136, 191-193).  Optional outputs may be null.  pcg_log
// (capacity log_cap) receives the per-inner max-over-columns PCG iteration
// counts; *n_inner the number of inner iterations run.
int orc_solve(int mode, int n, int m, const int* ei, const int* ej, const double* w, const double* deg,
              const orc_params* prm, const double* y0, double* y_out, double* p_out, double* breg_out,
              double* sb_out, double* ss_out, int* pcg_log, int log_cap, long* n_inner) {
  return orc_solve_timed(mode, n, m, ei, ej, w, deg, prm, y0, y_out, p_out, breg_out, sb_out, ss_out, pcg_log,
                         log_cap, n_inner, nullptr);
}

// orc_solve plus wall seconds {set-up, inner iterations, projections} in
// times[0..2] (bench.py's CPU baseline times the inner loop only).
int orc_solve_timed(int mode, int n, int m, const int* ei, const int* ej, const double* w, const double* deg,
                    const orc_params* prm, const double* y0, double* y_out, double* p_out, double* breg_out,
                    double* sb_out, double* ss_out, int* pcg_log, int log_cap, long* n_inner, double* times) {
  return guard([&] {
    Graph g = make_graph(n, m, ei, ej, w, deg);
    Params params = to_params(prm);
    RunLog log;
    const auto t0 = std::chrono::steady_clock::now();
    PfeSolver s(g, params);
    s.log = &log;
    State st = s.make_state(make_mat(n, params.dim, y0));
    log.t_setup = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    s.run_soc(st, params.soc_max, params.sb_max_stage1);
    if (mode == 1 && params.sb_max_stage2 > 0) s.split_bregman(st, params.sb_max_stage2);
    put(st.y, y_out);
    put(st.p, p_out);
    put(st.bregman, breg_out);
    put(st.split_b, sb_out);
    put(st.split_s, ss_out);
    if (pcg_log)
      for (int i = 0; i < log_cap && i < static_cast<int>(log.pcg_iters.size()); ++i) pcg_log[i] = log.pcg_iters[i];
    if (n_inner) *n_inner = log.inner_iterations;
    if (times) {
      times[0] = log.t_setup;
      times[1] = log.t_inner;
      times[2] = log.t_outer;
    }
  });
}

// A resident oracle solve for bench.py's CPU legs: the solver and state are
// built once (orc_session_create, set-up seconds reported), then each
// orc_session_step runs the next `inner` inner iterations of the soc
// schedule (solver.cpp:110-126: b = s = 0 at the start of an outer
// iteration, the projection after its sb_max-th inner iteration), so a
// bounded sample of steps walks the same trajectory the full run does.
struct orc_session {
  PfeSolver solver;
  State st;
  RunLog log;
  int sb_max = 1;
  long pos = 0;  // inner iterations run so far
  orc_session(const Graph& g, const Params& p) : solver(g, p), sb_max(p.sb_max_stage1) {}
};

int orc_session_create(int n, int m, const int* ei, const int* ej, const double* w, const double* deg,
                       const orc_params* prm, const double* y0, orc_session** out, double* setup_s) {
  return guard([&] {
    Graph g = make_graph(n, m, ei, ej, w, deg);
    Params params = to_params(prm);
    const auto t0 = std::chrono::steady_clock::now();
    auto* ss = new orc_session(g, params);
    ss->solver.log = &ss->log;
    try {
      ss->st = ss->solver.make_state(make_mat(n, params.dim, y0));
    } catch (...) {
      delete ss;
      throw;
    }
    if (setup_s) *setup_s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    *out = ss;
  });
}

// times[0] = inner-iteration seconds, times[1] = projection seconds of this
// call; pcg_max[i] = PCG iterations (max over columns) of its i-th inner iteration.
int orc_session_step(orc_session* ss, int inner, double* times, int* pcg_max) {
  return guard([&] {
    const double ti = ss->log.t_inner, to = ss->log.t_outer;
    const size_t before = ss->log.pcg_iters.size();
    for (int k = 0; k < inner; ++k) {
      if (ss->pos % ss->sb_max == 0) {
        std::fill(ss->st.split_b.a.begin(), ss->st.split_b.a.end(), 0.0);
        std::fill(ss->st.split_s.a.begin(), ss->st.split_s.a.end(), 0.0);
      }
      ss->solver.split_bregman(ss->st, 1);
      ++ss->pos;
      if (ss->pos % ss->sb_max == 0) ss->solver.outer_update(ss->st);
    }
    if (times) {
      times[0] = ss->log.t_inner - ti;
      times[1] = ss->log.t_outer - to;
    }
    if (pcg_max)
      for (size_t i = before; i < ss->log.pcg_iters.size(); ++i) pcg_max[i - before] = ss->log.pcg_iters[i];
  });
}

void orc_session_destroy(orc_session* ss) { delete ss; }

// PfeSolver::split_bregman on a caller-supplied state (solver.cpp:73-108);
// state arrays are updated in place.  traj (max_iter*n*d, may be null)
// receives Y after each inner iteration (the IterateCallback slow path).
int orc_state_split_bregman(int n, int m, const int* ei, const int* ej, const double* w, const double* deg,
                            const orc_params* prm, int max_iter, double* y, double* p, double* breg, double* sb,
                            double* ss, double* traj, int* n_traj) {
  return guard([&] {
    Graph g = make_graph(n, m, ei, ej, w, deg);
    Params params = to_params(prm);
    PfeSolver s(g, params);
    const int d = params.dim;
    State st;
    st.y = make_mat(n, d, y);
    st.p = make_mat(n, d, p);
    st.bregman = make_mat(n, d, breg);
    st.split_b = make_mat(m, d, sb);
    st.split_s = make_mat(m, d, ss);
    int cnt = 0;
    s.split_bregman(st, max_iter, [&](int, const Mat& yy) {
      if (traj) std::memcpy(traj + static_cast<size_t>(cnt) * n * d, yy.a.data(), sizeof(double) * yy.a.size());
      ++cnt;
    });
    if (n_traj) *n_traj = cnt;
    put(st.y, y);
    put(st.p, p);
    put(st.bregman, breg);
    put(st.split_b, sb);
    put(st.split_s, ss);
  });
}

// Standalone split_bregman (solver.cpp:138-182) with M = difference_matrix(g).
int orc_split_bregman(int n, int m, const int* ei, const int* ej, const double* w, const double* d_vec,
                      const double* p, const double* b, const orc_params* prm, int d, const double* y_init,
                      int max_iter, double* y_out, double* traj, int* n_traj) {
  return guard([&] {
    Graph g = make_graph(n, m, ei, ej, w, d_vec);
    Csr mm = difference_matrix(g);
    Params params = to_params(prm);
    int cnt = 0;
    Mat y = split_bregman(mm, g.degree, make_mat(n, d, p), make_mat(n, d, b), params, make_mat(n, d, y_init),
                          max_iter, [&](int, const Mat& yy) {
                            if (traj)
                              std::memcpy(traj + static_cast<size_t>(cnt) * n * d, yy.a.data(),
                                          sizeof(double) * yy.a.size());
                            ++cnt;
                          });
    if (n_traj) *n_traj = cnt;
    put(y, y_out);
  });
}

// A = form_normal_matrix(difference_matrix(g), deg, lambda, r) as CSR.
// Call with vals == null to get *nnz, then again with buffers.
int orc_normal_matrix(int n, int m, const int* ei, const int* ej, const double* w, const double* deg,
                      double lambda, double r, int* nnz, int* ptr, int* idx, double* vals) {
  return guard([&] {
    Graph g = make_graph(n, m, ei, ej, w, deg);
    Csr a = form_normal_matrix(difference_matrix(g), g.degree, lambda, r);
    *nnz = a.nnz();
    if (!vals) return;
    std::memcpy(ptr, a.ptr.data(), sizeof(int) * a.ptr.size());
    std::memcpy(idx, a.idx.data(), sizeof(int) * a.idx.size());
    std::memcpy(vals, a.val.data(), sizeof(double) * a.val.size());
  });
}

// PcgOperator::solve_multi (pcg.cpp:94-114) on a caller CSR matrix.
int orc_pcg_solve_multi(int n, const int* ptr, const int* idx, const double* vals, int d, const double* b,
                        const double* x0, double rel_tol, int max_iter, int prec, double* x_out, int* iters,
                        int* converged, double* resid) {
  return guard([&] {
    Csr a;
    a.nrows = a.ncols = n;
    a.ptr.assign(ptr, ptr + n + 1);
    a.idx.assign(idx, idx + ptr[n]);
    a.val.assign(vals, vals + ptr[n]);
    PcgConfig cfg{rel_tol, max_iter, prec};
    PcgOperator op(std::move(a), cfg);
    Mat x;
    std::vector<PcgReport> reps = op.solve_multi(make_mat(n, d, b), make_mat(n, d, x0), x);
    put(x, x_out);
    for (int j = 0; j < d; ++j) {
      if (iters) iters[j] = reps[j].iterations;
      if (converged) converged[j] = reps[j].converged ? 1 : 0;
      if (resid) resid[j] = reps[j].final_rel_residual;
    }
  });
}

int orc_project_orthogonal(int n, int d, const double* a, double* p_out) {
  return guard([&] { put(project_orthogonal(make_mat(n, d, a)), p_out); });
}

int orc_shrink(long count, const double* v, double gamma, double* out) {
  return guard([&] { put(shrink(make_mat(count, 1, v), gamma), out); });
}

int orc_objective(int n, int m, const int* ei, const int* ej, const double* w, int d, const double* y,
                  double* out) {
  return guard([&] {
    Graph g = make_graph(n, m, ei, ej, w, nullptr);
    *out = objective(difference_matrix(g), make_mat(n, d, y));
  });
}

int orc_kmeans(int n, int d, const double* pts, int k, unsigned long long seed, int max_iter, int* labels) {
  return guard([&] {
    std::vector<int> l = kmeans(make_mat(n, d, pts), k, seed, max_iter);
    std::memcpy(labels, l.data(), sizeof(int) * l.size());
  });
}

int orc_covering(int n, const int* pred, const int* gt, double* out) {
  return guard([&] { *out = covering(std::vector<int>(pred, pred + n), std::vector<int>(gt, gt + n)); });
}

// 4-neighbour image graph (graph.cpp:105-159).  rgb row-major n x 3.  sigma
// <= 0 selects median_neighbor_distance.  Call with ei == null for *m.
int orc_build_image_graph(int h, int w, const double* rgb, double sigma, int* m, int* ei, int* ej, double* wt,
                          double* deg, double* sigma_out) {
  return guard([&] {
    std::vector<double> f(rgb, rgb + static_cast<size_t>(h) * w * 3);
    const double s = sigma > 0.0 ? sigma : median_neighbor_distance(h, w, f);
    Graph g = build_image_graph(h, w, f, s);
    *m = g.m();
    if (sigma_out) *sigma_out = s;
    if (!ei) return;
    std::memcpy(ei, g.ei.data(), sizeof(int) * g.ei.size());
    std::memcpy(ej, g.ej.data(), sizeof(int) * g.ej.size());
    std::memcpy(wt, g.w.data(), sizeof(double) * g.w.size());
    std::memcpy(deg, g.degree.data(), sizeof(double) * g.degree.size());
  });
}

// GMM init (init.cpp:45-170) for an n x 3 row-major feature image.
int orc_gmm_init_embedding(int n, const double* rgb, int k, unsigned long long seed, const double* deg,
                           double* out) {
  return guard([&] {
    Mat f(n, 3);
    for (int v = 0; v < n; ++v)
      for (int c = 0; c < 3; ++c) f(v, c) = rgb[3 * v + c];
    Gmm g = gmm_fit(f, k, seed);
    put(init_embedding(g, f, Vec(deg, deg + n)), out);
  });
}

int orc_quadrant_rgb(int size, double noise, unsigned long long seed, double* out) {
  return guard([&] {
    std::vector<double> v = quadrant_rgb(size, noise, seed);
    std::memcpy(out, v.data(), sizeof(double) * v.size());
  });
}

// out = {obj0, obj1, covering, seconds, inner_iterations}
int orc_golden_quadrant(int size, double* out) {
  return guard([&] {
    GoldenResult r = run_golden_quadrant(size);
    out[0] = r.obj0;
    out[1] = r.obj1;
    out[2] = r.covering;
    out[3] = r.seconds;
    out[4] = static_cast<double>(r.inner_iterations);
  });
}

}  // extern "C"
