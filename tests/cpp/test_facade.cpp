// C++ facade test: the reference's own unit-test cases (proj/tests/
// test_solver.cpp, test_pcg.cpp) written against include/pfe/b200.hpp, i.e.
// what a user of the reference library compiles after switching headers.
// Exit code = number of failed checks.
#include <cmath>
#include <cstdio>
#include <random>

#include "pfe/b200.hpp"

static int failures = 0;
#define CHECK(c)                                                   \
  do {                                                             \
    if (!(c)) {                                                    \
      ++failures;                                                  \
      std::printf("FAIL %s:%d: %s\n", __FILE__, __LINE__, #c);     \
    }                                                              \
  } while (0)

template <class E, class F>
bool throws(F&& f) {
  try {
    f();
  } catch (const E&) {
    return true;
  } catch (...) {
    return false;
  }
  return false;
}

static pfe::WeightedGraph chain_graph(int n, std::mt19937_64& rng) {
  std::uniform_real_distribution<double> w(0.1, 2.0);
  pfe::WeightedGraph g;
  g.n = n;
  for (int i = 0; i + 1 < n; ++i) g.edges.push_back({i, i + 1, w(rng)});
  for (int i = 0; i + 3 < n; i += 2) g.edges.push_back({i, i + 3, w(rng)});
  std::sort(g.edges.begin(), g.edges.end(),
            [](const auto& a, const auto& b) { return a.i != b.i ? a.i < b.i : a.j < b.j; });
  g.degree = pfe::degree_vector(g);
  return g;
}

int main() {
  // shrink known answers (test_solver.cpp:30-35)
  {
    pfe::Matrix v(2, 1);
    v(0, 0) = 2.5;
    v(1, 0) = -0.5;
    pfe::Matrix s = pfe::shrink(v, 1.0);
    CHECK(s(0, 0) == 1.5);
    CHECK(s(1, 0) == 0.0);
    CHECK(throws<pfe::ConfigError>([&] { pfe::shrink(v, -1.0); }));
  }
  // objective single edge (test_solver.cpp:98-106)
  {
    pfe::WeightedGraph g;
    g.n = 2;
    g.edges = {{0, 1, 2.0}};
    g.degree = pfe::degree_vector(g);
    pfe::Matrix y(2, 1);
    y(0, 0) = 0.0;
    y(1, 0) = 1.0;
    CHECK(pfe::objective(pfe::difference_matrix(g), y) == 2.0);
  }
  // projection removes scaling, rank deficiency throws (test_solver.cpp:65-87)
  {
    pfe::Matrix a(6, 3);
    for (int k = 0; k < 3; ++k) a(k, k) = 2.0;
    pfe::Matrix p = pfe::project_orthogonal(a);
    double dev = 0.0;
    for (int i = 0; i < 6; ++i)
      for (int j = 0; j < 3; ++j) dev = std::max(dev, std::abs(p(i, j) - (i == j ? 1.0 : 0.0)));
    CHECK(dev < 1e-12);
    pfe::Matrix r(4, 2);
    for (int i = 0; i < 4; ++i) {
      r(i, 0) = 1.0;
      r(i, 1) = 2.0;
    }
    CHECK(throws<pfe::NumericalError>([&] { pfe::project_orthogonal(r); }));
  }
  // single edge, one iteration, hand-rolled (test_solver.cpp:194-219)
  {
    pfe::WeightedGraph g;
    g.n = 2;
    g.edges = {{0, 1, 1.0}};
    g.degree = pfe::degree_vector(g);
    const double lam = 2.0, r = 1.0;
    pfe::Matrix p(2, 1), b(2, 1), y0(2, 1);
    p(0, 0) = 1.0;
    p(1, 0) = -1.0;
    // (lam/2 + r/2) y0 - lam/2 y1 = r/2, -lam/2 y0 + (lam/2 + r/2) y1 = -r/2
    const double a11 = lam / 2 + r / 2, a12 = -lam / 2, det = a11 * a11 - a12 * a12;
    const double h0 = (a11 * (r / 2) - a12 * (-r / 2)) / det, h1 = (a11 * (-r / 2) - a12 * (r / 2)) / det;
    pfe::PfeParams prm;
    prm.dim = 1;
    prm.lambda = lam;
    prm.r = r;
    prm.conv_tol = 0.0;
    prm.pcg.rel_tol = 1e-13;
    prm.pcg.max_iter = 2000;
    std::vector<pfe::Matrix> traj;
    pfe::split_bregman(pfe::difference_matrix(g), g.degree, p, b, prm, y0, 1,
                       [&](int, const pfe::Matrix& y) { traj.push_back(y); });
    CHECK(traj.size() == 1);
    if (!traj.empty()) {
      CHECK(std::abs(traj[0](0, 0) - h0) < 1e-10);
      CHECK(std::abs(traj[0](1, 0) - h1) < 1e-10);
    }
  }
  // two-stage with stage II disabled equals soc; determinism; P^T P = I
  {
    std::mt19937_64 rng(37);
    pfe::WeightedGraph g = chain_graph(24, rng);
    pfe::PfeParams prm;
    prm.dim = 3;
    prm.soc_max = 4;
    prm.sb_max_stage1 = 3;
    prm.sb_max_stage2 = 0;
    pfe::Matrix y0 = pfe::random_embedding(g.n, 3, 1, g.degree);
    pfe::Embedding a = pfe::pfe_two_stage(g, prm, y0);
    pfe::Embedding s = pfe::soc(g, prm, y0);
    CHECK(a == s);
    pfe::PfeSolver solver(g, prm, pfe::ExecOptions{0, true, false, false, true});
    pfe::SolverState st = solver.make_state(y0);
    solver.run_soc(st, prm.soc_max, prm.sb_max_stage1);
    double dev = 0.0;
    for (int i = 0; i < 3; ++i)
      for (int j = 0; j < 3; ++j) {
        double acc = 0.0;
        for (int v = 0; v < g.n; ++v) acc += st.p(v, i) * st.p(v, j);
        dev = std::max(dev, std::abs(acc - (i == j ? 1.0 : 0.0)));
      }
    CHECK(dev < 1e-8);
    CHECK(st.y == s);
    CHECK(st.split_b.rows() == g.edge_count());
    CHECK(throws<pfe::ConfigError>([&] { solver.make_state(pfe::Matrix(g.n, 2)); }));
  }
  // PCG identity and zero rhs (test_pcg.cpp:19-39)
  {
    pfe::CsrMatrix eye;
    eye.nrows = eye.ncols = 3;
    eye.row_ptr = {0, 1, 2, 3};
    eye.col_idx = {0, 1, 2};
    eye.values = {1.0, 1.0, 1.0};
    pfe::Matrix b(3, 1), x0(3, 1);
    b(0, 0) = 0.3;
    b(1, 0) = -1.0;
    b(2, 0) = 2.0;
    pfe::PcgConfig cfg;
    cfg.preconditioner = pfe::Preconditioner::Jacobi;
    auto [x, reps] = pfe::pcg_solve_multi(eye, b, x0, cfg);
    CHECK(reps[0].converged && reps[0].iterations <= 1);
    CHECK(std::abs(x(2, 0) - 2.0) < 1e-12);
    pfe::Matrix z(3, 1);
    auto [x2, r2] = pfe::pcg_solve_multi(eye, z, b, cfg);
    CHECK(r2[0].converged && r2[0].iterations == 0 && x2(0, 0) == 0.0);
    pfe::PcgConfig bad;
    bad.rel_tol = 0.0;
    CHECK(throws<pfe::ConfigError>([&] { pfe::PcgOperator(eye, bad); }));
    // PcgOperator::solve / pcg_solve (one right-hand side, pcg.hpp:131-158)
    pfe::Vector bv(3), xv0(3);
    bv[0] = 0.3;
    bv[1] = -1.0;
    bv[2] = 2.0;
    const pfe::PcgOperator op(eye, cfg);
    auto [xs, rs] = op.solve(bv, xv0);
    CHECK(rs.converged && rs.iterations <= 1 && std::abs(xs[1] + 1.0) < 1e-12);
    auto [xf, rf] = pfe::pcg_solve(eye, bv, xv0, cfg);
    CHECK(rf.converged && std::abs(xf[0] - 0.3) < 1e-12);
    CHECK(!op.jacobi_fallback());
    // the default IC(0): the constructor's breakdown test (pcg.cpp:22-28) on
    // an SPD matrix keeps IC(0)
    pfe::PcgConfig ic;
    const pfe::PcgOperator op_ic(eye, ic);
    CHECK(!op_ic.jacobi_fallback());
    auto [xi, ri] = op_ic.solve(bv, xv0);
    CHECK(ri.converged && std::abs(xi[2] - 2.0) < 1e-12);
  }
  std::printf("%s (%d failures)\n", failures ? "FACADE TEST FAILED" : "facade test passed", failures);
  // GMM initial embedding (init.hpp: gmm_fit + init_embedding) on the GPU:
  // Y0^T D Y0 = I, weights on the simplex, variances floored
  {
    std::mt19937_64 rng(3);
    std::normal_distribution<double> nz(0.0, 0.03);
    const int n = 600;
    pfe::Matrix f(n, 3);
    pfe::Vector deg(n);
    for (int i = 0; i < n; ++i) {
      const int q = i % 3;
      for (int c = 0; c < 3; ++c) f(i, c) = (c == q ? 0.8 : 0.2) + nz(rng);
      deg[i] = 1.0 + 0.01 * (i % 7);
    }
    pfe::GmmModel model;
    pfe::Matrix y = pfe::gmm_init_embedding(f, 3, 0, deg, &model);
    double dev = 0.0;
    for (int a = 0; a < 3; ++a)
      for (int b = 0; b < 3; ++b) {
        double acc = 0.0;
        for (int i = 0; i < n; ++i) acc += y(i, a) * deg[i] * y(i, b);
        dev = std::max(dev, std::abs(acc - (a == b ? 1.0 : 0.0)));
      }
    CHECK(dev < 1e-10);
    CHECK(model.k == 3);
    double ws = 0.0;
    for (int j = 0; j < 3; ++j) {
      ws += model.weights[j];
      for (int c = 0; c < 3; ++c) CHECK(model.variances(j, c) >= 1e-6);
    }
    CHECK(std::abs(ws - 1.0) < 1e-12);
    CHECK(throws<pfe::ConfigError>([&] { pfe::gmm_init_embedding(f, 0, 0, deg); }));
  }
  return failures;
}
