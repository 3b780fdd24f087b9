// TEST: the reference's own solver API, compiled from the reference's
// headers (/root/reference/proj/core/include/pfe/*.hpp), linked against the
// link-level B200 backend (paper_1612_06496_b200/binding/pfe_core_b200.cpp)
// and libpfe_b200.so -- the combination a maintainer gets by swapping
// solver.cpp / pcg.cpp for the binding.  The calls below are
// the ones tools/main.cpp (pfe_two_stage, main.cpp:121; objective) and the
// reference tests (test_solver.cpp, test_pcg.cpp) make.
//
// usage: test_ref_binding <in.bin> <out.bin>
//   in.bin  (little-endian): int32 n, m, d, soc, sb1, sb2, pcg_max, precond;
//           f64 lambda, r, conv_tol, pcg_tol; int32 ei[m], ej[m]; f64 w[m],
//           degree[n], y0[n*d] (column-major); int32 an, annz; int32
//           aptr[an+1], aidx[annz]; f64 aval[annz], ab[an*2], ax0[an*2]
//   out.bin: f64 y_soc[n*d], y_state[n*d], y_two_stage[n*d], y_cb[n*d],
//           objective, callbacks; f64 pcg_x[an*2]; int32 pcg_iters[2];
//           f64 vec_x[an]; int32 vec_iters; int32 fallback
// Exit status: 0, or the CLI mapping of the first exception (main.cpp:431-446:
// Io 1, Numerical 2, Config 3), with "<Type>: <message>" on stdout.
#include <cstdio>
#include <cstring>
#include <fstream>
#include <iostream>
#include <string>
#include <vector>

#include "pfe/errors.hpp"
#include "pfe/graph.hpp"
#include "pfe/pcg.hpp"
#include "pfe/solver.hpp"

namespace pfe {
// graph.cpp:161-170 restated for the test (graph.cpp itself needs real
// Eigen): one row per edge, +w at column min(i,j), -w at max(i,j).
CsrMatrix difference_matrix(const WeightedGraph& g) {
  CsrMatrix m;
  m.nrows = g.edge_count();
  m.ncols = g.n;
  m.row_ptr.push_back(0);
  for (const auto& e : g.edges) {
    if (e.w != 0.0 && e.i != e.j) {
      m.col_idx.push_back(e.i < e.j ? e.i : e.j);
      m.values.push_back(e.i < e.j ? e.w : -e.w);
      m.col_idx.push_back(e.i < e.j ? e.j : e.i);
      m.values.push_back(e.i < e.j ? -e.w : e.w);
    }
    m.row_ptr.push_back(static_cast<int>(m.values.size()));
  }
  return m;
}
}  // namespace pfe

namespace {
template <class T>
void rd(std::ifstream& f, T* p, size_t n) {
  f.read(reinterpret_cast<char*>(p), static_cast<std::streamsize>(sizeof(T) * n));
  if (!f) throw pfe::IoError("short input file");
}
template <class T>
T rd1(std::ifstream& f) {
  T v{};
  rd(f, &v, 1);
  return v;
}
template <class T>
void wr(std::ofstream& f, const T* p, size_t n) {
  f.write(reinterpret_cast<const char*>(p), static_cast<std::streamsize>(sizeof(T) * n));
}

int run(const char* in_path, const char* out_path) {
  std::ifstream in(in_path, std::ios::binary);
  if (!in) throw pfe::IoError(std::string("cannot open ") + in_path);
  const int n = rd1<int32_t>(in), m = rd1<int32_t>(in), d = rd1<int32_t>(in);
  pfe::PfeParams prm;
  prm.dim = d;
  prm.soc_max = rd1<int32_t>(in);
  prm.sb_max_stage1 = rd1<int32_t>(in);
  prm.sb_max_stage2 = rd1<int32_t>(in);
  prm.pcg.max_iter = rd1<int32_t>(in);
  prm.pcg.preconditioner = static_cast<pfe::Preconditioner>(rd1<int32_t>(in));
  prm.lambda = rd1<double>(in);
  prm.r = rd1<double>(in);
  prm.conv_tol = rd1<double>(in);
  prm.pcg.rel_tol = rd1<double>(in);
  std::vector<int32_t> ei(m), ej(m);
  std::vector<double> w(m);
  rd(in, ei.data(), m);
  rd(in, ej.data(), m);
  rd(in, w.data(), m);
  pfe::WeightedGraph g;
  g.n = n;
  g.degree = Eigen::VectorXd(n);
  rd(in, g.degree.data(), n);
  for (int k = 0; k < m; ++k) g.edges.push_back({ei[k], ej[k], w[k]});
  Eigen::MatrixXd y0 = Eigen::MatrixXd::Zero(n, d);
  rd(in, y0.data(), static_cast<size_t>(n) * d);
  const int an = rd1<int32_t>(in), annz = rd1<int32_t>(in);
  pfe::CsrMatrix a;
  a.nrows = a.ncols = an;
  a.row_ptr.resize(an + 1);
  a.col_idx.resize(annz);
  a.values.resize(annz);
  rd(in, a.row_ptr.data(), an + 1);
  rd(in, a.col_idx.data(), annz);
  rd(in, a.values.data(), annz);
  Eigen::MatrixXd ab = Eigen::MatrixXd::Zero(an, 2), ax0 = Eigen::MatrixXd::Zero(an, 2);
  rd(in, ab.data(), static_cast<size_t>(an) * 2);
  rd(in, ax0.data(), static_cast<size_t>(an) * 2);

  std::ofstream out(out_path, std::ios::binary);
  const size_t nd = static_cast<size_t>(n) * d;
  // 1. the one-call soc (solver.cpp:184-189)
  pfe::PfeParams p1 = prm;
  pfe::Embedding y_soc = pfe::soc(g, p1, y0);
  wr(out, y_soc.data(), nd);
  // 2. the same through PfeSolver + SolverState (solver.cpp:60-71, 110-126)
  pfe::PfeSolver solver(g, prm);
  pfe::SolverState st = solver.make_state(y0);
  solver.run_soc(st, prm.soc_max, prm.sb_max_stage1);
  wr(out, st.y.data(), nd);
  // 3. pfe_two_stage (solver.cpp:191-193), what tools/main.cpp:121 calls
  pfe::Embedding y_ts = pfe::pfe_two_stage(g, prm, y0);
  wr(out, y_ts.data(), nd);
  // 4. split_bregman continued on the state with the iterate callback
  //    (solver.cpp:73-108, the IterateCallback slow path)
  double callbacks = 0.0;
  solver.split_bregman(st, 3, [&](int, const Eigen::MatrixXd& y) {
    if (y.rows() == n && y.cols() == d) callbacks += 1.0;
  });
  wr(out, st.y.data(), nd);
  const double obj = pfe::objective(solver.diff_matrix(), y_soc);
  wr(out, &obj, 1);
  wr(out, &callbacks, 1);
  // 5. PcgOperator (pcg.cpp:9-127)
  pfe::PcgConfig cfg{1e-10, 200, pfe::Preconditioner::Jacobi};
  auto [x, reps] = pfe::pcg_solve_multi(a, ab, ax0, cfg);
  wr(out, x.data(), static_cast<size_t>(an) * 2);
  int32_t its[2] = {reps[0].iterations, reps[1].iterations};
  wr(out, its, 2);
  Eigen::VectorXd b1(an), x01(an);
  std::memcpy(b1.data(), ab.data(), sizeof(double) * an);
  std::memcpy(x01.data(), ax0.data(), sizeof(double) * an);
  pfe::PcgOperator op(a, cfg);
  auto [xv, rv] = op.solve(b1, x01);
  wr(out, xv.data(), static_cast<size_t>(an));
  int32_t vi = rv.iterations;
  wr(out, &vi, 1);
  pfe::PcgOperator op_ic(a, pfe::PcgConfig{});
  int32_t fb = op_ic.jacobi_fallback() ? 1 : 0;
  wr(out, &fb, 1);
  // 6. the reference's precondition errors surface as its exception types
  pfe::PfeParams bad = prm;
  bad.dim = 0;
  try {
    pfe::PfeSolver s2(g, bad);
    std::printf("no ConfigError for dim = 0\n");
    return 5;
  } catch (const pfe::ConfigError& e) {
    std::printf("expected ConfigError: %s\n", e.what());
  }
  return 0;
}
}  // namespace

int main(int argc, char** argv) {
  if (argc != 3) {
    std::fprintf(stderr, "usage: %s in.bin out.bin\n", argv[0]);
    return 64;
  }
  try {
    return run(argv[1], argv[2]);
  } catch (const pfe::IoError& e) {
    std::printf("IoError: %s\n", e.what());
    return 1;
  } catch (const pfe::NumericalError& e) {
    std::printf("NumericalError: %s\n", e.what());
    return 2;
  } catch (const pfe::ConfigError& e) {
    std::printf("ConfigError: %s\n", e.what());
    return 3;
  }
}
