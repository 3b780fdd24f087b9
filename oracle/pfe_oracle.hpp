// TEST INFRASTRUCTURE ONLY — CPU oracle for the PFE split-Bregman hot path.
//
// An Eigen-free C++ restatement of the reference solver in
// /root/reference/proj/core (Eigen3 is absent in this image, so the reference
// itself cannot be compiled).  Only tests/,
// __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference leg
// may load this code, and only as the checker.  Nothing in the product
// package links or imports it.
//
// Every routine cites the reference file:line it restates.  Loop structure,
// per-row summation order (left to right over sorted CSR rows), elementwise
// operation order and control flow follow the reference; Eigen's BLAS-1
// reductions (dot / norm / sum), whose order Eigen leaves unspecified, are
// plain sequential sums here.
//
// Parity pin: the restatement reproduces the reference's recorded end-to-end
// run (proj/test_output.txt:29-30; acceptance.cpp:310-335) — see
// oracle/golden_quadrant.cpp and tests/test_oracle_golden.py.
#pragma once

#include <cstdint>
#include <functional>
#include <stdexcept>
#include <string>
#include <vector>

namespace orc {

// errors.hpp:9-24
struct IoError : std::runtime_error {
  explicit IoError(const std::string& s) : std::runtime_error(s) {}
};
struct NumericalError : std::runtime_error {
  explicit NumericalError(const std::string& s) : std::runtime_error(s) {}
};
struct ConfigError : std::invalid_argument {
  explicit ConfigError(const std::string& s) : std::invalid_argument(s) {}
};

// Column-major dense matrix (the reference's Eigen::MatrixXd layout).
struct Mat {
  long rows = 0, cols = 0;
  std::vector<double> a;
  Mat() = default;
  Mat(long r, long c, double fill = 0.0) : rows(r), cols(c), a(static_cast<size_t>(r * c), fill) {}
  double& operator()(long i, long j) { return a[static_cast<size_t>(i + j * rows)]; }
  double operator()(long i, long j) const { return a[static_cast<size_t>(i + j * rows)]; }
  double* col(long j) { return a.data() + j * rows; }
  const double* col(long j) const { return a.data() + j * rows; }
};
using Vec = std::vector<double>;

// ---------------------------------------------------------------- sparse ----
// sparse.hpp:9-25
struct Trip {
  int row, col;
  double val;
};
struct Csr {
  int nrows = 0, ncols = 0;
  std::vector<int> ptr, idx;
  std::vector<double> val;
  int nnz() const { return static_cast<int>(val.size()); }
};

Csr csr_from_triplets(int nrows, int ncols, const std::vector<Trip>& t);  // sparse.cpp:11-50
Csr transpose(const Csr& a);                                            // sparse.cpp:52-72
Vec spmv(const Csr& a, const Vec& x);                                   // sparse.cpp:74-85
void spmv_raw(const Csr& a, const double* x, double* y);
Mat spmm_dense(const Csr& a, const Mat& x);                             // sparse.cpp:87-94
Csr form_normal_matrix(const Csr& m, const Vec& deg, double lambda, double r);  // sparse.cpp:96-122

struct IcFactor {  // sparse.hpp:45-49
  Csr lower;
  double shift = 0.0;
};
IcFactor incomplete_cholesky(const Csr& a);                             // sparse.cpp:184-203
void triangular_solve(const IcFactor& f, double* x, bool forward);     // sparse.cpp:205-238 (in place)

// ------------------------------------------------------------------- pcg ----
enum Prec { kIc0 = 0, kJacobi = 1, kNone = 2 };  // pcg.hpp:13
struct PcgConfig {                               // pcg.hpp:15-19
  double rel_tol = 1e-6;
  int max_iter = 1000;
  int prec = kIc0;
};
struct PcgReport {  // pcg.hpp:21-26
  int iterations = 0;
  double final_rel_residual = 0.0;
  bool converged = false;
  bool jacobi_fallback = false;
};

class PcgOperator {  // pcg.hpp:31-54, pcg.cpp:9-114
 public:
  PcgOperator() = default;
  PcgOperator(Csr a, PcgConfig cfg);
  PcgReport solve(const double* b, const double* x0, double* x) const;
  std::vector<PcgReport> solve_multi(const Mat& b, const Mat& x0, Mat& x) const;
  const Csr& matrix() const { return a_; }

 private:
  void precondition(const double* r, double* z) const;
  Csr a_;
  PcgConfig cfg_;
  bool have_ic_ = false;
  IcFactor ic_;
  Vec inv_diag_;
  bool fallback_ = false;
};

// ----------------------------------------------------------------- graph ----
struct Graph {  // graph.hpp:15-28
  int n = 0;
  std::vector<int> ei, ej;
  Vec w;
  Vec degree;
  double sigma = 0.0;
  int m() const { return static_cast<int>(w.size()); }
};
Csr difference_matrix(const Graph& g);     // graph.cpp:161-170
Vec degree_vector(const Graph& g);         // graph.cpp:172-174

// 4-neighbour image graph (graph.cpp:105-159) and its sigma heuristic (87-103).
// features: n x 3 (row-major RGB), vertex = row*width + col.
double median_neighbor_distance(int h, int w, const std::vector<double>& rgb);
Graph build_image_graph(int h, int w, const std::vector<double>& rgb, double sigma);

// ---------------------------------------------------------------- solver ----
struct Params {  // solver.hpp:16-25
  int dim = 5;
  double lambda = 100.0;
  double r = 1.0;
  int soc_max = 10;
  int sb_max_stage1 = 5;
  int sb_max_stage2 = 100;
  double conv_tol = 1e-4;
  PcgConfig pcg{1e-6, 1000, kIc0};
};
struct State {  // solver.hpp:28-34
  Mat y, p, bregman, split_b, split_s;
};
using IterCb = std::function<void(int, const Mat&)>;

double objective(const Csr& m, const Mat& y);          // solver.cpp:14-17
Mat shrink(const Mat& v, double gamma);                 // solver.cpp:19-25
Mat project_orthogonal(const Mat& a);                   // solver.cpp:27-41

// Per-inner-iteration PCG statistics (not in the reference: a run report
// so that inner iterations/s is interpretable).
struct RunLog {
  std::vector<int> pcg_iters;  // per inner iteration, max over columns
  long inner_iterations = 0;
  // wall seconds: solver construction + make_state, the inner split-Bregman
  // iterations (rhs, PCG, shrink / Bregman update), the per-outer projection
  double t_setup = 0.0, t_inner = 0.0, t_outer = 0.0;
};

class PfeSolver {  // solver.hpp:51-83, solver.cpp:43-136
 public:
  PfeSolver(const Graph& g, const Params& params);
  State make_state(const Mat& y0) const;
  void split_bregman(State& st, int max_iter, const IterCb& cb = {}) const;
  void run_soc(State& st, int soc_max, int sb_max) const;
  void outer_update(State& st) const;  // solver.cpp:116-118 (the body of one outer iteration after the inner loop)
  State two_stage(const Mat& y0) const;
  const Csr& diff_matrix() const { return m_; }
  RunLog* log = nullptr;

 private:
  Params params_;
  int n_;
  Csr m_, mt_;
  Vec degree_, sqrt_degree_;
  PcgOperator op_;
};

Mat split_bregman(const Csr& m, const Vec& d_vec, const Mat& p, const Mat& b, const Params& params,
                  const Mat& y_init, int max_iter, const IterCb& cb = {});  // solver.cpp:138-182
Mat soc(const Graph& g, const Params& params, const Mat& y0);                 // solver.cpp:184-189
Mat pfe_two_stage(const Graph& g, const Params& params, const Mat& y0);      // solver.cpp:191-193

// ------------------------------------------------------------------ init ----
struct Gmm {  // init.hpp:10-16
  int k = 0;
  Mat means, variances;
  Vec weights;
};
Gmm gmm_fit(const Mat& features, int k, uint64_t seed);                       // init.cpp:45-121
Mat responsibilities(const Gmm& g, const Mat& features);                      // init.cpp:123-138
Mat d_orthonormalize(const Mat& a, const Vec& degrees);                       // init.cpp:140-155
Mat init_embedding(const Gmm& g, const Mat& features, const Vec& degrees);    // init.cpp:157-170
Mat random_embedding(int n, int d, uint64_t seed, const Vec& degrees);       // init.cpp:172-181

// --------------------------------------------------------------- cluster ----
std::vector<int> kmeans(const Mat& points, int k, uint64_t seed, int max_iter = 100);  // cluster.cpp:54-124
double covering(const std::vector<int>& pred, const std::vector<int>& gt);              // metrics.cpp:57-72

// Worker threads for the column loop of solve_multi / spmm_dense.  Columns are
// independent, so any thread count gives bitwise-identical results
// (SPEC.md:239); 1 reproduces the reference's sequential execution.
void set_threads(int t);
int get_threads();

// Golden pin (golden_quadrant.cpp): oracles.hpp:179-213 + acceptance.cpp:310-335.
std::vector<double> quadrant_rgb(int size, double noise, uint64_t seed);
std::vector<int> quadrant_truth(int size);
struct GoldenResult {
  double obj0, obj1, covering, seconds;
  long inner_iterations;
};
GoldenResult run_golden_quadrant(int size);

}  // namespace orc
