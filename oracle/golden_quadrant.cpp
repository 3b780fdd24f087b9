// TEST INFRASTRUCTURE ONLY — pins the oracle to the reference's recorded run.
//
// Reproduces acceptance criteria 7 + 8 (proj/tests/acceptance.cpp:310-335) on
// the oracle: 64x64 quadrant image (proj/tests/oracles.hpp:179-213), sigma =
// median neighbour distance, default PfeParams (d=5, lambda=100, r=1, 10 SOC x
// 5 SB then 100 SB, conv_tol 1e-4, IC(0)-PCG), GMM init seed 0, k-means k=4
// seed 0.  The reference printed (proj/test_output.txt:29-30):
//   covering 1.000000 ; final objective 0.001466 <= 0.5 x initial 26.055418
#include <algorithm>
#include <chrono>
#include <cstdio>
#include <random>

#include "pfe_oracle.hpp"

namespace orc {

// oracles.hpp:179-198 — seeded jittered 4-colour quadrants, row-major RGB.
std::vector<double> quadrant_rgb(int size, double noise, uint64_t seed) {
  static const double colors[4][3] = {{0.95, 0.1, 0.1}, {0.1, 0.85, 0.15}, {0.15, 0.2, 0.9}, {0.9, 0.9, 0.1}};
  std::mt19937_64 rng(seed);
  std::uniform_real_distribution<double> jitter(-noise, noise);
  std::vector<double> img(static_cast<size_t>(size) * size * 3);
  for (int r = 0; r < size; ++r)
    for (int c = 0; c < size; ++c) {
      const int q = (r < size / 2 ? 0 : 2) + (c < size / 2 ? 0 : 1);
      for (int ch = 0; ch < 3; ++ch)
        img[(static_cast<size_t>(r) * size + c) * 3 + ch] = std::clamp(colors[q][ch] + jitter(rng), 0.0, 1.0);
    }
  return img;
}

// oracles.hpp:200-213
std::vector<int> quadrant_truth(int size) {
  std::vector<int> t(static_cast<size_t>(size) * size);
  for (int r = 0; r < size; ++r)
    for (int c = 0; c < size; ++c) t[static_cast<size_t>(r) * size + c] = (r < size / 2 ? 0 : 2) + (c < size / 2 ? 0 : 1);
  return t;
}

GoldenResult run_golden_quadrant(int size) {
  auto t0 = std::chrono::steady_clock::now();
  std::vector<double> rgb = quadrant_rgb(size, 0.02, 7);
  const long n = static_cast<long>(size) * size;
  Mat feats(n, 3);
  for (long v = 0; v < n; ++v)
    for (int c = 0; c < 3; ++c) feats(v, c) = rgb[static_cast<size_t>(3 * v + c)];
  const double sigma = median_neighbor_distance(size, size, rgb);
  Graph g = build_image_graph(size, size, rgb, sigma);
  Params params;  // reference defaults
  Gmm gmm = gmm_fit(feats, params.dim, 0);
  Mat y0 = init_embedding(gmm, feats, g.degree);
  PfeSolver solver(g, params);
  RunLog log;
  solver.log = &log;
  Mat y = solver.two_stage(y0).y;
  std::vector<int> seg = kmeans(y, 4, 0);
  GoldenResult res;
  res.covering = covering(seg, quadrant_truth(size));
  res.seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  Csr m = difference_matrix(g);
  res.obj0 = objective(m, y0);
  res.obj1 = objective(m, y);
  res.inner_iterations = log.inner_iterations;
  return res;
}

}  // namespace orc

#ifndef ORC_NO_MAIN
int main() {
  orc::GoldenResult r = orc::run_golden_quadrant(64);
  std::printf("covering %.6f in %.6f s\n", r.covering, r.seconds);
  std::printf("final objective %.6f initial %.6f\n", r.obj1, r.obj0);
  std::printf("inner iterations %ld\n", r.inner_iterations);
  const bool ok = std::abs(r.covering - 1.0) < 5e-7 && std::abs(r.obj1 - 0.001466) < 5e-7 &&
                  std::abs(r.obj0 - 26.055418) < 5e-7;
  std::printf("%s\n", ok ? "GOLDEN MATCH (proj/test_output.txt:29-30)" : "GOLDEN MISMATCH");
  return ok ? 0 : 1;
}
#endif
