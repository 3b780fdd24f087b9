// Host-side boundary helpers of the C ABI (no GPU work): the seeded initial
// embedding and the k-means "labels out" step.  They must consume the same
// libstdc++ random streams as the reference so that CPU and GPU runs start
// from the identical Y0 and cluster with identical seeding.
//
//   pfe_d_orthonormalize  init.cpp:140-155 (Gram-Schmidt in the D inner product)
//   pfe_random_embedding  init.cpp:172-181
//   pfe_kmeans            cluster.cpp:15-124 (k-means++ seeding + Lloyd)
//
// The k-means assignment sweep is parallelised over point blocks with
// std::thread (labels and inertia are order independent: each point's
// argmin is computed exactly as the reference does; inertia is summed per
// block in fixed order).
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <limits>
#include <random>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include "pfe_b200.h"
#include "pfe_errors.h"

namespace pfe_host {

namespace {

// Column-major view helpers.
inline double& at(std::vector<double>& a, long n, long i, long j) { return a[static_cast<size_t>(i + j * n)]; }

void d_orthonormalize_inplace(std::vector<double>& q, long n, long d, const double* deg) {
  for (long j = 0; j < d; ++j) {
    double* qj = q.data() + j * n;
    for (long i = 0; i < j; ++i) {
      const double* qi = q.data() + i * n;
      double proj = 0.0;
      for (long t = 0; t < n; ++t) proj += qj[t] * (deg[t] * qi[t]);
      for (long t = 0; t < n; ++t) qj[t] -= proj * qi[t];
    }
    double s = 0.0;
    for (long t = 0; t < n; ++t) s += qj[t] * (deg[t] * qj[t]);
    const double nrm = std::sqrt(s);
    if (nrm < 1e-10) throw Error(PFE_NUMERICAL_ERROR, "d_orthonormalize: dependent column " + std::to_string(j));
    for (long t = 0; t < n; ++t) qj[t] /= nrm;
  }
}

double row_dist2(const double* pts, long n, long d, long i, const std::vector<double>& cen, long k, long c) {
  double s = 0.0;
  for (long t = 0; t < d; ++t) {
    const double df = pts[i + t * n] - cen[static_cast<size_t>(c + t * k)];
    s += df * df;
  }
  return s;
}

}  // namespace

void random_embedding(int n, int d, uint64_t seed, const double* deg, double* out) {
  if (n < 1 || d < 1) throw Error(PFE_CONFIG_ERROR, "random_embedding: n and d must be >= 1");
  std::mt19937_64 rng(seed);
  std::normal_distribution<double> dist(0.0, 1.0);
  std::vector<double> a(static_cast<size_t>(n) * d);
  for (long i = 0; i < n; ++i)
    for (long j = 0; j < d; ++j) at(a, n, i, j) = dist(rng);
  d_orthonormalize_inplace(a, n, d, deg);
  std::copy(a.begin(), a.end(), out);
}

void d_orthonormalize(int n, int d, const double* a, const double* deg, double* out) {
  std::vector<double> q(a, a + static_cast<size_t>(n) * d);
  d_orthonormalize_inplace(q, n, d, deg);
  std::copy(q.begin(), q.end(), out);
}

void kmeans(int n_, int d_, const double* pts, int k_, uint64_t seed, int max_iter, int32_t* labels) {
  const long n = n_, d = d_, k = k_;
  if (k < 1) throw Error(PFE_CONFIG_ERROR, "kmeans: k must be >= 1");
  if (k > n) throw Error(PFE_CONFIG_ERROR, "kmeans: k exceeds point count");
  std::mt19937_64 rng(seed);
  std::vector<double> cen(static_cast<size_t>(k * d));
  // k-means++ seeding (cluster.cpp:15-51)
  std::uniform_int_distribution<long> first(0, n - 1);
  {
    const long f0 = first(rng);
    for (long t = 0; t < d; ++t) cen[static_cast<size_t>(t * k)] = pts[f0 + t * n];
    std::vector<double> d2(static_cast<size_t>(n));
    for (long i = 0; i < n; ++i) d2[i] = row_dist2(pts, n, d, i, cen, k, 0);
    std::uniform_real_distribution<double> uni(0.0, 1.0);
    for (long c = 1; c < k; ++c) {
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
      for (long t = 0; t < d; ++t) cen[static_cast<size_t>(c + t * k)] = pts[chosen + t * n];
      for (long i = 0; i < n; ++i) d2[i] = std::min(d2[i], row_dist2(pts, n, d, i, cen, k, c));
    }
  }
  // Lloyd (cluster.cpp:67-121)
  const int nthreads = std::max(1, std::min<int>(static_cast<int>(std::thread::hardware_concurrency()), 16));
  const long chunk = (n + nthreads - 1) / nthreads;
  std::vector<double> part(static_cast<size_t>(nthreads));
  double prev = std::numeric_limits<double>::infinity();
  for (int iter = 0; iter < max_iter; ++iter) {
    auto assign = [&](int w) {
      const long lo = w * chunk, hi = std::min(n, lo + chunk);
      double s = 0.0;
      for (long i = lo; i < hi; ++i) {
        int best = 0;
        double bd = row_dist2(pts, n, d, i, cen, k, 0);
        for (long c = 1; c < k; ++c) {
          const double dd = row_dist2(pts, n, d, i, cen, k, c);
          if (dd < bd) {
            bd = dd;
            best = static_cast<int>(c);
          }
        }
        labels[i] = best;
        s += bd;
      }
      part[w] = s;
    };
    if (n >= 65536 && nthreads > 1) {
      std::vector<std::thread> pool;
      for (int w = 0; w < nthreads; ++w) pool.emplace_back(assign, w);
      for (auto& t : pool) t.join();
    } else {
      for (int w = 0; w < nthreads; ++w) assign(w);
    }
    double inertia = 0.0;
    for (int w = 0; w < nthreads; ++w) inertia += part[w];
    std::vector<double> sums(static_cast<size_t>(k * d), 0.0);
    std::vector<long> cnt(static_cast<size_t>(k), 0);
    for (long i = 0; i < n; ++i) {
      for (long t = 0; t < d; ++t) sums[static_cast<size_t>(labels[i] + t * k)] += pts[i + t * n];
      ++cnt[labels[i]];
    }
    for (long c = 0; c < k; ++c) {
      if (cnt[c] > 0) {
        for (long t = 0; t < d; ++t)
          cen[static_cast<size_t>(c + t * k)] = sums[static_cast<size_t>(c + t * k)] / static_cast<double>(cnt[c]);
        continue;
      }
      long largest = 0;
      for (long c2 = 1; c2 < k; ++c2)
        if (cnt[c2] > cnt[largest]) largest = c2;
      long far_i = -1;
      double far_d = -1.0;
      for (long i = 0; i < n; ++i) {
        if (labels[i] != largest) continue;
        const double dd = row_dist2(pts, n, d, i, cen, k, largest);
        if (dd > far_d) {
          far_d = dd;
          far_i = i;
        }
      }
      for (long t = 0; t < d; ++t) cen[static_cast<size_t>(c + t * k)] = pts[far_i + t * n];
      labels[far_i] = static_cast<int32_t>(c);
      cnt[c] = 1;
      cnt[largest]--;
    }
    if (prev - inertia <= 1e-6 * std::max(prev, 1e-300) && inertia <= prev) break;
    prev = inertia;
  }
}

// ------------------------------------------------------------ IC(0) ------
// sparse.cpp:124-203.  The factor is set-up for the device triangular solves
// (pfe_runtime.cu, k_ic_apply); the per-row arithmetic (sparse dot over the
// columns below j, pivot sqrt, off-diagonal division) follows the reference
// operation for operation, so the factor is the reference's bit for bit.
namespace {
bool ic0_sweep(IcFactorHost& l, int n) {
  for (int i = 0; i < n; ++i) {
    const int b = l.ptr[i], e = l.ptr[i + 1];
    if (b == e || l.idx[e - 1] != i) return false;  // no diagonal
    for (int k = b; k < e; ++k) {
      const int j = l.idx[k];
      double dot = 0.0;
      int pi = b, pj = l.ptr[j];
      const int ej = l.ptr[j + 1];
      while (pi < k && pj < ej && l.idx[pj] < j) {
        const int ci = l.idx[pi], cj = l.idx[pj];
        if (ci == cj) {
          dot += l.val[pi] * l.val[pj];
          ++pi;
          ++pj;
        } else if (ci < cj) {
          ++pi;
        } else {
          ++pj;
        }
      }
      if (j == i) {
        const double piv = l.val[k] - dot;
        if (!(piv > 0.0)) return false;
        l.val[k] = std::sqrt(piv);
      } else {
        l.val[k] = (l.val[k] - dot) / l.val[l.ptr[j + 1] - 1];
      }
    }
  }
  return true;
}
}  // namespace

bool ic0_factor(int n, const int* ptr, const int* idx, const double* val, IcFactorHost& out) {
  double dmax = 0.0;
  for (int r = 0; r < n; ++r)
    for (int k = ptr[r]; k < ptr[r + 1]; ++k)
      if (idx[k] == r) dmax = std::max(dmax, val[k]);
  double shift = 0.0;
  for (int attempt = 0; attempt <= 8; ++attempt) {
    IcFactorHost l;
    l.shift = shift;
    l.ptr.assign(static_cast<size_t>(n) + 1, 0);
    for (int r = 0; r < n; ++r) {
      for (int k = ptr[r]; k < ptr[r + 1]; ++k) {
        if (idx[k] > r) continue;
        l.idx.push_back(idx[k]);
        l.val.push_back(idx[k] == r ? val[k] + shift : val[k]);
      }
      l.ptr[r + 1] = static_cast<int>(l.val.size());
    }
    if (ic0_sweep(l, n)) {
      out = std::move(l);
      return true;
    }
    shift = shift == 0.0 ? 1e-3 * std::max(dmax, 1.0) : 2.0 * shift;
  }
  return false;
}

}  // namespace pfe_host
