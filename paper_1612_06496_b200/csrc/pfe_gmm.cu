// GMM initial embedding on the GPU (gmm_fit /
// responsibilities / init_embedding, init.cpp:45-170).
//
// Same algorithm and control flow as the reference:
//   * k-means (cluster.cpp, 20 Lloyd iterations, same seed) on the GPU
//     (pfe_kmeans.cu) for the starting means; the per-label means are then
//     summed on the host in point order, exactly as init.cpp does;
//   * up to 50 EM iterations of a diagonal-covariance GMM on RGB features:
//     the E step (log-likelihoods, log-sum-exp, responsibilities, total
//     log-likelihood) and the M-step sums run on the device; the scalar
//     logic (empty-component repair with the farthest point, variance floor
//     1e-6, weight normalisation, stop when the log-likelihood gain is
//     < 1e-7) runs on the host on k-sized arrays;
//   * Y0 = responsibilities, D-orthonormalised by modified Gram-Schmidt on
//     the device (init.cpp:140-155); if a column is dependent, the
//     reference's fallback adds N(0, 1e-6) noise from std::mt19937_64
//     (seed 0x9e3779b97f4a7c15, row-major draw order) and retries.
//
// Sums are deterministic: one warp per component sums a fixed stripe of
// points per lane, lanes are combined by a fixed butterfly, blocks by the
// host in block order.  Per-point arithmetic follows the reference's
// operation order; exp / log are CUDA's (within an ulp of glibc's), so the
// result agrees with the CPU oracle to rounding (tests/test_gpu_gmm.py).
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <limits>
#include <random>
#include <string>
#include <vector>

#include "pfe_b200.h"
#include "pfe_errors.h"

namespace pfe_host {
void kmeans_device(int n_, int d_, const double* pts, int k_, uint64_t seed, int max_iter, int32_t* labels);
}

namespace pfe_dev {

constexpr int kGmmMaxK = 16;
constexpr int kGmmPts = 8192;  // points per block in the sum kernels

struct GmmParams {
  int k;
  double c0;  // -1.5 log(2 pi)       (host libm, as the reference)
  double logw[kGmmMaxK];              // log(w_j)
  double mean[kGmmMaxK][3];
  double var[kGmmMaxK][3];
  double logvar[kGmmMaxK][3];         // log(var_jc)
};

// E step (init.cpp:72-86 / 123-138): resp[i + j n] and the per-point
// log-likelihood term mx + log(s).
__global__ void k_gmm_estep(const double* __restrict__ f, long n, GmmParams p, double* __restrict__ resp,
                            double* __restrict__ ll) {
  const double c0 = p.c0;
  for (long i = blockIdx.x * static_cast<long>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<long>(gridDim.x) * blockDim.x) {
    const double x[3] = {f[3 * i], f[3 * i + 1], f[3 * i + 2]};
    double lp[kGmmMaxK];
    double mx = 0.0;
#pragma unroll
    for (int j = 0; j < kGmmMaxK; ++j) {
      if (j >= p.k) break;
      double l = c0;
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        const double df = x[c] - p.mean[j][c];
        l -= 0.5 * (p.logvar[j][c] + df * df / p.var[j][c]);
      }
      lp[j] = p.logw[j] + l;
      mx = j == 0 ? lp[j] : fmax(mx, lp[j]);
    }
    double s = 0.0;
#pragma unroll
    for (int j = 0; j < kGmmMaxK; ++j) {
      if (j >= p.k) break;
      lp[j] = exp(lp[j] - mx);
      s += lp[j];
    }
#pragma unroll
    for (int j = 0; j < kGmmMaxK; ++j) {
      if (j >= p.k) break;
      resp[i + j * n] = lp[j] / s;
    }
    if (ll) ll[i] = mx + log(s);
  }
}

// Block partials of the M step.  Warp w handles component w; lane l sums
// points b*kGmmPts + l, + 32, ...  mode 0: [w][0] = sum r, [w][1..3] =
// sum r f_c, and warp 0 also sums ll into slot k*4; mode 1: [w][c] =
// sum r (f_c - mean_c)^2.  part: [block][4k+1].
__global__ void k_gmm_sums(const double* __restrict__ f, const double* __restrict__ resp, const double* __restrict__ ll,
                           long n, GmmParams p, int mode, double* __restrict__ part) {
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nq = 4 * p.k + 1;
  const long b0 = static_cast<long>(blockIdx.x) * kGmmPts;
  const long b1 = b0 + kGmmPts < n ? b0 + kGmmPts : n;
  if (w < p.k) {
    double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0, al = 0.0;
    for (long i = b0 + lane; i < b1; i += 32) {
      const double r = resp[i + static_cast<long>(w) * n];
      const double x0 = f[3 * i], x1 = f[3 * i + 1], x2 = f[3 * i + 2];
      if (mode == 0) {
        a0 += r;
        a1 += r * x0;
        a2 += r * x1;
        a3 += r * x2;
        if (w == 0) al += ll[i];
      } else {
        const double d0 = x0 - p.mean[w][0], d1 = x1 - p.mean[w][1], d2 = x2 - p.mean[w][2];
        a1 += r * (d0 * d0);
        a2 += r * (d1 * d1);
        a3 += r * (d2 * d2);
      }
    }
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) {
      a0 += __shfl_xor_sync(0xffffffffu, a0, o);
      a1 += __shfl_xor_sync(0xffffffffu, a1, o);
      a2 += __shfl_xor_sync(0xffffffffu, a2, o);
      a3 += __shfl_xor_sync(0xffffffffu, a3, o);
      al += __shfl_xor_sync(0xffffffffu, al, o);
    }
    if (lane == 0) {
      double* o = part + static_cast<long>(blockIdx.x) * nq;
      o[4 * w] = a0;
      o[4 * w + 1] = a1;
      o[4 * w + 2] = a2;
      o[4 * w + 3] = a3;
      if (w == 0) o[4 * p.k] = al;
    }
  }
}

// Block partials of sum_t a[t] * (deg[t] * b[t]) (init.cpp:146-150).
__global__ void k_gmm_ddot(const double* __restrict__ a, const double* __restrict__ b, const double* __restrict__ deg,
                           long n, double* __restrict__ part) {
  __shared__ double red[32];
  double s = 0.0;
  const long b0 = static_cast<long>(blockIdx.x) * kGmmPts;
  const long b1 = b0 + kGmmPts < n ? b0 + kGmmPts : n;
  for (long i = b0 + threadIdx.x; i < b1; i += blockDim.x) s += a[i] * (deg[i] * b[i]);
#pragma unroll
  for (int o = 16; o >= 1; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < static_cast<int>(blockDim.x >> 5); ++w) t += red[w];
    part[blockIdx.x] = t;
  }
}

// q -= proj * qi  (mode 0)  or  q /= nrm  (mode 1)  or  q += noise  (mode 2)
__global__ void k_gmm_axpy(double* __restrict__ q, const double* __restrict__ qi, double s, long n, int mode) {
  for (long i = blockIdx.x * static_cast<long>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<long>(gridDim.x) * blockDim.x) {
    if (mode == 0)
      q[i] -= s * qi[i];
    else if (mode == 1)
      q[i] /= s;
    else
      q[i] += qi[i];
  }
}

}  // namespace pfe_dev

namespace pfe_host {
namespace {

using pfe_dev::GmmParams;

#define GK(call)                                                                                 \
  do {                                                                                           \
    const cudaError_t e_ = (call);                                                               \
    if (e_ != cudaSuccess) throw Error(PFE_CUDA_ERROR, std::string(#call) + ": " + cudaGetErrorString(e_)); \
  } while (0)

struct DevBuf {
  double* p = nullptr;
  explicit DevBuf(size_t count) { GK(cudaMalloc(&p, std::max<size_t>(1, count) * sizeof(double))); }
  ~DevBuf() { cudaFree(p); }
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
};

// init.cpp:30-41 (host: rare repair step; features are host memory)
long farthest_point(const double* f, long n, const std::vector<double>& means, int k) {
  long best = 0;
  double best_d = -1.0;
  for (long i = 0; i < n; ++i) {
    double dmin = std::numeric_limits<double>::infinity();
    for (int j = 0; j < k; ++j) {
      double s = 0.0;
      for (int c = 0; c < 3; ++c) {
        const double df = means[j * 3 + c] - f[3 * i + c];
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

void gmm_init_device(int n_, const double* feat, int k, uint64_t seed, const double* degree, double* y_out,
                     double* means_out, double* vars_out, double* weights_out) {
  using namespace pfe_dev;
  const long n = n_;
  if (!feat || !degree || !y_out) throw Error(PFE_CONFIG_ERROR, "gmm_init: null argument");
  if (k < 1) throw Error(PFE_CONFIG_ERROR, "gmm_fit: k must be >= 1");
  if (k > kGmmMaxK) throw Error(PFE_CONFIG_ERROR, "gmm_init_device: k must be <= 16");
  if (n < k) throw Error(PFE_CONFIG_ERROR, "gmm_fit: fewer points than components");
  for (long i = 0; i < 3 * n; ++i)
    if (!std::isfinite(feat[i])) throw Error(PFE_CONFIG_ERROR, "gmm_fit: non-finite features");

  // k-means (20 iterations, same seed) on the device; column-major points
  std::vector<double> fcm(static_cast<size_t>(3 * n));
  for (long i = 0; i < n; ++i)
    for (int c = 0; c < 3; ++c) fcm[static_cast<size_t>(i + c * n)] = feat[3 * i + c];
  std::vector<int32_t> lab(static_cast<size_t>(n));
  kmeans_device(n_, 3, fcm.data(), k, seed, 20, lab.data());

  // init.cpp:55-64: per-label means (point order), variances 1e-2, weights 1/k
  std::vector<double> means(static_cast<size_t>(3 * k), 0.0), vars(static_cast<size_t>(3 * k), 1e-2),
      wts(static_cast<size_t>(k), 1.0 / k), cnt(static_cast<size_t>(k), 0.0);
  for (long i = 0; i < n; ++i) {
    for (int c = 0; c < 3; ++c) means[lab[i] * 3 + c] += feat[3 * i + c];
    cnt[lab[i]] += 1.0;
  }
  for (int j = 0; j < k; ++j)
    if (cnt[j] > 0.0)
      for (int c = 0; c < 3; ++c) means[j * 3 + c] /= cnt[j];

  DevBuf df(static_cast<size_t>(3 * n)), dresp(static_cast<size_t>(n) * k), dll(static_cast<size_t>(n)),
      ddeg(static_cast<size_t>(n));
  GK(cudaMemcpy(df.p, feat, sizeof(double) * 3 * n, cudaMemcpyHostToDevice));
  GK(cudaMemcpy(ddeg.p, degree, sizeof(double) * n, cudaMemcpyHostToDevice));
  const int nblk = static_cast<int>((n + kGmmPts - 1) / kGmmPts);
  const int nq = 4 * k + 1;
  DevBuf dpart(static_cast<size_t>(nblk) * nq);
  std::vector<double> part(static_cast<size_t>(nblk) * nq);
  const int eblocks = static_cast<int>(std::min<long>(4096, (n + 255) / 256));

  auto params = [&]() {
    GmmParams p{};
    p.k = k;
    p.c0 = -1.5 * std::log(2.0 * M_PI);
    for (int j = 0; j < k; ++j) {
      p.logw[j] = std::log(wts[j]);
      for (int c = 0; c < 3; ++c) {
        p.mean[j][c] = means[j * 3 + c];
        p.var[j][c] = vars[j * 3 + c];
        p.logvar[j][c] = std::log(vars[j * 3 + c]);
      }
    }
    return p;
  };
  // sums over blocks in block order
  auto reduce = [&](std::vector<double>& tot) {
    GK(cudaMemcpy(part.data(), dpart.p, sizeof(double) * part.size(), cudaMemcpyDeviceToHost));
    tot.assign(static_cast<size_t>(nq), 0.0);
    for (int b = 0; b < nblk; ++b)
      for (int q = 0; q < nq; ++q) tot[q] += part[static_cast<size_t>(b) * nq + q];
  };

  // EM (init.cpp:66-120)
  double prev = -std::numeric_limits<double>::infinity();
  int repairs = 0;
  std::vector<double> s1, s2;
  for (int iter = 0; iter < 50; ++iter) {
    GmmParams p = params();
    k_gmm_estep<<<eblocks, 256>>>(df.p, n, p, dresp.p, dll.p);
    k_gmm_sums<<<nblk, 32 * k>>>(df.p, dresp.p, dll.p, n, p, 0, dpart.p);
    GK(cudaGetLastError());
    reduce(s1);
    const double loglik = s1[4 * k];
    // means of every component first (the variance pass needs them)
    std::vector<double> nmean(static_cast<size_t>(3 * k), 0.0);
    for (int j = 0; j < k; ++j) {
      const double nj = s1[4 * j];
      if (nj > 0.0)
        for (int c = 0; c < 3; ++c) nmean[j * 3 + c] = s1[4 * j + 1 + c] / nj;
    }
    GmmParams pv = p;
    for (int j = 0; j < k; ++j)
      for (int c = 0; c < 3; ++c) pv.mean[j][c] = nmean[j * 3 + c];
    k_gmm_sums<<<nblk, 32 * k>>>(df.p, dresp.p, dll.p, n, pv, 1, dpart.p);
    GK(cudaGetLastError());
    reduce(s2);
    bool repaired = false;
    for (int j = 0; j < k; ++j) {
      const double nj = s1[4 * j];
      if (nj < 1e-8 && repairs < 5) {
        const long fi = farthest_point(feat, n, means, k);
        for (int c = 0; c < 3; ++c) {
          means[j * 3 + c] = feat[3 * fi + c];
          vars[j * 3 + c] = 1e-2;
        }
        wts[j] = 1.0 / n;
        ++repairs;
        repaired = true;
        continue;
      }
      if (nj <= 0.0) continue;
      for (int c = 0; c < 3; ++c) {
        means[j * 3 + c] = nmean[j * 3 + c];
        vars[j * 3 + c] = std::max(s2[4 * j + 1 + c] / nj, 1e-6);
      }
      wts[j] = nj / n;
    }
    double ws = 0.0;
    for (int j = 0; j < k; ++j) ws += wts[j];
    for (int j = 0; j < k; ++j) wts[j] /= ws;
    if (!repaired && loglik - prev < 1e-7 && iter > 0) break;
    prev = loglik;
  }
  if (means_out) std::copy(means.begin(), means.end(), means_out);
  if (vars_out) std::copy(vars.begin(), vars.end(), vars_out);
  if (weights_out) std::copy(wts.begin(), wts.end(), weights_out);

  // responsibilities of the fitted model (init.cpp:123-138)
  {
    GmmParams p = params();
    k_gmm_estep<<<eblocks, 256>>>(df.p, n, p, dresp.p, nullptr);
    GK(cudaGetLastError());
  }

  // D-orthonormalisation (init.cpp:140-155) on a copy; fallback with noise
  DevBuf dq(static_cast<size_t>(n) * k), dparts(static_cast<size_t>(nblk));
  std::vector<double> pp(static_cast<size_t>(nblk));
  auto ddot = [&](const double* a, const double* b) {
    pfe_dev::k_gmm_ddot<<<nblk, 256>>>(a, b, ddeg.p, n, dparts.p);
    GK(cudaGetLastError());
    GK(cudaMemcpy(pp.data(), dparts.p, sizeof(double) * nblk, cudaMemcpyDeviceToHost));
    double s = 0.0;
    for (int b = 0; b < nblk; ++b) s += pp[b];
    return s;
  };
  auto mgs = [&]() -> bool {
    for (int j = 0; j < k; ++j) {
      double* qj = dq.p + static_cast<long>(j) * n;
      for (int i = 0; i < j; ++i) {
        const double* qi = dq.p + static_cast<long>(i) * n;
        const double proj = ddot(qj, qi);
        pfe_dev::k_gmm_axpy<<<eblocks, 256>>>(qj, qi, proj, n, 0);
      }
      const double nrm = std::sqrt(ddot(qj, qj));
      if (nrm < 1e-10) return false;
      pfe_dev::k_gmm_axpy<<<eblocks, 256>>>(qj, nullptr, nrm, n, 1);
    }
    GK(cudaGetLastError());
    return true;
  };
  GK(cudaMemcpy(dq.p, dresp.p, sizeof(double) * n * k, cudaMemcpyDeviceToDevice));
  if (!mgs()) {
    // init.cpp:160-168: resp(i, j) += N(0, 1e-6), drawn row by row
    std::mt19937_64 rng(0x9e3779b97f4a7c15ull);
    std::normal_distribution<double> dist(0.0, 1e-6);
    std::vector<double> noise(static_cast<size_t>(n) * k);
    for (long i = 0; i < n; ++i)
      for (int j = 0; j < k; ++j) noise[static_cast<size_t>(i + j * n)] = dist(rng);
    GK(cudaMemcpy(dq.p, noise.data(), sizeof(double) * n * k, cudaMemcpyHostToDevice));
    pfe_dev::k_gmm_axpy<<<eblocks, 256>>>(dq.p, dresp.p, 0.0, n * k, 2);
    GK(cudaGetLastError());
    if (!mgs()) throw Error(PFE_NUMERICAL_ERROR, "d_orthonormalize: dependent column");
  }
  GK(cudaMemcpy(y_out, dq.p, sizeof(double) * n * k, cudaMemcpyDeviceToHost));
}

}  // namespace pfe_host
