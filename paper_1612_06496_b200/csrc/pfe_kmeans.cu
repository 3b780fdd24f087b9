// k-means "labels out" on the GPU (kmeans, cluster.cpp:15-124).
//
// Same algorithm and random stream as the host kmeans (pfe_host.cpp): k-means++
// seeding driven by std::mt19937_64 with libstdc++'s uniform distributions,
// then Lloyd iterations with the lowest-index tie-break, the empty-cluster
// split and the relative-inertia stop.  The O(n k d) work runs on the device:
//
//   * seeding: d2[i] = min_c |x_i - c|^2 is kept on the device; for every new
//     centre the device writes sequential sums of d2 over fixed chunks of
//     points, the host walks the chunk sums to the chunk holding the sampled
//     target and scans that chunk's d2 values sequentially (one 32 KB copy);
//   * assignment: centres in shared memory, one thread per point, distances
//     summed over dimensions in the reference's order;
//   * update: per-chunk per-cluster sums in point order (one thread per
//     cluster scans the chunk's labels), then the chunk partials summed in
//     chunk order.
//
// Distances are bitwise those of the host; the sums of d2, of the inertia and
// of the cluster coordinates associate by chunk instead of one running sum,
// so centroids can differ in the last bits (the north_star label gate is
// >= 99.9 % agreement with the oracle's labels).
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <limits>
#include <random>
#include <string>
#include <utility>
#include <vector>

#include "pfe_b200.h"
#include "pfe_errors.h"

namespace pfe_dev {

constexpr int kKmChunk = 4096;   // points per sequential chunk
constexpr int kKmThreads = 256;

__device__ __forceinline__ double km_dist2(const double* __restrict__ pts, long n, int d, long i,
                                           const double* cen, int k, int c) {
  double s = 0.0;
  for (int t = 0; t < d; ++t) {
    const double df = pts[i + t * n] - cen[c + t * k];
    s += df * df;
  }
  return s;
}

// d2[i] = |x_i - c0|^2 (first) or min(d2[i], |x_i - c|^2); chunk sums of d2.
__global__ void k_km_seed_update(const double* __restrict__ pts, long n, int d, const double* __restrict__ c_new,
                                 double* __restrict__ d2, int first) {
  const long i = static_cast<long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < n) {
    double s = 0.0;
    for (int t = 0; t < d; ++t) {
      const double df = pts[i + t * n] - c_new[t];
      s += df * df;
    }
    d2[i] = first ? s : fmin(d2[i], s);
  }
}

// Sequential sum of d2 over chunk b (one thread per chunk).
__global__ void k_km_chunk_sums(const double* __restrict__ d2, long n, double* __restrict__ chunk_sum, long nchunks) {
  const long b = static_cast<long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (b >= nchunks) return;
  const long lo = b * kKmChunk, hi = min(n, lo + kKmChunk);
  double s = 0.0;
  for (long i = lo; i < hi; ++i) s += d2[i];
  chunk_sum[b] = s;
}

// Lloyd assignment: labels and per-point best distances.
template <int D>
__global__ void k_km_assign(const double* __restrict__ pts, long n, const double* __restrict__ cen, int k,
                            int32_t* __restrict__ labels, double* __restrict__ best_d) {
  extern __shared__ double sc[];  // centres [D][k]
  for (int e = threadIdx.x; e < k * D; e += blockDim.x) sc[e] = cen[e];
  __syncthreads();
  const long i = static_cast<long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n) return;
  double x[D];
#pragma unroll
  for (int t = 0; t < D; ++t) x[t] = pts[i + t * n];
  int best = 0;
  double bd = 0.0;
  for (int c = 0; c < k; ++c) {
    double s = 0.0;
#pragma unroll
    for (int t = 0; t < D; ++t) {
      const double df = x[t] - sc[c + t * k];
      s += df * df;
    }
    if (c == 0 || s < bd) {
      bd = s;
      best = c;
    }
  }
  labels[i] = best;
  best_d[i] = bd;
}

// Per chunk: sequential sums of the best distances (inertia), and per cluster
// the sums of its points' coordinates in point order plus the count.
template <int D>
__global__ void k_km_chunk_update(const double* __restrict__ pts, long n, int k,
                                  const int32_t* __restrict__ labels, const double* __restrict__ best_d,
                                  double* __restrict__ part_sum, long* __restrict__ part_cnt,
                                  double* __restrict__ part_inertia) {
  __shared__ int32_t lab[kKmChunk];
  const long lo = static_cast<long>(blockIdx.x) * kKmChunk, hi = min(n, lo + kKmChunk);
  const int cnt = static_cast<int>(hi - lo);
  for (int e = threadIdx.x; e < cnt; e += blockDim.x) lab[e] = labels[lo + e];
  __syncthreads();
  if (threadIdx.x == 0) {
    double s = 0.0;
    for (long i = lo; i < hi; ++i) s += best_d[i];
    part_inertia[blockIdx.x] = s;
  }
  for (int c = threadIdx.x; c < k; c += blockDim.x) {
    double acc[D];
#pragma unroll
    for (int t = 0; t < D; ++t) acc[t] = 0.0;
    long m = 0;
    for (int e = 0; e < cnt; ++e) {
      if (lab[e] != c) continue;
#pragma unroll
      for (int t = 0; t < D; ++t) acc[t] += pts[lo + e + t * n];
      ++m;
    }
    const long base = static_cast<long>(blockIdx.x) * k + c;
#pragma unroll
    for (int t = 0; t < D; ++t) part_sum[base * D + t] = acc[t];
    part_cnt[base] = m;
  }
}

// Chunk partials -> per cluster sums and counts, in chunk order.
__global__ void k_km_reduce(const double* __restrict__ part_sum, const long* __restrict__ part_cnt, long nchunks, int k,
                            int d, double* __restrict__ sums, long* __restrict__ cnts) {
  const int e = blockIdx.x * blockDim.x + threadIdx.x;  // (cluster, t) or count
  if (e >= k * (d + 1)) return;
  const int c = e / (d + 1), t = e - c * (d + 1);
  if (t < d) {
    double s = 0.0;
    for (long b = 0; b < nchunks; ++b) s += part_sum[(b * k + c) * d + t];
    sums[c * d + t] = s;
  } else {
    long m = 0;
    for (long b = 0; b < nchunks; ++b) m += part_cnt[b * k + c];
    cnts[c] = m;
  }
}

}  // namespace pfe_dev

namespace pfe_host {

namespace {

#define KMCK(x)                                                                             \
  do {                                                                                      \
    cudaError_t e_ = (x);                                                                   \
    if (e_ != cudaSuccess) throw Error(PFE_CUDA_ERROR, std::string(#x) + ": " + cudaGetErrorString(e_)); \
  } while (0)

struct DevBuf {
  void* p = nullptr;
  cudaStream_t s;
  DevBuf(size_t bytes, cudaStream_t st) : s(st) {
    if (cudaMallocAsync(&p, std::max<size_t>(bytes, 8), st) != cudaSuccess)
      throw Error(PFE_CUDA_ERROR, "kmeans: device allocation failed");
  }
  ~DevBuf() { cudaFreeAsync(p, s); }
  template <class T>
  T* as() const {
    return static_cast<T*>(p);
  }
};

template <int D>
void lloyd_step_d(int gpts, int gchunks, cudaStream_t st, const double* pts, long n, const double* cen, int k,
                  int32_t* lab, double* best, double* psum, long* pcnt, double* pin) {
  pfe_dev::k_km_assign<D><<<gpts, pfe_dev::kKmThreads, sizeof(double) * k * D, st>>>(pts, n, cen, k, lab, best);
  KMCK(cudaGetLastError());
  pfe_dev::k_km_chunk_update<D><<<gchunks, pfe_dev::kKmThreads, 0, st>>>(pts, n, k, lab, best, psum, pcnt, pin);
  KMCK(cudaGetLastError());
}

template <int... Ds>
void lloyd_dispatch(int d, std::integer_sequence<int, Ds...>, int gpts, int gchunks, cudaStream_t st, const double* pts,
                    long n, const double* cen, int k, int32_t* lab, double* best, double* psum, long* pcnt,
                    double* pin) {
  ((d == Ds + 1 ? (lloyd_step_d<Ds + 1>(gpts, gchunks, st, pts, n, cen, k, lab, best, psum, pcnt, pin), true) : false),
   ...);
}

void lloyd_step(int d, int gpts, int gchunks, cudaStream_t st, const double* pts, long n, const double* cen, int k,
                int32_t* lab, double* best, double* psum, long* pcnt, double* pin) {
  lloyd_dispatch(d, std::make_integer_sequence<int, 16>{}, gpts, gchunks, st, pts, n, cen, k, lab, best, psum, pcnt,
                 pin);
}

}  // namespace

void kmeans_device(int n_, int d_, const double* pts, int k_, uint64_t seed, int max_iter, int32_t* labels) {
  using namespace pfe_dev;
  const long n = n_;
  const int d = d_, k = k_;
  if (k < 1) throw Error(PFE_CONFIG_ERROR, "kmeans: k must be >= 1");
  if (k > n) throw Error(PFE_CONFIG_ERROR, "kmeans: k exceeds point count");
  if (d < 1 || d > 16) throw Error(PFE_CONFIG_ERROR, "kmeans (device): dimension must be in [1, 16]");
  if (static_cast<long>(k) * d * 8 > 48 * 1024) throw Error(PFE_CONFIG_ERROR, "kmeans (device): k * d too large");
  cudaStream_t st;
  KMCK(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
  struct StreamGuard {
    cudaStream_t s;
    ~StreamGuard() {
      cudaStreamSynchronize(s);
      cudaStreamDestroy(s);
    }
  } sg{st};
  const long nchunks = (n + kKmChunk - 1) / kKmChunk;
  DevBuf dpts(sizeof(double) * n * d, st), dd2(sizeof(double) * n, st), dcs(sizeof(double) * nchunks, st),
      dcen(sizeof(double) * k * d, st), dlab(sizeof(int32_t) * n, st), dbest(sizeof(double) * n, st),
      dpsum(sizeof(double) * nchunks * k * d, st), dpcnt(sizeof(long) * nchunks * k, st),
      dpin(sizeof(double) * nchunks, st), dsums(sizeof(double) * k * d, st), dcnts(sizeof(long) * k, st),
      dcnew(sizeof(double) * d, st);
  KMCK(cudaMemcpyAsync(dpts.p, pts, sizeof(double) * n * d, cudaMemcpyHostToDevice, st));
  const int gpts = static_cast<int>((n + kKmThreads - 1) / kKmThreads);
  const int gchunks = static_cast<int>((nchunks + kKmThreads - 1) / kKmThreads);

  std::mt19937_64 rng(seed);
  std::vector<double> cen(static_cast<size_t>(k) * d);  // [t][c] (column-major k x d, as the reference)
  std::vector<double> cnew(d), csum(nchunks), chunk(kKmChunk);
  // k-means++ seeding (cluster.cpp:15-51)
  std::uniform_int_distribution<long> first(0, n - 1);
  auto set_centre = [&](int c, long i, int first_call) {
    for (int t = 0; t < d; ++t) cnew[t] = cen[static_cast<size_t>(c) + static_cast<size_t>(t) * k] = pts[i + t * n];
    KMCK(cudaMemcpyAsync(dcnew.p, cnew.data(), sizeof(double) * d, cudaMemcpyHostToDevice, st));
    k_km_seed_update<<<gpts, kKmThreads, 0, st>>>(dpts.as<double>(), n, d, dcnew.as<double>(), dd2.as<double>(),
                                                   first_call);
    KMCK(cudaGetLastError());
  };
  set_centre(0, first(rng), 1);
  std::uniform_real_distribution<double> uni(0.0, 1.0);
  for (int c = 1; c < k; ++c) {
    k_km_chunk_sums<<<gchunks, kKmThreads, 0, st>>>(dd2.as<double>(), n, dcs.as<double>(), nchunks);
    KMCK(cudaGetLastError());
    KMCK(cudaMemcpyAsync(csum.data(), dcs.p, sizeof(double) * nchunks, cudaMemcpyDeviceToHost, st));
    KMCK(cudaStreamSynchronize(st));
    double total = 0.0;
    for (long b = 0; b < nchunks; ++b) total += csum[b];
    long chosen = 0;
    if (total > 0.0) {
      const double target = uni(rng) * total;
      double acc = 0.0;
      long b = 0;
      for (; b < nchunks - 1 && acc + csum[b] < target; ++b) acc += csum[b];
      const long lo = b * kKmChunk, cnt = std::min<long>(kKmChunk, n - lo);
      KMCK(cudaMemcpyAsync(chunk.data(), dd2.as<double>() + lo, sizeof(double) * cnt, cudaMemcpyDeviceToHost, st));
      KMCK(cudaStreamSynchronize(st));
      chosen = 0;  // as the reference when rounding leaves the running sum short of the target
      for (long e = 0; e < cnt; ++e) {
        acc += chunk[e];
        if (acc >= target) {
          chosen = lo + e;
          break;
        }
      }
    } else {
      chosen = first(rng);
    }
    set_centre(c, chosen, 0);
  }
  // Lloyd (cluster.cpp:67-121)
  std::vector<double> sums(static_cast<size_t>(k) * d), pin(nchunks);
  std::vector<long> cnts(k);
  std::vector<int32_t> hlab;
  std::vector<double> ccm(static_cast<size_t>(k) * d);  // device layout [t][c]
  double prev = std::numeric_limits<double>::infinity();
  for (int iter = 0; iter < max_iter; ++iter) {
    KMCK(cudaMemcpyAsync(dcen.p, cen.data(), sizeof(double) * k * d, cudaMemcpyHostToDevice, st));
    lloyd_step(d, gpts, static_cast<int>(nchunks), st, dpts.as<double>(), n, dcen.as<double>(), k, dlab.as<int32_t>(),
               dbest.as<double>(), dpsum.as<double>(), dpcnt.as<long>(), dpin.as<double>());
    k_km_reduce<<<(k * (d + 1) + 127) / 128, 128, 0, st>>>(dpsum.as<double>(), dpcnt.as<long>(), nchunks, k, d,
                                                           dsums.as<double>(), dcnts.as<long>());
    KMCK(cudaGetLastError());
    KMCK(cudaMemcpyAsync(sums.data(), dsums.p, sizeof(double) * k * d, cudaMemcpyDeviceToHost, st));
    KMCK(cudaMemcpyAsync(cnts.data(), dcnts.p, sizeof(long) * k, cudaMemcpyDeviceToHost, st));
    KMCK(cudaMemcpyAsync(pin.data(), dpin.p, sizeof(double) * nchunks, cudaMemcpyDeviceToHost, st));
    KMCK(cudaStreamSynchronize(st));
    double inertia = 0.0;
    for (long b = 0; b < nchunks; ++b) inertia += pin[b];
    bool relabelled = false;
    for (int c = 0; c < k; ++c) {
      if (cnts[c] > 0) {
        for (int t = 0; t < d; ++t)
          cen[static_cast<size_t>(c) + static_cast<size_t>(t) * k] =
              sums[static_cast<size_t>(c) * d + t] / static_cast<double>(cnts[c]);
        continue;
      }
      // empty cluster: the farthest point of the largest cluster (cluster.cpp:96-115)
      if (hlab.empty()) {
        hlab.resize(n);
        KMCK(cudaMemcpyAsync(hlab.data(), dlab.p, sizeof(int32_t) * n, cudaMemcpyDeviceToHost, st));
        KMCK(cudaStreamSynchronize(st));
      }
      int largest = 0;
      for (int c2 = 1; c2 < k; ++c2)
        if (cnts[c2] > cnts[largest]) largest = c2;
      long far_i = -1;
      double far_d = -1.0;
      for (long i = 0; i < n; ++i) {
        if (hlab[i] != largest) continue;
        double s = 0.0;
        for (int t = 0; t < d; ++t) {
          const double df = pts[i + t * n] - cen[static_cast<size_t>(largest) + static_cast<size_t>(t) * k];
          s += df * df;
        }
        if (s > far_d) {
          far_d = s;
          far_i = i;
        }
      }
      for (int t = 0; t < d; ++t) cen[static_cast<size_t>(c) + static_cast<size_t>(t) * k] = pts[far_i + t * n];
      hlab[far_i] = c;
      cnts[c] = 1;
      cnts[largest]--;
      relabelled = true;
    }
    if (relabelled) KMCK(cudaMemcpyAsync(dlab.p, hlab.data(), sizeof(int32_t) * n, cudaMemcpyHostToDevice, st));
    hlab.clear();
    if (prev - inertia <= 1e-6 * std::max(prev, 1e-300) && inertia <= prev) break;
    prev = inertia;
  }
  KMCK(cudaMemcpyAsync(labels, dlab.p, sizeof(int32_t) * n, cudaMemcpyDeviceToHost, st));
  KMCK(cudaStreamSynchronize(st));
}

}  // namespace pfe_host
