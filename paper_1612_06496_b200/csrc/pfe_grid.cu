// Pixel-grid graph builder on the GPU (configs C2-C4).
//
// Semantics of build_image_graph (graph.cpp:105-159) generalised to the
// 8-neighbour and 5x5 neighbourhoods, exactly as the harness builder
// paper_1612_06496_b200/inputs.py grid_graph defines them:
//
//   1. every forward stencil pair (v, v + off_s), off_s = dy * W + dx in
//      lexicographic order, inside the image, is a candidate with
//      w = exp(-(|f_v - f_u|^2 / (2 sigma_rgb^2) [+ (dy^2 + dx^2) / (2 sigma_xy^2)]))
//      (|.|^2 summed over the 3 channels left to right, as numpy sums a row
//      of 3);
//   2. candidates with w < 1e-12 are dropped;
//   3. a vertex left without an edge keeps its strongest incident candidate
//      (first in edge order on ties), its weight floored at 1e-12;
//   4. edges in lexicographic (i < j) order: pixel-major, slot order;
//   5. degree summed in edge order: a vertex's "j" contributions (backward
//      slots, i ascending) before its "i" contributions (forward slots).
//
// Steps 1, 2, 4, 5 run on the device: a candidate kernel writes the [n][S]
// slot weights (-1 = no candidate) and the per-vertex kept-edge counts, a
// block-scan pass gives every vertex its first edge index, and a second
// kernel writes the compacted edge list and the degrees.  Step 3 is rare
// (none in the benchmark images) and runs on the host for the flagged
// vertices only, on their few candidate weights.  Weights equal the host
// builder's up to the last ulp of exp (CUDA's exp vs the host libm's).
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <string>
#include <vector>

#include "pfe_b200.h"
#include "pfe_errors.h"

namespace pfe_dev {

constexpr int kGridThreads = 256;
constexpr double kWeightFloor = 1e-12;

template <int R>
struct Stencil;
template <>
struct Stencil<1> {
  static constexpr int S = 4;
  __host__ __device__ static constexpr int dy(int s) { return s == 0 ? 0 : 1; }
  __host__ __device__ static constexpr int dx(int s) { return s == 0 ? 1 : s - 2; }
};
template <>
struct Stencil<2> {
  static constexpr int S = 12;
  __host__ __device__ static constexpr int dy(int s) { return s < 2 ? 0 : (s < 7 ? 1 : 2); }
  __host__ __device__ static constexpr int dx(int s) { return s < 2 ? s + 1 : (s < 7 ? s - 4 : s - 9); }
};

// Candidate weights of every (v, s): wc[v][s] = w, or -1 outside the image.
// kept[v] = number of kept forward edges of v.
template <int R>
__global__ void __launch_bounds__(kGridThreads) k_grid_candidates(int H, int W, const double* __restrict__ rgb,
                                                                 double inv_rgb, double inv_xy, int use_xy,
                                                                 double* __restrict__ wc, int* __restrict__ kept) {
  using T = Stencil<R>;
  const long n = static_cast<long>(H) * W;
  for (long v = static_cast<long>(blockIdx.x) * blockDim.x + threadIdx.x; v < n; v += static_cast<long>(gridDim.x) * blockDim.x) {
    const int y = static_cast<int>(v / W), x = static_cast<int>(v - static_cast<long>(y) * W);
    const double f0 = __ldg(rgb + 3 * v), f1 = __ldg(rgb + 3 * v + 1), f2 = __ldg(rgb + 3 * v + 2);
    int cnt = 0;
#pragma unroll
    for (int s = 0; s < T::S; ++s) {
      const int yy = y + T::dy(s), xx = x + T::dx(s);
      double wt = -1.0;
      if (yy < H && xx >= 0 && xx < W) {
        const long u = static_cast<long>(yy) * W + xx;
        const double a0 = f0 - __ldg(rgb + 3 * u), a1 = f1 - __ldg(rgb + 3 * u + 1), a2 = f2 - __ldg(rgb + 3 * u + 2);
        const double d2 = ((0.0 + a0 * a0) + a1 * a1) + a2 * a2;
        double e = d2 * inv_rgb;
        if (use_xy) e = e + static_cast<double>(T::dy(s) * T::dy(s) + T::dx(s) * T::dx(s)) * inv_xy;
        wt = exp(-e);
        cnt += wt >= kWeightFloor;
      }
      wc[v * T::S + s] = wt;
    }
    kept[v] = cnt;
  }
}

// Vertices without any kept incident edge (forward or backward).
template <int R>
__global__ void __launch_bounds__(kGridThreads) k_grid_isolated(int H, int W, const double* __restrict__ wc,
                                                               const int* __restrict__ kept, int* __restrict__ iso,
                                                               int* __restrict__ n_iso, int cap) {
  using T = Stencil<R>;
  const long n = static_cast<long>(H) * W;
  for (long v = static_cast<long>(blockIdx.x) * blockDim.x + threadIdx.x; v < n; v += static_cast<long>(gridDim.x) * blockDim.x) {
    if (kept[v] > 0) continue;
    const int y = static_cast<int>(v / W), x = static_cast<int>(v - static_cast<long>(y) * W);
    bool any = false;
#pragma unroll
    for (int s = 0; s < T::S; ++s) {
      const int yy = y - T::dy(s), xx = x - T::dx(s);
      if (yy >= 0 && xx >= 0 && xx < W) any |= wc[(static_cast<long>(yy) * W + xx) * T::S + s] >= kWeightFloor;
    }
    if (!any) {
      const int slot = atomicAdd(n_iso, 1);
      if (slot < cap) iso[slot] = static_cast<int>(v);
    }
  }
}

// Exclusive scan of kept[] in blocks of kGridThreads * 4 vertices: block sums.
__global__ void __launch_bounds__(kGridThreads) k_block_sums(long n, const int* __restrict__ kept, long* __restrict__ sums) {
  __shared__ long red[kGridThreads / 32];
  const long base = static_cast<long>(blockIdx.x) * kGridThreads * 4;
  long acc = 0;
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const long v = base + j * kGridThreads + threadIdx.x;
    if (v < n) acc += kept[v];
  }
#pragma unroll
  for (int o = 16; o >= 1; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    long s = 0;
    for (int w = 0; w < kGridThreads / 32; ++w) s += red[w];
    sums[blockIdx.x] = s;
  }
}

// Compacted edge list (pixel-major, slot order) and degrees in edge order.
template <int R>
__global__ void __launch_bounds__(kGridThreads) k_grid_edges(int H, int W, const double* __restrict__ wc,
                                                            const int* __restrict__ kept,
                                                            const long* __restrict__ block_off, int32_t* __restrict__ ei,
                                                            int32_t* __restrict__ ej, double* __restrict__ w,
                                                            double* __restrict__ degree) {
  using T = Stencil<R>;
  constexpr int CH = kGridThreads * 4;
  __shared__ long wsum[kGridThreads / 32];
  const long n = static_cast<long>(H) * W;
  const long base = static_cast<long>(blockIdx.x) * CH;
  // thread t owns vertices base + 4t .. base + 4t + 3 (contiguous, so the
  // block-local exclusive scan keeps pixel order)
  int c[4];
  long tsum = 0;
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const long v = base + 4 * threadIdx.x + j;
    c[j] = v < n ? kept[v] : 0;
    tsum += c[j];
  }
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  long incl = tsum;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const long t = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += t;
  }
  if (lane == 31) wsum[warp] = incl;
  __syncthreads();
  long woff = 0;
  for (int q = 0; q < warp; ++q) woff += wsum[q];
  long pos = block_off[blockIdx.x] + woff + incl - tsum;
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const long v = base + 4 * threadIdx.x + j;
    if (v >= n) break;
    const int y = static_cast<int>(v / W), x = static_cast<int>(v - static_cast<long>(y) * W);
    // edges owned by v, slot order
#pragma unroll
    for (int s = 0; s < T::S; ++s) {
      const double wt = wc[v * T::S + s];
      if (wt >= kWeightFloor) {
        ei[pos] = static_cast<int32_t>(v);
        ej[pos] = static_cast<int32_t>(v + T::dy(s) * W + T::dx(s));
        w[pos] = wt;
        ++pos;
      }
    }
    // degree: backward edges (u < v ascending = slot descending), then forward
    double dg = 0.0;
#pragma unroll
    for (int s = T::S - 1; s >= 0; --s) {
      const int yy = y - T::dy(s), xx = x - T::dx(s);
      if (yy >= 0 && xx >= 0 && xx < W) {
        const double wt = wc[(static_cast<long>(yy) * W + xx) * T::S + s];
        if (wt >= kWeightFloor) dg += wt;
      }
    }
#pragma unroll
    for (int s = 0; s < T::S; ++s) {
      const double wt = wc[v * T::S + s];
      if (wt >= kWeightFloor) dg += wt;
    }
    degree[v] = dg;
  }
}

}  // namespace pfe_dev

namespace pfe_host {

#define GCK(x)                                                                                      \
  do {                                                                                              \
    cudaError_t e_ = (x);                                                                           \
    if (e_ != cudaSuccess) throw Error(PFE_CUDA_ERROR, std::string(#x) + ": " + cudaGetErrorString(e_)); \
  } while (0)

namespace {

// Device buffers of one build, freed on every path.
struct GridBufs {
  cudaStream_t st = nullptr;
  std::vector<void*> ptrs;
  template <class T>
  T* alloc(size_t count) {
    void* p = nullptr;
    GCK(cudaMallocAsync(&p, std::max<size_t>(count, 1) * sizeof(T), st));
    ptrs.push_back(p);
    return static_cast<T*>(p);
  }
  ~GridBufs() {
    for (void* p : ptrs) cudaFreeAsync(p, st);
    if (st) {
      cudaStreamSynchronize(st);
      cudaStreamDestroy(st);
    }
  }
};

template <int R>
long build(int H, int W, const double* rgb, double sigma_rgb, double sigma_xy, int32_t* ei, int32_t* ej, double* w,
           double* degree) {
  using T = pfe_dev::Stencil<R>;
  constexpr int S = T::S;
  const long n = static_cast<long>(H) * W;
  GridBufs b;
  GCK(cudaStreamCreateWithFlags(&b.st, cudaStreamNonBlocking));
  int sms = 148, dev = 0;
  GCK(cudaGetDevice(&dev));
  GCK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  double* drgb = b.alloc<double>(static_cast<size_t>(n) * 3);
  double* wc = b.alloc<double>(static_cast<size_t>(n) * S);
  int* kept = b.alloc<int>(n);
  GCK(cudaMemcpyAsync(drgb, rgb, sizeof(double) * 3 * n, cudaMemcpyHostToDevice, b.st));
  const double inv_rgb = 1.0 / ((2.0 * sigma_rgb) * sigma_rgb);
  const bool use_xy = sigma_xy > 0.0;
  const double inv_xy = use_xy ? 1.0 / ((2.0 * sigma_xy) * sigma_xy) : 0.0;
  const int grid = static_cast<int>(std::min<long>((n + pfe_dev::kGridThreads - 1) / pfe_dev::kGridThreads, 16L * sms));
  pfe_dev::k_grid_candidates<R><<<grid, pfe_dev::kGridThreads, 0, b.st>>>(H, W, drgb, inv_rgb, inv_xy, use_xy, wc, kept);
  GCK(cudaGetLastError());
  // isolated vertices (step 3) -> host repair on their candidate weights
  constexpr int kIsoCap = 1 << 16;
  int* iso = b.alloc<int>(kIsoCap);
  int* n_iso = b.alloc<int>(1);
  GCK(cudaMemsetAsync(n_iso, 0, sizeof(int), b.st));
  pfe_dev::k_grid_isolated<R><<<grid, pfe_dev::kGridThreads, 0, b.st>>>(H, W, wc, kept, iso, n_iso, kIsoCap);
  GCK(cudaGetLastError());
  int niso = 0;
  GCK(cudaMemcpyAsync(&niso, n_iso, sizeof(int), cudaMemcpyDeviceToHost, b.st));
  GCK(cudaStreamSynchronize(b.st));
  if (niso > kIsoCap) throw Error(PFE_CONFIG_ERROR, "grid_graph: more than 65536 isolated pixels");
  if (niso > 0) {
    std::vector<int> iv(niso);
    GCK(cudaMemcpyAsync(iv.data(), iso, sizeof(int) * niso, cudaMemcpyDeviceToHost, b.st));
    GCK(cudaStreamSynchronize(b.st));
    std::sort(iv.begin(), iv.end());
    // every choice is made on the ORIGINAL candidate weights (two isolated
    // neighbours may pick the same edge; it is added once)
    struct Pick {
      long u;
      int s;
      double w;
    };
    std::vector<Pick> picks;
    for (int v : iv) {
      const int y = static_cast<int>(v / W), x = static_cast<int>(v % W);
      Pick best{-1, -1, -1.0};
      auto consider = [&](long u, int s) {
        double wt = 0.0;
        GCK(cudaMemcpyAsync(&wt, wc + u * S + s, sizeof(double), cudaMemcpyDeviceToHost, b.st));
        GCK(cudaStreamSynchronize(b.st));
        if (wt > best.w) best = {u, s, wt};  // strict: the first maximum in edge order wins
      };
      // candidates of v in edge order: backward (u ascending = slot
      // descending), then forward slots
      for (int s = S - 1; s >= 0; --s) {
        const int yy = y - T::dy(s), xx = x - T::dx(s);
        if (yy >= 0 && xx >= 0 && xx < W) consider(static_cast<long>(yy) * W + xx, s);
      }
      for (int s = 0; s < S; ++s) {
        const int yy = y + T::dy(s), xx = x + T::dx(s);
        if (yy < H && xx >= 0 && xx < W) consider(v, s);
      }
      if (best.u < 0) throw Error(PFE_CONFIG_ERROR, "grid_graph: pixel " + std::to_string(v) + " has no neighbour");
      picks.push_back(best);
    }
    std::sort(picks.begin(), picks.end(), [](const Pick& a, const Pick& c) { return a.u != c.u ? a.u < c.u : a.s < c.s; });
    picks.erase(std::unique(picks.begin(), picks.end(), [](const Pick& a, const Pick& c) { return a.u == c.u && a.s == c.s; }),
                picks.end());
    for (const Pick& pk : picks) {
      const double fixed = std::max(pk.w, pfe_dev::kWeightFloor);
      int kcount = 0;
      GCK(cudaMemcpyAsync(wc + pk.u * S + pk.s, &fixed, sizeof(double), cudaMemcpyHostToDevice, b.st));
      GCK(cudaMemcpyAsync(&kcount, kept + pk.u, sizeof(int), cudaMemcpyDeviceToHost, b.st));
      GCK(cudaStreamSynchronize(b.st));
      ++kcount;  // the candidate was not kept (its endpoints were isolated)
      GCK(cudaMemcpyAsync(kept + pk.u, &kcount, sizeof(int), cudaMemcpyHostToDevice, b.st));
      GCK(cudaStreamSynchronize(b.st));
    }
  }
  // block offsets (exclusive scan of the per-block kept counts, on the host)
  constexpr int CH = pfe_dev::kGridThreads * 4;
  const long nblk = (n + CH - 1) / CH;
  long* bsum = b.alloc<long>(nblk);
  pfe_dev::k_block_sums<<<static_cast<int>(nblk), pfe_dev::kGridThreads, 0, b.st>>>(n, kept, bsum);
  GCK(cudaGetLastError());
  std::vector<long> hs(nblk);
  GCK(cudaMemcpyAsync(hs.data(), bsum, sizeof(long) * nblk, cudaMemcpyDeviceToHost, b.st));
  GCK(cudaStreamSynchronize(b.st));
  long m = 0;
  for (long i = 0; i < nblk; ++i) {
    const long c = hs[i];
    hs[i] = m;
    m += c;
  }
  GCK(cudaMemcpyAsync(bsum, hs.data(), sizeof(long) * nblk, cudaMemcpyHostToDevice, b.st));
  int32_t* dei = b.alloc<int32_t>(m);
  int32_t* dej = b.alloc<int32_t>(m);
  double* dw = b.alloc<double>(m);
  double* ddeg = b.alloc<double>(n);
  pfe_dev::k_grid_edges<R><<<static_cast<int>(nblk), pfe_dev::kGridThreads, 0, b.st>>>(H, W, wc, kept, bsum, dei, dej,
                                                                                       dw, ddeg);
  GCK(cudaGetLastError());
  GCK(cudaMemcpyAsync(ei, dei, sizeof(int32_t) * m, cudaMemcpyDeviceToHost, b.st));
  GCK(cudaMemcpyAsync(ej, dej, sizeof(int32_t) * m, cudaMemcpyDeviceToHost, b.st));
  GCK(cudaMemcpyAsync(w, dw, sizeof(double) * m, cudaMemcpyDeviceToHost, b.st));
  GCK(cudaMemcpyAsync(degree, ddeg, sizeof(double) * n, cudaMemcpyDeviceToHost, b.st));
  GCK(cudaStreamSynchronize(b.st));
  return m;
}

}  // namespace

long grid_graph_device(int H, int W, const double* rgb, double sigma_rgb, int radius, double sigma_xy, int32_t* ei,
                       int32_t* ej, double* w, double* degree) {
  if (H < 1 || W < 1 || static_cast<long>(H) * W > 0x7fffffffL) throw Error(PFE_CONFIG_ERROR, "grid_graph: bad image size");
  if (!(sigma_rgb > 0.0)) throw Error(PFE_CONFIG_ERROR, "grid_graph: sigma_rgb must be > 0");
  if (static_cast<long>(H) * W < 2) throw Error(PFE_CONFIG_ERROR, "grid_graph: need at least 2 pixels");
  if (radius == 1) return build<1>(H, W, rgb, sigma_rgb, sigma_xy, ei, ej, w, degree);
  if (radius == 2) return build<2>(H, W, rgb, sigma_rgb, sigma_xy, ei, ej, w, degree);
  throw Error(PFE_CONFIG_ERROR, "grid_graph: radius must be 1 (8-neighbour) or 2 (5x5)");
}

}  // namespace pfe_host
