// Device side of the B200 PFE solver: graph topologies, row access helpers,
// deterministic block/grid reductions and the per-column PCG control block.
//
// Layout: every n x d iterate (Y, P, B, r, p, q, rhs) is a
// row-major [n][d] fp64 array, so one vertex's d columns are one contiguous
// 8d-byte row; edge arrays (split_b, split_s) are row-major [rows][d] where a
// row is one undirected edge (CSR topology: edge order as given; grid
// topology: the (vertex, forward stencil slot) pair owning the edge).
//
// Bitwise contract with the reference (proj/core/src): every elementwise
// formula and every sparse row sum is evaluated in the reference's operation
// order with separate multiply and add (the library is compiled with
// -fmad=false), so the only rounding differences against the CPU oracle are
// the orders of the BLAS-1 reductions (dot products and norms).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

namespace pfe_dev {

constexpr int kMaxD = 16;
constexpr int kBlock = 256;

enum ColStatus : int {
  kActive = 0,     // still iterating
  kConverged = 1,  // rel <= tol after >= 1 iteration
  kZeroRhs = 2,    // ||b|| == 0: x = 0, 0 iterations (pcg.cpp:50-53)
  kFailed = 3,     // curvature / NaN breakdown: x = x0, residual = inf (pcg.cpp:71-77, 106-111)
  kMaxIter = 4,    // hit max_iter without converging
  kConvInit = 5,   // initial residual already below tol: x = x0 (pcg.cpp:56-62)
};

struct PcgCol {
  double bnorm, rz, pq, alpha, beta, rel;
  int iters, status;
};

// Device-resident control block shared by the kernels of one solver.
struct Ctl {
  PcgCol col[kMaxD];   // per-column state after the latest SpMV prologue
  PcgCol colu[kMaxD];  // per-column state after the latest update prologue
  int iter;          // PCG iterations executed in the current solve
  int any_active;    // PCG loop condition
  int need_fix;      // finalize must patch some column of the result
  int nonfinite_y;   // sticky: NaN/Inf seen in Y (solver.cpp:94)
  int deficient;     // sticky: rank-deficient columns in the last projection (solver.cpp:31-39)
  int inner_count;   // inner iterations completed (index into the PCG log)
  unsigned int ticket;
  int log_cap;       // capacity (inner iterations) of the PCG log below
  double scalar[4];  // reduction outputs (objective, norms)
  int* log_iters;    // [log_cap][d] PCG iterations per column
  int* log_status;   // [log_cap][d] ColStatus per column
  double* log_rel;   // [log_cap][d] final relative residual per column
};

// --------------------------------------------------------------------------
// Column grouping: each thread owns V consecutive columns of one vertex row;
// TPV = D / V threads cooperate on a row.  d = 16 rows (128 B) are read as
// four 32-byte (256-bit, LDG.256) pieces: a warp instruction then gathers 8
// rows instead of 4, which halves the load instructions of the
// gather-bound general-graph kernels (C5; SpMV 495 -> 428 us in
// scripts/spmv_lab.py).  Other even D that divide 32-lane warps use 16-byte
// double2 accesses; the rest use one thread per row.
template <int D>
struct Cols {
  static constexpr int V = D == 16 ? 4 : ((D == 2 || D == 4 || D == 8) ? 2 : D);
  static constexpr int TPV = D / V;
};
// row gathers issued together per batch by the general-graph kernels
template <int V>
constexpr int kGatherBatch = V >= 4 ? 4 : 8;

template <int V>
struct Row {
  double a[V];
};

template <int V>
__device__ __forceinline__ Row<V> ldg_row(const double* __restrict__ p) {
  Row<V> r;
  if constexpr (V % 4 == 0) {
#pragma unroll
    for (int k = 0; k < V / 4; ++k)
      asm volatile("ld.global.nc.v4.f64 {%0,%1,%2,%3}, [%4];"
                   : "=d"(r.a[4 * k]), "=d"(r.a[4 * k + 1]), "=d"(r.a[4 * k + 2]), "=d"(r.a[4 * k + 3])
                   : "l"(p + 4 * k));
  } else if constexpr (V % 2 == 0) {
#pragma unroll
    for (int k = 0; k < V / 2; ++k) {
      const double2 t = __ldg(reinterpret_cast<const double2*>(p) + k);
      r.a[2 * k] = t.x;
      r.a[2 * k + 1] = t.y;
    }
  } else {
#pragma unroll
    for (int k = 0; k < V; ++k) r.a[k] = __ldg(p + k);
  }
  return r;
}

// Coherent load (data written earlier in the same kernel by the same thread,
// or buffers that are both read and written by the kernel).
template <int V>
__device__ __forceinline__ Row<V> ld_row(const double* p) {
  Row<V> r;
  if constexpr (V % 4 == 0) {
#pragma unroll
    for (int k = 0; k < V / 4; ++k)
      asm volatile("ld.global.v4.f64 {%0,%1,%2,%3}, [%4];"
                   : "=d"(r.a[4 * k]), "=d"(r.a[4 * k + 1]), "=d"(r.a[4 * k + 2]), "=d"(r.a[4 * k + 3])
                   : "l"(p + 4 * k)
                   : "memory");
  } else if constexpr (V % 2 == 0) {
#pragma unroll
    for (int k = 0; k < V / 2; ++k) {
      const double2 t = reinterpret_cast<const double2*>(p)[k];
      r.a[2 * k] = t.x;
      r.a[2 * k + 1] = t.y;
    }
  } else {
#pragma unroll
    for (int k = 0; k < V; ++k) r.a[k] = p[k];
  }
  return r;
}

template <int V>
__device__ __forceinline__ void st_row(double* p, const Row<V>& r) {
  if constexpr (V % 4 == 0) {
#pragma unroll
    for (int k = 0; k < V / 4; ++k)
      asm volatile("st.global.v4.f64 [%0], {%1,%2,%3,%4};" ::"l"(p + 4 * k), "d"(r.a[4 * k]), "d"(r.a[4 * k + 1]),
                   "d"(r.a[4 * k + 2]), "d"(r.a[4 * k + 3])
                   : "memory");
  } else if constexpr (V % 2 == 0) {
#pragma unroll
    for (int k = 0; k < V / 2; ++k) reinterpret_cast<double2*>(p)[k] = make_double2(r.a[2 * k], r.a[2 * k + 1]);
  } else {
#pragma unroll
    for (int k = 0; k < V; ++k) p[k] = r.a[k];
  }
}

// --------------------------------------------------------------------------
// Topologies.  Both expose, for a vertex v:
//   visitA(v, f(u, a))         : the row of A = (lambda/2) M^T M + (r/2) D in
//                                ascending column order, diagonal included
//                                (sparse.cpp:96-122 + spmv order 74-85);
//   visitE(v, f(u, w, slot, fwd)): incident edges in ascending edge index
//                                (the row order of M^T, sparse.cpp:52-72);
//                                fwd = v is the edge's first endpoint i.
// plus inv_diag(v) (pcg.cpp:15-20).

// Pixel grid with the (2R+1)^2 - 1 neighbourhood (R=1: 8-nbr, R=2: 5x5).
// Edge weights are stored per vertex for its S forward slots (the edges
// (v, v+off_s), off_s > 0), so an undirected edge has exactly one owner and
// the lexicographic edge order of the reference equals slot order.  A zero
// weight marks an absent edge (out of image or dropped by the builder).
template <int R>
struct GridTopo;

template <>
struct GridTopo<1> {
  static constexpr int S = 4;
  __device__ static constexpr int dy(int s) { return s == 0 ? 0 : 1; }
  __device__ static constexpr int dx(int s) { return s == 0 ? 1 : s - 2; }
};
template <>
struct GridTopo<2> {
  static constexpr int S = 12;
  __device__ static constexpr int dy(int s) { return s < 2 ? 0 : (s < 7 ? 1 : 2); }
  __device__ static constexpr int dx(int s) { return s < 2 ? s + 1 : (s < 7 ? s - 4 : s - 9); }
};

template <int R>
struct Grid {
  using T = GridTopo<R>;
  static constexpr int S = T::S;
  static constexpr bool kGrid = true;
  int n, H, W;
  double hl;  // lambda / 2
  const double* __restrict__ wf;        // [n][S]
  const double* __restrict__ diag;      // A_vv
  const double* __restrict__ invd;      // Jacobi
  // Rows whose vertices this solver owns (outputs and reductions); the rows
  // outside [row_lo, row_hi) are a halo copied from neighbouring row bands.
  // A single-GPU solver owns every row.
  int row_lo, row_hi;
  // [n][S] off-diagonal entries of A per forward slot, -((hl w) w), +0.0 for
  // an absent edge (tiled stencil kernels; set by the host after construction)
  const double* __restrict__ cf = nullptr;
  __device__ __forceinline__ double inv_diag(int v) const { return __ldg(invd + v); }
  __device__ __forceinline__ int vbeg() const { return row_lo * W; }
  __device__ __forceinline__ int vend() const { return row_hi * W; }

  template <class F>
  __device__ __forceinline__ void visitE(int v, F&& f) const {
    const int y = v / W, x = v - y * W;
#pragma unroll
    for (int s = S - 1; s >= 0; --s) {  // backward edges (u, v), u < v ascending
      const int yy = y - T::dy(s), xx = x - T::dx(s);
      if (yy >= 0 && xx >= 0 && xx < W) {
        const int u = v - T::dy(s) * W - T::dx(s);
        const long slot = static_cast<long>(u) * S + s;
        const double w = __ldg(wf + slot);
        if (w != 0.0) f(u, w, slot, false);
      }
    }
#pragma unroll
    for (int s = 0; s < S; ++s) {  // forward edges (v, u), u > v ascending
      const int yy = y + T::dy(s), xx = x + T::dx(s);
      if (yy < H && xx >= 0 && xx < W) {
        const int u = v + T::dy(s) * W + T::dx(s);
        const long slot = static_cast<long>(v) * S + s;
        const double w = __ldg(wf + slot);
        if (w != 0.0) f(u, w, slot, true);
      }
    }
  }

  template <class F>
  __device__ __forceinline__ void visitA(int v, F&& f) const {
    const int y = v / W, x = v - y * W;
#pragma unroll
    for (int s = S - 1; s >= 0; --s) {
      const int yy = y - T::dy(s), xx = x - T::dx(s);
      if (yy >= 0 && xx >= 0 && xx < W) {
        const int u = v - T::dy(s) * W - T::dx(s);
        const double w = __ldg(wf + static_cast<long>(u) * S + s);
        // (hl * (+-w)) * (-+w) == -((hl * w) * w) exactly (sparse.cpp:114)
        if (w != 0.0) f(u, -((hl * w) * w));
      }
    }
    f(v, __ldg(diag + v));
#pragma unroll
    for (int s = 0; s < S; ++s) {
      const int yy = y + T::dy(s), xx = x + T::dx(s);
      if (yy < H && xx >= 0 && xx < W) {
        const int u = v + T::dy(s) * W + T::dx(s);
        const double w = __ldg(wf + static_cast<long>(v) * S + s);
        if (w != 0.0) f(u, -((hl * w) * w));
      }
    }
  }
  // same interface as Csr::visitA_b / visitE_b (stencil rows need no batching)
  template <int B, class L, class F>
  __device__ __forceinline__ void visitA_b(int v, L&& load, F&& use) const {
    visitA(v, [&](int u, double av) { use(av, load(u)); });
  }
  template <int B, class L, class F>
  __device__ __forceinline__ void visitE_b(int v, L&& load, F&& use) const {
    visitE(v, [&](int u, double w, long slot, bool fwd) { use(u, w, slot, fwd, load(u, slot)); });
  }
};

// General graph (k-NN, arbitrary edge lists): explicit CSR of A (diagonal in
// its sorted position, duplicates pre-summed in edge order exactly like
// csr_from_triplets) and an incidence list sorted by edge index.
struct Csr {
  static constexpr bool kGrid = false;
  int n;
  const int* __restrict__ aptr;
  const int* __restrict__ acol;
  const double* __restrict__ aval;
  const int* __restrict__ iptr;
  const int* __restrict__ inbr;  // incidence: neighbour (device row)
  const int* __restrict__ ieid;  // edge id << 1 | [this vertex is the edge's first endpoint]
  const double* __restrict__ iw;
  const double* __restrict__ invd;
  int vb, ve;  // owned vertex range
  __device__ __forceinline__ double inv_diag(int v) const { return __ldg(invd + v); }
  __device__ __forceinline__ int vbeg() const { return vb; }
  __device__ __forceinline__ int vend() const { return ve; }

  template <class F>
  __device__ __forceinline__ void visitA(int v, F&& f) const {
    const int b = __ldg(aptr + v), e = __ldg(aptr + v + 1);
    for (int k = b; k < e; ++k) f(__ldg(acol + k), __ldg(aval + k));
  }
  template <class F>
  __device__ __forceinline__ void visitE(int v, F&& f) const {
    const int b = __ldg(iptr + v), e = __ldg(iptr + v + 1);
    for (int k = b; k < e; ++k) {
      const int code = __ldg(ieid + k);  // edge id << 1 | [v is the first endpoint]
      f(__ldg(inbr + k), __ldg(iw + k), static_cast<long>(code >> 1), (code & 1) != 0);
    }
  }
  // Batched visits for gather-bound k-NN rows: a batch's B gathers load(...)
  // (and its weights) are all issued before use(...) consumes them in row /
  // edge order (the summation order is unchanged; only the memory round
  // trips overlap).  The neighbour indices of the next batch are loaded
  // before the current batch is consumed, so each batch costs one dependent
  // round trip (its gathers), not two.
  template <int B, class L, class F>
  __device__ __forceinline__ void visitA_b(int v, L&& load, F&& use) const {
    const int b = __ldg(aptr + v), e = __ldg(aptr + v + 1);
    using G = decltype(load(0));
    int cu[B];
#pragma unroll
    for (int j = 0; j < B; ++j) cu[j] = b + j < e ? __ldg(acol + b + j) : -1;
    for (int k0 = b; k0 < e; k0 += B) {
      G g[B];
      double av[B];
#pragma unroll
      for (int j = 0; j < B; ++j)
        if (cu[j] >= 0) {
          g[j] = load(cu[j]);
          av[j] = __ldg(aval + k0 + j);
        }
      int cn[B];
#pragma unroll
      for (int j = 0; j < B; ++j) cn[j] = k0 + B + j < e ? __ldg(acol + k0 + B + j) : -1;
#pragma unroll
      for (int j = 0; j < B; ++j)
        if (cu[j] >= 0) use(av[j], g[j]);
#pragma unroll
      for (int j = 0; j < B; ++j) cu[j] = cn[j];
    }
  }
  template <int B, class L, class F>
  __device__ __forceinline__ void visitE_b(int v, L&& load, F&& use) const {
    const int b = __ldg(iptr + v), e = __ldg(iptr + v + 1);
    using G = decltype(load(0, 0L));
    int cu[B], cc[B];
#pragma unroll
    for (int j = 0; j < B; ++j) {
      const bool ok = b + j < e;
      cu[j] = ok ? __ldg(inbr + b + j) : -1;
      cc[j] = ok ? __ldg(ieid + b + j) : 0;
    }
    for (int k0 = b; k0 < e; k0 += B) {
      G g[B];
      double cw[B];
#pragma unroll
      for (int j = 0; j < B; ++j)
        if (cu[j] >= 0) {
          g[j] = load(cu[j], static_cast<long>(cc[j] >> 1));
          cw[j] = __ldg(iw + k0 + j);
        }
      int un[B], cn[B];
#pragma unroll
      for (int j = 0; j < B; ++j) {
        const bool ok = k0 + B + j < e;
        un[j] = ok ? __ldg(inbr + k0 + B + j) : -1;
        cn[j] = ok ? __ldg(ieid + k0 + B + j) : 0;
      }
#pragma unroll
      for (int j = 0; j < B; ++j)
        if (cu[j] >= 0) use(cu[j], cw[j], static_cast<long>(cc[j] >> 1), (cc[j] & 1) != 0, g[j]);
#pragma unroll
      for (int j = 0; j < B; ++j) {
        cu[j] = un[j];
        cc[j] = cn[j];
      }
    }
  }
};

// --------------------------------------------------------------------------
// Deterministic reductions.  Each thread holds acc[NQ][V] for its column
// group g = lane % TPV.  Warp butterfly over lanes with equal g, then warps
// combined in fixed order through shared memory; block b writes
// partials[b][NQ][D].  The last block to finish (ticket) reduces the block
// partials in a fixed order and runs the scalar epilogue.
template <int NQ, int D, int V, int NT = kBlock>
__device__ __forceinline__ void block_reduce_store(double (&acc)[NQ][V], double* __restrict__ partials) {
  constexpr int TPV = D / V;
  __shared__ double red[NT / 32][NQ][D];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int o = 16; o >= TPV; o >>= 1) {
#pragma unroll
    for (int q = 0; q < NQ; ++q)
#pragma unroll
      for (int k = 0; k < V; ++k) acc[q][k] += __shfl_xor_sync(0xffffffffu, acc[q][k], o);
  }
  if (lane < TPV) {
#pragma unroll
    for (int q = 0; q < NQ; ++q)
#pragma unroll
      for (int k = 0; k < V; ++k) red[warp][q][lane * V + k] = acc[q][k];
  }
  __syncthreads();
  if (threadIdx.x < NQ * D) {
    const int q = threadIdx.x / D, c = threadIdx.x - q * D;
    double s = 0.0;
#pragma unroll
    for (int w = 0; w < NT / 32; ++w) s += red[w][q][c];
    partials[static_cast<long>(q * D + c) * gridDim.x + blockIdx.x] = s;  // pair-major
  }
}

// Returns true in exactly one block (the last to arrive); that block's
// shared `out[NQ][D]` then holds the grid totals.  The final reduction uses
// every thread of the last block: thread t owns blocks t, t+256, ... of each
// (quantity, column) pair (coalesced: partials are stored pair-major), then a
// warp butterfly and a fixed-order sum over warps — deterministic.
template <int NQ, int D, int NT = kBlock>
__device__ __forceinline__ bool grid_reduce_last(const double* partials, Ctl* ctl, double (&out)[NQ][D]) {
  constexpr int P = NQ * D;
  constexpr int CH = P < 16 ? P : 16;  // pairs reduced per pass
  __shared__ bool last;
  __shared__ double wsum[NT / 32][CH];
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned t = atomicAdd(&ctl->ticket, 1u);
    last = (t == gridDim.x - 1);
  }
  __syncthreads();
  if (!last) return false;
  __threadfence();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int nb = gridDim.x;
  for (int base = 0; base < P; base += CH) {
    double acc[CH];
#pragma unroll
    for (int k = 0; k < CH; ++k) acc[k] = 0.0;
    for (int b = threadIdx.x; b < nb; b += NT) {
#pragma unroll
      for (int k = 0; k < CH; ++k)
        if (base + k < P) acc[k] += __ldcg(partials + static_cast<long>(base + k) * nb + b);
    }
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1)
#pragma unroll
      for (int k = 0; k < CH; ++k) acc[k] += __shfl_xor_sync(0xffffffffu, acc[k], o);
    if (lane == 0)
#pragma unroll
      for (int k = 0; k < CH; ++k) wsum[warp][k] = acc[k];
    __syncthreads();
    if (threadIdx.x < CH && base + threadIdx.x < P) {
      double s = 0.0;
#pragma unroll
      for (int w = 0; w < NT / 32; ++w) s += wsum[w][threadIdx.x];
      const int pr = base + threadIdx.x;
      out[pr / D][pr % D] = s;
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) ctl->ticket = 0;
  return true;
}

// Soft threshold, exactly solver.cpp:21-24.
__device__ __forceinline__ double shrink1(double x, double gamma) {
  const double mag = fabs(x) - gamma;
  return mag > 0.0 ? (x > 0.0 ? mag : -mag) : 0.0;
}

}  // namespace pfe_dev
