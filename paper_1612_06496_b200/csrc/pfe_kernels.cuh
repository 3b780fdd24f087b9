// Hot-path kernels of the PFE nested Bregman loop (templates; instantiated per
// topology and embedding dimension in pfe_kernels_*.cu).
//
//   k_pcg_init    r = b - A x0, p = D^-1 r, partials of ||b||^2, r.r, r.z  (pcg.cpp:49-66)
//   k_pcg_spmv    [stop test, beta] p = D^-1 r + beta p, q = A p, partial p.q
//                                                              (pcg.cpp:56-62, 68-72, 79-88)
//   k_pcg_update  [alpha] x += alpha p, r -= alpha q, partials r.r, r.D^-1 r, NaN
//                                                              (pcg.cpp:71-78)
//   k_pcg_finalize  per-column result selection + PCG log      (pcg.cpp:50-53, 56-62, 101-112)
//   k_sb_pass     M Y, shrink, Bregman b update, next rhs       (solver.cpp:83-84, 96-98)
//   k_rhs_quad / k_rhs_from_state                               (solver.cpp:79-84)
//   k_objective   sum |M Y|                                     (solver.cpp:14-17)
//
// All d columns are iterated together; each column keeps its own alpha,
// beta, residual and stopping state exactly as solve_multi runs them one by
// one (pcg.cpp:94-114).
//
// Reductions are consumer-side: a kernel only writes its per-block partial
// sums; every block of the NEXT kernel reduces them (same fixed order in
// every block, so all blocks derive bit-identical scalars) while its own data
// loads are in flight, runs the scalar logic of pcg.cpp (alpha, beta,
// convergence, breakdown) in warp 0, and block 0 persists the per-column
// state to the control block.  No kernel has a serial last-block tail.  The
// stop decision for iteration k is taken by the SpMV of iteration k+1, which
// then exits immediately and clears the CUDA-graph loop condition.
#pragma once

#include "pfe_device.cuh"

namespace pfe_dev {

struct PcgArgs {
  const double* x0;    // Y (warm start), row-major [n][D]
  double* x;           // Y2: solve result buffer
  const double* rhs;   // right-hand side (may alias r)
  double* r;
  double* pbuf[2];     // ping-pong search directions
  double* q;
  Ctl* ctl;
  double* part_a;      // partials of init / update (3 x D pairs, pair-major)
  double* part_b;      // partials of spmv (D pairs)
  const double* rd_a;  // what the consumers reduce: part_a / part_b, or the
  const double* rd_b;  // per-rank totals gathered from every row band
  int nb_init;         // block counts of the producers (consumers reduce that many)
  int nb_update;
  int nb_spmv;
  double tol;
  int max_iter;
  cudaGraphConditionalHandle cond;  // loop handle when running inside a graph
  int use_cond;
  // Iteration parity, fixed per launch so no buffer address depends on the
  // device control block: 0 = first iteration (p from init in pbuf[0],
  // x read from x0), 1 = odd iteration >= 3 (p' -> pbuf[0], p_old = pbuf[1]),
  // 2 = even iteration (p' -> pbuf[1], p_old = pbuf[0]).
  int phase;
  // Row-band solvers: part_a / part_b hold the per-rank totals gathered from
  // every band ([rank][pair], nb = ranks) instead of this grid's block partials.
  int rank_major;
  int skip_pdir;  // host side: pcg_spmv does not launch the CSR direction pass
  // IC(0): z = M^-1 r of the latest update (the direction pass then forms
  // p' = z + beta p, pcg.cpp:86-88); null: Jacobi z = D^-1 r on the fly
  const double* zbuf;
  // Producer-side totals (single-domain solvers): the last block of each
  // producer reduces the block partials in a fixed order and writes the NQ*D
  // totals to tot_a (init / update) or tot_b (spmv); consumers then read
  // those (rd_* = tot_*, nb = 1) instead of every block re-reducing all
  // partials, which costs nb^2 loads (dominant for 10^3-block grids).
  double* tot_a;
  double* tot_b;
  int totals;
};

__host__ __device__ __forceinline__ int pcg_phase(int it) { return it == 1 ? 0 : ((it & 1) ? 1 : 2); }
__device__ __forceinline__ double* pcg_pnew(const PcgArgs& a) { return a.phase == 2 ? a.pbuf[1] : a.pbuf[0]; }
__device__ __forceinline__ const double* pcg_pold(const PcgArgs& a) { return a.phase == 1 ? a.pbuf[1] : a.pbuf[0]; }

constexpr double kInf = __builtin_huge_val();

// Producer epilogue: block partials, then (a.totals) the grid totals written
// by the last block to arrive (deterministic fixed-order reduction).
template <int NQ, int D, int V, int NT = kBlock>
__device__ __forceinline__ void store_partials(const PcgArgs& a, double (&acc)[NQ][V], double* __restrict__ partials,
                                               double* __restrict__ tot) {
  block_reduce_store<NQ, D, V, NT>(acc, partials);
  if (a.totals) {
    __shared__ double out[NQ][D];
    if (grid_reduce_last<NQ, D, NT>(partials, a.ctl, out) && threadIdx.x < NQ * D)
      tot[threadIdx.x] = out[threadIdx.x / D][threadIdx.x % D];
  }
}

// Block-wide fixed-order reduction of a producer's pair-major partials
// (nb blocks x NQ*D pairs) into shared out[NQ][D]; all NT threads take part.
template <int NQ, int D, int NT>
__device__ __forceinline__ void reduce_partials(const double* __restrict__ part, int nb, double (&out)[NQ][D],
                                                bool rank_major = false) {
  constexpr int P = NQ * D;
  constexpr int CH = P < 16 ? P : 16;
  __shared__ double wsum[NT / 32][CH];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int base = 0; base < P; base += CH) {
    double acc[CH];
#pragma unroll
    for (int k = 0; k < CH; ++k) acc[k] = 0.0;
    for (int b = threadIdx.x; b < nb; b += NT) {
#pragma unroll
      for (int k = 0; k < CH; ++k)
        if (base + k < P)
          acc[k] += __ldcg(part + (rank_major ? static_cast<long>(b) * P + base + k : static_cast<long>(base + k) * nb + b));
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
}

// Column state is double-buffered in the control block: SpMV prologues read
// Ctl::colu (written by the previous update) and write Ctl::col; update
// prologues read Ctl::col and write Ctl::colu.

// Shared per-block view of the column state after a prologue.
template <int D>
struct ColView {
  double coef[D];  // beta (spmv) or alpha (update); 0 for inactive columns
  int act[D];
  int any;
};

// SpMV prologue: the stop test of the previous iteration (or the initial
// residual test after init) and beta.  Mirrors pcg.cpp:50-62 (init) and
// pcg.cpp:75-88 (after an update).  Returns whether any column is active.
template <int D, int NT>
__device__ __forceinline__ bool spmv_prologue(const PcgArgs& a, ColView<D>& cv) {
  __shared__ double tot[3][D];
  const bool first = a.phase == 0;
  reduce_partials<3, D, NT>(a.rd_a, first ? a.nb_init : a.nb_update, tot, a.rank_major != 0);
  if (threadIdx.x < 32) {
    const int j = threadIdx.x;
    const int done = a.ctl->iter;  // PCG iterations completed so far
    bool act = false;
    if (j < D) {
      PcgCol col;
      if (first) {  // tot = ||b||^2, r.r, r.z of the initial residual
        col = PcgCol{};
        col.bnorm = sqrt(tot[0][j]);
        if (col.bnorm == 0.0) {
          col.status = kZeroRhs;
          col.rel = 0.0;
        } else {
          col.rel = sqrt(tot[1][j]) / col.bnorm;
          if (col.rel <= a.tol) {
            col.status = kConvInit;
          } else {
            col.status = kActive;
            col.rz = tot[2][j];
          }
        }
      } else {  // tot = r.r, r.D^-1 r, NaN count of iteration `done`
        col = a.ctl->colu[j];
        if (col.status == kActive) {
          if (tot[2][j] > 0.0) {  // pcg.cpp:75
            col.status = kFailed;
            col.iters = 0;
            col.rel = kInf;
          } else {
            col.rel = sqrt(tot[0][j]) / col.bnorm;
            col.iters = done;
            if (col.rel <= a.tol) {
              col.status = kConverged;
            } else if (done >= a.max_iter) {
              col.status = kMaxIter;
            } else {
              col.beta = tot[1][j] / col.rz;
              col.rz = tot[1][j];
            }
          }
        }
      }
      act = col.status == kActive;
      cv.act[j] = act;
      cv.coef[j] = act ? col.beta : 0.0;
      if (blockIdx.x == 0) a.ctl->col[j] = col;
    }
    const bool any = __any_sync(0xffffffffu, act);
    if (j == 0) {
      cv.any = any;
      if (blockIdx.x == 0) {
        a.ctl->any_active = any;
        if (first) a.ctl->iter = 0;
        if (!any && a.use_cond) cudaGraphSetConditional(a.cond, 0u);
      }
    }
  }
  __syncthreads();
  return cv.any != 0;
}

// Update prologue: alpha = rz / p.q with the curvature check (pcg.cpp:70-72).
template <int D, int NT>
__device__ __forceinline__ bool update_prologue(const PcgArgs& a, ColView<D>& cv) {
  __shared__ double tot[1][D];
  const int active = a.ctl->any_active;  // written by this iteration's SpMV
  if (!active) return false;             // uniform across the grid
  reduce_partials<1, D, NT>(a.rd_b, a.nb_spmv, tot, a.rank_major != 0);
  if (threadIdx.x < 32) {
    const int j = threadIdx.x;
    bool act = false;
    if (j < D) {
      PcgCol col = a.ctl->col[j];
      if (col.status == kActive) {
        const double pq = tot[0][j];
        col.pq = pq;
        if (!(pq > 0.0) || !isfinite(pq)) {
          col.status = kFailed;
          col.iters = 0;
          col.rel = kInf;
        } else {
          col.alpha = col.rz / pq;
        }
      }
      // the state is double-buffered (col -> colu) so no block reads a
      // column another block of the same kernel has already advanced
      if (blockIdx.x == 0) a.ctl->colu[j] = col;
      act = col.status == kActive;
      cv.act[j] = act;
      cv.coef[j] = act ? col.alpha : 0.0;
    }
    const bool any = __any_sync(0xffffffffu, act);
    if (j == 0) {
      cv.any = any;
      if (blockIdx.x == 0) a.ctl->iter = a.ctl->iter + 1;
    }
  }
  __syncthreads();
  return true;  // even with every column failed, write (inert) partials
}

// Vertex rows of a gather-bound kernel: grid-stride order, so block b takes
// chunks b, b + nb, ... of blockDim / TPV consecutive vertices and the whole
// GPU sweeps one window of the storage order at a time.  For general graphs
// in breadth-first storage order the rows gathered at any moment then come
// from a window a few MB wide that stays in L2 (C5 SpMV: DRAM reads 1.34 GB
// -> 0.45 GB = compulsory, 429 -> 319 us, scripts/spmv_lab.py), and an edge
// row read by both endpoints is often still in L2 for the second read
// (split-Bregman pass).  kContig (one contiguous range per block; more L1
// reuse, but the whole vector is gathered at once and misses L2) is kept
// for comparison.
template <int TPV, bool kContig = false, class Topo>
__device__ __forceinline__ void row_range(const Topo& topo, long& e0, long& e1, long& step) {
  const long first = static_cast<long>(topo.vbeg()) * TPV, total = static_cast<long>(topo.vend()) * TPV;
  if constexpr (Topo::kGrid || !kContig) {
    e0 = first + static_cast<long>(blockIdx.x) * blockDim.x + threadIdx.x;
    e1 = total;
    step = static_cast<long>(gridDim.x) * blockDim.x;
  } else {
    const long cnt = total - first;
    const long per = ((cnt + gridDim.x - 1) / gridDim.x + blockDim.x - 1) / blockDim.x * blockDim.x;
    e0 = first + static_cast<long>(blockIdx.x) * per + threadIdx.x;
    e1 = first + static_cast<long>(blockIdx.x + 1) * per;
    e1 = e1 < total ? e1 : total;
    step = blockDim.x;
  }
}

// ---------------------------------------------------------------- PCG init --
template <int D, class Topo>
__global__ void __launch_bounds__(kBlock, 2) k_pcg_init(Topo topo, PcgArgs a) {
  constexpr int V = Cols<D>::V, TPV = Cols<D>::TPV;
  double acc[3][V] = {};
  long e0, e1, step;
  row_range<TPV>(topo, e0, e1, step);
  for (long e = e0; e < e1; e += step) {
    const int v = static_cast<int>(e / TPV);
    const int c0 = static_cast<int>(e - static_cast<long>(v) * TPV) * V;
    double ax[V] = {};
    topo.template visitA_b<kGatherBatch<V>>(
        v, [&](int u) { return ldg_row<V>(a.x0 + static_cast<long>(u) * D + c0); },
        [&](double av, const Row<V>& xu) {
#pragma unroll
          for (int k = 0; k < V; ++k) ax[k] += av * xu.a[k];
        });
    const Row<V> b = ld_row<V>(a.rhs + static_cast<long>(v) * D + c0);
    const double id = topo.inv_diag(v);
    Row<V> r, z;
#pragma unroll
    for (int k = 0; k < V; ++k) {
      r.a[k] = b.a[k] - ax[k];
      z.a[k] = id * r.a[k];
      acc[0][k] += b.a[k] * b.a[k];
      acc[1][k] += r.a[k] * r.a[k];
      acc[2][k] += r.a[k] * z.a[k];
    }
    st_row<V>(a.r + static_cast<long>(v) * D + c0, r);
    st_row<V>(a.pbuf[0] + static_cast<long>(v) * D + c0, z);
  }
  store_partials<3, D, V>(a, acc, a.part_a, a.tot_a);
}

// Gathers rows (ghost exchange packing).
template <int D>
__global__ void k_pack_rows(const double* __restrict__ src, const int* __restrict__ rows, int cnt,
                            double* __restrict__ dst) {
  const long total = static_cast<long>(cnt) * D, stride = static_cast<long>(gridDim.x) * blockDim.x;
  for (long e = static_cast<long>(blockIdx.x) * blockDim.x + threadIdx.x; e < total; e += stride) {
    const long i = e / D;
    dst[e] = src[static_cast<long>(__ldg(rows + i)) * D + (e - i * D)];
  }
}

// ----------------------------------------------- PCG direction (CSR rows) --
// [stop test, beta] p' = D^-1 r + beta p_old for every vertex (pcg.cpp:86-88),
// ahead of k_pcg_spmv on general graphs: their SpMV then gathers p' once per
// neighbour instead of re-forming it from r and p_old.  The SpMV repeats the
// same prologue (same partials, same decisions; its writes are idempotent).
template <int D, class Topo>
__global__ void __launch_bounds__(kBlock) k_pcg_pdir(Topo topo, PcgArgs a) {
  constexpr int V = Cols<D>::V, TPV = Cols<D>::TPV;
  __shared__ ColView<D> cv;
  if (!spmv_prologue<D, kBlock>(a, cv)) return;
  const int gfirst = (static_cast<int>(threadIdx.x) % TPV) * V;
  double beta[V];
#pragma unroll
  for (int k = 0; k < V; ++k) beta[k] = cv.coef[gfirst + k];
  double* pnew = pcg_pnew(a);
  const double* pold = pcg_pold(a);
  long e0, e1, step;
  row_range<TPV>(topo, e0, e1, step);
  for (long e = e0; e < e1; e += step) {
    const int v = static_cast<int>(e / TPV);
    const int c0 = static_cast<int>(e - static_cast<long>(v) * TPV) * V;
    const Row<V> po = ldg_row<V>(pold + static_cast<long>(v) * D + c0);
    Row<V> pu;
    if (a.zbuf) {
      const Row<V> zv = ldg_row<V>(a.zbuf + static_cast<long>(v) * D + c0);
#pragma unroll
      for (int k = 0; k < V; ++k) pu.a[k] = zv.a[k] + beta[k] * po.a[k];
    } else {
      const Row<V> rv = ldg_row<V>(a.r + static_cast<long>(v) * D + c0);
      const double id = topo.inv_diag(v);
#pragma unroll
      for (int k = 0; k < V; ++k) pu.a[k] = id * rv.a[k] + beta[k] * po.a[k];
    }
    st_row<V>(pnew + static_cast<long>(v) * D + c0, pu);
  }
}

// ------------------------------------------------------- PCG SpMV (+ p update)
template <int D, class Topo>
__global__ void __launch_bounds__(kBlock, 2) k_pcg_spmv(Topo topo, PcgArgs a) {
  constexpr int V = Cols<D>::V, TPV = Cols<D>::TPV;
  __shared__ ColView<D> cv;
  if (!spmv_prologue<D, kBlock>(a, cv)) return;
  const bool first = a.phase == 0;
  const int gfirst = (static_cast<int>(threadIdx.x) % TPV) * V;
  double beta[V];
#pragma unroll
  for (int k = 0; k < V; ++k) beta[k] = cv.coef[gfirst + k];
  double* pnew = pcg_pnew(a);
  const double* pold = pcg_pold(a);
  double acc[1][V] = {};
  long e0, e1, step;
  row_range<TPV>(topo, e0, e1, step);
  for (long e = e0; e < e1; e += step) {
    const int v = static_cast<int>(e / TPV);
    const int c0 = static_cast<int>(e - static_cast<long>(v) * TPV) * V;
    double q[V] = {};
    Row<V> pv;
    if (first || !Topo::kGrid) {
      // CSR rows: p' was formed for every vertex by k_pcg_pdir (one gather per
      // neighbour instead of three); first iteration: p = z from the init
      pv = ldg_row<V>(pnew + static_cast<long>(v) * D + c0);
      topo.template visitA_b<kGatherBatch<V>>(
          v, [&](int u) { return ldg_row<V>(pnew + static_cast<long>(u) * D + c0); },
          [&](double av, const Row<V>& pu) {
#pragma unroll
            for (int k = 0; k < V; ++k) q[k] += av * pu.a[k];
          });
    } else {
      // p_u = z_u + beta p_u with z_u = D^-1_u r_u, recomputed identically
      // for every row that reads vertex u (pcg.cpp:86-88).
      auto pdir = [&](int u) {
        const Row<V> ru = ldg_row<V>(a.r + static_cast<long>(u) * D + c0);
        const Row<V> po = ldg_row<V>(pold + static_cast<long>(u) * D + c0);
        const double id = topo.inv_diag(u);
        Row<V> pu;
#pragma unroll
        for (int k = 0; k < V; ++k) pu.a[k] = id * ru.a[k] + beta[k] * po.a[k];
        return pu;
      };
      pv = pdir(v);
      topo.visitA(v, [&](int u, double av) {
        const Row<V> pu = pdir(u);
#pragma unroll
        for (int k = 0; k < V; ++k) q[k] += av * pu.a[k];
      });
      st_row<V>(pnew + static_cast<long>(v) * D + c0, pv);
    }
    Row<V> qv;
#pragma unroll
    for (int k = 0; k < V; ++k) {
      qv.a[k] = q[k];
      acc[0][k] += pv.a[k] * q[k];
    }
    st_row<V>(a.q + static_cast<long>(v) * D + c0, qv);
  }
  store_partials<1, D, V>(a, acc, a.part_b, a.tot_b);
}

// ----------------------------------------------------------- PCG update -----
template <int D, class Topo>
__global__ void __launch_bounds__(kBlock) k_pcg_update(Topo topo, PcgArgs a) {
  constexpr int V = Cols<D>::V, TPV = Cols<D>::TPV;
  __shared__ ColView<D> cv;
  const int gfirst = (static_cast<int>(threadIdx.x) % TPV) * V;
  const double* xsrc = a.phase == 0 ? a.x0 : a.x;
  const double* pin = pcg_pnew(a);
  const long total = static_cast<long>(topo.vend()) * TPV;
  const long stride = static_cast<long>(gridDim.x) * blockDim.x;
  long e = static_cast<long>(topo.vbeg()) * TPV + static_cast<long>(blockIdx.x) * blockDim.x + threadIdx.x;
  // first item's data is loaded before the prologue's reduction so both
  // memory round trips overlap
  Row<V> x{}, r{}, p{}, q{};
  double id = 0.0;
  auto load = [&](long ee) {
    const int v = static_cast<int>(ee / TPV);
    const long o = static_cast<long>(v) * D + static_cast<int>(ee - static_cast<long>(v) * TPV) * V;
    x = ld_row<V>(xsrc + o);
    r = ld_row<V>(a.r + o);
    p = ldg_row<V>(pin + o);
    q = ldg_row<V>(a.q + o);
    id = topo.inv_diag(v);
  };
  if (e < total) load(e);
  if (!update_prologue<D, kBlock>(a, cv)) return;
  double alpha[V];
  bool act[V];
#pragma unroll
  for (int k = 0; k < V; ++k) {
    act[k] = cv.act[gfirst + k] != 0;
    alpha[k] = cv.coef[gfirst + k];
  }
  double acc[3][V] = {};
  for (; e < total; e += stride) {
    const int v = static_cast<int>(e / TPV);
    const long o = static_cast<long>(v) * D + static_cast<int>(e - static_cast<long>(v) * TPV) * V;
#pragma unroll
    for (int k = 0; k < V; ++k) {
      if (act[k]) {
        x.a[k] = x.a[k] + alpha[k] * p.a[k];
        r.a[k] = r.a[k] - alpha[k] * q.a[k];
        if (!isfinite(x.a[k])) acc[2][k] += 1.0;
      }
      const double z = id * r.a[k];
      acc[0][k] += r.a[k] * r.a[k];
      acc[1][k] += r.a[k] * z;
    }
    st_row<V>(a.x + o, x);
    st_row<V>(a.r + o, r);
    if (e + stride < total) load(e + stride);
  }
  store_partials<3, D, V>(a, acc, a.part_a, a.tot_a);
}

// --------------------------------------------------------- PCG finalize -----
// Columns that never iterated (zero rhs / converged at x0) or that broke down
// take their value from x0 / zero; every other column is already in x.  Also
// appends the per-column report of this solve to the PCG log.
template <int D>
__global__ void __launch_bounds__(kBlock) k_pcg_finalize(int n, const double* __restrict__ x0, double* x, Ctl* ctl) {
  __shared__ int mode[D];  // 0 keep, 1 from x0, 2 zero
  __shared__ int need;
  if (threadIdx.x < 32) {
    const int j = threadIdx.x;
    const bool never_iterated = ctl->iter == 0;
    int md = 0;
    if (j < D) {
      const PcgCol col = ctl->col[j];
      md = col.status == kZeroRhs ? 2 : ((col.status == kConvInit || col.status == kFailed || never_iterated) ? 1 : 0);
      mode[j] = md;
      if (blockIdx.x == 0) {
        const int idx = ctl->inner_count;
        if (idx < ctl->log_cap) {
          ctl->log_iters[static_cast<long>(idx) * D + j] = col.iters;
          ctl->log_status[static_cast<long>(idx) * D + j] = col.status;
          ctl->log_rel[static_cast<long>(idx) * D + j] = col.rel;
        }
      }
    }
    const bool anyfix = __any_sync(0xffffffffu, md != 0);
    if (j == 0) {
      need = anyfix;
      if (blockIdx.x == 0) ctl->inner_count = ctl->inner_count + 1;  // no other block reads it
    }
  }
  __syncthreads();
  if (!need) return;
  const long total = static_cast<long>(n) * D;
  const long stride = static_cast<long>(gridDim.x) * blockDim.x;
  for (long e = static_cast<long>(blockIdx.x) * blockDim.x + threadIdx.x; e < total; e += stride) {
    const int j = static_cast<int>(e % D);
    if (mode[j] == 1) x[e] = x0[e];
    else if (mode[j] == 2) x[e] = 0.0;
  }
}

// Reduces one grid's block partials (pair-major, nb blocks) to NQ*D totals;
// row-band solvers then gather these totals from every band so all bands
// derive the same PCG scalars (reduced in rank order).
template <int NQ, int D>
__global__ void __launch_bounds__(kBlock) k_local_totals(const double* part, int nb, double* out) {
  __shared__ double tot[NQ][D];
  reduce_partials<NQ, D, kBlock>(part, nb, tot);
  if (threadIdx.x < NQ * D) out[threadIdx.x] = tot[threadIdx.x / D][threadIdx.x % D];
}

// ----------------------------------------------------- split-Bregman pass ---
struct SbArgs {
  const double* y;      // new Y
  const double* b_old;  // null => zero
  double* b_new;
  double* s_out;        // null => do not materialize split_s
  const double* rq;     // rhs_quad
  double* rhs;          // null => do not produce the next rhs
  double hl;            // lambda / 2
  double gamma;         // 1 / lambda
  Ctl* ctl;
  int prefetch;         // general graphs: L2-prefetch a vertex's b_old rows ahead of its edge loop
};

// Per vertex v and column group: for every incident edge e (ascending edge
// index): my_e = w y_i + (-w) y_j (spmm_dense over M, sparse.cpp:77-83),
// s_e = shrink(my_e + b_e) (solver.cpp:97), b_e' = b_e + (my_e - s_e)
// (solver.cpp:98); the owner (v == i) stores b_e' (and s_e).  The next
// right-hand side (solver.cpp:83-84) is accumulated from the same edge values:
// rhs_v = hl * sum_e M_ev (s_e - b_e') + rq_v.
template <int D, class Topo>
__global__ void __launch_bounds__(kBlock, D == 16 ? 2 : 3) k_sb_pass(Topo topo, SbArgs a) {
  constexpr int V = Cols<D>::V, TPV = Cols<D>::TPV;
  int bad = 0;
  long e0, e1, step;
  row_range<TPV>(topo, e0, e1, step);
  for (long e = e0; e < e1; e += step) {
    const int v = static_cast<int>(e / TPV);
    const int c0 = static_cast<int>(e - static_cast<long>(v) * TPV) * V;
    const Row<V> yv = ldg_row<V>(a.y + static_cast<long>(v) * D + c0);
#pragma unroll
    for (int k = 0; k < V; ++k) bad |= !isfinite(yv.a[k]);
    if constexpr (!Topo::kGrid) {
      // The b_old rows of a vertex's edges are the pass's DRAM reads (its own
      // rows stream, the rows owned by neighbours are scattered): ask L2 for
      // all of them now, one request per row, split over the vertex's lanes,
      // so the batches below find them in L2 or on their way instead of each
      // batch paying a DRAM round trip with its registers pinned.
      if (a.prefetch && a.b_old) {
        const int kb = __ldg(topo.iptr + v), ke = __ldg(topo.iptr + v + 1);
        for (int k = kb + static_cast<int>(e - static_cast<long>(v) * TPV); k < ke; k += TPV) {
          const double* row = a.b_old + static_cast<long>(__ldg(topo.ieid + k) >> 1) * D;
          asm volatile("prefetch.global.L2 [%0];" ::"l"(row));
          if constexpr ((D * 8) % 128 != 0) asm volatile("prefetch.global.L2 [%0];" ::"l"(row + D - 1));
        }
      }
    }
    double acc[V] = {};
    struct YB {
      Row<V> y, b;
    };
    auto load = [&](int u, long slot) {
      YB g;
      g.y = ldg_row<V>(a.y + static_cast<long>(u) * D + c0);
      if (a.b_old) {
        g.b = ldg_row<V>(a.b_old + slot * D + c0);
      } else {
#pragma unroll
        for (int k = 0; k < V; ++k) g.b.a[k] = 0.0;
      }
      return g;
    };
    topo.template visitE_b<(V >= 4 ? 3 : 4)>(v, load, [&](int u, double w, long slot, bool fwd, const YB& g) {
      const Row<V>& yu = g.y;
      const Row<V>& bo = g.b;
      Row<V> bn, sv;
      const double nw = -w;
#pragma unroll
      for (int k = 0; k < V; ++k) {
        const double yi = fwd ? yv.a[k] : yu.a[k];
        const double yj = fwd ? yu.a[k] : yv.a[k];
        const double t1 = w * yi;
        const double my = t1 + nw * yj;
        const double s = shrink1(my + bo.a[k], a.gamma);
        bn.a[k] = bo.a[k] + (my - s);
        sv.a[k] = s;
        acc[k] += (fwd ? w : nw) * (s - bn.a[k]);
      }
      // the owner (first endpoint) stores b and s; in a vertex-range
      // partition, edges owned by a ghost vertex are local replicas that this
      // range updates identically (CSR only: u >= vend() is a ghost row)
      if (fwd || (!Topo::kGrid && u >= topo.vend())) {
        st_row<V>(a.b_new + slot * D + c0, bn);
        if (a.s_out) st_row<V>(a.s_out + slot * D + c0, sv);
      }
    });
    if (a.rhs) {
      const Row<V> rq = ldg_row<V>(a.rq + static_cast<long>(v) * D + c0);
      Row<V> out;
#pragma unroll
      for (int k = 0; k < V; ++k) out.a[k] = a.hl * acc[k] + rq.a[k];
      st_row<V>(a.rhs + static_cast<long>(v) * D + c0, out);
    }
  }
  if (__syncthreads_or(bad) && threadIdx.x == 0) atomicOr(&a.ctl->nonfinite_y, 1);
}

// rhs_v = hl * sum_e M_ev (s_e - b_e) + rq_v for a caller-supplied inner
// state (first iteration of split_bregman when b, s are not known zero).
template <int D, class Topo>
__global__ void __launch_bounds__(kBlock) k_rhs_from_state(Topo topo, const double* __restrict__ s,
                                                          const double* __restrict__ b,
                                                          const double* __restrict__ rq, double* rhs, double hl) {
  constexpr int V = Cols<D>::V, TPV = Cols<D>::TPV;
  const long total = static_cast<long>(topo.vend()) * TPV;
  const long stride = static_cast<long>(gridDim.x) * blockDim.x;
  for (long e = static_cast<long>(topo.vbeg()) * TPV + static_cast<long>(blockIdx.x) * blockDim.x + threadIdx.x; e < total; e += stride) {
    const int v = static_cast<int>(e / TPV);
    const int c0 = static_cast<int>(e - static_cast<long>(v) * TPV) * V;
    double acc[V] = {};
    topo.visitE(v, [&](int, double w, long slot, bool fwd) {
      const Row<V> sv = ldg_row<V>(s + slot * D + c0);
      const Row<V> bv = ldg_row<V>(b + slot * D + c0);
      const double coef = fwd ? w : -w;
#pragma unroll
      for (int k = 0; k < V; ++k) acc[k] += coef * (sv.a[k] - bv.a[k]);
    });
    const Row<V> q = ldg_row<V>(rq + static_cast<long>(v) * D + c0);
    Row<V> out;
#pragma unroll
    for (int k = 0; k < V; ++k) out.a[k] = hl * acc[k] + q.a[k];
    st_row<V>(rhs + static_cast<long>(v) * D + c0, out);
  }
}

// rq = (r/2) * (sqrt(deg) * (P - B))   (solver.cpp:79-80)
template <int D>
__global__ void __launch_bounds__(kBlock) k_rhs_quad(int n, const double* __restrict__ sqd, const double* __restrict__ p,
                                                    const double* __restrict__ breg, double* rq, double hr) {
  const long total = static_cast<long>(n) * D;
  const long stride = static_cast<long>(gridDim.x) * blockDim.x;
  for (long e = static_cast<long>(blockIdx.x) * blockDim.x + threadIdx.x; e < total; e += stride) {
    const int v = static_cast<int>(e / D);
    rq[e] = hr * (__ldg(sqd + v) * (__ldg(p + e) - __ldg(breg + e)));
  }
}

// objective = sum over edges and columns of |w y_i + (-w) y_j| (solver.cpp:14-17).
template <int D, class Topo>
__global__ void __launch_bounds__(kBlock) k_objective(Topo topo, const double* __restrict__ y, double* partials,
                                                     Ctl* ctl) {
  constexpr int V = Cols<D>::V, TPV = Cols<D>::TPV;
  double acc[1][V] = {};
  const long total = static_cast<long>(topo.vend()) * TPV;
  const long stride = static_cast<long>(gridDim.x) * blockDim.x;
  for (long e = static_cast<long>(topo.vbeg()) * TPV + static_cast<long>(blockIdx.x) * blockDim.x + threadIdx.x; e < total; e += stride) {
    const int v = static_cast<int>(e / TPV);
    const int c0 = static_cast<int>(e - static_cast<long>(v) * TPV) * V;
    const Row<V> yv = ldg_row<V>(y + static_cast<long>(v) * D + c0);
    topo.visitE(v, [&](int u, double w, long, bool fwd) {
      if (!fwd) return;
      const Row<V> yu = ldg_row<V>(y + static_cast<long>(u) * D + c0);
#pragma unroll
      for (int k = 0; k < V; ++k) acc[0][k] += fabs(w * yv.a[k] + (-w) * yu.a[k]);
    });
  }
  block_reduce_store<1, D, V>(acc, partials);
  __shared__ double tot[1][D];
  if (!grid_reduce_last<1, D>(partials, ctl, tot)) return;
  if (threadIdx.x == 0) {
    double s = 0.0;
    for (int j = 0; j < D; ++j) s += tot[0][j];
    ctl->scalar[0] = s;
  }
}

// ||Y_new - Y_old||^2 and ||Y_old||^2 for the relative-change test
// (solver.cpp:102-106, 120-124).
template <int D>
__global__ void __launch_bounds__(kBlock) k_diff_norms(int n, const double* __restrict__ ynew,
                                                      const double* __restrict__ yold, double* partials, Ctl* ctl) {
  double acc[2][D] = {};
  const long stride = static_cast<long>(gridDim.x) * blockDim.x;
  for (long v = static_cast<long>(blockIdx.x) * blockDim.x + threadIdx.x; v < n; v += stride) {
#pragma unroll
    for (int k = 0; k < D; ++k) {
      const double o = __ldg(yold + v * D + k);
      const double df = __ldg(ynew + v * D + k) - o;
      acc[0][k] += df * df;
      acc[1][k] += o * o;
    }
  }
  block_reduce_store<2, D, D>(acc, partials);
  __shared__ double tot[2][D];
  if (!grid_reduce_last<2, D>(partials, ctl, tot)) return;
  if (threadIdx.x == 0) {
    double a = 0.0, b = 0.0;
    for (int j = 0; j < D; ++j) {
      a += tot[0][j];
      b += tot[1][j];
    }
    ctl->scalar[1] = a;
    ctl->scalar[2] = b;
  }
}

}  // namespace pfe_dev
