// Shared-memory tiled stencil kernels for pixel-grid graphs (Grid<R>).
//
// A block owns a TW x TH tile of the image (one thread per tile vertex).
// Everything the tile needs from HBM is staged with cp.async (LDGSTS) in one
// batch: the (TW+2R) x (TH+2R) halo of the input rows, the forward-slot edge
// weights of those positions, the interior rows (rhs, diag, ...) and, for
// the split-Bregman pass on 8-neighbour grids, b_old of every edge touching
// the tile.  The copies are all in flight together (one memory round trip
// per tile instead of one per neighbour and per array), go straight to shared
// memory without register staging, and are zero-filled outside the image.
// The stencil is then evaluated from shared memory in the reference's exact
// summation order (see pfe_device.cuh); control-block values (alpha, beta,
// status) are read while the copies are in flight.
//
//   k_grid_pcg_init   r = b - A x0, p = D^-1 r, ||b||^2, r.r, r.z
//   k_grid_pcg_spmv   p' = D^-1 r + beta p (halo recomputed), q = A p', p'.q, alpha
//   k_grid_sb_pass    M Y, shrink, b update, next rhs (split-Bregman pass)
#pragma once

#include "pfe_kernels.cuh"

namespace pfe_dev {

// ------------------------------------------------------------ cp.async ----
__device__ __forceinline__ void cp_async(double* dst, const double* src, bool pred, int bytes) {
  const unsigned d = static_cast<unsigned>(__cvta_generic_to_shared(dst));
  const int sz = pred ? bytes : 0;  // 0 => zero-fill, nothing read
  if (bytes == 16)
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(d), "l"(src), "r"(sz));
  else
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(d), "l"(src), "r"(sz));
}
__device__ __forceinline__ void cp_async_wait_all() {
  asm volatile("cp.async.commit_group;\n" ::);
  asm volatile("cp.async.wait_all;\n" ::: "memory");
}

// ------------------------------------------------------------ geometry ----
template <int R, int D>
struct TileGeo {
  static constexpr int TW = 32;
  static constexpr int TH = (D <= 4 || R == 2) ? 8 : 4;  // keeps sb staging within 2+ blocks/SM
  static constexpr int NT = TW * TH;                     // threads per block
  static constexpr int HW = TW + 2 * R, HH = TH + 2 * R, NP = HW * HH;
  static constexpr int S = GridTopo<R>::S;
  static constexpr int NO = (TH + R) * HW;  // positions owning edges that touch the tile
  static constexpr bool kStageB = (R == 1);
  // shared-memory footprints (doubles)
  static constexpr int kInit = NP * D + NP * S + NT * D + 2 * NT;
  static constexpr int kSpmv = 2 * NP * D + NP + NP * S + NT;
  static constexpr int kSb = NP * D + NP * S + NT * D + (kStageB ? NO * S * D : 0);
};

struct TileIdx {
  int y0, x0;
};

template <int R, int D>
__device__ __forceinline__ int num_tiles(const Grid<R>& g) {
  using G = TileGeo<R, D>;
  return ((g.W + G::TW - 1) / G::TW) * ((g.H + G::TH - 1) / G::TH);
}
template <int R, int D>
__device__ __forceinline__ TileIdx tile_of(const Grid<R>& g, int t) {
  using G = TileGeo<R, D>;
  const int tiles_x = (g.W + G::TW - 1) / G::TW;
  const int ty = t / tiles_x;
  return {ty * G::TH, (t - ty * tiles_x) * G::TW};
}

// Issues cp.async copies of a [n][W] row-major array for the halo positions
// (rows [r0, r0+nrows) of the halo tile) into dst[pos][W].
template <int R, int D, int W>
__device__ __forceinline__ void stage_halo(const Grid<R>& g, TileIdx ti, const double* __restrict__ src, double* dst,
                                           int nrows) {
  using G = TileGeo<R, D>;
  constexpr int CH = (W % 2 == 0) ? 2 : 1;
  constexpr int PER = W / CH;
  const int total = nrows * G::HW * PER;
  for (int c = threadIdx.x; c < total; c += G::NT) {
    const int pos = c / PER, k = (c - pos * PER) * CH;
    const int hy = pos / G::HW, hx = pos - hy * G::HW;
    const int y = ti.y0 - R + hy, x = ti.x0 - R + hx;
    const bool in = y >= 0 && y < g.H && x >= 0 && x < g.W;
    const double* s = in ? src + (static_cast<long>(y) * g.W + x) * W + k : src;
    cp_async(dst + pos * W + k, s, in, CH * 8);
  }
}

// Interior rows [NT][W] of a [n][W] array.
template <int R, int D, int W>
__device__ __forceinline__ void stage_interior(const Grid<R>& g, TileIdx ti, const double* __restrict__ src,
                                               double* dst) {
  using G = TileGeo<R, D>;
  constexpr int CH = (W % 2 == 0) ? 2 : 1;
  constexpr int PER = W / CH;
  for (int c = threadIdx.x; c < G::NT * PER; c += G::NT) {
    const int pos = c / PER, k = (c - pos * PER) * CH;
    const int ty = pos / G::TW, tx = pos - ty * G::TW;
    const int y = ti.y0 + ty, x = ti.x0 + tx;
    const bool in = y < g.H && x < g.W;
    const double* s = in ? src + (static_cast<long>(y) * g.W + x) * W + k : src;
    cp_async(dst + pos * W + k, s, in, CH * 8);
  }
}

// q_v = sum over the row of A in ascending column order (sparse.cpp:77-83)
// from the staged tile: backward slots, diagonal, forward slots.
template <int D, int R>
__device__ __forceinline__ void tile_apply_A(double hl, const double* P, const double* Wt, int hpos, double diag_v,
                                             double (&q)[D]) {
  using G = TileGeo<R, D>;
  using T = GridTopo<R>;
#pragma unroll
  for (int c = 0; c < D; ++c) q[c] = 0.0;
#pragma unroll
  for (int s = G::S - 1; s >= 0; --s) {
    const int npos = hpos - T::dy(s) * G::HW - T::dx(s);
    const double w = Wt[npos * G::S + s];
    if (w != 0.0) {
      const double a = -((hl * w) * w);
#pragma unroll
      for (int c = 0; c < D; ++c) q[c] += a * P[npos * D + c];
    }
  }
#pragma unroll
  for (int c = 0; c < D; ++c) q[c] += diag_v * P[hpos * D + c];
#pragma unroll
  for (int s = 0; s < G::S; ++s) {
    const int npos = hpos + T::dy(s) * G::HW + T::dx(s);
    const double w = Wt[hpos * G::S + s];
    if (w != 0.0) {
      const double a = -((hl * w) * w);
#pragma unroll
      for (int c = 0; c < D; ++c) q[c] += a * P[npos * D + c];
    }
  }
}

// ---------------------------------------------------------------- init ----
template <int D, int R>
__global__ void __launch_bounds__(TileGeo<R, D>::NT) k_grid_pcg_init(Grid<R> g, PcgArgs a) {
  using G = TileGeo<R, D>;
  extern __shared__ double smem[];
  double* P = smem;                   // x0 halo [NP][D]
  double* Wt = P + G::NP * D;         // [NP][S]
  double* Bv = Wt + G::NP * G::S;     // rhs interior [NT][D]
  double* Dg = Bv + G::NT * D;        // diag interior
  double* Iv = Dg + G::NT;            // inv diag interior
  double acc[3][D] = {};
  const int tx = threadIdx.x % G::TW, ty = threadIdx.x / G::TW;
  const int hpos = (ty + R) * G::HW + (tx + R);
  const int nt = num_tiles<R, D>(g);
  for (int t = blockIdx.x; t < nt; t += gridDim.x) {
    const TileIdx ti = tile_of<R, D>(g, t);
    stage_halo<R, D, D>(g, ti, a.x0, P, G::HH);
    stage_halo<R, D, G::S>(g, ti, g.wf, Wt, G::HH);
    stage_interior<R, D, D>(g, ti, a.rhs, Bv);
    stage_interior<R, D, 1>(g, ti, g.diag, Dg);
    stage_interior<R, D, 1>(g, ti, g.invd, Iv);
    cp_async_wait_all();
    __syncthreads();
    const int y = ti.y0 + ty, x = ti.x0 + tx;
    if (y < g.H && x < g.W) {
      const long v = static_cast<long>(y) * g.W + x;
      double ax[D];
      tile_apply_A<D, R>(g.hl, P, Wt, hpos, Dg[threadIdx.x], ax);
      const double id = Iv[threadIdx.x];
#pragma unroll
      for (int c = 0; c < D; ++c) {
        const double b = Bv[threadIdx.x * D + c];
        const double r = b - ax[c];
        const double z = id * r;
        a.r[v * D + c] = r;
        a.pbuf[0][v * D + c] = z;
        acc[0][c] += b * b;
        acc[1][c] += r * r;
        acc[2][c] += r * z;
      }
    }
    __syncthreads();
  }
  block_reduce_store<3, D, D, G::NT>(acc, a.partials);
  __shared__ double tot[3][D];
  if (!grid_reduce_last<3, D, G::NT>(a.partials, a.ctl, tot)) return;
  if (threadIdx.x < 32) pcg_init_epilogue<D>(a, tot);
}

// ---------------------------------------------------------------- spmv ----
template <int D, int R>
__global__ void __launch_bounds__(TileGeo<R, D>::NT) k_grid_pcg_spmv(Grid<R> g, PcgArgs a) {
  using G = TileGeo<R, D>;
  extern __shared__ double smem[];
  double* P = smem;                   // p (phase 0) or p_old -> p' in place [NP][D]
  double* Rs = P + G::NP * D;         // r halo [NP][D]
  double* Iv = Rs + G::NP * D;        // inv diag halo [NP]
  double* Wt = Iv + G::NP;            // [NP][S]
  double* Dg = Wt + G::NP * G::S;     // diag interior [NT]
  __shared__ double beta[D];
  __shared__ int active;
  const bool first = a.phase == 0;
  double* pnew = pcg_pnew(a);
  const double* pold = first ? a.pbuf[0] : pcg_pold(a);
  double acc[1][D] = {};
  const int tx = threadIdx.x % G::TW, ty = threadIdx.x / G::TW;
  const int hpos = (ty + R) * G::HW + (tx + R);
  const int nt = num_tiles<R, D>(g);
  bool checked = false;
  for (int t = blockIdx.x; t < nt; t += gridDim.x) {
    const TileIdx ti = tile_of<R, D>(g, t);
    stage_halo<R, D, D>(g, ti, pold, P, G::HH);
    if (!first) {
      stage_halo<R, D, D>(g, ti, a.r, Rs, G::HH);
      stage_halo<R, D, 1>(g, ti, g.invd, Iv, G::HH);
    }
    stage_halo<R, D, G::S>(g, ti, g.wf, Wt, G::HH);
    stage_interior<R, D, 1>(g, ti, g.diag, Dg);
    if (!checked) {  // control block read while the copies are in flight
      if (threadIdx.x < D) {
        const PcgCol& col = a.ctl->col[threadIdx.x];
        beta[threadIdx.x] = col.status == kActive ? col.beta : 0.0;
      }
      if (threadIdx.x == 0) active = a.ctl->any_active;
    }
    cp_async_wait_all();
    __syncthreads();
    if (!checked) {
      if (!active) return;
      checked = true;
    }
    if (!first) {
      // p_u = z_u + beta p_u, z_u = D^-1_u r_u (pcg.cpp:86-88) for every tile
      // + halo position; halo values are recomputed bit-identically.
      for (int e = threadIdx.x; e < G::NP * D; e += G::NT) {
        const int pos = e / D, c = e - pos * D;
        P[e] = Iv[pos] * Rs[e] + beta[c] * P[e];
      }
      __syncthreads();
    }
    const int y = ti.y0 + ty, x = ti.x0 + tx;
    if (y < g.H && x < g.W) {
      const long v = static_cast<long>(y) * g.W + x;
      double q[D];
      tile_apply_A<D, R>(g.hl, P, Wt, hpos, Dg[threadIdx.x], q);
#pragma unroll
      for (int c = 0; c < D; ++c) {
        const double pv = P[hpos * D + c];
        a.q[v * D + c] = q[c];
        if (!first) pnew[v * D + c] = pv;
        acc[0][c] += pv * q[c];
      }
    }
    __syncthreads();
  }
  if (!checked) {  // block without tiles still votes
    if (threadIdx.x == 0) active = a.ctl->any_active;
    __syncthreads();
    if (!active) return;
  }
  block_reduce_store<1, D, D, G::NT>(acc, a.partials);
  __shared__ double tot[1][D];
  if (!grid_reduce_last<1, D, G::NT>(a.partials, a.ctl, tot)) return;
  if (threadIdx.x < 32) pcg_spmv_epilogue<D>(a, tot);
}

// ----------------------------------------------------- split-Bregman pass -
// Per interior vertex v: incident edges in edge order (backward slots
// S-1..0 owned by neighbours, then forward slots 0..S-1 owned by v), each
// evaluated as solver.cpp:96-98 and accumulated into the next rhs
// (solver.cpp:83-84).  8-neighbour grids stage b_old of all those edges; 5x5
// grids read it from global memory two columns at a time.
template <int D, int R>
__global__ void __launch_bounds__(TileGeo<R, D>::NT) k_grid_sb_pass(Grid<R> g, SbArgs a) {
  using G = TileGeo<R, D>;
  using T = GridTopo<R>;
  constexpr int CW = (D % 2 == 0) ? 2 : 1;
  extern __shared__ double smem[];
  double* P = smem;                 // Y halo [NP][D]
  double* Wt = P + G::NP * D;       // [NP][S]
  double* Rq = Wt + G::NP * G::S;   // rq interior [NT][D]
  double* Bo = Rq + G::NT * D;      // b_old of owner rows [NO][S][D] (8-nbr only)
  const int tx = threadIdx.x % G::TW, ty = threadIdx.x / G::TW;
  const int hpos = (ty + R) * G::HW + (tx + R);
  const int nt = num_tiles<R, D>(g);
  int bad = 0;
  for (int t = blockIdx.x; t < nt; t += gridDim.x) {
    const TileIdx ti = tile_of<R, D>(g, t);
    stage_halo<R, D, D>(g, ti, a.y, P, G::HH);
    stage_halo<R, D, G::S>(g, ti, g.wf, Wt, G::HH);
    if (a.rhs) stage_interior<R, D, D>(g, ti, a.rq, Rq);
    if constexpr (G::kStageB) {
      if (a.b_old) stage_halo<R, D, G::S * D>(g, ti, a.b_old, Bo, G::TH + R);
    }
    cp_async_wait_all();
    __syncthreads();
    const int y = ti.y0 + ty, x = ti.x0 + tx;
    if (y < g.H && x < g.W) {
      const long v = static_cast<long>(y) * g.W + x;
#pragma unroll
      for (int c = 0; c < D; ++c) bad |= !isfinite(P[hpos * D + c]);
#pragma unroll
      for (int c0 = 0; c0 < D; c0 += CW) {
        double acc[CW];
#pragma unroll
        for (int k = 0; k < CW; ++k) acc[k] = 0.0;
#pragma unroll
        for (int e = 0; e < 2 * G::S; ++e) {
          const bool fwd = e >= G::S;
          const int s = fwd ? e - G::S : G::S - 1 - e;
          const int npos = fwd ? hpos + T::dy(s) * G::HW + T::dx(s) : hpos - T::dy(s) * G::HW - T::dx(s);
          const int opos = fwd ? hpos : npos;  // owner (first endpoint i)
          const int jpos = fwd ? npos : hpos;
          const double w = Wt[opos * G::S + s];
          if (w == 0.0) continue;
          const long slot = fwd ? v * G::S + s : (v - T::dy(s) * g.W - T::dx(s)) * G::S + s;
          double bo[CW];
#pragma unroll
          for (int k = 0; k < CW; ++k) {
            if (!a.b_old)
              bo[k] = 0.0;
            else if constexpr (G::kStageB)
              bo[k] = Bo[(opos * G::S + s) * D + c0 + k];
            else
              bo[k] = __ldg(a.b_old + slot * D + c0 + k);
          }
          const double nw = -w;
          double bn[CW], sv[CW];
#pragma unroll
          for (int k = 0; k < CW; ++k) {
            const double my = w * P[opos * D + c0 + k] + nw * P[jpos * D + c0 + k];
            const double sh = shrink1(my + bo[k], a.gamma);
            bn[k] = bo[k] + (my - sh);
            sv[k] = sh;
            acc[k] += (fwd ? w : nw) * (sh - bn[k]);
          }
          if (fwd) {
#pragma unroll
            for (int k = 0; k < CW; ++k) {
              a.b_new[slot * D + c0 + k] = bn[k];
              if (a.s_out) a.s_out[slot * D + c0 + k] = sv[k];
            }
          }
        }
        if (a.rhs)
#pragma unroll
          for (int k = 0; k < CW; ++k) a.rhs[v * D + c0 + k] = a.hl * acc[k] + Rq[threadIdx.x * D + c0 + k];
      }
    }
    __syncthreads();
  }
  if (__syncthreads_or(bad) && threadIdx.x == 0) atomicOr(&a.ctl->nonfinite_y, 1);
}

}  // namespace pfe_dev
