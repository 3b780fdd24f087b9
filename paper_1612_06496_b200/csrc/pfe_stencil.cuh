// Shared-memory tiled stencil kernels for pixel-grid graphs (Grid<R>).
//
// A block owns a TW x TH tile of the image.  Everything the tile needs from
// HBM is staged with cp.async (LDGSTS) in one batch: the (TW+2R) x (TH+2R)
// halo of the input rows, the forward-slot edge weights of those positions,
// the interior rows (rhs, diag, ...) and, for the split-Bregman pass on
// 8-neighbour grids, b_old of every edge touching the tile.  All copies are
// in flight together (one memory round trip per tile), go straight to shared
// memory and are zero-filled outside the image.  The stencil is then
// evaluated from shared memory in the reference's exact summation order (see
// pfe_device.cuh), one (vertex, column) element per thread so that
// consecutive lanes read consecutive words (row data [pos][d]; weights and
// edge variables stored slot-planar [s][pos][d]): no bank conflicts.
// Control-block values (beta, status) are read while the copies are in flight.
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
  static constexpr int TH = (D <= 4 || R == 2) ? 8 : 4;  // keeps the sb staging at >= 3 blocks/SM
  static constexpr int NV = TW * TH;                     // tile vertices
  // threads per block: 5x5 tiles need ~100-200 KB of shared memory (one
  // block per SM), so they get 16 warps to keep enough loads in flight
  static constexpr int NT = R == 2 ? 512 : 256;
  static constexpr int HW = TW + 2 * R, HH = TH + 2 * R, NP = HW * HH;
  static constexpr int S = GridTopo<R>::S;
  static constexpr int NO = (TH + R) * HW;  // positions owning edges that touch the tile
  static constexpr bool kStageB = (R == 1);
  // element-parallel compute: thread owns column tid % D of successive vertices
  static constexpr bool kEl = (32 % D == 0);
  static constexpr int V = kEl ? 1 : D;  // columns accumulated per thread
  // shared-memory footprints (doubles); every array offset stays 16-byte aligned
  static constexpr int kInit = NP * D + S * NP + NV * D + 2 * NV;
  static constexpr int kSpmv = 2 * NP * D + NP + S * NP + NV;
  static constexpr int kSb = NP * D + S * NP + NV * D + (kStageB ? S * NO * D : 0);
  static_assert(NP % 2 == 0 && NO % 2 == 0, "alignment of staged arrays");
};

struct TileIdx {
  int y0, x0;
};

template <int R, int D>
__device__ __forceinline__ int num_tiles(const Grid<R>& g) {
  using G = TileGeo<R, D>;
  return ((g.W + G::TW - 1) / G::TW) * ((g.row_hi - g.row_lo + G::TH - 1) / G::TH);
}
template <int R, int D>
__device__ __forceinline__ TileIdx tile_of(const Grid<R>& g, int t) {
  using G = TileGeo<R, D>;
  const int tiles_x = (g.W + G::TW - 1) / G::TW;
  const int ty = t / tiles_x;
  return {g.row_lo + ty * G::TH, (t - ty * tiles_x) * G::TW};
}

template <int R, int D>
__device__ __forceinline__ bool halo_in(const Grid<R>& g, TileIdx ti, int pos, long& u) {
  using G = TileGeo<R, D>;
  const int hy = pos / G::HW, hx = pos - hy * G::HW;
  const int y = ti.y0 - R + hy, x = ti.x0 - R + hx;
  u = static_cast<long>(y) * g.W + x;
  return y >= 0 && y < g.H && x >= 0 && x < g.W;
}

// Rows [n][W] -> dst[pos][W] for halo rows [0, nrows) (16-byte copies when W even).
template <int R, int D, int W>
__device__ __forceinline__ void stage_rows(const Grid<R>& g, TileIdx ti, const double* __restrict__ src, double* dst,
                                           int nrows) {
  using G = TileGeo<R, D>;
  constexpr int CH = (W % 2 == 0) ? 2 : 1;
  constexpr int PER = W / CH;
  const int total = nrows * G::HW * PER;
  for (int c = threadIdx.x; c < total; c += G::NT) {
    const int pos = c / PER, k = (c - pos * PER) * CH;
    long u;
    const bool in = halo_in<R, D>(g, ti, pos, u);
    cp_async(dst + pos * W + k, in ? src + u * W + k : src, in, CH * 8);
  }
}

// Slot-major planes: src [n][S][W] -> dst[s][pos][W] for halo rows [0, nrows)
// (npos = nrows * HW positions per plane).
template <int R, int D, int S, int W>
__device__ __forceinline__ void stage_planes(const Grid<R>& g, TileIdx ti, const double* __restrict__ src, double* dst,
                                             int nrows) {
  using G = TileGeo<R, D>;
  constexpr int CH = (W % 2 == 0) ? 2 : 1;
  constexpr int PER = W / CH;
  const int npos = nrows * G::HW;
  const int total = npos * S * PER;
  for (int c = threadIdx.x; c < total; c += G::NT) {
    const int pos = c / (S * PER);
    const int rem = c - pos * (S * PER);
    const int s = rem / PER, k = (rem - s * PER) * CH;
    long u;
    const bool in = halo_in<R, D>(g, ti, pos, u);
    cp_async(dst + (s * npos + pos) * W + k, in ? src + (u * S + s) * W + k : src, in, CH * 8);
  }
}

// Interior rows [NV][W].
template <int R, int D, int W>
__device__ __forceinline__ void stage_interior(const Grid<R>& g, TileIdx ti, const double* __restrict__ src,
                                               double* dst) {
  using G = TileGeo<R, D>;
  constexpr int CH = (W % 2 == 0) ? 2 : 1;
  constexpr int PER = W / CH;
  for (int c = threadIdx.x; c < G::NV * PER; c += G::NT) {
    const int tv = c / PER, k = (c - tv * PER) * CH;
    const int ty = tv / G::TW, tx = tv - ty * G::TW;
    const int y = ti.y0 + ty, x = ti.x0 + tx;
    const bool in = y < g.row_hi && x < g.W;
    cp_async(dst + tv * W + k, in ? src + (static_cast<long>(y) * g.W + x) * W + k : src, in, CH * 8);
  }
}

// Iterates the tile's (vertex, column) elements owned by this thread:
// f(tv, c, hpos, v, k) with k the accumulator slot (0 in element mode, c in
// vertex mode).  Vertices outside the image are skipped.
template <int R, int D, class F>
__device__ __forceinline__ void for_tile_elements(const Grid<R>& g, TileIdx ti, F&& f) {
  using G = TileGeo<R, D>;
  if constexpr (G::kEl) {
    const int c = threadIdx.x % D;
    for (int e = threadIdx.x; e < G::NV * D; e += G::NT) {
      const int tv = e / D;
      const int ty = tv / G::TW, tx = tv - ty * G::TW;
      const int y = ti.y0 + ty, x = ti.x0 + tx;
      if (y < g.row_hi && x < g.W)
        f(tv, c, (ty + R) * G::HW + (tx + R), static_cast<long>(y) * g.W + x, 0);
    }
  } else {
    for (int tv = threadIdx.x; tv < G::NV; tv += G::NT) {
      const int ty = tv / G::TW, tx = tv - ty * G::TW;
      const int y = ti.y0 + ty, x = ti.x0 + tx;
      if (y < g.row_hi && x < g.W)
#pragma unroll
        for (int c = 0; c < D; ++c) f(tv, c, (ty + R) * G::HW + (tx + R), static_cast<long>(y) * g.W + x, c);
    }
  }
}

// (A p)_v, column c, in ascending column order (sparse.cpp:77-83): backward
// slots, diagonal, forward slots.  Wt is slot-planar [S][NP].
template <int D, int R>
__device__ __forceinline__ double tile_apply_A(double hl, const double* P, const double* Wt, int hpos, int c,
                                               double diag_v) {
  using G = TileGeo<R, D>;
  using T = GridTopo<R>;
  // branch-free: every term is loaded and formed, absent edges (w == 0) are
  // skipped by a select, so all loads are in flight before the serial
  // reference-order additions
  double t[2 * G::S + 1];
  bool nz[2 * G::S + 1];
#pragma unroll
  for (int j = 0; j < G::S; ++j) {
    const int s = G::S - 1 - j;
    const int npos = hpos - T::dy(s) * G::HW - T::dx(s);
    const double w = Wt[s * G::NP + npos];
    nz[j] = w != 0.0;
    t[j] = -((hl * w) * w) * P[npos * D + c];
  }
  nz[G::S] = true;
  t[G::S] = diag_v * P[hpos * D + c];
#pragma unroll
  for (int s = 0; s < G::S; ++s) {
    const int npos = hpos + T::dy(s) * G::HW + T::dx(s);
    const double w = Wt[s * G::NP + hpos];
    nz[G::S + 1 + s] = w != 0.0;
    t[G::S + 1 + s] = -((hl * w) * w) * P[npos * D + c];
  }
  double q = 0.0;
#pragma unroll
  for (int j = 0; j < 2 * G::S + 1; ++j) q = nz[j] ? q + t[j] : q;
  return q;
}

// ---------------------------------------------------------------- init ----
template <int D, int R>
__global__ void __launch_bounds__(TileGeo<R, D>::NT) k_grid_pcg_init(Grid<R> g, PcgArgs a) {
  using G = TileGeo<R, D>;
  constexpr int V = G::V;
  extern __shared__ double smem[];
  double* P = smem;                  // x0 halo [NP][D]
  double* Wt = P + G::NP * D;        // [S][NP]
  double* Bv = Wt + G::S * G::NP;    // rhs interior [NV][D]
  double* Dg = Bv + G::NV * D;       // diag interior [NV]
  double* Iv = Dg + G::NV;           // inv diag interior [NV]
  double acc[3][V] = {};
  const int nt = num_tiles<R, D>(g);
  for (int t = blockIdx.x; t < nt; t += gridDim.x) {
    const TileIdx ti = tile_of<R, D>(g, t);
    stage_rows<R, D, D>(g, ti, a.x0, P, G::HH);
    stage_planes<R, D, G::S, 1>(g, ti, g.wf, Wt, G::HH);
    stage_interior<R, D, D>(g, ti, a.rhs, Bv);
    stage_interior<R, D, 1>(g, ti, g.diag, Dg);
    stage_interior<R, D, 1>(g, ti, g.invd, Iv);
    cp_async_wait_all();
    __syncthreads();
    for_tile_elements<R, D>(g, ti, [&](int tv, int c, int hpos, long v, int k) {
      const double ax = tile_apply_A<D, R>(g.hl, P, Wt, hpos, c, Dg[tv]);
      const double b = Bv[tv * D + c];
      const double r = b - ax;
      const double z = Iv[tv] * r;
      a.r[v * D + c] = r;
      a.pbuf[0][v * D + c] = z;
      acc[0][k] += b * b;
      acc[1][k] += r * r;
      acc[2][k] += r * z;
    });
    __syncthreads();
  }
  block_reduce_store<3, D, V, G::NT>(acc, a.part_a);  // reduced by the first SpMV
}

// ---------------------------------------------------------------- spmv ----
template <int D, int R>
__global__ void __launch_bounds__(TileGeo<R, D>::NT) k_grid_pcg_spmv(Grid<R> g, PcgArgs a) {
  using G = TileGeo<R, D>;
  constexpr int V = G::V;
  extern __shared__ double smem[];
  double* P = smem;                  // p (phase 0) or p_old -> p' in place [NP][D]
  double* Rs = P + G::NP * D;        // r halo [NP][D]
  double* Iv = Rs + G::NP * D;       // inv diag halo [NP]
  double* Wt = Iv + G::NP;           // [S][NP]
  double* Dg = Wt + G::S * G::NP;    // diag interior [NV]
  __shared__ ColView<D> cv;
  const bool first = a.phase == 0;
  double* pnew = pcg_pnew(a);
  const double* pold = first ? a.pbuf[0] : pcg_pold(a);
  double acc[1][V] = {};
  const int nt = num_tiles<R, D>(g);
  bool checked = false;
  for (int t = blockIdx.x; t < nt; t += gridDim.x) {
    const TileIdx ti = tile_of<R, D>(g, t);
    stage_rows<R, D, D>(g, ti, pold, P, G::HH);
    if (!first) {
      stage_rows<R, D, D>(g, ti, a.r, Rs, G::HH);
      stage_rows<R, D, 1>(g, ti, g.invd, Iv, G::HH);
    }
    stage_planes<R, D, G::S, 1>(g, ti, g.wf, Wt, G::HH);
    stage_interior<R, D, 1>(g, ti, g.diag, Dg);
    if (!checked) {  // stop test + beta while the copies are in flight
      if (!spmv_prologue<D, G::NT>(a, cv)) {
        cp_async_wait_all();
        return;
      }
      checked = true;
    }
    cp_async_wait_all();
    __syncthreads();
    if (!first) {
      // p_u = z_u + beta p_u, z_u = D^-1_u r_u (pcg.cpp:86-88) for every tile
      // + halo position; halo values are recomputed bit-identically.
      for (int e = threadIdx.x; e < G::NP * D; e += G::NT) {
        const int pos = e / D, c = e - pos * D;
        P[e] = Iv[pos] * Rs[e] + cv.coef[c] * P[e];
      }
      __syncthreads();
    }
    for_tile_elements<R, D>(g, ti, [&](int tv, int c, int hpos, long v, int k) {
      const double q = tile_apply_A<D, R>(g.hl, P, Wt, hpos, c, Dg[tv]);
      const double pv = P[hpos * D + c];
      a.q[v * D + c] = q;
      if (!first) pnew[v * D + c] = pv;
      acc[0][k] += pv * q;
    });
    __syncthreads();
  }
  if (!checked && !spmv_prologue<D, G::NT>(a, cv)) return;  // block without tiles
  block_reduce_store<1, D, V, G::NT>(acc, a.part_b);  // reduced by the update
}

// ----------------------------------------------------- split-Bregman pass -
// Per interior vertex v and column: incident edges in edge order (backward
// slots S-1..0 owned by neighbours, then forward slots 0..S-1 owned by v),
// each evaluated as solver.cpp:96-98 and accumulated into the next rhs
// (solver.cpp:83-84).  8-neighbour grids stage b_old of all those edges
// (slot-planar); 5x5 grids read it from global memory.
template <int D, int R>
__global__ void __launch_bounds__(TileGeo<R, D>::NT) k_grid_sb_pass(Grid<R> g, SbArgs a) {
  using G = TileGeo<R, D>;
  using T = GridTopo<R>;
  extern __shared__ double smem[];
  double* P = smem;                 // Y halo [NP][D]
  double* Wt = P + G::NP * D;       // [S][NP]
  double* Rq = Wt + G::S * G::NP;   // rq interior [NV][D]
  double* Bo = Rq + G::NV * D;      // b_old of owners [S][NO][D] (8-nbr only)
  const int nt = num_tiles<R, D>(g);
  int bad = 0;
  for (int t = blockIdx.x; t < nt; t += gridDim.x) {
    const TileIdx ti = tile_of<R, D>(g, t);
    stage_rows<R, D, D>(g, ti, a.y, P, G::HH);
    stage_planes<R, D, G::S, 1>(g, ti, g.wf, Wt, G::HH);
    if (a.rhs) stage_interior<R, D, D>(g, ti, a.rq, Rq);
    if constexpr (G::kStageB) {
      if (a.b_old) stage_planes<R, D, G::S, D>(g, ti, a.b_old, Bo, G::TH + R);
    }
    cp_async_wait_all();
    __syncthreads();
    for_tile_elements<R, D>(g, ti, [&](int tv, int c, int hpos, long v, int) {
      bad |= !isfinite(P[hpos * D + c]);
      double acc = 0.0;
#pragma unroll
      for (int e = 0; e < 2 * G::S; ++e) {
        const bool fwd = e >= G::S;
        const int s = fwd ? e - G::S : G::S - 1 - e;
        const int npos = fwd ? hpos + T::dy(s) * G::HW + T::dx(s) : hpos - T::dy(s) * G::HW - T::dx(s);
        const int opos = fwd ? hpos : npos;  // owner = first endpoint i
        const int jpos = fwd ? npos : hpos;
        const double w = Wt[s * G::NP + opos];
        if (w == 0.0) continue;
        const long slot = fwd ? v * G::S + s : (v - T::dy(s) * g.W - T::dx(s)) * G::S + s;
        double bo = 0.0;
        if (a.b_old) {
          if constexpr (G::kStageB)
            bo = Bo[(s * G::NO + opos) * D + c];
          else
            bo = __ldg(a.b_old + slot * D + c);
        }
        const double nw = -w;
        const double my = w * P[opos * D + c] + nw * P[jpos * D + c];
        const double sh = shrink1(my + bo, a.gamma);
        const double bn = bo + (my - sh);
        acc += (fwd ? w : nw) * (sh - bn);
        // the owner stores b (and s); in a row band, edges owned by the halo
        // rows above are replicas that this band updates identically
        if (fwd || static_cast<int>(v / g.W) - T::dy(s) < g.row_lo) {
          a.b_new[slot * D + c] = bn;
          if (a.s_out) a.s_out[slot * D + c] = sh;
        }
      }
      if (a.rhs) a.rhs[v * D + c] = a.hl * acc + Rq[tv * D + c];
    });
    __syncthreads();
  }
  if (__syncthreads_or(bad) && threadIdx.x == 0) atomicOr(&a.ctl->nonfinite_y, 1);
}

}  // namespace pfe_dev
