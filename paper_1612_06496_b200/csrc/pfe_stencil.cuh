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
#include "pfe_tma.cuh"

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
  // Shared-memory layouts (offsets in doubles, every array 128-byte aligned
  // so it can be a TMA destination).  Everything is position-major: rows
  // [pos][D], weights / coefficients [pos][S], b_old [opos][S][D] -- the
  // layout of the global arrays, so a halo box is one rectangular copy.
  static constexpr int al(int x) { return (x + 15) / 16 * 16; }
  // init: x0 halo, coefficient halo, rhs / diag / inv diag interior
  static constexpr int kI_W = al(NP * D), kI_B = kI_W + al(NP * S), kI_Dg = kI_B + al(NV * D),
                       kI_Iv = kI_Dg + al(NV), kInit = kI_Iv + al(NV);
  // spmv: p_old halo, r halo, inv diag halo, coefficient halo, diag interior
  static constexpr int kS_Rs = al(NP * D), kS_Iv = kS_Rs + al(NP * D), kS_W = kS_Iv + al(NP),
                       kS_Dg = kS_W + al(NP * S), kSpmv = kS_Dg + al(NV);
  // sb pass: Y halo, weight halo, rq interior, b_old of owners (8-nbr only)
  static constexpr int kB_W = al(NP * D), kB_Rq = kB_W + al(NP * S), kB_Bo = kB_Rq + al(NV * D),
                       kSb = kB_Bo + (kStageB ? al(NO * S * D) : 0);
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

// Bulk staging (cp.async.bulk): row hy of a tile box is one contiguous run
// of a row-major [H][W][K] array, so it is one bulk copy of its in-image
// part instead of (BW * K / 2) 16-byte cp.async with per-element address
// arithmetic.  Lanes of warp 0 issue one row each, after lane 0 posted the
// bytes (span_bytes) on the buffer's mbarrier.  Positions outside the image
// are zero-filled with ordinary stores by span_zero (border tiles only).
struct Span {
  int r0, r1;  // box rows [r0, r1) inside the image
  int c0, c1;  // box columns [c0, c1) inside the image
  int ylo, xlo;
};
// Box of bw x nrows positions with top-left image position (xlo, ylo); rows
// at or past ymax and columns past W are outside.
template <int R>
__device__ __forceinline__ Span box_span(const Grid<R>& g, int xlo, int ylo, int bw, int nrows, int ymax) {
  Span sp;
  sp.ylo = ylo;
  sp.xlo = xlo;
  sp.r0 = ylo < 0 ? -ylo : 0;
  sp.r1 = ylo + nrows > ymax ? ymax - ylo : nrows;
  sp.c0 = xlo < 0 ? -xlo : 0;
  sp.c1 = xlo + bw > g.W ? g.W - xlo : bw;
  if (sp.r1 < sp.r0) sp.r1 = sp.r0;
  if (sp.c1 < sp.c0) sp.c1 = sp.c0;
  return sp;
}
template <int K>
__device__ __forceinline__ uint32_t span_bytes(const Span& sp) {
  return static_cast<uint32_t>((sp.r1 - sp.r0) * (sp.c1 - sp.c0) * K * 8);
}
template <int K, int BW, int R>
__device__ __forceinline__ void span_issue(const Grid<R>& g, const Span& sp, const double* __restrict__ src,
                                           double* dst, uint64_t* bar, int lane) {
  if constexpr (K % 2 != 0) {
    return;  // odd widths never stage in bulk (the host requires even d)
  } else {
  if (sp.c1 <= sp.c0) return;
  const uint32_t bytes = static_cast<uint32_t>((sp.c1 - sp.c0) * K * 8);
  for (int hy = sp.r0 + lane; hy < sp.r1; hy += 32) {
    const long u = static_cast<long>(sp.ylo + hy) * g.W + (sp.xlo + sp.c0);
    bulk_copy(dst + (hy * BW + sp.c0) * K, src + u * K, bytes, bar);
  }
  }
}
template <int K, int BW, int NT>
__device__ __forceinline__ void span_zero(const Span& sp, double* dst, int nrows) {
  if constexpr (K % 2 != 0) return;
  if (sp.r0 == 0 && sp.r1 == nrows && sp.c0 == 0 && sp.c1 == BW) return;
  constexpr int PER = K / 2 > 0 ? K / 2 : 1;
  const int total = nrows * BW * PER;
  for (int c = threadIdx.x; c < total; c += NT) {
    const int pos = c / PER, k = (c - pos * PER) * 2;
    const int hy = pos / BW, hx = pos - hy * BW;
    if (hy < sp.r0 || hy >= sp.r1 || hx < sp.c0 || hx >= sp.c1)
      *reinterpret_cast<double2*>(dst + pos * K + k) = make_double2(0.0, 0.0);
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
// slots, diagonal, forward slots.  Ct is position-major [NP][S] and holds the
// off-diagonal entries -((hl w) w) (Grid::cf, sparse.cpp:114), +0.0 for an
// absent edge: a present edge's entry always has its sign bit set (it is
// negative, or -0.0 if hl w^2 underflows), so the sign bit is the presence test.
template <int D, int R>
__device__ __forceinline__ double tile_apply_A(const double* P, const double* Ct, int hpos, int c, double diag_v) {
  using G = TileGeo<R, D>;
  using T = GridTopo<R>;
  // branch-free: every term is loaded and formed, absent edges are skipped by
  // a select, so all loads are in flight before the serial reference-order
  // additions
  double t[2 * G::S + 1];
  bool nz[2 * G::S + 1];
#pragma unroll
  for (int j = 0; j < G::S; ++j) {
    const int s = G::S - 1 - j;
    const int npos = hpos - T::dy(s) * G::HW - T::dx(s);
    const double cw = Ct[npos * G::S + s];
    nz[j] = __double_as_longlong(cw) < 0;
    t[j] = cw * P[npos * D + c];
  }
  nz[G::S] = true;
  t[G::S] = diag_v * P[hpos * D + c];
#pragma unroll
  for (int s = 0; s < G::S; ++s) {
    const int npos = hpos + T::dy(s) * G::HW + T::dx(s);
    const double cw = Ct[hpos * G::S + s];
    nz[G::S + 1 + s] = __double_as_longlong(cw) < 0;
    t[G::S + 1 + s] = cw * P[npos * D + c];
  }
  double q = 0.0;
#pragma unroll
  for (int j = 0; j < 2 * G::S + 1; ++j) q = nz[j] ? q + t[j] : q;
  return q;
}

// Pair mode (even D, NV * D == 4 * NT): a thread evaluates two vertically
// adjacent pixels (tile rows 2i and 2i + 1) for two adjacent columns.  The
// terms of a row of A, in the order tile_apply_A adds them (backward slots
// S-1..0, the diagonal, forward slots 0..S-1), are exactly the positions of
// the (2R+1) x (2R+1) window around the pixel in raster order.  The pair
// therefore walks the (2R+2) x (2R+1) window covering both pixels row by
// row: every P position is read once (16 bytes: both columns) and used by
// both pixels, each pixel still adding its terms in its own raster order.
// Same products, same selected additions in the same sequence as
// tile_apply_A -- bitwise the same q -- with about a quarter of the
// shared-memory load instructions (the stencil phases were bound by those,
// profiles/r01/ncu_k_sb_persistent_c3.txt).
template <int R, int D>
struct PairMode {
  using G = TileGeo<R, D>;
  static constexpr bool kOn = (D % 2 == 0) && (G::NV * D == 4 * G::NT) && (G::TH % 2 == 0);
  static constexpr int CP = D / 2;  // column pairs per pixel
  static constexpr int V = kOn ? 2 : G::V;  // columns a thread accumulates (partial sums)
};

// forward slot of offset (dy, dx) (dy > 0, or dy == 0 and dx > 0)
template <int R>
__host__ __device__ constexpr int fwd_slot(int dy, int dx) {
  return dy == 0 ? dx - 1 : R + (dy - 1) * (2 * R + 1) + (dx + R);
}

// The thread's pixel pair: f(tv, hpos, v, c0, q[2], pv[2]) for each pixel of
// the pair inside the image, q = (A p)_v and pv = p_v for columns c0, c0 + 1.
template <int R, int D, class F>
__device__ __forceinline__ void for_tile_pairs(const Grid<R>& g, TileIdx ti, const double* P, const double* Ct,
                                               const double* Dg, F&& f) {
  using G = TileGeo<R, D>;
  constexpr int CP = PairMode<R, D>::CP;
  constexpr int WS = 2 * R + 1;
  const int c0 = (threadIdx.x % CP) * 2;
  const int pi = threadIdx.x / CP;
  const int tx = pi % G::TW, tyA = (pi / G::TW) * 2;
  const int x = ti.x0 + tx, yA = ti.y0 + tyA;
  if (x >= g.W || yA >= g.row_hi) return;
  const bool hasB = yA + 1 < g.row_hi;
  const int cA = (tyA + R) * G::HW + (tx + R), cB = cA + G::HW;  // centres (halo positions)
  double qa0 = 0.0, qa1 = 0.0, qb0 = 0.0, qb1 = 0.0;
  double2 pa{}, pb{};
#pragma unroll
  for (int wr = 0; wr <= 2 * R + 1; ++wr) {
    double2 row[WS];
#pragma unroll
    for (int wc = 0; wc < WS; ++wc)
      row[wc] = *reinterpret_cast<const double2*>(P + ((tyA + wr) * G::HW + tx + wc) * D + c0);
    // pixel A: window row wr = offset dy = wr - R; pixel B: dy = wr - 1 - R
#pragma unroll
    for (int who = 0; who < 2; ++who) {
      const int dy = who == 0 ? wr - R : wr - 1 - R;
      if (dy < -R || dy > R) continue;
      const int cpos = who == 0 ? cA : cB;
      double& q0 = who == 0 ? qa0 : qb0;
      double& q1 = who == 0 ? qa1 : qb1;
#pragma unroll
      for (int wc = 0; wc < WS; ++wc) {
        const int dx = wc - R;
        const double2 pv = row[wc];
        if (dy == 0 && dx == 0) {  // the diagonal
          const double dg = Dg[(tyA + who) * G::TW + tx];
          q0 = q0 + dg * pv.x;
          q1 = q1 + dg * pv.y;
          if (who == 0) pa = pv; else pb = pv;
          continue;
        }
        const bool bwd = dy < 0 || (dy == 0 && dx < 0);
        const int s = bwd ? fwd_slot<R>(-dy, -dx) : fwd_slot<R>(dy, dx);
        const int npos = cpos + dy * G::HW + dx;
        const double cw = Ct[(bwd ? npos : cpos) * G::S + s];
        const bool nz = __double_as_longlong(cw) < 0;
        const double t0 = cw * pv.x, t1 = cw * pv.y;
        q0 = nz ? q0 + t0 : q0;
        q1 = nz ? q1 + t1 : q1;
      }
    }
  }
  {
    const double q[2] = {qa0, qa1}, pv[2] = {pa.x, pa.y};
    f(tyA * G::TW + tx, cA, static_cast<long>(yA) * g.W + x, c0, q, pv);
  }
  if (hasB) {
    const double q[2] = {qb0, qb1}, pv[2] = {pb.x, pb.y};
    f((tyA + 1) * G::TW + tx, cB, static_cast<long>(yA + 1) * g.W + x, c0, q, pv);
  }
}

// PCG init of one staged tile (pcg.cpp:49-66): r = b - A x0, z = D^-1 r,
// partial sums of b.b, r.r, r.z per column.
template <int R, int D, int V>
__device__ __forceinline__ void tile_init_body(const Grid<R>& g, TileIdx ti, const double* P, const double* Wt,
                                               const double* Bv, const double* Dg, const double* Iv, double* r_out,
                                               double* z_out, double (&acc)[3][V]) {
  if constexpr (PairMode<R, D>::kOn) {
    for_tile_pairs<R, D>(g, ti, P, Wt, Dg, [&](int tv, int, long v, int c0, const double (&q)[2], const double (&)[2]) {
      const double2 b = *reinterpret_cast<const double2*>(Bv + tv * D + c0);
      const double iv = Iv[tv];
      const double r0 = b.x - q[0], r1 = b.y - q[1];
      const double z0 = iv * r0, z1 = iv * r1;
      *reinterpret_cast<double2*>(r_out + v * D + c0) = make_double2(r0, r1);
      *reinterpret_cast<double2*>(z_out + v * D + c0) = make_double2(z0, z1);
      acc[0][0] += b.x * b.x;
      acc[0][1] += b.y * b.y;
      acc[1][0] += r0 * r0;
      acc[1][1] += r1 * r1;
      acc[2][0] += r0 * z0;
      acc[2][1] += r1 * z1;
    });
  } else {
    for_tile_elements<R, D>(g, ti, [&](int tv, int c, int hpos, long v, int k) {
      const double ax = tile_apply_A<D, R>(P, Wt, hpos, c, Dg[tv]);
      const double b = Bv[tv * D + c];
      const double r = b - ax;
      const double z = Iv[tv] * r;
      r_out[v * D + c] = r;
      z_out[v * D + c] = z;
      acc[0][k] += b * b;
      acc[1][k] += r * r;
      acc[2][k] += r * z;
    });
  }
}

// PCG SpMV of one staged tile (P holds p' on the halo): q = A p', p' stored
// to pnew (unless null), partial sums of p'.q per column.
template <int R, int D, int V>
__device__ __forceinline__ void tile_spmv_body(const Grid<R>& g, TileIdx ti, const double* P, const double* Wt,
                                               const double* Dg, double* q_out, double* pnew, double (&acc)[1][V]) {
  if constexpr (PairMode<R, D>::kOn) {
    for_tile_pairs<R, D>(g, ti, P, Wt, Dg,
                         [&](int, int, long v, int c0, const double (&q)[2], const double (&pv)[2]) {
                           *reinterpret_cast<double2*>(q_out + v * D + c0) = make_double2(q[0], q[1]);
                           if (pnew) *reinterpret_cast<double2*>(pnew + v * D + c0) = make_double2(pv[0], pv[1]);
                           acc[0][0] += pv[0] * q[0];
                           acc[0][1] += pv[1] * q[1];
                         });
  } else {
    for_tile_elements<R, D>(g, ti, [&](int tv, int c, int hpos, long v, int k) {
      const double qv = tile_apply_A<D, R>(P, Wt, hpos, c, Dg[tv]);
      const double pv = P[hpos * D + c];
      q_out[v * D + c] = qv;
      if (pnew) pnew[v * D + c] = pv;
      acc[0][k] += pv * qv;
    });
  }
}

// ---------------------------------------------------------------- init ----
template <int D, int R>
__global__ void __launch_bounds__(TileGeo<R, D>::NT) k_grid_pcg_init(Grid<R> g, PcgArgs a) {
  using G = TileGeo<R, D>;
  constexpr int V = PairMode<R, D>::V;
  extern __shared__ double smem[];
  double* P = smem;                  // x0 halo [NP][D]
  double* Wt = smem + G::kI_W;       // coefficients [NP][S]
  double* Bv = smem + G::kI_B;       // rhs interior [NV][D]
  double* Dg = smem + G::kI_Dg;      // diag interior [NV]
  double* Iv = smem + G::kI_Iv;      // inv diag interior [NV]
  double acc[3][V] = {};
  const int nt = num_tiles<R, D>(g);
  for (int t = blockIdx.x; t < nt; t += gridDim.x) {
    const TileIdx ti = tile_of<R, D>(g, t);
    stage_rows<R, D, D>(g, ti, a.x0, P, G::HH);
    stage_rows<R, D, G::S>(g, ti, g.cf, Wt, G::HH);
    stage_interior<R, D, D>(g, ti, a.rhs, Bv);
    stage_interior<R, D, 1>(g, ti, g.diag, Dg);
    stage_interior<R, D, 1>(g, ti, g.invd, Iv);
    cp_async_wait_all();
    __syncthreads();
    tile_init_body<R, D, V>(g, ti, P, Wt, Bv, Dg, Iv, a.r, a.pbuf[0], acc);
    __syncthreads();
  }
  store_partials<3, D, V, G::NT>(a, acc, a.part_a, a.tot_a);  // reduced by the first SpMV
}

// ---------------------------------------------------------------- spmv ----
template <int D, int R>
__global__ void __launch_bounds__(TileGeo<R, D>::NT) k_grid_pcg_spmv(Grid<R> g, PcgArgs a) {
  using G = TileGeo<R, D>;
  constexpr int V = PairMode<R, D>::V;
  extern __shared__ double smem[];
  double* P = smem;                  // p (phase 0) or p_old -> p' in place [NP][D]
  double* Rs = smem + G::kS_Rs;      // r halo [NP][D]
  double* Iv = smem + G::kS_Iv;      // inv diag halo [NP]
  double* Wt = smem + G::kS_W;       // coefficients [NP][S]
  double* Dg = smem + G::kS_Dg;      // diag interior [NV]
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
    stage_rows<R, D, G::S>(g, ti, g.cf, Wt, G::HH);
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
    tile_spmv_body<R, D, V>(g, ti, P, Wt, Dg, a.q, first ? nullptr : pnew, acc);
    if (!first && (g.row_lo > 0 || g.row_hi < g.H)) {
      // Row band: the halo rows of p' above / below the band were formed in
      // shared memory from exchanged r and the previous p (bit-identical to
      // the neighbouring band's own p'); storing them saves the halo
      // exchange of p before the next SpMV (pcg.cpp:86-88).
      const int top0 = ti.y0 == g.row_lo ? max(g.row_lo - R, 0) : 0, top1 = ti.y0 == g.row_lo ? g.row_lo : 0;
      const bool bot = ti.y0 + G::TH >= g.row_hi;
      const int bot0 = bot ? g.row_hi : 0, bot1 = bot ? min(g.row_hi + R, g.H) : 0;
      const int cols = min(G::TW, g.W - ti.x0);
      for (int band = 0; band < 2; ++band) {
        const int y0 = band == 0 ? top0 : bot0, y1 = band == 0 ? top1 : bot1;
        const int cnt = (y1 - y0) * cols * D;
        for (int e = threadIdx.x; e < cnt; e += G::NT) {
          const int pix = e / D, c = e - pix * D;
          const int y = y0 + pix / cols, x = ti.x0 + pix % cols;
          const int hpos = (y - ti.y0 + R) * G::HW + (x - ti.x0 + R);
          pnew[(static_cast<long>(y) * g.W + x) * D + c] = P[hpos * D + c];
        }
      }
    }
    __syncthreads();
  }
  if (!checked && !spmv_prologue<D, G::NT>(a, cv)) return;  // block without tiles
  store_partials<1, D, V, G::NT>(a, acc, a.part_b, a.tot_b);  // reduced by the update
}

// ----------------------------------------------------- split-Bregman pass -
// One (vertex, column) element of the pass from a staged tile: every incident
// edge in edge order (backward slots S-1..0, owned by neighbours, then forward
// slots 0..S-1, owned by v) evaluated as solver.cpp:96-98; returns
// sum_e M_ev (s_e - b_e') for the next rhs (solver.cpp:83-84).  The owner
// stores b' (and s); in a row band, edges owned by the halo rows above are
// replicas this band updates identically (vy = image row of v).  b_old comes from the staged
// owner planes Bo (8-neighbour grids) or from global memory, in which case
// all 2S loads are issued before the first use (one round trip, not 2S).
template <int D, int R, bool kNc>
__device__ __forceinline__ double tile_sb_element(const Grid<R>& g, const double* P, const double* Wt, const double* Bo,
                                                  const double* __restrict__ b_old, double* b_new, double* s_out,
                                                  double gamma, int hpos, int c, long v, int vy, int vx) {
  using G = TileGeo<R, D>;
  using T = GridTopo<R>;
  double bo[2 * G::S];
#pragma unroll
  for (int e = 0; e < 2 * G::S; ++e) {
    const bool fwd = e >= G::S;
    const int s = fwd ? e - G::S : G::S - 1 - e;
    const int opos = fwd ? hpos : hpos - T::dy(s) * G::HW - T::dx(s);
    bo[e] = 0.0;
    // staged: only present edges are read (the staged owner rows may be
    // stale for absent ones); global: every edge whose owner lies inside the
    // stored rows has a slot (absent edges hold zeros and are skipped
    // below), so the load needs no shared-memory weight first
    const bool valid = G::kStageB ? Wt[opos * G::S + s] != 0.0
                                  : (fwd || (vy - T::dy(s) >= 0 && vx - T::dx(s) >= 0 && vx - T::dx(s) < g.W));
    if (b_old && valid) {
      if constexpr (G::kStageB) {
        bo[e] = Bo[(opos * G::S + s) * D + c];
      } else {
        const long slot = fwd ? v * G::S + s : (v - T::dy(s) * g.W - T::dx(s)) * G::S + s;
        // kNc: b_old is read-only for this launch (multi-kernel path: the
        // non-coherent path); else it was written earlier in the same
        // persistent launch, before a grid barrier: a plain (coherent) load,
        // still L1-cached so the other endpoint's read of the edge can hit
        bo[e] = kNc ? __ldg(b_old + slot * D + c) : b_old[slot * D + c];
      }
    }
  }
  double acc = 0.0;
#pragma unroll
  for (int e = 0; e < 2 * G::S; ++e) {
    const bool fwd = e >= G::S;
    const int s = fwd ? e - G::S : G::S - 1 - e;
    const int npos = fwd ? hpos + T::dy(s) * G::HW + T::dx(s) : hpos - T::dy(s) * G::HW - T::dx(s);
    const int opos = fwd ? hpos : npos;  // owner = first endpoint i
    const int jpos = fwd ? npos : hpos;
    const double w = Wt[opos * G::S + s];
    if (w == 0.0) continue;
    const double nw = -w;
    const double my = w * P[opos * D + c] + nw * P[jpos * D + c];
    const double sh = shrink1(my + bo[e], gamma);
    const double bn = bo[e] + (my - sh);
    acc += (fwd ? w : nw) * (sh - bn);
    if (fwd || vy - T::dy(s) < g.row_lo) {
      const long slot = fwd ? v * G::S + s : (v - T::dy(s) * g.W - T::dx(s)) * G::S + s;
      b_new[slot * D + c] = bn;
      if (s_out) s_out[slot * D + c] = sh;
    }
  }
  return acc;
}

// Column-pair form of tile_sb_element (even D): one pixel, columns c0 and
// c0 + 1, every shared / global access 16 bytes wide (half the load and
// store instructions of two elements).  The same operations per column, in
// the same order, so b', s and the rhs are bitwise those of
// tile_sb_element.  b_old is loaded for a group of incident edges at a time
// (all 2S edges in two groups for 8-neighbour grids, four groups of 6 for
// 5x5 grids), each group's loads issued before its first use.
template <int D, int R, bool kNc>
__device__ __forceinline__ double2 tile_sb_pair(const Grid<R>& g, const double* P, const double* Wt, const double* Bo,
                                                const double* __restrict__ b_old, double* b_new, double* s_out,
                                                double gamma, int hpos, int c0, long v, int vy, int vx) {
  using G = TileGeo<R, D>;
  using T = GridTopo<R>;
  double acc0 = 0.0, acc1 = 0.0;
  const double2 pself = *reinterpret_cast<const double2*>(P + hpos * D + c0);
  // edge e = 0 .. 2S-1 in edge order: backward slots S-1..0, then forward
  // slots 0..S-1; b_old of a group of GS edges is loaded before its first use
  constexpr int GS = G::S > 6 ? G::S / 2 : G::S;
#pragma unroll
  for (int e0 = 0; e0 < 2 * G::S; e0 += GS) {
    double2 bo[GS];
#pragma unroll
    for (int i = 0; i < GS; ++i) {
      const int e = e0 + i;
      const bool fwd = e >= G::S;
      const int s = fwd ? e - G::S : G::S - 1 - e;
      const int opos = fwd ? hpos : hpos - T::dy(s) * G::HW - T::dx(s);
      bo[i] = make_double2(0.0, 0.0);
      const bool valid = G::kStageB ? Wt[opos * G::S + s] != 0.0
                                    : (fwd || (vy - T::dy(s) >= 0 && vx - T::dx(s) >= 0 && vx - T::dx(s) < g.W));
      if (b_old && valid) {
        if constexpr (G::kStageB) {
          bo[i] = *reinterpret_cast<const double2*>(Bo + (opos * G::S + s) * D + c0);
        } else {
          const long slot = fwd ? v * G::S + s : (v - T::dy(s) * g.W - T::dx(s)) * G::S + s;
          const double2* src = reinterpret_cast<const double2*>(b_old + slot * D + c0);
          bo[i] = kNc ? __ldg(src) : *src;
        }
      }
    }
#pragma unroll
    for (int i = 0; i < GS; ++i) {
      const int e = e0 + i;
      const bool fwd = e >= G::S;
      const int s = fwd ? e - G::S : G::S - 1 - e;
      const int npos = fwd ? hpos + T::dy(s) * G::HW + T::dx(s) : hpos - T::dy(s) * G::HW - T::dx(s);
      const int opos = fwd ? hpos : npos;  // owner = first endpoint i
      const double w = Wt[opos * G::S + s];
      if (w == 0.0) continue;
      const double nw = -w;
      const double2 pn = *reinterpret_cast<const double2*>(P + npos * D + c0);
      const double2 pi = fwd ? pself : pn, pj = fwd ? pn : pself;
      const double my0 = w * pi.x + nw * pj.x, my1 = w * pi.y + nw * pj.y;
      const double sh0 = shrink1(my0 + bo[i].x, gamma), sh1 = shrink1(my1 + bo[i].y, gamma);
      const double bn0 = bo[i].x + (my0 - sh0), bn1 = bo[i].y + (my1 - sh1);
      const double cf = fwd ? w : nw;
      acc0 += cf * (sh0 - bn0);
      acc1 += cf * (sh1 - bn1);
      if (fwd || vy - T::dy(s) < g.row_lo) {
        const long slot = fwd ? v * G::S + s : (v - T::dy(s) * g.W - T::dx(s)) * G::S + s;
        *reinterpret_cast<double2*>(b_new + slot * D + c0) = make_double2(bn0, bn1);
        if (s_out) *reinterpret_cast<double2*>(s_out + slot * D + c0) = make_double2(sh0, sh1);
      }
    }
  }
  return make_double2(acc0, acc1);
}

// The split-Bregman pass over one staged tile (solver.cpp:83-84, 96-98):
// column pairs for even D, elements otherwise.  Returns nonzero if a Y
// value of the tile is not finite (solver.cpp:94).
template <int D, int R, bool kNc>
__device__ __forceinline__ int tile_sb_body(const Grid<R>& g, TileIdx ti, const double* P, const double* Wt,
                                            const double* Bo, const double* Rq, const double* __restrict__ b_old,
                                            double* b_new, double* s_out, double* rhs_out, double hl, double gamma) {
  using G = TileGeo<R, D>;
  int bad = 0;
  if constexpr (D % 2 == 0) {
    constexpr int CP = D / 2;
    for (int it = threadIdx.x; it < G::NV * CP; it += G::NT) {
      const int tv = it / CP, c0 = (it - tv * CP) * 2;
      const int ty = tv / G::TW, tx = tv - ty * G::TW;
      const int y = ti.y0 + ty, x = ti.x0 + tx;
      if (y >= g.row_hi || x >= g.W) continue;
      const int hpos = (ty + R) * G::HW + (tx + R);
      const long v = static_cast<long>(y) * g.W + x;
      const double2 pv = *reinterpret_cast<const double2*>(P + hpos * D + c0);
      bad |= !isfinite(pv.x) || !isfinite(pv.y);
      const double2 acc = tile_sb_pair<D, R, kNc>(g, P, Wt, Bo, b_old, b_new, s_out, gamma, hpos, c0, v, y, x);
      if (rhs_out) {
        const double2 rq = *reinterpret_cast<const double2*>(Rq + tv * D + c0);
        *reinterpret_cast<double2*>(rhs_out + v * D + c0) = make_double2(hl * acc.x + rq.x, hl * acc.y + rq.y);
      }
    }
  } else {
    for_tile_elements<R, D>(g, ti, [&](int tv, int c, int hpos, long v, int) {
      bad |= !isfinite(P[hpos * D + c]);
      const double acc = tile_sb_element<D, R, kNc>(g, P, Wt, Bo, b_old, b_new, s_out, gamma, hpos, c, v,
                                                    ti.y0 + hpos / G::HW - R, ti.x0 + hpos % G::HW - R);
      if (rhs_out) rhs_out[v * D + c] = hl * acc + Rq[tv * D + c];
    });
  }
  return bad;
}

// The pass over a tile grid (tile_sb_element per element).
template <int D, int R>
__global__ void __launch_bounds__(TileGeo<R, D>::NT) k_grid_sb_pass(Grid<R> g, SbArgs a) {
  using G = TileGeo<R, D>;
  using T = GridTopo<R>;
  extern __shared__ double smem[];
  double* P = smem;                 // Y halo [NP][D]
  double* Wt = smem + G::kB_W;      // weights [NP][S]
  double* Rq = smem + G::kB_Rq;     // rq interior [NV][D]
  double* Bo = smem + G::kB_Bo;     // b_old of owners [NO][S][D] (8-nbr only)
  const int nt = num_tiles<R, D>(g);
  int bad = 0;
  for (int t = blockIdx.x; t < nt; t += gridDim.x) {
    const TileIdx ti = tile_of<R, D>(g, t);
    stage_rows<R, D, D>(g, ti, a.y, P, G::HH);
    stage_rows<R, D, G::S>(g, ti, g.wf, Wt, G::HH);
    if (a.rhs) stage_interior<R, D, D>(g, ti, a.rq, Rq);
    if constexpr (G::kStageB) {
      if (a.b_old) stage_rows<R, D, G::S * D>(g, ti, a.b_old, Bo, G::TH + R);
    }
    cp_async_wait_all();
    __syncthreads();
    bad |= tile_sb_body<D, R, true>(g, ti, P, Wt, Bo, Rq, a.b_old, a.b_new, a.s_out, a.rhs, a.hl, a.gamma);
    __syncthreads();
  }
  if (__syncthreads_or(bad) && threadIdx.x == 0) atomicOr(&a.ctl->nonfinite_y, 1);
}

}  // namespace pfe_dev
