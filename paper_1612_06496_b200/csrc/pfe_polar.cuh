// Orthogonality projection P = polar(A), A = sqrt(D) Y + B (solver.cpp:27-41,
// 116-118), as a communication-avoiding TSQR:
//
//   k_tsqr_local  each block folds its contiguous rows of A, tile by tile,
//                 into a D x D triangular factor with Householder QR held in
//                 registers (thread t owns row t of the (D+T) x D stack).
//   k_tsqr_final  one block folds the per-block factors into R, runs a
//                 parallel one-sided Jacobi SVD R V = U S, checks rank the way
//                 the reference does (s_i <= 1e-12 max(1, s_max)) and forms
//                 W = V S^-1 V^T, so that P = A W = Q U V^T.
//   k_project_apply  P = A W, B += sqrt(D) Y - P and the next rhs_quad in
//                 one pass.
//
// Householder QR keeps the accuracy of the reference's JacobiSVD (backward
// stable, no Gram squaring), so rank deficiency is detected at the same
// 1e-12 threshold; the result is the same unique polar factor.
#pragma once

#include <utility>

#include "pfe_device.cuh"

namespace pfe_dev {

constexpr int kQrRows = kBlock;  // rows of the stacked [R; tile] matrix

// Block-wide sum of NV values per thread (all 256 threads participate);
// every thread receives the totals.  Fixed order => deterministic.
template <int NV>
__device__ __forceinline__ void block_allsum(double (&x)[NV]) {
  __shared__ double red[kBlock / 32][NV];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int o = 16; o >= 1; o >>= 1)
#pragma unroll
    for (int i = 0; i < NV; ++i) x[i] += __shfl_xor_sync(0xffffffffu, x[i], o);
  __syncthreads();
  if (lane == 0)
#pragma unroll
    for (int i = 0; i < NV; ++i) red[warp][i] = x[i];
  __syncthreads();
#pragma unroll
  for (int i = 0; i < NV; ++i) {
    double s = 0.0;
#pragma unroll
    for (int w = 0; w < kBlock / 32; ++w) s += red[w][i];
    x[i] = s;
  }
}

// In-place Householder QR of the kQrRows x D matrix whose row t lives in
// thread t's registers.  Afterwards rows 0..D-1 hold R, the rest are zero.
//
// Step K reduces over the block only what it needs: sum_{t>K} a_tK^2 and
// sum_{t>K} a_tK a_tj for j > K (D - K values), and takes row K from shared
// memory, written by thread K.  (Round 1 all-reduced 1 + 2D values in every
// step -- the unused dot products and row K as a sum of one value and 255
// zeros -- and the kernel was bound by its shuffles: C4 5.0 ms per
// projection.  The reduced values keep their summation tree and the
// broadcast its rounding -- "+ 0.0" is what summing a value with zeros does
// to -0.0 -- so R is bit for bit what it was.)
template <int D, int K>
__device__ __forceinline__ void householder_step(double (&row)[D], double (&bc)[D][D]) {
  constexpr int NV = D - K;
  constexpr int NW = kBlock / 32;
  __shared__ double part[NW][D];  // per-warp sums
  __shared__ double coef[D + 2];  // [0] alpha, [1] v0, [2..] tau * w_j for j = K+1.., written by warp 0
  __shared__ int skip;            // zero column: nothing to annihilate
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  double red[NV];  // [0]: sum_{t>K} a_tK^2 ; [j-K]: sum_{t>K} a_tK a_tj, j = K+1..D-1
#pragma unroll
  for (int i = 0; i < NV; ++i) red[i] = 0.0;
  if (t > K) {
    red[0] = row[K] * row[K];
#pragma unroll
    for (int j = K + 1; j < D; ++j) red[j - K] = row[K] * row[j];
  } else if (t == K) {
#pragma unroll
    for (int j = K; j < D; ++j) bc[K][j] = row[j] + 0.0;
  }
  // the same tree as block_allsum: warp butterfly, then the warps in order
#pragma unroll
  for (int o = 16; o >= 1; o >>= 1)
#pragma unroll
    for (int i = 0; i < NV; ++i) red[i] += __shfl_xor_sync(0xffffffffu, red[i], o);
  if (lane == 0)
#pragma unroll
    for (int i = 0; i < NV; ++i) part[warp][i] = red[i];
  __syncthreads();
  // Warp 0 finishes the totals and the step's scalars once for the block
  // (every thread used to repeat the 8 * NV additions, the square root and
  // the division; the FP64 pipe was the kernel's limit): lane i owns total i.
  if (warp == 0) {
    double tot = 0.0;
    if (lane < NV)
#pragma unroll
      for (int w = 0; w < NW; ++w) tot += part[w][lane];
    double v0 = 0.0, tau = 0.0;
    if (lane == 0) {
      const double x0 = bc[K][K];
      const double nrm = sqrt(x0 * x0 + tot);
      skip = nrm == 0.0 ? 1 : 0;
      const double alpha = x0 > 0.0 ? -nrm : nrm;
      v0 = x0 - alpha;
      tau = 2.0 / (v0 * v0 + tot);
      coef[0] = alpha;
      coef[1] = v0;
    }
    v0 = __shfl_sync(0xffffffffu, v0, 0);
    tau = __shfl_sync(0xffffffffu, tau, 0);
    if (lane >= 1 && lane < NV) {
      const double wj = v0 * bc[K][K + lane] + tot;
      coef[1 + lane] = tau * wj;
    }
  }
  __syncthreads();
  if (skip) return;
  const double vt = (t == K) ? coef[1] : (t > K ? row[K] : 0.0);
  if (t >= K) {
#pragma unroll
    for (int j = K + 1; j < D; ++j) row[j] -= coef[1 + (j - K)] * vt;
    row[K] = (t == K) ? coef[0] : 0.0;
  }
}
template <int D, int... Ks>
__device__ __forceinline__ void householder_steps(double (&row)[D], double (&bc)[D][D], std::integer_sequence<int, Ks...>) {
  (householder_step<D, Ks>(row, bc), ...);
}
template <int D>
__device__ __forceinline__ void householder_fold(double (&row)[D]) {
  __shared__ double bc[D][D];  // row K of step K (columns K..D-1)
  householder_steps<D>(row, bc, std::make_integer_sequence<int, D>{});
}

// A row: sqd ? (sqrt(d_v) * y_v + B_v) : y_v   (solver.cpp:116-117)
template <int D>
__device__ __forceinline__ void load_a_row(double (&row)[D], long v, const double* __restrict__ y,
                                           const double* __restrict__ sqd, const double* __restrict__ breg) {
  const Row<D> yr = ldg_row<D>(y + v * D);  // the row as 16 / 32-byte pieces
  if (sqd) {
    const double s = __ldg(sqd + v);
    const Row<D> br = ldg_row<D>(breg + v * D);
#pragma unroll
    for (int k = 0; k < D; ++k) row[k] = s * yr.a[k] + br.a[k];
  } else {
#pragma unroll
    for (int k = 0; k < D; ++k) row[k] = yr.a[k];
  }
}

template <int D>
__global__ void __launch_bounds__(kBlock) k_tsqr_local(int n, const double* __restrict__ y,
                                                      const double* __restrict__ sqd,
                                                      const double* __restrict__ breg, double* rbuf) {
  constexpr int T = kQrRows - D;
  const long per = (static_cast<long>(n) + gridDim.x - 1) / gridDim.x;
  const long lo = per * blockIdx.x, hi = min(static_cast<long>(n), lo + per);
  const int t = threadIdx.x;
  double row[D];
#pragma unroll
  for (int k = 0; k < D; ++k) row[k] = 0.0;
  for (long base = lo; base < hi; base += T) {
    if (t >= D) {
      const long v = base + (t - D);
      if (v < hi) {
        load_a_row<D>(row, v, y, sqd, breg);
      } else {
#pragma unroll
        for (int k = 0; k < D; ++k) row[k] = 0.0;
      }
    }
    householder_fold<D>(row);
  }
  if (t < D)
#pragma unroll
    for (int k = 0; k < D; ++k) rbuf[(static_cast<long>(blockIdx.x) * D + t) * D + k] = row[k];
}

// Single block.  W (row-major D x D) receives V S^-1 V^T; ctl->deficient the
// number of singular values at or below 1e-12 * max(1, s_max).
template <int D>
__global__ void __launch_bounds__(kBlock) k_tsqr_final(int nblk, const double* __restrict__ rbuf, double* wout,
                                                      Ctl* ctl) {
  constexpr int T = kQrRows - D;
  constexpr int DP = (D % 2) ? D + 1 : D;  // padded to even for round-robin pairing
  const int t = threadIdx.x;
  double row[D];
#pragma unroll
  for (int k = 0; k < D; ++k) row[k] = 0.0;
  const long rows = static_cast<long>(nblk) * D;
  for (long base = 0; base < rows; base += T) {
    if (t >= D) {
      const long i = base + (t - D);
#pragma unroll
      for (int k = 0; k < D; ++k) row[k] = (i < rows) ? rbuf[i * D + k] : 0.0;
    }
    householder_fold<D>(row);
  }
  // One-sided Jacobi on the columns of R: R V = U S.
  __shared__ double Rm[D][DP];
  __shared__ double Vm[DP][DP];
  __shared__ int done;
  __shared__ double offmax[kBlock / 16];
  if (t < D)
#pragma unroll
    for (int k = 0; k < D; ++k) Rm[t][k] = row[k];
  for (int i = t; i < D * DP; i += kBlock)
    if (i % DP >= D) Rm[i / DP][i % DP] = 0.0;
  for (int i = t; i < DP * DP; i += kBlock) Vm[i / DP][i % DP] = (i / DP == i % DP) ? 1.0 : 0.0;
  __syncthreads();
  const int pair = t >> 4, ri = t & 15;  // 16 threads per column pair; ri = row index
  for (int sweep = 0; sweep < 40; ++sweep) {
    double local_off = 0.0;
    for (int step = 0; step < DP - 1; ++step) {
      int p = -1, q = -1;
      if (pair < DP / 2) {
        if (pair == 0) {
          p = DP - 1;
          q = step;
        } else {
          p = (step + pair) % (DP - 1);
          q = (step - pair + DP - 1) % (DP - 1);
        }
      }
      double al = 0.0, be = 0.0, ga = 0.0;
      if (p >= 0 && ri < D) {
        const double x = Rm[ri][p], y = Rm[ri][q];
        al = x * x;
        be = y * y;
        ga = x * y;
      }
#pragma unroll
      for (int o = 8; o >= 1; o >>= 1) {
        al += __shfl_xor_sync(0xffffffffu, al, o);
        be += __shfl_xor_sync(0xffffffffu, be, o);
        ga += __shfl_xor_sync(0xffffffffu, ga, o);
      }
      double cs = 1.0, sn = 0.0;
      bool rot = false;
      if (p >= 0 && ga != 0.0 && al > 0.0 && be > 0.0) {
        const double rel = fabs(ga) / sqrt(al * be);
        if (rel > 1e-15) {
          local_off = fmax(local_off, rel);
          const double zeta = (be - al) / (2.0 * ga);
          const double tt = (zeta >= 0.0 ? 1.0 : -1.0) / (fabs(zeta) + sqrt(1.0 + zeta * zeta));
          cs = 1.0 / sqrt(1.0 + tt * tt);
          sn = cs * tt;
          rot = true;
        }
      }
      __syncthreads();
      if (rot) {
        if (ri < D) {
          const double x = Rm[ri][p], y = Rm[ri][q];
          Rm[ri][p] = cs * x - sn * y;
          Rm[ri][q] = sn * x + cs * y;
        }
        if (ri < DP) {
          const double x = Vm[ri][p], y = Vm[ri][q];
          Vm[ri][p] = cs * x - sn * y;
          Vm[ri][q] = sn * x + cs * y;
        }
      }
      __syncthreads();
    }
#pragma unroll
    for (int o = 8; o >= 1; o >>= 1) local_off = fmax(local_off, __shfl_xor_sync(0xffffffffu, local_off, o));
    if (ri == 0) offmax[pair] = local_off;
    __syncthreads();
    if (t == 0) {
      double m = 0.0;
      for (int i = 0; i < kBlock / 16; ++i) m = fmax(m, offmax[i]);
      done = m <= 1e-15;
    }
    __syncthreads();
    if (done) break;
  }
  __shared__ double sig[DP];
  if (t < D) {
    double s = 0.0;
    for (int i = 0; i < D; ++i) s += Rm[i][t] * Rm[i][t];
    sig[t] = sqrt(s);
  }
  __syncthreads();
  if (t == 0) {
    double smax = 0.0;
    for (int j = 0; j < D; ++j) smax = fmax(smax, sig[j]);
    const double tol = 1e-12 * fmax(1.0, smax);
    int def = 0;
    for (int j = 0; j < D; ++j) def += sig[j] <= tol;
    ctl->deficient = def;
  }
  for (int i = t; i < D * D; i += kBlock) {
    const int r = i / D, c = i % D;
    double s = 0.0;
    for (int j = 0; j < D; ++j) s += Vm[r][j] * (Vm[c][j] / sig[j]);
    wout[i] = s;
  }
}

// P = A W; B' = B + (dy - P); rq' = (r/2) * (sqrt(d) * (P - B'))
// (solver.cpp:116-118 fused with the next split_bregman's rhs_quad, 79-80).
// With sqd == null: plain P = A W for the standalone projection.
template <int D>
__global__ void __launch_bounds__(kBlock) k_project_apply(int n, const double* __restrict__ y,
                                                         const double* __restrict__ sqd, double* breg,
                                                         const double* __restrict__ wmat, double* pout, double* rq,
                                                         double hr) {
  __shared__ double W[D * D];
  for (int i = threadIdx.x; i < D * D; i += blockDim.x) W[i] = wmat[i];
  __syncthreads();
  const long stride = static_cast<long>(gridDim.x) * blockDim.x;
  // one row per thread, moved as whole 16 / 32-byte pieces (the scalar
  // version wrote three arrays 8 bytes at a time from 32 rows per warp)
  for (long v = static_cast<long>(blockIdx.x) * blockDim.x + threadIdx.x; v < n; v += stride) {
    double dy[D], a[D];
    const Row<D> yr = ldg_row<D>(y + v * D);
    Row<D> br;
    double sq = 0.0;
    if (sqd) {
      sq = __ldg(sqd + v);
      br = ld_row<D>(breg + v * D);
#pragma unroll
      for (int k = 0; k < D; ++k) {
        dy[k] = sq * yr.a[k];
        a[k] = dy[k] + br.a[k];
      }
    } else {
#pragma unroll
      for (int k = 0; k < D; ++k) a[k] = yr.a[k];
    }
    Row<D> po, bnew, rqv;
#pragma unroll
    for (int j = 0; j < D; ++j) {
      double s = 0.0;
#pragma unroll
      for (int k = 0; k < D; ++k) s += a[k] * W[k * D + j];
      po.a[j] = s;
      if (sqd) {
        const double bn = br.a[j] + (dy[j] - s);
        bnew.a[j] = bn;
        rqv.a[j] = hr * (sq * (s - bn));
      }
    }
    st_row<D>(pout + v * D, po);
    if (sqd) {
      st_row<D>(breg + v * D, bnew);
      st_row<D>(rq + v * D, rqv);
    }
  }
}

}  // namespace pfe_dev
