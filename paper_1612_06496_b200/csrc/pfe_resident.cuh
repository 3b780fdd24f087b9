// Shared-memory-resident persistent split-Bregman kernel for pixel grids
// whose PCG state fits in the SMs' shared memory (e.g. a 481x321 image at
// d = 4: 154k vertices x 18 doubles ~ 22 MB against 148 x 227 KB).
//
// Same algorithm and per-element arithmetic as k_sb_persistent (and so as
// PfeSolver::split_bregman, solver.cpp:82-107, with the Jacobi-PCG of
// pcg.cpp:40-113), different data placement.  The image is cut into
// rgx x rgy rectangular regions, one per block (one block per SM).  A block
// keeps its region plus an R-pixel ring of neighbour pixels in shared memory
// for the whole launch:
//
//   A1 [np][D]  p (PCG direction), and Y between PCG solves
//   A2 [np][D]  r (PCG residual), and the next rhs between passes
//   A3 [np][D]  x (PCG iterate; interior only)
//   Wt [S][np]  forward-slot weights, Iv [np] D^-1, Dg [np] diag(A)  (static)
//
// Only ring values cross blocks, through the global arrays at their natural
// positions: every block writes the boundary pixels of r (and of x) it owns,
// and after the grid barrier that follows reads its ring from them.  The
// direction p' = D^-1 r + beta p is recomputed on the ring from the
// exchanged r and the ring's previous p' (bit-identical to the owner's), so a
// PCG iteration moves a few KB per block instead of the whole state.  Per
// inner iteration: 1 + 2 k grid barriers (k PCG iterations); the result
// selection and the split-Bregman pass need none because Y's ring comes
// from the x boundary values of the last update.  b_old / b_new (4-12 edge
// variables per pixel and column) and rq stream through L2.
#pragma once

#include "pfe_persist.cuh"

namespace pfe_dev {

template <int D, int R>
struct ResGeo {
  static constexpr int NT = 768;   // threads per block (one block per SM, <= 85 registers)
  static constexpr int EPT = 6;    // interior (vertex, column) elements per thread, max
  static constexpr int HR = 2;     // ring elements per thread, max
  static constexpr int kMaxBlocks = 256;  // reduce_partials_warp limit
  static constexpr int S = GridTopo<R>::S;
  static constexpr int U = D;                     // units (pixel, column) per pixel
  static constexpr int kPerPos = 3 * D + 2 * S + 2;  // shared doubles per ring/interior position
  static constexpr bool kFix = (32 % D == 0);
  static constexpr int V = kFix ? 1 : D;
};

// Fixed-order reduction of nb <= 256 pair-major block partials into out[NQ][D]
// (identical in every block): warp w sums pairs w, w + NT/32, ...; lane l
// loads blocks l, l + 32, ... (all loads in flight at once), then a butterfly.
template <int NQ, int D, int NT>
__device__ __forceinline__ void reduce_partials_warp(const double* __restrict__ part, int nb,
                                                     double (&out)[NQ][D]) {
  constexpr int P = NQ * D, NW = NT / 32;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int p = warp; p < P; p += NW) {
    double v[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const int b = lane + 32 * j;
      v[j] = b < nb ? __ldcg(part + static_cast<long>(p) * nb + b) : 0.0;
    }
    double acc = v[0];
#pragma unroll
    for (int j = 1; j < 8; ++j) acc += v[j];
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (lane == 0) out[p / D][p % D] = acc;
  }
  __syncthreads();
}

// acc[q][.] += val for column c (V == 1: one column per thread)
template <int NQ, int V>
__device__ __forceinline__ void acc_add(double (&acc)[NQ][V], int q, int c, double val) {
  if constexpr (V == 1) {
    acc[q][0] += val;
  } else {
#pragma unroll
    for (int j = 0; j < V; ++j)
      if (j == c) acc[q][j] += val;
  }
}

template <int D, int R>
__global__ void __launch_bounds__(768, 1) k_sb_resident(PersistArgs<R> a) {
  using G = ResGeo<D, R>;
  using T = GridTopo<R>;
  constexpr int NT = G::NT, EPT = G::EPT, HR = G::HR, S = G::S, V = G::V;
  constexpr bool kColFix = (NT % D == 0);  // all elements of a thread share column tid % D
  extern __shared__ double smem[];
  __shared__ PersistCols<D> pc;
  __shared__ double tot[3][D];
  __shared__ double tot1[1][D];
  __shared__ int mode[D];
  cg::grid_group grid = cg::this_grid();
  const Grid<R>& g = a.g;
  const int nb = gridDim.x;
  const int tid = threadIdx.x;

  // ---- this block's region [y0, y0+rh) x [x0, x0+rw)
  const int by = blockIdx.x / a.rgx, bx = blockIdx.x - by * a.rgx;
  const int y0 = by * g.H / a.rgy, x0 = bx * g.W / a.rgx;
  const int rh = (by + 1) * g.H / a.rgy - y0, rw = (bx + 1) * g.W / a.rgx - x0;
  const int HW = a.rhw, NP = a.rnp;
  const int hwb = rw + 2 * R;                  // this region's ring width
  const int nring = 2 * R * hwb + 2 * R * rh;  // ring positions
  const int ne = rh * rw * D;                  // interior elements
  double* A1 = smem;
  double* A2 = A1 + NP * D;
  double* A3 = A2 + NP * D;
  double* Wt = A3 + NP * D;
  double* Iv = Wt + S * NP;
  double* Dg = Iv + NP;
  double* Ct = Dg + NP;  // [S][NP] off-diagonal entries of A (Grid::cf), +0.0 = absent edge

  // this thread's interior elements e_k = tid + k NT, k < nk: smem position
  // hpk[k], column col(k), vertex vert(k); bit k of bnd: on the region boundary
  int hpk[EPT];
  unsigned bnd = 0;
  int nk = 0;
#pragma unroll
  for (int k = 0; k < EPT; ++k) {
    const int e = tid + k * NT;
    hpk[k] = 0;
    if (e < ne) {
      const int lv = e / D;
      const int ly = lv / rw, lx = lv - ly * rw;
      hpk[k] = (ly + R) * HW + lx + R;
      if (ly < R || ly >= rh - R || lx < R || lx >= rw - R) bnd |= 1u << k;
      nk = k + 1;
    }
  }
  auto col = [&](int k) { return kColFix ? tid % D : (tid + k * NT) % D; };
  const float rhw = 1.0f / static_cast<float>(HW);
  const long vbase = static_cast<long>(y0 - R) * g.W + (x0 - R);
  auto vert = [&](int k) -> long {  // hp = (ly + R) HW + lx + R  ->  vertex
    const int t = static_cast<int>((static_cast<float>(hpk[k]) + 0.5f) * rhw);
    return vbase + static_cast<long>(t) * g.W + (hpk[k] - t * HW);
  };

  // q_k = (A P)_{v_k, col(k)}, each in the order of tile_apply_A
  // (sparse.cpp:77-83).  Branch-free: every term is loaded and formed, and
  // absent edges (w == 0) are skipped by a select, so the loads of a row are
  // all in flight before the (serial, reference-order) additions.  Elements
  // k >= nk evaluate a valid interior position and are discarded.
  auto apply_A = [&](const double* P, double (&q)[EPT]) {
#pragma unroll
    for (int k = 0; k < EPT; ++k) {
      const int hp = k < nk ? hpk[k] : R * HW + R;
      const double* Pc = P + col(k);
      double t[2 * S + 1];
      bool nz[2 * S + 1];
#pragma unroll
      for (int j = 0; j < S; ++j) {  // backward slots S-1 .. 0
        const int s = S - 1 - j;
        const int pn = hp - T::dy(s) * HW - T::dx(s);
        const double cw = Ct[s * NP + pn];  // -((hl w) w); present edges have the sign bit set
        nz[j] = __double_as_longlong(cw) < 0;
        t[j] = cw * Pc[pn * D];
      }
      nz[S] = true;
      t[S] = Dg[hp] * Pc[hp * D];
#pragma unroll
      for (int s = 0; s < S; ++s) {
        const int pn = hp + T::dy(s) * HW + T::dx(s);
        const double cw = Ct[s * NP + hp];
        nz[S + 1 + s] = __double_as_longlong(cw) < 0;
        t[S + 1 + s] = cw * Pc[pn * D];
      }
      double acc = 0.0;
#pragma unroll
      for (int j = 0; j < 2 * S + 1; ++j) acc = nz[j] ? acc + t[j] : acc;
      q[k] = acc;
    }
  };

  // ring element i (position i / D, column i % D): smem index and global index
  auto ring_elem = [&](int i, int& si, long& gi) -> bool {
    const int p = i / D, c = i - p * D;
    int ly, lx;
    if (p < 2 * R * hwb) {
      const int t = p / hwb;
      lx = p - t * hwb - R;
      ly = t < R ? t - R : rh + (t - R);
    } else {
      const int j = p - 2 * R * hwb;
      const int t = j / (2 * R), k = j - t * (2 * R);
      ly = t;
      lx = k < R ? k - R : rw + (k - R);
    }
    const int y = y0 + ly, x = x0 + lx;
    if (y < 0 || y >= g.H || x < 0 || x >= g.W) return false;
    si = ((ly + R) * HW + lx + R) * D + c;
    gi = (static_cast<long>(y) * g.W + x) * D + c;
    return true;
  };
  // ring of a global [n][D] array: loads issued now, stored by ring_store
  double hv[HR];
  int hs[HR];
  auto ring_load = [&](const double* src) {
#pragma unroll
    for (int j = 0; j < HR; ++j) {
      hs[j] = -1;
      long gi;
      int si;
      const int i = tid + j * NT;
      if (i < nring * D && ring_elem(i, si, gi)) {
        hv[j] = __ldcg(src + gi);
        hs[j] = si;
      }
    }
  };
  auto ring_store = [&](double* dst) {
#pragma unroll
    for (int j = 0; j < HR; ++j)
      if (hs[j] >= 0) dst[hs[j]] = hv[j];
  };

  int ycur = a.ycur, ebcur = a.ebcur;
  bool b_zero = a.b_zero != 0;
  int bad = 0;
  int trace_n = 0;
  PFE_TRACE(0);

  // ---- resident data: zero, then the static operator and the first Y / rhs
  for (int i = tid; i < NP * G::kPerPos; i += NT) smem[i] = 0.0;
  __syncthreads();
  {
    const int npos = (rh + 2 * R) * hwb;
    const double* y = a.ybuf[ycur];
    for (int i = tid; i < npos; i += NT) {
      const int t = i / hwb;
      const int ly = t - R, lx = i - t * hwb - R;
      const int yy = y0 + ly, xx = x0 + lx;
      if (yy < 0 || yy >= g.H || xx < 0 || xx >= g.W) continue;
      const long u = static_cast<long>(yy) * g.W + xx;
      const int hp = (ly + R) * HW + lx + R;
#pragma unroll
      for (int s = 0; s < S; ++s) {
        Wt[s * NP + hp] = __ldg(g.wf + u * S + s);
        Ct[s * NP + hp] = __ldg(g.cf + u * S + s);
      }
      Iv[hp] = __ldg(g.invd + u);
      Dg[hp] = __ldg(g.diag + u);
#pragma unroll
      for (int c = 0; c < D; ++c) A1[hp * D + c] = y[u * D + c];
    }
#pragma unroll
    for (int k = 0; k < EPT; ++k)
      if (k < nk) A2[hpk[k] * D + col(k)] = a.rhs0[vert(k) * D + col(k)];
  }
  __syncthreads();

  for (int inner = 0; inner < a.n_inner; ++inner) {
    const bool last = inner == a.n_inner - 1;
    const double* x0g = a.ybuf[ycur];  // Y at the start of this iteration (global, complete)
    double* xg = a.ybuf[ycur ^ 1];     // x boundary values during PCG, then the new Y
    double* part_i = a.part_c + (inner & 1) * 3 * D * nb;

    // ---------------- PCG init: r = b - A x0, p = D^-1 r (pcg.cpp:49-66)
    {
      double ax[EPT];
      apply_A(A1, ax);
      double acc[3][V] = {};
#pragma unroll
      for (int k = 0; k < EPT; ++k) {
        if (k >= nk) continue;
        const int c = col(k);
        const int si = hpk[k] * D + c;
        const double b = A2[si];
        const double rr = b - ax[k];
        const double z = Iv[hpk[k]] * rr;
        A2[si] = rr;
        A3[si] = A1[si];
        if (bnd >> k & 1u) a.r[vert(k) * D + c] = rr;
        acc_add(acc, 0, c, b * b);
        acc_add(acc, 1, c, rr * rr);
        acc_add(acc, 2, c, rr * z);
      }
      block_reduce_store<3, D, V, NT>(acc, part_i);
    }
    grid.sync();
    PFE_TRACE(1);
    if (*reinterpret_cast<volatile int*>(&a.ctl->nonfinite_y)) break;  // NaN in the previous Y
    ring_load(a.r);
    reduce_partials_warp<3, D, NT>(part_i, nb, tot);
    ring_store(A2);
    if (tid < 32) {  // initial residual test (pcg.cpp:50-62)
      const int j = tid;
      bool act = false;
      if (j < D) {
        PcgCol col{};
        col.bnorm = sqrt(tot[0][j]);
        if (col.bnorm == 0.0) {
          col.status = kZeroRhs;
        } else {
          col.rel = sqrt(tot[1][j]) / col.bnorm;
          if (col.rel <= a.tol) {
            col.status = kConvInit;
          } else {
            col.status = kActive;
            col.rz = tot[2][j];
          }
        }
        pc.col[j] = col;
        act = col.status == kActive;
        pc.act[j] = act;
        pc.coef[j] = 0.0;
      }
      const bool any = __any_sync(0xffffffffu, act);
      if (j == 0) pc.any = any;
    }
    __syncthreads();

    // ---------------- PCG iterations (pcg.cpp:68-89)
    int it = 0;
    while (pc.any && it < a.max_iter) {
      ++it;
      const bool first = it == 1;
      // p' = D^-1 r (first) or D^-1 r + beta p (pcg.cpp:86-88) on region +
      // ring (positions outside the region's box hold zeros and stay zero)
      for (int i = tid; i < NP * D; i += NT) {
        const int hp = i / D, c = i - hp * D;
        A1[i] = first ? Iv[hp] * A2[i] : Iv[hp] * A2[i] + pc.coef[c] * A1[i];
      }
      __syncthreads();
      PFE_TRACE(11);
      // q = A p', p'.q
      double qv[EPT];
      apply_A(A1, qv);
      {
        double acc[1][V] = {};
#pragma unroll
        for (int k = 0; k < EPT; ++k)
          if (k < nk) acc_add(acc, 0, col(k), A1[hpk[k] * D + col(k)] * qv[k]);
        block_reduce_store<1, D, V, NT>(acc, a.part_b);
      }
      PFE_TRACE(12);
      grid.sync();
      PFE_TRACE(3);
      reduce_partials_warp<1, D, NT>(a.part_b, nb, tot1);
      PFE_TRACE(14);
      if (tid < D) {  // alpha and the curvature check (pcg.cpp:70-72)
        const int j = tid;
        PcgCol& col = pc.col[j];
        if (pc.act[j]) {
          const double pq = tot1[0][j];
          col.pq = pq;
          if (!(pq > 0.0) || !isfinite(pq)) {
            col.status = kFailed;
            col.iters = 0;
            col.rel = kInf;
            pc.act[j] = 0;
          } else {
            col.alpha = col.rz / pq;
          }
        }
        pc.coef[j] = pc.act[j] ? col.alpha : 0.0;
      }
      __syncthreads();
      // x += alpha p, r -= alpha q (pcg.cpp:73-78); boundary values of r and x
      // go to global memory for the neighbours' rings
      {
        double acc[3][V] = {};
#pragma unroll
        for (int k = 0; k < EPT; ++k) {
          if (k >= nk) continue;
          const int c = col(k);
          const int si = hpk[k] * D + c;
          double xv = A3[si], rv = A2[si];
          if (pc.act[c]) {
            const double alpha = pc.coef[c];
            xv = xv + alpha * A1[si];
            rv = rv - alpha * qv[k];
            if (!isfinite(xv)) acc_add(acc, 2, c, 1.0);
            A3[si] = xv;
            A2[si] = rv;
          }
          const double z = Iv[hpk[k]] * rv;
          acc_add(acc, 0, c, rv * rv);
          acc_add(acc, 1, c, rv * z);
          if (bnd >> k & 1u) {
            const long gi = vert(k) * D + c;
            a.r[gi] = rv;
            xg[gi] = xv;
          }
        }
        block_reduce_store<3, D, V, NT>(acc, a.part);
      }
      PFE_TRACE(13);
      grid.sync();
      PFE_TRACE(5);
      ring_load(a.r);  // speculative: dead if every column stops here
      reduce_partials_warp<3, D, NT>(a.part, nb, tot);
      ring_store(A2);
      if (tid < 32) {  // stop test and beta (pcg.cpp:75-88)
        const int j = tid;
        bool act = false;
        if (j < D) {
          PcgCol& col = pc.col[j];
          if (pc.act[j]) {
            if (tot[2][j] > 0.0) {
              col.status = kFailed;
              col.iters = 0;
              col.rel = kInf;
            } else {
              col.rel = sqrt(tot[0][j]) / col.bnorm;
              col.iters = it;
              if (col.rel <= a.tol) {
                col.status = kConverged;
              } else if (it >= a.max_iter) {
                col.status = kMaxIter;
              } else {
                col.beta = tot[1][j] / col.rz;
                col.rz = tot[1][j];
              }
            }
          }
          act = col.status == kActive;
          pc.act[j] = act;
          pc.coef[j] = act ? col.beta : 0.0;
        }
        const bool any = __any_sync(0xffffffffu, act);
        if (j == 0) pc.any = any;
      }
      __syncthreads();
      PFE_TRACE(10);
    }

    // ---------------- result selection + log (pcg.cpp:50-62, 101-112)
    if (tid < D) {
      const PcgCol& col = pc.col[tid];
      mode[tid] = col.status == kZeroRhs ? 2 : ((col.status == kConvInit || col.status == kFailed || it == 0) ? 1 : 0);
      if (blockIdx.x == 0) {
        a.ctl->col[tid] = col;
        const int idx = a.ctl->inner_count;
        if (idx < a.ctl->log_cap) {
          a.ctl->log_iters[static_cast<long>(idx) * D + tid] = col.iters;
          a.ctl->log_status[static_cast<long>(idx) * D + tid] = col.status;
          a.ctl->log_rel[static_cast<long>(idx) * D + tid] = col.rel;
        }
      }
    }
    __syncthreads();
    if (blockIdx.x == 0 && tid == 0) {
      a.ctl->inner_count += 1;
      a.ctl->iter = it;
    }
    // new Y -> A1 (interior and ring) and to global memory (interior)
#pragma unroll
    for (int k = 0; k < EPT; ++k) {
      if (k >= nk) continue;
      const int c = col(k);
      const int si = hpk[k] * D + c;
      const long gi = vert(k) * D + c;
      const int m = mode[c];
      const double y = m == 0 ? A3[si] : (m == 1 ? __ldcg(x0g + gi) : 0.0);
      A1[si] = y;
      xg[gi] = y;
    }
    for (int i = tid; i < nring * D; i += NT) {
      int si;
      long gi;
      if (!ring_elem(i, si, gi)) continue;
      const int m = mode[i % D];
      A1[si] = m == 0 ? __ldcg(xg + gi) : (m == 1 ? __ldcg(x0g + gi) : 0.0);
    }
    ycur ^= 1;
    __syncthreads();
    PFE_TRACE(6);

    // ---------------- split-Bregman pass (solver.cpp:96-98, 83-84)
    // Per element: the 2S incident edges in edge order (backward slots owned
    // by neighbours, then forward slots); b_old of a chunk of CH edges (and
    // rq) are loaded before any of them is evaluated.
    {
      const double* b_old = b_zero ? nullptr : a.eb[ebcur];
      double* b_new = a.eb[ebcur ^ 1];
      double* s_out = (last && a.write_s_last) ? a.es : nullptr;
      const bool need_rhs = !last || a.rhs_last;
      double* rhs_g = (last && a.rhs_last) ? a.r : nullptr;
      constexpr int CH = S <= 4 ? 2 * S : S;
#pragma unroll
      for (int k = 0; k < EPT; ++k) {
        if (k >= nk) continue;
        const int hp = hpk[k], c = col(k);
        const long v = vert(k);
        bad |= !isfinite(A1[hp * D + c]);
        const double rqv = need_rhs ? __ldg(a.rq + v * D + c) : 0.0;
        double acc = 0.0;
#pragma unroll
        for (int e0 = 0; e0 < 2 * S; e0 += CH) {
          double bo[CH];
#pragma unroll
          for (int j = 0; j < CH; ++j) {
            const int e = e0 + j;
            const bool fwd = e >= S;
            const int s = fwd ? e - S : S - 1 - e;
            const int opos = fwd ? hp : hp - T::dy(s) * HW - T::dx(s);
            const long slot = fwd ? v * S + s : (v - T::dy(s) * g.W - T::dx(s)) * S + s;
            bo[j] = (b_old && Wt[s * NP + opos] != 0.0) ? __ldcg(b_old + slot * D + c) : 0.0;
          }
#pragma unroll
          for (int j = 0; j < CH; ++j) {
            const int e = e0 + j;
            const bool fwd = e >= S;
            const int s = fwd ? e - S : S - 1 - e;
            const int npos = fwd ? hp + T::dy(s) * HW + T::dx(s) : hp - T::dy(s) * HW - T::dx(s);
            const int opos = fwd ? hp : npos;
            const int jpos = fwd ? npos : hp;
            const double w = Wt[s * NP + opos];
            if (w == 0.0) continue;
            const double nw = -w;
            const double my = w * A1[opos * D + c] + nw * A1[jpos * D + c];
            const double sh = shrink1(my + bo[j], a.gamma);
            const double bn = bo[j] + (my - sh);
            acc += (fwd ? w : nw) * (sh - bn);
            if (fwd) {
              const long slot = v * S + s;
              b_new[slot * D + c] = bn;
              if (s_out) s_out[slot * D + c] = sh;
            }
          }
        }
        if (need_rhs) {
          const double rn = a.hl * acc + rqv;
          A2[hp * D + c] = rn;
          if (rhs_g) rhs_g[v * D + c] = rn;
        }
      }
    }
    ebcur ^= 1;
    b_zero = false;
    // NaN / Inf in this iteration's Y (solver.cpp:94): published now, seen by
    // every block after the next grid barrier, where the launch stops
    if (__syncthreads_or(bad) && tid == 0) atomicOr(&a.ctl->nonfinite_y, 1);
    bad = 0;
    PFE_TRACE(8);
  }
}

}  // namespace pfe_dev
