// Persistent cooperative split-Bregman kernel for pixel-grid graphs.
//
// One cooperative launch runs whole inner iterations of PfeSolver::
// split_bregman (solver.cpp:82-107) on the device: for every inner iteration
// the PCG solve of all d columns (init, then SpMV / update pairs until every
// column has stopped, then the per-column result selection) followed by the
// fused shrink / Bregman / next-rhs pass.  Phases are separated by grid-wide
// barriers; after each barrier every block reduces the producers' block
// partials in the same fixed order, so all blocks hold bit-identical PCG
// scalars (alpha, beta, stop flags) in shared memory and the loop needs no
// host round trip, no kernel launch and no serial reduction tail.
//
// The stencil phases (init, SpMV) stage their tiles with double-buffered
// cp.async: the copies of the block's next tile are in flight while the
// current tile is evaluated from shared memory.  The update phase streams
// with a 4-deep software pipeline (all loads of a batch issued before any
// store).  Per-element arithmetic is exactly that of the multi-kernel path
// (pfe_stencil.cuh / pfe_kernels.cuh); only the reduction tree differs.
#pragma once

#include <cooperative_groups.h>

#include "pfe_stencil.cuh"
#include "pfe_tma.cuh"

namespace pfe_dev {

namespace cg = cooperative_groups;

// Optional phase trace (block 0, thread 0): code and %globaltimer after each
// grid barrier, for the per-phase timing breakdown in scripts/prof_run.py.
#define PFE_TRACE(code)                                                                      \
  do {                                                                                       \
    if (a.trace && blockIdx.x == 0 && threadIdx.x == 0 && trace_n < a.trace_cap) {            \
      unsigned long long t_;                                                                 \
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));                                 \
      a.trace[trace_n++] = (static_cast<unsigned long long>(code) << 56) | (t_ & ((1ull << 56) - 1)); \
    }                                                                                        \
  } while (0)

template <int R>
struct PersistArgs {
  Grid<R> g;
  double* ybuf[2];   // the two Y buffers
  int ycur;          // index of Y (the warm start) at kernel start
  double* r;         // residual; also the rhs buffer written by the sb phase
  double* pbuf[2];
  double* q;
  double* eb[2];     // split_b ping-pong
  int ebcur;
  double* es;        // split_s (materialised on the last iteration when asked)
  const double* rq;  // (r/2) sqrt(D) (P - B)
  const double* rhs0;  // rhs of the first inner iteration
  int b_zero;        // split_b == split_s == 0 at kernel start
  int n_inner;
  int write_s_last;
  int rhs_last;      // produce the rhs after the last iteration too
  double tol;
  int max_iter;
  double hl, gamma;
  Ctl* ctl;
  double* part;      // init / update block partials [3*D][gridDim.x]
  unsigned long long* trace;  // optional phase trace (null: off)
  int trace_cap;
  double* part_b;    // SpMV block partials: alternating buffers so a fast block never
                     // overwrites partials a slow block is still reducing
  // shared-memory-resident variant (pfe_resident.cuh) only
  double* part_c;    // init partials, two buffers alternating by inner iteration
  int rgx, rgy;      // region grid: blocks = rgx * rgy, block b owns region (b / rgx, b % rgx)
  int rhw, rnp;      // smem pitch (max region width + 2R) and positions per plane
  // tiled persistent kernel: phases staging their tiles with TMA (bit 0
  // init, 1 SpMV, 2 split-Bregman pass, 3 b_old owner rows) or cp.async
  int tma;
  // 8-neighbour grids (no TMA): halo rows staged as cp.async.bulk row copies
  int bulk;
  TileMaps tm;
};

// Per-block column state (identical in every block).
template <int D>
struct PersistCols {
  PcgCol col[D];
  double coef[D];
  int act[D];
  int any;
};

template <int D, int R>
struct PersistGeo {
  using G = TileGeo<R, D>;
  // tile buffers of the init and SpMV phases: a ring of kRing (one tile
  // evaluated while kRing - 1 are staged)
  static constexpr int kRing = 2;
  static constexpr int kInit2 = kRing * G::kInit, kSpmv2 = kRing * G::kSpmv;
  static constexpr int kA = kInit2 > kSpmv2 ? kInit2 : kSpmv2;
  static constexpr int kSbB = G::kStageB ? G::kSb : 2 * G::kSb;  // sb phase (double-buffered for 5x5)
  static constexpr int kSmem = kA > kSbB ? kA : kSbB;  // doubles
};

__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory");
}

template <int D, int R>
__global__ void __launch_bounds__(TileGeo<R, D>::NT, R == 2 ? 1 : 2)
    k_sb_persistent(const __grid_constant__ PersistArgs<R> a) {
  using G = TileGeo<R, D>;
  using T = GridTopo<R>;
  constexpr int V = PairMode<R, D>::V;
  constexpr int NT = G::NT;
  extern __shared__ __align__(1024) double smem[];  // 1024: TMA box destinations
  __shared__ PersistCols<D> pc;
  __shared__ double tot[3][D];
  __shared__ double tot1[1][D];
  cg::grid_group grid = cg::this_grid();
  const Grid<R>& g = a.g;
  const int nt = num_tiles<R, D>(g);
  const int nb = gridDim.x;
  int ycur = a.ycur, ebcur = a.ebcur;
  bool b_zero = a.b_zero != 0;
  int bad = 0;
  int trace_n = 0;
  PFE_TRACE(0);
  // TMA staging: one mbarrier per tile buffer; tph holds each buffer's
  // expected phase parity (identical in every thread)
  constexpr int NB = PersistGeo<D, R>::kRing > 2 ? PersistGeo<D, R>::kRing : 2;  // mbarriers / tile buffers
  __shared__ alignas(8) uint64_t tbar[NB];
  const bool tma_any = a.tma != 0;
  const bool bulk_any = a.bulk != 0;
  uint32_t tph = 0;
  if ((tma_any || bulk_any) && threadIdx.x == 0) {
    for (int i = 0; i < NB; ++i) mbar_init(&tbar[i], 1);
    mbar_fence_init();
  }
  __syncthreads();
  const bool bulk = a.bulk != 0;
  // ring form for the init / SpMV phases: NR - 1 tiles staged ahead
  constexpr int NR = PersistGeo<D, R>::kRing;
  auto ring_wait = [&](bool tma, int buf) {
    if (tma || bulk) {
      mbar_wait(&tbar[buf], (tph >> buf) & 1u);
      tph ^= 1u << buf;
    }
    cp_async_wait<NR - 1>();
  };
  auto tile_wait = [&](bool tma, int buf, bool more) {
    if (tma || bulk) {
      mbar_wait(&tbar[buf], (tph >> buf) & 1u);
      tph ^= 1u << buf;
    }
    if (more)
      cp_async_wait<1>();
    else
      cp_async_wait<0>();
  };
  constexpr uint32_t kHalo = G::NP * 8, kInt = G::NV * 8;

  for (int inner = 0; inner < a.n_inner; ++inner) {
    const bool last = inner == a.n_inner - 1;
    const double* x0 = a.ybuf[ycur];
    double* x = a.ybuf[ycur ^ 1];
    const double* rhs = inner == 0 ? a.rhs0 : a.r;

    // ---------------- PCG init: r = b - A x0, p = D^-1 r (pcg.cpp:49-66)
    {
      double acc[3][V] = {};
      const bool tma = (a.tma & 1) != 0, tma1 = (a.tma & 16) != 0;
      auto stage = [&](int t, int buf) {
        double* P = smem + buf * G::kInit;
        double* Wt = P + G::kI_W;
        double* Bv = P + G::kI_B;
        double* Dg = P + G::kI_Dg;
        double* Iv = P + G::kI_Iv;
        const TileIdx ti = tile_of<R, D>(g, t);
        if (tma) {
          if (threadIdx.x == 0) {
            fence_proxy_async();
            mbar_expect_tx(&tbar[buf], kHalo * (D + G::S) + kInt * (D + (tma1 ? 2 : 0)));
            tma_rows<D>(P, &a.tm.y[ycur], ti.x0 - R, ti.y0 - R, &tbar[buf]);
            tma_rows<G::S>(Wt, &a.tm.cf_halo, ti.x0 - R, ti.y0 - R, &tbar[buf]);
            tma_rows<D>(Bv, inner == 0 ? &a.tm.rhs0_int : &a.tm.r_int, ti.x0, ti.y0, &tbar[buf]);
            if (tma1) {
              tma_rows<1>(Dg, &a.tm.dg_int, ti.x0, ti.y0, &tbar[buf]);
              tma_rows<1>(Iv, &a.tm.iv_int, ti.x0, ti.y0, &tbar[buf]);
            }
          }
          if (!tma1) {
            stage_interior<R, D, 1>(g, ti, g.diag, Dg);
            stage_interior<R, D, 1>(g, ti, g.invd, Iv);
          }
          return;
        }
        if (bulk) {
          const Span sh = box_span(g, ti.x0 - R, ti.y0 - R, G::HW, G::HH, g.H);
          const Span si = box_span(g, ti.x0, ti.y0, G::TW, G::TH, g.row_hi);
          if (threadIdx.x < 32) {
            if (threadIdx.x == 0) {
              fence_proxy_async();
              mbar_expect_tx(&tbar[buf], span_bytes<D>(sh) + span_bytes<G::S>(sh) + span_bytes<D>(si));
            }
            __syncwarp();
            span_issue<D, G::HW>(g, sh, x0, P, &tbar[buf], threadIdx.x);
            span_issue<G::S, G::HW>(g, sh, g.cf, Wt, &tbar[buf], threadIdx.x);
            span_issue<D, G::TW>(g, si, rhs, Bv, &tbar[buf], threadIdx.x);
          }
          span_zero<D, G::HW, NT>(sh, P, G::HH);
          span_zero<G::S, G::HW, NT>(sh, Wt, G::HH);
          stage_interior<R, D, 1>(g, ti, g.diag, Dg);
          stage_interior<R, D, 1>(g, ti, g.invd, Iv);
          return;
        }
        stage_rows<R, D, D>(g, ti, x0, P, G::HH);
        stage_rows<R, D, G::S>(g, ti, g.cf, Wt, G::HH);
        stage_interior<R, D, D>(g, ti, rhs, Bv);
        stage_interior<R, D, 1>(g, ti, g.diag, Dg);
        stage_interior<R, D, 1>(g, ti, g.invd, Iv);
      };
      for (int j = 0; j < NR - 1; ++j) {
        if (blockIdx.x + j * nb < nt) stage(blockIdx.x + j * nb, j);
        cp_async_commit();
      }
      int buf = 0;
      for (int t = blockIdx.x; t < nt; t += nb) {
        if (t + (NR - 1) * nb < nt) stage(t + (NR - 1) * nb, (buf + NR - 1) % NR);
        cp_async_commit();
        ring_wait(tma, buf);
        __syncthreads();
        const double* P = smem + buf * G::kInit;
        const double* Wt = P + G::kI_W;
        const double* Bv = P + G::kI_B;
        const double* Dg = P + G::kI_Dg;
        const double* Iv = P + G::kI_Iv;
        const TileIdx ti = tile_of<R, D>(g, t);
        tile_init_body<R, D, V>(g, ti, P, Wt, Bv, Dg, Iv, a.r, a.pbuf[0], acc);
        if (bulk) fence_proxy_async();  // zero-fill stores before later async writes
        __syncthreads();
        buf = (buf + 1) % NR;
      }
      cp_async_wait<0>();
      block_reduce_store<3, D, V, NT>(acc, a.part);
    }
    grid.sync();
    PFE_TRACE(1);
    reduce_partials<3, D, NT>(a.part, nb, tot);
    if (threadIdx.x < 32) {  // initial residual test (pcg.cpp:50-62)
      const int j = threadIdx.x;
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
      double* pnew = (it & 1) ? a.pbuf[0] : a.pbuf[1];
      const double* pold = first ? a.pbuf[0] : ((it & 1) ? a.pbuf[1] : a.pbuf[0]);
      if (threadIdx.x < D) pc.coef[threadIdx.x] = pc.act[threadIdx.x] ? pc.col[threadIdx.x].beta : 0.0;
      // SpMV with the fused direction update p = z + beta p
      {
        double acc[1][V] = {};
        const bool tma = (a.tma & 2) != 0, tma1 = (a.tma & 16) != 0;
        auto stage = [&](int t, int buf) {
          double* P = smem + buf * G::kSpmv;
          double* Rs = P + G::kS_Rs;
          double* Iv = P + G::kS_Iv;
          double* Wt = P + G::kS_W;
          double* Dg = P + G::kS_Dg;
          const TileIdx ti = tile_of<R, D>(g, t);
          if (tma) {
            if (threadIdx.x == 0) {
              fence_proxy_async();
              mbar_expect_tx(&tbar[buf], kHalo * (D + G::S) + (tma1 ? kInt : 0u) +
                                             (first ? 0u : kHalo * (D + (tma1 ? 1 : 0))));
              tma_rows<D>(P, &a.tm.p[pold == a.pbuf[1] ? 1 : 0], ti.x0 - R, ti.y0 - R, &tbar[buf]);
              if (!first) {
                tma_rows<D>(Rs, &a.tm.r_halo, ti.x0 - R, ti.y0 - R, &tbar[buf]);
                if (tma1) tma_rows<1>(Iv, &a.tm.iv_halo, ti.x0 - R, ti.y0 - R, &tbar[buf]);
              }
              tma_rows<G::S>(Wt, &a.tm.cf_halo, ti.x0 - R, ti.y0 - R, &tbar[buf]);
              if (tma1) tma_rows<1>(Dg, &a.tm.dg_int, ti.x0, ti.y0, &tbar[buf]);
            }
            if (!tma1) {
              if (!first) stage_rows<R, D, 1>(g, ti, g.invd, Iv, G::HH);
              stage_interior<R, D, 1>(g, ti, g.diag, Dg);
            }
            return;
          }
          if (bulk) {
            const Span sh = box_span(g, ti.x0 - R, ti.y0 - R, G::HW, G::HH, g.H);
            if (threadIdx.x < 32) {
              if (threadIdx.x == 0) {
                fence_proxy_async();
                mbar_expect_tx(&tbar[buf], span_bytes<D>(sh) * (first ? 1u : 2u) + span_bytes<G::S>(sh));
              }
              __syncwarp();
              span_issue<D, G::HW>(g, sh, pold, P, &tbar[buf], threadIdx.x);
              if (!first) span_issue<D, G::HW>(g, sh, a.r, Rs, &tbar[buf], threadIdx.x);
              span_issue<G::S, G::HW>(g, sh, g.cf, Wt, &tbar[buf], threadIdx.x);
            }
            span_zero<D, G::HW, NT>(sh, P, G::HH);
            if (!first) {
              span_zero<D, G::HW, NT>(sh, Rs, G::HH);
              stage_rows<R, D, 1>(g, ti, g.invd, Iv, G::HH);
            }
            span_zero<G::S, G::HW, NT>(sh, Wt, G::HH);
            stage_interior<R, D, 1>(g, ti, g.diag, Dg);
            return;
          }
          stage_rows<R, D, D>(g, ti, pold, P, G::HH);
          if (!first) {
            stage_rows<R, D, D>(g, ti, a.r, Rs, G::HH);
            stage_rows<R, D, 1>(g, ti, g.invd, Iv, G::HH);
          }
          stage_rows<R, D, G::S>(g, ti, g.cf, Wt, G::HH);
          stage_interior<R, D, 1>(g, ti, g.diag, Dg);
        };
        for (int j = 0; j < NR - 1; ++j) {
          if (blockIdx.x + j * nb < nt) stage(blockIdx.x + j * nb, j);
          cp_async_commit();
        }
        int buf = 0;
        for (int t = blockIdx.x; t < nt; t += nb) {
          if (t + (NR - 1) * nb < nt) stage(t + (NR - 1) * nb, (buf + NR - 1) % NR);
          cp_async_commit();
          ring_wait(tma, buf);
          __syncthreads();
          double* P = smem + buf * G::kSpmv;
          const double* Rs = P + G::kS_Rs;
          const double* Iv = P + G::kS_Iv;
          const double* Wt = P + G::kS_W;
          const double* Dg = P + G::kS_Dg;
          if (!first) {
            for (int e = threadIdx.x; e < G::NP * D; e += NT) {
              const int pos = e / D, c = e - pos * D;
              P[e] = Iv[pos] * Rs[e] + pc.coef[c] * P[e];
            }
            __syncthreads();
          }
          const TileIdx ti = tile_of<R, D>(g, t);
          tile_spmv_body<R, D, V>(g, ti, P, Wt, Dg, a.q, first ? nullptr : pnew, acc);
          // p' was formed in place (generic proxy); a later TMA copy into
          // this buffer (async proxy) must be ordered after those writes
          if (tma || bulk) fence_proxy_async();
          __syncthreads();
          buf = (buf + 1) % NR;
        }
        cp_async_wait<0>();
        block_reduce_store<1, D, V, NT>(acc, a.part_b);
      }
      grid.sync();
    PFE_TRACE(3);
      reduce_partials<1, D, NT>(a.part_b, nb, tot1);
      if (threadIdx.x < 32) {  // alpha and the curvature check (pcg.cpp:70-72)
        const int j = threadIdx.x;
        if (j < D) {
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
      }
      __syncthreads();
      // update x += alpha p, r -= alpha q (pcg.cpp:73-78); element e owns
      // column e % D; batches of U elements per thread are loaded before any
      // of them is stored (the buffers alias, so the compiler cannot hoist)
      {
        constexpr bool kFix = (32 % D == 0);
        constexpr int VA = kFix ? 1 : D;
        constexpr int U = 4;
        double acc[3][VA] = {};
        const double* __restrict__ xs = first ? x0 : x;
        const double* __restrict__ pin = first ? a.pbuf[0] : pnew;
        const long total = static_cast<long>(g.n) * D;
        const long stride = static_cast<long>(nb) * NT;
        for (long e0 = static_cast<long>(blockIdx.x) * NT + threadIdx.x; e0 < total; e0 += U * stride) {
          double xv[U], rv[U], pv[U], qv[U], iv[U];
#pragma unroll
          for (int u = 0; u < U; ++u) {
            const long e = e0 + u * stride;
            if (e < total) {
              xv[u] = xs[e];
              rv[u] = a.r[e];
              pv[u] = __ldcg(pin + e);  // written earlier in this kernel: L2-coherent loads
              qv[u] = __ldcg(a.q + e);
              iv[u] = __ldg(g.invd + e / D);
            }
          }
#pragma unroll
          for (int u = 0; u < U; ++u) {
            const long e = e0 + u * stride;
            if (e >= total) break;
            const int c = static_cast<int>(e % D);
            const int k = kFix ? 0 : c;
            if (pc.act[c]) {
              const double alpha = pc.coef[c];
              xv[u] = xv[u] + alpha * pv[u];
              rv[u] = rv[u] - alpha * qv[u];
              if (!isfinite(xv[u])) acc[2][k] += 1.0;
            }
            const double z = iv[u] * rv[u];
            acc[0][k] += rv[u] * rv[u];
            acc[1][k] += rv[u] * z;
            x[e] = xv[u];
            a.r[e] = rv[u];
          }
        }
        block_reduce_store<3, D, VA, NT>(acc, a.part);
      }
      grid.sync();
    PFE_TRACE(5);
      reduce_partials<3, D, NT>(a.part, nb, tot);
      if (threadIdx.x < 32) {  // stop test and beta (pcg.cpp:75-88)
        const int j = threadIdx.x;
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
        }
        const bool any = __any_sync(0xffffffffu, act);
        if (j == 0) pc.any = any;
      }
      __syncthreads();
    }

    // ---------------- result selection + log (pcg.cpp:50-62, 101-112)
    {
      __shared__ int mode[D];
      if (threadIdx.x < D) {
        const PcgCol& col = pc.col[threadIdx.x];
        mode[threadIdx.x] =
            col.status == kZeroRhs ? 2 : ((col.status == kConvInit || col.status == kFailed || it == 0) ? 1 : 0);
        if (blockIdx.x == 0) {
          a.ctl->col[threadIdx.x] = col;
          const int idx = a.ctl->inner_count;
          if (idx < a.ctl->log_cap) {
            a.ctl->log_iters[static_cast<long>(idx) * D + threadIdx.x] = col.iters;
            a.ctl->log_status[static_cast<long>(idx) * D + threadIdx.x] = col.status;
            a.ctl->log_rel[static_cast<long>(idx) * D + threadIdx.x] = col.rel;
          }
        }
      }
      __syncthreads();
      if (blockIdx.x == 0 && threadIdx.x == 0) {
        a.ctl->inner_count += 1;
        a.ctl->iter = it;
      }
      bool need = false;
#pragma unroll
      for (int j = 0; j < D; ++j) need |= mode[j] != 0;
      if (need) {
        const long total = static_cast<long>(g.n) * D;
        for (long e = static_cast<long>(blockIdx.x) * NT + threadIdx.x; e < total; e += static_cast<long>(nb) * NT) {
          const int j = static_cast<int>(e % D);
          if (mode[j] == 1) x[e] = x0[e];
          else if (mode[j] == 2) x[e] = 0.0;
        }
      }
    }
    ycur ^= 1;
    grid.sync();
    PFE_TRACE(6);

    // ---------------- split-Bregman pass (solver.cpp:96-98, 83-84)
    {
      const double* y = a.ybuf[ycur];
      const double* b_old = b_zero ? nullptr : a.eb[ebcur];
      double* b_new = a.eb[ebcur ^ 1];
      double* s_out = (last && a.write_s_last) ? a.es : nullptr;
      double* rhs_out = (!last || a.rhs_last) ? a.r : nullptr;
      // 8-neighbour grids stage b_old (the tile fills shared memory: single
      // buffer); 5x5 grids read b_old from global memory and double-buffer
      // the tile staging like the SpMV
      constexpr bool kDB = !G::kStageB;
      const bool tma = (a.tma & 4) != 0, tma_b = (a.tma & 8) != 0;
      auto stage = [&](int t, int buf) {
        double* P = smem + buf * G::kSb;
        double* Wt = P + G::kB_W;
        double* Rq = P + G::kB_Rq;
        double* Bo = P + G::kB_Bo;
        const TileIdx ti = tile_of<R, D>(g, t);
        if (tma) {
          if (threadIdx.x == 0) {
            fence_proxy_async();
            const bool stage_b = G::kStageB && b_old && tma_b;
            mbar_expect_tx(&tbar[buf], kHalo * (D + G::S) + (rhs_out ? kInt * D : 0u) +
                                           (stage_b ? static_cast<uint32_t>(G::NO * G::S * D * 8) : 0u));
            tma_rows<D>(P, &a.tm.y[ycur], ti.x0 - R, ti.y0 - R, &tbar[buf]);
            tma_rows<G::S>(Wt, &a.tm.wf_halo, ti.x0 - R, ti.y0 - R, &tbar[buf]);
            if (rhs_out) tma_rows<D>(Rq, &a.tm.rq_int, ti.x0, ti.y0, &tbar[buf]);
            if constexpr (G::kStageB) {
              if (stage_b) tma_rows<G::S * D>(Bo, &a.tm.bo[ebcur], ti.x0 - R, ti.y0 - R, &tbar[buf]);
            }
          }
          if constexpr (G::kStageB) {
            if (b_old && !tma_b) stage_rows<R, D, G::S * D>(g, ti, b_old, Bo, G::TH + R);
          }
          return;
        }
        if (bulk) {
          const Span sh = box_span(g, ti.x0 - R, ti.y0 - R, G::HW, G::HH, g.H);
          const Span sb = box_span(g, ti.x0 - R, ti.y0 - R, G::HW, G::TH + R, g.H);
          const Span si = box_span(g, ti.x0, ti.y0, G::TW, G::TH, g.row_hi);
          const bool stage_b = G::kStageB && b_old;
          if (threadIdx.x < 32) {
            if (threadIdx.x == 0) {
              fence_proxy_async();
              mbar_expect_tx(&tbar[buf], span_bytes<D>(sh) + span_bytes<G::S>(sh) + (rhs_out ? span_bytes<D>(si) : 0u) +
                                             (stage_b ? span_bytes<G::S * D>(sb) : 0u));
            }
            __syncwarp();
            span_issue<D, G::HW>(g, sh, y, P, &tbar[buf], threadIdx.x);
            span_issue<G::S, G::HW>(g, sh, g.wf, Wt, &tbar[buf], threadIdx.x);
            if (rhs_out) span_issue<D, G::TW>(g, si, a.rq, Rq, &tbar[buf], threadIdx.x);
            if constexpr (G::kStageB) {
              if (stage_b) span_issue<G::S * D, G::HW>(g, sb, b_old, Bo, &tbar[buf], threadIdx.x);
            }
          }
          span_zero<D, G::HW, NT>(sh, P, G::HH);
          span_zero<G::S, G::HW, NT>(sh, Wt, G::HH);
          return;
        }
        stage_rows<R, D, D>(g, ti, y, P, G::HH);
        stage_rows<R, D, G::S>(g, ti, g.wf, Wt, G::HH);
        if (rhs_out) stage_interior<R, D, D>(g, ti, a.rq, Rq);
        if constexpr (G::kStageB) {
          if (b_old) stage_rows<R, D, G::S * D>(g, ti, b_old, Bo, G::TH + R);
        }
      };
      int buf = 0;
      if (kDB && blockIdx.x < nt) stage(blockIdx.x, 0);
      cp_async_commit();
      for (int t = blockIdx.x; t < nt; t += nb) {
        if constexpr (kDB) {
          if (t + nb < nt) stage(t + nb, buf ^ 1);
          cp_async_commit();
          tile_wait(tma, buf, true);
        } else {
          stage(t, 0);
          cp_async_commit();
          tile_wait(tma, 0, false);
        }
        __syncthreads();
        const double* P = smem + buf * G::kSb;
        const double* Wt = P + G::kB_W;
        const double* Rq = P + G::kB_Rq;
        const double* Bo = P + G::kB_Bo;
        const TileIdx ti = tile_of<R, D>(g, t);
        bad |= tile_sb_body<D, R, false>(g, ti, P, Wt, Bo, Rq, b_old, b_new, s_out, rhs_out, a.hl, a.gamma);
        if (bulk) fence_proxy_async();  // zero-fill stores before later async writes
        __syncthreads();
        if constexpr (kDB) buf ^= 1;
      }
      cp_async_wait<0>();
    }
    ebcur ^= 1;
    b_zero = false;
    // NaN / Inf in this iteration's Y (solver.cpp:94): published before the
    // barrier, so every block sees it after and the launch stops here, as the
    // reference aborts the inner loop (the host then raises NumericalError)
    if (__syncthreads_or(bad) && threadIdx.x == 0) atomicOr(&a.ctl->nonfinite_y, 1);
    grid.sync();
    PFE_TRACE(8);
    if (*reinterpret_cast<volatile int*>(&a.ctl->nonfinite_y)) break;
  }
}

}  // namespace pfe_dev
