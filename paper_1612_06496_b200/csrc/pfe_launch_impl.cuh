// Template bodies of the launch table (included by pfe_kernels_d*.cu only).
#pragma once

#include "pfe_kernels.cuh"
#include "pfe_launch.h"
#include "pfe_polar.cuh"

namespace pfe_host {

using namespace pfe_dev;

template <int D>
struct Impl {
  template <class F>
  static void on_topo(const TopoDesc& t, F&& f) {
    switch (t.kind) {
      case kTopoGrid1:
        f(t.g1);
        break;
      case kTopoGrid2:
        f(t.g2);
        break;
      default:
        f(t.csr);
        break;
    }
  }

  static void pcg_init(const TopoDesc& t, const PcgArgs& a, Launch l) {
    on_topo(t, [&](const auto& topo) {
      using T = std::decay_t<decltype(topo)>;
      k_pcg_init<D, T><<<l.grid, kBlock, 0, l.stream>>>(topo, a);
    });
  }
  static void pcg_spmv(const TopoDesc& t, const PcgArgs& a, Launch l) {
    on_topo(t, [&](const auto& topo) {
      using T = std::decay_t<decltype(topo)>;
      k_pcg_spmv<D, T><<<l.grid, kBlock, 0, l.stream>>>(topo, a);
    });
  }
  static void pcg_update(const TopoDesc& t, const PcgArgs& a, Launch l) {
    on_topo(t, [&](const auto& topo) {
      using T = std::decay_t<decltype(topo)>;
      k_pcg_update<D, T><<<l.grid, kBlock, 0, l.stream>>>(topo, a);
    });
  }
  static void pcg_finalize(int n, const double* x0, double* x, Ctl* ctl, Launch l) {
    k_pcg_finalize<D><<<l.grid, kBlock, 0, l.stream>>>(n, x0, x, ctl);
    k_inner_done<<<1, 32, 0, l.stream>>>(ctl);
  }
  static void sb_pass(const TopoDesc& t, const SbArgs& a, Launch l) {
    on_topo(t, [&](const auto& topo) {
      using T = std::decay_t<decltype(topo)>;
      k_sb_pass<D, T><<<l.grid, kBlock, 0, l.stream>>>(topo, a);
    });
  }
  static void rhs_from_state(const TopoDesc& t, const double* s, const double* b, const double* rq, double* rhs,
                             double hl, Launch l) {
    on_topo(t, [&](const auto& topo) {
      using T = std::decay_t<decltype(topo)>;
      k_rhs_from_state<D, T><<<l.grid, kBlock, 0, l.stream>>>(topo, s, b, rq, rhs, hl);
    });
  }
  static void rhs_quad(int n, const double* sqd, const double* p, const double* b, double* rq, double hr, Launch l) {
    k_rhs_quad<D><<<l.grid, kBlock, 0, l.stream>>>(n, sqd, p, b, rq, hr);
  }
  static void objective(const TopoDesc& t, const double* y, double* partials, Ctl* ctl, Launch l) {
    on_topo(t, [&](const auto& topo) {
      using T = std::decay_t<decltype(topo)>;
      k_objective<D, T><<<l.grid, kBlock, 0, l.stream>>>(topo, y, partials, ctl);
    });
  }
  static void diff_norms(int n, const double* ynew, const double* yold, double* partials, Ctl* ctl, Launch l) {
    k_diff_norms<D><<<l.grid, kBlock, 0, l.stream>>>(n, ynew, yold, partials, ctl);
  }
  static void tsqr_local(int n, const double* y, const double* sqd, const double* breg, double* rbuf, Launch l) {
    k_tsqr_local<D><<<l.grid, kBlock, 0, l.stream>>>(n, y, sqd, breg, rbuf);
  }
  static void tsqr_final(int nblk, const double* rbuf, double* w, Ctl* ctl, Launch l) {
    k_tsqr_final<D><<<1, kBlock, 0, l.stream>>>(nblk, rbuf, w, ctl);
  }
  static void project_apply(int n, const double* y, const double* sqd, double* breg, const double* w, double* p,
                            double* rq, double hr, Launch l) {
    k_project_apply<D><<<l.grid, kBlock, 0, l.stream>>>(n, y, sqd, breg, w, p, rq, hr);
  }
  static int max_blocks_per_sm() {
    int worst = 8, nb = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, k_pcg_spmv<D, Grid<2>>, kBlock, 0);
    worst = nb < worst ? nb : worst;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, k_sb_pass<D, Grid<2>>, kBlock, 0);
    worst = nb < worst ? nb : worst;
    return worst < 1 ? 1 : worst;
  }
};

template <int D>
LaunchTable make_table() {
  using I = Impl<D>;
  return LaunchTable{D,
                     &I::pcg_init,
                     &I::pcg_spmv,
                     &I::pcg_update,
                     &I::pcg_finalize,
                     &I::sb_pass,
                     &I::rhs_from_state,
                     &I::rhs_quad,
                     &I::objective,
                     &I::diff_norms,
                     &I::tsqr_local,
                     &I::tsqr_final,
                     &I::project_apply,
                     &I::max_blocks_per_sm};
}

}  // namespace pfe_host
