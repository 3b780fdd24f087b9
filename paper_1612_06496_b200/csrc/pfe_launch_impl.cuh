// Template bodies of the launch table (included by pfe_kernels_d*.cu only).
#pragma once

#include <cudaTypedefs.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <mutex>
#include <stdexcept>
#include <string>

#include "pfe_kernels.cuh"
#include "pfe_launch.h"
#include "pfe_polar.cuh"
#include "pfe_stencil.cuh"
#include "pfe_persist.cuh"
#include "pfe_resident.cuh"

namespace pfe_host {

using namespace pfe_dev;

// Every launch is checked: a failed launch (bad configuration, resources)
// must surface as an error, never as silently missing work.
inline void check_launch(const char* what) {
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) throw std::runtime_error(std::string("kernel launch failed (") + what + "): " + cudaGetErrorString(e));
}
#define PFE_LAUNCHED(name) check_launch(name)

// A value computed once per device (function attributes such as the
// dynamic shared-memory opt-in are per device, and one process may drive
// several devices from several host threads).
struct PerDeviceValue {
  std::mutex mu;
  long v[64] = {};
  bool set[64] = {};
  template <class F>
  long get(F&& f) {
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev < 0 || dev >= 64) dev = 0;
    std::lock_guard<std::mutex> lk(mu);
    if (!set[dev]) {
      v[dev] = f();
      set[dev] = true;
    }
    return v[dev];
  }
};

// cuTensorMapEncodeTiled through the runtime's driver entry point (no
// link-time dependency on libcuda).
inline PFN_cuTensorMapEncodeTiled_v12000 tma_encoder() {
  static const PFN_cuTensorMapEncodeTiled_v12000 fn = []() -> PFN_cuTensorMapEncodeTiled_v12000 {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q{};
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
    return nullptr;
  }();
  return fn;
}

// Map of an image-row array [H][W][K] (fp64) with box (K, bw, bh); K == 1
// arrays are 2-D.  Fails (false) when TMA's alignment rules are not met.
inline bool encode_rows(CUtensorMap* m, const void* base, int K, int W, int H, int bw, int bh) {
  auto enc = tma_encoder();
  if (!enc || !base || (reinterpret_cast<uintptr_t>(base) & 15) != 0) return false;
  const cuuint32_t es[3] = {1, 1, 1};
  CUresult r;
  if (K == 1) {
    if ((W * 8) % 16 != 0 || (bw * 8) % 16 != 0) return false;
    const cuuint64_t dims[2] = {static_cast<cuuint64_t>(W), static_cast<cuuint64_t>(H)};
    const cuuint64_t strides[1] = {static_cast<cuuint64_t>(W) * 8};
    const cuuint32_t box[2] = {static_cast<cuuint32_t>(bw), static_cast<cuuint32_t>(bh)};
    r = enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, const_cast<void*>(base), dims, strides, box, es,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  } else {
    if ((K * 8) % 16 != 0 || K > 256) return false;
    const cuuint64_t dims[3] = {static_cast<cuuint64_t>(K), static_cast<cuuint64_t>(W), static_cast<cuuint64_t>(H)};
    const cuuint64_t strides[2] = {static_cast<cuuint64_t>(K) * 8, static_cast<cuuint64_t>(W) * K * 8};
    const cuuint32_t box[3] = {static_cast<cuuint32_t>(K), static_cast<cuuint32_t>(bw), static_cast<cuuint32_t>(bh)};
    r = enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, const_cast<void*>(base), dims, strides, box, es,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  }
  return r == CUDA_SUCCESS;
}

// Phases of the persistent kernel that stage with TMA (PersistArgs::tma
// bits: 1 init, 2 SpMV, 4 split-Bregman, 8 b_old, 16 the one-wide arrays
// diag / inv diag).  Default: every phase.  PFE_TMA=0 forces cp.async
// everywhere (A/B tests), PFE_TMA=1 every phase, PFE_TMA=<mask> selects
// phases.
//
// Bit 16 is never set for odd R.  Root cause of the round-1 "illegal
// instruction" on 8-neighbour grids (scripts/tma_probe.cu, run case by case
// on B200): a 2-D box of a one-wide fp64 array whose first column is odd
// starts at an 8-byte but not 16-byte aligned global address, and the TMA
// unit faults; 3-D boxes of even row width are always 16-byte aligned.  The
// halo box of inv diag starts at column x0 - R (x0 a multiple of 32), odd
// for R = 1, so those arrays stay on cp.async there.
inline int tma_mask(int radius) {
  const char* e = std::getenv("PFE_TMA");
  int m = 31;  // every phase (C4: 57.4 -> 63.6 inner it/s over cp.async tiles)
  if (e && e[0]) m = std::atoi(e) == 1 ? 31 : std::atoi(e);
  if (radius % 2 != 0) m &= ~16;
  return m;
}

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

  // Tiled stencil kernels: grid = min(tiles, resident blocks), dynamic smem.
  template <int R, auto Kern>
  static int tiled_grid(size_t smem, const Grid<R>& g, int sm) {
    using G = TileGeo<R, D>;
    static PerDeviceValue cache;  // one value per kernel instantiation and device
    const int per_sm = static_cast<int>(cache.get([&]() -> long {
      if (smem > 48 * 1024) cudaFuncSetAttribute(Kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      int nb = 0;
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, Kern, G::NT, smem);
      return nb < 1 ? 1 : nb;
    }));
    const long tiles = static_cast<long>((g.W + G::TW - 1) / G::TW) * ((g.H + G::TH - 1) / G::TH);
    return static_cast<int>(tiles < static_cast<long>(per_sm) * sm ? tiles : static_cast<long>(per_sm) * sm);
  }
  template <int R>
  static void grid_init(const Grid<R>& g, const PcgArgs& a, Launch l) {
    using G = TileGeo<R, D>;
    constexpr size_t sm_bytes = sizeof(double) * G::kInit;
    const int grid = tiled_grid<R, k_grid_pcg_init<D, R>>(sm_bytes, g, l.sm);
    k_grid_pcg_init<D, R><<<grid, G::NT, sm_bytes, l.stream>>>(g, a); PFE_LAUNCHED(__func__);
  }
  template <int R>
  static void grid_spmv(const Grid<R>& g, const PcgArgs& a, Launch l) {
    using G = TileGeo<R, D>;
    constexpr size_t sm_bytes = sizeof(double) * G::kSpmv;
    const int grid = tiled_grid<R, k_grid_pcg_spmv<D, R>>(sm_bytes, g, l.sm);
    k_grid_pcg_spmv<D, R><<<grid, G::NT, sm_bytes, l.stream>>>(g, a); PFE_LAUNCHED(__func__);
  }
  template <int R>
  static void grid_sb(const Grid<R>& g, const SbArgs& a, Launch l) {
    using G = TileGeo<R, D>;
    constexpr size_t sm_bytes = sizeof(double) * G::kSb;
    const int grid = tiled_grid<R, k_grid_sb_pass<D, R>>(sm_bytes, g, l.sm);
    k_grid_sb_pass<D, R><<<grid, G::NT, sm_bytes, l.stream>>>(g, a); PFE_LAUNCHED(__func__);
  }

  // General-graph (CSR) gather kernels sweep the storage order in
  // grid-stride chunks (row_range); that is a sweep of one window only if
  // every block is resident at once, so their grid is capped at the
  // resident block count (SMs x occupancy).  With more blocks, the first
  // resident wave would walk its chunks over the whole vertex range before
  // later blocks start, and the gathered rows would miss L2.
  template <auto Kern>
  static int csr_grid(Launch l) {
    static PerDeviceValue cache;  // one value per kernel instantiation and device
    const int per_sm = static_cast<int>(cache.get([&]() -> long {
      int nb = 0;
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, Kern, kBlock, 0);
      return nb < 1 ? 1 : nb;
    }));
    return std::max(1, std::min(l.grid, per_sm * l.sm));
  }

  static void pcg_grids(const TopoDesc& t, Launch l, int* nb_init, int* nb_spmv, int* nb_update) {
    *nb_update = l.grid;
    if (t.kind == kTopoGrid1) {
      using G = TileGeo<1, D>;
      *nb_init = tiled_grid<1, k_grid_pcg_init<D, 1>>(sizeof(double) * G::kInit, t.g1, l.sm);
      *nb_spmv = tiled_grid<1, k_grid_pcg_spmv<D, 1>>(sizeof(double) * G::kSpmv, t.g1, l.sm);
    } else if (t.kind == kTopoGrid2) {
      using G = TileGeo<2, D>;
      *nb_init = tiled_grid<2, k_grid_pcg_init<D, 2>>(sizeof(double) * G::kInit, t.g2, l.sm);
      *nb_spmv = tiled_grid<2, k_grid_pcg_spmv<D, 2>>(sizeof(double) * G::kSpmv, t.g2, l.sm);
    } else {
      *nb_init = csr_grid<k_pcg_init<D, Csr>>(l);
      *nb_spmv = csr_grid<k_pcg_spmv<D, Csr>>(l);
    }
  }
  static void pcg_init(const TopoDesc& t, const PcgArgs& a, Launch l) {
    if (t.kind == kTopoGrid1) return grid_init<1>(t.g1, a, l);
    if (t.kind == kTopoGrid2) return grid_init<2>(t.g2, a, l);
    k_pcg_init<D, Csr><<<csr_grid<k_pcg_init<D, Csr>>(l), kBlock, 0, l.stream>>>(t.csr, a); PFE_LAUNCHED(__func__);
  }
  static void pcg_spmv(const TopoDesc& t, const PcgArgs& a, Launch l) {
    if (t.kind == kTopoGrid1) return grid_spmv<1>(t.g1, a, l);
    if (t.kind == kTopoGrid2) return grid_spmv<2>(t.g2, a, l);
    if (a.phase != 0 && !a.skip_pdir) {
      k_pcg_pdir<D, Csr><<<csr_grid<k_pcg_pdir<D, Csr>>(l), kBlock, 0, l.stream>>>(t.csr, a); PFE_LAUNCHED(__func__);
    }
    k_pcg_spmv<D, Csr><<<csr_grid<k_pcg_spmv<D, Csr>>(l), kBlock, 0, l.stream>>>(t.csr, a); PFE_LAUNCHED(__func__);
  }
  static void pcg_pdir(const TopoDesc& t, const PcgArgs& a, Launch l) {
    if (t.kind != kTopoCsr) throw std::runtime_error("pcg_pdir: CSR topologies only");
    k_pcg_pdir<D, Csr><<<csr_grid<k_pcg_pdir<D, Csr>>(l), kBlock, 0, l.stream>>>(t.csr, a); PFE_LAUNCHED(__func__);
  }
  static void pack_rows(const double* src, const int* rows, int cnt, double* dst, cudaStream_t s) {
    if (cnt <= 0) return;
    const int grid = static_cast<int>(std::min<long>(4096, (static_cast<long>(cnt) * D + kBlock - 1) / kBlock));
    k_pack_rows<D><<<grid, kBlock, 0, s>>>(src, rows, cnt, dst); PFE_LAUNCHED(__func__);
  }
  static void pcg_update(const TopoDesc& t, const PcgArgs& a, Launch l) {
    on_topo(t, [&](const auto& topo) {
      using T = std::decay_t<decltype(topo)>;
      k_pcg_update<D, T><<<l.grid, kBlock, 0, l.stream>>>(topo, a); PFE_LAUNCHED(__func__);
    });
  }
  static void pcg_finalize(int n, const double* x0, double* x, Ctl* ctl, Launch l) {
    k_pcg_finalize<D><<<l.grid, kBlock, 0, l.stream>>>(n, x0, x, ctl); PFE_LAUNCHED(__func__);
  }
  static void sb_pass(const TopoDesc& t, const SbArgs& a, Launch l) {
    if (t.kind == kTopoGrid1) return grid_sb<1>(t.g1, a, l);
    if (t.kind == kTopoGrid2) return grid_sb<2>(t.g2, a, l);
    k_sb_pass<D, Csr><<<csr_grid<k_sb_pass<D, Csr>>(l), kBlock, 0, l.stream>>>(t.csr, a); PFE_LAUNCHED(__func__);
  }
  static void rhs_from_state(const TopoDesc& t, const double* s, const double* b, const double* rq, double* rhs,
                             double hl, Launch l) {
    on_topo(t, [&](const auto& topo) {
      using T = std::decay_t<decltype(topo)>;
      k_rhs_from_state<D, T><<<l.grid, kBlock, 0, l.stream>>>(topo, s, b, rq, rhs, hl); PFE_LAUNCHED(__func__);
    });
  }
  static void rhs_quad(int n, const double* sqd, const double* p, const double* b, double* rq, double hr, Launch l) {
    k_rhs_quad<D><<<l.grid, kBlock, 0, l.stream>>>(n, sqd, p, b, rq, hr); PFE_LAUNCHED(__func__);
  }
  static void objective(const TopoDesc& t, const double* y, double* partials, Ctl* ctl, Launch l) {
    on_topo(t, [&](const auto& topo) {
      using T = std::decay_t<decltype(topo)>;
      k_objective<D, T><<<l.grid, kBlock, 0, l.stream>>>(topo, y, partials, ctl); PFE_LAUNCHED(__func__);
    });
  }
  static void diff_norms(int n, const double* ynew, const double* yold, double* partials, Ctl* ctl, Launch l) {
    k_diff_norms<D><<<l.grid, kBlock, 0, l.stream>>>(n, ynew, yold, partials, ctl); PFE_LAUNCHED(__func__);
  }
  static void tsqr_local(int n, const double* y, const double* sqd, const double* breg, double* rbuf, Launch l) {
    k_tsqr_local<D><<<l.grid, kBlock, 0, l.stream>>>(n, y, sqd, breg, rbuf); PFE_LAUNCHED(__func__);
  }
  static void tsqr_final(int nblk, const double* rbuf, double* w, Ctl* ctl, Launch l) {
    k_tsqr_final<D><<<1, kBlock, 0, l.stream>>>(nblk, rbuf, w, ctl); PFE_LAUNCHED(__func__);
  }
  static void project_apply(int n, const double* y, const double* sqd, double* breg, const double* w, double* p,
                            double* rq, double hr, Launch l) {
    k_project_apply<D><<<l.grid, kBlock, 0, l.stream>>>(n, y, sqd, breg, w, p, rq, hr); PFE_LAUNCHED(__func__);
  }
  // Region grid of the shared-memory-resident kernel: rgx x rgy <= #SMs
  // regions minimising the largest region + ring (the per-block work), under
  // the shared-memory, per-thread element and ring limits.  ok = false: the
  // state does not fit; the tiled persistent kernel runs instead.
  struct ResPlan {
    bool ok = false;
    int gx = 0, gy = 0, hw = 0, np = 0;
    size_t smem = 0;
  };
  template <int R>
  static ResPlan res_plan(const Grid<R>& g, int sms) {
    using G = ResGeo<D, R>;
    static PerDeviceValue cache;
    const size_t avail = static_cast<size_t>(cache.get([]() -> long {
      int dev = 0, optin = 0;
      cudaGetDevice(&dev);
      cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
      cudaFuncAttributes fa{};
      cudaFuncGetAttributes(&fa, k_sb_resident<D, R>);
      const long av = static_cast<long>(optin) - static_cast<long>(fa.sharedSizeBytes);
      cudaFuncSetAttribute(k_sb_resident<D, R>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)av);
      return av;
    }));
    ResPlan best;
    if (g.row_lo != 0 || g.row_hi != g.H) return best;  // single-domain solvers only
    const int max_blocks = std::min(sms, G::kMaxBlocks);
    for (int gy = 1; gy <= g.H && gy <= max_blocks; ++gy) {
      const int gx = std::min(g.W, max_blocks / gy);
      const int rh = (g.H + gy - 1) / gy, rw = (g.W + gx - 1) / gx;
      const int hw = rw + 2 * R, np = hw * (rh + 2 * R);
      const size_t smem = sizeof(double) * static_cast<size_t>(np) * G::kPerPos;
      const long ring = 2L * R * hw + 2L * R * rh;
      if (smem > avail || static_cast<long>(rh) * rw * G::U > static_cast<long>(G::NT) * G::EPT ||
          ring * D > static_cast<long>(G::NT) * G::HR)
        continue;
      if (!best.ok || np < best.np || (np == best.np && gx * gy < best.gx * best.gy)) {
        best.ok = true;
        best.gx = gx;
        best.gy = gy;
        best.hw = hw;
        best.np = np;
        best.smem = smem;
      }
    }
    return best;
  }
  template <int R>
  static int persist_grid(const Grid<R>& g, const PersistIn& in, Launch l) {
    constexpr size_t smem = sizeof(double) * PersistGeo<D, R>::kSmem;
    static PerDeviceValue cache;
    const int per_sm = static_cast<int>(cache.get([]() -> long {
      cudaFuncSetAttribute(k_sb_persistent<D, R>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      int nb = 0;
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, k_sb_persistent<D, R>, TileGeo<R, D>::NT, smem);
      if (const char* e = std::getenv("PFE_SETUP_TIMING"); e && e[0] == '1')
        std::fprintf(stderr, "k_sb_persistent<%d,%d>: %zu B dynamic shared memory, %d block(s) per SM\n", D, R, smem, nb);
      return nb;
    }));
    if (per_sm < 1) throw std::runtime_error("persistent split-Bregman kernel does not fit on an SM");
    PersistArgs<R> a{};
    a.g = g;
    a.ybuf[0] = in.ybuf[0];
    a.ybuf[1] = in.ybuf[1];
    a.ycur = in.ycur;
    a.r = in.r;
    a.pbuf[0] = in.pbuf[0];
    a.pbuf[1] = in.pbuf[1];
    a.q = in.q;
    a.eb[0] = in.eb[0];
    a.eb[1] = in.eb[1];
    a.ebcur = in.ebcur;
    a.es = in.es;
    a.rq = in.rq;
    a.rhs0 = in.rhs0;
    a.b_zero = in.b_zero;
    a.n_inner = in.n_inner;
    a.write_s_last = in.write_s_last;
    a.rhs_last = in.rhs_last;
    a.tol = in.tol;
    a.max_iter = in.max_iter;
    a.hl = in.hl;
    a.gamma = in.gamma;
    a.ctl = in.ctl;
    a.part = in.part;
    a.part_b = in.part_b;
    a.trace = in.trace;
    a.trace_cap = in.trace_cap;
    a.part_c = in.part_c;
    void* args[] = {&a};
    if (in.allow_resident) {
      const ResPlan rp = res_plan<R>(g, l.sm);
      if (rp.ok) {
        a.rgx = rp.gx;
        a.rgy = rp.gy;
        a.rhw = rp.hw;
        a.rnp = rp.np;
        const cudaError_t e = cudaLaunchCooperativeKernel(reinterpret_cast<const void*>(&k_sb_resident<D, R>),
                                                          dim3(rp.gx * rp.gy), dim3(ResGeo<D, R>::NT), args,
                                                          rp.smem, l.stream);
        if (e != cudaSuccess)
          throw std::runtime_error(std::string("cooperative launch failed: ") + cudaGetErrorString(e));
        return 2;
      }
    }
    // TMA staging: every tile array is a box of one tensor map (even d and
    // image width; pfe_tma.cuh)
    using G = TileGeo<R, D>;
    a.tma = 0;
    if (tma_mask(R) != 0 && D % 2 == 0 && g.W % 2 == 0) {
      TileMaps& tm = a.tm;
      const int W = g.W, H = g.H;
      bool ok = true;
      for (int i = 0; i < 2; ++i) {
        ok = ok && encode_rows(&tm.y[i], in.ybuf[i], D, W, H, G::HW, G::HH);
        ok = ok && encode_rows(&tm.p[i], in.pbuf[i], D, W, H, G::HW, G::HH);
      }
      ok = ok && encode_rows(&tm.r_halo, in.r, D, W, H, G::HW, G::HH);
      ok = ok && encode_rows(&tm.r_int, in.r, D, W, H, G::TW, G::TH);
      ok = ok && encode_rows(&tm.rhs0_int, in.rhs0, D, W, H, G::TW, G::TH);
      ok = ok && encode_rows(&tm.iv_halo, g.invd, 1, W, H, G::HW, G::HH);
      ok = ok && encode_rows(&tm.iv_int, g.invd, 1, W, H, G::TW, G::TH);
      ok = ok && encode_rows(&tm.dg_int, g.diag, 1, W, H, G::TW, G::TH);
      ok = ok && encode_rows(&tm.cf_halo, g.cf, G::S, W, H, G::HW, G::HH);
      ok = ok && encode_rows(&tm.wf_halo, g.wf, G::S, W, H, G::HW, G::HH);
      if (in.rq) ok = ok && encode_rows(&tm.rq_int, in.rq, D, W, H, G::TW, G::TH);
      if (G::kStageB)
        for (int i = 0; i < 2; ++i) ok = ok && encode_rows(&tm.bo[i], in.eb[i], G::S * D, W, H, G::HW, G::TH + R);
      a.tma = ok ? tma_mask(R) : 0;
    }
    // PFE_BULK=1 (no TMA, even d): halo rows as cp.async.bulk row copies.
    // Off by default: bit-identical, but on C4 (8-neighbour, d = 8) it
    // measured 49.9 vs 50.9 inner it/s for per-element cp.async -- that
    // kernel is bound by DRAM latency / pipeline depth, not by the staging
    // instructions.
    {
      const char* b = std::getenv("PFE_BULK");
      a.bulk = (a.tma == 0 && D % 2 == 0 && b && b[0] == '1') ? 1 : 0;
    }
    const char* one = std::getenv("PFE_PERSIST_ONE_CTA");  // debugging: one block per SM
    const int grid = (one && one[0] == '1' ? 1 : per_sm) * l.sm;
    const cudaError_t e = cudaLaunchCooperativeKernel(reinterpret_cast<const void*>(&k_sb_persistent<D, R>),
                                                      dim3(grid), dim3(TileGeo<R, D>::NT), args, smem, l.stream);
    if (e != cudaSuccess)
      throw std::runtime_error(std::string("cooperative launch failed: ") + cudaGetErrorString(e));
    return 1;
  }
  static int sb_persistent(const TopoDesc& t, const PersistIn& in, Launch l) {
    if (t.kind == kTopoGrid1) return persist_grid<1>(t.g1, in, l);
    if (t.kind == kTopoGrid2) return persist_grid<2>(t.g2, in, l);
    return 0;
  }
  static void local_totals(int nq, const double* part, int nb, double* out, cudaStream_t s) {
    if (nq == 3)
      k_local_totals<3, D><<<1, kBlock, 0, s>>>(part, nb, out);
    else
      k_local_totals<1, D><<<1, kBlock, 0, s>>>(part, nb, out);
    PFE_LAUNCHED(__func__);
  }
  static int max_blocks_per_sm() {
    int worst = 8, nb = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, k_pcg_spmv<D, Csr>, kBlock, 0);
    worst = nb < worst ? nb : worst;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, k_sb_pass<D, Csr>, kBlock, 0);
    worst = nb < worst ? nb : worst;
    return worst < 1 ? 1 : worst;
  }
};

template <int D>
LaunchTable make_table() {
  using I = Impl<D>;
  return LaunchTable{D,
                     &I::pcg_grids,
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
                     &I::max_blocks_per_sm,
                     &I::sb_persistent,
                     &I::local_totals,
                     &I::pcg_pdir,
                     &I::pack_rows};
}

}  // namespace pfe_host
