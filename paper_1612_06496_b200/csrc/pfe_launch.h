// Host-side launch table: one entry set per embedding dimension D (1..16),
// each dispatching on the graph topology.  The kernels are instantiated in
// pfe_kernels_d*.cu so the 16 x 3 template sets compile in parallel.
#pragma once

#include <cuda_runtime.h>

#include "pfe_device.cuh"

namespace pfe_dev {
struct PcgArgs;
struct SbArgs;
}  // namespace pfe_dev

namespace pfe_host {

enum TopoKind : int { kTopoCsr = 0, kTopoGrid1 = 1, kTopoGrid2 = 2 };

struct TopoDesc {
  int kind = kTopoCsr;
  pfe_dev::Grid<1> g1{};
  pfe_dev::Grid<2> g2{};
  pfe_dev::Csr csr{};
};

struct Launch {
  int grid;             // blocks (vertex-parallel kernels)
  cudaStream_t stream;
  int sm = 148;         // multiprocessors (tiled kernels size their own grid)
};

// Host view of pfe_dev::PersistArgs (topology supplied separately).
struct PersistIn {
  double* ybuf[2];
  int ycur;
  double* r;
  double* pbuf[2];
  double* q;
  double* eb[2];
  int ebcur;
  double* es;
  const double* rq;
  const double* rhs0;
  int b_zero, n_inner, write_s_last, rhs_last;
  double tol;
  int max_iter;
  double hl, gamma;
  pfe_dev::Ctl* ctl;
  double* part;
  double* part_b;
  unsigned long long* trace;  // optional phase trace (null: off)
  int trace_cap;
  int allow_resident;  // run the shared-memory-resident kernel when the state fits
  double* part_c;      // its init partials (2 x 3 x kMaxD x #SMs)
};

struct LaunchTable {
  int d;
  // block counts the PCG kernels launch with (consumers reduce that many partials)
  void (*pcg_grids)(const TopoDesc&, Launch, int* nb_init, int* nb_spmv, int* nb_update);
  void (*pcg_init)(const TopoDesc&, const pfe_dev::PcgArgs&, Launch);
  void (*pcg_spmv)(const TopoDesc&, const pfe_dev::PcgArgs&, Launch);
  void (*pcg_update)(const TopoDesc&, const pfe_dev::PcgArgs&, Launch);
  void (*pcg_finalize)(int n, const double* x0, double* x, pfe_dev::Ctl* ctl, Launch);
  void (*sb_pass)(const TopoDesc&, const pfe_dev::SbArgs&, Launch);
  void (*rhs_from_state)(const TopoDesc&, const double* s, const double* b, const double* rq, double* rhs,
                         double hl, Launch);
  void (*rhs_quad)(int n, const double* sqd, const double* p, const double* b, double* rq, double hr, Launch);
  void (*objective)(const TopoDesc&, const double* y, double* partials, pfe_dev::Ctl* ctl, Launch);
  void (*diff_norms)(int n, const double* ynew, const double* yold, double* partials, pfe_dev::Ctl* ctl, Launch);
  void (*tsqr_local)(int n, const double* y, const double* sqd, const double* breg, double* rbuf, Launch);
  void (*tsqr_final)(int nblk, const double* rbuf, double* w, pfe_dev::Ctl* ctl, Launch);
  void (*project_apply)(int n, const double* y, const double* sqd, double* breg, const double* w, double* p,
                        double* rq, double hr, Launch);
  // Largest resident grid (blocks) of the heaviest kernels, for partial sizing.
  int (*max_blocks_per_sm)();
  // Persistent cooperative split-Bregman kernel (grid topologies only).
  // Returns the variant launched: 0 none (topology without one), 1 tiled,
  // 2 shared-memory resident.
  int (*sb_persistent)(const TopoDesc&, const PersistIn&, Launch);
  // block partials -> nq * D totals (nq = 1 or 3), one block
  void (*local_totals)(int nq, const double* part, int nb, double* out, cudaStream_t);
  // CSR only: the direction pass p' = D^-1 r + beta p on its own (pcg_spmv
  // runs it first unless PcgArgs::skip_pdir), for partitioned solvers that
  // exchange p' ghosts between the two
  void (*pcg_pdir)(const TopoDesc&, const pfe_dev::PcgArgs&, Launch);
  // dst[i][D] = src[rows[i]][D] for i < cnt (ghost exchange packing)
  void (*pack_rows)(const double* src, const int* rows, int cnt, double* dst, cudaStream_t);
};

const LaunchTable& table_for(int d);  // d in [1, 16]

template <int D>
LaunchTable make_table();

}  // namespace pfe_host
