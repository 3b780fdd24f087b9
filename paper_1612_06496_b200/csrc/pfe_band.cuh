// Row-band decomposition of pixel-grid graphs over several GPUs
// (DESIGN.md §6).  Included by pfe_runtime.cu inside its
// anonymous namespace (needs pfe_solver / pfe_state).
//
// Band p of P owns global image rows [r0, r1) and stores rows [lo, hi) =
// [r0 - R, r1 + R) clipped to the image: its owned rows plus an R-row halo
// (R = stencil radius).  Every kernel processes owned rows only (Grid::row_lo
// / row_hi); the halo rows are copies refreshed from the neighbouring bands:
//   * p0 after init and r after every update (the fused SpMV recomputes
//     p' = D^-1 r + beta p on its halo from exchanged r and stores the halo
//     rows of p' itself, so p' needs no exchange: one halo exchange per PCG
//     iteration),
//   * Y after every result selection (init and the split-Bregman pass read
//     the neighbours' rows).
// split_b / split_s of an edge crossing a band boundary are replicated in both
// bands: the lower band updates its copy with exactly the arithmetic the
// owning band uses, so no edge data is ever exchanged.  PCG reductions: each
// band reduces its block partials to d or 3d totals, the totals of all bands
// are gathered, and every band sums them in rank order, so all bands take
// identical alpha / beta / stop decisions.  The TSQR factors of all bands are
// gathered the same way before the d x d polar step.
//
// Transport: bands in separate processes (one GPU each) use NCCL send/recv
// for halos and all-gathers for totals (loaded at run time from
// libnccl.so.2); bands emulated inside one process (pfe_solve_banded, used to
// validate the decomposition on one GPU) use device-to-device copies.

struct BandPlan {
  int r0, r1, lo, hi;
};

BandPlan band_plan(int H, int P, int R, int p) {
  const int r0 = static_cast<int>(static_cast<long>(H) * p / P);
  const int r1 = static_cast<int>(static_cast<long>(H) * (p + 1) / P);
  return {r0, r1, p > 0 ? std::max(0, r0 - R) : r0, p < P - 1 ? std::min(H, r1 + R) : r1};
}

// ------------------------------------------------------------------ NCCL --
struct NcclApi {
  void* h = nullptr;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommInitAll)(ncclComm_t*, int, const int*) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

NcclApi& nccl() {
  static NcclApi api;
  if (api.h) return api;
  void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
  if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
  if (!h) config_error(std::string("multi-GPU row bands need NCCL: ") + dlerror());
  auto sym = [&](const char* name) {
    void* f = dlsym(h, name);
    if (!f) config_error(std::string("NCCL symbol missing: ") + name);
    return f;
  };
  api.GetUniqueId = reinterpret_cast<decltype(api.GetUniqueId)>(sym("ncclGetUniqueId"));
  api.CommInitRank = reinterpret_cast<decltype(api.CommInitRank)>(sym("ncclCommInitRank"));
  api.CommInitAll = reinterpret_cast<decltype(api.CommInitAll)>(sym("ncclCommInitAll"));
  api.CommDestroy = reinterpret_cast<decltype(api.CommDestroy)>(sym("ncclCommDestroy"));
  api.AllGather = reinterpret_cast<decltype(api.AllGather)>(sym("ncclAllGather"));
  api.Send = reinterpret_cast<decltype(api.Send)>(sym("ncclSend"));
  api.Recv = reinterpret_cast<decltype(api.Recv)>(sym("ncclRecv"));
  api.GroupStart = reinterpret_cast<decltype(api.GroupStart)>(sym("ncclGroupStart"));
  api.GroupEnd = reinterpret_cast<decltype(api.GroupEnd)>(sym("ncclGroupEnd"));
  api.GetErrorString = reinterpret_cast<decltype(api.GetErrorString)>(sym("ncclGetErrorString"));
  api.h = h;
  g_comm_destroy = [](void* c) { nccl().CommDestroy(static_cast<ncclComm_t>(c)); };
  return api;
}

void nccl_check(ncclResult_t r, const char* what) {
  if (r != ncclSuccess)
    throw Error(PFE_CUDA_ERROR, std::string(what) + " failed: " + nccl().GetErrorString(r));
}

// ------------------------------------------------------ band construction --
// Global slot weights -> this band's rows; diag(A) and its inverse are taken
// from the GLOBAL graph (halo vertices have edges outside the band).
void setup_band_grid(pfe_solver* S, const HostGraph& g, int gh, int gw, int grad, const BandPlan& bp) {
  const int S_ = grad == 1 ? 4 : 12;
  if (!(gh > 0 && gw > 0 && static_cast<long>(gh) * gw == g.n && (grad == 1 || grad == 2) && gw >= 2 * grad + 2))
    config_error("row bands need a pixel-grid graph (grid_h * grid_w == n, radius 1 or 2)");
  const double hl = 0.5 * S->prm.lambda, dterm = 0.5 * S->prm.r;
  std::vector<double> wf(static_cast<size_t>(g.n) * S_, 0.0);
  for (long k = 0; k < g.m; ++k) {
    if (k > 0 && !(g.ei[k - 1] < g.ei[k] || (g.ei[k - 1] == g.ei[k] && g.ej[k - 1] < g.ej[k])))
      config_error("row bands need lexicographically ordered grid edges");
    const int s = grid_slot(grad, gw, g.ei[k], g.ej[k]);
    if (s < 0) config_error("row bands: edge " + std::to_string(k) + " is not a stencil neighbour");
    wf[static_cast<size_t>(g.ei[k]) * S_ + s] = g.w[k];
  }
  const long vb = static_cast<long>(bp.lo) * gw, ve = static_cast<long>(bp.hi) * gw, nl = ve - vb;
  std::vector<double> wl(wf.begin() + vb * S_, wf.begin() + ve * S_);
  std::vector<double> diag(nl), invd(nl), deg(nl), sqd(nl);
  for (long v = vb; v < ve; ++v) {
    const int y = static_cast<int>(v / gw), x = static_cast<int>(v % gw);
    double acc = 0.0;
    for (int s = S_ - 1; s >= 0; --s) {  // backward slots (u ascending)
      const int dy = grad == 1 ? (s == 0 ? 0 : 1) : (s < 2 ? 0 : (s < 7 ? 1 : 2));
      const int dx = grad == 1 ? (s == 0 ? 1 : s - 2) : (s < 2 ? s + 1 : (s < 7 ? s - 4 : s - 9));
      const int yy = y - dy, xx = x - dx;
      if (yy < 0 || xx < 0 || xx >= gw) continue;
      const double w = wf[static_cast<size_t>(static_cast<long>(yy) * gw + xx) * S_ + s];
      acc += (hl * w) * w;
    }
    for (int s = 0; s < S_; ++s) {
      const double w = wf[static_cast<size_t>(v) * S_ + s];
      acc += (hl * w) * w;
    }
    const long l = v - vb;
    diag[l] = acc + dterm * g.deg[v];
    invd[l] = S->prm.preconditioner == PFE_PRECOND_NONE ? 1.0 : (diag[l] > 0.0 ? 1.0 / diag[l] : 1.0);
    deg[l] = g.deg[v];
    sqd[l] = std::sqrt(g.deg[v]);
  }
  S->n = static_cast<int>(nl);
  S->deg = S->mem.upload(deg, S->stream);
  S->sqd = S->mem.upload(sqd, S->stream);
  S->diag = S->mem.upload(diag, S->stream);
  S->invd = S->mem.upload(invd, S->stream);
  double* dwf = S->mem.upload(wl, S->stream);
  S->row_lo = bp.r0 - bp.lo;
  S->row_hi = bp.r1 - bp.lo;
  S->part = 1;
  S->own_vb = static_cast<long>(S->row_lo) * gw;
  S->own_cnt = (S->row_hi - S->row_lo) * gw;
  S->band_h = gh;
  S->band_w = gw;
  S->band_rad = grad;
  S->band_r0 = bp.r0;
  S->band_r1 = bp.r1;
  S->band_lo = bp.lo;
  S->edge_rows = nl * S_;
  const int hloc = bp.hi - bp.lo;
  double* dcf = grid_coef(S, dwf, nl * S_, hl, S->stream);
  if (grad == 1) {
    S->topo.kind = pfe_host::kTopoGrid1;
    S->topo.g1 = pfe_dev::Grid<1>{S->n, hloc, gw, hl, dwf, S->diag, S->invd, S->row_lo, S->row_hi};
    S->topo.g1.cf = dcf;
  } else {
    S->topo.kind = pfe_host::kTopoGrid2;
    S->topo.g2 = pfe_dev::Grid<2>{S->n, hloc, gw, hl, dwf, S->diag, S->invd, S->row_lo, S->row_hi};
    S->topo.g2.cf = dcf;
  }
}

// IC(0) for partitioned solvers (the reference default, pcg.cpp:22-28).  The
// factor depends on the global row order, and its triangular solves are
// sequential across any row partition, so every rank keeps the factor of the
// GLOBAL matrix (built exactly as the single-GPU solver builds it) and
// applies it to the gathered global residual; it then uses its own rows of
// z.  All ranks compute the same z and the same r.z total (bitwise the
// single-GPU values), so no rank waits on another inside a sweep.  `pos`
// maps a vertex to its row in the team's global order (identity for row
// bands, the breadth-first storage position for vertex ranges).
void setup_team_ic(pfe_solver* S, const HostGraph& hg, const Incidence& inc, const std::vector<int>& pos) {
  const int n = hg.n;
  const double hl = 0.5 * S->prm.lambda, dterm = 0.5 * S->prm.r;
  std::vector<double> diag(static_cast<size_t>(n));
  parallel_for(n, [&](long vb, long ve) {
    for (long v = vb; v < ve; ++v) {
      double acc = 0.0;
      for (int k = inc.iptr[v]; k < inc.iptr[v + 1]; ++k) acc += (hl * inc.iw[k]) * inc.iw[k];
      diag[v] = acc + dterm * hg.deg[v];  // the (r/2) d_v triplet is summed last
    }
  }, 4096);
  std::vector<int> nptr, ncol;
  std::vector<double> nval;
  natural_rows(n, inc, hl, diag.data(), nptr, ncol, nval);
  const int n_local = S->n;
  S->ic = true;
  build_ic(S, n, nptr, ncol, nval, pos);  // clears S->ic and sets jacobi_fallback on a breakdown
  S->ic_team = S->ic;
  S->ic = false;  // the single-GPU IC loop is not used by teams
  S->jacobi_fallback = !S->ic_team;
  if (S->ic_team) {
    S->rfull = S->mem.alloc<double>(static_cast<size_t>(n) * S->d);
    S->ic_part = S->mem.alloc<double>(static_cast<size_t>(std::max(1, std::min(S->max_grid, (n + 255) / 256))) * S->d);
    std::vector<double> one(static_cast<size_t>(n_local), 1.0);
    S->ones = S->mem.upload(one, S->stream);
    CK(cudaStreamSynchronize(S->stream));
  }
}

// The same band arrays derived on the device (round 2): only the edges whose
// first endpoint lies in the band's rows, plus the R rows above (their
// weights enter diag(A) of the band's first rows), are uploaded -- a
// contiguous slice of the lexicographic edge list -- and the slot weights,
// diag, inv diag, sqrt(deg) and coefficients come from the kernels of the
// single-GPU grid builder run on that sub-grid.  Per band this costs O(m / P)
// instead of the O(n + m) host loops of setup_band_grid (C4: ~1.5 s per
// band), which is what the one-call multi-GPU path pays once per band.
// Returns false when the slice breaks the grid contract (the caller then
// takes the host path, which reports the offending edge).
bool setup_band_grid_device(pfe_solver* S, const HostGraph& g, int gh, int gw, int grad, const BandPlan& bp) {
  const int S_ = grad == 1 ? 4 : 12;
  if (!(gh > 0 && gw > 0 && static_cast<long>(gh) * gw == g.n && (grad == 1 || grad == 2) && gw >= 2 * grad + 2))
    return false;
  // first endpoints must ascend for the slice search (full order is checked on the slice by the kernel)
  std::atomic<bool> sorted{true};
  parallel_for(g.m, [&](long kb, long ke) {
    for (long k = std::max(1L, kb); k < ke; ++k)
      if (g.ei[k - 1] > g.ei[k]) {
        sorted = false;
        return;
      }
  });
  if (!sorted) return false;
  const double hl = 0.5 * S->prm.lambda, dterm = 0.5 * S->prm.r;
  const int elo = std::max(0, bp.lo - grad), ehi = bp.hi;  // rows whose edges are needed
  const int voff = elo * gw;
  const long k0 = std::lower_bound(g.ei, g.ei + g.m, voff) - g.ei;
  const long k1 = std::lower_bound(g.ei, g.ei + g.m, ehi * gw) - g.ei;
  const long ms = k1 - k0, ne = static_cast<long>(ehi - elo) * gw, nl = static_cast<long>(bp.hi - bp.lo) * gw;
  const long off = static_cast<long>(bp.lo - elo) * gw;  // local row 0 inside the extended sub-grid
  cudaStream_t st = S->stream;
  DevPool tmp;
  tmp.stream = tmp.fstream = st;
  int32_t* d_ei = tmp.alloc<int32_t>(static_cast<size_t>(std::max(ms, 1L)));
  int32_t* d_ej = tmp.alloc<int32_t>(static_cast<size_t>(std::max(ms, 1L)));
  double* d_w = tmp.alloc<double>(static_cast<size_t>(std::max(ms, 1L)));
  int* d_bad = tmp.alloc<int>(1);
  double* wf_e = S->mem.alloc<double>(static_cast<size_t>(ne) * S_);
  double* deg_e = S->mem.alloc<double>(static_cast<size_t>(ne));
  double* diag_e = S->mem.alloc<double>(static_cast<size_t>(ne));
  double* invd_e = S->mem.alloc<double>(static_cast<size_t>(ne));
  double* sqd_e = S->mem.alloc<double>(static_cast<size_t>(ne));
  if (ms > 0) {
    copy_h2d(d_ei, g.ei + k0, sizeof(int32_t) * ms, st);
    copy_h2d(d_ej, g.ej + k0, sizeof(int32_t) * ms, st);
    copy_h2d(d_w, g.w + k0, sizeof(double) * ms, st);
  }
  copy_h2d(deg_e, g.deg + voff, sizeof(double) * ne, st);
  CK(cudaMemsetAsync(wf_e, 0, sizeof(double) * ne * S_, st));
  CK(cudaMemsetAsync(d_bad, 0, sizeof(int), st));
  const int eb = static_cast<int>(std::min<long>(std::max<long>(1, (ms + 255) / 256), 32L * S->sm));
  if (ms > 0) k_grid_slots<<<eb, 256, 0, st>>>(ms, gw, grad, d_ei, d_ej, d_w, wf_e, nullptr, d_bad, voff);
  CK(cudaGetLastError());
  int bad = 0;
  CK(cudaMemcpyAsync(&bad, d_bad, sizeof(int), cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  // edges of the slice must stay inside the rows the band stores (+ R below)
  if (bad) {
    S->mem.release(wf_e);
    S->mem.release(deg_e);
    S->mem.release(diag_e);
    S->mem.release(invd_e);
    S->mem.release(sqd_e);
    return false;
  }
  const int vb = static_cast<int>(std::max<long>(1, std::min<long>((ne + 255) / 256, 32L * S->sm)));
  k_grid_diag<<<vb, 256, 0, st>>>(ehi - elo, gw, grad, hl, dterm, S->prm.preconditioner == PFE_PRECOND_NONE, wf_e,
                                  deg_e, diag_e, invd_e);
  k_sqrt<<<vb, 256, 0, st>>>(ne, deg_e, sqd_e);
  CK(cudaGetLastError());
  S->n = static_cast<int>(nl);
  S->deg = deg_e + off;
  S->sqd = sqd_e + off;
  S->diag = diag_e + off;
  S->invd = invd_e + off;
  double* dwf = wf_e + off * S_;
  S->row_lo = bp.r0 - bp.lo;
  S->row_hi = bp.r1 - bp.lo;
  S->part = 1;
  S->own_vb = static_cast<long>(S->row_lo) * gw;
  S->own_cnt = (S->row_hi - S->row_lo) * gw;
  S->band_h = gh;
  S->band_w = gw;
  S->band_rad = grad;
  S->band_r0 = bp.r0;
  S->band_r1 = bp.r1;
  S->band_lo = bp.lo;
  S->edge_rows = nl * S_;
  const int hloc = bp.hi - bp.lo;
  double* dcf = grid_coef(S, dwf, nl * S_, hl, st);
  CK(cudaStreamSynchronize(st));  // the temporaries are freed next
  if (grad == 1) {
    S->topo.kind = pfe_host::kTopoGrid1;
    S->topo.g1 = pfe_dev::Grid<1>{S->n, hloc, gw, hl, dwf, S->diag, S->invd, S->row_lo, S->row_hi};
    S->topo.g1.cf = dcf;
  } else {
    S->topo.kind = pfe_host::kTopoGrid2;
    S->topo.g2 = pfe_dev::Grid<2>{S->n, hloc, gw, hl, dwf, S->diag, S->invd, S->row_lo, S->row_hi};
    S->topo.g2.cf = dcf;
  }
  return true;
}

pfe_solver* create_band_solver(const pfe_graph* g, const pfe_params* p, const pfe_exec* x, int nranks, int rank,
                               void* comm) {
  if (!g || !p) config_error("null graph or params");
  const auto t0 = std::chrono::steady_clock::now();
  HostGraph hg{g->n, static_cast<long>(g->m), g->ei, g->ej, g->w, g->degree};
  validate(hg, *p, true);
  const int R = g->grid_radius;
  if (nranks < 1 || rank < 0 || rank >= nranks) config_error("row bands: bad rank / rank count");
  if (g->grid_h / nranks < std::max(R, 1)) config_error("row bands: every band needs at least R image rows");
  auto S = std::make_unique<pfe_solver>();
  S->prm = *p;
  S->jacobi_fallback = p->preconditioner == PFE_PRECOND_IC0;
  init_common(S.get(), x, p->dim);
  S->persistent = false;  // grid-wide barriers cannot span GPUs
  S->use_graphs = false;
  S->nranks = nranks;
  S->rank = rank;
  S->comm = comm;
  S->m = g->m;
  S->global_n = g->n;
  const BandPlan bp = band_plan(g->grid_h, nranks, R, rank);
  const bool host_only = std::getenv("PFE_HOST_TOPOLOGY") && std::getenv("PFE_HOST_TOPOLOGY")[0] == '1';
  if (host_only || !setup_band_grid_device(S.get(), hg, g->grid_h, g->grid_w, R, bp))
    setup_band_grid(S.get(), hg, g->grid_h, g->grid_w, R, bp);
  int maxrows = 0;
  for (int q = 0; q < nranks; ++q) {
    const BandPlan b = band_plan(g->grid_h, nranks, R, q);
    maxrows = std::max(maxrows, b.r1 - b.r0);
  }
  S->band_maxrows = maxrows;
  S->max_own = maxrows * g->grid_w;
  const int d = S->d;
  S->qr_blocks = qr_blocks_for(S.get(), static_cast<long>(maxrows) * g->grid_w);  // equal on every band
  S->rbuf = S->mem.alloc<double>(static_cast<size_t>(S->qr_blocks) * d * d);
  S->rgather = S->mem.alloc<double>(static_cast<size_t>(nranks) * S->qr_blocks * d * d);
  S->wmat = S->mem.alloc<double>(static_cast<size_t>(d) * d);
  S->tot_local = S->mem.alloc<double>(3 * pfe_dev::kMaxD);
  S->gathered_a = S->mem.alloc<double>(static_cast<size_t>(nranks) * 3 * d);
  S->gathered_b = S->mem.alloc<double>(static_cast<size_t>(nranks) * d);
  const size_t rows = static_cast<size_t>(S->max_own) * d;
  S->ystage = S->mem.alloc<double>(rows);
  S->yall = S->mem.alloc<double>(rows * nranks);
  if (p->preconditioner == PFE_PRECOND_IC0) {
    std::vector<int> ident(static_cast<size_t>(g->n));
    std::iota(ident.begin(), ident.end(), 0);
    setup_team_ic(S.get(), hg, build_incidence(hg), ident);
  }
  S->ensure_log(64);
  CK(cudaStreamSynchronize(S->stream));
  S->setup_s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  return S.release();
}

// Band state: y0 is the GLOBAL column-major n x d embedding.
pfe_state* create_band_state(pfe_solver* S, const double* y0_global) {
  // the band's rows of every column are contiguous in the global matrix
  const long gn = S->global_n, vb = static_cast<long>(S->band_lo) * S->band_w;
  return create_state(S, y0_global + vb, gn);
}

// ------------------------------------------------------------------ team --
// The bands a host thread drives: one band per process (NCCL, one GPU each),
// every band of an image on its own GPU of this process (NCCL, one
// communicator per device from ncclCommInitAll, pfe_solve_multi_gpu), or every
// band emulated on one device (device copies, pfe_solve_banded).
struct Team {
  std::vector<pfe_state*> st;
  bool emulated = false;
  pfe_solver* S(size_t i) const { return st[i]->s; }
  size_t size() const { return st.size(); }
};

// Makes member S's device current (kernel launches need their stream's
// device); a no-op when the team lives on one device.
inline pfe_solver* on(pfe_solver* S) {
  int cur = -1;
  cudaGetDevice(&cur);
  if (cur != S->device) CK(cudaSetDevice(S->device));
  return S;
}

void team_sync(Team& t) {
  for (auto* st : t.st) CK(cudaStreamSynchronize(on(st->s)->stream));
}

// NCCL calls of every member of a multi-device team go into one group (one
// host thread issues them for all communicators).
struct NcclGroup {
  const int unwinding = std::uncaught_exceptions();
  NcclGroup() { nccl_check(nccl().GroupStart(), "ncclGroupStart"); }
  ~NcclGroup() noexcept(false) {
    const ncclResult_t r = nccl().GroupEnd();
    if (std::uncaught_exceptions() == unwinding) nccl_check(r, "ncclGroupEnd");
  }
};

// Emulated transport: a device copy ordered on the receiving band's stream
// (the solver streams are non-blocking, so a legacy-stream copy would not be
// ordered before the receiver's next kernels).  Callers team_sync() before
// (sources ready) and after (sources reusable).
void emu_copy(pfe_solver* dst_owner, double* dst, const double* src, size_t doubles) {
  if (doubles == 0) return;
  CK(cudaMemcpyAsync(dst, src, sizeof(double) * doubles, cudaMemcpyDeviceToDevice, dst_owner->stream));
}

// Per-band totals of the producer's partials, then the totals of all bands.
void team_gather_totals(Team& t, int nq, bool spmv_partials, int nb_producer_of(const pfe_solver*, bool)) {
  const int d = t.S(0)->d, P = t.S(0)->nranks;
  const size_t cnt = static_cast<size_t>(nq) * d;
  for (auto* st : t.st) {
    pfe_solver* S = on(st->s);
    S->tab->local_totals(nq, spmv_partials ? S->partials_b : S->partials, nb_producer_of(S, spmv_partials),
                         S->tot_local, S->stream);
  }
  if (t.emulated) {
    team_sync(t);
    for (size_t j = 0; j < t.size(); ++j)
      for (size_t i = 0; i < t.size(); ++i) {
        double* dst = (spmv_partials ? t.S(j)->gathered_b : t.S(j)->gathered_a) + i * cnt;
        emu_copy(t.S(j), dst, t.S(i)->tot_local, cnt);
      }
    team_sync(t);
    return;
  }
  (void)P;
  NcclGroup grp;
  for (auto* st : t.st) {
    pfe_solver* S = on(st->s);
    nccl_check(nccl().AllGather(S->tot_local, spmv_partials ? S->gathered_b : S->gathered_a, cnt, ncclDouble,
                                static_cast<ncclComm_t>(S->comm), S->stream),
               "ncclAllGather(totals)");
  }
}

// Refreshes the R halo rows of `field` (a [n_local][d] array) from the
// neighbouring bands.
template <class F>
void team_ghosts(Team& t, F&& field);

template <class F>
void team_halo(Team& t, F&& field) {
  if (t.S(0)->part == 2) return team_ghosts(t, field);
  const pfe_solver* S0 = t.S(0);
  const int d = S0->d, R = S0->band_rad, W = S0->band_w;
  const size_t blk = static_cast<size_t>(R) * W * d;  // doubles per halo block
  auto rows = [&](pfe_state* st, int local_row) { return field(st) + static_cast<size_t>(local_row) * W * d; };
  if (t.emulated) {
    team_sync(t);
    for (size_t p = 1; p < t.size(); ++p) {
      pfe_state* up = t.st[p - 1];
      pfe_state* dn = t.st[p];
      // dn's top owned rows -> up's bottom halo; up's bottom owned rows -> dn's top halo
      emu_copy(up->s, rows(up, up->s->row_hi), rows(dn, dn->s->row_lo), blk);
      emu_copy(dn->s, rows(dn, 0), rows(up, up->s->row_hi - R), blk);
    }
    team_sync(t);
    return;
  }
  NcclGroup grp;
  for (pfe_state* st : t.st) {
    pfe_solver* S = on(st->s);
    auto comm = static_cast<ncclComm_t>(S->comm);
    if (S->rank > 0) {
      nccl_check(nccl().Send(rows(st, S->row_lo), blk, ncclDouble, S->rank - 1, comm, S->stream), "ncclSend");
      nccl_check(nccl().Recv(rows(st, 0), blk, ncclDouble, S->rank - 1, comm, S->stream), "ncclRecv");
    }
    if (S->rank < S->nranks - 1) {
      nccl_check(nccl().Send(rows(st, S->row_hi - R), blk, ncclDouble, S->rank + 1, comm, S->stream), "ncclSend");
      nccl_check(nccl().Recv(rows(st, S->row_hi), blk, ncclDouble, S->rank + 1, comm, S->stream), "ncclRecv");
    }
  }
}

int nb_producer(const pfe_solver* S, bool spmv) {
  int nb_init = 0, nb_spmv = 0, nb_update = 0;
  S->tab->pcg_grids(S->topo, S->lv(), &nb_init, &nb_spmv, &nb_update);
  return spmv ? nb_spmv : nb_update;
}
int nb_producer_init(const pfe_solver* S, bool) {
  int nb_init = 0, nb_spmv = 0, nb_update = 0;
  S->tab->pcg_grids(S->topo, S->lv(), &nb_init, &nb_spmv, &nb_update);
  return nb_init;
}

// First row of a member's owned block in the team's global row order.
long team_global_first(const pfe_solver* S) {
  return S->part == 2 ? static_cast<long>(S->range_start[S->rank]) : static_cast<long>(S->band_r0) * S->band_w;
}

// Owned rows of `field` from every member -> every member's S->rfull, a
// [global n][d] array in the team's global row order (IC(0) residual).
template <class F>
void team_gather_rows(Team& t, F&& field) {
  const pfe_solver* S0 = t.S(0);
  const int d = S0->d, P = S0->nranks;
  if (t.emulated) {
    team_sync(t);
    for (size_t j = 0; j < t.size(); ++j)
      for (size_t i = 0; i < t.size(); ++i) {
        const pfe_solver* Si = t.S(i);
        emu_copy(t.S(j), t.S(j)->rfull + static_cast<size_t>(team_global_first(Si)) * d,
                 field(t.st[i]) + Si->own_vb * d, static_cast<size_t>(Si->own_cnt) * d);
      }
    team_sync(t);
    return;
  }
  const size_t slot = static_cast<size_t>(S0->max_own) * d;
  {
    NcclGroup grp;
    for (pfe_state* st : t.st) {
      pfe_solver* S = on(st->s);
      CK(cudaMemcpyAsync(S->ystage, field(st) + S->own_vb * d, sizeof(double) * S->own_cnt * d,
                         cudaMemcpyDeviceToDevice, S->stream));
      nccl_check(nccl().AllGather(S->ystage, S->yall, slot, ncclDouble, static_cast<ncclComm_t>(S->comm), S->stream),
                 "ncclAllGather(r)");
    }
  }
  for (pfe_state* st : t.st) {
    pfe_solver* S = on(st->s);
    for (int q = 0; q < P; ++q) {
      long first, cnt;
      if (S->part == 2) {
        first = S->range_start[q];
        cnt = S->range_start[q + 1] - S->range_start[q];
      } else {
        const BandPlan bp = band_plan(S->band_h, P, S->band_rad, q);
        first = static_cast<long>(bp.r0) * S->band_w;
        cnt = static_cast<long>(bp.r1 - bp.r0) * S->band_w;
      }
      CK(cudaMemcpyAsync(S->rfull + static_cast<size_t>(first) * d, S->yall + q * slot, sizeof(double) * cnt * d,
                         cudaMemcpyDeviceToDevice, S->stream));
    }
  }
}

// One PCG solve of every band (pcg.cpp:40-114 for all d columns).
//
// The host does not read the device control block after every PCG
// iteration.  It issues iterations in chunks and reads the control block
// (one stream synchronisation) only at the end of a chunk: the first chunk
// is as long as the previous solve (warm-started solves inside the
// split-Bregman loop take about the same number of iterations), later ones
// are short.  Iterations issued after every column stopped are no-ops: the
// SpMV prologue finds no active column, clears any_active, and the update
// and direction kernels return at once; their halo exchanges and gathers
// move unchanged values.  So the chunking changes no result, and a typical
// solve costs one host round trip instead of one per PCG iteration.
void team_pcg(Team& t, const std::vector<const double*>& rhs) {
  NvtxRange nv("pfe band pcg");
  const size_t B = t.size();
  std::vector<PcgArgs> a(B);
  for (size_t i = 0; i < B; ++i) {
    pfe_solver* S = on(t.S(i));
    a[i] = pcg_args(t.st[i], rhs[i]);
    a[i].rd_a = S->gathered_a;
    a[i].rd_b = S->gathered_b;
    a[i].rank_major = 1;
    a[i].totals = 0;  // per-band totals are gathered across ranks instead
    a[i].nb_init = a[i].nb_update = a[i].nb_spmv = S->nranks;
  }
  const int maxit = t.S(0)->prm.pcg_max_iter;
  const bool ranges = t.S(0)->part == 2;
  const bool ic = t.S(0)->ic_team;
  // IC(0): z = M^-1 r on the gathered global residual, on every member; the
  // r.z total the consumers read (slot 2 after init, slot 1 after an update)
  // becomes the preconditioned one: member 0's entry holds the global total
  // (k_ic_dot over the global vectors, the single-GPU value), the others 0.
  std::vector<pfe_dev::PcgArgs> az(a);  // SpMV arguments when z replaces D^-1 r
  std::vector<TopoDesc> tz(B);
  for (size_t i = 0; i < B && ic; ++i) {
    pfe_solver* S = t.S(i);
    const long g0 = team_global_first(S) - S->own_vb;  // global row of local row 0 (row bands)
    tz[i] = S->topo;
    if (ranges) {
      a[i].zbuf = S->zbuf + static_cast<size_t>(team_global_first(S)) * S->d;  // owned rows are contiguous
    } else {
      az[i].r = S->zbuf + static_cast<size_t>(g0) * S->d;  // band rows incl. halo are contiguous global rows
      tz[i].g1.invd = S->ones;
      tz[i].g2.invd = S->ones;
    }
  }
  using DSeq = std::make_integer_sequence<int, pfe_dev::kMaxD>;
  auto ic_z = [&](int slot, bool to_p0) {
    if (!ic) return;
    team_gather_rows(t, [](pfe_state* st) { return st->r; });
    for (size_t i = 0; i < B; ++i) {
      pfe_solver* S = on(t.S(i));
      const int d = S->d, P = S->nranks;
      const int gn = static_cast<int>(S->global_n);
      ic_apply_dispatch(d, DSeq{}, S->icd, S->rfull, S->zbuf, S->stream);
      const int grid = std::min(S->max_grid, std::max(1, (gn + 255) / 256));
      // (its own partials: iterations issued after every column stopped re-read
      // the update's block partials, which must stay as that update left them)
      ic_dot_dispatch(d, DSeq{}, gn, S->rfull, S->zbuf, S->ic_part, S->ctl, S->gathered_a + slot * d, grid, S->stream);
      for (int q = 1; q < P; ++q)
        CK(cudaMemsetAsync(S->gathered_a + (static_cast<size_t>(q) * 3 + slot) * d, 0, sizeof(double) * d, S->stream));
      if (to_p0)  // p = z for the first iteration: owned rows (halo / ghost rows are exchanged next)
        CK(cudaMemcpyAsync(t.st[i]->pb[0] + S->own_vb * d,
                           S->zbuf + static_cast<size_t>(team_global_first(S)) * d,
                           sizeof(double) * S->own_cnt * d, cudaMemcpyDeviceToDevice, S->stream));
      CK(cudaGetLastError());
    }
  };
  for (size_t i = 0; i < B; ++i) on(t.S(i))->tab->pcg_init(t.S(i)->topo, a[i], t.S(i)->lv());
  team_gather_totals(t, 3, false, nb_producer_init);
  ic_z(2, true);
  team_halo(t, [](pfe_state* st) { return st->pb[0]; });
  auto spmv = [&](int k) {
    for (size_t i = 0; i < B; ++i) {
      a[i].phase = az[i].phase = pfe_dev::pcg_phase(k);
      const bool zdir = ic && !ranges;
      on(t.S(i))->tab->pcg_spmv(zdir ? tz[i] : t.S(i)->topo, zdir ? az[i] : a[i], t.S(i)->lv());
    }
    team_gather_totals(t, 1, true, nb_producer);
  };
  // one PCG iteration after the SpMV of iteration k: update k, SpMV k + 1
  auto iteration = [&](int k) {
    // (row bands need no halo exchange of p here: the SpMV stored the halo
    // rows of p' it formed from exchanged r, k_grid_pcg_spmv)
    for (size_t i = 0; i < B; ++i) {
      a[i].phase = pfe_dev::pcg_phase(k);
      on(t.S(i))->tab->pcg_update(t.S(i)->topo, a[i], t.S(i)->lv());
    }
    team_gather_totals(t, 3, false, nb_producer);
    ic_z(1, false);
    const int kn = k + 1;
    if (ranges) {
      // vertex ranges: p' = D^-1 r + beta p on owned rows, then its ghosts
      for (size_t i = 0; i < B; ++i) {
        a[i].phase = pfe_dev::pcg_phase(kn);
        a[i].skip_pdir = 1;
        on(t.S(i))->tab->pcg_pdir(t.S(i)->topo, a[i], t.S(i)->lv());
      }
      team_halo(t, [kn](pfe_state* st) { return (kn & 1) ? st->pb[0] : st->pb[1]; });
    } else if (!ic) {  // with IC(0) every band already holds z on its halo rows
      team_halo(t, [](pfe_state* st) { return st->r; });
    }
    spmv(kn);
  };
  pfe_solver* S0 = t.S(0);
  int k = 1;
  spmv(1);
  int chunk = std::max(1, S0->band_chunk_hint);
  for (;;) {
    for (int c = 0; c < chunk && k <= maxit; ++c) iteration(k++);
    on(S0)->read_ctl();  // every band took the same decision
    if (!S0->h_ctl->any_active || k > maxit) break;
    chunk = 2;
  }
  // the next solve's first chunk: this solve's iteration count
  const int done = S0->h_ctl->iter;
  for (size_t i = 0; i < B; ++i) t.S(i)->band_chunk_hint = std::max(1, done);
  for (size_t i = 0; i < B; ++i) {
    pfe_state* st = t.st[i];
    pfe_solver* S = on(st->s);
    const long vb = S->own_vb * S->d;
    const int cnt = S->own_cnt;
    S->tab->pcg_finalize(cnt, st->y + vb, st->y2 + vb, S->ctl, {S->grid_for(static_cast<long>(cnt) * S->d), S->stream, S->sm});
    ++S->inner_launched;
    std::swap(st->y, st->y2);
  }
  team_halo(t, [](pfe_state* st) { return st->y; });
}

// PfeSolver::split_bregman (solver.cpp:73-108) over every band.
void team_split_bregman(Team& t, int max_iter) {
  NvtxRange nv("pfe band split_bregman");
  const size_t B = t.size();
  std::vector<const double*> rhs(B);
  for (size_t i = 0; i < B; ++i) {
    pfe_state* st = t.st[i];
    pfe_solver* S = on(st->s);
    const long vb = S->own_vb;
    const int cnt = S->own_cnt;
    if (!st->rq_valid) {
      S->tab->rhs_quad(cnt, S->sqd + vb, st->p + vb * S->d, st->breg + vb * S->d, st->rq + vb * S->d,
                       0.5 * S->prm.r, {S->grid_for(static_cast<long>(cnt) * S->d), S->stream, S->sm});
      st->rq_valid = true;
    }
    rhs[i] = st->rq;
    if (!st->inner_zero) {
      S->tab->rhs_from_state(S->topo, st->es, st->eb[st->eb_cur], st->rq, st->r, 0.5 * S->prm.lambda, S->lv());
      rhs[i] = st->r;
    }
  }
  for (int it = 0; it < max_iter; ++it) {
    const bool last = it == max_iter - 1;
    team_pcg(t, rhs);
    for (size_t i = 0; i < B; ++i) {
      pfe_state* st = t.st[i];
      pfe_solver* S = on(st->s);
      SbArgs sa{};
      sa.y = st->y;
      sa.b_old = st->inner_zero ? nullptr : st->eb[st->eb_cur];
      sa.b_new = st->eb[st->eb_cur ^ 1];
      sa.s_out = last ? st->es : nullptr;
      sa.rq = st->rq;
      sa.rhs = last ? nullptr : st->r;
      sa.hl = 0.5 * S->prm.lambda;
      sa.gamma = 1.0 / S->prm.lambda;
      sa.ctl = S->ctl;
      sa.prefetch = sb_prefetch();
      S->tab->sb_pass(S->topo, sa, S->lv());
      st->eb_cur ^= 1;
      st->inner_zero = false;
      rhs[i] = st->r;
    }
  }
}

// Projection (solver.cpp:116-118): TSQR factors of every band folded in rank
// order on every band, so all bands apply the same W.
void team_project(Team& t) {
  NvtxRange nv("pfe band projection");
  const size_t B = t.size();
  const int d = t.S(0)->d;
  const size_t fac = static_cast<size_t>(t.S(0)->qr_blocks) * d * d;
  for (size_t i = 0; i < B; ++i) {
    pfe_state* st = t.st[i];
    pfe_solver* S = on(st->s);
    const long vb = S->own_vb;
    const int cnt = S->own_cnt;
    S->tab->tsqr_local(cnt, st->y + vb * d, S->sqd + vb, st->breg + vb * d, S->rbuf, {S->qr_blocks, S->stream, S->sm});
  }
  if (t.emulated) {
    team_sync(t);
    for (size_t j = 0; j < B; ++j)
      for (size_t i = 0; i < B; ++i)
        emu_copy(t.S(j), t.S(j)->rgather + i * fac, t.S(i)->rbuf, fac);
    team_sync(t);
  } else {
    NcclGroup grp;
    for (size_t i = 0; i < B; ++i) {
      pfe_solver* S = on(t.S(i));
      nccl_check(nccl().AllGather(S->rbuf, S->rgather, fac, ncclDouble, static_cast<ncclComm_t>(S->comm), S->stream),
                 "ncclAllGather(R factors)");
    }
  }
  for (size_t i = 0; i < B; ++i) {
    pfe_state* st = t.st[i];
    pfe_solver* S = on(st->s);
    const long vb = S->own_vb;
    const int cnt = S->own_cnt;
    S->tab->tsqr_final(S->nranks * S->qr_blocks, S->rgather, S->wmat, S->ctl, {1, S->stream, S->sm});
    S->tab->project_apply(cnt, st->y + vb * d, S->sqd + vb, st->breg + vb * d, S->wmat, st->p + vb * d,
                          st->rq + vb * d, 0.5 * S->prm.r, {S->grid_for(cnt), S->stream, S->sm});
    st->rq_valid = true;
  }
}

void team_check(Team& t) {
  for (auto* st : t.st) check_flags(on(st->s));
}

// PfeSolver::run_soc (solver.cpp:110-126) over every band (fixed counts;
// the relative-change test is not supported across bands).
void team_run_soc(Team& t, int soc_max, int sb_max) {
  for (auto* st : t.st) st->s->ensure_log(static_cast<long>(soc_max) * sb_max);
  for (int k = 0; k < soc_max; ++k) {
    for (auto* st : t.st) st->inner_zero = true;
    team_split_bregman(t, sb_max);
    team_project(t);
    team_check(t);
  }
}

// Global column-major Y from the owned rows of every band / range.
void team_gather_y(Team& t, double* out) {
  NvtxRange nv("pfe band gather Y");
  const pfe_solver* S0 = t.S(0);
  const int d = S0->d, P = S0->nranks;
  const long gn = S0->global_n;
  const size_t slot = static_cast<size_t>(S0->max_own) * d;
  if (!t.emulated && S0->part == 1 && static_cast<int>(t.size()) == P) {
    // every band lives in this process: each device writes its owned rows
    // straight into the caller's column-major matrix (its rows of a column
    // are contiguous there), no gather through a host copy of all of Y
    for (pfe_state* st : t.st) {
      pfe_solver* S = on(st->s);
      const long cnt = S->own_cnt, v0 = static_cast<long>(S->band_r0) * S->band_w;
      k_rows_to_colmajor<<<S->grid_for(cnt * d), pfe_dev::kBlock, 0, S->stream>>>(cnt, d, st->y + S->own_vb * d,
                                                                                S->ystage, nullptr);
      CK(cudaGetLastError());
      for (int j = 0; j < d; ++j)
        copy_d2h(out + v0 + j * gn, S->ystage + static_cast<size_t>(j) * cnt, sizeof(double) * cnt, S->stream);
    }
    return;
  }
  std::vector<double> all;
  if (t.emulated) {
    all.assign(slot * P, 0.0);
    for (size_t i = 0; i < t.size(); ++i) {
      const pfe_solver* S = t.S(i);
      stream_copy(all.data() + i * slot, t.st[i]->y + S->own_vb * d, sizeof(double) * S->own_cnt * d,
                  cudaMemcpyDeviceToHost, S->stream);
    }
  } else {
    {
      NcclGroup grp;
      for (pfe_state* st : t.st) {
        pfe_solver* S = on(st->s);
        CK(cudaMemcpyAsync(S->ystage, st->y + S->own_vb * d, sizeof(double) * S->own_cnt * d,
                           cudaMemcpyDeviceToDevice, S->stream));
        nccl_check(nccl().AllGather(S->ystage, S->yall, slot, ncclDouble, static_cast<ncclComm_t>(S->comm), S->stream),
                   "ncclAllGather(Y)");
      }
    }
    pfe_solver* S = on(t.S(0));
    all.resize(slot * P);
    CK(cudaMemcpyAsync(all.data(), S->yall, sizeof(double) * all.size(), cudaMemcpyDeviceToHost, S->stream));
    CK(cudaStreamSynchronize(S->stream));
    for (size_t i = 1; i < t.size(); ++i) CK(cudaStreamSynchronize(on(t.S(i))->stream));
  }
  for (int p = 0; p < P; ++p) {
    long cnt, v0 = 0;
    if (S0->part == 2) {
      cnt = S0->range_start[p + 1] - S0->range_start[p];
    } else {
      const BandPlan bp = band_plan(S0->band_h, P, S0->band_rad, p);
      v0 = static_cast<long>(bp.r0) * S0->band_w;
      cnt = static_cast<long>(bp.r1 - bp.r0) * S0->band_w;
    }
    parallel_for(cnt, [&](long ib, long ie) {
      for (long i = ib; i < ie; ++i) {
        const long v = S0->part == 2 ? S0->range_vertex[S0->range_start[p] + i] : v0 + i;
        for (int j = 0; j < d; ++j) out[v + j * gn] = all[p * slot + static_cast<size_t>(i) * d + j];
      }
    }, 1L << 14);
  }
}

// Device time of a band call (CUDA events on the band's stream).
template <class F>
void band_timed(pfe_solver* S, F&& f) {
  CK(cudaEventRecord(S->ev0, S->stream));
  f();
  CK(cudaEventRecord(S->ev1, S->stream));
  CK(cudaEventSynchronize(S->ev1));
  float ms = 0.f;
  CK(cudaEventElapsedTime(&ms, S->ev0, S->ev1));
  S->last_ms = ms;
}

// ------------------------------------------------------ vertex ranges ----
// General graphs (k-NN) over several GPUs.  The vertices,
// in the BFS storage order of the whole graph (bfs_storage_order), are cut
// into contiguous ranges, one per rank.  A rank stores its owned vertices
// (local rows [0, own)) and then its ghosts -- neighbours owned elsewhere --
// grouped by owner and in storage order.  Kernels process owned rows only
// (Csr::vb / ve); ghost rows of p' (after the direction pass) and of Y (after
// the result selection) are refreshed from their owners.  Every edge incident
// to an owned vertex is stored locally; an edge crossing two ranges is a
// replica on both, updated identically (k_sb_pass writes the edges of ghost
// owners too).  Rows of A and incidence lists keep the reference's term
// order, so per-vertex arithmetic is that of the single-GPU solver.
// Host-only statistics of the vertex-range partition create_range_solver
// builds (same BFS storage order, same contiguous ranges): per rank the
// owned vertices, the ghost rows it receives per exchange and the rows it
// sends (with multiplicity per peer).
void range_partition_stats(const pfe_graph* g, int nranks, int64_t* owned, int64_t* ghosts, int64_t* sends) {
  if (!g || g->n < 1 || g->m < 0) config_error("vertex ranges: bad graph");
  if (nranks < 1 || g->n < nranks) config_error("vertex ranges: bad rank count");
  HostGraph hg{g->n, static_cast<long>(g->m), g->ei, g->ej, g->w, g->degree};
  const int n = g->n, P = nranks;
  const Incidence inc = build_incidence(hg);
  const std::vector<int> pos = bfs_storage_order(n, inc.iptr, inc.inbr.data());
  std::vector<int> vat(n);
  for (int v = 0; v < n; ++v) vat[pos[v]] = v;
  std::vector<int> start(P + 1);
  for (int q = 0; q <= P; ++q) start[q] = static_cast<int>(static_cast<long>(n) * q / P);
  for (int r = 0; r < P; ++r) {
    const int s0 = start[r], s1 = start[r + 1];
    std::vector<int> gh;
    std::vector<std::vector<int>> sendl(P);
    for (int l = 0; l < s1 - s0; ++l) {
      const int v = vat[s0 + l];
      for (int k = inc.iptr[v]; k < inc.iptr[v + 1]; ++k) {
        const int pu = pos[inc.inbr[k]];
        if (pu >= s0 && pu < s1) continue;
        gh.push_back(pu);
        const int q = static_cast<int>(std::upper_bound(start.begin(), start.end(), pu) - start.begin()) - 1;
        sendl[q].push_back(l);
      }
    }
    std::sort(gh.begin(), gh.end());
    gh.erase(std::unique(gh.begin(), gh.end()), gh.end());
    long snd = 0;
    for (auto& sl : sendl) {
      std::sort(sl.begin(), sl.end());
      snd += std::unique(sl.begin(), sl.end()) - sl.begin();
    }
    if (owned) owned[r] = s1 - s0;
    if (ghosts) ghosts[r] = static_cast<int64_t>(gh.size());
    if (sends) sends[r] = snd;
  }
}

pfe_solver* create_range_solver(const pfe_graph* g, const pfe_params* p, const pfe_exec* x, int nranks, int rank,
                                void* comm) {
  if (!g || !p) config_error("null graph or params");
  const auto t0 = std::chrono::steady_clock::now();
  HostGraph hg{g->n, static_cast<long>(g->m), g->ei, g->ej, g->w, g->degree};
  validate(hg, *p, true);
  if (nranks < 1 || rank < 0 || rank >= nranks) config_error("vertex ranges: bad rank / rank count");
  if (g->n < nranks) config_error("vertex ranges: fewer vertices than ranks");
  if (g->m > 0x3fffffffL) config_error("graph too large for 32-bit edge indices");
  auto S = std::make_unique<pfe_solver>();
  S->prm = *p;
  S->jacobi_fallback = p->preconditioner == PFE_PRECOND_IC0;
  init_common(S.get(), x, p->dim);
  S->persistent = false;
  S->use_graphs = false;
  S->nranks = nranks;
  S->rank = rank;
  S->comm = comm;
  S->m = g->m;
  S->global_n = g->n;
  S->part = 2;
  const int n = g->n, P = nranks, d = S->d;
  const double hl = 0.5 * S->prm.lambda, dterm = 0.5 * S->prm.r;
  const Incidence inc = build_incidence(hg);
  const std::vector<int> pos = bfs_storage_order(n, inc.iptr, inc.inbr.data());
  std::vector<int> vat(n);
  for (int v = 0; v < n; ++v) vat[pos[v]] = v;
  S->range_vertex = vat;
  S->range_start.resize(P + 1);
  for (int q = 0; q <= P; ++q) S->range_start[q] = static_cast<int>(static_cast<long>(n) * q / P);
  const int s0 = S->range_start[rank], s1 = S->range_start[rank + 1], own = s1 - s0;
  auto owner = [&](int ps) {
    return static_cast<int>(std::upper_bound(S->range_start.begin(), S->range_start.end(), ps) -
                            S->range_start.begin()) - 1;
  };
  std::vector<int> ghost;  // storage positions of the ghosts, sorted (grouped by owner)
  std::vector<std::vector<int>> sendl(P);
  for (int l = 0; l < own; ++l) {
    const int v = vat[s0 + l];
    for (int k = inc.iptr[v]; k < inc.iptr[v + 1]; ++k) {
      const int pu = pos[inc.inbr[k]];
      if (pu >= s0 && pu < s1) continue;
      ghost.push_back(pu);
      sendl[owner(pu)].push_back(l);
    }
  }
  std::sort(ghost.begin(), ghost.end());
  ghost.erase(std::unique(ghost.begin(), ghost.end()), ghost.end());
  const int nloc = own + static_cast<int>(ghost.size());
  auto lid = [&](int pu) {
    if (pu >= s0 && pu < s1) return pu - s0;
    return own + static_cast<int>(std::lower_bound(ghost.begin(), ghost.end(), pu) - ghost.begin());
  };
  S->local_vertex.resize(nloc);
  for (int l = 0; l < nloc; ++l) S->local_vertex[l] = vat[l < own ? s0 + l : ghost[l - own]];
  // diag(A) from the global incidence (edge order, (r/2) d_v last)
  std::vector<double> diag(nloc), invd(nloc), deg(nloc), sqd(nloc);
  parallel_for(nloc, [&](long lb, long le) {
    for (long l = lb; l < le; ++l) {
      const int v = S->local_vertex[l];
      double acc = 0.0;
      for (int k = inc.iptr[v]; k < inc.iptr[v + 1]; ++k) acc += (hl * inc.iw[k]) * inc.iw[k];
      diag[l] = acc + dterm * g->degree[v];
      invd[l] = S->prm.preconditioner == PFE_PRECOND_NONE ? 1.0 : (diag[l] > 0.0 ? 1.0 / diag[l] : 1.0);
      deg[l] = g->degree[v];
      sqd[l] = std::sqrt(g->degree[v]);
    }
  }, 4096);
  // A rows of the owned vertices in the reference's column order: merged in
  // parallel into an upper-bound layout (degree + 1 entries per row), then
  // compacted (the single-GPU builder's scheme)
  std::vector<long> ub(static_cast<size_t>(own) + 1, 0);
  for (int l = 0; l < own; ++l) {
    const int v = S->local_vertex[l];
    ub[l + 1] = ub[l] + (inc.iptr[v + 1] - inc.iptr[v]) + 1;
  }
  uvec<int> tcol(static_cast<size_t>(ub[own])), tlen(static_cast<size_t>(own));
  uvec<double> tval(static_cast<size_t>(ub[own]));
  parallel_for(own, [&](long lb, long le) {
    std::vector<std::pair<int, double>> row;
    for (long l = lb; l < le; ++l) {
      const int v = S->local_vertex[l];
      row.clear();
      for (int k = inc.iptr[v]; k < inc.iptr[v + 1]; ++k) row.emplace_back(inc.inbr[k], -((hl * inc.iw[k]) * inc.iw[k]));
      row.emplace_back(v, diag[l]);
      std::stable_sort(row.begin(), row.end(), [](const auto& a, const auto& b) { return a.first < b.first; });
      long at = ub[l];
      for (size_t t = 0; t < row.size();) {
        const int col = row[t].first;
        double sum = 0.0;
        if (col == v) {
          sum = row[t].second;
          ++t;
        } else {
          for (; t < row.size() && row[t].first == col; ++t) sum += row[t].second;
        }
        if (sum != 0.0) {
          tcol[static_cast<size_t>(at)] = lid(pos[col]);
          tval[static_cast<size_t>(at)] = sum;
          ++at;
        }
      }
      tlen[l] = static_cast<int>(at - ub[l]);
    }
  }, 2048);
  std::vector<int> aptr(static_cast<size_t>(own) + 1, 0);
  for (int l = 0; l < own; ++l) aptr[l + 1] = aptr[l] + tlen[l];
  uvec<int> acol(static_cast<size_t>(aptr[own]));
  uvec<double> aval(static_cast<size_t>(aptr[own]));
  parallel_for(own, [&](long lb, long le) {
    for (long l = lb; l < le; ++l) {
      std::copy(tcol.begin() + ub[l], tcol.begin() + ub[l] + tlen[l], acol.begin() + aptr[l]);
      std::copy(tval.begin() + ub[l], tval.begin() + ub[l] + tlen[l], aval.begin() + aptr[l]);
    }
  }, 4096);
  // local edge rows (first visit order: vertex by vertex, each in edge order)
  // and incidence lists of the owned vertices.  An edge is first visited at
  // its owned endpoint with the smaller local index, so every vertex can
  // count the edges it visits first; a prefix sum then numbers them.
  auto local_of = [&](int u) {  // local index if owned, else -1
    const int pu = pos[u];
    return pu >= s0 && pu < s1 ? pu - s0 : -1;
  };
  std::vector<int> first(static_cast<size_t>(own) + 1, 0), iptr2(static_cast<size_t>(own) + 1, 0);
  parallel_for(own, [&](long lb, long le) {
    for (long l = lb; l < le; ++l) {
      const int v = S->local_vertex[l];
      int c = 0;
      for (int k = inc.iptr[v]; k < inc.iptr[v + 1]; ++k) {
        const int lu = local_of(inc.inbr[k]);
        c += (lu < 0 || lu > l) ? 1 : 0;
      }
      first[l + 1] = c;
      iptr2[l + 1] = inc.iptr[v + 1] - inc.iptr[v];
    }
  }, 4096);
  for (int l = 0; l < own; ++l) {
    first[l + 1] += first[l];
    iptr2[l + 1] += iptr2[l];
  }
  const int ne = first[own];
  uvec<int> erow(static_cast<size_t>(g->m));  // written for every edge incident to an owned vertex
  parallel_for(own, [&](long lb, long le) {
    for (long l = lb; l < le; ++l) {
      const int v = S->local_vertex[l];
      int next = first[l];
      for (int k = inc.iptr[v]; k < inc.iptr[v + 1]; ++k) {
        const int lu = local_of(inc.inbr[k]);
        if (lu < 0 || lu > l) erow[inc.ieid[k]] = next++;
      }
    }
  }, 4096);
  uvec<int> inbr2(static_cast<size_t>(iptr2[own])), ieid2(static_cast<size_t>(iptr2[own]));
  uvec<double> iw2(static_cast<size_t>(iptr2[own]));
  parallel_for(own, [&](long lb, long le) {
    for (long l = lb; l < le; ++l) {
      const int v = S->local_vertex[l];
      int at = iptr2[l];
      for (int k = inc.iptr[v]; k < inc.iptr[v + 1]; ++k, ++at) {
        const int e = inc.ieid[k], u = inc.inbr[k];
        inbr2[at] = lid(pos[u]);
        ieid2[at] = (erow[e] << 1) | (u > v ? 1 : 0);
        iw2[at] = inc.iw[k];
      }
    }
  }, 4096);
  cudaStream_t st = S->stream;
  S->n = nloc;
  S->deg = S->mem.upload(deg, st);
  S->sqd = S->mem.upload(sqd, st);
  S->diag = S->mem.upload(diag, st);
  S->invd = S->mem.upload(invd, st);
  pfe_dev::Csr c{};
  c.n = nloc;
  c.vb = 0;
  c.ve = own;
  c.aptr = S->mem.upload(aptr, st);
  c.acol = S->mem.upload(acol, st);
  c.aval = S->mem.upload(aval, st);
  c.iptr = S->mem.upload(iptr2, st);
  c.inbr = S->mem.upload(inbr2, st);
  c.ieid = S->mem.upload(ieid2, st);
  c.iw = S->mem.upload(iw2, st);
  c.invd = S->invd;
  S->topo.kind = pfe_host::kTopoCsr;
  S->topo.csr = c;
  S->edge_rows = std::max(ne, 1);
  S->own_vb = 0;
  S->own_cnt = own;
  for (int q = 0; q < P; ++q) S->max_own = std::max(S->max_own, S->range_start[q + 1] - S->range_start[q]);
  // peers: ghost blocks (contiguous, by owner) and send lists (same order)
  long send_total = 0;
  for (int q = 0; q < P; ++q) {
    if (q == rank) continue;
    auto& sl = sendl[q];
    std::sort(sl.begin(), sl.end());
    sl.erase(std::unique(sl.begin(), sl.end()), sl.end());
    const int r_lo = static_cast<int>(std::lower_bound(ghost.begin(), ghost.end(), S->range_start[q]) - ghost.begin());
    const int r_hi = static_cast<int>(std::lower_bound(ghost.begin(), ghost.end(), S->range_start[q + 1]) - ghost.begin());
    if (sl.empty() && r_hi == r_lo) continue;
    pfe_solver::Peer pr{};
    pr.rank = q;
    pr.send_cnt = static_cast<int>(sl.size());
    pr.send_rows = sl.empty() ? nullptr : S->mem.upload(sl, st);
    pr.send_off = send_total;
    pr.recv_off = own + r_lo;
    pr.recv_cnt = r_hi - r_lo;
    send_total += pr.send_cnt;
    S->peers.push_back(pr);
  }
  S->sendbuf = S->mem.alloc<double>(static_cast<size_t>(std::max<long>(send_total, 1)) * d);
  S->qr_blocks = qr_blocks_for(S.get(), S->max_own);  // equal on every rank
  S->rbuf = S->mem.alloc<double>(static_cast<size_t>(S->qr_blocks) * d * d);
  S->rgather = S->mem.alloc<double>(static_cast<size_t>(P) * S->qr_blocks * d * d);
  S->wmat = S->mem.alloc<double>(static_cast<size_t>(d) * d);
  S->tot_local = S->mem.alloc<double>(3 * pfe_dev::kMaxD);
  S->gathered_a = S->mem.alloc<double>(static_cast<size_t>(P) * 3 * d);
  S->gathered_b = S->mem.alloc<double>(static_cast<size_t>(P) * d);
  S->ystage = S->mem.alloc<double>(static_cast<size_t>(S->max_own) * d);
  S->yall = S->mem.alloc<double>(static_cast<size_t>(S->max_own) * d * P);
  if (p->preconditioner == PFE_PRECOND_IC0) setup_team_ic(S.get(), hg, inc, pos);
  S->ensure_log(64);
  CK(cudaStreamSynchronize(S->stream));
  S->setup_s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  return S.release();
}

// Range state: y0 is the GLOBAL column-major n x d embedding.
pfe_state* create_range_state(pfe_solver* S, const double* y0_global) {
  const long gn = S->global_n;
  std::vector<double> loc(static_cast<size_t>(S->n) * S->d);
  for (int j = 0; j < S->d; ++j)
    for (int l = 0; l < S->n; ++l) loc[static_cast<size_t>(j) * S->n + l] = y0_global[S->local_vertex[l] + j * gn];
  return create_state(S, loc.data());
}

// Ghost rows of `field` ([n_local][d]) from their owners.
template <class F>
void team_ghosts(Team& t, F&& field) {
  const int d = t.S(0)->d;
  for (auto* st : t.st) {
    pfe_solver* S = on(st->s);
    for (const auto& pr : S->peers)
      S->tab->pack_rows(field(st), pr.send_rows, pr.send_cnt, S->sendbuf + pr.send_off * d, S->stream);
  }
  if (t.emulated) {
    team_sync(t);
    for (size_t i = 0; i < t.size(); ++i) {
      const pfe_solver* Si = t.S(i);
      for (const auto& pr : Si->peers) {
        pfe_state* dst = t.st[pr.rank];
        for (const auto& back : dst->s->peers) {
          if (back.rank != Si->rank) continue;
          if (back.recv_cnt != pr.send_cnt) throw Error(PFE_CUDA_ERROR, "vertex ranges: inconsistent ghost lists");
          emu_copy(dst->s, field(dst) + static_cast<size_t>(back.recv_off) * d, Si->sendbuf + pr.send_off * d,
                   static_cast<size_t>(pr.send_cnt) * d);
        }
      }
    }
    team_sync(t);
    return;
  }
  NcclGroup grp;
  for (pfe_state* st : t.st) {
    pfe_solver* S = on(st->s);
    auto comm = static_cast<ncclComm_t>(S->comm);
    for (const auto& pr : S->peers) {
      if (pr.send_cnt > 0)
        nccl_check(nccl().Send(S->sendbuf + pr.send_off * d, static_cast<size_t>(pr.send_cnt) * d, ncclDouble,
                               pr.rank, comm, S->stream),
                   "ncclSend");
      if (pr.recv_cnt > 0)
        nccl_check(nccl().Recv(field(st) + static_cast<size_t>(pr.recv_off) * d,
                               static_cast<size_t>(pr.recv_cnt) * d, ncclDouble, pr.rank, comm, S->stream),
                   "ncclRecv");
    }
  }
}
