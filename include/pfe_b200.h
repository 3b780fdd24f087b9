/*
 * pfe_b200.h — C ABI of the B200-native piecewise-flat-embedding solver.
 *
 * Drop-in boundary for the reference's solver entry points in
 * /root/reference/proj/core (namespace pfe).  Each function below names the
 * reference interface it replaces.  Plain pointers and sizes only; no C++ or
 * torch types cross this boundary.
 *
 * Conventions
 *   - Host matrices are column-major n x d (the reference's Eigen::MatrixXd,
 *     solver.hpp:14).  Edge-indexed matrices (split_b, split_s) are |E| x d in
 *     the caller's edge order (difference_matrix row order, graph.cpp:161-170).
 *   - Status codes mirror the reference CLI's exception mapping
 *     (proj/tools/main.cpp:431-446): 0 ok, 1 IoError, 2 NumericalError,
 *     3 ConfigError; 4 = CUDA/driver failure.  pfe_last_error() returns the
 *     message of the last failure on the calling thread.
 *   - There is no CPU fallback: without a usable sm_100 device every entry
 *     point that computes returns 3 with a message.
 *   - A solver/state handle may be driven by one host thread at a time
 *     (solver.hpp:51-83 is const and state is caller-owned).
 */
#ifndef PFE_B200_H
#define PFE_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PFE_OK 0
#define PFE_IO_ERROR 1
#define PFE_NUMERICAL_ERROR 2
#define PFE_CONFIG_ERROR 3
#define PFE_CUDA_ERROR 4

/* Preconditioner ids (pcg.hpp:13).  Ic0 (the reference default) on a
 * single-GPU solver: the reference's IC(0) factor (sparse.cpp:124-203, host
 * set-up) applied by level-scheduled device triangular solves, host-driven
 * PCG loop on the general-graph kernels.  A factor that breaks down after
 * every shift runs Jacobi and reports jacobi_fallback = 1, as the reference
 * does (pcg.cpp:22-28).  Row-band / vertex-range (multi-GPU) solvers keep the
 * factor of the GLOBAL matrix on every rank and apply it to the all-gathered
 * residual, so they reproduce the single-GPU IC(0) iterates.
 * pfe_split_bregman_standalone and pfe_pcg_solve_multi
 * (PcgOperator::solve_multi) factor their matrix the same way. */
#define PFE_PRECOND_IC0 0
#define PFE_PRECOND_JACOBI 1
#define PFE_PRECOND_NONE 2

/* Topology actually used by a solver (pfe_report.topology). */
#define PFE_TOPO_CSR 0
#define PFE_TOPO_GRID8 1  /* 3x3 neighbourhood stencil */
#define PFE_TOPO_GRID24 2 /* 5x5 neighbourhood stencil */

/* WeightedGraph (graph.hpp:15-28): undirected edges stored once with i < j,
 * w finite; degree[] is used as given (solver.cpp:48-50) and must be > 0.
 * Optional grid hint: when grid_h * grid_w == n and every edge is a forward
 * stencil neighbour of radius grid_radius (1: 8-nbr, 2: 5x5) listed in
 * lexicographic order, the solver uses the stencil kernels (no index
 * arrays); otherwise it uses the general CSR kernels.  Results are identical
 * either way. */
typedef struct pfe_graph {
  int32_t n;
  int64_t m;
  const int32_t* ei;
  const int32_t* ej;
  const double* w;
  const double* degree;
  int32_t grid_h;
  int32_t grid_w;
  int32_t grid_radius;
} pfe_graph;

/* PfeParams (solver.hpp:16-25) with PcgConfig (pcg.hpp:15-19) flattened.
 * pfe_params_default() returns the reference defaults. */
typedef struct pfe_params {
  int32_t dim;
  double lambda;
  double r;
  int32_t soc_max;
  int32_t sb_max_stage1;
  int32_t sb_max_stage2;
  double conv_tol;
  double pcg_rel_tol;
  int32_t pcg_max_iter;
  int32_t preconditioner;
} pfe_params;

/* Execution options (no reference counterpart). */
typedef struct pfe_exec {
  int32_t device;       /* CUDA ordinal */
  int32_t use_graphs;   /* 1: capture the PCG loop as a CUDA graph with a
                           device-side WHILE node (no host sync per PCG
                           iteration); 0: host-driven loop */
  int32_t warn;         /* 1: print the reference's non-converged-column
                           warning to stderr (solver.cpp:87-92) */
  int32_t profile;      /* 1: time every kernel launch with CUDA events */
  int32_t persistent;   /* 1: pixel-grid graphs run each split_bregman call as
                           one persistent cooperative kernel (grid barriers,
                           device-side PCG control), keeping the PCG state in
                           shared memory when it fits; 2: the same kernel
                           without the shared-memory-resident variant;
                           0: one kernel per phase */
} pfe_exec;

/* Run report (PcgReport aggregation, pcg.hpp:21-26). */
typedef struct pfe_report {
  int64_t inner_iterations;      /* split-Bregman iterations executed */
  int64_t pcg_iterations;        /* sum over inner iterations of max-over-columns PCG iterations */
  int64_t pcg_column_iterations; /* sum over inner iterations and columns */
  int64_t nonconverged;          /* column solves that stopped unconverged (incl. failures) */
  int64_t failed;                /* column solves that broke down (x kept at x0) */
  int32_t jacobi_fallback;
  int32_t topology;
  int64_t n;
  int64_t m;
  int32_t d;
  int32_t persistent_kind;       /* kernel of the last persistent launch: 0 none,
                                    1 tiled (streams HBM/L2), 2 shared-memory resident */
  double setup_seconds;          /* host + device setup of pfe_solver_create */
} pfe_report;

/* Per-kernel-class timing when pfe_exec.profile = 1. */
#define PFE_KERNEL_CLASSES 8
/* 0 pcg_init, 1 pcg_spmv, 2 pcg_update (+ IC(0) triangular solves), 3 pcg_finalize, 4 sb_pass,
 * 5 rhs (quad / from state), 6 projection (tsqr + apply),
 * 7 persistent split-Bregman kernel */
typedef struct pfe_kernel_times {
  double ms[PFE_KERNEL_CLASSES];
  int64_t launches[PFE_KERNEL_CLASSES];
} pfe_kernel_times;

typedef struct pfe_solver pfe_solver;
typedef struct pfe_state pfe_state;

/* IterateCallback (solver.hpp:36): Y (column-major host copy) after each
 * inner iteration; forces the host-driven slow path. */
typedef void (*pfe_iterate_fn)(int iteration, const double* y_colmajor, int32_t n, int32_t d, void* user);

const char* pfe_last_error(void);
pfe_params pfe_params_default(void);
pfe_exec pfe_exec_default(void);
int pfe_device_check(int32_t device); /* 0 if an sm_100-class device is usable */
/* Destroyed solvers and states park their large device arrays in a per-device
 * cache (exact-size reuse by the next solver: the one-call pfe_solve otherwise
 * spends 0.1-1.4 s per call re-carving 24 GB for C4).  This returns the cached
 * blocks of `device` to the driver; the result is the number of bytes released.
 * Environment PFE_CACHE_MB caps the cache (default 40 % of device memory, 0 = off). */
int64_t pfe_release_cached_memory(int32_t device);

/* PfeSolver::PfeSolver (solver.hpp:53, solver.cpp:43-58): builds the
 * operator A = (lambda/2) M^T M + (r/2) D, its Jacobi preconditioner and the
 * graph topology on the device. */
int pfe_solver_create(const pfe_graph* g, const pfe_params* p, const pfe_exec* x, pfe_solver** out);
void pfe_solver_destroy(pfe_solver* s);
int pfe_solver_report(const pfe_solver* s, pfe_report* out);
/* PCG log: per inner iteration x column iterations / status / final residual
 * (status codes: 0 active, 1 converged, 2 zero rhs, 3 failed, 4 max_iter,
 * 5 converged at x0).  Returns the number of logged inner iterations. */
int64_t pfe_solver_pcg_log(const pfe_solver* s, int32_t* iters, int32_t* status, double* rel, int64_t cap);
int pfe_solver_kernel_times(const pfe_solver* s, pfe_kernel_times* out, int reset);
/* Device time (CUDA events on the solver's stream) of the last
 * split_bregman / run_soc / two_stage call, in milliseconds. */
double pfe_solver_last_ms(const pfe_solver* s);
/* Phase trace of the last persistent launch (environment PFE_TRACE=1 at
 * solver creation): entries are (phase code << 56) | %globaltimer ns,
 * recorded by block 0 after each grid barrier.  Returns the entry count. */
int64_t pfe_solver_trace(const pfe_solver* s, uint64_t* out, int64_t cap);

/* PfeSolver::make_state (solver.cpp:60-71): Y = y0, P = sqrt(D) y0, B = 0,
 * split_b = split_s = 0.  y0 is host column-major n x dim. */
int pfe_state_create(pfe_solver* s, const double* y0, pfe_state** out);
/* Re-initialise an existing state from the y0 it was created with (device
 * copy; no host transfer). */
int pfe_state_reset(pfe_state* st);
void pfe_state_destroy(pfe_state* st);

/* SolverState fields (solver.hpp:28-34). */
#define PFE_FIELD_Y 0
#define PFE_FIELD_P 1
#define PFE_FIELD_BREGMAN 2
#define PFE_FIELD_SPLIT_B 3
#define PFE_FIELD_SPLIT_S 4
int pfe_state_get(pfe_state* st, int32_t field, double* out);
int pfe_state_set(pfe_state* st, int32_t field, const double* in);

/* PfeSolver::split_bregman (solver.cpp:73-108). */
int pfe_split_bregman(pfe_solver* s, pfe_state* st, int32_t max_iter, pfe_iterate_fn cb, void* user);
/* PfeSolver::run_soc (solver.cpp:110-126). */
int pfe_run_soc(pfe_solver* s, pfe_state* st, int32_t soc_max, int32_t sb_max);
/* PfeSolver::two_stage (solver.cpp:128-136) on a state fresh from make_state. */
int pfe_two_stage(pfe_solver* s, pfe_state* st);
/* objective(diff_matrix(), Y of the state) (solver.cpp:14-17). */
int pfe_state_objective(pfe_solver* s, pfe_state* st, double* out);

/* One-call drop-ins, host buffers in and out:
 *   mode 0: soc(g, params, y0)            (solver.cpp:184-189)
 *   mode 1: pfe_two_stage(g, params, y0)  (solver.cpp:191-193)          */
int pfe_solve(const pfe_graph* g, const pfe_params* p, const pfe_exec* x, int32_t mode, const double* y0,
              double* y_out, pfe_report* rep);

/* Standalone split_bregman(M, d_vec, P, B, params, y_init, max_iter, cb)
 * (solver.cpp:138-182) with M = difference_matrix(g): fresh zero inner
 * variables, operator built for this call. */
int pfe_split_bregman_standalone(const pfe_graph* g, const double* p, const double* b, const pfe_params* prm,
                                 int32_t d, const double* y_init, int32_t max_iter, const pfe_exec* x,
                                 double* y_out, pfe_iterate_fn cb, void* user);

/* PcgOperator(A, cfg).solve_multi(B, X0) (pcg.cpp:94-114) on a caller CSR
 * matrix (row_ptr[n+1], col_idx, values; rows sorted, no duplicates as
 * csr_from_triplets produces, sparse.hpp:17-25).  Per column: iterations,
 * converged flag, final relative residual, jacobi_fallback. */
int pfe_pcg_solve_multi(int32_t n, const int32_t* row_ptr, const int32_t* col_idx, const double* values,
                        int32_t d, const double* b, const double* x0, double rel_tol, int32_t max_iter,
                        int32_t preconditioner, const pfe_exec* x, double* x_out, int32_t* iterations,
                        int32_t* converged, double* residual, int32_t* jacobi_fallback);

/* The IC(0) breakdown test of the PcgOperator constructor (pcg.cpp:22-28):
 * factors the CSR matrix on the host exactly as incomplete_cholesky does
 * (sparse.cpp:124-203, up to 8 diagonal shifts) and sets *jacobi_fallback
 * to 1 if the breakdown persisted.  Host only (no device needed). */
int pfe_ic0_probe(int32_t n, const int32_t* row_ptr, const int32_t* col_idx, const double* values,
                  int32_t* jacobi_fallback);
/* Multi-GPU row bands for pixel-grid graphs: one process
 * per GPU; rank 0 calls pfe_nccl_unique_id and shares the bytes (e.g. via
 * torch.distributed), then every rank creates its band solver from the SAME
 * global graph.  The band owns image rows [H*rank/nranks, H*(rank+1)/nranks)
 * plus an R-row halo exchanged with NCCL send/recv; PCG scalars and TSQR
 * factors are all-gathered.  pfe_state_create takes the global y0;
 * pfe_run_soc / pfe_two_stage / pfe_split_bregman run the banded solve
 * (fixed iteration counts); pfe_state_get(PFE_FIELD_Y) returns the global Y
 * on every rank.  NCCL is loaded at run time (libnccl.so.2). */
#define PFE_NCCL_ID_BYTES 128
/* Host only: band `rank` of `nranks` over `height` rows owns [out[0], out[1])
 * and stores [out[2], out[3]) (owned rows plus the radius-row halo). */
int pfe_band_plan(int32_t height, int32_t nranks, int32_t radius, int32_t rank, int32_t* out);
int pfe_nccl_unique_id(uint8_t* out);
int pfe_solver_create_band(const pfe_graph* g, const pfe_params* p, const pfe_exec* x, const uint8_t* nccl_id,
                           int32_t nranks, int32_t rank, pfe_solver** out);
/* Host only: the vertex-range partition pfe_solver_create_band builds for a
 * general graph over `nranks` ranks (BFS storage order, contiguous ranges):
 * per rank the owned vertices, the ghost rows it receives in every ghost
 * exchange, and the owned rows it sends (one per peer that needs them).
 * Arrays of nranks entries; any may be null. */
int pfe_range_partition_stats(const pfe_graph* g, int32_t nranks, int64_t* owned, int64_t* ghosts, int64_t* sends);
/* The same banded algorithm with `nbands` bands emulated in this process on
 * one device (device copies instead of NCCL): validates the decomposition.
 * mode 0: soc, 1: pfe_two_stage. */
int pfe_solve_banded(const pfe_graph* g, const pfe_params* p, const pfe_exec* x, int32_t nbands, int32_t mode,
                     const double* y0, double* y_out, pfe_report* rep);

/* Multi-GPU inside ONE call: soc (mode 0) or
 * pfe_two_stage (mode 1) of one graph over the `ndev` distinct CUDA devices
 * listed, from one host thread.  Pixel grids are cut into row bands, general
 * graphs into vertex ranges (the same decomposition as
 * pfe_solver_create_band); the communicators come from ncclCommInitAll and
 * every NCCL call of a step is issued for all devices in one group.  The
 * drop-in for pfe_two_stage(g, params, y0) (solver.cpp:191-193) on N GPUs.
 * device_ms (may be null): device time of the solve, max over the GPUs. */
int pfe_solve_multi_gpu(const pfe_graph* g, const pfe_params* p, const pfe_exec* x, int32_t ndev,
                        const int32_t* devices, int32_t mode, const double* y0, double* y_out, pfe_report* rep,
                        double* device_ms);

/* objective(M, Y) (solver.cpp:14-17) with M = difference_matrix(g). */
int pfe_objective(const pfe_graph* g, int32_t d, const double* y, const pfe_exec* x, double* out);
/* shrink(V, gamma) (solver.cpp:19-25), elementwise on count values. */
int pfe_shrink(int64_t count, const double* v, double gamma, const pfe_exec* x, double* out);
/* project_orthogonal(A) (solver.cpp:27-41): polar factor of n x d A. */
int pfe_project_orthogonal(int32_t n, int32_t d, const double* a, const pfe_exec* x, double* p_out);

/* Host-side boundary helpers (init.cpp:140-155, 172-181; cluster.cpp:54-124):
 * seeded Y0 and the k-means "labels out" step, same RNG streams as the
 * reference (std::mt19937_64 + libstdc++ distributions). */
int pfe_d_orthonormalize(int32_t n, int32_t d, const double* a, const double* degree, double* out);
int pfe_random_embedding(int32_t n, int32_t d, uint64_t seed, const double* degree, double* out);
int pfe_kmeans(int32_t n, int32_t d, const double* points, int32_t k, uint64_t seed, int32_t max_iter,
               int32_t* labels);

/* pfe_kmeans on the GPU: same seeding random stream,
 * tie-breaks, empty-cluster split and stop rule as pfe_kmeans; distances are
 * bitwise the host's, sums associate by chunks of 4096 points (labels agree
 * with the host's up to ties).  d <= 16, k * d <= 6144. */
int pfe_kmeans_device(int32_t n, int32_t d, const double* points, int32_t k, uint64_t seed, int32_t max_iter,
                      int32_t device, int32_t* labels);

/* GMM initial embedding on the GPU (gmm_fit +
 * init_embedding, init.cpp:45-170): k-means (20 iterations, seed) for the
 * starting means, <= 50 EM iterations of a diagonal GMM on the n x 3
 * features (row-major RGB triples, as imgio.cpp produces them), then the
 * responsibilities D-orthonormalised (Gram-Schmidt in <u, v> = u^T D v,
 * noise fallback of init.cpp:160-168).  Replaces the host init path of
 * main.cpp:109-110.  y_out: n x k column-major; means_out / vars_out
 * (k x 3 row-major) and weights_out (k) may be null.  1 <= k <= 16. */
int pfe_gmm_init_device(int32_t n, const double* features, int32_t k, uint64_t seed, const double* degree,
                        int32_t device, double* y_out, double* means_out, double* vars_out, double* weights_out);

/* k-NN graph builder for point sets (configs C1 / C5).  No reference
 * counterpart: the reference has no k-NN builder; this
 * is the harness definition of paper_1612_06496_b200/inputs.py knn_graph --
 * exact k nearest neighbours (ascending distance, then index) on the GPU,
 * sigma = median directed k-NN distance, union-symmetrised edges (i < j,
 * lexicographic), w = exp(-|x_i - x_j|^2 / (2 sigma^2)) dropped below 1e-12,
 * degree summed in edge order (graph.cpp:15-22).  points: row-major n x dim
 * (dim <= 32); k <= 32; ei / ej / w need capacity n * k, degree n.  Writes the
 * edge count to *m_out and sigma to *sigma_out. */
int pfe_knn_graph(int32_t n, int32_t dim, const double* points, int32_t k, int32_t device, int32_t* ei, int32_t* ej,
                  double* w, double* degree, int64_t* m_out, double* sigma_out);

/* Pixel-grid graph builder on the GPU (configs C2-C4):
 * build_image_graph (graph.cpp:105-159) generalised to the 8-neighbour
 * (radius 1) and 5x5 (radius 2) neighbourhoods, as the harness builder
 * paper_1612_06496_b200/inputs.py grid_graph defines it: heat kernel
 * w = exp(-|drgb|^2 / (2 sigma_rgb^2) [- |dxy|^2 / (2 sigma_xy^2) if sigma_xy > 0]),
 * weights below 1e-12 dropped, an isolated pixel keeps its strongest
 * incident candidate floored at 1e-12, edges lexicographic (i < j), degree
 * summed in edge order (graph.cpp:15-22).  rgb: row-major height x width x 3.
 * ei / ej / w need capacity n * (4 or 12), degree n; *m_out = edge count.
 * Weights equal the host builder's up to the last ulp of exp. */
int pfe_grid_graph(int32_t height, int32_t width, const double* rgb, double sigma_rgb, int32_t radius,
                   double sigma_xy, int32_t device, int32_t* ei, int32_t* ej, double* w, double* degree,
                   int64_t* m_out);

#ifdef __cplusplus
}
#endif

#endif /* PFE_B200_H */
