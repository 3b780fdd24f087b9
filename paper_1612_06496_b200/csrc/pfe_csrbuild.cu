// General-graph (CSR) solver topology built on the GPU.
//
// pfe_solver_create for a k-NN / arbitrary edge list used to build the
// solver's device arrays on the host (incidence lists, breadth-first storage
// order, the rows of A = (lambda/2) M^T M + (r/2) D, edge-row assignment,
// permuted copies) and upload them: 0.47-0.51 s for C5 (10^6 vertices,
// 12.7 M edges) against 0.83 s for the whole soc solve.  Here the edge list is
// uploaded once and every array is derived by kernels and CUB radix sorts /
// scans, reproducing the host builder bit for bit:
//
//   * incidence lists in increasing edge index (the row order of M^T,
//     sparse.cpp:52-72): stable sort of the 2m (vertex, entry) pairs;
//   * diag(A): sum over incident edges in edge order of (hl w) w, then
//     + (r/2) deg_v last (csr_from_triplets order, sparse.cpp:96-122);
//   * storage order: the breadth-first order of the sequential queue
//     (components in vertex order, neighbours in incidence order).  Level by
//     level, every frontier vertex at queue position p offers each unvisited
//     neighbour the key (p, index in p's list); atomicMin keeps the first
//     discoverer, and sorting the discovered vertices by key gives exactly the
//     order in which the sequential queue appends them;
//   * rows of A: stable sort of the 2m + n (row, column) entries, duplicate
//     columns summed in edge order, exact zeros dropped, columns renamed to
//     storage rows (form_normal_matrix / csr_from_triplets semantics);
//   * edge rows: the edges a vertex owns (it is their first endpoint)
//     consecutive, vertices in storage order; incidence lists rewritten with
//     storage rows and edge rows.
//
// tests/test_gpu_csrbuild.py compares solves on both builders bit for bit.
#include <cuda_runtime.h>

#include <cub/cub.cuh>
#include <nvtx3/nvToolsExt.h>

#include <algorithm>
#include <climits>
#include <memory>
#include <string>
#include <vector>

#include "pfe_b200.h"
#include "pfe_errors.h"

namespace {

using pfe_host::Error;
using ull = unsigned long long;
constexpr int kT = 256;
constexpr ull kNoKey = ~0ull;

void ck(cudaError_t e, const char* what) {
  if (e != cudaSuccess) throw Error(PFE_CUDA_ERROR, std::string(what) + ": " + cudaGetErrorString(e));
}
#define CKB(x) ck((x), #x)

int blocks_for(long items) { return static_cast<int>(std::max<long>(1, std::min<long>((items + kT - 1) / kT, 148L * 32))); }
int bits_for(long maxval) {  // bits needed to represent values in [0, maxval]
  int b = 1;
  while ((maxval >> b) != 0) ++b;
  return b;
}

// Stream-ordered scratch, returned to the pool when the build ends.
struct Scratch {
  cudaStream_t st;
  std::vector<void*> ptrs;
  explicit Scratch(cudaStream_t s) : st(s) {}
  template <class T>
  T* get(size_t count) {
    void* p = nullptr;
    CKB(cudaMallocAsync(&p, std::max<size_t>(count, 1) * sizeof(T), st));
    ptrs.push_back(p);
    return static_cast<T*>(p);
  }
  ~Scratch() {
    for (void* p : ptrs) cudaFreeAsync(p, st);
  }
};

// NVTX range for a scope (popped on every exit path)
struct Nvtx {
  explicit Nvtx(const char* name) { nvtxRangePushA(name); }
  ~Nvtx() { nvtxRangePop(); }
};

#define GRID_STRIDE(i, n) for (long i = blockIdx.x * static_cast<long>(blockDim.x) + threadIdx.x; i < (n); i += static_cast<long>(gridDim.x) * blockDim.x)

// ------------------------------------------------------------- incidence --
__global__ void k_inc_keys(long m, const int32_t* __restrict__ ei, const int32_t* __restrict__ ej, int* keys, int* vals) {
  GRID_STRIDE(k, m) {
    keys[2 * k] = ei[k];
    vals[2 * k] = static_cast<int>(2 * k);
    keys[2 * k + 1] = ej[k];
    vals[2 * k + 1] = static_cast<int>(2 * k + 1);
  }
}
__global__ void k_inc_fill(long m2, const int* __restrict__ svals, const int32_t* __restrict__ ei,
                           const int32_t* __restrict__ ej, const double* __restrict__ w, int* inbr, int* ie, double* iw) {
  GRID_STRIDE(i, m2) {
    const int e = svals[i] >> 1;
    inbr[i] = (svals[i] & 1) ? ei[e] : ej[e];
    ie[i] = e;
    iw[i] = w[e];
  }
}
// ptr[v] = first index i with keys[i] >= v (keys ascending), v in [0, n]
__global__ void k_row_ptr(int n, long cnt, const int* __restrict__ keys, int* ptr) {
  GRID_STRIDE(v, static_cast<long>(n) + 1) {
    long lo = 0, hi = cnt;
    while (lo < hi) {
      const long mid = (lo + hi) >> 1;
      if (keys[mid] < v) lo = mid + 1;
      else hi = mid;
    }
    ptr[v] = static_cast<int>(lo);
  }
}
__global__ void k_diag(int n, const int* __restrict__ iptr, const double* __restrict__ iw, const double* __restrict__ deg,
                       double hl, double dterm, double* diag, int* degree_count) {
  GRID_STRIDE(v, n) {
    double acc = 0.0;
    for (int k = iptr[v]; k < iptr[v + 1]; ++k) acc += (hl * iw[k]) * iw[k];
    diag[v] = acc + dterm * deg[v];  // the (r/2) d_v triplet is summed last
    degree_count[v] = iptr[v + 1] - iptr[v];
  }
}

// ------------------------------------------------- breadth-first order ----
__global__ void k_find_seed(int n, int start, const int* __restrict__ pos, int* out) {
  GRID_STRIDE(i, static_cast<long>(n) - start) {
    const int v = start + static_cast<int>(i);
    if (pos[v] < 0) {
      atomicMin(out, v);
      return;  // later vertices of this thread are larger
    }
  }
}
__global__ void k_place_seed(const int* seed, int at, int* order, int* pos) {
  order[at] = *seed;
  pos[*seed] = at;
}
// Frontier = queue positions [f0, f1).  Every unvisited neighbour keeps the
// smallest (relative queue position, index in that vertex's list) offered.
__global__ void k_expand(int f0, int f1, int jbits, const int* __restrict__ order, const int* __restrict__ iptr,
                         const int* __restrict__ inbr, const int* __restrict__ pos, ull* key, int* cand, int* ncand) {
  GRID_STRIDE(i, static_cast<long>(f1) - f0) {
    const int u = order[f0 + i];
    const int b = iptr[u], e = iptr[u + 1];
    for (int k = b; k < e; ++k) {
      const int nb = inbr[k];
      if (pos[nb] >= 0) continue;
      const ull mine = (static_cast<ull>(i) << jbits) | static_cast<ull>(k - b);
      const ull old = atomicMin(&key[nb], mine);
      if (old == kNoKey) cand[atomicAdd(ncand, 1)] = nb;
    }
  }
}
__global__ void k_gather_keys(int nc, const int* __restrict__ cand, const ull* __restrict__ key, ull* out) {
  GRID_STRIDE(i, nc) out[i] = key[cand[i]];
}
__global__ void k_place(int nc, const int* __restrict__ sorted, int at, int* order, int* pos) {
  GRID_STRIDE(i, nc) {
    order[at + i] = sorted[i];
    pos[sorted[i]] = at + static_cast<int>(i);
  }
}

// --------------------------------------------------------------- A rows ----
// entries: i < m2 -> incidence entry i of vertex vert[i]; i >= m2 -> the
// diagonal of vertex i - m2.  key = storage row << cbits | column (vertex id)
__global__ void k_row_keys(long m2, int n, int cbits, const int* __restrict__ vert, const int* __restrict__ inbr,
                           const int* __restrict__ pos, ull* keys, int* idx) {
  GRID_STRIDE(i, m2 + n) {
    const int v = i < m2 ? vert[i] : static_cast<int>(i - m2);
    const int col = i < m2 ? inbr[i] : v;
    keys[i] = (static_cast<ull>(pos[v]) << cbits) | static_cast<ull>(col);
    idx[i] = static_cast<int>(i);
  }
}
// Group heads sum their group in edge order (the stable sort kept it).
__global__ void k_row_groups(long cnt, long m2, const ull* __restrict__ skey, const int* __restrict__ sidx,
                             const double* __restrict__ iw, const double* __restrict__ diag, double hl, int* flag,
                             double* val) {
  GRID_STRIDE(i, cnt + 1) {
    if (i == cnt) {
      flag[i] = 0;
      continue;
    }
    const ull k = skey[i];
    if (i > 0 && skey[i - 1] == k) {
      flag[i] = 0;
      continue;
    }
    double s = 0.0;
    for (long t = i; t < cnt && skey[t] == k; ++t) {
      const int id = sidx[t];
      if (id < m2) s += -((hl * iw[id]) * iw[id]);
      else s = diag[id - m2];  // the diagonal, already accumulated in csr_from_triplets order
    }
    val[i] = s;
    flag[i] = s != 0.0 ? 1 : 0;
  }
}
__global__ void k_row_compact(long cnt, int cbits, const ull* __restrict__ skey, const int* __restrict__ flag,
                              const int* __restrict__ opos, const double* __restrict__ val, const int* __restrict__ pos,
                              int* acol, double* aval) {
  GRID_STRIDE(i, cnt) {
    if (!flag[i]) continue;
    const int col = static_cast<int>(skey[i] & ((1ull << cbits) - 1));
    acol[opos[i]] = pos[col];
    aval[opos[i]] = val[i];
  }
}
__global__ void k_row_aptr(int n, long cnt, int cbits, const ull* __restrict__ skey, const int* __restrict__ opos, int* aptr) {
  GRID_STRIDE(x, static_cast<long>(n) + 1) {
    const ull want = static_cast<ull>(x) << cbits;
    long lo = 0, hi = cnt;
    while (lo < hi) {
      const long mid = (lo + hi) >> 1;
      if (skey[mid] < want) lo = mid + 1;
      else hi = mid;
    }
    aptr[x] = opos[lo];
  }
}

// ------------------------------------------- storage-order incidence ------
__global__ void k_own_count(int n, const int* __restrict__ order, const int* __restrict__ iptr, const int* __restrict__ inbr,
                            int* own, int* len) {
  GRID_STRIDE(x, static_cast<long>(n) + 1) {
    if (x == n) {
      own[x] = 0;
      len[x] = 0;
      continue;
    }
    const int v = order[x];
    int c = 0;
    for (int k = iptr[v]; k < iptr[v + 1]; ++k) c += inbr[k] > v ? 1 : 0;
    own[x] = c;
    len[x] = iptr[v + 1] - iptr[v];
  }
}
__global__ void k_edge_rows(int n, const int* __restrict__ order, const int* __restrict__ iptr, const int* __restrict__ inbr,
                            const int* __restrict__ ie, const int* __restrict__ own, int32_t* epos) {
  GRID_STRIDE(x, n) {
    const int v = order[x];
    int next = own[x];
    for (int k = iptr[v]; k < iptr[v + 1]; ++k)
      if (inbr[k] > v) epos[ie[k]] = next++;
  }
}
__global__ void k_final_incidence(int n, const int* __restrict__ order, const int* __restrict__ iptr,
                                  const int* __restrict__ inbr, const int* __restrict__ ie, const double* __restrict__ iw,
                                  const int* __restrict__ pos, const int32_t* __restrict__ epos,
                                  const int* __restrict__ iptr2, int* inbr2, int* ieid2, double* iw2) {
  GRID_STRIDE(x, n) {
    const int v = order[x];
    int at = iptr2[x];
    for (int k = iptr[v]; k < iptr[v + 1]; ++k, ++at) {
      inbr2[at] = pos[inbr[k]];
      ieid2[at] = (epos[ie[k]] << 1) | (inbr[k] > v ? 1 : 0);
      iw2[at] = iw[k];
    }
  }
}
__global__ void k_vertex_arrays(int n, const int* __restrict__ order, const double* __restrict__ diag_nat,
                                const double* __restrict__ deg_nat, int precond_none, double* diag, double* invd,
                                double* deg, double* sqd) {
  GRID_STRIDE(x, n) {
    const int v = order[x];
    const double dg = diag_nat[v];
    diag[x] = dg;
    invd[x] = precond_none ? 1.0 : (dg > 0.0 ? 1.0 / dg : 1.0);
    deg[x] = deg_nat[v];
    sqd[x] = sqrt(deg_nat[v]);
  }
}

}  // namespace

namespace pfe_host {

bool csr_topology_device(int n, long m, const int32_t* ei, const int32_t* ej, const double* w, const double* degree,
                         double hl, double dterm, bool precond_none, void* stream, DevAllocFn alloc, void* alloc_ctx,
                         H2dFn h2d, int max_components, CsrDevArrays* out) {
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const long m2 = 2 * m, ent = m2 + n;
  if (ent >= INT_MAX) return false;
  auto keep = [&](size_t bytes) { return alloc(alloc_ctx, std::max<size_t>(bytes, 8)); };
  Scratch tmp(st);

  // edge list and degrees on the device
  int32_t* d_ei = tmp.get<int32_t>(m);
  int32_t* d_ej = tmp.get<int32_t>(m);
  double* d_w = tmp.get<double>(m);
  double* d_degn = tmp.get<double>(n);
  if (m > 0) {
    h2d(d_ei, ei, sizeof(int32_t) * m, st);
    h2d(d_ej, ej, sizeof(int32_t) * m, st);
    h2d(d_w, w, sizeof(double) * m, st);
  }
  h2d(d_degn, degree, sizeof(double) * n, st);

  // CUB scratch sized for the largest call (the row sort)
  size_t cub_bytes = 0;
  {
    size_t b = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, b, static_cast<ull*>(nullptr), static_cast<ull*>(nullptr),
                                    static_cast<int*>(nullptr), static_cast<int*>(nullptr), ent, 0, 64, st);
    cub_bytes = std::max(cub_bytes, b);
    cub::DeviceRadixSort::SortPairs(nullptr, b, static_cast<int*>(nullptr), static_cast<int*>(nullptr),
                                    static_cast<int*>(nullptr), static_cast<int*>(nullptr), m2, 0, 32, st);
    cub_bytes = std::max(cub_bytes, b);
    cub::DeviceScan::ExclusiveSum(nullptr, b, static_cast<int*>(nullptr), static_cast<int*>(nullptr), ent + 1, st);
    cub_bytes = std::max(cub_bytes, b);
    cub::DeviceReduce::Max(nullptr, b, static_cast<int*>(nullptr), static_cast<int*>(nullptr), n, st);
    cub_bytes = std::max(cub_bytes, b);
  }
  void* cub_tmp = tmp.get<char>(cub_bytes);

  // ---- incidence lists, natural vertex order, increasing edge index
  auto nv = std::make_unique<Nvtx>("pfe csr build: incidence");
  int* keys = tmp.get<int>(m2);
  int* vals = tmp.get<int>(m2);
  int* vert = tmp.get<int>(m2);   // sorted keys: the vertex of every incidence entry
  int* svals = tmp.get<int>(m2);
  int* iptr = tmp.get<int>(static_cast<size_t>(n) + 1);
  int* inbr = tmp.get<int>(m2);
  int* ie = tmp.get<int>(m2);
  double* iw = tmp.get<double>(m2);
  const int vbits = bits_for(std::max(1, n - 1));
  if (m > 0) {
    k_inc_keys<<<blocks_for(m), kT, 0, st>>>(m, d_ei, d_ej, keys, vals);
    size_t b = cub_bytes;
    CKB(cub::DeviceRadixSort::SortPairs(cub_tmp, b, keys, vert, vals, svals, m2, 0, vbits, st));
    k_inc_fill<<<blocks_for(m2), kT, 0, st>>>(m2, svals, d_ei, d_ej, d_w, inbr, ie, iw);
  }
  k_row_ptr<<<blocks_for(n + 1), kT, 0, st>>>(n, m2, vert, iptr);
  double* diag_nat = tmp.get<double>(n);
  int* degcnt = tmp.get<int>(n);
  k_diag<<<blocks_for(n), kT, 0, st>>>(n, iptr, iw, d_degn, hl, dterm, diag_nat, degcnt);
  int* d_scalar = tmp.get<int>(2);  // [0] max degree / seed, [1] candidate count
  {
    size_t b = cub_bytes;
    CKB(cub::DeviceReduce::Max(cub_tmp, b, degcnt, d_scalar, n, st));
  }
  int maxdeg = 0;
  CKB(cudaMemcpyAsync(&maxdeg, d_scalar, sizeof(int), cudaMemcpyDeviceToHost, st));
  CKB(cudaStreamSynchronize(st));
  const int jbits = bits_for(std::max(1, maxdeg));

  // ---- breadth-first storage order (the sequential queue's order)
  nv.reset();
  nv = std::make_unique<Nvtx>("pfe csr build: breadth-first order");
  int* pos = static_cast<int*>(keep(sizeof(int) * n));  // vertex -> storage row (kept: perm)
  int* order = tmp.get<int>(n);
  ull* key = tmp.get<ull>(n);
  ull* ckey = tmp.get<ull>(n);
  ull* ckey2 = tmp.get<ull>(n);
  int* cand = tmp.get<int>(n);
  int* cand2 = tmp.get<int>(n);
  CKB(cudaMemsetAsync(pos, 0xff, sizeof(int) * n, st));
  CKB(cudaMemsetAsync(key, 0xff, sizeof(ull) * n, st));
  int placed = 0, start = 0, comps = 0, levels = 0;
  int* seed = d_scalar;
  int* ncand = d_scalar + 1;
  while (placed < n) {
    if (++comps > max_components) return false;  // many tiny components: the host builder handles those
    const int big = INT_MAX;
    CKB(cudaMemcpyAsync(seed, &big, sizeof(int), cudaMemcpyHostToDevice, st));
    k_find_seed<<<blocks_for(n - start), kT, 0, st>>>(n, start, pos, seed);
    k_place_seed<<<1, 1, 0, st>>>(seed, placed, order, pos);
    int s = 0;
    CKB(cudaMemcpyAsync(&s, seed, sizeof(int), cudaMemcpyDeviceToHost, st));
    int f0 = placed, f1 = placed + 1;
    placed = f1;
    for (;;) {
      // every level costs a host round trip: chain-like graphs (thousands of
      // levels, or levels of a few vertices) are left to the host builder as well
      if (++levels > 4 * max_components || (levels > 256 && placed < 64L * levels)) return false;
      CKB(cudaMemsetAsync(ncand, 0, sizeof(int), st));
      k_expand<<<blocks_for(f1 - f0), kT, 0, st>>>(f0, f1, jbits, order, iptr, inbr, pos, key, cand, ncand);
      int nc = 0;
      CKB(cudaMemcpyAsync(&nc, ncand, sizeof(int), cudaMemcpyDeviceToHost, st));
      CKB(cudaStreamSynchronize(st));
      if (nc == 0) break;
      k_gather_keys<<<blocks_for(nc), kT, 0, st>>>(nc, cand, key, ckey);
      size_t b = cub_bytes;
      CKB(cub::DeviceRadixSort::SortPairs(cub_tmp, b, ckey, ckey2, cand, cand2, nc, 0,
                                          jbits + bits_for(std::max(1, f1 - f0 - 1)), st));
      k_place<<<blocks_for(nc), kT, 0, st>>>(nc, cand2, f1, order, pos);
      f0 = f1;
      f1 += nc;
      placed = f1;
    }
    start = s + 1;  // (s was read by the first synchronisation of the level loop)
  }
  CKB(cudaGetLastError());

  // ---- rows of A in storage order
  nv.reset();
  nv = std::make_unique<Nvtx>("pfe csr build: rows of A, incidence");
  ull* rkeys = tmp.get<ull>(ent);
  ull* rkeys2 = tmp.get<ull>(ent);
  int* ridx = tmp.get<int>(ent);
  int* ridx2 = tmp.get<int>(ent);
  int* flag = tmp.get<int>(ent + 1);
  int* opos = tmp.get<int>(ent + 1);
  double* gval = tmp.get<double>(ent);
  k_row_keys<<<blocks_for(ent), kT, 0, st>>>(m2, n, vbits, vert, inbr, pos, rkeys, ridx);
  {
    size_t b = cub_bytes;
    CKB(cub::DeviceRadixSort::SortPairs(cub_tmp, b, rkeys, rkeys2, ridx, ridx2, ent, 0, 2 * vbits, st));
  }
  k_row_groups<<<blocks_for(ent + 1), kT, 0, st>>>(ent, m2, rkeys2, ridx2, iw, diag_nat, hl, flag, gval);
  {
    size_t b = cub_bytes;
    CKB(cub::DeviceScan::ExclusiveSum(cub_tmp, b, flag, opos, ent + 1, st));
  }
  int nnz = 0;
  CKB(cudaMemcpyAsync(&nnz, opos + ent, sizeof(int), cudaMemcpyDeviceToHost, st));
  CKB(cudaStreamSynchronize(st));
  out->aptr = static_cast<int*>(keep(sizeof(int) * (static_cast<size_t>(n) + 1)));
  out->acol = static_cast<int*>(keep(sizeof(int) * static_cast<size_t>(nnz)));
  out->aval = static_cast<double*>(keep(sizeof(double) * static_cast<size_t>(nnz)));
  k_row_compact<<<blocks_for(ent), kT, 0, st>>>(ent, vbits, rkeys2, flag, opos, gval, pos, out->acol, out->aval);
  k_row_aptr<<<blocks_for(n + 1), kT, 0, st>>>(n, ent, vbits, rkeys2, opos, out->aptr);
  out->nnz = nnz;

  // ---- edge rows and incidence lists in storage order
  int* own = tmp.get<int>(static_cast<size_t>(n) + 1);
  int* len = tmp.get<int>(static_cast<size_t>(n) + 1);
  int* own_off = tmp.get<int>(static_cast<size_t>(n) + 1);
  out->iptr = static_cast<int*>(keep(sizeof(int) * (static_cast<size_t>(n) + 1)));
  out->inbr = static_cast<int*>(keep(sizeof(int) * static_cast<size_t>(m2)));
  out->ieid = static_cast<int*>(keep(sizeof(int) * static_cast<size_t>(m2)));
  out->iw = static_cast<double*>(keep(sizeof(double) * static_cast<size_t>(m2)));
  out->edge_row = static_cast<int32_t*>(keep(sizeof(int32_t) * static_cast<size_t>(m)));
  k_own_count<<<blocks_for(n + 1), kT, 0, st>>>(n, order, iptr, inbr, own, len);
  {
    size_t b = cub_bytes;
    CKB(cub::DeviceScan::ExclusiveSum(cub_tmp, b, own, own_off, n + 1, st));
    b = cub_bytes;
    CKB(cub::DeviceScan::ExclusiveSum(cub_tmp, b, len, out->iptr, n + 1, st));
  }
  k_edge_rows<<<blocks_for(n), kT, 0, st>>>(n, order, iptr, inbr, ie, own_off, out->edge_row);
  k_final_incidence<<<blocks_for(n), kT, 0, st>>>(n, order, iptr, inbr, ie, iw, pos, out->edge_row, out->iptr, out->inbr,
                                                  out->ieid, out->iw);
  out->diag = static_cast<double*>(keep(sizeof(double) * n));
  out->invd = static_cast<double*>(keep(sizeof(double) * n));
  out->deg = static_cast<double*>(keep(sizeof(double) * n));
  out->sqd = static_cast<double*>(keep(sizeof(double) * n));
  k_vertex_arrays<<<blocks_for(n), kT, 0, st>>>(n, order, diag_nat, d_degn, precond_none ? 1 : 0, out->diag, out->invd,
                                                out->deg, out->sqd);
  out->perm = pos;
  out->components = comps;
  CKB(cudaGetLastError());
  CKB(cudaStreamSynchronize(st));  // the scratch is released after the last kernel that reads it
  return true;
}

}  // namespace pfe_host
