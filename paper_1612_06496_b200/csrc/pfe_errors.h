// Error type carried from the implementation to the C ABI status codes
// (errors.hpp:9-24 -> proj/tools/main.cpp:431-446 numbering).
#pragma once

#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

namespace pfe_host {

struct Error : std::runtime_error {
  int code;
  Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

void random_embedding(int n, int d, uint64_t seed, const double* deg, double* out);
void d_orthonormalize(int n, int d, const double* a, const double* deg, double* out);
void kmeans(int n, int d, const double* pts, int k, uint64_t seed, int max_iter, int32_t* labels);
void knn_search(int n, int dim, const double* pts, int k, double* d2, int32_t* idx);
void kmeans_device(int n, int d, const double* pts, int k, uint64_t seed, int max_iter, int32_t* labels);
// IC(0) factor L (A ~ L L^T) of a natural-order CSR matrix, exactly as
// incomplete_cholesky (sparse.cpp:124-203): lower triangle with a diagonal
// shift, row-oriented sweep, shift retries.  false: breakdown persisted
// (the reference then falls back to Jacobi, pcg.cpp:22-28).
struct IcFactorHost {
  std::vector<int> ptr, idx;  // rows of L, ascending columns, diagonal last
  std::vector<double> val;
  double shift = 0.0;
};
bool ic0_factor(int n, const int* ptr, const int* idx, const double* val, IcFactorHost& out);
void gmm_init_device(int n, const double* feat, int k, uint64_t seed, const double* degree, double* y_out,
                     double* means_out, double* vars_out, double* weights_out);
long grid_graph_device(int H, int W, const double* rgb, double sigma_rgb, int radius, double sigma_xy, int32_t* ei,
                       int32_t* ej, double* w, double* degree);
long knn_graph_from_lists(int n, int k, const double* d2, const int32_t* idx, int32_t* ei, int32_t* ej, double* w,
                          double* degree, double* sigma_out);

// General-graph solver topology built on the device (pfe_csrbuild.cu): all
// pointers are device arrays in storage order, allocated through `alloc`.
struct CsrDevArrays {
  int* aptr = nullptr;   // [n + 1] rows of A
  int* acol = nullptr;   // [nnz] storage rows, reference column order
  double* aval = nullptr;
  int* iptr = nullptr;   // [n + 1] incidence lists, increasing edge index
  int* inbr = nullptr;   // [2m] neighbour storage row
  int* ieid = nullptr;   // [2m] edge row << 1 | [vertex is the edge's first endpoint]
  double* iw = nullptr;  // [2m]
  double* diag = nullptr;
  double* invd = nullptr;
  double* deg = nullptr;
  double* sqd = nullptr;
  int* perm = nullptr;          // [n] vertex -> storage row
  int32_t* edge_row = nullptr;  // [m] edge -> row of the edge arrays
  long nnz = 0;
  int components = 0;
};
using DevAllocFn = void* (*)(void* ctx, size_t bytes);
using H2dFn = void (*)(void* dst, const void* src, size_t bytes, void* stream);
// false: more than max_components connected components or 4 * max_components
// breadth-first levels (the level-synchronous device BFS would crawl; the
// caller builds on the host instead).
bool csr_topology_device(int n, long m, const int32_t* ei, const int32_t* ej, const double* w, const double* degree,
                         double hl, double dterm, bool precond_none, void* stream, DevAllocFn alloc, void* alloc_ctx,
                         H2dFn h2d, int max_components, CsrDevArrays* out);

}  // namespace pfe_host
