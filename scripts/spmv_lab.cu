// Kernel lab for the general-graph (k-NN, CSR) PCG SpMV q = A p, d = 16
// (C5's operator).  NOT product code: variants of the gather loop timed side by
// side on the real C5 matrix (scripts/spmv_lab.py builds it) to choose the
// design that goes into csrc/.  Every variant sums each row left to right with
// separate multiply and add (-fmad=false), so all must agree bit for bit.
//
// nvcc -O3 -gencode arch=compute_100a,code=sm_100a -fmad=false -lineinfo -shared -Xcompiler -fPIC \
//      scripts/spmv_lab.cu -o scripts/libspmv_lab.so
#include <cuda_runtime.h>

#include <cstdio>
#include <vector>

namespace {

constexpr int D = 16;

// ---- V0: the shipped round-1 loop (8 lanes per row, 2 columns per lane,
// batches of B gathers in registers, next batch's indices prefetched)
template <int B, int MINB>
__global__ void __launch_bounds__(256, MINB) v_regs(int n, const int* __restrict__ aptr, const int* __restrict__ acol,
                                                   const double* __restrict__ aval, const double* __restrict__ p,
                                                   double* __restrict__ q) {
  const long total = static_cast<long>(n) * 8;
  const long per = ((total + gridDim.x - 1) / gridDim.x + blockDim.x - 1) / blockDim.x * blockDim.x;
  const long e0 = static_cast<long>(blockIdx.x) * per + threadIdx.x;
  long e1 = static_cast<long>(blockIdx.x + 1) * per;
  e1 = e1 < total ? e1 : total;
  for (long e = e0; e < e1; e += blockDim.x) {
    const int v = static_cast<int>(e >> 3);
    const int c0 = static_cast<int>(e & 7) * 2;
    double q0 = 0.0, q1 = 0.0;
    const int b = __ldg(aptr + v), en = __ldg(aptr + v + 1);
    int cu[B];
#pragma unroll
    for (int j = 0; j < B; ++j) cu[j] = b + j < en ? __ldg(acol + b + j) : -1;
    for (int k0 = b; k0 < en; k0 += B) {
      double2 g[B];
      double av[B];
#pragma unroll
      for (int j = 0; j < B; ++j)
        if (cu[j] >= 0) {
          g[j] = __ldg(reinterpret_cast<const double2*>(p + static_cast<long>(cu[j]) * D + c0));
          av[j] = __ldg(aval + k0 + j);
        }
      int cn[B];
#pragma unroll
      for (int j = 0; j < B; ++j) cn[j] = k0 + B + j < en ? __ldg(acol + k0 + B + j) : -1;
#pragma unroll
      for (int j = 0; j < B; ++j)
        if (cu[j] >= 0) {
          q0 += av[j] * g[j].x;
          q1 += av[j] * g[j].y;
        }
#pragma unroll
      for (int j = 0; j < B; ++j) cu[j] = cn[j];
    }
    reinterpret_cast<double2*>(q + static_cast<long>(v) * D + c0)[0] = make_double2(q0, q1);
  }
}

// ---- V2: 4 lanes per row, 32-byte (256-bit) loads: a warp gathers 8 rows
// per instruction.
__device__ __forceinline__ void ldg256(const double* p, double (&r)[4]) {
  asm volatile("ld.global.nc.v4.f64 {%0,%1,%2,%3}, [%4];" : "=d"(r[0]), "=d"(r[1]), "=d"(r[2]), "=d"(r[3]) : "l"(p));
}
template <int B, int MINB>
__global__ void __launch_bounds__(256, MINB) v_regs4(int n, const int* __restrict__ aptr, const int* __restrict__ acol,
                                                    const double* __restrict__ aval, const double* __restrict__ p,
                                                    double* __restrict__ q) {
  const long total = static_cast<long>(n) * 4;
  const long per = ((total + gridDim.x - 1) / gridDim.x + blockDim.x - 1) / blockDim.x * blockDim.x;
  const long e0 = static_cast<long>(blockIdx.x) * per + threadIdx.x;
  long e1 = static_cast<long>(blockIdx.x + 1) * per;
  e1 = e1 < total ? e1 : total;
  for (long e = e0; e < e1; e += blockDim.x) {
    const int v = static_cast<int>(e >> 2);
    const int c0 = static_cast<int>(e & 3) * 4;
    double acc[4] = {0.0, 0.0, 0.0, 0.0};
    const int b = __ldg(aptr + v), en = __ldg(aptr + v + 1);
    int cu[B];
#pragma unroll
    for (int j = 0; j < B; ++j) cu[j] = b + j < en ? __ldg(acol + b + j) : -1;
    for (int k0 = b; k0 < en; k0 += B) {
      double g[B][4];
      double av[B];
#pragma unroll
      for (int j = 0; j < B; ++j)
        if (cu[j] >= 0) {
          ldg256(p + static_cast<long>(cu[j]) * D + c0, g[j]);
          av[j] = __ldg(aval + k0 + j);
        }
      int cn[B];
#pragma unroll
      for (int j = 0; j < B; ++j) cn[j] = k0 + B + j < en ? __ldg(acol + k0 + B + j) : -1;
#pragma unroll
      for (int j = 0; j < B; ++j)
        if (cu[j] >= 0)
#pragma unroll
          for (int k = 0; k < 4; ++k) acc[k] += av[j] * g[j][k];
#pragma unroll
      for (int j = 0; j < B; ++j) cu[j] = cn[j];
    }
    double* o = q + static_cast<long>(v) * D + c0;
    reinterpret_cast<double2*>(o)[0] = make_double2(acc[0], acc[1]);
    reinterpret_cast<double2*>(o)[1] = make_double2(acc[2], acc[3]);
  }
}

// ---- V4: as V2, but the blocks sweep the storage order together: block b
// takes chunks b, b + nb, ... of 64 consecutive rows, so the rows gathered
// at any moment come from a narrow window of the breadth-first order
// (L2-resident) instead of the whole 128 MB vector.
template <int B, int MINB, int CHUNK>
__global__ void __launch_bounds__(256, MINB) v_sweep4(int n, const int* __restrict__ aptr, const int* __restrict__ acol,
                                                     const double* __restrict__ aval, const double* __restrict__ p,
                                                     double* __restrict__ q) {
  const long total = static_cast<long>(n) * 4;
  constexpr int ITEMS = CHUNK * 4;
  for (long base = static_cast<long>(blockIdx.x) * ITEMS; base < total; base += static_cast<long>(gridDim.x) * ITEMS) {
    for (long e = base + threadIdx.x; e < base + ITEMS && e < total; e += blockDim.x) {
      const int v = static_cast<int>(e >> 2);
      const int c0 = static_cast<int>(e & 3) * 4;
      double acc[4] = {0.0, 0.0, 0.0, 0.0};
      const int b = __ldg(aptr + v), en = __ldg(aptr + v + 1);
      int cu[B];
#pragma unroll
      for (int j = 0; j < B; ++j) cu[j] = b + j < en ? __ldg(acol + b + j) : -1;
      for (int k0 = b; k0 < en; k0 += B) {
        double g[B][4];
        double av[B];
#pragma unroll
        for (int j = 0; j < B; ++j)
          if (cu[j] >= 0) {
            ldg256(p + static_cast<long>(cu[j]) * D + c0, g[j]);
            av[j] = __ldg(aval + k0 + j);
          }
        int cn[B];
#pragma unroll
        for (int j = 0; j < B; ++j) cn[j] = k0 + B + j < en ? __ldg(acol + k0 + B + j) : -1;
#pragma unroll
        for (int j = 0; j < B; ++j)
          if (cu[j] >= 0)
#pragma unroll
            for (int k = 0; k < 4; ++k) acc[k] += av[j] * g[j][k];
#pragma unroll
        for (int j = 0; j < B; ++j) cu[j] = cn[j];
      }
      double* o = q + static_cast<long>(v) * D + c0;
      reinterpret_cast<double2*>(o)[0] = make_double2(acc[0], acc[1]);
      reinterpret_cast<double2*>(o)[1] = make_double2(acc[2], acc[3]);
    }
  }
}

// ---- V3: stream reference: reads aval/acol and p rows contiguously (what a
// perfectly local gather would cost), writes q.
__global__ void __launch_bounds__(256) v_stream(int n, const int* __restrict__ aptr, const int* __restrict__ acol,
                                               const double* __restrict__ aval, const double* __restrict__ p,
                                               double* __restrict__ q) {
  const long total = static_cast<long>(n) * 8;
  for (long e = static_cast<long>(blockIdx.x) * blockDim.x + threadIdx.x; e < total; e += static_cast<long>(gridDim.x) * blockDim.x) {
    const int v = static_cast<int>(e >> 3);
    const int c0 = static_cast<int>(e & 7) * 2;
    const int b = __ldg(aptr + v), en = __ldg(aptr + v + 1);
    double s = 0.0;
    for (int k = b + (c0 >> 1); k < en; k += 8) s += __ldg(aval + k) * static_cast<double>(__ldg(acol + k));
    const double2 pv = __ldg(reinterpret_cast<const double2*>(p + static_cast<long>(v) * D + c0));
    reinterpret_cast<double2*>(q + static_cast<long>(v) * D + c0)[0] = make_double2(pv.x + s, pv.y);
  }
}

// ---- V1: shared-memory gather ring.  A group of 8 lanes owns a contiguous
// vertex range, i.e. a contiguous stream of nonzeros [k0, k1).  Step t
// consumes nonzero t (landed in the ring L steps earlier) and issues the
// cp.async gather of nonzero t + L (its column index was itself copied into
// the index ring L steps earlier), so ~L row gathers per group are in flight
// without holding registers.
__device__ __forceinline__ void cp_async16(void* smem, const void* g) {
  const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.ca.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(g));
}
__device__ __forceinline__ void cp_async8(void* smem, const void* g) {
  const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(s), "l"(g));
}
__device__ __forceinline__ void cp_async4(void* smem, const void* g) {
  const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(s), "l"(g));
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

template <int L>
struct RingGeo {
  static constexpr int kGroups = 32;                              // 256 threads / 8 lanes
  static constexpr int kGather = L * 8 * 16;                      // [L][8] double2
  static constexpr int kVal = L * 8;                              // [L] double
  static constexpr int kIdx = 2 * L * 4;                          // [2L] int
  static constexpr int kPerGroup = kGather + kVal + kIdx;
  static constexpr int kBytes = kGroups * kPerGroup;
};

template <int L, int MINB, bool kBalance>
__global__ void __launch_bounds__(256, MINB) v_ring(int n, const int* __restrict__ aptr, const int* __restrict__ acol,
                                                   const double* __restrict__ aval, const double* __restrict__ p,
                                                   double* __restrict__ q) {
  using G = RingGeo<L>;
  extern __shared__ __align__(16) unsigned char smem[];
  const int grp = threadIdx.x >> 3, c = threadIdx.x & 7;
  unsigned char* base = smem + grp * G::kPerGroup;
  double2* gring = reinterpret_cast<double2*>(base);
  double* vring = reinterpret_cast<double*>(base + G::kGather);
  int* iring = reinterpret_cast<int*>(base + G::kGather + G::kVal);
  // block range (equal vertex counts), then the group's share
  const long vb0 = static_cast<long>(n) * blockIdx.x / gridDim.x, vb1 = static_cast<long>(n) * (blockIdx.x + 1) / gridDim.x;
  int v0, v1;
  if constexpr (kBalance) {
    // split the block's nonzeros evenly among the groups (vertex-aligned)
    const int kb0 = __ldg(aptr + vb0), kb1 = __ldg(aptr + vb1);
    auto find = [&](long target) {  // first vertex v in [vb0, vb1] with aptr[v] >= target
      long lo = vb0, hi = vb1;
      while (lo < hi) {
        const long mid = (lo + hi) >> 1;
        if (__ldg(aptr + mid) >= target) hi = mid; else lo = mid + 1;
      }
      return static_cast<int>(lo);
    };
    v0 = find(kb0 + (static_cast<long>(kb1 - kb0) * grp) / G::kGroups);
    v1 = find(kb0 + (static_cast<long>(kb1 - kb0) * (grp + 1)) / G::kGroups);
  } else {
    v0 = static_cast<int>(vb0 + (vb1 - vb0) * grp / G::kGroups);
    v1 = static_cast<int>(vb0 + (vb1 - vb0) * (grp + 1) / G::kGroups);
  }
  const int k0 = __ldg(aptr + v0), k1 = __ldg(aptr + v1);
  const int cnt = k1 - k0;
  // warp-uniform step count
  int steps = cnt;
#pragma unroll
  for (int o = 8; o < 32; o <<= 1) steps = max(steps, __shfl_xor_sync(0xffffffffu, steps, o));
  // prologue: indices of nonzeros [0, 2L), gathers of [0, L)
  if (c == 0)
    for (int t = 0; t < 2 * L; ++t)
      if (t < cnt) cp_async4(iring + t, acol + k0 + t);
  cp_commit();
  cp_wait<0>();
  __syncwarp();
  for (int t = 0; t < L; ++t) {
    if (t < cnt) {
      const int u = iring[t];
      cp_async16(gring + t * 8 + c, p + static_cast<long>(u) * D + 2 * c);
      if (c == 0) cp_async8(vring + t, aval + k0 + t);
    }
    cp_commit();
  }
  int v = v0;
  int kend = v < v1 ? __ldg(aptr + v + 1) - k0 : cnt;
  int knext = v + 1 < v1 ? __ldg(aptr + v + 2) - k0 : cnt;
  double q0 = 0.0, q1 = 0.0;
  for (int t = 0; t < steps; ++t) {
    cp_wait<L - 1>();
    __syncwarp();
    const int slot = t % L;
    if (t < cnt) {
      const double a = vring[slot];
      const double2 g = gring[slot * 8 + c];
      q0 += a * g.x;
      q1 += a * g.y;
      if (t + 1 == kend) {
        reinterpret_cast<double2*>(q + static_cast<long>(v) * D + 2 * c)[0] = make_double2(q0, q1);
        q0 = q1 = 0.0;
        ++v;
        // (no empty rows in A: the diagonal is always present)
        kend = knext;
        knext = v + 1 < v1 ? __ldg(aptr + v + 2) - k0 : cnt;
      }
    }
    __syncwarp();
    const int tn = t + L;
    if (tn < cnt) {
      const int u = iring[tn % (2 * L)];
      cp_async16(gring + slot * 8 + c, p + static_cast<long>(u) * D + 2 * c);
      if (c == 0) {
        cp_async8(vring + slot, aval + k0 + tn);
        if (tn + L < cnt) cp_async4(iring + (tn + L) % (2 * L), acol + k0 + tn + L);
      }
    }
    cp_commit();
  }
  cp_wait<0>();
}

}  // namespace

extern "C" {

// Storage order built from small breadth-first clusters: grow a cluster of
// up to C unassigned vertices by BFS from a seed, give them consecutive
// positions, take the next seed from a FIFO of the vertices discovered next
// to earlier clusters (so consecutive clusters stay adjacent), repeat.
// perm[v] = storage position of vertex v.
void lab_cluster_order(int n, const int* indptr, const int* indices, int C, int* perm) {
  std::vector<int> fifo;
  fifo.reserve(n);
  std::vector<char> queued(n, 0);
  for (int v = 0; v < n; ++v) perm[v] = -1;
  int next = 0;
  size_t head = 0;
  std::vector<int> cl;
  for (int s0 = 0; s0 < n; ++s0) {
    if (perm[s0] >= 0) continue;
    fifo.push_back(s0);
    queued[s0] = 1;
    while (head < fifo.size()) {
      const int seed = fifo[head++];
      if (perm[seed] >= 0) continue;
      // grow one cluster
      cl.clear();
      cl.push_back(seed);
      perm[seed] = next++;
      for (size_t h = 0; h < cl.size() && static_cast<int>(cl.size()) < C; ++h) {
        const int v = cl[h];
        for (int k = indptr[v]; k < indptr[v + 1] && static_cast<int>(cl.size()) < C; ++k) {
          const int u = indices[k];
          if (perm[u] < 0) {
            perm[u] = next++;
            cl.push_back(u);
          }
        }
      }
      // the cluster's unassigned neighbours seed the next clusters
      for (int v : cl)
        for (int k = indptr[v]; k < indptr[v + 1]; ++k) {
          const int u = indices[k];
          if (perm[u] < 0 && !queued[u]) {
            queued[u] = 1;
            fifo.push_back(u);
          }
        }
    }
  }
}

// variant ids: 0..3 registers (B, minBlocks) = (8,2) (8,3) (4,4) (12,2);
// 10.. ring: L in {8, 16, 24, 32} x balance
int lab_spmv(int variant, int n, const int* aptr, const int* acol, const double* aval, const double* p, double* q,
             int reps, float* ms_out) {
  int dev = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  auto launch = [&]() -> int {
    int nb = 0;
    switch (variant) {
#define REGS(id, B, M)                                                              \
  case id:                                                                          \
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, v_regs<B, M>, 256, 0);       \
    v_regs<B, M><<<sms * nb, 256>>>(n, aptr, acol, aval, p, q);                     \
    return nb;
      REGS(0, 8, 2)
      REGS(1, 8, 3)
      REGS(2, 4, 4)
      REGS(3, 12, 2)
      REGS(4, 16, 1)
#define REGS4(id, B, M)                                                             \
  case id:                                                                          \
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, v_regs4<B, M>, 256, 0);      \
    v_regs4<B, M><<<sms * nb, 256>>>(n, aptr, acol, aval, p, q);                    \
    return nb;
      REGS4(5, 4, 3)
      REGS4(6, 8, 2)
      REGS4(7, 4, 4)
#define SWEEP(id, B, M, CH)                                                          \
  case id:                                                                           \
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, v_sweep4<B, M, CH>, 256, 0);  \
    v_sweep4<B, M, CH><<<sms * nb, 256>>>(n, aptr, acol, aval, p, q);                \
    return nb;
      SWEEP(20, 4, 3, 64)
      SWEEP(21, 4, 3, 16)
      SWEEP(22, 4, 3, 256)
      SWEEP(23, 4, 4, 64)
      SWEEP(24, 8, 2, 64)
      case 9:
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, v_stream, 256, 0);
        v_stream<<<sms * nb, 256>>>(n, aptr, acol, aval, p, q);
        return nb;
#define RING(id, L, M, BAL)                                                                                  \
  case id: {                                                                                                 \
    constexpr int sm = RingGeo<L>::kBytes;                                                                   \
    cudaFuncSetAttribute(v_ring<L, M, BAL>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm);                 \
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, v_ring<L, M, BAL>, 256, sm);                          \
    if (nb < 1) return -1;                                                                                   \
    v_ring<L, M, BAL><<<sms * nb, 256, sm>>>(n, aptr, acol, aval, p, q);                                     \
    return nb;                                                                                               \
  }
      RING(10, 8, 4, false)
      RING(11, 16, 2, false)
      RING(12, 16, 3, false)
      RING(13, 24, 2, false)
      RING(14, 16, 2, true)
      RING(15, 24, 2, true)
      RING(16, 12, 3, true)
      RING(17, 32, 1, true)
      default:
        return -2;
    }
  };
  int nb = launch();
  if (nb < 0) return nb;
  cudaDeviceSynchronize();
  cudaEventRecord(e0);
  for (int r = 0; r < reps; ++r) launch();
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms = 0.f;
  cudaEventElapsedTime(&ms, e0, e1);
  *ms_out = reps > 0 ? ms / reps : 0.f;
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  const cudaError_t err = cudaGetLastError();
  if (err != cudaSuccess) {
    std::fprintf(stderr, "lab_spmv variant %d: %s\n", variant, cudaGetErrorString(err));
    return -3;
  }
  return nb;
}
}
