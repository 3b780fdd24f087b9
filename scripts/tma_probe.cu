// TMA box probe (NOT product code): loads one halo box of a [H][W][K] fp64
// array with cp.async.bulk.tensor into shared memory, for the box shapes the
// persistent grid kernel uses (8-neighbour: R = 1, 5x5: R = 2), at interior
// and edge positions (negative / past-the-edge coordinates are zero filled),
// and compares with the expected box.  Prints one line per case before
// launching it, so a faulting case is the last line printed.
//
// nvcc -O2 -gencode arch=compute_100a,code=sm_100a scripts/tma_probe.cu -o scripts/tma_probe -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <string>
#include <vector>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }

template <int DIMS>
__global__ void k_probe(const __grid_constant__ CUtensorMap m, int x, int y, int bytes, double* out, int count,
                        int dst_off) {
  extern __shared__ __align__(1024) double sm[];
  __shared__ alignas(8) uint64_t bar;
  double* dst = sm + dst_off;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(smem_u32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(&bar)), "r"(bytes) : "memory");
    if constexpr (DIMS == 3)
      asm volatile(
          "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];\n" ::"r"(
              smem_u32(dst)),
          "l"(reinterpret_cast<uint64_t>(&m)), "r"(0), "r"(x), "r"(y), "r"(smem_u32(&bar))
          : "memory");
    else
      asm volatile(
          "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];\n" ::"r"(
              smem_u32(dst)),
          "l"(reinterpret_cast<uint64_t>(&m)), "r"(x), "r"(y), "r"(smem_u32(&bar))
          : "memory");
  }
  asm volatile(
      "{\n.reg .pred p;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n@!p bra W_%=;\n}\n" ::"r"(
          smem_u32(&bar))
      : "memory");
  for (int i = threadIdx.x; i < count; i += blockDim.x) out[i] = dst[i];
}

int main(int argc, char** argv) {
  // argv[1]: run only case i (a fault kills the context, so the driver
  // script runs every case in its own process); "count": print the count
  const int H = 64, W = 96;
  struct Case {
    int K, bw, bh, x, y, dst_off;
  };
  std::vector<Case> cases;
  for (int K : {1, 2, 4, 8})
    for (int bw : {32, 33, 34, 35, 36, 38, 40})
      cases.push_back({K, bw, 6, -1, -1, 0});
  // box heights 1..16 (2-D and 3-D) and the interior boxes of the tiles
  for (int K : {1, 4, 8})
    for (int bh = 1; bh <= 16; ++bh) cases.push_back({K, 32, bh, 0, 0, 0});
  for (int K : {1, 4, 8})
    for (int bh : {4, 8}) cases.push_back({K, 32, bh, 32, 16, 0});
  for (int K : {1, 4, 8, 12, 32})
    for (int R : {1, 2})
      for (int TH : {4, 8}) {
        const int bw = 32 + 2 * R, bh = TH + 2 * R;
        for (int pos = 0; pos < 3; ++pos) {
          const int x = pos == 0 ? -R : (pos == 1 ? 32 - R : W - 32 - R);
          const int y = pos == 0 ? -R : (pos == 1 ? 16 - R : H - TH - R);
          cases.push_back({K, bw, bh, x, y, 0});
        }
        cases.push_back({K, bw, bh, -R, -R, 16 * 27});  // a non-zero 128-byte aligned destination offset
      }
  if (argc > 1 && std::string(argv[1]) == "count") {
    std::printf("%zu\n", cases.size());
    return 0;
  }
  const int only = argc > 1 ? std::atoi(argv[1]) : -1;
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q{};
  if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess || !fn) {
    std::printf("no cuTensorMapEncodeTiled\n");
    return 1;
  }
  auto enc = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);

  std::vector<double> host(static_cast<size_t>(H) * W * 32);
  for (size_t i = 0; i < host.size(); ++i) host[i] = 1.0 + static_cast<double>(i);
  double *dsrc = nullptr, *dout = nullptr;
  cudaMalloc(&dsrc, host.size() * sizeof(double));
  cudaMalloc(&dout, 1 << 22);
  cudaFuncSetAttribute(k_probe<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  cudaFuncSetAttribute(k_probe<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  int fails = 0;
  for (size_t ci = 0; ci < cases.size(); ++ci) {
    if (only >= 0 && static_cast<int>(ci) != only) continue;
    const Case& c = cases[ci];
    cudaMemcpy(dsrc, host.data(), sizeof(double) * H * W * c.K, cudaMemcpyHostToDevice);
    CUtensorMap m;
    const cuuint32_t es[3] = {1, 1, 1};
    CUresult r;
    if (c.K == 1) {
      const cuuint64_t dims[2] = {static_cast<cuuint64_t>(W), static_cast<cuuint64_t>(H)};
      const cuuint64_t strides[1] = {static_cast<cuuint64_t>(W) * 8};
      const cuuint32_t box[2] = {static_cast<cuuint32_t>(c.bw), static_cast<cuuint32_t>(c.bh)};
      r = enc(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, dsrc, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
              CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    } else {
      const cuuint64_t dims[3] = {static_cast<cuuint64_t>(c.K), static_cast<cuuint64_t>(W), static_cast<cuuint64_t>(H)};
      const cuuint64_t strides[2] = {static_cast<cuuint64_t>(c.K) * 8, static_cast<cuuint64_t>(W) * c.K * 8};
      const cuuint32_t box[3] = {static_cast<cuuint32_t>(c.K), static_cast<cuuint32_t>(c.bw), static_cast<cuuint32_t>(c.bh)};
      r = enc(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, dsrc, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
              CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    }
    const int count = c.K * c.bw * c.bh;
    std::printf("K=%2d box %dx%d at (%d,%d) dst+%d: encode %d ... ", c.K, c.bw, c.bh, c.x, c.y, c.dst_off * 8,
                static_cast<int>(r));
    std::fflush(stdout);
    if (r != CUDA_SUCCESS) {
      std::printf("ENCODE FAILED\n");
      ++fails;
      continue;
    }
    const size_t smem = static_cast<size_t>(count + c.dst_off) * 8 + 1024;
    if (c.K == 1)
      k_probe<2><<<1, 128, smem>>>(m, c.x, c.y, count * 8, dout, count, c.dst_off);
    else
      k_probe<3><<<1, 128, smem>>>(m, c.x, c.y, count * 8, dout, count, c.dst_off);
    const cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) {
      std::printf("FAULT: %s\n", cudaGetErrorString(e));
      return 2;
    }
    std::vector<double> got(count);
    cudaMemcpy(got.data(), dout, sizeof(double) * count, cudaMemcpyDeviceToHost);
    int bad = 0;
    for (int by = 0; by < c.bh; ++by)
      for (int bx = 0; bx < c.bw; ++bx)
        for (int k = 0; k < c.K; ++k) {
          const int yy = c.y + by, xx = c.x + bx;
          const double want = (yy >= 0 && yy < H && xx >= 0 && xx < W) ? host[(static_cast<size_t>(yy) * W + xx) * c.K + k] : 0.0;
          if (got[(by * c.bw + bx) * c.K + k] != want) ++bad;
        }
    std::printf("%s (%d mismatches)\n", bad ? "WRONG" : "ok", bad);
    fails += bad != 0;
  }
  std::printf("%d failing cases of %zu\n", fails, cases.size());
  return fails ? 3 : 0;
}
