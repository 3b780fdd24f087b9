// Microbenchmark: cost of a grid-wide barrier (cooperative groups vs a
// sense-reversing atomic barrier) and of back-to-back dependent kernel
// launches on this GPU.  Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mb microbench_sync.cu
#include <cooperative_groups.h>
#include <cstdio>

namespace cg = cooperative_groups;

__global__ void k_cg(int iters, double* sink) {
  cg::grid_group grid = cg::this_grid();
  double acc = 0;
  for (int i = 0; i < iters; ++i) {
    acc += i * 1e-9;
    grid.sync();
  }
  if (acc < 0) sink[0] = acc;
}

__device__ unsigned g_count = 0;
__device__ volatile unsigned g_gen = 0;

__device__ __forceinline__ void bar(unsigned nb) {
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned gen = g_gen;
    __threadfence();
    if (atomicAdd(&g_count, 1u) == nb - 1) {
      g_count = 0;
      __threadfence();
      g_gen = gen + 1;
    } else {
      while (g_gen == gen) {
      }
    }
    __threadfence();
  }
  __syncthreads();
}

__global__ void k_atomic(int iters, double* sink) {
  double acc = 0;
  for (int i = 0; i < iters; ++i) {
    acc += i * 1e-9;
    bar(gridDim.x);
  }
  if (acc < 0) sink[0] = acc;
}

__global__ void k_empty(double* sink) {
  if (threadIdx.x == 1023) sink[0] = 1;
}

int main() {
  int sm = 0;
  cudaDeviceGetAttribute(&sm, cudaDevAttrMultiProcessorCount, 0);
  double* sink;
  cudaMalloc(&sink, 8);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (int per : {1, 2, 4}) {
    int iters = 2000;
    void* args[] = {&iters, &sink};
    const int nb = sm * per;
    cudaLaunchCooperativeKernel((void*)k_cg, nb, 256, args, 0, 0);
    cudaEventRecord(a);
    cudaLaunchCooperativeKernel((void*)k_cg, nb, 256, args, 0, 0);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    std::printf("cg grid.sync     blocks=%4d : %.3f us per barrier (%s)\n", nb, 1e3 * ms / iters,
                cudaGetErrorString(cudaGetLastError()));
    cudaLaunchCooperativeKernel((void*)k_atomic, nb, 256, args, 0, 0);
    cudaEventRecord(a);
    cudaLaunchCooperativeKernel((void*)k_atomic, nb, 256, args, 0, 0);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    cudaEventElapsedTime(&ms, a, b);
    std::printf("atomic barrier   blocks=%4d : %.3f us per barrier (%s)\n", nb, 1e3 * ms / iters,
                cudaGetErrorString(cudaGetLastError()));
  }
  for (int nb : {148, 592, 1184}) {
    cudaStream_t s;
    cudaStreamCreate(&s);
    for (int i = 0; i < 10; ++i) k_empty<<<nb, 256, 0, s>>>(sink);
    cudaEventRecord(a, s);
    for (int i = 0; i < 1000; ++i) k_empty<<<nb, 256, 0, s>>>(sink);
    cudaEventRecord(b, s);
    cudaEventSynchronize(b);
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    std::printf("stream launches  blocks=%4d : %.3f us per empty kernel\n", nb, 1e3 * ms / 1000);
    // graph of 1000 launches
    cudaGraph_t g;
    cudaGraphExec_t ge;
    cudaStreamBeginCapture(s, cudaStreamCaptureModeRelaxed);
    for (int i = 0; i < 1000; ++i) k_empty<<<nb, 256, 0, s>>>(sink);
    cudaStreamEndCapture(s, &g);
    cudaGraphInstantiate(&ge, g, 0);
    cudaGraphLaunch(ge, s);
    cudaEventRecord(a, s);
    cudaGraphLaunch(ge, s);
    cudaEventRecord(b, s);
    cudaEventSynchronize(b);
    cudaEventElapsedTime(&ms, a, b);
    std::printf("graph launches   blocks=%4d : %.3f us per empty kernel\n", nb, 1e3 * ms / 1000);
  }
  return 0;
}
