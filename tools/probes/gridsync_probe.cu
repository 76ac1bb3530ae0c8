// Grid-barrier cost on this GPU: cooperative_groups grid.sync() vs a
// flag barrier, K barriers per launch, for several grid sizes.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o gridsync_probe gridsync_probe.cu
#include <cooperative_groups.h>
#include <cstdio>
namespace cg = cooperative_groups;

__global__ void k_cg(int iters, double* sink) {
  cg::grid_group g = cg::this_grid();
  double s = 0;
  for (int i = 0; i < iters; ++i) {
    s += i;
    g.sync();
  }
  if (s == -1) sink[0] = s;
}

__device__ unsigned ldacq(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
// monotonic arrival counter, each CTA waits for count >= (epoch+1)*grid
__global__ void k_flag(int iters, unsigned* ctr, double* sink) {
  double s = 0;
  for (int i = 0; i < iters; ++i) {
    s += i;
    __syncthreads();
    if (threadIdx.x == 0) {
      __threadfence();
      atomicAdd(ctr, 1u);
      const unsigned target = (unsigned)(i + 1) * gridDim.x;
      while (ldacq(ctr) < target) __nanosleep(32);
    }
    __syncthreads();
  }
  if (s == -1) sink[0] = s;
}

int main() {
  double* sink;
  unsigned* ctr;
  cudaMalloc(&sink, 8);
  cudaMalloc(&ctr, 4);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int iters = 1000;
  for (int grid : {1, 8, 35, 74, 148}) {
    for (int variant = 0; variant < 2; ++variant) {
      float best = 1e9;
      for (int rep = 0; rep < 3; ++rep) {
        cudaMemset(ctr, 0, 4);
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(grid);
        cfg.blockDim = dim3(256);
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeCooperative;
        at[0].val.cooperative = 1;
        cfg.attrs = at;
        cfg.numAttrs = 1;
        cudaEventRecord(e0);
        cudaError_t err = variant == 0 ? cudaLaunchKernelEx(&cfg, k_cg, iters, sink)
                                       : cudaLaunchKernelEx(&cfg, k_flag, iters, ctr, sink);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        if (err != cudaSuccess) printf("launch error %s\n", cudaGetErrorString(err));
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        if (ms < best) best = ms;
      }
      printf("grid %3d %-10s %.3f us per barrier\n", grid, variant == 0 ? "grid.sync" : "flag", best * 1e3 / iters);
    }
  }
  return 0;
}
