// Latency / throughput probes of the fp64 and shared-memory paths on this GPU:
// dependent DFMA chain latency, DFMA throughput of one warp with k independent
// chains, LDS.64 round-trip latency, and shfl latency.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o lat_probe lat_probe.cu && ./lat_probe
#include <cstdio>
#include <cuda_runtime.h>

template <int K>
__global__ void k_dfma(double* out, long long* cyc, int iters, double a, double b) {
  double v[K];
#pragma unroll
  for (int k = 0; k < K; ++k) v[k] = threadIdx.x + k;
  __syncwarp();
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < K; ++k) v[k] = fma(v[k], a, b);
  }
  long long t1 = clock64();
  double s = 0;
#pragma unroll
  for (int k = 0; k < K; ++k) s += v[k];
  out[threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

__global__ void k_lds(double* out, long long* cyc, int iters) {
  __shared__ long long buf[1024];
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) buf[i] = (i * 7 + 1) & 1023;
  __syncthreads();
  long long idx = threadIdx.x;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) idx = buf[idx];
  long long t1 = clock64();
  out[threadIdx.x] = (double)idx;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

__global__ void k_shfl(double* out, long long* cyc, int iters) {
  double v = threadIdx.x;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) v = __shfl_sync(0xffffffffu, v, (threadIdx.x + 1) & 31) + 1.0;
  long long t1 = clock64();
  out[threadIdx.x] = v;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

int main() {
  double* out;
  long long* cyc;
  cudaMalloc(&out, 1 << 20);
  cudaMalloc(&cyc, 1 << 16);
  long long h;
  const int it = 4096;
  auto run = [&](const char* name, auto kern, int threads, double per) {
    kern<<<1, threads>>>(out, cyc, it, 1.0000001, 1e-9);
    cudaDeviceSynchronize();
    kern<<<1, threads>>>(out, cyc, it, 1.0000001, 1e-9);
    cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
    printf("%-28s threads %4d  cycles/iter %.2f  cycles/op %.2f\n", name, threads, (double)h / it, (double)h / it / per);
  };
  run("dfma 1 chain", k_dfma<1>, 32, 1);
  run("dfma 2 chains", k_dfma<2>, 32, 2);
  run("dfma 4 chains", k_dfma<4>, 32, 4);
  run("dfma 8 chains", k_dfma<8>, 32, 8);
  run("dfma 16 chains", k_dfma<16>, 32, 16);
  run("dfma 8 chains 4 warps", k_dfma<8>, 128, 8);
  run("dfma 8 chains 8 warps", k_dfma<8>, 256, 8);
  run("dfma 16 chains 4 warps", k_dfma<16>, 128, 16);
  k_lds<<<1, 32>>>(out, cyc, it);
  k_lds<<<1, 32>>>(out, cyc, it);
  cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
  printf("%-28s cycles/iter %.2f\n", "lds.64 dependent chain", (double)h / it);
  k_shfl<<<1, 32>>>(out, cyc, it);
  k_shfl<<<1, 32>>>(out, cyc, it);
  cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
  printf("%-28s cycles/iter %.2f\n", "shfl.f64 + dadd chain", (double)h / it);
  return 0;
}
