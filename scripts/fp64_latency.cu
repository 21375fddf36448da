// Microbenchmark: latency of dependent DFMA / DMUL / DADD chains and LDS on
// this GPU (one warp), and throughput with k independent chains per warp.
#include <cstdio>
#include <cuda_runtime.h>

__global__ void chain(double* out, long long* cyc, int iters, double a, double b)
{
  double x = threadIdx.x * 1e-3;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < 16; ++u) x = fma(x, a, b);
  }
  long long t1 = clock64();
  out[threadIdx.x] = x;
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
}

template <int K>
__global__ void multi(double* out, long long* cyc, int iters, double a, double b)
{
  double x[K];
#pragma unroll
  for (int k = 0; k < K; ++k) x[k] = threadIdx.x * 1e-3 + k;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < 16; ++u)
#pragma unroll
      for (int k = 0; k < K; ++k) x[k] = fma(x[k], a, b);
  }
  long long t1 = clock64();
  double s = 0;
#pragma unroll
  for (int k = 0; k < K; ++k) s += x[k];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0 && blockIdx.x == 0) cyc[0] = t1 - t0;
}

__global__ void lds_chain(double* out, long long* cyc, int iters)
{
  __shared__ int idx[1024];
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) idx[i] = (i + 33) & 1023;
  __syncthreads();
  int p = threadIdx.x;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) p = idx[p];
  long long t1 = clock64();
  out[threadIdx.x] = p;
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
}

int main()
{
  double* d;
  long long* c;
  cudaMalloc(&d, 1 << 20);
  cudaMalloc(&c, 64);
  long long h;
  const int it = 1000;
  chain<<<1, 32>>>(d, c, it, 1.0000001, 1e-9);
  chain<<<1, 32>>>(d, c, it, 1.0000001, 1e-9);
  cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
  printf("DFMA dependent latency: %.2f cycles\n", (double)h / (it * 16));
#define M(K, W)                                                                      \
  multi<K><<<1, 32 * W>>>(d, c, it, 1.0000001, 1e-9);                                \
  cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);                                     \
  printf("warps/SM %2d chains/warp %d: %.2f cycles per chain step (%.2f DFMA/clk/SM)\n", W, K, \
         (double)h / (it * 16), (double)K * W * 32 * it * 16 / h);
  M(1, 1) M(2, 1) M(4, 1) M(8, 1) M(1, 4) M(2, 4) M(4, 4) M(1, 8) M(2, 8) M(4, 8) M(1, 16) M(2, 16)
  M(1, 32) M(2, 32) M(4, 32)
  lds_chain<<<1, 32>>>(d, c, it);
  cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
  printf("LDS dependent latency: %.2f cycles\n", (double)h / it);
  return 0;
}
