// Development probe: fp64 latencies on the B200 (DFMA chain, DMMA chain, DMMA
// throughput per SMSP with k independent chains, DFMA/DMMA co-issue).
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void dmma(double (&d)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(d[0]), "+d"(d[1]) : "d"(a), "d"(b));
}

__global__ void dfma_chain(double* out, long long* cyc, int n) {
  double x = threadIdx.x * 1e-3, y = 1.0000001;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) x = fma(x, y, 1e-9);
  long long t1 = clock64();
  out[threadIdx.x] = x;
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
}

template <int C>
__global__ void dmma_chains(double* out, long long* cyc, int n) {
  double acc[C][2];
  for (int c = 0; c < C; ++c) acc[c][0] = acc[c][1] = 0.0;
  double a = 1.0 + threadIdx.x * 1e-6, b = 1.0 - threadIdx.x * 1e-6;
  __syncwarp();
  long long t0 = clock64();
  for (int i = 0; i < n; ++i)
#pragma unroll
    for (int c = 0; c < C; ++c) dmma(acc[c], a, b);
  long long t1 = clock64();
  double s = 0;
  for (int c = 0; c < C; ++c) s += acc[c][0] + acc[c][1];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

int main() {
  double* out; long long* cyc;
  cudaMalloc(&out, 1 << 20); cudaMalloc(&cyc, 4096);
  long long h[64];
  const int n = 4096;
  dfma_chain<<<1, 32>>>(out, cyc, n); cudaDeviceSynchronize();
  cudaMemcpy(h, cyc, 8, cudaMemcpyDeviceToHost);
  printf("DFMA dependent chain: %.1f cyc/op\n", double(h[0]) / n);
  // one warp per SMSP (block of 32 threads -> one warp), chains C
#define RUN(C, W)                                                                          \
  dmma_chains<C><<<1, 32 * W>>>(out, cyc, n); cudaDeviceSynchronize();                     \
  cudaMemcpy(h, cyc, 8, cudaMemcpyDeviceToHost);                                           \
  printf("DMMA %d warps x %d chains: %.1f cyc per DMMA per warp-chain step, %.2f cyc/DMMA per SM\n", W, C, \
         double(h[0]) / n, double(h[0]) / (n * (double)C * W));
  RUN(1, 1) RUN(2, 1) RUN(4, 1) RUN(8, 1) RUN(1, 4) RUN(2, 4) RUN(4, 4) RUN(8, 4) RUN(2, 8) RUN(4, 8) RUN(3, 8) RUN(6, 8) RUN(4, 16)
  return 0;
}
