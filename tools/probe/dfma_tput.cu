// Scalar FP64 throughput (DFMA, DADD, DMUL) on every SM: 8 independent chains
// per thread, W warps per SM; prints TFLOP/s-equivalent and lanes/cycle/SM.
#include <cstdio>
#include <cuda_runtime.h>

template <int OP>
__global__ void k(double* out, int iters, double s) {
  double c[8];
  for (int i = 0; i < 8; ++i) c[i] = threadIdx.x * 1e-3 + i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (OP == 0) c[i] = fma(c[i], s, 1e-9);
      if (OP == 1) c[i] = c[i] + s;
      if (OP == 2) c[i] = c[i] * s;
    }
  }
  double t = 0;
  for (int i = 0; i < 8; ++i) t += c[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = t;
}

int main() {
  int sms, clk;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  double* d;
  cudaMalloc(&d, 1 << 26);
  const char* nm[3] = {"DFMA", "DADD", "DMUL"};
  for (int op = 0; op < 3; ++op)
    for (int w : {4, 8, 16, 32}) {
      void (*kern)(double*, int, double) = op == 0 ? k<0> : op == 1 ? k<1> : k<2>;
      const int iters = 20000;
      kern<<<sms, 32 * w>>>(d, 100, 0.999999);
      cudaEvent_t a, b;
      cudaEventCreate(&a);
      cudaEventCreate(&b);
      cudaEventRecord(a);
      kern<<<sms, 32 * w>>>(d, iters, 0.999999);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      const double ops = 8.0 * iters * sms * 32 * w;
      const double lanes_per_cycle = ops / (ms * 1e-3) / sms / (clk * 1e3);
      printf("%s warps/SM=%2d  %.2f Gop/s  %.1f lanes/cycle/SM (at %d MHz nominal)\n", nm[op], w, ops / ms / 1e6,
             lanes_per_cycle, clk / 1000);
    }
  return 0;
}
