// DMMA latency, F2F.F64.F32 throughput, and DMMA throughput when each DMMA's
// A operand is converted from fp32 (the pass kernel's pattern).
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k_lat(double* out, long long* cyc, int iters) {
  double c[2] = {1.0, 2.0};
  double a = threadIdx.x * 1e-3, b = 1.0;
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it)
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                 : "+d"(c[0]), "+d"(c[1]) : "d"(a), "d"(b));
  long long t1 = clock64();
  if (threadIdx.x == 0) *cyc = t1 - t0;
  out[threadIdx.x] = c[0] + c[1];
}
template <int C>
__global__ void k_f2f(double* out, const float* in, int iters) {
  __shared__ float sx[1024];
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) sx[i] = in[i];
  __syncthreads();
  double c[C][2];
  for (int i = 0; i < C; ++i) c[i][0] = c[i][1] = i;
  double b = 1.0 + threadIdx.x * 1e-4;
  const int lane = threadIdx.x & 31;
  for (int it = 0; it < iters; ++it) {
    const double a = (double)sx[((it * 4) & 1023) ^ lane];
#pragma unroll
    for (int i = 0; i < C; ++i)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
  }
  double s = 0;
  for (int i = 0; i < C; ++i) s += c[i][0] + c[i][1];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void k_cvt(double* out, const float* in, int iters) {
  __shared__ float sx[1024];
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) sx[i] = in[i];
  __syncthreads();
  double s0 = 0, s1 = 0, s2 = 0, s3 = 0;
  const int lane = threadIdx.x & 31;
  for (int it = 0; it < iters; ++it) {
    float f = sx[((it * 4) & 1023) ^ lane];
    s0 += (double)f; s1 += (double)(f + 1.f); s2 += (double)(f + 2.f); s3 += (double)(f + 3.f);
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = s0 + s1 + s2 + s3;
}
int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* d; cudaMalloc(&d, 1 << 24);
  float* f; cudaMalloc(&f, 4096 * 4); cudaMemset(f, 0, 4096 * 4);
  long long* cyc; cudaMalloc(&cyc, 8);
  k_lat<<<1, 32>>>(d, cyc, 1000); cudaDeviceSynchronize();
  long long h; cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
  printf("DMMA dependent-chain latency: %.1f cycles\n", h / 1000.0);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int warps : {8, 16}) {
    int iters = 4000;
    k_f2f<3><<<sms, warps * 32>>>(d, f, 10);
    cudaEventRecord(e0); k_f2f<3><<<sms, warps * 32>>>(d, f, iters); cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    printf("DMMA with F2F operand, %d warps/SM, 3 chains: %.2f TF/s\n", warps, 2.0 * 256 * 3 * iters * (double)sms * warps / ms / 1e9);
    k_cvt<<<sms, warps * 32>>>(d, f, 10);
    cudaEventRecord(e0); k_cvt<<<sms, warps * 32>>>(d, f, iters); cudaEventRecord(e1); cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    printf("F2F.F64.F32 + DADD: %d warps/SM: %.3f G cvt-add pairs/s per SM\n", warps, 4.0 * iters * warps * 32 * sms / ms / 1e6 / sms);
  }
  return 0;
}
