// DMMA throughput vs warps/SM and independent accumulator chains, with
// operands from registers (R) or loaded from shared memory per k-step (S).
#include <cstdio>
#include <cuda_runtime.h>
template <int C, bool SMEM>
__global__ void k(double* out, int iters) {
  __shared__ double sa[64 * 8], sb[64 * 8];
  for (int i = threadIdx.x; i < 512; i += blockDim.x) { sa[i] = i * 1e-3; sb[i] = 1.0 + i * 1e-4; }
  __syncthreads();
  double a = threadIdx.x * 1e-3, b = 1.0 + threadIdx.x * 1e-4;
  double c[C][2];
  for (int i = 0; i < C; ++i) c[i][0] = c[i][1] = i;
  const int lane = threadIdx.x & 31;
  for (int it = 0; it < iters; ++it) {
    if (SMEM) { b = sb[(it & 63) * 8 + (lane & 7)]; }
#pragma unroll
    for (int i = 0; i < C; ++i) {
      double ai = SMEM ? sa[((it + i) & 63) * 8 + (lane >> 2)] : a;
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(ai), "d"(b));
    }
  }
  double s = 0;
  for (int i = 0; i < C; ++i) s += c[i][0] + c[i][1];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
template <int C, bool SMEM>
void run(int warps_per_sm, double* d, int sms) {
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int threads = 32 * (warps_per_sm > 16 ? warps_per_sm / 2 : warps_per_sm);
  int bps = warps_per_sm > 16 ? 2 : 1;
  int blocks = sms * bps;
  int iters = 4000;
  k<C, SMEM><<<blocks, threads>>>(d, 10);
  cudaEventRecord(e0);
  k<C, SMEM><<<blocks, threads>>>(d, iters);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  double fl = 2.0 * 256 * C * (double)iters * blocks * threads / 32;
  printf("%s warps/SM=%2d chains=%d  %.2f TF/s\n", SMEM ? "S" : "R", warps_per_sm, C, fl / ms / 1e9);
}
int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* d; cudaMalloc(&d, 1 << 24);
  for (int w : {4, 8, 12, 16, 32}) {
    run<1, false>(w, d, sms); run<2, false>(w, d, sms); run<3, false>(w, d, sms); run<4, false>(w, d, sms); run<8, false>(w, d, sms);
    run<1, true>(w, d, sms); run<2, true>(w, d, sms); run<3, true>(w, d, sms); run<4, true>(w, d, sms); run<8, true>(w, d, sms);
  }
  return 0;
}
