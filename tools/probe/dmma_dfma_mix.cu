// Does scalar fp64 work share the pipe with DMMA?  Warps [0, Wm) run DMMA
// (register operands, 4 chains), warps [Wm, Wm+Wf) run DFMA (8 chains); each
// group's issue rate is timed alone and together.
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k(double* out, long long* cyc, int wm, int wf, int it_m, int it_f) {
  const int w = threadIdx.x >> 5;
  long long t0 = clock64();
  double s = 0;
  if (w < wm) {
    double c[4][2];
    for (int i = 0; i < 4; ++i) c[i][0] = c[i][1] = i;
    double a = threadIdx.x * 1e-3, b = 1.0 + threadIdx.x * 1e-4;
    for (int it = 0; it < it_m; ++it)
#pragma unroll
      for (int i = 0; i < 4; ++i)
        asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                     : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
    for (int i = 0; i < 4; ++i) s += c[i][0] + c[i][1];
  } else if (w < wm + wf) {
    double c[8];
    for (int i = 0; i < 8; ++i) c[i] = threadIdx.x * 1e-3 + i;
    for (int it = 0; it < it_f; ++it)
#pragma unroll
      for (int i = 0; i < 8; ++i) c[i] = fma(c[i], 0.999999, 1e-9);
    for (int i = 0; i < 8; ++i) s += c[i];
  }
  long long t1 = clock64();
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if ((threadIdx.x & 31) == 0 && blockIdx.x == 0) cyc[w] = t1 - t0;
}

int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* d;
  long long* cyc;
  cudaMalloc(&d, 1 << 24);
  cudaMalloc(&cyc, 64 * 8);
  const int it_m = 4000, it_f = 8000;
  struct Case { int wm, wf; };
  for (Case cs : {Case{8, 0}, Case{0, 8}, Case{8, 8}, Case{8, 4}, Case{8, 2}}) {
    k<<<sms, 32 * (cs.wm + cs.wf)>>>(d, cyc, cs.wm, cs.wf, 10, 10);
    k<<<sms, 32 * (cs.wm + cs.wf)>>>(d, cyc, cs.wm, cs.wf, it_m, it_f);
    cudaDeviceSynchronize();
    long long h[64];
    cudaMemcpy(h, cyc, 64 * 8, cudaMemcpyDeviceToHost);
    double dm = 0, df = 0;
    for (int w = 0; w < cs.wm; ++w) dm = h[w] > dm ? h[w] : dm;
    for (int w = cs.wm; w < cs.wm + cs.wf; ++w) df = h[w] > df ? h[w] : df;
    // DMMA: 4 per iteration per warp; DFMA: 8 warp-instructions per iteration per warp
    printf("DMMA warps %d, DFMA warps %d:  DMMA %.1f cycles/DMMA/SMSP   DFMA %.2f warp-instr/cycle/SM\n", cs.wm, cs.wf,
           cs.wm ? dm / (4.0 * it_m * cs.wm / 4) : 0.0, cs.wf ? (8.0 * it_f * cs.wf) / df : 0.0);
  }
  return 0;
}
