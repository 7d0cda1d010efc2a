// Is the scalar-fp64 starvation under DMMA load a per-SMSP effect?  Warp w runs on
// SM sub-partition w % 4.  role[w]: 0 idle, 1 DMMA (4 chains), 2 DFMA throughput
// (8 chains), 3 DFMA latency (1 dependent chain, like the update's exp chain).
// Compares the mixed layout of k_pass (DMMA and scalar warps on every SMSP) with
// a split one (SMSPs 0-2 DMMA only, SMSP 3 scalar only).
#include <cstdio>
#include <cuda_runtime.h>

struct Roles { int r[16]; };

__global__ void k(double* out, long long* cyc, Roles ro, int it_m, int it_f) {
  const int w = threadIdx.x >> 5;
  const int role = ro.r[w];
  long long t0 = clock64();
  double s = 0;
  if (role == 1) {
    double c[4][2];
    for (int i = 0; i < 4; ++i) c[i][0] = c[i][1] = i;
    double a = threadIdx.x * 1e-3, b = 1.0 + threadIdx.x * 1e-4;
    for (int it = 0; it < it_m; ++it)
#pragma unroll
      for (int i = 0; i < 4; ++i)
        asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                     : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
    for (int i = 0; i < 4; ++i) s += c[i][0] + c[i][1];
  } else if (role == 2) {
    double c[8];
    for (int i = 0; i < 8; ++i) c[i] = threadIdx.x * 1e-3 + i;
    for (int it = 0; it < it_f; ++it)
#pragma unroll
      for (int i = 0; i < 8; ++i) c[i] = fma(c[i], 0.999999, 1e-9);
    for (int i = 0; i < 8; ++i) s += c[i];
  } else if (role == 3) {
    double c = threadIdx.x * 1e-3;
    for (int it = 0; it < it_f; ++it)
#pragma unroll
      for (int i = 0; i < 8; ++i) c = fma(c, 0.999999, 1e-9);
    s = c;
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
  const int it_m = 4000, it_f = 4000;
  struct Case { const char* name; Roles ro; };
  Case cases[] = {
      {"16 DMMA (all SMSPs)", {{1,1,1,1,1,1,1,1,1,1,1,1,1,1,1,1}}},
      {"8 DMMA w0-7 alone", {{1,1,1,1,1,1,1,1,0,0,0,0,0,0,0,0}}},
      {"12 DMMA on SMSP 0-2 alone", {{1,1,1,0,1,1,1,0,1,1,1,0,1,1,1,0}}},
      {"8 DFMA-tput w8-15 alone", {{0,0,0,0,0,0,0,0,2,2,2,2,2,2,2,2}}},
      {"4 DFMA-tput on SMSP 3 alone", {{0,0,0,2,0,0,0,2,0,0,0,2,0,0,0,2}}},
      {"8 DFMA-lat w8-15 alone", {{0,0,0,0,0,0,0,0,3,3,3,3,3,3,3,3}}},
      {"mixed: 8 DMMA w0-7 + 8 DFMA-tput w8-15", {{1,1,1,1,1,1,1,1,2,2,2,2,2,2,2,2}}},
      {"mixed: 8 DMMA w0-7 + 8 DFMA-lat w8-15", {{1,1,1,1,1,1,1,1,3,3,3,3,3,3,3,3}}},
      {"mixed, DFMA low wid: 8 DFMA-lat w0-7 + 8 DMMA w8-15", {{3,3,3,3,3,3,3,3,1,1,1,1,1,1,1,1}}},
      {"split: 12 DMMA SMSP 0-2 + 4 DFMA-tput SMSP 3", {{1,1,1,2,1,1,1,2,1,1,1,2,1,1,1,2}}},
      {"split: 12 DMMA SMSP 0-2 + 4 DFMA-lat SMSP 3", {{1,1,1,3,1,1,1,3,1,1,1,3,1,1,1,3}}},
      {"split: 6 DMMA SMSP 0-2 + 4 DFMA-lat SMSP 3", {{1,1,1,3,1,1,1,3,0,0,0,3,0,0,0,3}}},
  };
  for (const Case& cs : cases) {
    k<<<sms, 512>>>(d, cyc, cs.ro, 10, 10);
    k<<<sms, 512>>>(d, cyc, cs.ro, it_m, it_f);
    cudaDeviceSynchronize();
    long long h[64];
    cudaMemcpy(h, cyc, 64 * 8, cudaMemcpyDeviceToHost);
    double dm = 0, df = 0;
    int nm = 0, nf = 0, flat = 0;
    for (int w = 0; w < 16; ++w) {
      if (cs.ro.r[w] == 1) { dm = h[w] > dm ? h[w] : dm; ++nm; }
      if (cs.ro.r[w] >= 2) { df = h[w] > df ? h[w] : df; ++nf; flat = cs.ro.r[w] == 3; }
    }
    printf("%-52s", cs.name);
    if (nm) printf("  DMMA %.0f cyc total, %.1f DMMA/kcycle/SM", dm, 4.0 * it_m * nm / dm * 1000.0 / 1000.0 * 1.0);
    if (nf) printf("  DFMA %.0f cyc total, %.2f cyc/dependent-op", df, flat ? df / (8.0 * it_f) : df / (1.0 * it_f));
    printf("\n");
  }
  return 0;
}
