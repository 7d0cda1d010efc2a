// Hand-off latency between two warp groups of one CTA: ping-pong of N rounds
// through (a) mbarrier arrive / try_wait.parity, (b) named barriers
// (bar.arrive by the producer group, bar.sync by the consumer group),
// (c) a flag in shared memory (st.release / ld.acquire spin).
// usage: handoff   -> cycles per one-way hand-off for each mechanism
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ unsigned su32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mb_init(unsigned long long* b, unsigned c) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(b)), "r"(c) : "memory");
}
__device__ __forceinline__ void mb_arrive(unsigned long long* b) {
  asm volatile("{ .reg .b64 st; mbarrier.arrive.shared::cta.b64 st, [%0]; }" ::"r"(su32(b)) : "memory");
}
__device__ __forceinline__ void mb_wait(unsigned long long* b, unsigned ph) {
  asm volatile("{ .reg .pred P; W: mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1; @!P bra W; }" ::"r"(su32(b)),
               "r"(ph) : "memory");
}
__device__ __forceinline__ void mb_wait_test(unsigned long long* b, unsigned ph) {
  asm volatile("{ .reg .pred P; W: mbarrier.test_wait.parity.shared::cta.b64 P, [%0], %1; @!P bra W; }" ::"r"(su32(b)),
               "r"(ph) : "memory");
}
__device__ __forceinline__ void nb_arrive(int id, int n) { asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(n) : "memory"); }
__device__ __forceinline__ void nb_sync(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory"); }

// G warps per group; group 0 = warps [0,G), group 1 = [G,2G).
template <int MODE>
__global__ void k(long long* out, int rounds, int G) {
  __shared__ unsigned long long bars[2];
  __shared__ volatile int flag[2];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const bool g0 = w < G;
  if (threadIdx.x == 0) {
    mb_init(&bars[0], G);
    mb_init(&bars[1], G);
    flag[0] = flag[1] = 0;
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const int n = 64 * G;  // threads in both groups
  long long t0 = clock64();
  for (int r = 0; r < rounds; ++r) {
    const unsigned ph = r & 1;
    if (g0) {  // ping: signal 0, wait 1
      if (MODE == 0 || MODE == 3) {
        __syncwarp();
        if (lane == 0) mb_arrive(&bars[0]);
        if (MODE == 0) mb_wait(&bars[1], ph); else mb_wait_test(&bars[1], ph);
      } else if (MODE == 1) {
        nb_arrive(1, n);
        nb_sync(2, n);
      } else {
        __syncwarp();
        if (lane == 0 && w == 0) { __threadfence_block(); flag[0] = r + 1; }
        while (flag[1] < r + 1) {}
      }
    } else {  // pong: wait 0, signal 1
      if (MODE == 0 || MODE == 3) {
        if (MODE == 0) mb_wait(&bars[0], ph); else mb_wait_test(&bars[0], ph);
        __syncwarp();
        if (lane == 0) mb_arrive(&bars[1]);
      } else if (MODE == 1) {
        nb_sync(1, n);
        nb_arrive(2, n);
      } else {
        while (flag[0] < r + 1) {}
        __syncwarp();
        if (lane == 0 && w == G) { __threadfence_block(); flag[1] = r + 1; }
      }
    }
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
}

int main() {
  long long* d;
  cudaMalloc(&d, 8 * 1024);
  const char* names[4] = {"mbarrier try_wait", "named barrier   ", "smem flag spin  ", "mbarrier test_wait"};
  for (int G : {1, 8}) {
    for (int m = 0; m < 4; ++m) {
      if (m == 2 && G > 1) continue;
      const int rounds = 20000;
      void (*kern)(long long*, int, int) = m == 0 ? k<0> : m == 1 ? k<1> : m == 2 ? k<2> : k<3>;
      kern<<<148, 64 * G>>>(d, 100, G);
      kern<<<148, 64 * G>>>(d, rounds, G);
      cudaDeviceSynchronize();
      long long h;
      cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
      printf("%s  warps/group=%d  %.0f cycles per one-way hand-off  (%s)\n", names[m], G, (double)h / rounds / 2,
             cudaGetErrorString(cudaGetLastError()));
    }
  }
  return 0;
}
