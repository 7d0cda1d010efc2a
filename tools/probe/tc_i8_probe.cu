// tcgen05 kind::i8 probe for the Ozaki (int8-sliced fp64) route of the EDAA contractions
// (VERDICT r1 item 4).  Measures, on one B200:
//   1. correctness of a hand-written tcgen05.mma.kind::i8 (SS operands, K-major, no swizzle,
//      int32 accumulators in TMEM, read back with tcgen05.ld) against a CPU product;
//   2. the int8 MMA issue rate per SM for the tile shapes the contractions would use
//      (M = 128, N = 32 .. 256, K = 32 per instruction);
//   3. the TMEM -> register -> fp64 reconstruction rate (tcgen05.ld + I2F + DFMA);
//   4. the fp64 -> 7 x int8 slicing rate of the softmax weights (scalar fp64 work).
// and prints the projected B-pass time of cfg1 from them next to the DMMA pass.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -o tc_i8_probe tc_i8_probe.cu
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#include <cuda_runtime.h>

#define CK(x)                                                                      \
  do {                                                                             \
    cudaError_t e_ = (x);                                                          \
    if (e_ != cudaSuccess) {                                                       \
      std::printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e_), __FILE__, __LINE__); \
      std::exit(1);                                                                \
    }                                                                              \
  } while (0)

namespace {

constexpr int kM = 128;      // rows of D = TMEM lanes
constexpr int kKStep = 32;   // int8 elements per MMA along K

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }

// Shared-memory matrix descriptor, K-major, SWIZZLE_NONE ("interleave") canonical layout:
// core matrices of 8 rows x 16 bytes stored contiguously (128 B); SBO = byte distance of
// 8-row groups, LBO = byte distance of the two 16-byte K chunks of one MMA; version 1 (sm_100).
__device__ __forceinline__ uint64_t make_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  return static_cast<uint64_t>((saddr >> 4) & 0x3FFF) | (static_cast<uint64_t>((lbo >> 4) & 0x3FFF) << 16) |
         (static_cast<uint64_t>((sbo >> 4) & 0x3FFF) << 32) | (1ull << 46);
}
// Instruction descriptor, kind::i8: D = S32, A = B = signed 8 bit, both K-major, dense.
__host__ __device__ constexpr uint32_t make_idesc(int M, int N) {
  return (2u << 4) | (1u << 7) | (1u << 10) | (static_cast<uint32_t>(N >> 3) << 17) | (static_cast<uint32_t>(M >> 4) << 24);
}
// Byte offset of element (row r, k) of a rows x K int8 operand in the canonical layout above
// with the K chunks outermost: core matrix (r/8, k/16) at ((k/16)·rows/8 + r/8)·128.
__host__ __device__ inline int core_off(int r, int k, int rows) { return ((k >> 4) * (rows >> 3) + (r >> 3)) * 128 + (r & 7) * 16 + (k & 15); }

__device__ __forceinline__ void mma_i8(uint32_t taddr, uint64_t da, uint64_t db, uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, {%5, %5, %5, %5}, p;\n\t}\n" ::"r"(taddr),
      "l"(da), "l"(db), "r"(idesc), "r"(accumulate), "r"(0u)
      : "memory");
}
// the same instruction with kind::f16 (fp16 inputs, fp32 accumulators, K = 16 per instruction): rate reference
__device__ __forceinline__ void mma_f16(uint32_t taddr, uint64_t da, uint64_t db, uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, {%5, %5, %5, %5}, p;\n\t}\n" ::"r"(taddr),
      "l"(da), "l"(db), "r"(idesc), "r"(accumulate), "r"(0u)
      : "memory");
}
__device__ __forceinline__ void mma_commit(unsigned long long* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_init(unsigned long long* bar, unsigned n) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(n) : "memory");
}
// Bounded wait (a probe must not hang the box if a descriptor is wrong): gives up after ~2^22 polls.
__device__ __forceinline__ void mbar_wait(unsigned long long* bar, unsigned parity) {
  for (int spin = 0; spin < (1 << 22); ++spin) {
    unsigned ok;
    asm volatile("{\n.reg .pred P1;\nmbarrier.try_wait.parity.shared::cta.b64 P1, [%1], %2;\nselp.u32 %0, 1, 0, P1;\n}\n"
                 : "=r"(ok)
                 : "r"(smem_u32(bar)), "r"(parity)
                 : "memory");
    if (ok) return;
  }
  if ((threadIdx.x & 31) == 0) printf("mbarrier wait timed out (block %d warp %d)\n", blockIdx.x, threadIdx.x >> 5);
}
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t (&v)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];\n"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]), "=r"(v[8]),
        "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]), "=r"(v[16]),
        "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]), "=r"(v[24]),
        "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

struct Setup {
  uint32_t tmem;
};

// Common prologue: operands into shared memory (canonical layout), TMEM allocation (512 columns).
template <int N, int KTOT>
__device__ __forceinline__ uint32_t prologue(const int8_t* A, const int8_t* B, int8_t* sa, int8_t* sb, uint32_t* tslot,
                                             unsigned long long* bar) {
  for (int e = threadIdx.x; e < kM * KTOT; e += blockDim.x) sa[core_off(e / KTOT, e % KTOT, kM)] = A ? A[e] : static_cast<int8_t>(e * 7 + 3);
  for (int e = threadIdx.x; e < N * KTOT; e += blockDim.x) sb[core_off(e / KTOT, e % KTOT, N)] = B ? B[e] : static_cast<int8_t>(e * 5 + 1);
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // generic-proxy writes -> visible to the tensor core (async proxy)
  if (threadIdx.x == 0) {
    mbar_init(bar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(tslot)) : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  return *tslot;
}
__device__ __forceinline__ void epilogue_free(uint32_t tmem) {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem) : "memory");
}

// 1. D[128][N] = A[128][KTOT] · B[N][KTOT]ᵀ, int8 -> int32, one CTA.
template <int N, int KTOT>
__global__ void __launch_bounds__(128) k_check(const int8_t* A, const int8_t* B, int* D) {
  extern __shared__ __align__(1024) unsigned char smem[];
  int8_t* sa = reinterpret_cast<int8_t*>(smem);
  int8_t* sb = sa + kM * KTOT;
  __shared__ uint32_t tslot;
  __shared__ __align__(8) unsigned long long bar;
  const uint32_t tmem = prologue<N, KTOT>(A, B, sa, sb, &tslot, &bar);
  if (threadIdx.x == 0) {
    constexpr uint32_t idesc = make_idesc(kM, N);
    for (int ks = 0; ks < KTOT / kKStep; ++ks) {
      const uint64_t da = make_desc(smem_u32(sa) + ks * 2 * (kM / 8) * 128, (kM / 8) * 128, 128);
      const uint64_t db = make_desc(smem_u32(sb) + ks * 2 * (N / 8) * 128, (N / 8) * 128, 128);
      mma_i8(tmem, da, db, idesc, ks > 0);
    }
    mma_commit(&bar);
  }
  mbar_wait(&bar, 0);
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int c0 = 0; c0 < N; c0 += 32) {
    uint32_t v[32];
    tmem_ld32(tmem + (static_cast<uint32_t>(warp * 32) << 16) + c0, v);
    for (int i = 0; i < 32; ++i) D[(warp * 32 + lane) * N + c0 + i] = static_cast<int>(v[i]);
  }
  epilogue_free(tmem);
}

// 2. issue rate: `iters` MMAs of 128 x N x (32 bytes of K) per SM, 4 per loop trip (no address
// arithmetic between them), into 1 or 2 accumulators; F16 = the same shapes with kind::f16.
template <int N, bool F16>
__global__ void __launch_bounds__(128) k_rate(int iters, int nacc, long long* cyc) {
  extern __shared__ __align__(1024) unsigned char smem[];
  constexpr int KTOT = 128;  // 4 k-steps of operands, cycled
  int8_t* sa = reinterpret_cast<int8_t*>(smem);
  int8_t* sb = sa + kM * KTOT;
  __shared__ uint32_t tslot;
  __shared__ __align__(8) unsigned long long bar;
  const uint32_t tmem = prologue<N, KTOT>(nullptr, nullptr, sa, sb, &tslot, &bar);
  if (threadIdx.x == 0) {
    constexpr uint32_t idesc = F16 ? ((1u << 4) | (static_cast<uint32_t>(N >> 3) << 17) | (static_cast<uint32_t>(kM >> 4) << 24))
                                   : make_idesc(kM, N);
    uint64_t da[4], db[4];
    for (int ks = 0; ks < 4; ++ks) {
      da[ks] = make_desc(smem_u32(sa) + ks * 2 * (kM / 8) * 128, (kM / 8) * 128, 128);
      db[ks] = make_desc(smem_u32(sb) + ks * 2 * (N / 8) * 128, (N / 8) * 128, 128);
    }
    const uint32_t t1a = tmem + (nacc > 1 ? N : 0);
    const long long t0 = clock64();
    for (int it = 0; it < iters; it += 4) {
#pragma unroll
      for (int ks = 0; ks < 4; ++ks) {
        if (F16) mma_f16((ks & 1) ? t1a : tmem, da[ks], db[ks], idesc, it > 0);
        else mma_i8((ks & 1) ? t1a : tmem, da[ks], db[ks], idesc, it > 0);
      }
    }
    mma_commit(&bar);
    mbar_wait(&bar, 0);
    const long long t1 = clock64();
    if (blockIdx.x == 0) cyc[0] = t1 - t0;
  } else {
    mbar_wait(&bar, 0);
  }
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  epilogue_free(tmem);
}

// 3. reconstruction: read `ngroups` accumulators of 128 x N int32 from TMEM and fold them into
// fp64 with the slice weights (I2F + DFMA per value); cycles for the whole CTA (4 warps).
template <int N>
__global__ void __launch_bounds__(128) k_recon(int ngroups, int reps, long long* cyc, double* out) {
  extern __shared__ __align__(1024) unsigned char smem[];
  constexpr int KTOT = 32;
  int8_t* sa = reinterpret_cast<int8_t*>(smem);
  int8_t* sb = sa + kM * KTOT;
  __shared__ uint32_t tslot;
  __shared__ __align__(8) unsigned long long bar;
  const uint32_t tmem = prologue<N, KTOT>(nullptr, nullptr, sa, sb, &tslot, &bar);
  if (threadIdx.x == 0) {
    constexpr uint32_t idesc = make_idesc(kM, N);
    const uint64_t da = make_desc(smem_u32(sa), (kM / 8) * 128, 128);
    const uint64_t db = make_desc(smem_u32(sb), (N / 8) * 128, 128);
    for (int g = 0; g < ngroups; ++g) mma_i8(tmem + g * N, da, db, idesc, 0);
    mma_commit(&bar);
  }
  mbar_wait(&bar, 0);
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const int warp = threadIdx.x >> 5;
  double acc[N];
  for (int i = 0; i < N; ++i) acc[i] = 0.0;
  __syncthreads();
  const long long t0 = clock64();
  for (int r = 0; r < reps; ++r) {
    double wgt = 1.0;
    for (int g = 0; g < ngroups; ++g) {
#pragma unroll
      for (int c0 = 0; c0 < N; c0 += 32) {
        uint32_t v[32];
        tmem_ld32(tmem + (static_cast<uint32_t>(warp * 32) << 16) + g * N + c0, v);
#pragma unroll
        for (int i = 0; i < 32; ++i) acc[c0 + i] = fma(static_cast<double>(static_cast<int>(v[i])), wgt, acc[c0 + i]);
      }
      wgt *= 0.0078125;  // 2^-7 per slice group
    }
  }
  __syncthreads();
  const long long t1 = clock64();
  if (blockIdx.x == 0 && threadIdx.x == 0) cyc[0] = t1 - t0;
  double s = 0.0;
  for (int i = 0; i < N; ++i) s += acc[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  epilogue_free(tmem);
}

// 4. slicing: fp64 values in [0, 1] (softmax weights, per-column scale 1) -> 7 signed int8 digits
// base 128 (49 bits), error-free: d_k = rint(r·128), r <- r·128 − d_k.  Elements per thread `n`.
__global__ void k_slice(const double* w, int8_t* out, int n, long long* cyc) {
  const int tid = blockIdx.x * blockDim.x + threadIdx.x;
  const long long t0 = clock64();
  for (int e = 0; e < n; ++e) {
    double r = w[static_cast<size_t>(e) * gridDim.x * blockDim.x + tid];
    uint32_t lo = 0, hi = 0;
#pragma unroll
    for (int k = 0; k < 7; ++k) {
      r *= 128.0;
      const double d = rint(r);
      r -= d;
      const uint32_t b = static_cast<uint32_t>(static_cast<int>(d)) & 0xFF;
      if (k < 4) lo |= b << (8 * k); else hi |= b << (8 * (k - 4));
    }
    reinterpret_cast<uint2*>(out)[static_cast<size_t>(e) * gridDim.x * blockDim.x + tid] = make_uint2(lo, hi);
  }
  const long long t1 = clock64();
  if (tid == 0) cyc[0] = t1 - t0;
}

template <int N, int KTOT>
bool run_check() {
  std::vector<int8_t> A(kM * KTOT), B(N * KTOT);
  for (size_t i = 0; i < A.size(); ++i) A[i] = static_cast<int8_t>((i * 37 + 11) % 251 - 125);
  for (size_t i = 0; i < B.size(); ++i) B[i] = static_cast<int8_t>((i * 53 + 7) % 241 - 120);
  int8_t *dA, *dB;
  int* dD;
  CK(cudaMalloc(&dA, A.size()));
  CK(cudaMalloc(&dB, B.size()));
  CK(cudaMalloc(&dD, kM * N * 4));
  CK(cudaMemcpy(dA, A.data(), A.size(), cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dB, B.data(), B.size(), cudaMemcpyHostToDevice));
  const int smem = (kM + N) * KTOT;
  k_check<N, KTOT><<<1, 128, smem>>>(dA, dB, dD);
  CK(cudaDeviceSynchronize());
  std::vector<int> D(kM * N);
  CK(cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost));
  int bad = 0;
  for (int r = 0; r < kM; ++r)
    for (int c = 0; c < N; ++c) {
      int s = 0;
      for (int k = 0; k < KTOT; ++k) s += static_cast<int>(A[r * KTOT + k]) * static_cast<int>(B[c * KTOT + k]);
      if (s != D[r * N + c] && bad++ < 4) std::printf("  mismatch D[%d][%d] = %d, want %d\n", r, c, D[r * N + c], s);
    }
  std::printf("check  M=128 N=%-3d K=%-3d : %s (%d of %d entries differ)\n", N, KTOT, bad ? "FAIL" : "exact", bad, kM * N);
  cudaFree(dA); cudaFree(dB); cudaFree(dD);
  return bad == 0;
}

template <int N, bool F16 = false>
double run_rate(int sms, long long* dcyc, int nacc) {
  const int iters = 4096;
  const int smem = (kM + N) * 128;
  CK(cudaFuncSetAttribute(k_rate<N, F16>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  k_rate<N, F16><<<sms, 128, smem>>>(64, nacc, dcyc);
  k_rate<N, F16><<<sms, 128, smem>>>(iters, nacc, dcyc);
  CK(cudaDeviceSynchronize());
  long long c;
  CK(cudaMemcpy(&c, dcyc, 8, cudaMemcpyDeviceToHost));
  const double per = static_cast<double>(c) / iters;
  const double macs = 128.0 * N * (F16 ? 16.0 : 32.0);
  std::printf("rate   %s M=128 N=%-3d K=%d, %d accumulator(s): %7.1f cycles per MMA = %6.0f MAC/cycle/SM\n", F16 ? "f16" : "i8 ", N,
              F16 ? 16 : 32, nacc, per, macs / per);
  return per;
}

template <int N>
double run_recon(int sms, long long* dcyc, double* dout, int ngroups) {
  const int reps = 64;
  k_recon<N><<<sms, 128, (kM + N) * 32>>>(ngroups, reps, dcyc, dout);
  CK(cudaDeviceSynchronize());
  long long c;
  CK(cudaMemcpy(&c, dcyc, 8, cudaMemcpyDeviceToHost));
  const double per = static_cast<double>(c) / reps;
  std::printf("recon  128 x %-3d outputs x %d slice groups: %8.0f cycles per tile = %5.2f cycles per output\n", N, ngroups, per,
              per / (128.0 * N));
  return per / (128.0 * N);
}

}  // namespace

int main() {
  int sms = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  int khz = 0;
  CK(cudaDeviceGetAttribute(&khz, cudaDevAttrClockRate, 0));
  std::printf("tcgen05 kind::i8 probe: %d SMs, %.0f MHz\n", sms, khz / 1000.0);
  bool ok = run_check<64, 64>();
  ok &= run_check<32, 224>();
  ok &= run_check<256, 32>();
  long long* dcyc;
  double* dout;
  CK(cudaMalloc(&dcyc, 64));
  CK(cudaMalloc(&dout, sms * 128 * 8));
  run_rate<8>(sms, dcyc, 1);
  const double r32 = run_rate<32>(sms, dcyc, 1);
  const double r64 = run_rate<64>(sms, dcyc, 1);
  run_rate<64>(sms, dcyc, 2);
  const double r128 = run_rate<128>(sms, dcyc, 1);
  const double r256 = run_rate<256>(sms, dcyc, 1);
  run_rate<256>(sms, dcyc, 2);
  run_rate<32, true>(sms, dcyc, 1);
  run_rate<64, true>(sms, dcyc, 1);
  run_rate<128, true>(sms, dcyc, 1);
  run_rate<256, true>(sms, dcyc, 1);
  const double rec = run_recon<64>(sms, dcyc, dout, 7);
  // slicing
  const int n = 64, threads = 256, blocks = sms * 4;
  double* dw;
  int8_t* dsl;
  const size_t tot = static_cast<size_t>(n) * threads * blocks;
  CK(cudaMalloc(&dw, tot * 8));
  CK(cudaMalloc(&dsl, tot * 8));
  std::vector<double> hw(tot);
  // weights pre-scaled to [0, 1/2) (one exponent shift per column), so every digit is in [-64, 64]
  for (size_t i = 0; i < tot; ++i) hw[i] = 0.499 * static_cast<double>((i * 2654435761ull) % 1000003) / 1000003.0;
  CK(cudaMemcpy(dw, hw.data(), tot * 8, cudaMemcpyHostToDevice));
  k_slice<<<blocks, threads>>>(dw, dsl, n, dcyc);
  k_slice<<<blocks, threads>>>(dw, dsl, n, dcyc);
  CK(cudaDeviceSynchronize());
  long long c;
  CK(cudaMemcpy(&c, dcyc, 8, cudaMemcpyDeviceToHost));
  const double slice_cyc = static_cast<double>(c) / (static_cast<double>(n) * threads * 4);  // cycles per element per SM (4 CTAs of 256 resident)
  // check the digits reconstruct the value to 2^-49
  std::vector<int8_t> hs(tot * 8);
  CK(cudaMemcpy(hs.data(), dsl, tot * 8, cudaMemcpyDeviceToHost));
  double worst = 0.0;
  for (size_t i = 0; i < 4096; ++i) {
    double v = 0.0, wgt = 1.0;
    for (int k = 0; k < 7; ++k) {
      wgt /= 128.0;
      v += hs[i * 8 + k] * wgt;
    }
    worst = std::max(worst, std::abs(v - hw[i]));
  }
  std::printf("slice  fp64 -> 7 int8 digits: %.2f cycles per element per SM (1024 threads), max |error| %.2e (2^-50 = %.2e)\n",
              slice_cyc, worst, 1.0 / (1ull << 50));

  // ---- projection for the cfg1 B pass (L = 198 -> 224 = 7 k-steps, N = 10,000 pixels, M·p = 200 columns) ----
  // Per 128-pixel tile and 64-column chunk: P1 (g = XᵀZ) 28 slice products x 7 k-steps of 128x64x32;
  // P3 (Y += X·w) 2 row tiles x 28 products x 4 k-steps of 128x64x32; TMEM holds the 7 exponent groups of one
  // 64-column chunk (7 x 64 = 448 of 512 columns); the P3 groups of 2 x 64 columns do not fit beside them.
  const double tiles = (10000.0 / 128.0) * 4.0;  // 128-pixel tiles x 64-column chunks (200 -> 256 columns)
  const double p1 = 28 * 7 * r64, p3 = 2 * 28 * 4 * r64;
  const double recon_cyc = rec * 128 * 64 * 1.0;            // P1's g: 7 groups folded per output
  const double slice_c = slice_cyc * 128 * 64;              // the tile's softmax weights -> 7 digits
  const double per_tile = p1 + p3 + 0.0;                    // MMA pipe
  const double side = recon_cyc + slice_c;                  // CUDA-core side work per tile (overlappable at best)
  const double mhz = khz / 1000.0;
  std::printf("\nprojection, cfg1 B pass (%.0f tile-chunks over %d SMs = %.2f waves):\n", tiles, sms, tiles / sms);
  std::printf("  int8 MMA   : P1 %.0f + P3 %.0f = %.0f cycles per tile-chunk\n", p1, p3, per_tile);
  std::printf("  side work  : reconstruction %.0f + slicing %.0f = %.0f cycles per tile-chunk\n", recon_cyc, slice_c, side);
  const double waves = std::ceil(tiles / sms);
  std::printf("  pass time  : %.1f us if side work overlaps fully, %.1f us if serial  (DMMA B pass: 92.8 us measured, 43 us at its roof)\n",
              waves * std::max(per_tile, side) / mhz, waves * (per_tile + side) / mhz);
  (void)r32; (void)r128; (void)r256;
  std::printf(ok ? "all checks exact\n" : "CHECK FAILED\n");
  return ok ? 0 : 1;
}
