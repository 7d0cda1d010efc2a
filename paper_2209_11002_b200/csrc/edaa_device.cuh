// Device helpers shared by the EDAA kernel translation units.
#pragma once
#include <cmath>
#include <cstdint>

#include "edaa_internal.cuh"

namespace edaa {
namespace dev {

__device__ __forceinline__ double log_floor() { return -69.07755278982137; }  // log(1e-30)

// D = A·B + D for one 8×8×4 fp64 tile. Lane (g = lane>>2, t = lane&3) holds
// A[g][t], B[t][g] and D[g][2t], D[g][2t+1].
__device__ __forceinline__ void dmma(double (&d)[2], double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
      : "+d"(d[0]), "+d"(d[1])
      : "d"(a), "d"(b));
}

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait0() { asm volatile("cp.async.wait_group 0;\n" ::: "memory"); }

// SplitMix64 draw number `index` (0-based) of the stream seeded with `seed`:
// the state after index+1 increments (prng.hpp:15-26), mapped to [0,1)
// with the top 53 bits (prng.hpp:24-26).
__device__ __forceinline__ double splitmix_unit_at(uint64_t seed, uint64_t index) {
  uint64_t z = seed + (index + 1ull) * 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  z = z ^ (z >> 31);
  return static_cast<double>(z >> 11) * 0x1.0p-53;
}

__device__ __forceinline__ double max_like_std(double top, double s) {
  return (top < s) ? s : top;  // std::max(top, s): NaN in s is ignored
}

// Shared-memory plan of the pass kernel (one CTA per SM, two warp groups):
//   xs  nbuf × X tile          [Lpad][kXST] fp32/fp64  (tile i+2 loads while i, i+1 are used)
//   ws  W chunk (Y or Z)       [Lpad][WST]  fp64
//   ss  2 × projection/weights [QCpad][kSST] fp64 (band half 0; becomes the weights w)
//   sh  2 × projection half 1  [QCpad][kSST] fp64
//   st  2 × state tile         [QCpad][kNP] fp64 (A or logits of the chunk's columns)
//   gs  G blocks of the chunk's runs, then per-column and per-run scalars.
struct SmemLayout {
  int xs_off, xs_bytes, ws_off, ss_off, sh_off, st_off, buf_bytes, st_bytes, gs_off, col_off, total;
};

__host__ __device__ inline int align16(int b) { return (b + 15) & ~15; }

// W row stride (doubles): ≡ 8 mod 16 so a DMMA A-fragment (4 rows × 8 columns) hits 2 wavefronts.
__host__ __device__ inline int w_stride(int qcpad) { return qcpad + ((qcpad % 16 == 0) ? 8 : 0); }

__host__ __device__ inline SmemLayout smem_layout(const Dims& d, int nbuf) {
  SmemLayout s;
  int off = 0;
  s.xs_off = off;
  s.xs_bytes = align16(d.Lpad * kXST * d.xbytes);
  off += nbuf * s.xs_bytes;
  s.ws_off = off;
  off += align16(d.Lpad * w_stride(d.QCpad) * 8);
  s.buf_bytes = align16(d.QCpad * kSST * 8);
  s.ss_off = off;
  off += 2 * s.buf_bytes;
  s.sh_off = off;
  off += 2 * s.buf_bytes;
  s.st_bytes = align16(d.QCpad * kNP * 8);
  s.st_off = off;
  off += 2 * s.st_bytes;
  s.gs_off = off;
  off += align16(d.RC * d.p * d.p * 8);
  // m_run, S_run, colm, collogS, eta (QCpad each), fac[2][QCpad]; obj_run (RC), hobj (4·RC)
  s.col_off = off;
  off += align16((7 * d.QCpad + 5 * d.RC) * 8);
  s.total = off;
  return s;
}

__device__ __forceinline__ void bar_sync(int id, int n) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}
__device__ __forceinline__ void bar_arrive(int id, int n) {
  asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(n) : "memory");
}
__device__ __forceinline__ void cp_async_wait1() { asm volatile("cp.async.wait_group 1;\n" ::: "memory"); }

__device__ __forceinline__ double warp_max(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}
__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

}  // namespace dev
}  // namespace edaa
