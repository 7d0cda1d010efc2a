// EDAA hot-path kernels for sm_100a (B200).
//
// One "pass" streams the image X once and serves every run of the batch:
//   phase 1  S = Wᵀ·X_tile        (W = Y for the A-phase, Z for a B-step) on the
//                                 fp64 tensor pipe (DMMA m8n8k4), X widened
//                                 from the fp32 tile in shared memory;
//   phase 2  per-pixel update     A-phase: K1 entropic steps on the p-simplex of
//                                 every pixel (softmax in registers, fp64);
//                                 B-step: logit update + online column max;
//   phase 3  C += X_tile·wᵀ        (w = new A, or exp(ℓ − m_run) for B) on DMMA;
//                                 the A-phase appends w itself as pseudo-bands
//                                 so AAᵀ falls out of the same contraction.
// Partials per (pixel slice, run chunk) are reduced in a fixed order by the
// combine kernels, so a run's arithmetic does not depend on the batch it is
// in (bitwise replay, test_ensemble.cpp:150-169).
//
// Reference semantics followed (file:line under /root/reference/proj):
//   entropic step      solver.cpp:20-46   (1e-30 floor, max-subtracted softmax)
//   A block            solver.cpp:212-218 (XB fixed over K1 steps)
//   B block            solver.cpp:219-227 (Z_k = XAᵀ − (X·B_k)·AAᵀ, g = Xᵀ Z_k)
//   objective trace    solver.cpp:206,229 (½‖X − XB·A‖² before each A block)
//   B⁰ initialisation  solver.cpp:118-136 (SplitMix64 draw i·N+j, softmax(0.1u))
//   step sizes         solver.cpp:138-149, matrix.cpp:150-190
//   fit / coherence    ensemble.cpp:29-60; selection ensemble.cpp:71-94
#include <algorithm>
#include <cmath>
#include <cstdio>

#include "edaa_device.cuh"

namespace edaa {

namespace {

using namespace dev;

// check_iterate on a contribution column held as logits + normaliser
// (solver.cpp:65-90): b_j = e^{ℓ_j − m}/S.  Non-finite: the column max or sum
// is not finite (a NaN/Inf logit poisons both).  Negative entries cannot occur
// (an exponential over a positive sum).  Drift: the mass of the normalised
// column, accumulated slice by slice, is further than 1e-9 from 1.
__device__ __forceinline__ void post_column_check(const CombineArgs& ca, int r, int i, double m, double Ssum,
                                                  double nsum) {
  const unsigned tb = (static_cast<unsigned>(ca.t) << 1) | 1u;
  const unsigned long long col = static_cast<unsigned long long>(i) << 28;
  if (!(isfinite(m) && isfinite(Ssum) && Ssum > 0.0))
    atomicMin(ca.fail_key + r, fail_key_make(tb, ca.kin, col, kFailNonFinite));
  else if (!(fabs(nsum - 1.0) <= kSimplexTol))
    atomicMin(ca.fail_key + r, fail_key_make(tb, ca.kin, col | ((1ull << 28) - 1), kFailDrift));
}

// Final objective pass: trace[T] of every run = Σ over slices (ascending) of its objective terms.
__global__ void k_rowsum(CombineArgs ca, int /*rows*/) {
  griddep_launch_dependents();
  griddep_wait();
  const Dims& d = ca.d;
  const int S = d.nslices;
  if (blockIdx.x != 0 || blockIdx.y != 0) return;
  for (int r = threadIdx.y * 32 + threadIdx.x; r < d.M; r += 256) {
    double o = 0.0;
    for (int sl = 0; sl < S; ++sl) o += ca.part_obj[static_cast<size_t>(sl) * d.M + r];
    ca.trace[static_cast<size_t>(r) * ca.trace_stride + ca.trace_index] = o;
  }
}

// ---------------------------------------------------------------------------
// Combine of one pass's slice partials, fused with Z = XAᵀ − Y·AAᵀ
// (solver.cpp:221, anchored on the A block's XAᵀ/AAᵀ).  One CTA per (run
// chunk, kCR band rows); 256 threads = kCR rows × kCG slice groups × 32 lanes
// (lane x < kQMax = column of the chunk).  Group g sums the contiguous slice
// range [g·S/kCG, (g+1)·S/kCG) in ascending order and the kCG group sums are
// added in g order: one fixed order that depends on the slicing (a function of
// N) only, so a run's arithmetic stays independent of its batch and position
// (test_ensemble.cpp:150-169 analogue).
//   A:        XAᵀ rows = Σ_s C_s, then Z with the block's Y and AAᵀ (k_aat);
//   B / init: Y rows = Σ_s C_s·e^{m_s−m} / S with the column normalisers, then Z.
constexpr int kCR = 2;
constexpr int kCG = 4;

// A pass only (the B step / init combine is k_combine_b below, same summation order).
__global__ void __launch_bounds__(256) k_combine(CombineArgs ca) {
  griddep_launch_dependents();
  griddep_wait();
  __shared__ double red[kCR * kCG][kQMax];
  __shared__ double ys[kCR][kQMax];
  const Dims& d = ca.d;
  const int x = threadIdx.x & 31, y = threadIdx.x >> 5;
  const int rr = y % kCR, g = y / kCR;
  const int col0 = blockIdx.x * d.QCpad;
  const int S = d.nslices;
  const int p = d.p;
  const int ncol = min(d.RC, d.M - static_cast<int>(blockIdx.x) * d.RC) * p;
  const size_t sstride = static_cast<size_t>(d.Lrows) * d.Qs;
  const int l = blockIdx.y * kCR + rr;
  const bool live = (x < kQMax) && (l < d.Lpad);
  if (live) {
    const int s0 = (g * S) / kCG, s1 = ((g + 1) * S) / kCG;
    const double* src = ca.part_C + static_cast<size_t>(l) * d.Qs + col0 + x;
    double v = 0.0;
#pragma unroll 8
    for (int sl = s0; sl < s1; ++sl) v += src[sl * sstride];
    red[y][x] = v;
  }
  __syncthreads();
  if (g == 0 && live) {
    double v = red[rr][x];
    for (int k = 1; k < kCG; ++k) v += red[k * kCR + rr][x];
    const size_t o = static_cast<size_t>(l) * d.Qs + col0 + x;
    ca.XAt[o] = v;
    red[rr][x] = v;
    ys[rr][x] = ca.Y[o];
  }
  if (ca.Z == nullptr) return;
  __syncthreads();
  if (g == 0 && live && x < ncol) {
    // Z = XAᵀ − Y·AAᵀ for this row (m ascending, from 0)
    const int rl = x / p;
    const double* arow = ca.AAt + static_cast<size_t>(rl * p) * d.Qs + col0 + x;  // AAᵀ[rl·p+m][x]
    double sacc = 0.0;
    for (int mm = 0; mm < p; ++mm) sacc += ys[rr][rl * p + mm] * arow[static_cast<size_t>(mm) * d.Qs];
    ca.Z[static_cast<size_t>(l) * d.Qs + col0 + x] = red[rr][x] - sacc;
  }
}

// B step / init combine in ONE kernel: column normalisers, Y rows and Z rows.
// CTA = (run chunk, kBR band rows), 256 threads.  Every CTA of a chunk first
// recomputes that chunk's 24 column normalisers (the few-KB part_m/part_S
// columns; identical arithmetic in every CTA), keeps e^{m_s−m} in shared memory, then sums its rows'
// slice partials in kCG contiguous groups added in order (k_combine's order),
// and forms Z = XAᵀ − Y·AAᵀ.  One launch instead of two, and the rescale
// factors come from shared memory instead of a global scratch array.
#ifndef EDAA_KBR
#define EDAA_KBR 8
#endif
constexpr int kBRMax = EDAA_KBR;  // band rows per CTA for full grids (a row's slice-sum order does not depend on it)
// Small batches (few run chunks) launch the same kernel with fewer rows per CTA, so the
// combine — latency-bound on NCH·⌈Lpad/kBR⌉ CTAs — still fills the GPU: at cfg0 (one
// chunk) 8 rows per CTA is 20 CTAs and 15.7 µs per launch, as long as cfg1's 225.

template <int kBR>
__global__ void __launch_bounds__(256) k_combine_b(CombineArgs ca) {
  griddep_launch_dependents();
  griddep_wait();
  extern __shared__ __align__(16) double facs[];  // [nslices][kQMax]
  __shared__ double cS[kQMax];
  __shared__ double red[kCG][kBR][kQMax];
  __shared__ double ys[kBR][kQMax];
  const Dims& d = ca.d;
  const int tid = threadIdx.x;
  const int chunk = blockIdx.x;
  const int col0 = chunk * d.QCpad;
  const int S = d.nslices;
  const int ncol = min(d.RC, d.M - chunk * d.RC) * d.p;
  // The row sums' operands first: every thread owns up to kIt (group, row, column) sums
  // and issues the loads of its first kPre slices NOW, so their L2 latency overlaps the
  // normaliser phase below (the products need e^{m_s − m}, the loads do not).  The
  // accumulation order of a sum (slices ascending) is unchanged.
  const int l0 = blockIdx.y * kBR;
  const int nr = min(kBR, d.Lpad - l0);
  const size_t sstride = static_cast<size_t>(d.Lrows) * d.Qs;
  constexpr int kSums = kCG * kBR * kQMax;
  constexpr int kIt = (kSums + 255) / 256;
  constexpr int kPre = 4;
  const double* src[kIt];
  double v[kIt], pre[kIt][kPre];
  int s0[kIt], len[kIt], xs[kIt], slot[kIt];
  int maxlen = 0;
#pragma unroll
  for (int q = 0; q < kIt; ++q) {
    const int e0 = tid + 256 * q;
    const bool in = (kSums % 256 == 0) || e0 < kSums;
    const int e = in ? e0 : 0;
    const int x = e % kQMax, rest = e / kQMax;
    const int rr = rest % kBR, g = rest / kBR;
    s0[q] = (g * S) / kCG;
    len[q] = (in && rr < nr) ? ((g + 1) * S) / kCG - s0[q] : 0;
    src[q] = ca.part_C + static_cast<size_t>(l0 + min(rr, nr - 1)) * d.Qs + col0 + x;
    xs[q] = x;
    slot[q] = (g * kBR + rr) * kQMax + x;
    v[q] = 0.0;
    maxlen = max(maxlen, len[q]);
#pragma unroll
    for (int k = 0; k < kPre; ++k) pre[q][k] = (k < len[q]) ? src[q][(s0[q] + k) * sstride] : 0.0;
  }
  // Normalisers: 8 threads per column (192 threads for the 24 columns); thread t
  // of a column takes slices t, t+8, … with all its loads issued up front, then
  // an xor tree over the 8 (fixed order: a function of the slicing only).
  // The exponentials are exp_nonpos (table + polynomial, ~1 ulp; every argument
  // m_s − m ≤ 0): its table load is in flight with the partial loads, and it is
  // about half the fp64 work of libdevice exp on this latency-bound prologue.
  __shared__ double etab[kExpTab];
  const double tabv = (tid < kExpTab) ? kExp2Tab[tid] : 0.0;
  const bool nact = tid < kQMax * 8;
  const int cc = tid >> 3, t8 = tid & 7;
  const int col = col0 + cc;
  constexpr int kPer = (kMaxSlices + 7) / 8;
  double mv[kPer], sv[kPer];
  double m = -INFINITY;
  if (nact) {
#pragma unroll
    for (int k = 0; k < kPer; ++k) {
      const int sl = t8 + 8 * k;
      mv[k] = (sl < S) ? ca.part_m[static_cast<size_t>(sl) * d.Qs + col] : -INFINITY;
      sv[k] = (sl < S) ? ca.part_S[static_cast<size_t>(sl) * d.Qs + col] : 0.0;
      m = fmax(m, mv[k]);
    }
#pragma unroll
    for (int o = 4; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
  }
  if (tid < kExpTab) etab[tid] = tabv;
  __syncthreads();
  if (nact) {
    double Ssum = 0.0;
#pragma unroll
    for (int k = 0; k < kPer; ++k) {
      const int sl = t8 + 8 * k;
      if (sl < S) {
        const double f = (mv[k] == -INFINITY) ? 0.0 : exp_nonpos(mv[k] - m, etab);
        facs[sl * kQMax + cc] = f;
        Ssum += sv[k] * f;
      }
    }
#pragma unroll
    for (int o = 4; o > 0; o >>= 1) Ssum += __shfl_xor_sync(0xffffffffu, Ssum, o);
    if (blockIdx.y == 0) {  // one CTA per chunk runs check_iterate on the chunk's columns
      const double inv = 1.0 / Ssum;
      double nsum = 0.0;
#pragma unroll
      for (int k = 0; k < kPer; ++k) {
        const int sl = t8 + 8 * k;
        if (sl < S) nsum += sv[k] * facs[sl * kQMax + cc] * inv;
      }
#pragma unroll
      for (int o = 4; o > 0; o >>= 1) nsum += __shfl_xor_sync(0xffffffffu, nsum, o);
      const int r = chunk * d.RC + cc / d.p;
      if (t8 == 0 && cc < d.RC * d.p && r < d.M) post_column_check(ca, r, cc % d.p, m, Ssum, nsum);
    }
    if (t8 == 0) {
      cS[cc] = Ssum;
      if (blockIdx.y == 0) {
        ca.colm[col] = m;
        ca.colS[col] = Ssum;
        ca.collogS[col] = log(Ssum);
      }
    }
  }
  __syncthreads();
  {
#pragma unroll
    for (int k = 0; k < kPre; ++k) {
#pragma unroll
      for (int q = 0; q < kIt; ++q)
        if (k < len[q]) v[q] += pre[q][k] * facs[(s0[q] + k) * kQMax + xs[q]];
    }
#pragma unroll 5
    for (int k = kPre; k < maxlen; ++k) {
#pragma unroll
      for (int q = 0; q < kIt; ++q)
        if (k < len[q]) {
          const int sl = s0[q] + k;
          v[q] += src[q][sl * sstride] * facs[sl * kQMax + xs[q]];
        }
    }
#pragma unroll
    for (int q = 0; q < kIt; ++q)
      if ((kSums % 256 == 0) || tid + 256 * q < kSums) (&red[0][0][0])[slot[q]] = v[q];
  }  __syncthreads();
  for (int e = tid; e < nr * kQMax; e += blockDim.x) {
    const int x = e % kQMax, rr = e / kQMax;
    double v = red[0][rr][x];
    for (int k = 1; k < kCG; ++k) v += red[k][rr][x];
    v = (x < ncol) ? v / cS[x] : 0.0;  // padding columns carry no run
    ca.Y[static_cast<size_t>(l0 + rr) * d.Qs + col0 + x] = v;
    ys[rr][x] = v;
  }
  if (ca.Z == nullptr) return;
  __syncthreads();
  for (int e = tid; e < nr * kQMax; e += blockDim.x) {
    const int x = e % kQMax, rr = e / kQMax;
    if (x >= ncol) continue;
    const int rl = x / d.p;
    const double* arow = ca.AAt + static_cast<size_t>(rl * d.p) * d.Qs + col0 + x;  // AAᵀ[rl·p+m][x]
    double sacc = 0.0;
    for (int mm = 0; mm < d.p; ++mm) sacc += ys[rr][rl * d.p + mm] * arow[static_cast<size_t>(mm) * d.Qs];
    const size_t o = static_cast<size_t>(l0 + rr) * d.Qs + col0 + x;
    ca.Z[o] = ca.XAt[o] - sacc;
  }
}

// A block: the run-diagonal AAᵀ blocks (pseudo-band rows Lpad + rl·p + i of the
// slice partials) and the objective trace.  One warp per output: lane k sums
// the contiguous slice range [k·S/32, (k+1)·S/32) in ascending order, then a
// fixed xor tree — an order that depends on the slicing only.
// grid = (NCH, ⌈RC·p²/8⌉ + 1): the last y-row of CTAs folds the traces.
__global__ void __launch_bounds__(256) k_aat(CombineArgs ca) {
  griddep_launch_dependents();
  griddep_wait();
  const Dims& d = ca.d;
  const int S = d.nslices;
  const int p = d.p;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int s0 = (lane * S) / 32, s1 = ((lane + 1) * S) / 32;
  if (blockIdx.y + 1 == gridDim.y) {  // traces: runs r ≡ (blockIdx.x·8 + w) mod (NCH·8)
    for (int r = blockIdx.x * 8 + w; r < d.M; r += gridDim.x * 8) {
      double o = 0.0;
      for (int sl = s0; sl < s1; ++sl) o += ca.part_obj[static_cast<size_t>(sl) * d.M + r];
      o = warp_sum(o);
      if (lane == 0) ca.trace[static_cast<size_t>(r) * ca.trace_stride + ca.trace_index] = o;
    }
    return;
  }
  const int col0 = blockIdx.x * d.QCpad;
  const int RCe = min(d.RC, d.M - static_cast<int>(blockIdx.x) * d.RC);
  const int e = blockIdx.y * 8 + w;
  if (e >= RCe * p * p) return;
  const int rl = e / (p * p), rem = e - rl * p * p;
  const int i = rem / p, mcol = rem - i * p;
  const size_t sstride = static_cast<size_t>(d.Lrows) * d.Qs;
  const double* src = ca.part_C + static_cast<size_t>(d.Lpad + rl * p + i) * d.Qs + col0 + rl * p + mcol;
  double v = 0.0;
  for (int sl = s0; sl < s1; ++sl) v += src[sl * sstride];
  v = warp_sum(v);
  if (lane == 0) ca.AAt[static_cast<size_t>(rl * p + i) * d.Qs + col0 + rl * p + mcol] = v;
}

// G = YᵀY per run for the next A block (p×p, one warp per entry: lanes stride
// the bands, fixed xor tree).  The init Gram that feeds step_sizes keeps the
// reference's band-ascending order in k_post.
__global__ void __launch_bounds__(256) k_gram(PostArgs pa) {
  griddep_launch_dependents();
  griddep_wait();
  const Dims& d = pa.d;
  const int r = blockIdx.x;
  const int p = d.p;
  const int c0 = (r / d.RC) * d.QCpad + (r % d.RC) * p;
  const int lr0 = (r % d.RC) * p;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  for (int e = w; e < p * p; e += 8) {
    const int i = e / p, m = e - i * p;
    double s = 0.0;
    for (int l = lane; l < d.L; l += 32)
      s += pa.Y[static_cast<size_t>(l) * d.Qs + c0 + i] * pa.Y[static_cast<size_t>(l) * d.Qs + c0 + m];
    s = warp_sum(s);
    if (lane == 0) pa.Gbuf[static_cast<size_t>(lr0 + i) * d.Qs + c0 + m] = s;
  }
}

// ---------------------------------------------------------------------------
// Per-run small algebra: Z = XAᵀ − Y·AAᵀ, G = YᵀY, and (init) the step sizes.
__global__ void __launch_bounds__(256) k_post(PostArgs pa) {
  griddep_launch_dependents();
  griddep_wait();
  const Dims& d = pa.d;
  const int r = blockIdx.x;
  const int p = d.p;
  const int chunk = r / d.RC, rl = r % d.RC;
  const int c0 = chunk * d.QCpad + rl * p;  // first column of run r
  const int lr0 = rl * p;                    // its first row in AAt / Gbuf
  if (pa.mode == kPostZ) {
    for (int e = threadIdx.x; e < d.Lpad * p; e += blockDim.x) {
      const int l = e / p, i = e % p;
      const double* yrow = pa.Y + static_cast<size_t>(l) * d.Qs + c0;
      double s = 0.0;
      for (int m = 0; m < p; ++m) s += yrow[m] * pa.AAt[static_cast<size_t>(lr0 + m) * d.Qs + c0 + i];
      pa.Z[static_cast<size_t>(l) * d.Qs + c0 + i] = pa.XAt[static_cast<size_t>(l) * d.Qs + c0 + i] - s;
    }
    return;
  }
  // G = YᵀY, summed over bands in ascending order with separate multiply and
  // add (matrix.cpp:97-112 applied to m = XB, as spectral_norm's Gram).
  __shared__ double gram[kMaxP * kMaxP];
  for (int e = threadIdx.x; e < p * p; e += blockDim.x) {
    const int i = e / p, m = e % p;
    double s = 0.0;
    for (int l = 0; l < d.L; ++l)
      s = __dadd_rn(s, __dmul_rn(pa.Y[static_cast<size_t>(l) * d.Qs + c0 + i],
                                 pa.Y[static_cast<size_t>(l) * d.Qs + c0 + m]));
    gram[e] = s;
    pa.Gbuf[static_cast<size_t>(lr0 + i) * d.Qs + c0 + m] = s;
  }
  if (pa.mode != kPostInit) return;
  __syncthreads();
  if (threadIdx.x != 0) return;
  // step_sizes (solver.cpp:138-149): ‖XB⁰‖_F == 0 check, then spectral_norm.
  double fro = 0.0;
  bool finite = true;
  for (int l = 0; l < d.L; ++l)
    for (int i = 0; i < p; ++i) {
      const double v = pa.Y[static_cast<size_t>(l) * d.Qs + c0 + i];
      finite &= isfinite(v);
      fro = __dadd_rn(fro, __dmul_rn(v, v));
    }
  if (finite && sqrt(fro) == 0.0) {
    pa.fail_code[r] = kDegenerateInit;
    return;
  }
  if (!finite || !(sqrt(fro) != 0.0)) {
    pa.fail_code[r] = kSpectralBad;
    return;
  }
  // power iteration, matrix.cpp:154-189 (all-ones start, stop at tol/16)
  double v[kMaxP], gv[kMaxP];
  for (int i = 0; i < p; ++i) v[i] = 1.0 / sqrt(static_cast<double>(p));
  double lambda = 0.0;
  const double stop = 1e-6 / 16.0;
  const int max_iters = 1000;
  double sigma = -1.0;
  for (int it = 0; it < max_iters; ++it) {
    for (int i = 0; i < p; ++i) {
      double s = 0.0;
      for (int m = 0; m < p; ++m) s = __dadd_rn(s, __dmul_rn(gram[i * p + m], v[m]));
      gv[i] = s;
    }
    double next = 0.0;
    for (int i = 0; i < p; ++i) next = __dadd_rn(next, __dmul_rn(v[i], gv[i]));
    double norm = 0.0;
    for (int i = 0; i < p; ++i) norm = __dadd_rn(norm, __dmul_rn(gv[i], gv[i]));
    norm = sqrt(norm);
    if (norm == 0.0) {
      for (int i = 0; i < p; ++i) v[i] = 0.0;
      v[it % p] = 1.0;
      continue;
    }
    for (int i = 0; i < p; ++i) v[i] = gv[i] / norm;
    if (it > 0 && fabs(next - lambda) <= stop * fabs(next)) {
      sigma = sqrt(next);
      break;
    }
    lambda = next;
  }
  if (sigma < 0.0) {
    pa.fail_code[r] = kSpectralNoConv;
    pa.fail_value[r] = sqrt(fabs(lambda));
    return;
  }
  const double ea = pa.gamma[r] / __dmul_rn(sigma, sigma);
  pa.eta_a[r] = ea;
  pa.eta_b[r] = __dmul_rn(sqrt(static_cast<double>(p) / static_cast<double>(d.N)), ea);
}

template <class XT>
__global__ void k_xnorm(const XT* X, double* xnorm, Dims d) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= d.Npad) return;
  double s = 0.0;
  for (int l = 0; l < d.L; ++l) {
    const double v = X[static_cast<size_t>(l) * d.Npad + j];
    s += v * v;
  }
  xnorm[j] = s;
}

// b = exp(ℓ − m)/S, laid out like the logits: [M·p][Npad].
__global__ void k_materialize_b(const double* Lg, const double* colm, const double* colS,
                                double* Bv, Dims d) {
  const int col = blockIdx.y;  // r·p + i
  const int r = col / d.p, i = col % d.p;
  const int gc = (r / d.RC) * d.QCpad + (r % d.RC) * d.p + i;
  const double m = colm[gc], S = colS[gc];
  for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < d.Npad; j += gridDim.x * blockDim.x) {
    const size_t idx = static_cast<size_t>(col) * d.Npad + j;
    Bv[idx] = (j < d.N) ? exp(Lg[idx] - m) / S : 0.0;
  }
}

// E = X·B̂ in the reference's accumulation order (matrix.cpp:64-73: pixel
// index ascending, multiply then add, from 0.0) so E is bitwise the host
// matmul(X, B̂) of the same fp32-exact X. Output [M][Lpad][p].
template <class XT>
__global__ void __launch_bounds__(256) k_strict_e(const XT* X, const double* Bv, double* E, Dims d) {
  // One output per thread (8 band rows × 32 columns per CTA): the pixel-ascending
  // chain is inherently sequential, so throughput comes from running many chains
  // (L·M·p of them) on every SM at once.  The next 128-pixel chunk of X and B̂ is
  // loaded into registers while the current one is consumed from shared memory,
  // so the chains run at the dependent-DADD rate instead of waiting on L2 per chunk.
  constexpr int kJ = 128;
  constexpr int kXE = 8 * kJ / 256, kBE = 32 * kJ / 256;  // elements per thread per chunk
  __shared__ double xs[8][kJ];
  __shared__ double bs[32][kJ + 1];
  const int lane = threadIdx.x & 31, ry = threadIdx.x >> 5;
  const int l0 = blockIdx.x * 8, c0 = blockIdx.y * 32;
  const int ncol = d.M * d.p;
  double rx[kXE], rb[kBE];
  auto fetch = [&](int j0) {
#pragma unroll
    for (int k = 0; k < kXE; ++k) {
      const int e = threadIdx.x + 256 * k, rr = e / kJ, jj = e % kJ;
      const int l = l0 + rr, j = j0 + jj;
      rx[k] = (l < d.L && j < d.N) ? static_cast<double>(X[static_cast<size_t>(l) * d.Npad + j]) : 0.0;
    }
#pragma unroll
    for (int k = 0; k < kBE; ++k) {
      const int e = threadIdx.x + 256 * k, rr = e / kJ, jj = e % kJ;
      const int c = c0 + rr, j = j0 + jj;
      rb[k] = (c < ncol && j < d.N) ? Bv[static_cast<size_t>(c) * d.Npad + j] : 0.0;
    }
  };
  auto stage = [&]() {
#pragma unroll
    for (int k = 0; k < kXE; ++k) {
      const int e = threadIdx.x + 256 * k;
      xs[e / kJ][e % kJ] = rx[k];
    }
#pragma unroll
    for (int k = 0; k < kBE; ++k) {
      const int e = threadIdx.x + 256 * k;
      bs[e / kJ][e % kJ] = rb[k];
    }
  };
  double s = 0.0;
  fetch(0);
  stage();
  __syncthreads();
  for (int j0 = 0; j0 < d.N; j0 += kJ) {
    if (j0 + kJ < d.N) fetch(j0 + kJ);  // in flight during the chain below
    if (d.N - j0 >= kJ) {
#pragma unroll 16
      for (int jj = 0; jj < kJ; ++jj) s = __dadd_rn(s, __dmul_rn(xs[ry][jj], bs[lane][jj]));
    } else {
      for (int jj = 0; jj < d.N - j0; ++jj) s = __dadd_rn(s, __dmul_rn(xs[ry][jj], bs[lane][jj]));
    }
    __syncthreads();
    if (j0 + kJ < d.N) {
      stage();
      __syncthreads();
    }
  }
  const int c = c0 + lane;
  const int l = l0 + ry;
  if (c >= ncol || l >= d.L) return;
  const int r = c / d.p, i = c % d.p;
  E[(static_cast<size_t>(r) * d.Lpad + l) * d.p + i] = s;
}

// fit_l1 = Σ |X − E·A| (ensemble.cpp:29-39). Per element the reconstruction
// follows matmul's order (endmember index ascending, multiply then add);
// the sum over elements is a fixed-order tree (per block) then a fixed-order
// sum over blocks.
template <class XT>
__global__ void __launch_bounds__(256) k_fit_partial(const XT* X, const double* E, const double* A,
                                                     double* part, int nblk, Dims d) {
  __shared__ double es[kMaxLpad * kMaxP];
  __shared__ double red[256];
  const int r = blockIdx.y;
  const int p = d.p;
  for (int e = threadIdx.x; e < d.L * p; e += blockDim.x)
    es[e] = E[static_cast<size_t>(r) * d.Lpad * p + e];
  __syncthreads();
  double tot = 0.0;
  for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < d.N; j += nblk * blockDim.x) {
    double a[kMaxP];
    for (int i = 0; i < p; ++i) a[i] = A[(static_cast<size_t>(r) * p + i) * d.Npad + j];
    for (int l = 0; l < d.L; ++l) {
      double rec = 0.0;
      for (int i = 0; i < p; ++i) rec = __dadd_rn(rec, __dmul_rn(es[l * p + i], a[i]));
      tot += fabs(static_cast<double>(X[static_cast<size_t>(l) * d.Npad + j]) - rec);
    }
  }
  red[threadIdx.x] = tot;
  __syncthreads();
  for (int w = 128; w > 0; w >>= 1) {
    if (threadIdx.x < w) red[threadIdx.x] += red[threadIdx.x + w];
    __syncthreads();
  }
  if (threadIdx.x == 0) part[static_cast<size_t>(r) * nblk + blockIdx.x] = red[0];
}

__global__ void k_fit_final(const double* part, double* fit, int nblk, int M) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= M) return;
  double s = 0.0;
  for (int b = 0; b < nblk; ++b) s += part[static_cast<size_t>(r) * nblk + b];
  fit[r] = s;
}

// coherence (ensemble.cpp:41-60): raw max_{i<j} ⟨e_i, e_j⟩, reference order.
__global__ void k_coherence(const double* E, double* mu, Dims d) {
  // One warp per run, one lane per endmember pair (i < j): each dot product keeps
  // the reference's band-ascending multiply-then-add chain (ensemble.cpp:41-60), and
  // the max over pairs is order-free (std::max semantics: NaN dots never win).
  const int r = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (r >= d.M) return;
  const int p = d.p, npair = p * (p - 1) / 2;
  const double* e = E + static_cast<size_t>(r) * d.Lpad * p;
  double best = -INFINITY;
  for (int q = lane; q < npair; q += 32) {
    int i = 0, rem = q;
    while (rem >= p - 1 - i) {
      rem -= p - 1 - i;
      ++i;
    }
    const int j = i + 1 + rem;
    double dot = 0.0;
    for (int l = 0; l < d.L; ++l) dot = __dadd_rn(dot, __dmul_rn(e[l * p + i], e[l * p + j]));
    best = max_like_std(best, dot);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) best = max_like_std(best, __shfl_xor_sync(0xffffffffu, best, o));
  if (lane == 0) mu[r] = (best == -INFINITY) ? 0.0 : best;
}

// select_runs (ensemble.cpp:71-94) on device: fit_min over ok runs, cutoff
// fit_slack·fit_min, candidates ascending, strict-< coherence argmin.
__global__ void k_select(const double* fit, const double* mu, const int* fail_code,
                         const unsigned long long* fail_key, int M, double slack,
                         unsigned char* cand, long long* selected, double* fit_min) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  double fmin = INFINITY;
  for (int r = 0; r < M; ++r) {
    const bool ok = fail_code[r] == kOk && fail_key[r] == ~0ull;
    if (ok && fit[r] < fmin) fmin = fit[r];
  }
  if (fmin == INFINITY) {
    *selected = -1;
    *fit_min = fmin;
    for (int r = 0; r < M; ++r) cand[r] = 0;
    return;
  }
  const double cutoff = slack * fmin;
  long long best = -1;
  for (int r = 0; r < M; ++r) {
    const bool ok = fail_code[r] == kOk && fail_key[r] == ~0ull;
    cand[r] = (ok && fit[r] <= cutoff) ? 1 : 0;
    if (cand[r] && (best < 0 || mu[r] < mu[best])) best = r;
  }
  *selected = best;
  *fit_min = fmin;
}

}  // namespace

size_t pass_smem_bytes(const Dims& d, int nbuf) { return dev::smem_layout(d, nbuf).total; }

#define EDAA_DECL_PASS(X)                                             \
  cudaError_t launch_pass_##X##_init(const PassArgs&, cudaStream_t); \
  cudaError_t launch_pass_##X##_b(const PassArgs&, cudaStream_t);    \
  cudaError_t launch_pass_##X##_obj(const PassArgs&, cudaStream_t);  \
  cudaError_t launch_pass_##X##_alo(const PassArgs&, cudaStream_t);  \
  cudaError_t launch_pass_##X##_ahi(const PassArgs&, cudaStream_t);
EDAA_DECL_PASS(f32)
EDAA_DECL_PASS(f64)
#undef EDAA_DECL_PASS

cudaError_t launch_pass(int mode, const PassArgs& a, cudaStream_t st) {
  const bool f64 = a.d.xbytes == 8;
  const bool lo = a.d.p <= 5;
  switch (mode) {
    case kModeInit: return f64 ? launch_pass_f64_init(a, st) : launch_pass_f32_init(a, st);
    case kModeB:
      if (!f64 && a.d.npl == 2 && a.kprof == nullptr) return launch_pass_b64(a, st);
      return f64 ? launch_pass_f64_b(a, st) : launch_pass_f32_b(a, st);
    case kModeObj: return f64 ? launch_pass_f64_obj(a, st) : launch_pass_f32_obj(a, st);
    case kModeA:
      if (f64) return lo ? launch_pass_f64_alo(a, st) : launch_pass_f64_ahi(a, st);
      return lo ? launch_pass_f32_alo(a, st) : launch_pass_f32_ahi(a, st);
  }
  return cudaErrorInvalidValue;
}


cudaError_t launch_combine(const CombineArgs& a, cudaStream_t st) {
  const Dims& d = a.d;
  if (a.mode == kModeObj) {  // the final objective only
    cudaError_t e0 = launch_pdl(d.pdl != 0, k_rowsum, dim3(1, 1), dim3(32, 8), 0, st, a, 0);
    if (e0 != cudaSuccess) return e0;
    return cudaGetLastError();
  }
  if (a.mode != kModeA) {  // B step / init: normalisers, Y and Z in one kernel
    // rows per CTA: the largest of 8, 4, 2, 1 that still gives at least one CTA per SM
    int br = kBRMax;
    while (br > 1 && d.NCH * ((d.Lpad + br - 1) / br) < d.ncta) br >>= 1;
    const size_t smem = static_cast<size_t>(d.nslices) * kQMax * sizeof(double);
    void (*kern)(CombineArgs) = br >= kBRMax ? k_combine_b<kBRMax> : br >= 8 ? k_combine_b<8> : br >= 4 ? k_combine_b<4>
                                : br >= 2     ? k_combine_b<2>
                                              : k_combine_b<1>;
    const int rows = br >= kBRMax ? kBRMax : br >= 8 ? 8 : br >= 4 ? 4 : br >= 2 ? 2 : 1;
    // a constant, set on whichever device is current (per-device, per-function state)
    const cudaError_t ea = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                kMaxSlices * kQMax * static_cast<int>(sizeof(double)));
    if (ea != cudaSuccess) return ea;
    return launch_pdl(d.pdl != 0, kern, dim3(d.NCH, (d.Lpad + rows - 1) / rows), dim3(256), smem, st, a);
  }
  launch_pdl(d.pdl != 0, k_aat, dim3(d.NCH, (d.RC * d.p * d.p + 7) / 8 + 1), dim3(256), 0, st, a);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  launch_pdl(d.pdl != 0, k_combine, dim3(d.NCH, (d.Lpad + kCR - 1) / kCR), dim3(256), 0, st, a);
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// Pixel sharding, allreduce exchange (north_star: "NCCL allreduce of the L×p and
// p×p partial sums").  Each rank reduces the partials of the slices it owns into
// ONE block of Lrows×Qs (+ 2·Qs + M) doubles, the blocks are summed across ranks
// (log-sum-exp aware for the B step: column maxima first), and the unchanged
// combine kernels finish from the reduced block as if it were a single slice.
//   block layout (doubles): C [Lrows][Qs] | S [Qs] | obj [M] | m [Qs] | m_glob [Qs]
__host__ __device__ inline size_t red_off_S(const Dims& d) { return static_cast<size_t>(d.Lrows) * d.Qs; }
__host__ __device__ inline size_t red_off_obj(const Dims& d) { return red_off_S(d) + d.Qs; }
__host__ __device__ inline size_t red_off_m(const Dims& d) { return red_off_obj(d) + d.M; }
__host__ __device__ inline size_t red_off_mg(const Dims& d) { return red_off_m(d) + d.Qs; }

// B / init: per column, the max m_r of the owned slices' maxima, the rescale
// factors e^{m_s − m_r} (into ca.fac) and S_r = Σ_s S_s·e^{m_s − m_r}.  One warp
// per column, lanes stride the slices, fixed xor tree.
__global__ void k_shard_colmax(CombineArgs ca, int s0, int s1, double* red) {
  const Dims& d = ca.d;
  const int col = blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (col >= d.Qs) return;
  double m = -INFINITY;
  for (int sl = s0 + lane; sl < s1; sl += 32) m = fmax(m, ca.part_m[static_cast<size_t>(sl) * d.Qs + col]);
  m = warp_max(m);
  double S = 0.0;
  for (int sl = s0 + lane; sl < s1; sl += 32) {
    const double ms = ca.part_m[static_cast<size_t>(sl) * d.Qs + col];
    const double f = (ms == -INFINITY) ? 0.0 : exp(ms - m);
    ca.fac[static_cast<size_t>(sl) * d.Qs + col] = f;
    S += ca.part_S[static_cast<size_t>(sl) * d.Qs + col] * f;
  }
  S = warp_sum(S);
  if (lane == 0) {
    red[red_off_m(d) + col] = m;
    red[red_off_S(d) + col] = S;
  }
}

// Rows of the block: Σ_s C_s (A) or Σ_s C_s·e^{m_s − m_r} (B / init), slices in
// ascending order; block (0,0) also folds the owned slices' objective terms.
__global__ void k_shard_rowsum(CombineArgs ca, int s0, int s1, int rows, double* red) {
  const Dims& d = ca.d;
  const bool lse = ca.mode == kModeB || ca.mode == kModeInit;
  if (!lse && blockIdx.x == 0 && blockIdx.y == 0) {
    for (int r = threadIdx.y * 32 + threadIdx.x; r < d.M; r += 256) {
      double o = 0.0;
      for (int sl = s0; sl < s1; ++sl) o += ca.part_obj[static_cast<size_t>(sl) * d.M + r];
      red[red_off_obj(d) + r] = o;
    }
  }
  const int col = blockIdx.x * 32 + threadIdx.x;
  const int row = blockIdx.y * 8 + threadIdx.y;
  if (col >= d.Qs || row >= rows) return;
  const double* src = ca.part_C + static_cast<size_t>(row) * d.Qs + col;
  const size_t sstride = static_cast<size_t>(d.Lrows) * d.Qs;
  double s = 0.0;
  if (lse) {
    for (int sl = s0; sl < s1; ++sl) s += src[sl * sstride] * ca.fac[static_cast<size_t>(sl) * d.Qs + col];
  } else {
    for (int sl = s0; sl < s1; ++sl) s += src[sl * sstride];
  }
  red[static_cast<size_t>(row) * d.Qs + col] = s;
}

// B / init, after the column maxima were max-reduced across ranks: bring the
// rank's block to the common reference, C ← C·e^{m_r − m}, S ← S·e^{m_r − m}.
__global__ void k_shard_rescale(Dims d, double* red, const double* m_glob) {
  const int col = blockIdx.x * 32 + threadIdx.x;
  if (col >= d.Qs) return;
  const double mr = red[red_off_m(d) + col], mg = m_glob[col];
  const double f = (mr == -INFINITY) ? 0.0 : exp(mr - mg);
  for (int row = blockIdx.y * 8 + threadIdx.y; row < d.Lpad; row += gridDim.y * 8)
    red[static_cast<size_t>(row) * d.Qs + col] *= f;
  if (blockIdx.y == 0 && threadIdx.y == 0) red[red_off_S(d) + col] *= f;
}

// One-device emulation of the two collectives (tests): blocks of `world` ranks
// `stride` doubles apart; the max of their m into block 0's m_glob, and the sum
// of their first `n` doubles, in rank order, into block 0.
__global__ void k_shard_emul_max(Dims d, double* red, size_t stride, int world) {
  const int col = blockIdx.x * blockDim.x + threadIdx.x;
  if (col >= d.Qs) return;
  double m = -INFINITY;
  for (int q = 0; q < world; ++q) m = fmax(m, red[q * stride + red_off_m(d) + col]);
  red[red_off_mg(d) + col] = m;
}
__global__ void k_shard_emul_sum(double* red, size_t stride, int world, size_t n) {
  const size_t e = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (e >= n) return;
  double s = red[e];
  for (int q = 1; q < world; ++q) s += red[q * stride + e];
  red[e] = s;
}

// Final state exchange: a rank's pixel columns [j0, j0+w) of a [rows][Npad] array
// to / from a dense [rows][wmax] staging block (one all-gather per array).
__global__ void k_pack_cols(const double* src, double* stage, int rows, int Npad, int j0, int w, int wmax) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= w) return;
  for (int r = blockIdx.y; r < rows; r += gridDim.y)
    stage[static_cast<size_t>(r) * wmax + j] = src[static_cast<size_t>(r) * Npad + j0 + j];
}
__global__ void k_unpack_cols(double* dst, const double* stage, int rows, int Npad, int j0, int w, int wmax) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= w) return;
  for (int r = blockIdx.y; r < rows; r += gridDim.y)
    dst[static_cast<size_t>(r) * Npad + j0 + j] = stage[static_cast<size_t>(r) * wmax + j];
}

size_t shard_red_doubles(const Dims& d) { return red_off_mg(d) + d.Qs; }
size_t shard_red_sum_doubles(const Dims& d) { return red_off_m(d); }
size_t shard_red_off(const Dims& d, int what) {
  return what == 0 ? 0 : what == 1 ? red_off_S(d) : what == 2 ? red_off_obj(d) : what == 3 ? red_off_m(d) : red_off_mg(d);
}

cudaError_t launch_shard_reduce(const CombineArgs& a, int s0, int s1, double* red, cudaStream_t st) {
  const Dims& d = a.d;
  const bool lse = a.mode == kModeB || a.mode == kModeInit;
  if (lse) k_shard_colmax<<<(d.Qs + 7) / 8, 256, 0, st>>>(a, s0, s1, red);
  const int rows = a.mode == kModeObj ? 0 : (lse ? d.Lpad : d.Lrows);
  k_shard_rowsum<<<dim3((d.Qs + 31) / 32, std::max(1, (rows + 7) / 8)), dim3(32, 8), 0, st>>>(a, s0, s1, rows, red);
  return cudaGetLastError();
}
cudaError_t launch_shard_rescale(const Dims& d, double* red, const double* m_glob, cudaStream_t st) {
  k_shard_rescale<<<dim3((d.Qs + 31) / 32, std::min(32, (d.Lpad + 7) / 8)), dim3(32, 8), 0, st>>>(d, red, m_glob);
  return cudaGetLastError();
}
cudaError_t launch_shard_emul_max(const Dims& d, double* red, size_t stride, int world, cudaStream_t st) {
  k_shard_emul_max<<<(d.Qs + 127) / 128, 128, 0, st>>>(d, red, stride, world);
  return cudaGetLastError();
}
cudaError_t launch_shard_emul_sum(double* red, size_t stride, int world, size_t n, cudaStream_t st) {
  k_shard_emul_sum<<<static_cast<unsigned>((n + 255) / 256), 256, 0, st>>>(red, stride, world, n);
  return cudaGetLastError();
}
cudaError_t launch_pack_cols(const double* src, double* stage, int rows, int Npad, int j0, int w, int wmax,
                             bool unpack, double* dst, cudaStream_t st) {
  if (w <= 0 || rows <= 0) return cudaSuccess;
  const dim3 grid((w + 255) / 256, std::min(rows, 1024));
  if (unpack)
    k_unpack_cols<<<grid, 256, 0, st>>>(dst, stage, rows, Npad, j0, w, wmax);
  else
    k_pack_cols<<<grid, 256, 0, st>>>(src, stage, rows, Npad, j0, w, wmax);
  return cudaGetLastError();
}

cudaError_t launch_post(const PostArgs& a, cudaStream_t st) {
  if (a.mode == kPostG)
    launch_pdl(a.d.pdl != 0, k_gram, dim3(a.d.M), dim3(256), 0, st, a);
  else
    launch_pdl(a.d.pdl != 0, k_post, dim3(a.d.M), dim3(256), 0, st, a);
  return cudaGetLastError();
}

cudaError_t launch_xnorm(const void* X, double* xnorm, const Dims& d, cudaStream_t st) {
  if (d.xbytes == 8)
    k_xnorm<<<(d.Npad + 255) / 256, 256, 0, st>>>(static_cast<const double*>(X), xnorm, d);
  else
    k_xnorm<<<(d.Npad + 255) / 256, 256, 0, st>>>(static_cast<const float*>(X), xnorm, d);
  return cudaGetLastError();
}

cudaError_t launch_materialize_b(const double* Lg, const double* colm, const double* colS,
                                 double* Bv, const Dims& d, cudaStream_t st) {
  const dim3 grid(static_cast<unsigned>(std::min(64, (d.Npad + 255) / 256)), d.M * d.p);
  k_materialize_b<<<grid, 256, 0, st>>>(Lg, colm, colS, Bv, d);
  return cudaGetLastError();
}

cudaError_t launch_strict_e(const void* X, const double* Bv, double* E, const Dims& d,
                            cudaStream_t st) {
  const dim3 grid((d.L + 7) / 8, (d.M * d.p + 31) / 32);
  if (d.xbytes == 8)
    k_strict_e<<<grid, 256, 0, st>>>(static_cast<const double*>(X), Bv, E, d);
  else
    k_strict_e<<<grid, 256, 0, st>>>(static_cast<const float*>(X), Bv, E, d);
  return cudaGetLastError();
}

cudaError_t launch_fit(const void* X, const double* E, const double* A, double* part_fit,
                       double* fit, int fit_blocks, const Dims& d, cudaStream_t st) {
  if (d.xbytes == 8)
    k_fit_partial<<<dim3(fit_blocks, d.M), 256, 0, st>>>(static_cast<const double*>(X), E, A, part_fit, fit_blocks, d);
  else
    k_fit_partial<<<dim3(fit_blocks, d.M), 256, 0, st>>>(static_cast<const float*>(X), E, A, part_fit, fit_blocks, d);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  k_fit_final<<<(d.M + 127) / 128, 128, 0, st>>>(part_fit, fit, fit_blocks, d.M);
  return cudaGetLastError();
}

cudaError_t launch_coherence(const double* E, double* mu, const Dims& d, cudaStream_t st) {
  k_coherence<<<(d.M + 3) / 4, 128, 0, st>>>(E, mu, d);
  return cudaGetLastError();
}

cudaError_t launch_select(const double* fit, const double* mu, const int* fail_code,
                          const unsigned long long* fail_key, int M, double slack,
                          unsigned char* cand, long long* selected, double* fit_min,
                          cudaStream_t st) {
  k_select<<<1, 32, 0, st>>>(fit, mu, fail_code, fail_key, M, slack, cand, selected, fit_min);
  return cudaGetLastError();
}

}  // namespace edaa