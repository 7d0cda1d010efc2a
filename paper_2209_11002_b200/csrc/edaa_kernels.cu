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
#include <cmath>
#include <cstdio>

#include "edaa_internal.cuh"

namespace edaa {

namespace {

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

struct SmemLayout {
  int xs_off, ws_off, ss_off, sh_off, st_off, gs_off, col_off, total;
};

__host__ __device__ inline int align16(int b) { return (b + 15) & ~15; }

// W row stride (doubles): ≡ 8 mod 16 so a DMMA A-fragment (4 rows × 8 columns) hits 2 wavefronts.
__host__ __device__ inline int w_stride(int qcpad) { return qcpad + ((qcpad % 16 == 0) ? 8 : 0); }

__host__ __device__ inline SmemLayout smem_layout(const Dims& d, int /*nbuf*/) {
  SmemLayout s;
  int off = 0;
  s.xs_off = off;  // X tile, fp32 [Lpad][kXST]
  off += align16(d.Lpad * kXST * 4);
  s.ws_off = off;  // W chunk, fp64 [Lpad][WST]
  off += align16(d.Lpad * w_stride(d.QCpad) * 8);
  s.ss_off = off;  // projection / weights, fp64 [QCpad][kSST]
  off += align16(d.QCpad * kSST * 8);
  s.sh_off = off;  // second half of the band-split projection
  off += align16(d.QCpad * kSST * 8);
  s.st_off = off;  // state tile (A or logits) of the chunk, fp64 [QCpad][kNP]
  off += align16(d.QCpad * kNP * 8);
  s.gs_off = off;
  off += align16(d.RC * d.p * d.p * 8);
  s.col_off = off;  // m_run, S_run, fac, hmax, hsum (QCpad each) + obj_run (RC), hobj (4·RC)
  off += align16((5 * d.QCpad + 5 * d.RC) * 8);
  s.total = off;
  return s;
}

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

// ---------------------------------------------------------------------------
// Per-pixel A update: objective term + K1 entropic steps (solver.cpp:212-218),
// one pixel of one run per group of TPP lanes, each lane owning EPT of the p
// entries.  P (= Yᵀx_j) is the sum of the two band halves in ss/sh, G = YᵀY
// of the run and the pixel's current a are in shared memory.
// The softmax of solver.cpp:20-36, softmax(log max(a, 1e-30) + u) with
// u = η_a·(P − G·a), is evaluated in the equivalent multiplicative form
// a_i ← max(a_i,1e-30)·e^{u_i − max u} / Σ — the same shift-invariant
// quantity (every term ≤ 1, the largest ≥ 1e-30, so it neither overflows
// nor vanishes) without the logarithms.
// Returns the pixel's objective term ½‖x_j − Y a_j‖² = ½(‖x_j‖² − 2aᵀP + aᵀGa)
// for the pre-update a (on the group's sub-0 lane, 0 elsewhere).
template <int PT>
struct LanesPerPixel {
  static constexpr int value = PT <= 4 ? 1 : (PT <= 8 ? 2 : 4);
};

template <int PT, int TPP, bool UPDATE>
__device__ __forceinline__ double pixel_a_update(const PassArgs& pa, int r, int rl, int j, int pix,
                                                 bool valid, int sub, double* ss, const double* sh,
                                                 const double* st, const double* gs) {
  constexpr int EPT = (PT + TPP - 1) / TPP;
  const Dims& d = pa.d;
  const int p = d.p;
  const int gbase = (threadIdx.x & 31) - sub;
  double a[EPT], P[EPT];
#pragma unroll
  for (int e = 0; e < EPT; ++e) {
    const int i = sub * EPT + e;
    a[e] = 0.0;
    P[e] = 0.0;
    if (i < p) {
      const int c = rl * p + i;
      a[e] = st[c * kNP + j];
      P[e] = ss[c * kSST + j] + sh[c * kSST + j];
    }
  }
  const double* G = gs + rl * p * p;
  const double eta = pa.eta_a[r];
  double aPa = 0.0, aGa = 0.0;
  bool bad = false;
  const int steps = UPDATE ? d.K1 : 1;
  for (int k = 0; k < steps; ++k) {
    double ga[EPT];
#pragma unroll
    for (int e = 0; e < EPT; ++e) ga[e] = 0.0;
#pragma unroll
    for (int m = 0; m < PT; ++m) {
      if (m < p) {
        const double am = (TPP == 1) ? a[m % EPT] : __shfl_sync(0xffffffffu, a[m % EPT], gbase + m / EPT);
#pragma unroll
        for (int e = 0; e < EPT; ++e) {
          const int i = sub * EPT + e;
          if (i < p) ga[e] += G[i * p + m] * am;
        }
      }
    }
    double u[EPT];
    double umax = -INFINITY;
#pragma unroll
    for (int e = 0; e < EPT; ++e) {
      u[e] = -INFINITY;
      if (sub * EPT + e < p) {
        if (k == 0) {
          aPa += a[e] * P[e];
          aGa += a[e] * ga[e];
        }
        u[e] = (P[e] - ga[e]) * eta;  // −∇_A = (XB)ᵀ(X − XBA) = P − G·a, times η_a
        umax = fmax(umax, u[e]);
      }
    }
    if (!UPDATE) break;
#pragma unroll
    for (int o = 1; o < TPP; o <<= 1) umax = fmax(umax, __shfl_xor_sync(0xffffffffu, umax, o));
    double total = 0.0;
#pragma unroll
    for (int e = 0; e < EPT; ++e) {
      if (sub * EPT + e < p) {
        const double z = (a[e] < kLogFloorValue) ? kLogFloorValue : a[e];  // std::max(z, 1e-30)
        a[e] = z * exp(u[e] - umax);
        total += a[e];
      }
    }
#pragma unroll
    for (int o = 1; o < TPP; o <<= 1) total += __shfl_xor_sync(0xffffffffu, total, o);
    const double inv = 1.0 / total;
#pragma unroll
    for (int e = 0; e < EPT; ++e) {
      const int i = sub * EPT + e;
      if (i < p) {
        a[e] *= inv;
        bad |= !isfinite(a[e]);
        if (pa.observe_A != nullptr && valid)
          pa.observe_A[(static_cast<size_t>(k) * p + i) * d.Npad + pix] = a[e];
      }
    }
  }
#pragma unroll
  for (int o = 1; o < TPP; o <<= 1) {
    aPa += __shfl_xor_sync(0xffffffffu, aPa, o);
    aGa += __shfl_xor_sync(0xffffffffu, aGa, o);
  }
  if (UPDATE) {
    if (bad && valid) atomicMin(pa.fail_key + r, static_cast<unsigned long long>(pa.t) << 1);
    const size_t base = static_cast<size_t>(r) * p * d.Npad + pix;
#pragma unroll
    for (int e = 0; e < EPT; ++e) {
      const int i = sub * EPT + e;
      if (i < p) {
        if (valid) pa.A[base + static_cast<size_t>(i) * d.Npad] = a[e];
        ss[(rl * p + i) * kSST + j] = valid ? a[e] : 0.0;
      }
    }
  }
  return (valid && sub == 0) ? 0.5 * ((pa.xnorm[pix] - 2.0 * aPa) + aGa) : 0.0;
}

// X tile (rows < L) and the chunk's state rows (A or logits) for pixels
// [j0, j0+kNP), 16-byte cp.async into shared memory, one commit group.
template <int MODE>
__device__ __forceinline__ void load_tile(const PassArgs& pa, float* xs, double* st, int j0,
                                          int state_row0, int nstate) {
  const Dims& d = pa.d;
  for (int e = threadIdx.x; e < d.L * (kNP / 4); e += kThreads) {
    const int l = e / (kNP / 4), q = e % (kNP / 4);
    cp_async16(xs + l * kXST + q * 4, pa.X + static_cast<size_t>(l) * d.Npad + j0 + q * 4);
  }
  if (MODE != kModeInit) {
    const double* src = (MODE == kModeB) ? pa.Lg : pa.A;
    for (int e = threadIdx.x; e < nstate * (kNP / 2); e += kThreads) {
      const int c = e / (kNP / 2), q = e % (kNP / 2);
      cp_async16(st + c * kNP + q * 2, src + static_cast<size_t>(state_row0 + c) * d.Npad + j0 + q * 2);
    }
  }
  cp_async_commit();
}

// ---------------------------------------------------------------------------
// The pass kernel. grid = (nslices, NCH), block = 256, two CTAs per SM so one
// CTA's per-pixel phase overlaps the other's DMMA phases.
template <int MODE, int PT, int RTW, int MINB>
__global__ void __launch_bounds__(kThreads, MINB) k_pass(PassArgs pa) {
  extern __shared__ __align__(16) unsigned char smem[];
  const Dims& d = pa.d;
  const SmemLayout lay = smem_layout(d, 1);
  float* xs = reinterpret_cast<float*>(smem + lay.xs_off);
  double* ws = reinterpret_cast<double*>(smem + lay.ws_off);
  double* ss = reinterpret_cast<double*>(smem + lay.ss_off);
  double* sh = reinterpret_cast<double*>(smem + lay.sh_off);
  double* st = reinterpret_cast<double*>(smem + lay.st_off);
  double* gs = reinterpret_cast<double*>(smem + lay.gs_off);
  double* m_run = reinterpret_cast<double*>(smem + lay.col_off);
  double* S_run = m_run + d.QCpad;
  double* fac = S_run + d.QCpad;
  double* hmax = fac + d.QCpad;
  double* hsum = hmax + d.QCpad;
  double* obj_run = hsum + d.QCpad;
  double* hobj = obj_run + d.RC;

  const int tid = threadIdx.x;
  const int lane = tid & 31, warp = tid >> 5;
  const int g = lane >> 2, t4 = lane & 3;
  const int slice = blockIdx.x;
  const int chunk = blockIdx.y;
  const int p = d.p;
  const int run0 = chunk * d.RC;
  const int RCe = min(d.RC, d.M - run0);  // runs present in this chunk
  const int ncol_valid = RCe * p;
  const int nCT = d.QCpad / 8;
  const int nRTx = d.Lpad / 8;
  const int nRT = (MODE == kModeA) ? nRTx + d.QCpad / 8 : nRTx;
  const int WST = w_stride(d.QCpad);
  const int col0 = chunk * d.QCpad;
  const int srow0 = run0 * p;  // first state row (A / Lg) of this chunk

  const int tile_begin = static_cast<int>((static_cast<long long>(slice) * d.ntiles) / d.nslices);
  const int tile_end = static_cast<int>((static_cast<long long>(slice + 1) * d.ntiles) / d.nslices);

  // first tile in flight while the constants are staged
  load_tile<MODE>(pa, xs, st, tile_begin * kNP, srow0, ncol_valid);

  // ---- one-time staging: W chunk, G blocks, zero pad rows, running state ----
  if (MODE == kModeA || MODE == kModeB || MODE == kModeObj) {
    for (int e = tid; e < d.Lpad * d.QCpad; e += kThreads) {
      const int l = e / d.QCpad, c = e % d.QCpad;
      ws[l * WST + c] = pa.W[static_cast<size_t>(l) * d.Qs + col0 + c];
    }
  }
  if (MODE == kModeA || MODE == kModeObj) {
    for (int e = tid; e < RCe * p * p; e += kThreads) {
      const int rl = e / (p * p), rem = e % (p * p);
      const int i = rem / p, m = rem % p;
      gs[e] = pa.Gbuf[static_cast<size_t>(rl * p + i) * d.Qs + col0 + rl * p + m];
    }
  }
  for (int e = tid; e < (d.Lpad - d.L) * kNP; e += kThreads)
    xs[(d.L + e / kNP) * kXST + e % kNP] = 0.0f;
  if (tid < d.QCpad) {
    m_run[tid] = -INFINITY;
    S_run[tid] = 0.0;
    fac[tid] = 1.0;
  }
  if (tid < d.RC) obj_run[tid] = 0.0;

  double acc[RTW][kMaxCT][2];
#pragma unroll
  for (int i = 0; i < RTW; ++i)
#pragma unroll
    for (int c = 0; c < kMaxCT; ++c) acc[i][c][0] = acc[i][c][1] = 0.0;

  for (int tile = tile_begin; tile < tile_end; ++tile) {
    const int j0 = tile * kNP;
    cp_async_wait0();
    __syncthreads();

    // ---- phase 1: S[c][j] = Σ_l W[l][c]·X[l][j]  (DMMA; warp = 8 pixels × one band half) ----
    if (MODE != kModeInit) {
      const int pt = warp & 3, half = warp >> 2;
      const int kh = d.Lpad / 8;  // k-steps per band half
      double c1[kMaxCT][2];
#pragma unroll
      for (int c = 0; c < kMaxCT; ++c) c1[c][0] = c1[c][1] = 0.0;
      const float* xcol = xs + pt * 8 + g;
      const double* wcol = ws + g;
      for (int kk = half * kh; kk < (half + 1) * kh; ++kk) {
        const int l = kk * 4 + t4;
        const double bx = static_cast<double>(xcol[l * kXST]);
#pragma unroll
        for (int ct = 0; ct < kMaxCT; ++ct)
          if (ct < nCT) dmma(c1[ct], wcol[l * WST + ct * 8], bx);
      }
      double* dst = half ? sh : ss;
#pragma unroll
      for (int ct = 0; ct < kMaxCT; ++ct)
        if (ct < nCT)
          *reinterpret_cast<double2*>(dst + (ct * 8 + g) * kSST + pt * 8 + 2 * t4) =
              make_double2(c1[ct][0], c1[ct][1]);
    }
    __syncthreads();

    // ---- phase 2: per-pixel updates ----
    if (MODE == kModeA || MODE == kModeObj) {
      constexpr int TPP = LanesPerPixel<PT>::value;
      for (int q2 = tid; q2 < RCe * kNP * TPP; q2 += kThreads) {  // warp-uniform trip count
        const int q = q2 / TPP, sub = q2 % TPP;
        const int rl = q / kNP, j = q % kNP;
        const int pix = j0 + j;
        double o = pixel_a_update<PT, TPP, MODE == kModeA>(pa, run0 + rl, rl, j, pix, pix < d.N, sub,
                                                             ss, sh, st, gs);
        o = warp_sum(o);
        if (lane == 0) hobj[q2 >> 5] = o;  // warp-task q2/32 belongs to run (q2/32)/TPP
      }
      if (MODE == kModeA)
        for (int e = tid; e < (d.QCpad - ncol_valid) * kNP; e += kThreads)
          ss[(ncol_valid + e / kNP) * kSST + e % kNP] = 0.0;
      __syncthreads();
      if (tid < RCe) {
        double o = obj_run[tid];
        for (int h = 0; h < TPP; ++h) o += hobj[tid * TPP + h];
        obj_run[tid] = o;
      }
      if (MODE == kModeObj) {
        __syncthreads();
        if (tile + 1 < tile_end) load_tile<MODE>(pa, xs, st, j0 + kNP, srow0, ncol_valid);
        continue;
      }
    } else {  // B step or B⁰ initialisation: new logits, online column max
      constexpr int kPer = kQMax * kNP / kThreads;  // elements per thread at QCpad = kQMax
      double ell[kPer];
      const int per = d.QCpad * kNP / kThreads;
#pragma unroll
      for (int k = 0; k < kPer; ++k) {
        if (k < per) {
          const int e = tid + k * kThreads;  // warp = one column × 32 pixels
          const int c = e / kNP, j = e % kNP;
          const int pix = j0 + j;
          double v = -INFINITY;
          if (c < ncol_valid && pix < d.N) {
            const int rl = c / p, i = c % p, r = run0 + rl;
            if (MODE == kModeInit) {
              // solver.cpp:122-127: column i consumes draws i·N .. i·N+N−1.
              v = 0.1 * splitmix_unit_at(pa.seeds[r], static_cast<uint64_t>(i) * d.N +
                                                          static_cast<uint64_t>(pix));
            } else {
              const int gc = col0 + c;
              double lb = st[c * kNP + j] - pa.colm[gc] - pa.collogS[gc];  // log b_old
              lb = (lb < log_floor()) ? log_floor() : lb;                   // log max(b, 1e-30)
              v = lb + (ss[c * kSST + j] + sh[c * kSST + j]) * pa.eta_b[r]; // + η_b·(−∇_B)
            }
            pa.Lg[static_cast<size_t>(srow0 + c) * d.Npad + pix] = v;
          }
          ell[k] = v;
          const double hm = warp_max(v);
          if (lane == 0) hmax[c] = hm;
        }
      }
      __syncthreads();
#pragma unroll
      for (int k = 0; k < kPer; ++k) {
        if (k < per) {
          const int e = tid + k * kThreads;
          const int c = e / kNP, j = e % kNP;
          const double mn = fmax(m_run[c], hmax[c]);
          const double w = (mn == -INFINITY) ? 0.0 : exp(ell[k] - mn);
          ss[c * kSST + j] = w;
          const double hs = warp_sum(w);
          if (lane == 0) hsum[c] = hs;
        }
      }
      __syncthreads();
      if (tid < d.QCpad) {
        const double mo = m_run[tid];
        const double mn = fmax(mo, hmax[tid]);
        const double f = (mn == -INFINITY || mn == mo) ? 1.0 : exp(mo - mn);
        fac[tid] = f;
        S_run[tid] = S_run[tid] * f + hsum[tid];
        m_run[tid] = mn;
      }
      __syncthreads();
      // rescale running accumulators to the new column max
#pragma unroll
      for (int ct = 0; ct < kMaxCT; ++ct) {
        if (ct < nCT) {
          const double f0 = fac[ct * 8 + 2 * t4], f1 = fac[ct * 8 + 2 * t4 + 1];
          if (f0 != 1.0 || f1 != 1.0) {
#pragma unroll
            for (int i = 0; i < RTW; ++i) {
              acc[i][ct][0] *= f0;
              acc[i][ct][1] *= f1;
            }
          }
        }
      }
    }

    // ---- phase 3: C[l][c] += Σ_j X[l][j]·w[c][j]  (DMMA, warp owns row tiles) ----
    {
      const double* wrow = ss + g * kSST + t4;
#pragma unroll 2
      for (int kk = 0; kk < kNP / 4; ++kk) {
        double bw[kMaxCT];
#pragma unroll
        for (int ct = 0; ct < kMaxCT; ++ct) bw[ct] = (ct < nCT) ? wrow[ct * 8 * kSST + kk * 4] : 0.0;
#pragma unroll
        for (int i = 0; i < RTW; ++i) {
          const int rt = warp + 8 * i;
          if (rt < nRT) {
            double ax;
            if (rt < nRTx)
              ax = static_cast<double>(xs[(rt * 8 + g) * kXST + kk * 4 + t4]);
            else
              ax = ss[((rt - nRTx) * 8 + g) * kSST + kk * 4 + t4];
#pragma unroll
            for (int ct = 0; ct < kMaxCT; ++ct)
              if (ct < nCT) dmma(acc[i][ct], ax, bw[ct]);
          }
        }
      }
    }
    __syncthreads();
    if (tile + 1 < tile_end) load_tile<MODE>(pa, xs, st, j0 + kNP, srow0, ncol_valid);
  }

  // ---- write this CTA's partials ----
  if (MODE != kModeObj) {
#pragma unroll
    for (int i = 0; i < RTW; ++i) {
      const int rt = warp + 8 * i;
      if (rt < nRT) {
        const int row = rt * 8 + g;
#pragma unroll
        for (int ct = 0; ct < kMaxCT; ++ct) {
          if (ct < nCT) {
            double* dst = pa.part_C + (static_cast<size_t>(slice) * d.Lrows + row) * d.Qs + col0 +
                          ct * 8 + 2 * t4;
            *reinterpret_cast<double2*>(dst) = make_double2(acc[i][ct][0], acc[i][ct][1]);
          }
        }
      }
    }
  }
  if (MODE == kModeB || MODE == kModeInit) {
    if (tid < d.QCpad) {
      pa.part_m[static_cast<size_t>(slice) * d.Qs + col0 + tid] = m_run[tid];
      pa.part_S[static_cast<size_t>(slice) * d.Qs + col0 + tid] = S_run[tid];
    }
  } else {
    if (tid < RCe) pa.part_obj[static_cast<size_t>(slice) * d.M + run0 + tid] = obj_run[tid];
  }
}

// ---------------------------------------------------------------------------
// Combine, B/init: per column the log-sum-exp merge of the slice partials,
// m = max_s m_s, S = Σ_s S_s·e^{m_s − m}; one warp per column, lanes stride
// the slices, fixed xor-tree merge (deterministic).
__global__ void k_colnorm(CombineArgs ca) {
  const Dims& d = ca.d;
  const int col = blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (col >= d.Qs) return;
  const int S = d.nslices;
  double m = -INFINITY;
  for (int sl = lane; sl < S; sl += 32) m = fmax(m, ca.part_m[static_cast<size_t>(sl) * d.Qs + col]);
  m = warp_max(m);
  double Ssum = 0.0;
  for (int sl = lane; sl < S; sl += 32) {
    const double ms = ca.part_m[static_cast<size_t>(sl) * d.Qs + col];
    const double f = (ms == -INFINITY) ? 0.0 : exp(ms - m);
    ca.fac[static_cast<size_t>(sl) * d.Qs + col] = f;
    Ssum += ca.part_S[static_cast<size_t>(sl) * d.Qs + col] * f;
  }
  Ssum = warp_sum(Ssum);
  if (lane != 0) return;
  ca.colm[col] = m;
  ca.colS[col] = Ssum;
  ca.collogS[col] = log(Ssum);
  // A column of a real run must have a finite max and a finite positive sum.
  const int chunk = col / d.QCpad, c = col % d.QCpad;
  const int r = chunk * d.RC + c / d.p;
  if (c < d.RC * d.p && r < d.M && !(isfinite(m) && isfinite(Ssum) && Ssum > 0.0))
    atomicMin(ca.fail_key + r, (static_cast<unsigned long long>(ca.t) << 1) | 1ull);
}

// Row sums over slices (fixed order): A mode → XAt / AAt; B/init → Y = Σ C_s·fac_s / S.
// Block (32 columns × 8 rows); block (0,0) also folds the per-run objective.
__global__ void k_rowsum(CombineArgs ca, int rows) {
  const Dims& d = ca.d;
  const int col = blockIdx.x * 32 + threadIdx.x;
  const int row = blockIdx.y * 8 + threadIdx.y;
  const int S = d.nslices;
  if ((ca.mode == kModeA || ca.mode == kModeObj) && blockIdx.x == 0 && blockIdx.y == 0) {
    for (int r = threadIdx.y * 32 + threadIdx.x; r < d.M; r += 256) {
      double o = 0.0;
      for (int sl = 0; sl < S; ++sl) o += ca.part_obj[static_cast<size_t>(sl) * d.M + r];
      ca.trace[static_cast<size_t>(r) * ca.trace_stride + ca.trace_index] = o;
    }
  }
  if (col >= d.Qs || row >= rows) return;
  const double* src = ca.part_C + static_cast<size_t>(row) * d.Qs + col;
  const size_t sstride = static_cast<size_t>(d.Lrows) * d.Qs;
  double s = 0.0;
  if (ca.mode == kModeA) {
#pragma unroll 8
    for (int sl = 0; sl < S; ++sl) s += src[sl * sstride];
    if (row < d.Lpad)
      ca.XAt[static_cast<size_t>(row) * d.Qs + col] = s;
    else
      ca.AAt[static_cast<size_t>(row - d.Lpad) * d.Qs + col] = s;
  } else {
#pragma unroll 8
    for (int sl = 0; sl < S; ++sl) s += src[sl * sstride] * ca.fac[static_cast<size_t>(sl) * d.Qs + col];
    ca.Y[static_cast<size_t>(row) * d.Qs + col] = s / ca.colS[col];
  }
}

// ---------------------------------------------------------------------------
// Per-run small algebra: Z = XAᵀ − Y·AAᵀ, G = YᵀY, and (init) the step sizes.
__global__ void __launch_bounds__(256) k_post(PostArgs pa) {
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

__global__ void k_xnorm(const float* X, double* xnorm, Dims d) {
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
__global__ void __launch_bounds__(256) k_strict_e(const float* X, const double* Bv, double* E, Dims d) {
  __shared__ float xs[32][65];
  __shared__ double bs[32][65];
  const int lane = threadIdx.x & 31, ry = threadIdx.x >> 5;
  const int l0 = blockIdx.x * 32, c0 = blockIdx.y * 32;
  const int ncol = d.M * d.p;
  double s[4] = {0.0, 0.0, 0.0, 0.0};
  for (int j0 = 0; j0 < d.N; j0 += 64) {
    for (int e = threadIdx.x; e < 32 * 64; e += 256) {
      const int rr = e / 64, jj = e % 64;
      const int l = l0 + rr, c = c0 + rr, j = j0 + jj;
      xs[rr][jj] = (l < d.L && j < d.N) ? X[static_cast<size_t>(l) * d.Npad + j] : 0.0f;
      bs[rr][jj] = (c < ncol && j < d.N) ? Bv[static_cast<size_t>(c) * d.Npad + j] : 0.0;
    }
    __syncthreads();
    const int jn = min(64, d.N - j0);
    for (int jj = 0; jj < jn; ++jj) {
      const double b = bs[lane][jj];
#pragma unroll
      for (int q = 0; q < 4; ++q)
        s[q] = __dadd_rn(s[q], __dmul_rn(static_cast<double>(xs[ry + 8 * q][jj]), b));
    }
    __syncthreads();
  }
  const int c = c0 + lane;
  if (c >= ncol) return;
  const int r = c / d.p, i = c % d.p;
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const int l = l0 + ry + 8 * q;
    if (l < d.L) E[(static_cast<size_t>(r) * d.Lpad + l) * d.p + i] = s[q];
  }
}

// fit_l1 = Σ |X − E·A| (ensemble.cpp:29-39). Per element the reconstruction
// follows matmul's order (endmember index ascending, multiply then add);
// the sum over elements is a fixed-order tree (per block) then a fixed-order
// sum over blocks.
__global__ void __launch_bounds__(256) k_fit_partial(const float* X, const double* E, const double* A,
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
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= d.M) return;
  const int p = d.p;
  const double* e = E + static_cast<size_t>(r) * d.Lpad * p;
  double best = -INFINITY;
  for (int i = 0; i < p; ++i)
    for (int j = i + 1; j < p; ++j) {
      double dot = 0.0;
      for (int l = 0; l < d.L; ++l) dot = __dadd_rn(dot, __dmul_rn(e[l * p + i], e[l * p + j]));
      best = max_like_std(best, dot);
    }
  mu[r] = (best == -INFINITY) ? 0.0 : best;
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

template <int MODE, int RTW>
cudaError_t launch_pass_rtw(const PassArgs& a, cudaStream_t st, int pt) {
  constexpr int MB = (RTW <= 4) ? 2 : 1;
  const dim3 grid(a.d.nslices, a.d.NCH);
  const size_t smem = smem_layout(a.d, a.d.nbuf).total;
  void (*kern)(PassArgs) = nullptr;
  if (MODE == kModeInit || MODE == kModeB) {
    kern = k_pass<MODE, 1, RTW, MB>;
  } else {
    switch (pt) {
#define EDAA_PT_CASE(P)                                       \
  case P:                                                     \
    kern = k_pass<MODE, P, RTW, (P <= 12 ? MB : 1)>;          \
    break;
      EDAA_PT_CASE(2) EDAA_PT_CASE(3) EDAA_PT_CASE(4) EDAA_PT_CASE(5) EDAA_PT_CASE(6)
      EDAA_PT_CASE(7) EDAA_PT_CASE(8) EDAA_PT_CASE(10) EDAA_PT_CASE(12) EDAA_PT_CASE(16)
#undef EDAA_PT_CASE
      default:
        return cudaErrorInvalidValue;
    }
  }
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       static_cast<int>(smem));
  if (e != cudaSuccess) return e;
  kern<<<grid, kThreads, smem, st>>>(a);
  return cudaGetLastError();
}

int pt_bucket(int p) {
  if (p <= 8) return p;
  if (p <= 10) return 10;
  if (p <= 12) return 12;
  return 16;
}

}  // namespace

size_t pass_smem_bytes(const Dims& d, int nbuf) { return smem_layout(d, nbuf).total; }

cudaError_t launch_pass(int mode, const PassArgs& a, cudaStream_t st) {
  const int pt = pt_bucket(a.d.p);
  const bool wide = (a.d.Lpad / 8 + a.d.QCpad / 8) > 32;  // > 4 row tiles per warp
  switch (mode) {
    case kModeInit:
      return wide ? launch_pass_rtw<kModeInit, 6>(a, st, pt) : launch_pass_rtw<kModeInit, 4>(a, st, pt);
    case kModeA:
      return wide ? launch_pass_rtw<kModeA, 6>(a, st, pt) : launch_pass_rtw<kModeA, 4>(a, st, pt);
    case kModeB:
      return wide ? launch_pass_rtw<kModeB, 6>(a, st, pt) : launch_pass_rtw<kModeB, 4>(a, st, pt);
    case kModeObj:
      return launch_pass_rtw<kModeObj, 1>(a, st, pt);
  }
  return cudaErrorInvalidValue;
}

cudaError_t launch_combine(const CombineArgs& a, cudaStream_t st) {
  const Dims& d = a.d;
  if (a.mode == kModeB || a.mode == kModeInit) {
    k_colnorm<<<(d.Qs + 7) / 8, 256, 0, st>>>(a);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
  }
  const int rows = (a.mode == kModeA) ? d.Lrows : (a.mode == kModeObj ? 0 : d.Lpad);
  const dim3 grid((d.Qs + 31) / 32, rows > 0 ? (rows + 7) / 8 : 1);
  k_rowsum<<<grid, dim3(32, 8), 0, st>>>(a, rows);
  return cudaGetLastError();
}

cudaError_t launch_post(const PostArgs& a, cudaStream_t st) {
  k_post<<<a.d.M, 256, 0, st>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_xnorm(const float* X, double* xnorm, const Dims& d, cudaStream_t st) {
  k_xnorm<<<(d.Npad + 255) / 256, 256, 0, st>>>(X, xnorm, d);
  return cudaGetLastError();
}

cudaError_t launch_materialize_b(const double* Lg, const double* colm, const double* colS,
                                 double* Bv, const Dims& d, cudaStream_t st) {
  const dim3 grid(static_cast<unsigned>(std::min(64, (d.Npad + 255) / 256)), d.M * d.p);
  k_materialize_b<<<grid, 256, 0, st>>>(Lg, colm, colS, Bv, d);
  return cudaGetLastError();
}

cudaError_t launch_strict_e(const float* X, const double* Bv, double* E, const Dims& d,
                            cudaStream_t st) {
  const dim3 grid((d.L + 31) / 32, (d.M * d.p + 31) / 32);
  k_strict_e<<<grid, 256, 0, st>>>(X, Bv, E, d);
  return cudaGetLastError();
}

cudaError_t launch_fit(const float* X, const double* E, const double* A, double* part_fit,
                       double* fit, int fit_blocks, const Dims& d, cudaStream_t st) {
  k_fit_partial<<<dim3(fit_blocks, d.M), 256, 0, st>>>(X, E, A, part_fit, fit_blocks, d);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  k_fit_final<<<(d.M + 127) / 128, 128, 0, st>>>(part_fit, fit, fit_blocks, d.M);
  return cudaGetLastError();
}

cudaError_t launch_coherence(const double* E, double* mu, const Dims& d, cudaStream_t st) {
  k_coherence<<<(d.M + 63) / 64, 64, 0, st>>>(E, mu, d);
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
