// EDAA pass kernel (templated on the image element type) for sm_100a (B200).
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
#pragma once
#include <cmath>
#include <cstdio>

#include "edaa_device.cuh"

namespace edaa {
namespace pass_impl {

using namespace dev;

inline int pt_bucket(int p) {
  if (p <= 8) return p;
  if (p <= 10) return 10;
  if (p <= 12) return 12;
  return 16;
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
  // ½‖x − Ya‖² ≥ 0; the expanded form can round a few ulps below an exact zero.
  return (valid && sub == 0) ? fmax(0.5 * ((pa.xnorm[pix] - 2.0 * aPa) + aGa), 0.0) : 0.0;
}

// X tile (rows < L) and the chunk's state rows (A or logits) for pixels
// [j0, j0+kNP), 16-byte cp.async into shared memory, one commit group.
template <int MODE, class XT>
__device__ __forceinline__ void load_tile(const PassArgs& pa, XT* xs, double* st, int j0,
                                          int state_row0, int nstate) {
  const Dims& d = pa.d;
  constexpr int kV = 16 / sizeof(XT);  // elements per 16-byte copy
  const XT* X = static_cast<const XT*>(pa.X);
  for (int e = threadIdx.x; e < d.L * (kNP / kV); e += kThreads) {
    const int l = e / (kNP / kV), q = e % (kNP / kV);
    cp_async16(xs + l * kXST + q * kV, X + static_cast<size_t>(l) * d.Npad + j0 + q * kV);
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
template <int MODE, int PT, int RTW, int MINB, class XT>
__global__ void __launch_bounds__(kThreads, MINB) k_pass(PassArgs pa) {
  extern __shared__ __align__(16) unsigned char smem[];
  const Dims& d = pa.d;
  const SmemLayout lay = smem_layout(d, 1);
  XT* xs = reinterpret_cast<XT*>(smem + lay.xs_off);
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
  load_tile<MODE, XT>(pa, xs, st, tile_begin * kNP, srow0, ncol_valid);

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
    xs[(d.L + e / kNP) * kXST + e % kNP] = XT(0);
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
      const XT* xcol = xs + pt * 8 + g;
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
        if (tile + 1 < tile_end) load_tile<MODE, XT>(pa, xs, st, j0 + kNP, srow0, ncol_valid);
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
    if (tile + 1 < tile_end) load_tile<MODE, XT>(pa, xs, st, j0 + kNP, srow0, ncol_valid);
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
template <int MODE, int RTW, class XT>
cudaError_t launch_pass_rtw(const PassArgs& a, cudaStream_t st, int pt) {
  // two CTAs per SM for the fp32 image; the fp64 image tile needs the whole SM
  constexpr int MB = (RTW <= 4 && sizeof(XT) == 4) ? 2 : 1;
  const dim3 grid(a.d.nslices, a.d.NCH);
  const size_t smem = dev::smem_layout(a.d, a.d.nbuf).total;
  void (*kern)(PassArgs) = nullptr;
  if (MODE == kModeInit || MODE == kModeB) {
    kern = k_pass<MODE, 1, RTW, MB, XT>;
  } else {
    switch (pt) {
#define EDAA_PT_CASE(P)                                       \
  case P:                                                     \
    kern = k_pass<MODE, P, RTW, (P <= 12 ? MB : 1), XT>;      \
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


template <class XT>
cudaError_t launch_pass_xt(int mode, const PassArgs& a, cudaStream_t st) {
  const int pt = pt_bucket(a.d.p);
  const bool wide = (a.d.Lpad / 8 + a.d.QCpad / 8) > 32;  // > 4 row tiles per warp
  switch (mode) {
    case kModeInit:
      return wide ? launch_pass_rtw<kModeInit, 6, XT>(a, st, pt) : launch_pass_rtw<kModeInit, 4, XT>(a, st, pt);
    case kModeA:
      return wide ? launch_pass_rtw<kModeA, 6, XT>(a, st, pt) : launch_pass_rtw<kModeA, 4, XT>(a, st, pt);
    case kModeB:
      return wide ? launch_pass_rtw<kModeB, 6, XT>(a, st, pt) : launch_pass_rtw<kModeB, 4, XT>(a, st, pt);
    case kModeObj:
      return launch_pass_rtw<kModeObj, 1, XT>(a, st, pt);
  }
  return cudaErrorInvalidValue;
}


}  // namespace pass_impl
}  // namespace edaa
