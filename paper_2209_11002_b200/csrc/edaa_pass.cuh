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

// ---------------------------------------------------------------------------
// The pass kernel: grid = (nslices, NCH), block = 512 threads in two warp
// groups that run a two-stage software pipeline over the slice's 32-pixel
// tiles:
//   MMA group    (warps 0-7):  P1(i+1) = Wᵀ·X(i+1) on DMMA, then P3(i) += X(i)·w(i)ᵀ
//   update group (warps 8-15): P2(i)   the per-pixel simplex / logit update
// so the per-pixel math of tile i overlaps the tensor-pipe work of tiles i and
// i+1.  Hand-off through named barriers: S(i) ready (MMA → update) on id
// 1 + i%2, w(i) ready (update → MMA) on id 3 + i%2; each group also syncs
// internally (ids 5, 6).  X tiles are triple-buffered (cp.async, issued two
// tiles ahead), projections/weights and state tiles double-buffered.
namespace bars {
constexpr int kS = 1, kW = 3, kMma = 5, kUpd = 6;
}

// P3 for a warp owning R row tiles (gwarp + 8·i): C[l][c] += Σ_j X[l][j]·w[c][j]
// over the tile's 32 pixels; pseudo rows ≥ Lpad read w itself (AAᵀ).  R and the
// three column tiles are compile-time, so the DMMAs are unpredicated.
template <int R, int RTW, class XT>
__device__ __forceinline__ void accumulate_tiles(double (&ac)[RTW][kMaxCT][2], const XT* xs,
                                                 const double* w, int gwarp, int nRTx, int g, int t4) {
  const double* wrow = w + g * kSST + t4;
#pragma unroll
  for (int kk = 0; kk < kNP / 4; ++kk) {
    double bw[kMaxCT];
#pragma unroll
    for (int ct = 0; ct < kMaxCT; ++ct) bw[ct] = wrow[ct * 8 * kSST + kk * 4];
#pragma unroll
    for (int i = 0; i < R; ++i) {
      const int rt = gwarp + 8 * i;
      const double ax = (rt < nRTx) ? static_cast<double>(xs[(rt * 8 + g) * kXST + kk * 4 + t4])
                                    : w[((rt - nRTx) * 8 + g) * kSST + kk * 4 + t4];
#pragma unroll
      for (int ct = 0; ct < kMaxCT; ++ct) dmma(ac[i][ct], ax, bw[ct]);
    }
  }
}

template <int MODE, class XT>
__device__ __forceinline__ void issue_x(const PassArgs& pa, XT* xs, int j0, int gtid) {
  const Dims& d = pa.d;
  constexpr int kV = 16 / sizeof(XT);  // elements per 16-byte copy
  const XT* X = static_cast<const XT*>(pa.X);
  for (int e = gtid; e < d.L * (kNP / kV); e += kGroup) {
    const int l = e / (kNP / kV), q = e % (kNP / kV);
    cp_async16(xs + l * kXST + q * kV, X + static_cast<size_t>(l) * d.Npad + j0 + q * kV);
  }
  cp_async_commit();
}

template <int MODE>
__device__ __forceinline__ void issue_state(const PassArgs& pa, double* st, int j0, int row0,
                                            int nrows, int gtid) {
  if (MODE != kModeInit) {
    const double* src = (MODE == kModeB) ? pa.Lg : pa.A;
    for (int e = gtid; e < nrows * (kNP / 2); e += kGroup) {
      const int c = e / (kNP / 2), q = e % (kNP / 2);
      cp_async16(st + c * kNP + q * 2, src + static_cast<size_t>(row0 + c) * pa.d.Npad + j0 + q * 2);
    }
  }
  cp_async_commit();
}

template <int MODE, int PT, int RTW, class XT>
__global__ void __launch_bounds__(kThreads, 1) k_pass(PassArgs pa) {
  extern __shared__ __align__(16) unsigned char smem[];
  const Dims& d = pa.d;
  const int nbuf = d.nbuf;
  const SmemLayout lay = smem_layout(d, nbuf);
  double* ws = reinterpret_cast<double*>(smem + lay.ws_off);
  double* gs = reinterpret_cast<double*>(smem + lay.gs_off);
  double* m_run = reinterpret_cast<double*>(smem + lay.col_off);
  double* S_run = m_run + d.QCpad;
  double* c_m = S_run + d.QCpad;      // normaliser max of the previous logits (B pass)
  double* c_logS = c_m + d.QCpad;     // its log-sum
  double* c_eta = c_logS + d.QCpad;   // η of the column's run (η_b for B, η_a for A)
  double* facb = c_eta + d.QCpad;     // [2][QCpad] running-max rescale of tile i%2
  double* obj_run = facb + 2 * d.QCpad;
  double* hobj = obj_run + d.RC;
  auto xbuf = [&](int i) { return reinterpret_cast<XT*>(smem + lay.xs_off + (i % nbuf) * lay.xs_bytes); };
  auto sbuf = [&](int i) { return reinterpret_cast<double*>(smem + lay.ss_off + (i & 1) * lay.buf_bytes); };
  auto hbuf = [&](int i) { return reinterpret_cast<double*>(smem + lay.sh_off + (i & 1) * lay.buf_bytes); };
  auto stbuf = [&](int i) { return reinterpret_cast<double*>(smem + lay.st_off + (i & 1) * lay.st_bytes); };

  const int tid = threadIdx.x;
  const bool mma_group = tid < kGroup;
  const int gtid = tid & (kGroup - 1);
  const int lane = tid & 31, gwarp = gtid >> 5;
  const int g = lane >> 2, t4 = lane & 3;
  const int slice = blockIdx.x;
  const int chunk = blockIdx.y;
  const int p = d.p;
  const int run0 = chunk * d.RC;
  const int RCe = min(d.RC, d.M - run0);  // runs present in this chunk
  const int ncol_valid = RCe * p;
  const int nRTx = d.Lpad / 8;
  const int nRT = (MODE == kModeA) ? nRTx + d.QCpad / 8 : nRTx;
  const int WST = w_stride(d.QCpad);
  const int col0 = chunk * d.QCpad;
  const int srow0 = run0 * p;  // first state row (A / Lg) of this chunk

  const int tile_begin = static_cast<int>((static_cast<long long>(slice) * d.ntiles) / d.nslices);
  const int tile_end = static_cast<int>((static_cast<long long>(slice + 1) * d.ntiles) / d.nslices);
  const int ntile = tile_end - tile_begin;

  // First tiles in flight while the constants are staged.
  if (mma_group) {
    issue_x<MODE, XT>(pa, xbuf(0), tile_begin * kNP, gtid);
    if (ntile > 1) issue_x<MODE, XT>(pa, xbuf(1), (tile_begin + 1) * kNP, gtid);
  } else {
    issue_state<MODE>(pa, stbuf(0), tile_begin * kNP, srow0, ncol_valid, gtid);
  }
  // ---- one-time staging (all 512 threads) ----
  if (MODE != kModeInit) {
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
  for (int b = 0; b < nbuf; ++b)
    for (int e = tid; e < (d.Lpad - d.L) * kNP; e += kThreads)
      xbuf(b)[(d.L + e / kNP) * kXST + e % kNP] = XT(0);
  if (tid < d.QCpad) {
    const int c = tid;
    m_run[c] = -INFINITY;
    S_run[c] = 0.0;
    facb[c] = facb[d.QCpad + c] = 1.0;
    const bool real = c < ncol_valid;
    const int r = run0 + (real ? c / p : 0);
    c_m[c] = (MODE == kModeB && real) ? pa.colm[col0 + c] : 0.0;
    c_logS[c] = (MODE == kModeB && real) ? pa.collogS[col0 + c] : 0.0;
    c_eta[c] = real ? (MODE == kModeB ? pa.eta_b[r] : (MODE == kModeInit ? 0.0 : pa.eta_a[r])) : 0.0;
  }
  if (tid < d.RC) obj_run[tid] = 0.0;
  __syncthreads();

  if (mma_group) {
    // =========================== MMA group ===========================
    double acc[RTW][kMaxCT][2];
#pragma unroll
    for (int i = 0; i < RTW; ++i)
#pragma unroll
      for (int c = 0; c < kMaxCT; ++c) acc[i][c][0] = acc[i][c][1] = 0.0;

    // row tiles owned by this warp: gwarp + 8·i < nRT
    const int my_rt = (nRT - gwarp + 7) / 8;
    // P1(i): S[c][j] = Σ_l W[l][c]·X[l][j]; warp = 8 pixels × one band half.
    auto phase1 = [&](int i) {
      if (MODE != kModeInit) {
        const XT* xs = xbuf(i);
        const int pt = gwarp & 3, half = gwarp >> 2;
        const int kh = d.Lpad / 8;  // k-steps per band half
        double c1[kMaxCT][2];
#pragma unroll
        for (int c = 0; c < kMaxCT; ++c) c1[c][0] = c1[c][1] = 0.0;
        const XT* xcol = xs + pt * 8 + g;
        const double* wcol = ws + g;
#pragma unroll 4
        for (int kk = half * kh; kk < (half + 1) * kh; ++kk) {
          const int l = kk * 4 + t4;
          const double bx = static_cast<double>(xcol[l * kXST]);
#pragma unroll
          for (int ct = 0; ct < kMaxCT; ++ct) dmma(c1[ct], wcol[l * WST + ct * 8], bx);
        }
        double* dst = half ? hbuf(i) : sbuf(i);
#pragma unroll
        for (int ct = 0; ct < kMaxCT; ++ct)
          *reinterpret_cast<double2*>(dst + (ct * 8 + g) * kSST + pt * 8 + 2 * t4) =
              make_double2(c1[ct][0], c1[ct][1]);
      }
    };
    // wait for X(i) (the only other group in flight may be X(i+1)), publish to the group
    auto x_ready = [&](int i, bool newer_in_flight) {
      if (newer_in_flight) cp_async_wait1(); else cp_async_wait0();
      bar_sync(bars::kMma, kGroup);
    };

    x_ready(0, ntile > 1);
    phase1(0);
    bar_arrive(bars::kS + 0, kThreads);
    for (int it = 0; it < ntile; ++it) {
      if (it + 1 < ntile) {
        x_ready(it + 1, false);
        // three buffers: X(i+2) goes into X(i−1)'s slot, free since the barrier above
        if (nbuf > 2 && it + 2 < ntile) issue_x<MODE, XT>(pa, xbuf(it + 2), (tile_begin + it + 2) * kNP, gtid);
        phase1(it + 1);
        bar_arrive(bars::kS + ((it + 1) & 1), kThreads);
      }
      bar_sync(bars::kW + (it & 1), kThreads);  // w(i), fac(i) ready
      if (MODE != kModeObj) {
      const double* fac = facb + (it & 1) * d.QCpad;
      if (MODE == kModeB || MODE == kModeInit) {
#pragma unroll
        for (int ct = 0; ct < kMaxCT; ++ct) {
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
      // P3(i): C[l][c] += Σ_j X[l][j]·w[c][j]; warp owns row tiles gwarp, gwarp+8, …
      const XT* xs = xbuf(it);
      const double* w = sbuf(it);
      switch (my_rt) {  // warp-uniform: the DMMAs below are unpredicated
        case 1: accumulate_tiles<1>(acc, xs, w, gwarp, nRTx, g, t4); break;
        case 2: accumulate_tiles<2>(acc, xs, w, gwarp, nRTx, g, t4); break;
        case 3: accumulate_tiles<3>(acc, xs, w, gwarp, nRTx, g, t4); break;
        case 4: if constexpr (RTW >= 4) accumulate_tiles<4>(acc, xs, w, gwarp, nRTx, g, t4); break;
        case 5: if constexpr (RTW >= 5) accumulate_tiles<5>(acc, xs, w, gwarp, nRTx, g, t4); break;
        case 6: if constexpr (RTW >= 6) accumulate_tiles<6>(acc, xs, w, gwarp, nRTx, g, t4); break;
        default: break;
      }
      }  // MODE != kModeObj
      if (nbuf == 2 && it + 2 < ntile) {  // X(i) is consumed: reuse its buffer for X(i+2)
        bar_sync(bars::kMma, kGroup);
        issue_x<MODE, XT>(pa, xbuf(it + 2), (tile_begin + it + 2) * kNP, gtid);
      }
    }
    if (MODE != kModeObj) {
#pragma unroll
      for (int i = 0; i < RTW; ++i) {
        const int rt = gwarp + 8 * i;
        if (rt < nRT) {
          const int row = rt * 8 + g;
#pragma unroll
          for (int ct = 0; ct < kMaxCT; ++ct) {
            double* dst = pa.part_C + (static_cast<size_t>(slice) * d.Lrows + row) * d.Qs + col0 +
                          ct * 8 + 2 * t4;
            *reinterpret_cast<double2*>(dst) = make_double2(acc[i][ct][0], acc[i][ct][1]);
          }
        }
      }
    }
  } else {
    // ========================== update group ==========================
    for (int it = 0; it < ntile; ++it) {
      const int j0 = (tile_begin + it) * kNP;
      bar_sync(bars::kUpd, kGroup);  // everyone is done with st(i−1)
      const bool more = it + 1 < ntile;
      if (more) issue_state<MODE>(pa, stbuf(it + 1), j0 + kNP, srow0, ncol_valid, gtid);
      if (more) cp_async_wait1(); else cp_async_wait0();
      bar_sync(bars::kUpd, kGroup);  // st(i) visible
      bar_sync(bars::kS + (it & 1), kThreads);  // S(i) ready
      double* ss = sbuf(it);
      const double* sh = hbuf(it);
      const double* st = stbuf(it);
      double* fac = facb + (it & 1) * d.QCpad;

      if (MODE == kModeA || MODE == kModeObj) {
        constexpr int TPP = LanesPerPixel<PT>::value;
        for (int q2 = gtid; q2 < RCe * kNP * TPP; q2 += kGroup) {  // warp-uniform trip count
          const int q = q2 / TPP, sub = q2 % TPP;
          const int rl = q / kNP, j = q % kNP;
          const int pix = j0 + j;
          double o = pixel_a_update<PT, TPP, MODE == kModeA>(pa, run0 + rl, rl, j, pix, pix < d.N, sub,
                                                               ss, sh, st, gs);
          o = warp_sum(o);
          if (lane == 0) hobj[q2 >> 5] = o;  // warp-task q2/32 belongs to run (q2/32)/TPP
        }
        if (MODE == kModeA)
          for (int e = gtid; e < (d.QCpad - ncol_valid) * kNP; e += kGroup)
            ss[(ncol_valid + e / kNP) * kSST + e % kNP] = 0.0;
        bar_sync(bars::kUpd, kGroup);
        if (gtid < RCe) {
          double o = obj_run[gtid];
          for (int h = 0; h < TPP; ++h) o += hobj[gtid * TPP + h];
          obj_run[gtid] = o;
        }
      } else {
        // B step / B⁰: new logits; 8 lanes per column, 4 pixels per lane (j = k·8 + lane8).
        const int c = gtid >> 3, l8 = gtid & 7;
        const bool active = c < d.QCpad;  // QCpad·8 ≤ 192 threads carry columns
        double ell[4];
        double tmax = -INFINITY;
        if (active) {
          const bool real = c < ncol_valid;
          const int rl = real ? c / p : 0, i = real ? c % p : 0, r = run0 + rl;
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            const int j = k * 8 + l8, pix = j0 + j;
            double v = -INFINITY;
            if (real && pix < d.N) {
              if (MODE == kModeInit) {
                // solver.cpp:122-127: column i consumes draws i·N .. i·N+N−1.
                v = 0.1 * splitmix_unit_at(pa.seeds[r], static_cast<uint64_t>(i) * d.N +
                                                            static_cast<uint64_t>(pix));
              } else {
                double lb = st[c * kNP + j] - c_m[c] - c_logS[c];         // log b_old
                lb = (lb < log_floor()) ? log_floor() : lb;                // log max(b, 1e-30)
                v = lb + (ss[c * kSST + j] + sh[c * kSST + j]) * c_eta[c]; // + η_b·(−∇_B)
              }
              pa.Lg[static_cast<size_t>(srow0 + c) * d.Npad + pix] = v;
            }
            ell[k] = v;
            tmax = fmax(tmax, v);
          }
        }
        // column max over the 8 lanes (groups of 8 consecutive lanes)
#pragma unroll
        for (int o = 4; o > 0; o >>= 1) tmax = fmax(tmax, __shfl_xor_sync(0xffffffffu, tmax, o));
        double tsum = 0.0, mn = -INFINITY, mo = -INFINITY;
        if (active) {
          mo = m_run[c];
          mn = fmax(mo, tmax);
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            const double w = (mn == -INFINITY) ? 0.0 : exp(ell[k] - mn);
            ss[c * kSST + k * 8 + l8] = w;
            tsum += w;
          }
        }
#pragma unroll
        for (int o = 4; o > 0; o >>= 1) tsum += __shfl_xor_sync(0xffffffffu, tsum, o);
        if (active && l8 == 0) {
          const double f = (mn == -INFINITY || mn == mo) ? 1.0 : exp(mo - mn);
          fac[c] = f;
          S_run[c] = S_run[c] * f + tsum;
          m_run[c] = mn;
        }
      }
      bar_arrive(bars::kW + (it & 1), kThreads);  // w(i), fac(i) ready for P3(i)
    }
    bar_sync(bars::kUpd, kGroup);
    if (MODE == kModeB || MODE == kModeInit) {
      if (gtid < d.QCpad) {
        pa.part_m[static_cast<size_t>(slice) * d.Qs + col0 + gtid] = m_run[gtid];
        pa.part_S[static_cast<size_t>(slice) * d.Qs + col0 + gtid] = S_run[gtid];
      }
    } else {
      if (gtid < RCe) pa.part_obj[static_cast<size_t>(slice) * d.M + run0 + gtid] = obj_run[gtid];
    }
  }
}

template <int MODE, int RTW, class XT>
cudaError_t launch_pass_rtw(const PassArgs& a, cudaStream_t st, int pt) {
  const dim3 grid(a.d.nslices, a.d.NCH);
  const size_t smem = dev::smem_layout(a.d, a.d.nbuf).total;
  void (*kern)(PassArgs) = nullptr;
  if (MODE == kModeInit || MODE == kModeB) {
    kern = k_pass<MODE, 1, RTW, XT>;
  } else {
    switch (pt) {
#define EDAA_PT_CASE(P)                                       \
  case P:                                                     \
    kern = k_pass<MODE, P, RTW, XT>;                          \
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
