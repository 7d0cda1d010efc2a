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
#include <algorithm>
#include <cmath>
#include <cstdio>

#include <cuda.h>

#include "edaa_device.cuh"

#ifndef EDAA_P1_UNROLL
#define EDAA_P1_UNROLL 2
#endif

namespace edaa {
namespace pass_impl {

using namespace dev;
constexpr int kP1Unroll = EDAA_P1_UNROLL;  // P1 band-pair loop unroll (dev sweeps via -D)

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
// Lanes per (pixel, run) task of the A update.  Measured (A pass, ms): p = 6
// 1.55 with 2 lanes vs 2.36 with 1; p = 12 2.01 with 2 vs 2.25 with 4.
template <int PT>
struct LanesPerPixel {
  static constexpr int value = PT <= 4 ? 1 : (PT <= 12 ? 2 : 4);
};

// check_iterate (solver.cpp:65-90) on one pixel's column held by TPP lanes (EPT
// entries each, `ownbits` the valid ones), evaluated exactly and in the
// reference's scan order; posts the first failing check to the run's key.  Out of
// line: it is reached only when the update's range test on Σ fires, and must not
// cost the K1 loop registers.  All lanes of the pixel's group call it together.
template <int EPT, int TPP>
__device__ __noinline__ void post_simplex_failure(unsigned long long* slot, unsigned tb, int k, int pix, int e0,
                                                  unsigned gmask, const double* a, unsigned ownbits) {
  double csum = 0.0;
#pragma unroll
  for (int e = 0; e < EPT; ++e)
    if (ownbits >> e & 1u) csum += a[e];
#pragma unroll
  for (int o = 1; o < TPP; o <<= 1) csum += __shfl_xor_sync(gmask, csum, o);
  unsigned long long key = ~0ull;
#pragma unroll
  for (int e = EPT - 1; e >= 0; --e) {
    if ((ownbits >> e & 1u) && !(isfinite(a[e]) && a[e] >= 0.0))
      key = fail_key_make(tb, k, (static_cast<unsigned long long>(pix) << 5) | static_cast<unsigned>(e0 + e),
                          isfinite(a[e]) ? kFailNegative : kFailNonFinite);
  }
  // entries fine on this lane: the column-sum check comes after all of them
  if (key == ~0ull && !(fabs(csum - 1.0) <= kSimplexTol))
    key = fail_key_make(tb, k, (static_cast<unsigned long long>(pix) << 5) | 31u, kFailDrift);
  if (key != ~0ull) atomicMin(slot, key);  // later steps post larger keys: the first one survives
}

template <int PT, int TPP, bool UPDATE, bool EXACT>
__device__ __forceinline__ double pixel_a_update(const PassArgs& pa, int r, int rl, int j, int pix,
                                                 bool valid, int sub, double* ss, const double* sh,
                                                 const double* st, const double* gs, const double* T,
                                                 const double* ceta) {
  // EXACT: p == PT, so every index below is compile-time except the lane's `sub`.
  constexpr int EPT = (PT + TPP - 1) / TPP;
  constexpr bool kAllValid = EXACT && (PT % TPP == 0);
  constexpr bool kGinRegs = EXACT && EPT * PT <= 24;  // the lane's rows of G stay in registers (larger: smem; p = 7, 8 spilled)
  const Dims& d = pa.d;
  const int p = EXACT ? PT : d.p;
  const int gbase = (threadIdx.x & 31) - sub;
  const double xn = valid ? pa.xnorm[pix] : 0.0;
  const double eta = ceta[rl];  // η_a of the run, staged in shared memory at the chunk change
  double a[EPT], P[EPT];
  bool own[EPT];
#pragma unroll
  for (int e = 0; e < EPT; ++e) {
    const int i = sub * EPT + e;
    own[e] = kAllValid || i < p;
    a[e] = 0.0;
    P[e] = 0.0;
    if (own[e]) {
      const int c = rl * p + i;
      a[e] = st[c * kNP + j];
      P[e] = ss[c * kSST + j] + sh[c * kSST + j];
    }
  }
  const double* G = gs + rl * p * p;
  double Gr[kGinRegs ? EPT : 1][kGinRegs ? PT : 1];
  if constexpr (kGinRegs) {
#pragma unroll
    for (int e = 0; e < EPT; ++e)
#pragma unroll
      for (int m = 0; m < PT; ++m) Gr[e][m] = own[e] ? G[(sub * EPT + e) * PT + m] : 0.0;
  }
  double aPa = 0.0, aGa = 0.0;
  const int steps = UPDATE ? d.K1 : 1;
  for (int k = 0; k < steps; ++k) {
    double ga[EPT];
#pragma unroll
    for (int e = 0; e < EPT; ++e) ga[e] = 0.0;
#pragma unroll
    for (int m = 0; m < PT; ++m) {
      if (EXACT || m < p) {
        const double am = (TPP == 1) ? a[m % EPT] : __shfl_sync(0xffffffffu, a[m % EPT], gbase + m / EPT);
#pragma unroll
        for (int e = 0; e < EPT; ++e) {
          if constexpr (kGinRegs) {
            ga[e] = fma(Gr[e][m], am, ga[e]);
          } else {
            if (own[e]) ga[e] += G[(sub * EPT + e) * p + m] * am;
          }
        }
      }
    }
    double u[EPT];
    double umax = -INFINITY;
#pragma unroll
    for (int e = 0; e < EPT; ++e) {
      u[e] = -INFINITY;
      if (own[e]) {
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
      if (own[e]) {
        const double z = (a[e] < kLogFloorValue) ? kLogFloorValue : a[e];  // std::max(z, 1e-30)
        a[e] = z * exp_nonpos(u[e] - umax, T);
        total += a[e];
      }
    }
#pragma unroll
    for (int o = 1; o < TPP; o <<= 1) total += __shfl_xor_sync(0xffffffffu, total, o);
    // total ∈ [1e-30, p] (every factor ≤ 1, the largest ≥ 1e-30): a normal number.
    const double inv = __drcp_rn(total);  // IEEE 1/total (= the division's value)
#pragma unroll
    for (int e = 0; e < EPT; ++e)
      if (own[e]) a[e] *= inv;
    // check_iterate (solver.cpp:65-90) on this pixel's column: every entry finite
    // and >= 0, |Σ − 1| <= 1e-9.  None of the three can fail while `total` is a
    // positive normal number: the factors z·e^{u − max u} lie in [0, 1], so the
    // entries a_e = factor·(1/total) are finite and >= 0, and their sum is
    // total·(1/total) up to (2p + 2) roundings, < 4e-15 from 1 at p = 16.  A
    // NaN/Inf anywhere upstream (P, G·a, η, a) reaches `total` through the
    // exponentials.  So the fast path is ONE integer range test on total's high
    // word (the fp64 pipe is the A pass's bottleneck; a per-step column sum cost
    // 4–11% of the pass); the reference's conditions themselves are evaluated,
    // in its scan order, only behind that test.  `total` is uniform over the
    // pixel's TPP lanes, so the group takes the branch together.
    bool force = false;
    if (pa.dbg & 0xE000) {  // test hooks (EDAA_DBG): poison pixel 7 of run 1 at outer iteration 2, inner step 2
      if (r == 1 && pix == 7 && pa.t == 2 && k == 1) {
        force = true;
        if ((pa.dbg & 0x2000) && sub == 0) a[0] = __longlong_as_double(0x7FF8000000000000ll);  // NaN entry
        if ((pa.dbg & 0x4000) && sub == 0) a[0] = -a[0];                                        // negative entry
        if ((pa.dbg & 0x8000) && sub == 0) a[0] += 1e-8;                                        // drifted column
      }
    }
    if ((static_cast<unsigned>(__double2hiint(total)) - 0x00100000u >= 0x7FE00000u || force) && valid) {
      double tmp[EPT];  // a copy whose address may be taken: a[] itself stays in registers
      unsigned ownbits = 0;
#pragma unroll
      for (int e = 0; e < EPT; ++e) {
        tmp[e] = a[e];
        ownbits |= own[e] ? (1u << e) : 0u;
      }
      const unsigned gmask = (TPP == 32) ? 0xffffffffu : (((1u << TPP) - 1u) << gbase);
      post_simplex_failure<EPT, TPP>(pa.fail_key + r, static_cast<unsigned>(pa.t) << 1, k, pix, sub * EPT, gmask, tmp,
                                     ownbits);
    }
    if (pa.observe_A != nullptr && valid) {
#pragma unroll
      for (int e = 0; e < EPT; ++e)
        if (own[e]) pa.observe_A[(static_cast<size_t>(k) * p + sub * EPT + e) * d.Npad + pix] = a[e];
    }
  }
#pragma unroll
  for (int o = 1; o < TPP; o <<= 1) {
    aPa += __shfl_xor_sync(0xffffffffu, aPa, o);
    aGa += __shfl_xor_sync(0xffffffffu, aGa, o);
  }
  if (UPDATE) {
    const size_t base = static_cast<size_t>(r) * p * d.Npad + pix;
#pragma unroll
    for (int e = 0; e < EPT; ++e) {
      if (own[e]) {
        const int i = sub * EPT + e;
        if (valid) pa.A[base + static_cast<size_t>(i) * d.Npad] = a[e];
        ss[(rl * p + i) * kSST + j] = valid ? a[e] : 0.0;
      }
    }
  }
  // ½‖x − Ya‖² ≥ 0; the expanded form can round a few ulps below an exact zero.
  return (valid && sub == 0) ? fmax(0.5 * ((xn - 2.0 * aPa) + aGa), 0.0) : 0.0;
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

// Optional cycle accounting (PassArgs::kprof != nullptr, development only):
// warp 0 of each group adds the cycles of its phases into kprof[slot].
#define EDAA_TSTART() const long long t0_ = (pa.kprof && (lane == 0) && (gwarp == 0)) ? clock64() : 0
#define EDAA_TSTOP(slot)                                                        \
  do {                                                                          \
    if (pa.kprof && lane == 0 && gwarp == 0)                                    \
      atomicAdd(pa.kprof + 6 * MODE + (slot), static_cast<unsigned long long>(clock64() - t0_)); \
  } while (0)

// Row stride of the swizzled X tile in elements (one 128-byte smem row).
template <class XT>
constexpr int kXRow = 128 / sizeof(XT);

// P3 for a warp owning R X row tiles (gwarp + 8·i, i < R) and, when PSEUDO, one
// more row tile of pseudo-bands (rows ≥ Lpad read w itself: AAᵀ):
// C[l][c] += Σ_j X[l][j]·w[c][j] over the tile's 32 pixels.  Row tiles, column
// tiles and k-steps are compile-time, so the DMMAs are unpredicated and the
// swizzled X addresses reduce to a per-k-step table (row & 7 == g for every
// fragment row).
template <int R, bool PSEUDO, int CT, int RTW, class XT>
__device__ __forceinline__ void accumulate_tiles(double (&ac)[RTW][kMaxCT][2], const XT* xs,
                                                 const double* w, int gwarp, int nRTx, int g, int t4,
                                                 const int (&xo)[kNP / 4]) {
  const double* wrow = w + g * kSST + t4;
  const double* prow = w + ((gwarp + 8 * R - nRTx) * 8 + g) * kSST + t4;  // the pseudo tile's rows
#pragma unroll
  for (int kk = 0; kk < kNP / 4; ++kk) {
    double bw[CT];
#pragma unroll
    for (int ct = 0; ct < CT; ++ct) bw[ct] = wrow[ct * 8 * kSST + kk * 4];
#pragma unroll
    for (int i = 0; i < R; ++i) {
      const double ax = static_cast<double>(xs[(gwarp + 8 * i) * 8 * kXRow<XT> + xo[kk]]);
#pragma unroll
      for (int ct = 0; ct < CT; ++ct) dmma(ac[i][ct], ax, bw[ct]);
    }
    if constexpr (PSEUDO) {
      const double ax = prow[kk * 4];
#pragma unroll
      for (int ct = 0; ct < CT; ++ct) dmma(ac[R][ct], ax, bw[ct]);
    }
  }
}

template <int MODE>
__device__ __forceinline__ void issue_state(const PassArgs& pa, double* st, int j0, int row0,
                                            int nrows, int gtid) {
  if (MODE != kModeInit && !(pa.dbg & 8)) {
    const double* src = (MODE == kModeB) ? pa.Lg : pa.A;
    for (int e = gtid; e < nrows * (kNP / 2); e += kGroup) {
      const int c = e / (kNP / 2), q = e % (kNP / 2);
      cp_async16(st + c * kNP + q * 2, src + static_cast<size_t>(row0 + c) * pa.d.Npad + j0 + q * 2);
    }
  }
  cp_async_commit();
}

// Work decomposition: item k (0 ≤ k < NCH·nslices) is (slice k / NCH, chunk
// k % NCH) — slice-major, so a CTA sweeps the run chunks over the same pixel
// slice back to back and X is re-read from L2, not HBM; persistent CTA b of G
// processes items [b·K/G, (b+1)·K/G) as ONE flattened stream of 32-pixel
// tiles (the pipeline never drains between items), restaging the W chunk and
// the per-column constants when the chunk changes and flushing every item's
// partials when its last tile retires.
struct Cursor {
  int item, slice, chunk, tile, tstart, tend;
};

__host__ __device__ __forceinline__ int slice_tile(const Dims& d, int s) {
  return slice_first_tile(d.ntiles, d.nslices, s);  // tile pairs: every slice holds an even number of tiles
}
// slt: the CTA's shared-memory copy of slice_tile(d, 0 .. nslices) (no divisions per tile)
// Item order (local index k over the owned slices [sl0, sl1)):
//   chunk-major (Dims::cmajor): k = chunk·nsl + (slice − sl0) — a CTA's block of
//     items is consecutive slices of one run chunk, so the W chunk and the per-
//     column constants change about once per CTA instead of once per item; X is
//     re-read from L2 once per chunk (chosen when X fits in L2);
//   slice-major: k = (slice − sl0)·NCH + chunk — consecutive items re-read the
//     same X slice (large images).
// Either order computes the same per-(slice, chunk) partials: results are bitwise equal.
__host__ __device__ __forceinline__ int item_slice(const Dims& d, int k) {
  return d.cmajor ? d.sl0 + k % (d.sl1 - d.sl0) : d.sl0 + k / d.NCH;
}
__host__ __device__ __forceinline__ int item_chunk(const Dims& d, int k) {
  return d.cmajor ? k / (d.sl1 - d.sl0) : k % d.NCH;
}
__device__ __forceinline__ void cursor_set(Cursor& c, const Dims& d, const int* slt, int item) {
  c.item = item;
  c.slice = item_slice(d, item);
  c.chunk = item_chunk(d, item);
  c.tile = c.tstart = slt[c.slice];
  c.tend = slt[c.slice + 1];
}
__device__ __forceinline__ void cursor_next(Cursor& c, const Dims& d, const int* slt) {
  if (++c.tile != c.tend) return;
  ++c.item;
  if (d.cmajor) {  // the next slice of the same chunk, then the next chunk
    if (++c.slice == d.sl1) {
      c.slice = d.sl0;
      ++c.chunk;
    }
  } else if (++c.chunk == d.NCH) {  // the next chunk of the same slice, then the next slice
    c.chunk = 0;
    ++c.slice;
  }
  c.tile = c.tstart = slt[c.slice];
  c.tend = slt[c.slice + 1];
}

// Interleaved slice-major items (large images, Dims::ilv, the ILV instantiation
// of the A/B passes): CTA b's j-th item is slice-major item j·G + b, so the G
// CTAs always work on G consecutive items (~G/NCH slices, every chunk of each)
// and an X slice read from HBM by its first CTA is an L2 hit for the others —
// with one slice per CTA, plain slice-major keeps all of X in flight and
// re-reads it from HBM once per chunk. Same partials, bitwise the same results.
// The other instantiations (ILV = false) are the code above, unchanged.
template <bool ILV>
__device__ __forceinline__ int item_slice_t(const Dims& d, int k) {
  if constexpr (ILV) {
    const int per = d.NCH * (d.sl1 - d.sl0) / d.ncta;
    return d.sl0 + ((k % per) * d.ncta + k / per) / d.NCH;
  } else {
    return item_slice(d, k);
  }
}
template <bool ILV>
__device__ __forceinline__ int item_chunk_t(const Dims& d, int k) {
  if constexpr (ILV) {
    const int per = d.NCH * (d.sl1 - d.sl0) / d.ncta;
    return ((k % per) * d.ncta + k / per) % d.NCH;
  } else {
    return item_chunk(d, k);
  }
}
template <bool ILV>
__device__ __forceinline__ void cursor_set_t(Cursor& c, const Dims& d, const int* slt, int item) {
  if constexpr (ILV) {
    c.item = item;
    c.slice = item_slice_t<true>(d, item);
    c.chunk = item_chunk_t<true>(d, item);
    c.tile = c.tstart = slt[c.slice];
    c.tend = slt[c.slice + 1];
  } else {
    cursor_set(c, d, slt, item);
  }
}
template <bool ILV>
__device__ __forceinline__ void cursor_next_t(Cursor& c, const Dims& d, const int* slt) {
  if constexpr (ILV) {
    if (++c.tile != c.tend) return;
    cursor_set_t<true>(c, d, slt, c.item + 1);
  } else {
    cursor_next(c, d, slt);
  }
}
// Position in a ring of n slots walked one step at a time (slot = i % n, phase = (i / n) & 1).
struct Ring {
  int slot, phase;
  __device__ __forceinline__ void next(int n) {
    if (++slot == n) {
      slot = 0;
      phase ^= 1;
    }
  }
};

struct ChunkInfo {
  int chunk, run0, RCe, ncol, col0, srow0;
};
__device__ __forceinline__ ChunkInfo chunk_info(const Dims& d, int chunk) {
  ChunkInfo ci;
  ci.chunk = chunk;
  ci.run0 = ci.chunk * d.RC;
  ci.RCe = min(d.RC, d.M - ci.run0);
  ci.ncol = ci.RCe * d.p;
  ci.col0 = ci.chunk * kQMax;
  ci.srow0 = ci.run0 * d.p;
  return ci;
}

// CTF: DMMA column tiles computed per chunk — kMaxCT, or 1 when the whole batch
// fits one 8-column tile (a single run with p ≤ 8: cfg0, the pixel-sharded run),
// which skips the DMMAs of the empty tiles (their w is 0, their partials stay 0).
template <int MODE, int PT, int RTW, class XT, int CTF, bool ILV = false>
__global__ void __launch_bounds__(kThreads, 1) k_pass(PassArgs pa, const __grid_constant__ CUtensorMap xmap) {
  extern __shared__ __align__(16) unsigned char smem[];
  const long long t_kernel0 = pa.kprof ? clock64() : 0;
  const Dims& d = pa.d;
  const int nbuf = d.nbuf;
  const SmemLayout lay = smem_layout(d, nbuf);
  double* ws0 = reinterpret_cast<double*>(smem + lay.ws_off);  // W chunk buffers 0, 1
  int* slt = reinterpret_cast<int*>(smem + lay.slt_off);
  double* gs = reinterpret_cast<double*>(smem + lay.gs_off);
  double* m_run = reinterpret_cast<double*>(smem + lay.col_off);
  double* S_run = m_run + kQMax;
  double* c_m = S_run + kQMax;      // normaliser max of the previous logits (B pass)
  double* c_logS = c_m + kQMax;     // its log-sum
  double* c_eta = c_logS + kQMax;   // η_b of the column's run (B pass)
  double* facb = c_eta + kQMax;     // [2][QCpad] running-max rescale of tile i%2
  double* obj_run = facb + 2 * kQMax;
  double* hobj = obj_run + d.RC;
  double* etab = reinterpret_cast<double*>(smem + lay.tab_off);
  auto xslot = [&](int b) { return reinterpret_cast<XT*>(smem + lay.xs_off + b * lay.xs_bytes); };
  auto sbuf = [&](int i) { return reinterpret_cast<double*>(smem + lay.ss_off + (i & 1) * lay.buf_bytes); };
  auto hbuf = [&](int i) { return reinterpret_cast<double*>(smem + lay.sh_off + (i & 1) * lay.buf_bytes); };
  auto stslot = [&](int b) { return reinterpret_cast<double*>(smem + lay.st_off + b * lay.st_bytes); };

  const int tid = threadIdx.x;
  const bool mma_group = tid < kGroup;
  const int gtid = tid & (kGroup - 1);
  const int lane = tid & 31, gwarp = gtid >> 5;
  const int g = lane >> 2, t4 = lane & 3;
  const int p = d.p;
  const int nRTx = d.Lpad / 8;
  const int nRT = (MODE == kModeA) ? nRTx + kQMax / 8 : nRTx;
  const int WST = w_stride(kQMax);

  // the owned slices' items (all of them unless the pixels are sharded over devices)
  const int K = d.NCH * (d.sl1 - d.sl0);
  const int item_begin = static_cast<int>((static_cast<long long>(blockIdx.x) * K) / gridDim.x);
  const int item_end = static_cast<int>((static_cast<long long>(blockIdx.x + 1) * K) / gridDim.x);
  int ntile = 0;
  for (int k = item_begin; k < item_end; ++k) {
    const int s = item_slice_t<ILV>(d, k);
    ntile += slice_tile(d, s + 1) - slice_tile(d, s);
  }  // once per CTA
  if (ntile == 0) return;

  // ---- one-time setup (all 512 threads) ----
  unsigned long long* full = reinterpret_cast<unsigned long long*>(smem + lay.mbar_off);
  unsigned long long* empty = full + 4;
  unsigned long long* sready = empty + 4;  // [2] S(i) written by all 8 MMA warps
  unsigned long long* wready = sready + 2; // [2] w(i), fac(i) written by all 8 update warps
  unsigned long long* sfree = wready + 2;  // [kNSB] every MMA warp is done with w(i) (P3(i))
  for (int i = tid; i <= d.nslices; i += kThreads) slt[i] = slice_tile(d, i);
  if (tid == 0) {
    for (int b = 0; b < nbuf; ++b) {
      mbar_init(full + b, 1);   // the producer's arrive.expect_tx; TMA completes the bytes
      mbar_init(empty + b, 8);  // one arrive per MMA warp after its last read of the tile
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(sready + b, 8);
      mbar_init(wready + b, 8);
    }
    for (int b = 0; b < kNSB; ++b) mbar_init(sfree + b, 8);
    mbar_fence_init();
  }
  // Cross-group hand-offs on mbarriers: every warp arrives or waits on its own, so
  // no warp of one group ever waits for a slower warp of the same group.
  auto warp_arrive = [&](unsigned long long* bar) {
    __syncwarp();
    if (lane == 0) mbar_arrive(bar);
  };
  auto s_arrive = [&](int i) { warp_arrive(sready + (i & 1)); };
  auto s_wait = [&](int i) { mbar_wait(sready + (i & 1), (i >> 1) & 1); };
  auto w_arrive = [&](int i) { warp_arrive(wready + (i & 1)); };
  auto w_wait = [&](int i) { mbar_wait(wready + (i & 1), (i >> 1) & 1); };
  if (tid < kQMax) facb[tid] = facb[kQMax + tid] = 1.0;
  griddep_launch_dependents();
  griddep_wait();  // the previous kernel's W / partial normalisers / state are complete
  __syncthreads();
  if (pa.kprof && tid == 0) atomicAdd(pa.kprof + 36 + 4 * MODE, static_cast<unsigned long long>(clock64() - t_kernel0));

  if (mma_group) {
    // =========================== MMA group ===========================
    double acc[RTW][kMaxCT][2];
#pragma unroll
    for (int i = 0; i < RTW; ++i)
#pragma unroll
      for (int c = 0; c < kMaxCT; ++c) acc[i][c][0] = acc[i][c][1] = 0.0;
    const int my_rt = (nRT - gwarp + 7) / 8;  // row tiles gwarp + 8·i < nRT
    const int my_x = (nRTx - gwarp + 7) / 8;  // of which X rows (the rest: one pseudo tile)
    const bool my_pseudo = my_rt > my_x;
    Cursor xc, p1c, p3c;
    cursor_set_t<ILV>(xc, d, slt, item_begin);
    cursor_set_t<ILV>(p1c, d, slt, item_begin);
    cursor_set_t<ILV>(p3c, d, slt, item_begin);
    // W chunk double buffer: ws(wcur) holds chunk wchunk; the next item's chunk is
    // prefetched by cp.async into the other buffer while the current one is in use.
    int wcur = 0, wchunk = -1;
    auto ws_buf = [&](int b) { return reinterpret_cast<double*>(reinterpret_cast<unsigned char*>(ws0) + b * lay.ws_bytes); };
    auto w_fetch = [&](int chunk, int b) {  // one cp.async group per thread (possibly empty)
      double* dstw = ws_buf(b);
      constexpr int kV = kQMax / 2;  // 16-byte pieces per band row
      for (int e = gtid; e < d.Lpad * kV; e += kGroup) {
        const int l = e / kV, c2 = e - l * kV;
        cp_async16(dstw + l * WST + 2 * c2, pa.W + static_cast<size_t>(l) * d.Qs + chunk * kQMax + 2 * c2);
      }
      cp_async_commit();
    };

    const int xrows = x_rows(d), brows = x_box_rows(d);
    // Per-lane constants of the DMMA fragment addressing, hoisted out of the tile loop:
    // P3's swizzled X offsets per k-step and P1's two band-pair offsets / band range.
    int xo3[kNP / 4];
#pragma unroll
    for (int kk = 0; kk < kNP / 4; ++kk) xo3[kk] = xoff<XT>(g, kk * 4 + t4, xrows);
    const int p1_pt = gwarp & 3, p1_half = gwarp >> 2;
    const int p1_xo0 = xoff<XT>(2 * t4, p1_pt * 8 + g, xrows), p1_xo1 = xoff<XT>(2 * t4 + 1, p1_pt * 8 + g, xrows);
    const int p1_h0 = 2 * (d.Lpad / 16);
    const int p1_mb = (p1_half ? p1_h0 : 0) / 2;
    const int p1_mn = (p1_half ? d.Lpad / 4 - p1_h0 : p1_h0) / 2;
    const int nbox = xrows / brows, nhalf = sizeof(XT) / 4;  // row boxes × column halves
    const unsigned tile_tx = static_cast<unsigned>(nbox * nhalf * brows * 128);
    // Producer (MMA thread 0): X(f) into slot f % nbuf once the slot's previous
    // tile has been released by all 8 MMA warps (empty barrier).
    Ring ldr{0, 0}, xwr{0, 0}, p3r{0, 0};  // X ring: producer, P1 consumer, P3 consumer
    auto load_next_x = [&](int f) {
      if (gtid == 0 && !(pa.dbg & 4)) {
        const int b = ldr.slot;
        if (f >= nbuf) mbar_wait(empty + b, ldr.phase ^ 1);
        mbar_expect_tx(full + b, tile_tx);
        XT* dst = xslot(b);
        for (int h = 0; h < nhalf; ++h)
          for (int bx = 0; bx < nbox; ++bx)
            tma_load_2d(dst + h * xrows * (32 / nhalf) + bx * brows * (32 / nhalf), &xmap,
                        xc.tile * kNP + h * 16, bx * brows, full + b);
      }
      ldr.next(nbuf);
      cursor_next_t<ILV>(xc, d, slt);
    };
    auto x_wait = [&]() {  // the next tile for P1; returns its slot
      const int b = xwr.slot;
      if (!(pa.dbg & 4)) mbar_wait(full + b, xwr.phase);
      xwr.next(nbuf);
      return b;
    };
    auto x_release = [&]() {  // P3's tile
      __syncwarp();
      if (lane == 0 && !(pa.dbg & 4)) mbar_arrive(empty + p3r.slot);
      p3r.next(nbuf);
    };
    // P1: S[c][j] = Σ_l W[l][c]·X[l][j]; warp = 8 pixels × one band half.
    auto phase1 = [&](int i, int xb) {
      if (i >= kNSB) mbar_wait(sfree + (i & 1), ((i >> 1) - 1) & 1);  // w(i−2) consumed
      if (MODE == kModeInit || (pa.dbg & 65)) return;
      const int chunk = p1c.chunk;
      if (chunk != wchunk && !(pa.dbg & 4096)) {
        // Switch to the prefetched buffer once every MMA warp is past its previous
        // P1 (so the old buffer is free), then prefetch the following item's chunk.
        if (d.nwb == 2) {
          if (wchunk >= 0) wcur ^= 1;
          cp_async_wait0();
          if (pa.kprof && gtid == 0 && wchunk < 0)
            atomicAdd(pa.kprof + 38 + 4 * MODE, static_cast<unsigned long long>(clock64() - t_kernel0));
          bar_sync(bars::kMma, kGroup);
          // the next item with a different chunk (chunk-major: usually none in this CTA)
          int nx = p1c.item + 1;
          if (d.cmajor) nx = (item_chunk_t<ILV>(d, nx) == chunk) ? (chunk + 1) * (d.sl1 - d.sl0) : nx;
          if (nx < item_end && item_chunk_t<ILV>(d, nx) != chunk) w_fetch(item_chunk_t<ILV>(d, nx), wcur ^ 1);
        } else {  // one buffer: restage in place once every MMA warp is past its previous P1
          if (wchunk >= 0) {
            bar_sync(bars::kMma, kGroup);
            w_fetch(chunk, 0);
          }
          cp_async_wait0();
          bar_sync(bars::kMma, kGroup);
        }
        wchunk = chunk;
      }
      if (pa.dbg & 2048) return;
      const double* ws = ws_buf(wcur);
      const XT* xs = xslot(xb);
      const int pt = p1_pt, half = p1_half;
      double c1[CTF][2];
#pragma unroll
      for (int c = 0; c < CTF; ++c) c1[c][0] = c1[c][1] = 0.0;
      // Bands are taken in pairs of k-steps covering 8 bands: within pair m, lane
      // (g, t4) feeds band 8m + 2·t4 + par (par = 0, 1).  This band order makes
      // both the X B-fragment (rows 2·t4+par hit distinct 128-byte swizzle chunks)
      // and the W A-fragment (row stride 2·WST words ≡ 8 mod 32) conflict-free.
      const double* wcol = ws + 2 * t4 * WST + g;
      const int xo0 = p1_xo0, xo1 = p1_xo1;
      // band halves of even k-step length: K4 = Lpad/4 is even, split at h0 = 2⌊K4/4⌋
      const int mb = p1_mb, mn = p1_mn;
#pragma unroll kP1Unroll
      for (int m2 = 0; m2 < mn; ++m2) {
        const int m = mb + m2;
        const XT* xr = xs + m * 8 * kXRow<XT>;
        const double bx0 = static_cast<double>(xr[xo0]);
        const double bx1 = static_cast<double>(xr[xo1]);
        const double* w0 = wcol + m * 8 * WST;
        const double* w1 = w0 + WST;
#pragma unroll
        for (int ct = 0; ct < CTF; ++ct) dmma(c1[ct], w0[ct * 8], bx0);
#pragma unroll
        for (int ct = 0; ct < CTF; ++ct) dmma(c1[ct], w1[ct * 8], bx1);
      }
      double* dst = half ? hbuf(i) : sbuf(i);
#pragma unroll
      for (int ct = 0; ct < CTF; ++ct)
        *reinterpret_cast<double2*>(dst + (ct * 8 + g) * kSST + pt * 8 + 2 * t4) =
            make_double2(c1[ct][0], c1[ct][1]);
    };

    if (MODE != kModeInit && !(pa.dbg & 65)) w_fetch(item_chunk_t<ILV>(d, item_begin), 0);  // the first chunk (waited in P1(0))
    for (int f = 0; f < nbuf - 1 && f < ntile; ++f) load_next_x(f);  // X(0 .. nbuf−2) in flight
    {
      const int xb0 = x_wait();
      if (pa.kprof && gtid == 0) atomicAdd(pa.kprof + 37 + 4 * MODE, static_cast<unsigned long long>(clock64() - t_kernel0));
      phase1(0, xb0);
    }
    if (pa.kprof && gtid == 0) atomicAdd(pa.kprof + 24 + 3 * MODE, static_cast<unsigned long long>(clock64() - t_kernel0));
    cursor_next_t<ILV>(p1c, d, slt);
    s_arrive(0);
    // P1(i+1) overlaps the update of tile i (measured faster for both pass kinds than
    // the serial order P3(i) → P1(i+1), EDAA_DBG=1024, which keeps the scalar fp64
    // update chain clear of DMMA contention but leaves the tensor pipe idle meanwhile).
    const bool serial = (pa.dbg & 1024) != 0;
    auto next_p1 = [&](int it) {
      if (it + 1 < ntile) {
        int xb;
        {
          EDAA_TSTART();
          xb = x_wait();
          EDAA_TSTOP(0);
        }
        {
          EDAA_TSTART();
          phase1(it + 1, xb);
          EDAA_TSTOP(1);
        }
        cursor_next_t<ILV>(p1c, d, slt);
        s_arrive(it + 1);
      }
    };
    for (int it = 0; it < ntile; ++it) {
      // X(i+nbuf−1) into X(i−1)'s slot (released after P3(i−1)): nbuf−1 tiles of lead
      {
        const long long tq_ = (pa.kprof && lane == 0 && gwarp == 0) ? clock64() : 0;
        if (it + nbuf - 1 < ntile) load_next_x(it + nbuf - 1);
        if (pa.kprof && lane == 0 && gwarp == 0)
          atomicAdd(pa.kprof + 52 + 2 * MODE, static_cast<unsigned long long>(clock64() - tq_));
      }
      if (!serial) next_p1(it);
      {
        EDAA_TSTART();
        w_wait(it);  // w(i), fac(i) ready
        EDAA_TSTOP(2);
      }
      if (MODE != kModeObj) {
        if (MODE == kModeB || MODE == kModeInit) {
          const double* fac = facb + (it & 1) * kQMax;
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
        // P3: C[l][c] += Σ_j X[l][j]·w[c][j]; warp owns row tiles gwarp, gwarp+8, …
        const XT* xs = xslot(p3r.slot);
        const double* w = sbuf(it);
        EDAA_TSTART();
        if (!(pa.dbg & 129)) {
          switch (my_x + (my_pseudo ? 8 : 0)) {  // warp-uniform: the DMMAs below are unpredicated
            case 1: accumulate_tiles<1, false, CTF>(acc, xs, w, gwarp, nRTx, g, t4, xo3); break;
            case 2: accumulate_tiles<2, false, CTF>(acc, xs, w, gwarp, nRTx, g, t4, xo3); break;
            case 3: accumulate_tiles<3, false, CTF>(acc, xs, w, gwarp, nRTx, g, t4, xo3); break;
            case 4: if constexpr (RTW >= 4) accumulate_tiles<4, false, CTF>(acc, xs, w, gwarp, nRTx, g, t4, xo3); break;
            case 5: if constexpr (RTW >= 5) accumulate_tiles<5, false, CTF>(acc, xs, w, gwarp, nRTx, g, t4, xo3); break;
            case 6: if constexpr (RTW >= 6) accumulate_tiles<6, false, CTF>(acc, xs, w, gwarp, nRTx, g, t4, xo3); break;
            case 8: if constexpr (MODE == kModeA) accumulate_tiles<0, true, CTF>(acc, xs, w, gwarp, nRTx, g, t4, xo3); break;
            case 9: if constexpr (MODE == kModeA) accumulate_tiles<1, true, CTF>(acc, xs, w, gwarp, nRTx, g, t4, xo3); break;
            case 10: if constexpr (MODE == kModeA) accumulate_tiles<2, true, CTF>(acc, xs, w, gwarp, nRTx, g, t4, xo3); break;
            case 11: if constexpr (MODE == kModeA) accumulate_tiles<3, true, CTF>(acc, xs, w, gwarp, nRTx, g, t4, xo3); break;
            case 12: if constexpr (MODE == kModeA && RTW >= 5) accumulate_tiles<4, true, CTF>(acc, xs, w, gwarp, nRTx, g, t4, xo3); break;
            case 13: if constexpr (MODE == kModeA && RTW >= 6) accumulate_tiles<5, true, CTF>(acc, xs, w, gwarp, nRTx, g, t4, xo3); break;
            default: break;
          }
        }
        EDAA_TSTOP(3);
        if (p3c.tile + 1 == p3c.tend) {  // the item's last tile: flush and restart its partials
          const int slice = p3c.slice, col0 = p3c.chunk * kQMax;
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
#pragma unroll
            for (int ct = 0; ct < kMaxCT; ++ct) acc[i][ct][0] = acc[i][ct][1] = 0.0;
          }
        }
      }
      const long long tr_ = (pa.kprof && lane == 0 && gwarp == 0) ? clock64() : 0;
      x_release();  // this warp is done with X(i) (P1(i) and P3(i))
      warp_arrive(sfree + (it & 1));  // … and with S(i)/w(i)
      cursor_next_t<ILV>(p3c, d, slt);
      if (pa.kprof && lane == 0 && gwarp == 0)
        atomicAdd(pa.kprof + 53 + 2 * MODE, static_cast<unsigned long long>(clock64() - tr_));
      if (serial) next_p1(it);
    }
    if (pa.kprof && gtid == 0) {  // per-CTA MMA-loop end: sum and max over CTAs
      const unsigned long long tt = static_cast<unsigned long long>(clock64() - t_kernel0);
      atomicAdd(pa.kprof + 25 + 3 * MODE, tt);
      atomicMax(pa.kprof + 26 + 3 * MODE, tt);
    }
  } else {
    // ========================== update group ==========================
    // the exp table is this group's alone: loaded here, off the MMA group's path to its first
    // tile (the bar_sync at the top of the tile loop orders it before the first exp)
    if (gtid < kExpTab) etab[gtid] = kExp2Tab[gtid];
    Cursor sc, p2c;
    cursor_set_t<ILV>(sc, d, slt, item_begin);
    cursor_set_t<ILV>(p2c, d, slt, item_begin);
    int cchunk = -1;
    int stl = 0, stu = 0;  // state-tile ring (3 slots): next load, current use
    auto next_state = [&](int f) {  // one commit group per call (empty past the end)
      if (f < ntile) {
        const ChunkInfo cn = chunk_info(d, sc.chunk);
        issue_state<MODE>(pa, stslot(stl), sc.tile * kNP, cn.srow0, cn.ncol, gtid);
        stl = (stl == 2) ? 0 : stl + 1;
        cursor_next_t<ILV>(sc, d, slt);
      } else {
        cp_async_commit();
      }
    };
    next_state(0);
    next_state(1);
    if (pa.dbg & 256) {  // development: bare hand-shake, no update work
      for (int it = 0; it < ntile; ++it) {
        s_wait(it);
        w_arrive(it);
      }
      return;
    }
    for (int it = 0; it < ntile; ++it) {
      const ChunkInfo ci = chunk_info(d, p2c.chunk);
      const int j0 = p2c.tile * kNP;
      const bool item_first = p2c.tile == p2c.tstart;
      const bool item_last = p2c.tile + 1 == p2c.tend;
      bar_sync(bars::kUpd, kGroup);  // everyone is done with st(i−1) and the previous item's scalars
      next_state(it + 2);            // into st(i−1)'s slot
      if (ci.chunk != cchunk) {  // per-column constants and G blocks of the new chunk
        if (gtid < kQMax) {
          const int c = gtid;
          const bool real = c < ci.ncol;
          // log b_old = ℓ − (m + log S): one subtraction per element
          c_m[c] = (MODE == kModeB && real) ? pa.colm[ci.col0 + c] + pa.collogS[ci.col0 + c] : 0.0;
          c_eta[c] = (MODE == kModeB && real) ? pa.eta_b[ci.run0 + c / p]
                     : ((MODE == kModeA && c < ci.RCe) ? pa.eta_a[ci.run0 + c] : 0.0);  // B: per column, A: per run
        }
        if (MODE == kModeA || MODE == kModeObj) {
          for (int e = gtid; e < ci.RCe * p * p; e += kGroup) {
            const int rl = e / (p * p), rem = e % (p * p);
            const int i = rem / p, m = rem % p;
            gs[e] = pa.Gbuf[static_cast<size_t>(rl * p + i) * d.Qs + ci.col0 + rl * p + m];
          }
        }
        cchunk = ci.chunk;
      }
      if (item_first) {
        if (gtid < kQMax) {
          m_run[gtid] = -INFINITY;
          S_run[gtid] = 0.0;
        }
        if (gtid < d.RC) obj_run[gtid] = 0.0;
      }
      cp_async_wait2();  // st(i) landed (st(i+1), st(i+2) may still fly)
      bar_sync(bars::kUpd, kGroup);  // st(i), constants and resets visible
      {
        EDAA_TSTART();
        s_wait(it);  // S(i) ready
        EDAA_TSTOP(4);
      }
      EDAA_TSTART();
      double* ss = sbuf(it);
      const double* sh = hbuf(it);
      const double* st = stslot(stu);
      stu = (stu == 2) ? 0 : stu + 1;
      double* fac = facb + (it & 1) * kQMax;

      if (MODE == kModeA || MODE == kModeObj) {
        constexpr int TPP = LanesPerPixel<PT>::value;
        for (int q2 = gtid; q2 < ci.RCe * kNP * TPP; q2 += kGroup) {  // warp-uniform trip count
          const int q = q2 / TPP, sub = q2 % TPP;
          const int rl = q / kNP, j = q % kNP;
          const int pix = j0 + j;
          double o = (p == PT)
              ? pixel_a_update<PT, TPP, MODE == kModeA, true>(pa, ci.run0 + rl, rl, j, pix, pix < d.N, sub,
                                                              ss, sh, st, gs, etab, c_eta)
              : pixel_a_update<PT, TPP, MODE == kModeA, false>(pa, ci.run0 + rl, rl, j, pix, pix < d.N, sub,
                                                               ss, sh, st, gs, etab, c_eta);
          o = warp_sum(o);
          if (lane == 0) hobj[q2 >> 5] = o;  // warp-task q2/32 belongs to run (q2/32)/TPP
        }
        if (MODE == kModeA)
          for (int e = gtid; e < (kQMax - ci.ncol) * kNP; e += kGroup)
            ss[(ci.ncol + e / kNP) * kSST + e % kNP] = 0.0;
        bar_sync(bars::kUpd, kGroup);
        if (gtid < ci.RCe) {
          double o = obj_run[gtid];
          for (int h = 0; h < TPP; ++h) o += hobj[gtid * TPP + h];
          obj_run[gtid] = o;
        }
      } else if (!(pa.dbg & 2)) {
        // B step / B⁰: new logits; 8 lanes per column, 4 pixels per lane (j = k·8 + lane8).
        const int c = gtid >> 3, l8 = gtid & 7;
        const bool active = c < kQMax;  // QCpad·8 ≤ 192 threads carry columns
        double ell[4];
        double tmax = -INFINITY;
        if (active) {
          const bool real = c < ci.ncol;
          const int rl = real ? c / p : 0, i = real ? c % p : 0, r = ci.run0 + rl;
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
                double lb = st[c * kNP + j] - c_m[c];                      // log b_old
                lb = (lb < log_floor()) ? log_floor() : lb;                // log max(b, 1e-30)
                v = lb + (ss[c * kSST + j] + sh[c * kSST + j]) * c_eta[c]; // + η_b·(−∇_B)
              }
              pa.Lg[static_cast<size_t>(ci.srow0 + c) * d.Npad + pix] = v;
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
            const double w = (mn == -INFINITY) ? 0.0 : exp_nonpos(ell[k] - mn, etab);
            ss[c * kSST + k * 8 + l8] = w;
            tsum += w;
          }
        }
#pragma unroll
        for (int o = 4; o > 0; o >>= 1) tsum += __shfl_xor_sync(0xffffffffu, tsum, o);
        if (active && l8 == 0) {
          const double f = (mn == -INFINITY || mn == mo) ? 1.0 : exp_nonpos(mo - mn, etab);
          fac[c] = f;
          S_run[c] = S_run[c] * f + tsum;
          m_run[c] = mn;
        }
      }
      EDAA_TSTOP(5);
      if (item_last) {  // the item's softmax / objective partials
        bar_sync(bars::kUpd, kGroup);
        const int slice = p2c.slice;
        if (MODE == kModeB || MODE == kModeInit) {
          if (gtid < kQMax) {
            pa.part_m[static_cast<size_t>(slice) * d.Qs + ci.col0 + gtid] = m_run[gtid];
            pa.part_S[static_cast<size_t>(slice) * d.Qs + ci.col0 + gtid] = S_run[gtid];
          }
        } else {
          if (gtid < ci.RCe) pa.part_obj[static_cast<size_t>(slice) * d.M + ci.run0 + gtid] = obj_run[gtid];
        }
      }
      w_arrive(it);  // w(i), fac(i) ready for P3(i)
      cursor_next_t<ILV>(p2c, d, slt);
    }
  }
}

// PTS selects the p buckets this instantiation carries (kPtAll, kPtLo = 2-5,
// kPtHi = 6-16): a template parameter, not a macro, so translation units that
// carry different bucket sets never define the same function differently.
enum PtSet : int { kPtAll = 0, kPtLo = 1, kPtHi = 2 };

template <int MODE, int RTW, class XT, int PTS, int CTF>
cudaError_t launch_pass_ctf(const PassArgs& a, cudaStream_t st, int pt) {
  const dim3 grid(std::min(a.d.NCH * (a.d.sl1 - a.d.sl0), a.d.ncta));
  const size_t smem = dev::smem_layout(a.d, a.d.nbuf).total;
  void (*kern)(PassArgs, CUtensorMap) = nullptr;
  // The interleaved instantiation for the A/B passes of large images (Dims::ilv).
  constexpr bool kIlvOk = CTF == kMaxCT && (MODE == kModeA || MODE == kModeB);
  const bool ilv = kIlvOk && a.d.ilv != 0;
  if constexpr (MODE == kModeInit || MODE == kModeB) {
    kern = k_pass<MODE, 1, RTW, XT, CTF>;
    if constexpr (kIlvOk)
      if (ilv) kern = k_pass<MODE, 1, RTW, XT, CTF, true>;
  } else {
    switch (pt) {
#define EDAA_PT_CASE(P)                                                                         \
  case P:                                                                                       \
    if constexpr ((PTS == kPtAll || (PTS == kPtLo) == (P <= 5)) && (CTF == kMaxCT || P <= 8)) \
      kern = ilv ? k_pass<MODE, P, RTW, XT, CTF, kIlvOk> : k_pass<MODE, P, RTW, XT, CTF>;         \
    break;
      EDAA_PT_CASE(2) EDAA_PT_CASE(3) EDAA_PT_CASE(4) EDAA_PT_CASE(5)
      EDAA_PT_CASE(6) EDAA_PT_CASE(7) EDAA_PT_CASE(8) EDAA_PT_CASE(10) EDAA_PT_CASE(12) EDAA_PT_CASE(16)
#undef EDAA_PT_CASE
      default:
        break;
    }
    if (kern == nullptr) return cudaErrorInvalidValue;
  }
  // Always the device maximum, never this launch's size: the attribute is per-function
  // state shared by every context on the device, so two host threads solving different
  // batches concurrently would otherwise lower it under each other's launches.
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, kMaxSmem);
  if (e != cudaSuccess) return e;
  e = launch_pdl(a.d.pdl != 0, kern, grid, dim3(kThreads), smem, st, a, *static_cast<const CUtensorMap*>(a.xmap));
  if (e != cudaSuccess) return e;
  return cudaGetLastError();
}

// A batch that fits one 8-column DMMA tile (a single run with p ≤ 8) runs the
// CTF = 1 kernels; every other batch the full-chunk ones.
template <int MODE, int RTW, class XT, int PTS>
cudaError_t launch_pass_rtw(const PassArgs& a, cudaStream_t st, int pt) {
  return (a.d.NCH == 1 && a.d.M * a.d.p <= 8) ? launch_pass_ctf<MODE, RTW, XT, PTS, 1>(a, st, pt)
                                              : launch_pass_ctf<MODE, RTW, XT, PTS, kMaxCT>(a, st, pt);
}

// Per-mode entry points: each translation unit edaa_pass_<x>_<part>.cu instantiates
// one (image type, mode, p-bucket range) so the kernels compile in parallel.
template <int MODE, class XT, int PTS = kPtAll>
cudaError_t launch_pass_mode(const PassArgs& a, cudaStream_t st) {
  const int pt = pt_bucket(a.d.p);
  const bool wide = (a.d.Lpad / 8 + kQMax / 8) > 32;  // > 4 row tiles per warp
  if constexpr (MODE == kModeObj) {
    return launch_pass_rtw<kModeObj, 1, XT, PTS>(a, st, pt);
  } else {
    return wide ? launch_pass_rtw<MODE, 6, XT, PTS>(a, st, pt) : launch_pass_rtw<MODE, 4, XT, PTS>(a, st, pt);
  }
}

}  // namespace pass_impl
}  // namespace edaa
