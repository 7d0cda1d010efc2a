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
__device__ __forceinline__ void cp_async_wait_all() {
  asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;\n" ::: "memory");
}

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
  int xs_off, ws_off, ss_off, obj_off, gs_off, col_off, total;
};

__host__ __device__ inline int align16(int b) { return (b + 15) & ~15; }

__host__ __device__ inline int w_stride(int qcpad) { return qcpad + ((qcpad % 16 == 0) ? 8 : 0); }

__host__ __device__ inline SmemLayout smem_layout(const Dims& d) {
  SmemLayout s;
  int off = 0;
  s.xs_off = off;
  off += align16(d.Lpad * kXST * 4);
  s.ws_off = off;
  off += align16(d.Lpad * w_stride(d.QCpad) * 8);
  s.ss_off = off;
  off += align16(d.QCpad * kSST * 8);
  s.obj_off = off;
  off += align16(d.RC * kNP * 8);
  s.gs_off = off;
  off += align16(d.RC * d.p * d.p * 8);
  s.col_off = off;  // m_run, S_run, fac (QCpad each) + obj_run (RC)
  off += align16((3 * d.QCpad + d.RC) * 8);
  s.total = off;
  return s;
}

// ---------------------------------------------------------------------------
// Per-pixel A update: objective term + K1 entropic steps (solver.cpp:212-218).
// P (= Yᵀx_j, the projection) is read from the weight tile; G = YᵀY of the
// run is in shared memory; a is the pixel's p-vector.
// log(a_i) after a softmax is carried in the log domain,
// log a_i = s_i − top − log Σ, which equals log(e_i/Σ) up to rounding; the
// 1e-30 floor is applied to it as solver.cpp:25 does to a_i.
template <int PT, bool UPDATE>
__device__ __forceinline__ void pixel_a_update(const PassArgs& pa, int r, int rl, int j, int pix,
                                               double* ss, const double* gs, double* obj_s) {
  const Dims& d = pa.d;
  const int p = d.p;
  double a[PT], la[PT];
  const size_t base = static_cast<size_t>(r) * p * d.Npad + pix;
#pragma unroll
  for (int i = 0; i < PT; ++i) {
    if (i < p) {
      a[i] = pa.A[base + static_cast<size_t>(i) * d.Npad];
      const double z = (a[i] < kLogFloorValue) ? kLogFloorValue : a[i];  // std::max(z, 1e-30)
      la[i] = log(z);
    }
  }
  const double* G = gs + rl * p * p;
  const double* Pcol = ss + (rl * p) * kSST + j;
  const double eta = pa.eta_a[r];
  double aPa = 0.0, aGa = 0.0;
  const int steps = UPDATE ? d.K1 : 1;
  bool bad = false;
  for (int k = 0; k < steps; ++k) {
    double top = -INFINITY;
#pragma unroll
    for (int i = 0; i < PT; ++i) {
      if (i < p) {
        double ga = 0.0;
#pragma unroll
        for (int m = 0; m < PT; ++m)
          if (m < p) ga += G[i * p + m] * a[m];
        const double Pi = Pcol[i * kSST];
        if (k == 0) {
          aPa += a[i] * Pi;
          aGa += a[i] * ga;
        }
        // −∇_A = (XB)ᵀ(X − XBA) = P − G·a, scaled by η_a, added to log z.
        const double s = la[i] + (Pi - ga) * eta;
        la[i] = s;
        top = max_like_std(top, s);
      }
    }
    if (!UPDATE) break;
    double total = 0.0;
#pragma unroll
    for (int i = 0; i < PT; ++i) {
      if (i < p) {
        a[i] = exp(la[i] - top);
        total += a[i];
      }
    }
    const double ltot = log(total);
#pragma unroll
    for (int i = 0; i < PT; ++i) {
      if (i < p) {
        a[i] = a[i] / total;
        bad |= !isfinite(a[i]);
        const double l2 = la[i] - top - ltot;
        la[i] = (l2 < log_floor()) ? log_floor() : l2;
      }
    }
    if (pa.observe_A != nullptr) {
#pragma unroll
      for (int i = 0; i < PT; ++i)
        if (i < p) pa.observe_A[(static_cast<size_t>(k) * p + i) * d.Npad + pix] = a[i];
    }
  }
  obj_s[rl * kNP + j] = 0.5 * ((pa.xnorm[pix] - 2.0 * aPa) + aGa);
  if (UPDATE) {
    if (bad) atomicMin(pa.fail_key + r, static_cast<unsigned long long>(pa.t) << 1);
#pragma unroll
    for (int i = 0; i < PT; ++i) {
      if (i < p) {
        pa.A[base + static_cast<size_t>(i) * d.Npad] = a[i];
        ss[(rl * p + i) * kSST + j] = a[i];
      }
    }
  }
}

// ---------------------------------------------------------------------------
// The pass kernel. grid = (nslices, NCH), block = 256.
template <int MODE, int PT, int RTW>
__global__ void __launch_bounds__(kThreads, 1) k_pass(PassArgs pa) {
  extern __shared__ __align__(16) unsigned char smem[];
  const Dims& d = pa.d;
  const SmemLayout lay = smem_layout(d);
  float* xs = reinterpret_cast<float*>(smem + lay.xs_off);
  double* ws = reinterpret_cast<double*>(smem + lay.ws_off);
  double* ss = reinterpret_cast<double*>(smem + lay.ss_off);
  double* obj_s = reinterpret_cast<double*>(smem + lay.obj_off);
  double* gs = reinterpret_cast<double*>(smem + lay.gs_off);
  double* m_run = reinterpret_cast<double*>(smem + lay.col_off);
  double* S_run = m_run + d.QCpad;
  double* fac = S_run + d.QCpad;
  double* obj_run = fac + d.QCpad;

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

  double acc[RTW][4][2];
#pragma unroll
  for (int i = 0; i < RTW; ++i)
#pragma unroll
    for (int c = 0; c < 4; ++c) acc[i][c][0] = acc[i][c][1] = 0.0;

  const int tile_begin = static_cast<int>((static_cast<long long>(slice) * d.ntiles) / d.nslices);
  const int tile_end = static_cast<int>((static_cast<long long>(slice + 1) * d.ntiles) / d.nslices);

  for (int tile = tile_begin; tile < tile_end; ++tile) {
    const int j0 = tile * kNP;
    // ---- X tile → shared (16 B cp.async, rows < L) ----
    for (int e = tid; e < d.L * (kNP / 4); e += kThreads) {
      const int l = e / (kNP / 4), q = e % (kNP / 4);
      cp_async16(xs + l * kXST + q * 4, pa.X + static_cast<size_t>(l) * d.Npad + j0 + q * 4);
    }
    cp_async_wait_all();
    __syncthreads();

    // ---- phase 1: S[c][j] = Σ_l W[l][c]·X[l][j]  (DMMA, warp = 8 pixels) ----
    if (MODE != kModeInit) {
      double c1[4][2];
#pragma unroll
      for (int c = 0; c < 4; ++c) c1[c][0] = c1[c][1] = 0.0;
      const float* xcol = xs + warp * 8 + g;
      const double* wcol = ws + g;
      for (int kk = 0; kk < d.Lpad / 4; ++kk) {
        const int l = kk * 4 + t4;
        const double bx = static_cast<double>(xcol[l * kXST]);
#pragma unroll
        for (int ct = 0; ct < 4; ++ct)
          if (ct < nCT) dmma(c1[ct], wcol[l * WST + ct * 8], bx);
      }
#pragma unroll
      for (int ct = 0; ct < 4; ++ct)
        if (ct < nCT)
          *reinterpret_cast<double2*>(ss + (ct * 8 + g) * kSST + warp * 8 + 2 * t4) =
              make_double2(c1[ct][0], c1[ct][1]);
    }
    __syncthreads();

    // ---- phase 2: per-pixel updates ----
    if (MODE == kModeA || MODE == kModeObj) {
      for (int q = tid; q < RCe * kNP; q += kThreads) {
        const int rl = q / kNP, j = q % kNP;
        const int pix = j0 + j;
        if (pix < d.N) {
          pixel_a_update<PT, MODE == kModeA>(pa, run0 + rl, rl, j, pix, ss, gs, obj_s);
        } else {
          obj_s[rl * kNP + j] = 0.0;
          if (MODE == kModeA)
            for (int i = 0; i < p; ++i) ss[(rl * p + i) * kSST + j] = 0.0;
        }
      }
      if (MODE == kModeA)
        for (int e = tid; e < (d.QCpad - ncol_valid) * kNP; e += kThreads)
          ss[(ncol_valid + e / kNP) * kSST + e % kNP] = 0.0;
      __syncthreads();
      if (tid < RCe) {  // fixed-order per-run objective partial
        double s = obj_run[tid];
        const int jn = min(kNP, d.N - j0);
        for (int j = 0; j < jn; ++j) s += obj_s[tid * kNP + j];
        obj_run[tid] = s;
      }
      if (MODE == kModeObj) {
        __syncthreads();
        continue;
      }
    } else {  // B step or B⁰ initialisation: new logits, online column max
      for (int e = tid; e < d.QCpad * kNP; e += kThreads) {
        const int c = e / kNP, j = e % kNP;
        const int pix = j0 + j;
        double ell = -INFINITY;
        if (c < ncol_valid && pix < d.N) {
          const int rl = c / p, i = c % p, r = run0 + rl;
          const size_t idx = (static_cast<size_t>(r) * p + i) * d.Npad + pix;
          if (MODE == kModeInit) {
            // solver.cpp:122-127: column i consumes draws i·N .. i·N+N−1.
            ell = 0.1 * splitmix_unit_at(pa.seeds[r],
                                         static_cast<uint64_t>(i) * d.N + static_cast<uint64_t>(pix));
          } else {
            const int gc = col0 + c;
            double lb = pa.Lg[idx] - pa.colm[gc] - pa.collogS[gc];  // log b_old
            lb = (lb < log_floor()) ? log_floor() : lb;              // log max(b, 1e-30)
            ell = lb + ss[c * kSST + j] * pa.eta_b[r];               // + η_b·(−∇_B)
          }
          pa.Lg[idx] = ell;
        }
        ss[c * kSST + j] = ell;
      }
      __syncthreads();
      if (tid < d.QCpad) {
        double tmax = -INFINITY;
        for (int j = 0; j < kNP; ++j) tmax = max_like_std(tmax, ss[tid * kSST + j]);
        const double mo = m_run[tid];
        const double mn = max_like_std(mo, tmax);
        fac[tid] = (mn == -INFINITY || mn == mo) ? 1.0 : exp(mo - mn);
        m_run[tid] = mn;
      }
      __syncthreads();
      for (int e = tid; e < d.QCpad * kNP; e += kThreads) {
        const int c = e / kNP, j = e % kNP;
        const double m = m_run[c];
        const double v = ss[c * kSST + j];
        ss[c * kSST + j] = (m == -INFINITY) ? 0.0 : exp(v - m);
      }
      __syncthreads();
      if (tid < d.QCpad) {
        double s = S_run[tid] * fac[tid];
        for (int j = 0; j < kNP; ++j) s += ss[tid * kSST + j];
        S_run[tid] = s;
      }
      // rescale running accumulators to the new column max
#pragma unroll
      for (int ct = 0; ct < 4; ++ct) {
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
      for (int kk = 0; kk < kNP / 4; ++kk) {
        double bw[4];
#pragma unroll
        for (int ct = 0; ct < 4; ++ct) bw[ct] = (ct < nCT) ? wrow[ct * 8 * kSST + kk * 4] : 0.0;
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
            for (int ct = 0; ct < 4; ++ct)
              if (ct < nCT) dmma(acc[i][ct], ax, bw[ct]);
          }
        }
      }
    }
    __syncthreads();
  }

  // ---- write this CTA's partials ----
  if (MODE != kModeObj) {
#pragma unroll
    for (int i = 0; i < RTW; ++i) {
      const int rt = warp + 8 * i;
      if (rt < nRT) {
        const int row = rt * 8 + g;
#pragma unroll
        for (int ct = 0; ct < 4; ++ct) {
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
// Combine: block = 256 threads over 32 columns × 8 row lanes.
__global__ void __launch_bounds__(256) k_combine(CombineArgs ca) {
  extern __shared__ __align__(16) unsigned char smem[];
  const Dims& d = ca.d;
  const int lane = threadIdx.x & 31, ry = threadIdx.x >> 5;
  const int col = blockIdx.x * 32 + lane;
  const bool colv = col < d.Qs;
  const int S = d.nslices;
  if (ca.mode == kModeA || ca.mode == kModeObj) {
    for (int row = ry; ca.mode == kModeA && row < d.Lrows; row += 8) {
      if (!colv) continue;
      double s = 0.0;
      for (int sl = 0; sl < S; ++sl) s += ca.part_C[(static_cast<size_t>(sl) * d.Lrows + row) * d.Qs + col];
      if (row < d.Lpad)
        ca.XAt[static_cast<size_t>(row) * d.Qs + col] = s;
      else
        ca.AAt[static_cast<size_t>(row - d.Lpad) * d.Qs + col] = s;
    }
    if (blockIdx.x == 0) {
      for (int r = threadIdx.x; r < d.M; r += blockDim.x) {
        double o = 0.0;
        for (int sl = 0; sl < S; ++sl) o += ca.part_obj[static_cast<size_t>(sl) * d.M + r];
        ca.trace[static_cast<size_t>(r) * ca.trace_stride + ca.trace_index] = o;
      }
    }
    return;
  }
  // log-sum-exp combine of the per-slice column softmax partials
  double* fs = reinterpret_cast<double*>(smem);  // [S][32]
  __shared__ double Ssh[32];
  if (ry == 0) {
    double m = -INFINITY, Ssum = 0.0;
    if (colv) {
      for (int sl = 0; sl < S; ++sl) m = max_like_std(m, ca.part_m[static_cast<size_t>(sl) * d.Qs + col]);
      for (int sl = 0; sl < S; ++sl) {
        const double ms = ca.part_m[static_cast<size_t>(sl) * d.Qs + col];
        const double f = (ms == -INFINITY) ? 0.0 : exp(ms - m);
        fs[sl * 32 + lane] = f;
        Ssum += ca.part_S[static_cast<size_t>(sl) * d.Qs + col] * f;
      }
      ca.colm[col] = m;
      ca.colS[col] = Ssum;
      ca.collogS[col] = log(Ssum);
      // A B column is valid iff it belongs to a run; padded slots have m = −inf.
      const int chunk = col / d.QCpad, c = col % d.QCpad;
      const int r = chunk * d.RC + c / d.p;
      if (c < d.RC * d.p && r < d.M && m != -INFINITY) {
        if (!(isfinite(m) && isfinite(Ssum) && Ssum > 0.0))
          atomicMin(ca.fail_key + r, (static_cast<unsigned long long>(ca.t) << 1) | 1ull);
      } else if (c < d.RC * d.p && r < d.M) {
        atomicMin(ca.fail_key + r, (static_cast<unsigned long long>(ca.t) << 1) | 1ull);
      }
    }
    Ssh[lane] = Ssum;
  }
  __syncthreads();
  if (!colv) return;
  const double Ssum = Ssh[lane];
  for (int row = ry; row < d.Lpad; row += 8) {
    double s = 0.0;
    for (int sl = 0; sl < S; ++sl)
      s += ca.part_C[(static_cast<size_t>(sl) * d.Lrows + row) * d.Qs + col] * fs[sl * 32 + lane];
    ca.Y[static_cast<size_t>(row) * d.Qs + col] = s / Ssum;
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
  const dim3 grid(a.d.nslices, a.d.NCH);
  const size_t smem = smem_layout(a.d).total;
  void (*kern)(PassArgs) = nullptr;
  if (MODE == kModeInit || MODE == kModeB) {
    kern = k_pass<MODE, 1, RTW>;
  } else {
    switch (pt) {
#define EDAA_PT_CASE(P) \
  case P:               \
    kern = k_pass<MODE, P, RTW>; \
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

size_t pass_smem_bytes(int /*mode*/, const Dims& d) { return smem_layout(d).total; }

cudaError_t launch_pass(int mode, const PassArgs& a, cudaStream_t st) {
  const int pt = pt_bucket(a.d.p);
  const bool wide = (a.d.Lpad / 8 + a.d.QCpad / 8) > 32;
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
  const int blocks = (a.d.Qs + 31) / 32;
  const size_t smem = (a.mode == kModeA || a.mode == kModeObj) ? 0 : static_cast<size_t>(a.d.nslices) * 32 * 8;
  cudaError_t e = cudaFuncSetAttribute(k_combine, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       static_cast<int>(smem));
  if (e != cudaSuccess) return e;
  k_combine<<<blocks, 256, smem, st>>>(a);
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
