// Single-evaluation primitives of the solver API on the device: the residual
// R = X − (XB)·A and what the reference derives from it — ½‖R‖²
// (objective_l2, solver.cpp:184-188), Σ|R| (fit_l1, ensemble.cpp:29-39),
// −(XB)ᵀR (grad_abundances, solver.cpp:166-172), −Xᵀ(R·Aᵀ)
// (grad_contributions, solver.cpp:174-182) — and estimate_abundances
// (solver.cpp:240-259).  Every per-entry product follows the reference's
// accumulation order (inner index ascending, multiply then add, from 0.0), so
// with an fp32-exact or fp64 image the entries are the reference's bits; only
// the final sums over all pixels use a fixed-order tree.
// These are evaluation/test-surface functions, not the batched hot path.
#include <cmath>

#include "edaa_device.cuh"

namespace edaa {
namespace {

using namespace dev;

template <class XT>
__global__ void k_residual(const XT* X, const double* Y, const double* A, double* R, int L, int N,
                           int Npad, int p) {
  const size_t total = static_cast<size_t>(L) * Npad;
  for (size_t e = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; e < total;
       e += static_cast<size_t>(gridDim.x) * blockDim.x) {
    const int l = static_cast<int>(e / Npad), j = static_cast<int>(e % Npad);
    if (j >= N) {
      R[e] = 0.0;
      continue;
    }
    double rec = 0.0;
    for (int i = 0; i < p; ++i)
      rec = __dadd_rn(rec, __dmul_rn(Y[l * p + i], A[static_cast<size_t>(i) * Npad + j]));
    R[e] = __dsub_rn(static_cast<double>(X[e]), rec);
  }
}

// mode 0: Σ r², mode 1: Σ |r|; fixed per-thread order then a fixed tree.
__global__ void k_reduce(const double* R, size_t total, int mode, double* part) {
  __shared__ double red[256];
  double s = 0.0;
  for (size_t e = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; e < total;
       e += static_cast<size_t>(gridDim.x) * blockDim.x)
    s += (mode == 0) ? R[e] * R[e] : fabs(R[e]);
  red[threadIdx.x] = s;
  __syncthreads();
  for (int w = 128; w > 0; w >>= 1) {
    if (threadIdx.x < w) red[threadIdx.x] += red[threadIdx.x + w];
    __syncthreads();
  }
  if (threadIdx.x == 0) part[blockIdx.x] = red[0];
}

__global__ void k_sum_parts(const double* part, int n, double scale, double* out) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  double s = 0.0;
  for (int b = 0; b < n; ++b) s += part[b];
  *out = scale * s;
}

// g[i][j] = −Σ_l Y[l][i]·R[l][j]  (matrix.cpp:97-112 order, then ×(−1))
__global__ void k_grad_a(const double* Y, const double* R, double* G, int L, int N, int Npad, int p) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= N) return;
  for (int i = 0; i < p; ++i) {
    double s = 0.0;
    for (int l = 0; l < L; ++l) s = __dadd_rn(s, __dmul_rn(Y[l * p + i], R[static_cast<size_t>(l) * Npad + j]));
    G[static_cast<size_t>(i) * N + j] = -s;
  }
}

// rat[l][i] = Σ_j R[l][j]·A[i][j]  (matrix.cpp:114-131 order)
__global__ void k_rat(const double* R, const double* A, double* rat, int L, int N, int Npad, int p) {
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= L * p) return;
  const int l = e / p, i = e % p;
  double s = 0.0;
  for (int j = 0; j < N; ++j)
    s = __dadd_rn(s, __dmul_rn(R[static_cast<size_t>(l) * Npad + j], A[static_cast<size_t>(i) * Npad + j]));
  rat[e] = s;
}

// g[j][i] = −Σ_l X[l][j]·rat[l][i]
template <class XT>
__global__ void k_grad_b(const XT* X, const double* rat, double* G, int L, int N, int Npad, int p) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= N) return;
  for (int i = 0; i < p; ++i) {
    double s = 0.0;
    for (int l = 0; l < L; ++l)
      s = __dadd_rn(s, __dmul_rn(static_cast<double>(X[static_cast<size_t>(l) * Npad + j]), rat[l * p + i]));
    G[static_cast<size_t>(j) * p + i] = -s;
  }
}

// estimate_abundances (solver.cpp:240-259), one pixel per thread, E staged in shared
// memory; two forms of the step direction −∇ = Eᵀ(x − E·a):
//   FAST (default): the solver's A-pass form P − G·a with P = Eᵀx_j (one L×p
//     product per pixel, once) and G = EᵀE (p×p, once per block): an iteration
//     costs p² instead of 2·L·p multiply-adds, and the entropic
//     step is the solver's multiplicative softmax a ← max(a, 1e-30)·e^{u − max u}/Σ;
//   strict (EDAA_ESTIMATE_STRICT=1): the reference's explicit residual in its
//     operation order (separate multiply and add, log + exp).
// Both agree with the compiled reference to ≤ 1e-10 for contractive steps
// (η ≤ 1/λ_max(EᵀE)); for larger η the map is chaotic and ANY reordering —
// including the strict kernel's libm — drifts (measured at η = 0.5 on the
// unnormalised cfg3 endmembers: O(1) for both after 100 steps).
template <class XT, bool FAST>
__global__ void k_estimate(const XT* X, const double* E, double* A, int L, int N, int Npad, int p,
                           int iters, double eta) {
  extern __shared__ double es[];  // E [L][p], then G [p][p] (FAST)
  double* gsm = es + L * p;
  for (int e = threadIdx.x; e < L * p; e += blockDim.x) es[e] = E[e];
  __syncthreads();
  if (FAST) {
    for (int e = threadIdx.x; e < p * p; e += blockDim.x) {
      const int i = e / p, m = e % p;
      double s = 0.0;
      for (int l = 0; l < L; ++l) s = fma(es[l * p + i], es[l * p + m], s);
      gsm[e] = s;
    }
    __syncthreads();
  }
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= N) return;
  double a[kMaxP], g[kMaxP];
  for (int i = 0; i < p; ++i) a[i] = 1.0 / static_cast<double>(p);
  if (FAST) {
    double P[kMaxP];
    for (int i = 0; i < p; ++i) P[i] = 0.0;
    for (int l = 0; l < L; ++l) {
      const double x = static_cast<double>(X[static_cast<size_t>(l) * Npad + j]);
      for (int i = 0; i < p; ++i) P[i] = fma(es[l * p + i], x, P[i]);
    }
    for (int it = 0; it < iters; ++it) {
      double top = -INFINITY;
      for (int i = 0; i < p; ++i) {
        double ga = 0.0;
        for (int m = 0; m < p; ++m) ga = fma(gsm[i * p + m], a[m], ga);
        g[i] = (P[i] - ga) * eta;
        top = fmax(top, g[i]);
      }
      double total = 0.0;
      for (int i = 0; i < p; ++i) {
        const double z = (a[i] < kLogFloorValue) ? kLogFloorValue : a[i];
        g[i] = z * exp(g[i] - top);
        total += g[i];
      }
      for (int i = 0; i < p; ++i) a[i] = g[i] / total;
    }
  } else {
    for (int it = 0; it < iters; ++it) {
      for (int i = 0; i < p; ++i) g[i] = 0.0;
      for (int l = 0; l < L; ++l) {
        const double* el = es + l * p;
        double rec = 0.0;
        for (int i = 0; i < p; ++i) rec = __dadd_rn(rec, __dmul_rn(el[i], a[i]));
        const double r = __dsub_rn(static_cast<double>(X[static_cast<size_t>(l) * Npad + j]), rec);
        for (int i = 0; i < p; ++i) g[i] = __dadd_rn(g[i], __dmul_rn(el[i], r));
      }
      double top = -INFINITY;
      for (int i = 0; i < p; ++i) {
        const double z = (a[i] < kLogFloorValue) ? kLogFloorValue : a[i];
        g[i] = __dadd_rn(log(z), __dmul_rn(g[i], eta));  // log z + η·(−∇)
        top = max_like_std(top, g[i]);
      }
      double total = 0.0;
      for (int i = 0; i < p; ++i) {
        g[i] = exp(g[i] - top);
        total = __dadd_rn(total, g[i]);
      }
      for (int i = 0; i < p; ++i) a[i] = g[i] / total;
    }
  }
  for (int i = 0; i < p; ++i) A[static_cast<size_t>(i) * N + j] = a[i];
}

// check_iterate (solver.cpp:65-90) on a row-major d×n matrix, one column per
// thread, entries and the column sum in the reference's order.  The first
// failing check of the reference's column-by-column scan survives the
// atomicMin: key = column·2^36 + entry·4 + kind (entry = 2^34−1 for the sum).
__global__ void k_check_iterate(const double* m, int d, int n, unsigned long long* key) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= n) return;
  double sum = 0.0;
  for (int i = 0; i < d; ++i) {
    const double v = m[static_cast<size_t>(i) * n + j];
    if (!(isfinite(v) && v >= 0.0)) {
      atomicMin(key, (static_cast<unsigned long long>(j) << 36) | (static_cast<unsigned long long>(i) << 2) |
                         (isfinite(v) ? kFailNegative : kFailNonFinite));
      return;
    }
    sum = __dadd_rn(sum, v);
  }
  if (!(fabs(sum - 1.0) <= kSimplexTol))
    atomicMin(key, (static_cast<unsigned long long>(j) << 36) | (((1ull << 34) - 1) << 2) | kFailDrift);
}

inline int blocks_for(size_t n, int threads) {
  return static_cast<int>(std::min<size_t>((n + threads - 1) / threads, 4096));
}

}  // namespace

cudaError_t launch_residual(const void* X, int xbytes, const double* Y, const double* A, double* R,
                            int L, int N, int Npad, int p, cudaStream_t st) {
  const int nb = blocks_for(static_cast<size_t>(L) * Npad, 256);
  if (xbytes == 8)
    k_residual<<<nb, 256, 0, st>>>(static_cast<const double*>(X), Y, A, R, L, N, Npad, p);
  else
    k_residual<<<nb, 256, 0, st>>>(static_cast<const float*>(X), Y, A, R, L, N, Npad, p);
  return cudaGetLastError();
}

cudaError_t launch_reduce(const double* R, size_t total, int mode, double scale, double* part,
                          int nparts, double* out, cudaStream_t st) {
  k_reduce<<<nparts, 256, 0, st>>>(R, total, mode, part);
  k_sum_parts<<<1, 32, 0, st>>>(part, nparts, scale, out);
  return cudaGetLastError();
}

cudaError_t launch_grad_a(const double* Y, const double* R, double* G, int L, int N, int Npad, int p,
                          cudaStream_t st) {
  k_grad_a<<<(N + 127) / 128, 128, 0, st>>>(Y, R, G, L, N, Npad, p);
  return cudaGetLastError();
}

cudaError_t launch_grad_b(const void* X, int xbytes, const double* R, const double* A, double* rat,
                          double* G, int L, int N, int Npad, int p, cudaStream_t st) {
  k_rat<<<(L * p + 127) / 128, 128, 0, st>>>(R, A, rat, L, N, Npad, p);
  if (xbytes == 8)
    k_grad_b<<<(N + 127) / 128, 128, 0, st>>>(static_cast<const double*>(X), rat, G, L, N, Npad, p);
  else
    k_grad_b<<<(N + 127) / 128, 128, 0, st>>>(static_cast<const float*>(X), rat, G, L, N, Npad, p);
  return cudaGetLastError();
}

cudaError_t launch_check_iterate(const double* m, int rows, int cols, unsigned long long* key,
                                 cudaStream_t st) {
  k_check_iterate<<<(cols + 127) / 128, 128, 0, st>>>(m, rows, cols, key);
  return cudaGetLastError();
}

template <class XT>
static cudaError_t launch_estimate_t(const XT* X, const double* E, double* A, int L, int N, int Npad, int p,
                                     int iters, double eta, cudaStream_t st) {
  static const bool strict = [] {
    const char* v = std::getenv("EDAA_ESTIMATE_STRICT");
    return v && v[0] == '1';
  }();
  const size_t smem = (static_cast<size_t>(L) * p + static_cast<size_t>(p) * p) * sizeof(double);
  auto kern = strict ? k_estimate<XT, false> : k_estimate<XT, true>;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, kMaxSmem);
  kern<<<(N + 127) / 128, 128, smem, st>>>(X, E, A, L, N, Npad, p, iters, eta);
  return cudaGetLastError();
}

cudaError_t launch_estimate(const void* X, int xbytes, const double* E, double* A, int L, int N,
                            int Npad, int p, int iters, double eta, cudaStream_t st) {
  return xbytes == 8 ? launch_estimate_t(static_cast<const double*>(X), E, A, L, N, Npad, p, iters, eta, st)
                     : launch_estimate_t(static_cast<const float*>(X), E, A, L, N, Npad, p, iters, eta, st);
}

}  // namespace edaa
