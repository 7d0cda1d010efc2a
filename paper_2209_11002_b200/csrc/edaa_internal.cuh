// Internal declarations shared by the EDAA sm_100a kernels and the C-ABI.
//
// Data layout in HBM (one device, a batch of M runs, p endmembers each):
//   X       fp32 [L][Npad]       band-major, pixels contiguous (BSQ plane order,
//                                reference layout L×N, envi.cpp:160-174); zero
//                                padded to Npad = ceil(N/64)·64.
//   xnorm   fp64 [Npad]          ‖x_j‖² (fp64 sum of the fp32 values).
//   A       fp64 [M][p][Npad]    abundances, run-major then endmember (rows of
//                                the reference p×N matrix, solver.hpp:29-38).
//   Lg      fp64 [M][p][Npad]    contribution LOGITS ℓ; B = softmax over
//                                pixels: b_j = exp(ℓ_j − m)/S with the column
//                                normaliser (m, S) kept in colm/colS.
//   Columns of the batch live in a chunk-padded space of Qs = NCH·QCpad slots:
//   chunk k holds runs [k·RC, k·RC+RC), run-local column i at k·QCpad+rl·p+i.
//   Y, Z, XAt  fp64 [Lpad][Qs]   Y = X·B, Z = XAᵀ − Y·AAᵀ, XAt = X·Aᵀ.
//   AAt, G     fp64 [QCpad][Qs]  per-run p×p blocks on the chunk diagonal.
#pragma once
#include <cstddef>
#include <cstdint>
#include <cstdlib>
#include <cuda_runtime.h>

#ifndef EDAA_QMAX
#define EDAA_QMAX 24
#endif

namespace edaa {

constexpr int kThreads = 512;   // 16 warps per CTA: 8 MMA warps + 8 update warps
constexpr int kGroup = 256;     // threads per warp group
constexpr int kNP = 32;         // pixels per tile (one X ring slot)
constexpr int kNPad = 64;       // Npad granularity: an even number of tiles, so 64-pixel logical tiles never straddle a slice
constexpr int kXST = kNP + 8;   // fp32 X tile row stride (conflict-free DMMA B-frags)
constexpr int kSST = kNP + 4;   // fp64 weight tile row stride
constexpr int kQMax = EDAA_QMAX;  // columns per chunk (kQMax/8 DMMA column tiles)
constexpr int kMaxCT = kQMax / 8;
constexpr int kMaxSlices = 148; // bounds the slice-partial traffic (nslices·(L+24)·Q doubles per pass)
constexpr int kTilesPerSlice = 4;  // 128-pixel slices: ~5 (slice, chunk) items per CTA at cfg1
constexpr int kSmallTilesPerSlice = 2;  // images of at most 2·kMaxSlices tiles: 64-pixel slices
// Pixel slices of an image of `ntiles` 32-pixel tiles: a function of N ONLY (a run's
// partial sums, and so its bits, must not depend on the batch it is solved in).
// Small images (≤ 9,472 pixels) take 2-tile slices — twice the work items, so the
// passes fill more SMs and balance better: measured +9.5% on a single cfg0 run,
// +2.5–13% on batches of 20–50 runs at N = 2,500–9,025; cfg1 (313 tiles) is
// 10% slower with them (twice the slice partials), so larger images keep 4.
// First 32-pixel tile of slice s: slices are made of 64-pixel tile PAIRS (ntiles is even).
__host__ __device__ inline int slice_first_tile(int ntiles, int nslices, int s) {
  return 2 * static_cast<int>((static_cast<long long>(s) * (ntiles / 2)) / nslices);
}
inline int slice_count(int ntiles) {
  const int tps = ntiles <= 2 * kMaxSlices ? kSmallTilesPerSlice : kTilesPerSlice;
  const int n = (ntiles + tps - 1) / tps;
  return n < kMaxSlices ? n : kMaxSlices;
}
constexpr int kMaxP = 16;
constexpr int kMaxLpad = 320;
constexpr double kLogFloorValue = 1e-30;  // solver.cpp:15

enum PassMode : int { kModeInit = 0, kModeA = 1, kModeB = 2, kModeObj = 3 };

// Failure codes per run (map to the reference's archetype::Error messages).
enum FailCode : int {
  kOk = 0,
  kNonFiniteA = 1,       // "non-finite abundance iterate at outer iteration t"  solver.cpp:74
  kNonFiniteB = 2,       // "non-finite contribution iterate at outer iteration t"
  kDegenerateInit = 3,   // "degenerate initialization: X·B0 is zero"  solver.cpp:141
  kSpectralBad = 4,      // "spectral_norm: matrix must be finite and nonzero"  matrix.cpp:151
  kSpectralNoConv = 5,   // "spectral_norm: no convergence after ..."  matrix.cpp:186-189
  kSimplexA = 6,         // "abundance iterate left the simplex at outer iteration t"  solver.cpp:77-81
  kSimplexB = 7,         // "contribution iterate left the simplex ..."
  kDriftA = 8,           // "abundance column sum drifted from 1 at outer iteration t"  solver.cpp:84-88
  kDriftB = 9,           // "contribution column sum drifted from 1 ..."
};

// Per-run failure key of check_iterate (solver.cpp:65-90): the reference stops
// at the FIRST failing check of its scan (outer t, block A then B, inner step k,
// column, then per entry: finite, >= 0; then the column sum).  Every device
// check posts its position with atomicMin, so the surviving key is that first
// failure:  [t<<1|block : 23][k : 6][position : 33][kind : 2].
// Position: A block = pixel·32 + entry (31 = the column-sum check);
//           B block = endmember·2^28 + pixel (2^28−1 = the column-sum check).
enum FailKind : unsigned { kFailNonFinite = 0, kFailNegative = 1, kFailDrift = 2 };
constexpr double kSimplexTol = 1e-9;  // solver.cpp:84
__host__ __device__ inline unsigned long long fail_key_make(unsigned tb, unsigned k, unsigned long long pos,
                                                            unsigned kind) {
  return (static_cast<unsigned long long>(tb) << 41) | (static_cast<unsigned long long>(k < 63u ? k : 63u) << 35) |
         ((pos & ((1ull << 33) - 1)) << 2) | kind;
}
inline unsigned fail_key_tb(unsigned long long key) { return static_cast<unsigned>(key >> 41); }
inline unsigned fail_key_kind(unsigned long long key) { return static_cast<unsigned>(key & 3ull); }

struct Dims {
  int L, Lpad, N, Npad;
  int ntiles, nslices;
  int M, p, RC, QCpad, NCH, Qs;
  int Lrows;  // Lpad + QCpad (A-pass pseudo rows carry AAᵀ)
  int K1;
  int nbuf;   // X tile buffers in shared memory (2 = prefetch next tile)
  int nwb;    // W chunk buffers: 2 = next chunk prefetched, 1 = restaged in place
  int xbytes; // 4: fp32 image, 8: fp64 image (inputs not exactly representable in fp32)
  int ncta;   // persistent pass CTAs (one per SM)
  int sl0, sl1;  // pixel slices this device owns (pixel sharding; 0..nslices otherwise)
  int pdl;       // programmatic dependent launch for the schedule's kernels (small grids only)
  int cmajor;    // pass item order: 1 chunk-major (X fits in L2), 0 slice-major (edaa_pass.cuh)
  int ilv;       // slice-major items interleaved over the CTAs (A/B passes, separate instantiation)
  int npl;       // B pass: 2 = the 64-pixel logical-tile kernel (edaa_pass_b64.cu), 1 = k_pass
  int nbuf64;    // its X ring (32-pixel slots)
};

struct PassArgs {
  Dims d;
  int t;  // outer iteration (1-based); 0 for init
  const void* X;          // float or double [L][Npad] (Dims::xbytes)
  const double* xnorm;
  const double* W;        // Y (A/OBJ pass) or Z (B pass), [Lpad][Qs]
  double* A;              // [M][p][Npad]
  double* Lg;             // [M][p][Npad]
  const double* colm;     // [Qs] normaliser max of the current logits
  const double* collogS;  // [Qs] log of the normaliser sum
  const double* Gbuf;     // [QCpad][Qs]
  const double* eta_a;    // [M]
  const double* eta_b;    // [M]
  const uint64_t* seeds;  // [M]
  double* part_C;         // [nslices][Lrows][Qs]
  double* part_m;         // [nslices][Qs]
  double* part_S;         // [nslices][Qs]
  double* part_obj;       // [nslices][M]
  unsigned long long* fail_key;  // [M]  min over fail_key_make(...)
  double* observe_A;      // optional [K1][p][Npad] inner iterates (M == 1 observed mode)
  unsigned long long* kprof;  // optional cycle accounting (development)
  int dbg;                    // development switches (EDAA_DBG): 1 no DMMA, 2 no B update
  const void* xmap;           // host pointer to the CUtensorMap of X (passed by value at launch)
};

struct CombineArgs {
  Dims d;
  int t;
  int kin;   // inner B step (orders failures of one outer iteration; 0 otherwise)
  int mode;  // kModeA: plain sums (XAt, AAt, objective); kModeB/kModeInit: LSE combine into Y
  const double* part_C;
  const double* part_m;
  const double* part_S;
  const double* part_obj;
  double* Y;        // B/init output
  double* colm;
  double* colS;
  double* collogS;
  double* fac;      // [nslices][Qs] scratch: exp(m_s − m) per slice and column
  double* XAt;      // A output
  double* AAt;      // A output [QCpad][Qs] (run-diagonal p×p blocks)
  double* Z;        // A/B output: Z = XAᵀ − Y·AAᵀ (nullptr: not formed, init)
  double* trace;    // [M][T+1]
  int trace_stride;
  int trace_index;
  unsigned long long* fail_key;
};

enum PostMode : int { kPostZ = 0, kPostG = 1, kPostInit = 2 };

struct PostArgs {
  Dims d;
  int mode;
  const double* Y;
  const double* XAt;
  const double* AAt;
  double* Z;
  double* Gbuf;
  const double* gamma;  // [M]
  double* eta_a;
  double* eta_b;
  int* fail_code;       // [M]
  double* fail_value;   // [M]
};

// Launch with programmatic stream serialization (see griddep_wait in edaa_device.cuh)
// when `pdl`: the solve enables it only when the pass grid leaves SMs idle (small
// images), where hiding launch latency pays; measured slower for full-grid passes
// (cfg1: +2%), faster for cfg0 (-6%).  EDAA_NO_PDL=1 disables it everywhere.
inline bool pdl_enabled() {
  static const bool on = [] {
    const char* v = std::getenv("EDAA_NO_PDL");
    return !(v && v[0] == '1');
  }();
  return on;
}
template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl(bool pdl, void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                              Args... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = (pdl && pdl_enabled()) ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kern, static_cast<KArgs>(args)...);
}

// Kernel launchers (edaa_kernels.cu). All enqueue on `st`; none synchronise.
cudaError_t launch_pass(int mode, const PassArgs& a, cudaStream_t st);
cudaError_t launch_combine(const CombineArgs& a, cudaStream_t st);
cudaError_t launch_post(const PostArgs& a, cudaStream_t st);
cudaError_t launch_xnorm(const void* X, double* xnorm, const Dims& d, cudaStream_t st);
cudaError_t launch_materialize_b(const double* Lg, const double* colm, const double* colS,
                                 double* Bv, const Dims& d, cudaStream_t st);
cudaError_t launch_strict_e(const void* X, const double* Bv, double* E, const Dims& d,
                            cudaStream_t st);
cudaError_t launch_fit(const void* X, const double* E, const double* A, double* part_fit,
                       double* fit, int fit_blocks, const Dims& d, cudaStream_t st);
cudaError_t launch_coherence(const double* E, double* mu, const Dims& d, cudaStream_t st);
cudaError_t launch_select(const double* fit, const double* mu, const int* fail_code,
                          const unsigned long long* fail_key, int M, double slack,
                          unsigned char* cand, long long* selected, double* fit_min,
                          cudaStream_t st);
// pixel sharding, allreduce exchange (edaa_kernels.cu): the rank-local block of one pass
size_t shard_red_doubles(const Dims& d);       // whole block
size_t shard_red_sum_doubles(const Dims& d);   // its sum-reduced prefix (C | S | obj)
size_t shard_red_off(const Dims& d, int what); // 0 C, 1 S, 2 obj, 3 m (rank), 4 m (global)
cudaError_t launch_shard_reduce(const CombineArgs& a, int s0, int s1, double* red, cudaStream_t st);
cudaError_t launch_shard_rescale(const Dims& d, double* red, const double* m_glob, cudaStream_t st);
cudaError_t launch_shard_emul_max(const Dims& d, double* red, size_t stride, int world, cudaStream_t st);
cudaError_t launch_shard_emul_sum(double* red, size_t stride, int world, size_t n, cudaStream_t st);
cudaError_t launch_pack_cols(const double* src, double* stage, int rows, int Npad, int j0, int w, int wmax,
                             bool unpack, double* dst, cudaStream_t st);
size_t pass_smem_bytes(const Dims& d, int nbuf);
size_t pass_b64_smem_bytes(const Dims& d, int nbuf);
cudaError_t launch_pass_b64(const PassArgs& a, cudaStream_t st);
// primitives (edaa_prims.cu)
cudaError_t launch_residual(const void* X, int xbytes, const double* Y, const double* A, double* R,
                            int L, int N, int Npad, int p, cudaStream_t st);
cudaError_t launch_reduce(const double* R, size_t total, int mode, double scale, double* part,
                          int nparts, double* out, cudaStream_t st);
cudaError_t launch_grad_a(const double* Y, const double* R, double* G, int L, int N, int Npad, int p,
                          cudaStream_t st);
cudaError_t launch_grad_b(const void* X, int xbytes, const double* R, const double* A, double* rat,
                          double* G, int L, int N, int Npad, int p, cudaStream_t st);
cudaError_t launch_check_iterate(const double* m, int rows, int cols, unsigned long long* key,
                                 cudaStream_t st);
cudaError_t launch_estimate(const void* X, int xbytes, const double* E, double* A, int L, int N,
                            int Npad, int p, int iters, double eta, cudaStream_t st);
constexpr int kMaxSmem = 232448;  // sm_100 opt-in dynamic shared memory per block

}  // namespace edaa
