// C-ABI (include/edaa_b200.h): device context, buffer management and the
// per-solve launch schedule of the batched EDAA solver.
//
// Launch schedule of one solve (M runs batched, all on one stream):
//   init pass (B⁰ logits from SplitMix64, Y⁰ = X·B⁰)  → combine → post(init: G, η)
//   for t = 1..T:
//     A pass (trace[t-1], K1 steps, XAᵀ, AAᵀ)          → combine → post(Z)
//     for k = 1..K2:
//       B pass (g = XᵀZ, logits, online max, Y_{k+1})   → combine → post(Z or G)
//   objective pass (trace[T]) → combine; materialise B; E = X·B (reference
//   order); fit_l1; coherence.
#include <algorithm>
#include <atomic>
#include <cstdlib>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <string>
#include <type_traits>
#include <vector>

#include <cuda.h>
#include <dlfcn.h>
#include <nccl.h>
#include <nvtx3/nvToolsExt.h>  // header-only NVTX 3: ranges per solve phase (visible to nsys / ncu --nvtx)

#include "../../include/edaa_b200.h"
#include "edaa_device.cuh"

using edaa::Dims;

namespace {
// NVTX range of one schedule phase ("edaa/solve", "edaa/init", "edaa/A t=3", …): marks
// the host enqueue (and, outside a captured graph, brackets the phase's launches).
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  NvtxRange(const char* what, size_t t) {
    char buf[48];
    std::snprintf(buf, sizeof buf, "edaa/%s t=%zu", what, t);
    nvtxRangePushA(buf);
  }
  ~NvtxRange() { nvtxRangePop(); }
  NvtxRange(const NvtxRange&) = delete;
  NvtxRange& operator=(const NvtxRange&) = delete;
};
}  // namespace

struct GraphKey {
  Dims d;
  size_t T, K2;
  uint64_t gen;
  const void* comm;
  int emulate;
};

struct edaa_ctx {
  int device = 0;
  cudaStream_t stream = nullptr;
  std::string err;
  // image
  void* X = nullptr;  // float or double [L][Npad]
  int xbytes = 4;
  double* xnorm = nullptr;
  int L = 0, N = 0, Npad = 0;
  size_t x_cap = 0, xn_cap = 0;
  // solve state
  bool solved = false;
  Dims d{};
  size_t T = 0;
  struct Buf {
    void* p = nullptr;
    size_t cap = 0;
  };
  Buf A, Lg, Bv, Y, Z, XAt, AAt, Gbuf, colm, colS, collogS, eta_a, eta_b, gamma, trace, part_C,
      part_m, part_S, part_obj, fac, E, fit, mu, part_fit, seeds, fail_key, fail_code, fail_value, cand,
      selected, fit_min, obsA, pr_b, pr_a, pr_y, pr_r, pr_g, pr_rat, pr_part, pr_out, in_raw, in_x,
      in_flags, in_bad, shard_red, shard_stage;
  int fit_blocks = 0;
  // instrumentation
  bool profile = false;
  std::vector<cudaEvent_t> ev_pool;
  std::vector<int> ev_kind;
  size_t ev_used = 0;
  edaa_profile last_prof{};
  uint64_t launches = 0;
  void* kprof_buf = nullptr;  // EDAA_KPROF=1: per-phase cycle counters (dev only)
  int dbg = 0;                // EDAA_DBG: development switches, results invalid when set
  int num_sms = 148;
  alignas(64) CUtensorMap xmap;  // TMA descriptor of X for the current solve
  // CUDA graph of the last solve's device schedule and what it was captured for
  bool no_graph = false;
  uint64_t gen = 0;  // bumped whenever a device buffer or the image moves
  uint64_t image_gen = 0;
  cudaGraphExec_t graph_exec = nullptr;
  GraphKey graph_key{};
  uint64_t graph_launches = 0;
  // host copies of the per-run records
  std::vector<double> h_fit, h_mu, h_eta_a, h_eta_b, h_fail_value, h_trace;
  std::vector<int> h_fail_code;
  std::vector<unsigned long long> h_fail_key;
  // pixel sharding of one solve over the GPUs of a node (NCCL communicator; world 1 = off)
  ncclComm_t comm = nullptr;
  int shard_rank = 0, shard_world = 1;
  int shard_emulate = 0;  // > 1: run the slice ranges of that many ranks one after another here
  int shard_exchange = 0; // 0: allreduce of the rank-reduced L×Q / Q×Q / 2Q blocks; 1: broadcast of every slice partial (bitwise)
  int pass_order = 0;     // pass item order: 0 auto, 1 chunk-major, 2 slice-major (edaa_set_pass_order)
};

namespace {

int set_err(edaa_ctx* c, int code, const std::string& msg) {
  if (c) c->err = msg;
  return code;
}

int cuda_fail(edaa_ctx* c, cudaError_t e, const char* what) {
  return set_err(c, EDAA_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

#define EDAA_CUDA(ctx, call)                                   \
  do {                                                         \
    cudaError_t e_ = (call);                                   \
    if (e_ != cudaSuccess) return cuda_fail((ctx), e_, #call); \
  } while (0)

std::atomic<uint64_t> g_realloc_count{0};  // any device (re)allocation invalidates captured graphs (contexts on several host threads)

cudaError_t ensure(edaa_ctx::Buf& b, size_t bytes) {
  if (b.cap >= bytes && b.p) return cudaSuccess;
  ++g_realloc_count;
  if (b.p) cudaFree(b.p);
  b.p = nullptr;
  b.cap = 0;
  cudaError_t e = cudaMalloc(&b.p, std::max<size_t>(bytes, 16));
  if (e == cudaSuccess) b.cap = std::max<size_t>(bytes, 16);
  return e;
}

template <class T>
T* P(edaa_ctx::Buf& b) {
  return static_cast<T*>(b.p);
}

__global__ void k_fill_a(double* A, int M, int p, int N, int Npad) {
  const size_t total = static_cast<size_t>(M) * p * Npad;
  const double v = 1.0 / static_cast<double>(p);  // init_abundances, solver.cpp:113-116
  for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<size_t>(gridDim.x) * blockDim.x) {
    const int j = static_cast<int>(i % Npad);
    A[i] = (j < N) ? v : 0.0;
  }
}

template <class XT>
__global__ void k_pad_copy(const XT* src, size_t ld, XT* dst, int L, int N, int Npad) {
  const size_t total = static_cast<size_t>(L) * Npad;
  for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<size_t>(gridDim.x) * blockDim.x) {
    const int l = static_cast<int>(i / Npad), j = static_cast<int>(i % Npad);
    dst[i] = (j < N) ? src[static_cast<size_t>(l) * ld + j] : XT(0);
  }
}

// Device ingest (HsiImage::validate + l2_normalize, image.cpp:10-47): one thread
// per pixel.  Validation records the first offending element in the
// reference's scan order (row-major, i·N + j) per kind; the norm is
// Matrix::column_norm (matrix.cpp:44-51: s += v·v band-ascending, no fused
// multiply-add, sqrt) and every element of a nonzero pixel is divided by it, so
// the result is bitwise the reference's.  Zero pixels are flagged and left as
// they are; `inexact` is raised if any normalised value is not representable in
// fp32 (then the solve keeps the fp64 image).
// Source element (band i, pixel j) of the raw image: band-major L×N (BSQ, the
// HsiImage layout) or pixel-major N×L (an (H, W, L) NPY cube, npy.cpp:186-207,
// whose npy_to_image transpose is thereby done here). fp32 sources widen
// exactly, so every later step sees the reference's fp64 values.
template <class T, bool PIXEL_MAJOR>
__device__ __forceinline__ double raw_at(const T* raw, int L, int N, int i, int j) {
  return static_cast<double>(PIXEL_MAJOR ? raw[static_cast<size_t>(j) * L + i] : raw[static_cast<size_t>(i) * N + j]);
}

template <class T, bool PIXEL_MAJOR>
__global__ void k_ingest(const T* raw, double* xn, int L, int N, int Npad, unsigned long long* bad,
                         unsigned char* zero, unsigned int* inexact) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= Npad) return;
  if (j >= N) {
    for (int i = 0; i < L; ++i) xn[static_cast<size_t>(i) * Npad + j] = 0.0;
    return;
  }
  double s = 0.0;
  for (int i = 0; i < L; ++i) {
    const double v = raw_at<T, PIXEL_MAJOR>(raw, L, N, i, j);
    const unsigned long long idx = static_cast<unsigned long long>(i) * N + j;
    if (!isfinite(v))
      atomicMin(bad + 0, idx);
    else if (v < 0.0)
      atomicMin(bad + 1, idx);
    s = __dadd_rn(s, __dmul_rn(v, v));
  }
  const double norm = sqrt(s);
  const bool z = (norm == 0.0);
  zero[j] = z ? 1 : 0;
  bool exact = true;
  for (int i = 0; i < L; ++i) {
    const double v = raw_at<T, PIXEL_MAJOR>(raw, L, N, i, j);
    const double o = z ? v : __ddiv_rn(v, norm);
    xn[static_cast<size_t>(i) * Npad + j] = o;
    exact &= (static_cast<double>(static_cast<float>(o)) == o);
  }
  if (!exact) atomicOr(inexact, 1u);
}

// HsiImage::validate (image.cpp:10-27) of an uploaded fp32 image on the device:
// the first non-finite and the first negative element in the reference's
// row-major L×N scan order (atomicMin of the flat index; clean images issue no
// atomics).  Padding columns j ≥ N are skipped.
__global__ void k_check_f32(const float* X, int L, int N, int Npad, unsigned long long* bad) {
  const size_t total = static_cast<size_t>(L) * Npad;
  for (size_t e = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; e < total;
       e += static_cast<size_t>(gridDim.x) * blockDim.x) {
    const int i = static_cast<int>(e / Npad), j = static_cast<int>(e - static_cast<size_t>(i) * Npad);
    if (j >= N) continue;
    const float v = X[e];
    if (!isfinite(v))
      atomicMin(bad + 0, static_cast<unsigned long long>(i) * N + j);
    else if (v < 0.0f)
      atomicMin(bad + 1, static_cast<unsigned long long>(i) * N + j);
  }
}

__global__ void k_to_f32(const double* src, float* dst, size_t n) {
  for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<size_t>(gridDim.x) * blockDim.x)
    dst[i] = static_cast<float>(src[i]);
}

// Register-resident DMMA loop: 4 independent accumulators per lane.
__global__ void k_dmma_peak(double* out, int iters) {
  double a = threadIdx.x * 1e-3, b = 1.0 + threadIdx.x * 1e-4;
  double c[4][2];
  for (int i = 0; i < 4; ++i) c[i][0] = c[i][1] = i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 4; ++i)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(c[i][0]), "+d"(c[i][1])
                   : "d"(a), "d"(b));
  }
  double s = 0.0;
  for (int i = 0; i < 4; ++i) s += c[i][0] + c[i][1];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

// check_iterate's failure (solver.cpp:65-90) from a device fail key.
int fail_key_code(unsigned long long key, size_t* outer) {
  const unsigned tb = edaa::fail_key_tb(key);
  *outer = tb >> 1;
  const bool b = tb & 1u;
  switch (edaa::fail_key_kind(key)) {
    case edaa::kFailNonFinite: return b ? EDAA_RUN_NONFINITE_B : EDAA_RUN_NONFINITE_A;
    case edaa::kFailNegative: return b ? EDAA_RUN_SIMPLEX_B : EDAA_RUN_SIMPLEX_A;
    default: return b ? EDAA_RUN_DRIFT_B : EDAA_RUN_DRIFT_A;
  }
}

std::string run_message(int code, size_t outer, double value) {
  char buf[192];
  switch (code) {
    case EDAA_RUN_NONFINITE_A:
      std::snprintf(buf, sizeof buf, "non-finite abundance iterate at outer iteration %zu", outer);
      return buf;
    case EDAA_RUN_NONFINITE_B:
      std::snprintf(buf, sizeof buf, "non-finite contribution iterate at outer iteration %zu", outer);
      return buf;
    case EDAA_RUN_SIMPLEX_A:
      std::snprintf(buf, sizeof buf, "abundance iterate left the simplex at outer iteration %zu", outer);
      return buf;
    case EDAA_RUN_SIMPLEX_B:
      std::snprintf(buf, sizeof buf, "contribution iterate left the simplex at outer iteration %zu", outer);
      return buf;
    case EDAA_RUN_DRIFT_A:
      std::snprintf(buf, sizeof buf, "abundance column sum drifted from 1 at outer iteration %zu", outer);
      return buf;
    case EDAA_RUN_DRIFT_B:
      std::snprintf(buf, sizeof buf, "contribution column sum drifted from 1 at outer iteration %zu", outer);
      return buf;
    case EDAA_RUN_DEGENERATE:
      return "degenerate initialization: X\xc2\xb7" "B0 is zero";
    case EDAA_RUN_SPECTRAL_BAD:
      return "spectral_norm: matrix must be finite and nonzero";
    case EDAA_RUN_SPECTRAL_NOCONV:
      std::snprintf(buf, sizeof buf,
                    "spectral_norm: no convergence after 1000 iterations; best estimate %g", value);
      return buf;
    default:
      return "";
  }
}

// ---- NCCL, resolved at run time (libnccl.so.2: the one already loaded into the
// process, e.g. by torch, else the system copy) so the library links without it.
struct NcclApi {
  bool ok = false;
  std::string why;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*Broadcast)(const void*, void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

const NcclApi& nccl() {
  static NcclApi api = [] {
    NcclApi a;
    // EDAA_NCCL_LIB, else the copy already in the process (a host that loads its own
    // NCCL — torch — must do so first: a later load by soname would bind to ours).
    void* h = nullptr;
    if (const char* path = std::getenv("EDAA_NCCL_LIB")) h = dlopen(path, RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL | RTLD_NOLOAD);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
      a.why = "libnccl.so.2 not found";
      return a;
    }
    bool all = true;
    auto sym = [&](auto& fn, const char* name) {
      fn = reinterpret_cast<std::remove_reference_t<decltype(fn)>>(dlsym(h, name));
      all &= fn != nullptr;
    };
    sym(a.GetUniqueId, "ncclGetUniqueId");
    sym(a.CommInitRank, "ncclCommInitRank");
    sym(a.CommDestroy, "ncclCommDestroy");
    sym(a.Broadcast, "ncclBroadcast");
    sym(a.AllReduce, "ncclAllReduce");
    sym(a.AllGather, "ncclAllGather");
    sym(a.GroupStart, "ncclGroupStart");
    sym(a.GroupEnd, "ncclGroupEnd");
    sym(a.GetErrorString, "ncclGetErrorString");
    a.ok = all;
    if (!all) a.why = "libnccl.so.2 lacks a required symbol";
    return a;
  }();
  return api;
}

#define EDAA_NCCL(ctx, call)                                                                     \
  do {                                                                                           \
    ncclResult_t r_ = (call);                                                                    \
    if (r_ != ncclSuccess)                                                                       \
      return set_err((ctx), EDAA_ERR_CUDA, std::string(#call ": ") + nccl().GetErrorString(r_)); \
  } while (0)

// Slice range [sl0, sl1) of `rank` among `world` (slice boundaries depend on N only).
void shard_slices(const Dims& d, int rank, int world, int* sl0, int* sl1) {
  *sl0 = static_cast<int>((static_cast<long long>(rank) * d.nslices) / world);
  *sl1 = static_cast<int>((static_cast<long long>(rank + 1) * d.nslices) / world);
}
// Pixel range of a slice range (tile-aligned; the last slice ends at Npad).
void slice_pixels(const Dims& d, int sl0, int sl1, int* j0, int* j1) {
  *j0 = edaa::slice_first_tile(d.ntiles, d.nslices, sl0) * edaa::kNP;
  *j1 = edaa::slice_first_tile(d.ntiles, d.nslices, sl1) * edaa::kNP;
}

int make_dims(edaa_ctx* c, const edaa_solve_params* prm, Dims* out) {
  if (!prm || !prm->seeds || !prm->gammas) return set_err(c, EDAA_ERR_INVALID, "null params");
  if (c->X == nullptr) return set_err(c, EDAA_ERR_STATE, "no image set");
  const size_t p = prm->endmembers;
  if (p < 2) return set_err(c, EDAA_ERR_INVALID, "solver config: endmember count must be at least 2");
  if (prm->outer_iters < 1 || prm->inner_iters_a < 1 || prm->inner_iters_b < 1)
    return set_err(c, EDAA_ERR_INVALID, "solver config: iteration counts must be at least 1");
  if (prm->runs < 1) return set_err(c, EDAA_ERR_INVALID, "ensemble needs at least one run");
  if (p > static_cast<size_t>(edaa::kMaxP))
    return set_err(c, EDAA_ERR_UNSUPPORTED, "endmember count above the compiled maximum (16)");
  for (size_t r = 0; r < prm->runs; ++r)
    if (!(prm->gammas[r] > 0.0) || !std::isfinite(prm->gammas[r]))
      return set_err(c, EDAA_ERR_INVALID, "solver config: step factor gamma must be positive");
  Dims d{};
  d.L = c->L;
  d.xbytes = c->xbytes;
  d.Lpad = (c->L + 7) / 8 * 8;
  if (d.Lpad > edaa::kMaxLpad)
    return set_err(c, EDAA_ERR_UNSUPPORTED, "band count above the compiled maximum (320)");
  d.N = c->N;
  d.Npad = c->Npad;
  d.ntiles = d.Npad / edaa::kNP;
  d.nslices = edaa::slice_count(d.ntiles);
  d.sl0 = 0;
  d.sl1 = d.nslices;
  if (c->shard_world > 1) {
    if (d.nslices < c->shard_world)
      return set_err(c, EDAA_ERR_UNSUPPORTED, "image too small to shard its pixels over that many devices");
    shard_slices(d, c->shard_rank, c->shard_world, &d.sl0, &d.sl1);
  }
  d.M = static_cast<int>(prm->runs);
  d.p = static_cast<int>(p);
  d.RC = std::max(1, std::min(edaa::kQMax / d.p, d.M));
  d.QCpad = edaa::kQMax;  // fixed 3 DMMA column tiles: unpredicated tensor-core code
  d.NCH = (d.M + d.RC - 1) / d.RC;
  d.Qs = d.NCH * d.QCpad;
  d.Lrows = d.Lpad + d.QCpad;
  d.K1 = static_cast<int>(prm->inner_iters_a);
  d.ncta = c->num_sms;
  d.pdl = (d.NCH * (d.sl1 - d.sl0) < c->num_sms) ? 1 : 0;
  // Chunk-major pass items when X is comfortably L2-resident (126 MB L2 on B200,
  // shared with the slice partials), unless edaa_set_pass_order picks one.
  // Larger images: slice-major. Interleaved over the CTAs (A/B passes, when
  // every CTA gets the same number of items) only on request (order 3): it cuts
  // the cfg4 B pass's HBM reads 24.98 → 5.39 GB but runs 0.5% slower there.
  const bool even = (d.NCH * (d.sl1 - d.sl0)) % d.ncta == 0;
  if (c->pass_order >= 1 && c->pass_order <= 3)
    d.cmajor = (c->pass_order == 1) ? 1 : 0;
  else
    d.cmajor = (static_cast<size_t>(d.Lpad) * d.Npad * d.xbytes <= (size_t(96) << 20)) ? 1 : 0;
  // Images larger than L2 (slice-major): interleave the items over the CTAs whenever
  // they divide evenly, so every X slice comes from HBM once per pass and then from
  // L2 (cfg4 B pass: 9.8 GB of DRAM traffic instead of 29.4 GB at the same speed,
  // DESIGN §7); order 2 forces plain slice-major.
  d.ilv = (d.cmajor == 0 && even && (c->pass_order == 3 || c->pass_order == 0)) ? 1 : 0;
  // X ring depth and W chunk buffers, the deepest that fits shared memory.
  static const int kRing[][2] = {{4, 2}, {3, 2}, {3, 1}, {2, 2}, {2, 1}};
  for (const auto& rw : kRing) {
    d.nbuf = rw[0];
    d.nwb = rw[1];
    if (edaa::pass_smem_bytes(d, d.nbuf) <= static_cast<size_t>(edaa::kMaxSmem)) break;
  }
  if (edaa::pass_smem_bytes(d, d.nbuf) > static_cast<size_t>(edaa::kMaxSmem))
    return set_err(c, EDAA_ERR_UNSUPPORTED, "tile working set exceeds shared memory");
  // B pass with 64-pixel logical tiles (fp32 image) when its working set fits: 5 X slots, one W
  // buffer, the S tiles.  A function of (L, p, image type) only.  EDAA_NO_B64=1 keeps k_pass.
  d.npl = 1;
  d.nbuf64 = 0;
  static const bool no_b64 = [] {
    const char* v = std::getenv("EDAA_NO_B64");
    return v && v[0] == '1';
  }();
  if (!no_b64 && d.xbytes == 4 && (c->dbg & ~258) == 0 &&  // it honours EDAA_DBG bits 2 and 256 only
      edaa::pass_b64_smem_bytes(d, 5) <= static_cast<size_t>(edaa::kMaxSmem)) {
    d.npl = 2;
    d.nbuf64 = 5;
  }
  *out = d;
  return EDAA_OK;
}

// TMA descriptor of X: 2-D [L][Npad] (inner dimension = pixels), boxes of 128 bytes
// × x_box_rows rows with 128-byte swizzle; rows ≥ L read as zeros.
using EncodeTiledFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                   const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                   CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int make_xmap(edaa_ctx* c, const Dims& d) {
  static EncodeTiledFn encode = nullptr;
  if (!encode) {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess || !fn)
      return set_err(c, EDAA_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
    encode = reinterpret_cast<EncodeTiledFn>(fn);
  }
  const int esz = d.xbytes;
  const cuuint64_t dims[2] = {static_cast<cuuint64_t>(d.Npad), static_cast<cuuint64_t>(d.L)};
  const cuuint64_t strides[1] = {static_cast<cuuint64_t>(d.Npad) * esz};
  const cuuint32_t box[2] = {static_cast<cuuint32_t>(128 / esz), static_cast<cuuint32_t>(edaa::dev::x_box_rows(d))};
  const cuuint32_t estr[2] = {1, 1};
  const CUresult r = encode(&c->xmap, esz == 8 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT64 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2,
                            c->X, dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                            CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return set_err(c, EDAA_ERR_CUDA, "cuTensorMapEncodeTiled failed (" + std::to_string(r) + ")");
  return EDAA_OK;
}

// Staging plan of the final state exchange: widest pixel range of a rank, rows per all-gather.
void state_stage_plan(const edaa_ctx* c, const Dims& d, int* wmax, int* rblk) {
  const int W = c->shard_world;
  int w = 1;
  for (int q = 0; q < W; ++q) {
    int a = 0, b = 0, j0 = 0, j1 = 0;
    shard_slices(d, q, W, &a, &b);
    slice_pixels(d, a, b, &j0, &j1);
    w = std::max(w, j1 - j0);
  }
  const size_t cap = size_t(32) << 20;  // doubles of receive staging (256 MB)
  *wmax = w;
  *rblk = static_cast<int>(std::max<size_t>(1, std::min<size_t>(static_cast<size_t>(d.M) * d.p,
                                                                 cap / (static_cast<size_t>(W) * w))));
}

int alloc_solve(edaa_ctx* c, const Dims& d, size_t T) {
  if (c->comm || c->shard_emulate > 1)
    EDAA_CUDA(c, ensure(c->shard_red, edaa::shard_red_doubles(d) * std::max(1, c->shard_emulate) * 8));
  if (c->comm) {
    int wmax = 0, rblk = 0;
    state_stage_plan(c, d, &wmax, &rblk);
    EDAA_CUDA(c, ensure(c->shard_stage, static_cast<size_t>(rblk) * wmax * (c->shard_world + 1) * 8));
  }
  const size_t mpn = static_cast<size_t>(d.M) * d.p * d.Npad * 8;
  const size_t lq = static_cast<size_t>(d.Lpad) * d.Qs * 8;
  const size_t qq = static_cast<size_t>(d.QCpad) * d.Qs * 8;
  const size_t S = d.nslices;
  c->fit_blocks = std::max(1, std::min(64, (d.N + 255) / 256));
  EDAA_CUDA(c, ensure(c->A, mpn));
  EDAA_CUDA(c, ensure(c->Lg, mpn));
  EDAA_CUDA(c, ensure(c->Bv, mpn));
  EDAA_CUDA(c, ensure(c->Y, lq));
  EDAA_CUDA(c, ensure(c->Z, lq));
  EDAA_CUDA(c, ensure(c->XAt, lq));
  EDAA_CUDA(c, ensure(c->AAt, qq));
  EDAA_CUDA(c, ensure(c->Gbuf, qq));
  EDAA_CUDA(c, ensure(c->colm, d.Qs * 8));
  EDAA_CUDA(c, ensure(c->colS, d.Qs * 8));
  EDAA_CUDA(c, ensure(c->collogS, d.Qs * 8));
  EDAA_CUDA(c, ensure(c->eta_a, d.M * 8));
  EDAA_CUDA(c, ensure(c->eta_b, d.M * 8));
  EDAA_CUDA(c, ensure(c->gamma, d.M * 8));
  EDAA_CUDA(c, ensure(c->trace, static_cast<size_t>(d.M) * (T + 1) * 8));
  EDAA_CUDA(c, ensure(c->part_C, S * d.Lrows * d.Qs * 8));
  EDAA_CUDA(c, ensure(c->part_m, S * d.Qs * 8));
  EDAA_CUDA(c, ensure(c->part_S, S * d.Qs * 8));
  EDAA_CUDA(c, ensure(c->part_obj, S * d.M * 8));
  EDAA_CUDA(c, ensure(c->fac, S * d.Qs * 8));
  EDAA_CUDA(c, ensure(c->E, static_cast<size_t>(d.M) * d.Lpad * d.p * 8));
  EDAA_CUDA(c, ensure(c->fit, d.M * 8));
  EDAA_CUDA(c, ensure(c->mu, d.M * 8));
  EDAA_CUDA(c, ensure(c->part_fit, static_cast<size_t>(d.M) * c->fit_blocks * 8));
  EDAA_CUDA(c, ensure(c->seeds, d.M * 8));
  EDAA_CUDA(c, ensure(c->fail_key, d.M * 8));
  EDAA_CUDA(c, ensure(c->fail_code, d.M * 4));
  EDAA_CUDA(c, ensure(c->fail_value, d.M * 8));
  EDAA_CUDA(c, ensure(c->cand, d.M));
  EDAA_CUDA(c, ensure(c->selected, 8));
  EDAA_CUDA(c, ensure(c->fit_min, 8));
  return EDAA_OK;
}

edaa::PassArgs pass_args(edaa_ctx* c, int t, const double* W) {
  edaa::PassArgs a{};
  a.d = c->d;
  a.t = t;
  a.X = c->X;
  a.xnorm = c->xnorm;
  a.W = W;
  a.A = P<double>(c->A);
  a.Lg = P<double>(c->Lg);
  a.colm = P<double>(c->colm);
  a.collogS = P<double>(c->collogS);
  a.Gbuf = P<double>(c->Gbuf);
  a.eta_a = P<double>(c->eta_a);
  a.eta_b = P<double>(c->eta_b);
  a.seeds = P<uint64_t>(c->seeds);
  a.part_C = P<double>(c->part_C);
  a.part_m = P<double>(c->part_m);
  a.part_S = P<double>(c->part_S);
  a.part_obj = P<double>(c->part_obj);
  a.fail_key = P<unsigned long long>(c->fail_key);
  a.observe_A = nullptr;
  a.kprof = static_cast<unsigned long long*>(c->kprof_buf);
  a.dbg = c->dbg;
  a.xmap = &c->xmap;
  return a;
}

edaa::CombineArgs combine_args(edaa_ctx* c, int t, int mode, int trace_index, int kin = 0) {
  edaa::CombineArgs a{};
  a.d = c->d;
  a.t = t;
  a.mode = mode;
  a.part_C = P<double>(c->part_C);
  a.part_m = P<double>(c->part_m);
  a.part_S = P<double>(c->part_S);
  a.part_obj = P<double>(c->part_obj);
  a.Y = P<double>(c->Y);
  a.colm = P<double>(c->colm);
  a.colS = P<double>(c->colS);
  a.collogS = P<double>(c->collogS);
  a.fac = P<double>(c->fac);
  a.XAt = P<double>(c->XAt);
  a.AAt = P<double>(c->AAt);
  a.Z = (mode == edaa::kModeA || mode == edaa::kModeB) ? P<double>(c->Z) : nullptr;
  a.trace = P<double>(c->trace);
  a.trace_stride = static_cast<int>(c->T + 1);
  a.trace_index = trace_index;
  a.fail_key = P<unsigned long long>(c->fail_key);
  a.kin = kin;
  return a;
}

edaa::PostArgs post_args(edaa_ctx* c, int mode) {
  edaa::PostArgs a{};
  a.d = c->d;
  a.mode = mode;
  a.Y = P<double>(c->Y);
  a.XAt = P<double>(c->XAt);
  a.AAt = P<double>(c->AAt);
  a.Z = P<double>(c->Z);
  a.Gbuf = P<double>(c->Gbuf);
  a.gamma = P<double>(c->gamma);
  a.eta_a = P<double>(c->eta_a);
  a.eta_b = P<double>(c->eta_b);
  a.fail_code = P<int>(c->fail_code);
  a.fail_value = P<double>(c->fail_value);
  return a;
}

#define EDAA_LAUNCH_N(ctx, call, n)                                 \
  do {                                                              \
    cudaError_t e_ = (call);                                        \
    if (e_ != cudaSuccess) return cuda_fail((ctx), e_, #call);      \
    (ctx)->launches += (n);                                         \
  } while (0)
#define EDAA_LAUNCH(ctx, call) EDAA_LAUNCH_N(ctx, call, 1)

// Profiling brackets: an event pair of the given kind (0-3 = pass mode, 4 = combine) around
// whatever is enqueued between prof_begin and prof_end.
int prof_begin(edaa_ctx* c, int kind, cudaEvent_t* e1) {
  *e1 = nullptr;
  if (!c->profile) return EDAA_OK;
  while (c->ev_pool.size() < 2 * (c->ev_used + 1)) {
    cudaEvent_t e;
    EDAA_CUDA(c, cudaEventCreate(&e));
    c->ev_pool.push_back(e);
  }
  cudaEvent_t e0 = c->ev_pool[2 * c->ev_used];
  *e1 = c->ev_pool[2 * c->ev_used + 1];
  if (c->ev_kind.size() <= c->ev_used) c->ev_kind.resize(c->ev_used + 1);
  c->ev_kind[c->ev_used] = kind;
  ++c->ev_used;
  EDAA_CUDA(c, cudaEventRecord(e0, c->stream));
  return EDAA_OK;
}
int prof_end(edaa_ctx* c, cudaEvent_t e1) {
  if (e1) EDAA_CUDA(c, cudaEventRecord(e1, c->stream));
  return EDAA_OK;
}

// A pass launch, bracketed by events when profiling (kind = pass mode).
int launch_pass_profiled(edaa_ctx* c, int mode, const edaa::PassArgs& pa) {
  cudaEvent_t e1 = nullptr;
  int rc = prof_begin(c, mode, &e1);
  if (rc) return rc;
  EDAA_LAUNCH(c, edaa::launch_pass(mode, pa, c->stream));
  return prof_end(c, e1);
}

// Observer hooks used by edaa_solve_observed (null in the batched path).
struct ObserveHook {
  edaa_observer_fn fn = nullptr;
  void* user = nullptr;
  std::vector<double> a_host, b_host, obs;
};

int download_b(edaa_ctx* c, ObserveHook* h) {
  const Dims& d = c->d;
  EDAA_LAUNCH(c, edaa::launch_materialize_b(P<double>(c->Lg), P<double>(c->colm), P<double>(c->colS),
                                            P<double>(c->Bv), d, c->stream));
  std::vector<double> bv(static_cast<size_t>(d.p) * d.Npad);
  EDAA_CUDA(c, cudaMemcpyAsync(bv.data(), c->Bv.p, bv.size() * 8, cudaMemcpyDeviceToHost, c->stream));
  EDAA_CUDA(c, cudaStreamSynchronize(c->stream));
  h->b_host.resize(static_cast<size_t>(d.N) * d.p);
  for (int j = 0; j < d.N; ++j)
    for (int i = 0; i < d.p; ++i) h->b_host[static_cast<size_t>(j) * d.p + i] = bv[static_cast<size_t>(i) * d.Npad + j];
  return EDAA_OK;
}

bool all_finite(const double* v, size_t n) {
  for (size_t i = 0; i < n; ++i)
    if (!std::isfinite(v[i])) return false;
  return true;
}

int enqueue_solve(edaa_ctx* c, const edaa_solve_params* prm, ObserveHook* hook);

// One solve: per-run seeds and step factors go up, then the whole device
// schedule (≈ 3 + T·(3 + 4·K2) + 7 kernels) runs — replayed from a CUDA graph
// captured on the first solve of a given shape (EDAA_NO_GRAPH=1 disables).
int solve_impl(edaa_ctx* c, const edaa_solve_params* prm, ObserveHook* hook) {
  NvtxRange nv("edaa/solve");
  Dims d{};
  int rc = make_dims(c, prm, &d);
  if (rc) return rc;
  if (hook && (c->comm || c->shard_emulate > 1))
    return set_err(c, EDAA_ERR_UNSUPPORTED, "observed solves are not pixel-sharded");
  c->d = d;
  c->T = prm->outer_iters;
  c->solved = false;
  rc = alloc_solve(c, d, c->T);
  if (rc) return rc;
  rc = make_xmap(c, d);
  if (rc) return rc;
  c->gen = g_realloc_count.load() * 1000003ull + c->image_gen;
  cudaStream_t st = c->stream;
  EDAA_CUDA(c, cudaMemcpyAsync(c->seeds.p, prm->seeds, d.M * 8, cudaMemcpyHostToDevice, st));
  EDAA_CUDA(c, cudaMemcpyAsync(c->gamma.p, prm->gammas, d.M * 8, cudaMemcpyHostToDevice, st));
  const bool use_graph = !hook && !c->profile && !c->no_graph;
  if (!use_graph) return enqueue_solve(c, prm, hook);
  GraphKey key{};
  key.d = d;
  key.T = c->T;
  key.K2 = prm->inner_iters_b;
  key.gen = c->gen;
  key.comm = c->comm;
  key.emulate = c->shard_emulate * 2 + c->shard_exchange;
  if (!(c->graph_exec && std::memcmp(&key, &c->graph_key, sizeof key) == 0)) {
    if (c->graph_exec) cudaGraphExecDestroy(c->graph_exec);
    c->graph_exec = nullptr;
    const uint64_t l0 = c->launches;
    EDAA_CUDA(c, cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal));
    rc = enqueue_solve(c, prm, nullptr);
    cudaGraph_t graph = nullptr;
    const cudaError_t ce = cudaStreamEndCapture(st, &graph);
    if (rc) {
      if (graph) cudaGraphDestroy(graph);
      return rc;
    }
    if (ce != cudaSuccess) return cuda_fail(c, ce, "cudaStreamEndCapture");
    const cudaError_t ie = cudaGraphInstantiate(&c->graph_exec, graph, 0);
    cudaGraphDestroy(graph);
    if (ie != cudaSuccess) return cuda_fail(c, ie, "cudaGraphInstantiate");
    c->graph_launches = c->launches - l0;
    c->launches = l0;
    c->graph_key = key;
  }
  EDAA_CUDA(c, cudaGraphLaunch(c->graph_exec, st));
  c->launches += c->graph_launches;
  return EDAA_OK;
}

// Pixel sharding: after every pass each rank broadcasts the partials of the
// slices it owns (in place, every rank a root once), so every rank then runs
// the unchanged fixed-order combine over all slices — the sharded solve is
// bitwise the single-device solve.  Messages per pass ≈ nslices·(L+24)·Q·8 B
// in total (A/B) or nslices·M·8 B (objective).
int exchange_partials(edaa_ctx* c, int mode) {
  const Dims& d = c->d;
  const NcclApi& n = nccl();
  const size_t cblk = static_cast<size_t>(d.Lrows) * d.Qs;
  EDAA_NCCL(c, n.GroupStart());
  for (int q = 0; q < c->shard_world; ++q) {
    int a = 0, b = 0;
    shard_slices(d, q, c->shard_world, &a, &b);
    if (b <= a) continue;
    if (mode != edaa::kModeObj) {
      double* pc = P<double>(c->part_C) + a * cblk;
      EDAA_NCCL(c, n.Broadcast(pc, pc, (b - a) * cblk, ncclFloat64, q, c->comm, c->stream));
    }
    if (mode == edaa::kModeB || mode == edaa::kModeInit) {
      double* pm = P<double>(c->part_m) + static_cast<size_t>(a) * d.Qs;
      double* ps = P<double>(c->part_S) + static_cast<size_t>(a) * d.Qs;
      EDAA_NCCL(c, n.Broadcast(pm, pm, static_cast<size_t>(b - a) * d.Qs, ncclFloat64, q, c->comm, c->stream));
      EDAA_NCCL(c, n.Broadcast(ps, ps, static_cast<size_t>(b - a) * d.Qs, ncclFloat64, q, c->comm, c->stream));
    } else {
      double* po = P<double>(c->part_obj) + static_cast<size_t>(a) * d.M;
      EDAA_NCCL(c, n.Broadcast(po, po, static_cast<size_t>(b - a) * d.M, ncclFloat64, q, c->comm, c->stream));
    }
  }
  EDAA_NCCL(c, n.GroupEnd());
  return EDAA_OK;
}

// Before the final phase: every rank's A and logits pixel columns to everyone,
// and the per-run failure keys (set by the pass of the pixel's owner) min-reduced.
// A rank's columns are packed into a dense [rows][wmax] block, ONE all-gather per
// array (and per block of rows, bounded staging) moves them, and every rank's
// block is unpacked into place (its own too: the values it already holds).
int exchange_state(edaa_ctx* c) {
  const Dims& d = c->d;
  const NcclApi& n = nccl();
  const int W = c->shard_world;
  EDAA_NCCL(c, n.AllReduce(c->fail_key.p, c->fail_key.p, d.M, ncclUint64, ncclMin, c->comm, c->stream));
  int wmax = 0, rblk = 0;
  state_stage_plan(c, d, &wmax, &rblk);
  const int rows = d.M * d.p;
  double* send = P<double>(c->shard_stage);
  double* recv = send + static_cast<size_t>(rblk) * wmax;
  int mj0 = 0, mj1 = 0;
  slice_pixels(d, d.sl0, d.sl1, &mj0, &mj1);
  for (double* arr : {P<double>(c->A), P<double>(c->Lg)}) {
    for (int r0 = 0; r0 < rows; r0 += rblk) {
      const int nr = std::min(rblk, rows - r0);
      double* base = arr + static_cast<size_t>(r0) * d.Npad;
      EDAA_LAUNCH(c, edaa::launch_pack_cols(base, send, nr, d.Npad, mj0, mj1 - mj0, wmax, false, nullptr, c->stream));
      EDAA_NCCL(c, n.AllGather(send, recv, static_cast<size_t>(rblk) * wmax, ncclFloat64, c->comm, c->stream));
      for (int q = 0; q < W; ++q) {
        int a = 0, b = 0, j0 = 0, j1 = 0;
        shard_slices(d, q, W, &a, &b);
        slice_pixels(d, a, b, &j0, &j1);
        EDAA_LAUNCH(c, edaa::launch_pack_cols(nullptr, recv + static_cast<size_t>(q) * rblk * wmax, nr, d.Npad, j0,
                                              j1 - j0, wmax, true, base, c->stream));
      }
    }
  }
  return EDAA_OK;
}

// One pass over the owned slices, then (sharded) the partial exchange.  In
// emulation mode (development/tests, one device) the slice ranges of
// shard_emulate ranks are launched one after another instead.
int run_pass(edaa_ctx* c, int mode, edaa::PassArgs pa) {
  if (c->shard_emulate > 1) {
    for (int q = 0; q < c->shard_emulate; ++q) {
      shard_slices(pa.d, q, c->shard_emulate, &pa.d.sl0, &pa.d.sl1);
      if (pa.d.sl1 <= pa.d.sl0) continue;
      const int rc = launch_pass_profiled(c, mode, pa);
      if (rc) return rc;
    }
    return EDAA_OK;
  }
  const int rc = launch_pass_profiled(c, mode, pa);
  if (rc || c->comm == nullptr || c->shard_exchange == 0) return rc;
  return exchange_partials(c, mode);
}

// The combine of one pass.  Unsharded, or sharded with the broadcast exchange
// (every slice partial is already on every rank): the fixed-order combine over
// all slices.  Sharded with the allreduce exchange (the default; BASELINE
// north_star: "NCCL allreduce of the L×p and p×p partial sums"): every rank
// reduces the slices it owns into one block of Lrows×Qs + 2·Qs + M doubles, the
// blocks are combined across ranks — for the B step a max-allreduce of the 
// column maxima, a rescale to that common reference, then ONE sum-allreduce of
// C | S | obj — and the same combine kernels finish from the reduced block as
// if it were a single slice.  Per pass and rank that is ~(L+24)·Q·8 bytes
// (cfg4 single run: 47.6 KB) instead of nslices·(L+24)·Q·8 (7 MB).  The sum
// over ranks is NCCL's, so the sharded result equals the single-device one to
// rounding (not bitwise; the broadcast exchange keeps the bitwise property).
int combine_pass_impl(edaa_ctx* c, const edaa::CombineArgs& a, int nlaunch);
int combine_pass(edaa_ctx* c, const edaa::CombineArgs& a, int nlaunch) {
  cudaEvent_t e1 = nullptr;
  int rc = prof_begin(c, 4, &e1);  // kind 4: the combine kernels (and, sharded, the exchange) of one pass
  if (!rc) rc = combine_pass_impl(c, a, nlaunch);
  if (!rc) rc = prof_end(c, e1);
  return rc;
}
int combine_pass_impl(edaa_ctx* c, const edaa::CombineArgs& a, int nlaunch) {
  const Dims& d = c->d;
  const bool emul = c->shard_emulate > 1;
  if (c->shard_exchange != 0 || (!c->comm && !emul)) {
    EDAA_LAUNCH_N(c, edaa::launch_combine(a, c->stream), nlaunch);
    return EDAA_OK;
  }
  const bool lse = a.mode == edaa::kModeB || a.mode == edaa::kModeInit;
  const size_t blk = edaa::shard_red_doubles(d), nsum = edaa::shard_red_sum_doubles(d);
  const int world = emul ? c->shard_emulate : 1;
  double* red = P<double>(c->shard_red);
  EDAA_CUDA(c, cudaMemsetAsync(red, 0, blk * world * 8, c->stream));
  double* mg = red + edaa::shard_red_off(d, 4);
  if (emul) {
    for (int q = 0; q < world; ++q) {
      int s0 = 0, s1 = 0;
      shard_slices(d, q, world, &s0, &s1);
      EDAA_LAUNCH_N(c, edaa::launch_shard_reduce(a, s0, s1, red + q * blk, c->stream), lse ? 2 : 1);
    }
    if (lse) {
      EDAA_LAUNCH(c, edaa::launch_shard_emul_max(d, red, blk, world, c->stream));
      for (int q = 0; q < world; ++q) EDAA_LAUNCH(c, edaa::launch_shard_rescale(d, red + q * blk, mg, c->stream));
    }
    EDAA_LAUNCH(c, edaa::launch_shard_emul_sum(red, blk, world, nsum, c->stream));
  } else {
    const NcclApi& n = nccl();
    EDAA_LAUNCH_N(c, edaa::launch_shard_reduce(a, d.sl0, d.sl1, red, c->stream), lse ? 2 : 1);
    if (lse) {
      EDAA_NCCL(c, n.AllReduce(red + edaa::shard_red_off(d, 3), mg, d.Qs, ncclFloat64, ncclMax, c->comm, c->stream));
      EDAA_LAUNCH(c, edaa::launch_shard_rescale(d, red, mg, c->stream));
    }
    EDAA_NCCL(c, n.AllReduce(red, red, nsum, ncclFloat64, ncclSum, c->comm, c->stream));
  }
  edaa::CombineArgs f = a;  // finish from the reduced block: one slice holding everything
  f.d.nslices = 1;
  f.part_C = red;
  f.part_S = red + edaa::shard_red_off(d, 1);
  f.part_obj = red + edaa::shard_red_off(d, 2);
  f.part_m = mg;
  EDAA_LAUNCH_N(c, edaa::launch_combine(f, c->stream), nlaunch);
  return EDAA_OK;
}

int enqueue_solve(edaa_ctx* c, const edaa_solve_params* prm, ObserveHook* hook) {
  const Dims d = c->d;
  int rc = EDAA_OK;
  cudaStream_t st = c->stream;
  EDAA_CUDA(c, cudaMemsetAsync(c->fail_key.p, 0xFF, d.M * 8, st));
  EDAA_CUDA(c, cudaMemsetAsync(c->fail_code.p, 0, d.M * 4, st));
  EDAA_CUDA(c, cudaMemsetAsync(c->fail_value.p, 0, d.M * 8, st));
  // Zero the band-padding rows of Y/Z (and everything else) once.
  EDAA_CUDA(c, cudaMemsetAsync(c->Y.p, 0, static_cast<size_t>(d.Lpad) * d.Qs * 8, st));
  EDAA_CUDA(c, cudaMemsetAsync(c->Z.p, 0, static_cast<size_t>(d.Lpad) * d.Qs * 8, st));
  EDAA_CUDA(c, cudaMemsetAsync(c->Gbuf.p, 0, static_cast<size_t>(d.QCpad) * d.Qs * 8, st));
  EDAA_CUDA(c, cudaMemsetAsync(c->E.p, 0, static_cast<size_t>(d.M) * d.Lpad * d.p * 8, st));
  EDAA_CUDA(c, cudaMemsetAsync(c->Lg.p, 0, static_cast<size_t>(d.M) * d.p * d.Npad * 8, st));
  c->ev_used = 0;
  k_fill_a<<<592, 256, 0, st>>>(P<double>(c->A), d.M, d.p, d.N, d.Npad);
  EDAA_LAUNCH(c, cudaGetLastError());

  if (hook) {
    EDAA_CUDA(c, ensure(c->obsA, static_cast<size_t>(d.K1) * d.p * d.Npad * 8));
    hook->obs.resize(static_cast<size_t>(d.K1) * d.p * d.Npad);
    hook->a_host.resize(static_cast<size_t>(d.p) * d.N);
  }

  // ---- initialisation: B⁰, Y⁰ = X·B⁰, η, G ----
  {
    NvtxRange nv("edaa/init");
    edaa::PassArgs pa = pass_args(c, 0, nullptr);
    rc = run_pass(c, edaa::kModeInit, pa);
    if (rc) return rc;
    rc = combine_pass(c, combine_args(c, 0, edaa::kModeInit, 0), 1);
    if (rc) return rc;
    EDAA_LAUNCH(c, edaa::launch_post(post_args(c, edaa::kPostInit), st));
  }
  for (size_t t = 1; t <= c->T; ++t) {
    const int ti = static_cast<int>(t);
    NvtxRange nv_outer("outer", t);
    {
    NvtxRange nv_a("edaa/A block");
    edaa::PassArgs pa = pass_args(c, ti, P<double>(c->Y));
    if (hook) pa.observe_A = P<double>(c->obsA);
    rc = run_pass(c, edaa::kModeA, pa);
    if (rc) return rc;
    rc = combine_pass(c, combine_args(c, ti, edaa::kModeA, ti - 1), 2);
    if (rc) return rc;
    if (hook) {
      // B is fixed through the A block; snapshot it once, then replay the K1 iterates.
      rc = download_b(c, hook);
      if (rc) return rc;
      EDAA_CUDA(c, cudaMemcpyAsync(hook->obs.data(), c->obsA.p, hook->obs.size() * 8,
                                   cudaMemcpyDeviceToHost, st));
      EDAA_CUDA(c, cudaStreamSynchronize(st));
      for (int k = 0; k < d.K1; ++k) {
        for (int i = 0; i < d.p; ++i)
          std::memcpy(hook->a_host.data() + static_cast<size_t>(i) * d.N,
                      hook->obs.data() + (static_cast<size_t>(k) * d.p + i) * d.Npad, d.N * 8);
        if (!all_finite(hook->a_host.data(), hook->a_host.size())) break;  // run failed here
        hook->fn(t, 'A', static_cast<size_t>(k + 1), hook->a_host.data(), hook->b_host.data(),
                 d.p, d.N, hook->user);
      }
    }
    }
    NvtxRange nv_b("edaa/B block");
    for (size_t k = 1; k <= prm->inner_iters_b; ++k) {
      edaa::PassArgs pb = pass_args(c, ti, P<double>(c->Z));
      rc = run_pass(c, edaa::kModeB, pb);
      if (rc) return rc;
      rc = combine_pass(c, combine_args(c, ti, edaa::kModeB, 0, static_cast<int>(k)), 1);
      if (rc) return rc;
      if (k == prm->inner_iters_b) EDAA_LAUNCH(c, edaa::launch_post(post_args(c, edaa::kPostG), st));
      if (hook) {
        rc = download_b(c, hook);
        if (rc) return rc;
        if (!all_finite(hook->b_host.data(), hook->b_host.size())) break;
        hook->fn(t, 'B', k, hook->a_host.data(), hook->b_host.data(), d.p, d.N, hook->user);
      }
    }
    if (hook) {
      unsigned long long key = 0;
      int code = 0;
      EDAA_CUDA(c, cudaMemcpyAsync(&key, c->fail_key.p, 8, cudaMemcpyDeviceToHost, st));
      EDAA_CUDA(c, cudaMemcpyAsync(&code, c->fail_code.p, 4, cudaMemcpyDeviceToHost, st));
      EDAA_CUDA(c, cudaStreamSynchronize(st));
      if (key != ~0ull || code != 0) break;  // the reference stops at the first failure
    }
  }
  // ---- finalisation: trace[T], B̂, Ê = X·B̂, fit, coherence ----
  {
    NvtxRange nv("edaa/final");
    edaa::PassArgs po = pass_args(c, static_cast<int>(c->T), P<double>(c->Y));
    rc = run_pass(c, edaa::kModeObj, po);
    if (rc) return rc;
    edaa::CombineArgs co = combine_args(c, static_cast<int>(c->T), edaa::kModeObj, static_cast<int>(c->T));
    rc = combine_pass(c, co, 1);
    if (rc) return rc;
    if (c->comm) {
      rc = exchange_state(c);
      if (rc) return rc;
    }
    EDAA_LAUNCH(c, edaa::launch_materialize_b(P<double>(c->Lg), P<double>(c->colm), P<double>(c->colS),
                                              P<double>(c->Bv), d, st));
    EDAA_LAUNCH(c, edaa::launch_strict_e(c->X, P<double>(c->Bv), P<double>(c->E), d, st));
    EDAA_LAUNCH_N(c, edaa::launch_fit(c->X, P<double>(c->E), P<double>(c->A), P<double>(c->part_fit),
                                    P<double>(c->fit), c->fit_blocks, d, st), 2);
    EDAA_LAUNCH(c, edaa::launch_coherence(P<double>(c->E), P<double>(c->mu), d, st));
  }
  return EDAA_OK;
}

}  // namespace

extern "C" {

const char* edaa_version(void) { return "edaa-b200 0.1.0 (sm_100a, fp64 DMMA)"; }
size_t edaa_max_endmembers(void) { return edaa::kMaxP; }
size_t edaa_max_bands(void) { return edaa::kMaxLpad; }

int edaa_create(int device, edaa_ctx** out) {
  if (!out) return EDAA_ERR_INVALID;
  *out = nullptr;
  int n = 0;
  cudaError_t e = cudaGetDeviceCount(&n);
  if (e != cudaSuccess || device < 0 || device >= n) return EDAA_ERR_CUDA;
  e = cudaSetDevice(device);
  if (e != cudaSuccess) return EDAA_ERR_CUDA;
  edaa_ctx* c = new edaa_ctx();
  c->device = device;
  e = cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking);
  if (e != cudaSuccess) {
    delete c;
    return EDAA_ERR_CUDA;
  }
  if (const char* dbg = std::getenv("EDAA_DBG")) c->dbg = std::atoi(dbg);
  if (const char* ng = std::getenv("EDAA_NO_GRAPH")) c->no_graph = ng[0] == '1';
  cudaDeviceGetAttribute(&c->num_sms, cudaDevAttrMultiProcessorCount, device);
  if (const char* kp = std::getenv("EDAA_KPROF"))
    if (kp[0] == '1' && cudaMalloc(&c->kprof_buf, 64 * 8) == cudaSuccess) cudaMemset(c->kprof_buf, 0, 64 * 8);
  *out = c;
  return EDAA_OK;
}

int edaa_destroy(edaa_ctx* c) {
  if (!c) return EDAA_OK;
  cudaSetDevice(c->device);
  cudaStreamSynchronize(c->stream);
  edaa_ctx::Buf* bufs[] = {&c->A, &c->Lg, &c->Bv, &c->Y, &c->Z, &c->XAt, &c->AAt, &c->Gbuf,
                           &c->colm, &c->colS, &c->collogS, &c->eta_a, &c->eta_b, &c->gamma,
                           &c->trace, &c->part_C, &c->part_m, &c->part_S, &c->part_obj, &c->fac, &c->E,
                           &c->fit, &c->mu, &c->part_fit, &c->seeds, &c->fail_key, &c->fail_code,
                           &c->fail_value, &c->cand, &c->selected, &c->fit_min, &c->obsA,
                           &c->pr_b, &c->pr_a, &c->pr_y, &c->pr_r, &c->pr_g, &c->pr_rat,
                           &c->pr_part, &c->pr_out, &c->in_raw, &c->in_x, &c->in_flags, &c->in_bad};
  for (auto* b : bufs)
    if (b->p) cudaFree(b->p);
  if (c->X) cudaFree(c->X);
  if (c->xnorm) cudaFree(c->xnorm);
  if (c->graph_exec) cudaGraphExecDestroy(c->graph_exec);
  if (c->comm) nccl().CommDestroy(c->comm);
  cudaStreamDestroy(c->stream);
  delete c;
  return EDAA_OK;
}

const char* edaa_last_error(const edaa_ctx* c) { return c ? c->err.c_str() : "null context"; }

void* edaa_stream(edaa_ctx* c) { return c ? static_cast<void*>(c->stream) : nullptr; }

static int prepare_image(edaa_ctx* c, size_t bands, size_t pixels, int xbytes) {
  if (bands < 1 || pixels < 1)
    return set_err(c, EDAA_ERR_INVALID, "image: needs at least one band and one pixel");
  if (pixels > (1u << 30) || bands > (1u << 20)) return set_err(c, EDAA_ERR_UNSUPPORTED, "image too large");
  EDAA_CUDA(c, cudaSetDevice(c->device));
  c->L = static_cast<int>(bands);
  c->N = static_cast<int>(pixels);
  c->Npad = (c->N + edaa::kNPad - 1) / edaa::kNPad * edaa::kNPad;
  c->xbytes = xbytes;
  // A captured solve schedule reads X and ‖x‖² through their device addresses and
  // the shape through Dims (part of the graph key), so new contents in the same
  // buffers replay the same graph; only a reallocation invalidates it.
  const size_t xb = static_cast<size_t>(c->L) * c->Npad * xbytes;
  if (c->x_cap < xb) {
    ++c->image_gen;
    if (c->X) cudaFree(c->X);
    c->X = nullptr;
    c->x_cap = 0;
    EDAA_CUDA(c, cudaMalloc(&c->X, xb));
    c->x_cap = xb;
  }
  const size_t nb = static_cast<size_t>(c->Npad) * 8;
  if (c->xn_cap < nb) {
    ++c->image_gen;
    if (c->xnorm) cudaFree(c->xnorm);
    c->xnorm = nullptr;
    c->xn_cap = 0;
    EDAA_CUDA(c, cudaMalloc(&c->xnorm, nb));
    c->xn_cap = nb;
  }
  c->solved = false;
  return EDAA_OK;
}

static int upload_host(edaa_ctx* c, const void* x, size_t bands, size_t pixels, int xbytes) {
  if (!c || !x) return set_err(c, EDAA_ERR_INVALID, "null argument");
  int rc = prepare_image(c, bands, pixels, xbytes);
  if (rc) return rc;
  const size_t pitch = static_cast<size_t>(c->Npad) * xbytes;
  EDAA_CUDA(c, cudaMemcpy2DAsync(c->X, pitch, x, pixels * xbytes, pixels * xbytes, bands,
                                 cudaMemcpyHostToDevice, c->stream));
  if (c->Npad > c->N)
    EDAA_CUDA(c, cudaMemset2DAsync(static_cast<char*>(c->X) + pixels * xbytes, pitch, 0,
                                   static_cast<size_t>(c->Npad - c->N) * xbytes, bands, c->stream));
  Dims d{};
  d.L = c->L;
  d.N = c->N;
  d.Npad = c->Npad;
  d.xbytes = xbytes;
  EDAA_LAUNCH(c, edaa::launch_xnorm(c->X, c->xnorm, d, c->stream));
  return EDAA_OK;
}

int edaa_set_image_host(edaa_ctx* c, const float* x, size_t bands, size_t pixels) {
  return upload_host(c, x, bands, pixels, 4);
}

// HsiImage::validate (image.cpp:10-27) on the context's fp32 image: the
// reference's message for the first offending element in row-major order.
static int check_image_f32(edaa_ctx* c) {
  cudaStream_t st = c->stream;
  EDAA_CUDA(c, ensure(c->in_bad, 24));
  unsigned long long* bad = P<unsigned long long>(c->in_bad);
  EDAA_CUDA(c, cudaMemsetAsync(bad, 0xFF, 16, st));
  const size_t total = static_cast<size_t>(c->L) * c->Npad;
  const int blocks = static_cast<int>(std::min<size_t>((total + 255) / 256, static_cast<size_t>(c->num_sms) * 8));
  k_check_f32<<<blocks, 256, 0, st>>>(static_cast<const float*>(c->X), c->L, c->N, c->Npad, bad);
  EDAA_CUDA(c, cudaGetLastError());
  unsigned long long hb[2];
  EDAA_CUDA(c, cudaMemcpyAsync(hb, bad, 16, cudaMemcpyDeviceToHost, st));
  EDAA_CUDA(c, cudaStreamSynchronize(st));
  if (hb[0] != ~0ull || hb[1] != ~0ull) {  // the reference throws at the first offending element
    return set_err(c, EDAA_ERR_INVALID, hb[0] < hb[1] ? "image: non-finite reflectance" : "image: negative reflectance");
  }
  return EDAA_OK;
}

int edaa_set_image_host_checked(edaa_ctx* c, const float* x, size_t bands, size_t pixels) {
  int rc = upload_host(c, x, bands, pixels, 4);
  if (rc) return rc;
  return check_image_f32(c);
}

int edaa_set_image_host_f64(edaa_ctx* c, const double* x, size_t bands, size_t pixels) {
  return upload_host(c, x, bands, pixels, 8);
}

// The caller's buffer may have been produced on any stream of this device and
// may be freed as soon as the call returns: the copy is ordered after ALL work
// already enqueued on the device (cudaDeviceSynchronize — the C-ABI carries no
// stream) and finished before returning; the pointer must be device memory of
// the context's GPU; the image is then validated like the host paths.
int edaa_set_image_device(edaa_ctx* c, const float* x, size_t bands, size_t pixels, size_t ld) {
  if (!c || !x) return set_err(c, EDAA_ERR_INVALID, "null argument");
  if (ld < pixels) return set_err(c, EDAA_ERR_INVALID, "row pitch smaller than the pixel count");
  EDAA_CUDA(c, cudaSetDevice(c->device));
  cudaPointerAttributes attr{};
  if (cudaPointerGetAttributes(&attr, x) != cudaSuccess) {
    cudaGetLastError();
    return set_err(c, EDAA_ERR_INVALID, "image pointer is not CUDA memory");
  }
  if (attr.type != cudaMemoryTypeDevice && attr.type != cudaMemoryTypeManaged)
    return set_err(c, EDAA_ERR_INVALID, "image pointer is not device memory");
  if (attr.device != c->device)
    return set_err(c, EDAA_ERR_INVALID, "image pointer is on another device than the context");
  int rc = prepare_image(c, bands, pixels, 4);
  if (rc) return rc;
  EDAA_CUDA(c, cudaDeviceSynchronize());  // the producer's writes (any stream) are complete
  k_pad_copy<<<592, 256, 0, c->stream>>>(x, ld, static_cast<float*>(c->X), c->L, c->N, c->Npad);
  EDAA_LAUNCH(c, cudaGetLastError());
  Dims d{};
  d.L = c->L;
  d.N = c->N;
  d.Npad = c->Npad;
  d.xbytes = 4;
  EDAA_LAUNCH(c, edaa::launch_xnorm(c->X, c->xnorm, d, c->stream));
  return check_image_f32(c);  // synchronises c->stream: the caller may free x on return
}

// Shared by the fp64 and fp32 ingests: upload the raw image as given, then
// validate + normalise it on the device (k_ingest) into the solver's image.
}  // extern "C"

template <class T, bool PIXEL_MAJOR>
static int ingest_impl(edaa_ctx* c, const T* x, size_t bands, size_t pixels, size_t* zero_pixels,
                       size_t zero_cap, size_t* n_zero) {
  if (!c || !x) return set_err(c, EDAA_ERR_INVALID, "null argument");
  if (bands < 1 || pixels < 1) return set_err(c, EDAA_ERR_INVALID, "image: needs at least one band and one pixel");
  if (pixels > (1u << 30) || bands > (1u << 20)) return set_err(c, EDAA_ERR_UNSUPPORTED, "image too large");
  EDAA_CUDA(c, cudaSetDevice(c->device));
  const int L = static_cast<int>(bands), N = static_cast<int>(pixels);
  const int Npad = (N + edaa::kNPad - 1) / edaa::kNPad * edaa::kNPad;
  const size_t raw_bytes = bands * pixels * sizeof(T), xn_bytes = static_cast<size_t>(L) * Npad * 8;
  EDAA_CUDA(c, ensure(c->in_raw, raw_bytes));
  EDAA_CUDA(c, ensure(c->in_x, xn_bytes));
  EDAA_CUDA(c, ensure(c->in_flags, static_cast<size_t>(Npad)));
  EDAA_CUDA(c, ensure(c->in_bad, 24));
  cudaStream_t st = c->stream;
  EDAA_CUDA(c, cudaMemcpyAsync(c->in_raw.p, x, raw_bytes, cudaMemcpyHostToDevice, st));
  EDAA_CUDA(c, cudaMemsetAsync(c->in_bad.p, 0xFF, 16, st));
  EDAA_CUDA(c, cudaMemsetAsync(static_cast<char*>(c->in_bad.p) + 16, 0, 8, st));
  unsigned long long* bad = P<unsigned long long>(c->in_bad);
  k_ingest<T, PIXEL_MAJOR><<<(Npad + 127) / 128, 128, 0, st>>>(
      P<T>(c->in_raw), P<double>(c->in_x), L, N, Npad, bad, P<unsigned char>(c->in_flags),
      reinterpret_cast<unsigned int*>(bad + 2));
  EDAA_LAUNCH(c, cudaGetLastError());
  unsigned long long hb[3];
  std::vector<unsigned char> flags(N);
  EDAA_CUDA(c, cudaMemcpyAsync(hb, bad, 24, cudaMemcpyDeviceToHost, st));
  EDAA_CUDA(c, cudaMemcpyAsync(flags.data(), c->in_flags.p, N, cudaMemcpyDeviceToHost, st));
  EDAA_CUDA(c, cudaStreamSynchronize(st));
  if (hb[0] != ~0ull || hb[1] != ~0ull)  // the reference throws at the first offending element
    return set_err(c, EDAA_ERR_INVALID, hb[0] < hb[1] ? "image: non-finite reflectance" : "image: negative reflectance");
  size_t nz = 0;
  for (int j = 0; j < N; ++j)
    if (flags[j]) {
      if (zero_pixels && nz < zero_cap) zero_pixels[nz] = static_cast<size_t>(j);
      ++nz;
    }
  if (n_zero) *n_zero = nz;
  if (nz == pixels) return set_err(c, EDAA_ERR_INVALID, "degenerate input: all pixels are zero");
  const int xbytes = (static_cast<unsigned int>(hb[2]) == 0u) ? 4 : 8;  // fp32-exact → the fp32 image path
  int rc = prepare_image(c, bands, pixels, xbytes);
  if (rc) return rc;
  if (xbytes == 4) {
    k_to_f32<<<592, 256, 0, st>>>(P<double>(c->in_x), static_cast<float*>(c->X), static_cast<size_t>(L) * Npad);
    EDAA_LAUNCH(c, cudaGetLastError());
  } else {
    EDAA_CUDA(c, cudaMemcpyAsync(c->X, c->in_x.p, xn_bytes, cudaMemcpyDeviceToDevice, st));
  }
  Dims d{};
  d.L = c->L;
  d.N = c->N;
  d.Npad = c->Npad;
  d.xbytes = xbytes;
  EDAA_LAUNCH(c, edaa::launch_xnorm(c->X, c->xnorm, d, st));
  return EDAA_OK;
}

extern "C" {

int edaa_ingest_host(edaa_ctx* c, const double* x, size_t bands, size_t pixels, size_t* zero_pixels,
                     size_t zero_cap, size_t* n_zero) {
  return ingest_impl<double, false>(c, x, bands, pixels, zero_pixels, zero_cap, n_zero);
}

int edaa_ingest_host_f32(edaa_ctx* c, const float* x, size_t bands, size_t pixels, int pixel_major,
                         size_t* zero_pixels, size_t zero_cap, size_t* n_zero) {
  return pixel_major ? ingest_impl<float, true>(c, x, bands, pixels, zero_pixels, zero_cap, n_zero)
                     : ingest_impl<float, false>(c, x, bands, pixels, zero_pixels, zero_cap, n_zero);
}

int edaa_image_get(edaa_ctx* c, double* out, int* xbytes) {
  if (!c || !out) return EDAA_ERR_INVALID;
  if (!c->X) return set_err(c, EDAA_ERR_STATE, "no image set");
  EDAA_CUDA(c, cudaSetDevice(c->device));
  const size_t n = static_cast<size_t>(c->L) * c->Npad;
  std::vector<double> buf(n);
  if (c->xbytes == 8) {
    EDAA_CUDA(c, cudaMemcpyAsync(buf.data(), c->X, n * 8, cudaMemcpyDeviceToHost, c->stream));
  } else {
    std::vector<float> f(n);
    EDAA_CUDA(c, cudaMemcpyAsync(f.data(), c->X, n * 4, cudaMemcpyDeviceToHost, c->stream));
    EDAA_CUDA(c, cudaStreamSynchronize(c->stream));
    for (size_t i = 0; i < n; ++i) buf[i] = f[i];
  }
  EDAA_CUDA(c, cudaStreamSynchronize(c->stream));
  for (int l = 0; l < c->L; ++l)
    std::memcpy(out + static_cast<size_t>(l) * c->N, buf.data() + static_cast<size_t>(l) * c->Npad, c->N * 8);
  if (xbytes) *xbytes = c->xbytes;
  return EDAA_OK;
}

int edaa_solve_async(edaa_ctx* c, const edaa_solve_params* prm) {
  if (!c) return EDAA_ERR_INVALID;
  EDAA_CUDA(c, cudaSetDevice(c->device));
  return solve_impl(c, prm, nullptr);
}

int edaa_finish(edaa_ctx* c) {
  if (!c) return EDAA_ERR_INVALID;
  const Dims& d = c->d;
  EDAA_CUDA(c, cudaStreamSynchronize(c->stream));
  c->h_fit.resize(d.M);
  c->h_mu.resize(d.M);
  c->h_eta_a.resize(d.M);
  c->h_eta_b.resize(d.M);
  c->h_fail_value.resize(d.M);
  c->h_fail_code.resize(d.M);
  c->h_fail_key.resize(d.M);
  c->h_trace.resize(static_cast<size_t>(d.M) * (c->T + 1));
  EDAA_CUDA(c, cudaMemcpy(c->h_fit.data(), c->fit.p, d.M * 8, cudaMemcpyDeviceToHost));
  EDAA_CUDA(c, cudaMemcpy(c->h_mu.data(), c->mu.p, d.M * 8, cudaMemcpyDeviceToHost));
  EDAA_CUDA(c, cudaMemcpy(c->h_eta_a.data(), c->eta_a.p, d.M * 8, cudaMemcpyDeviceToHost));
  EDAA_CUDA(c, cudaMemcpy(c->h_eta_b.data(), c->eta_b.p, d.M * 8, cudaMemcpyDeviceToHost));
  EDAA_CUDA(c, cudaMemcpy(c->h_fail_value.data(), c->fail_value.p, d.M * 8, cudaMemcpyDeviceToHost));
  EDAA_CUDA(c, cudaMemcpy(c->h_fail_code.data(), c->fail_code.p, d.M * 4, cudaMemcpyDeviceToHost));
  EDAA_CUDA(c, cudaMemcpy(c->h_fail_key.data(), c->fail_key.p, d.M * 8, cudaMemcpyDeviceToHost));
  EDAA_CUDA(c, cudaMemcpy(c->h_trace.data(), c->trace.p, c->h_trace.size() * 8, cudaMemcpyDeviceToHost));
  c->last_prof = edaa_profile{};
  for (size_t i = 0; i < c->ev_used; ++i) {
    float ms = 0.f;
    EDAA_CUDA(c, cudaEventElapsedTime(&ms, c->ev_pool[2 * i], c->ev_pool[2 * i + 1]));
    const int k = c->ev_kind[i];
    c->last_prof.ms[k] += ms;
    c->last_prof.launches[k] += 1;
  }
  c->ev_used = 0;
  c->solved = true;
  if (c->kprof_buf) {
    unsigned long long v[64];
    cudaMemcpy(v, c->kprof_buf, sizeof v, cudaMemcpyDeviceToHost);
    const char* names[4] = {"init", "A", "B", "obj"};
    for (int m = 0; m < 4; ++m) {
      const unsigned long long* w = v + 6 * m;
      std::fprintf(stderr, "[edaa kprof] %4s mma: x_wait %llu p1 %llu w_wait %llu p3 %llu | upd: s_wait %llu p2 %llu"
                   " | cta: setup %llu x0 %llu w0 %llu first-tile %llu loop-end sum %llu max %llu | ldx %llu rel %llu\n",
                   names[m], w[0], w[1], w[2], w[3], w[4], w[5], v[36 + 4 * m], v[37 + 4 * m], v[38 + 4 * m],
                   v[24 + 3 * m], v[25 + 3 * m], v[26 + 3 * m], v[52 + 2 * m], v[53 + 2 * m]);
    }
    cudaMemset(c->kprof_buf, 0, sizeof v);
  }
  return EDAA_OK;
}

int edaa_set_pass_order(edaa_ctx* c, int order) {
  if (!c) return EDAA_ERR_INVALID;
  if (order < 0 || order > 3) return set_err(c, EDAA_ERR_INVALID, "pass order must be 0 (auto), 1, 2 or 3");
  c->pass_order = order;
  return EDAA_OK;
}

int edaa_profile_enable(edaa_ctx* c, int on) {
  if (!c) return EDAA_ERR_INVALID;
  c->profile = on != 0;
  return EDAA_OK;
}

int edaa_profile_read(edaa_ctx* c, edaa_profile* out) {
  if (!c || !out) return EDAA_ERR_INVALID;
  *out = c->last_prof;
  return EDAA_OK;
}

uint64_t edaa_launch_count(const edaa_ctx* c) { return c ? c->launches : 0; }

int edaa_probe_fp64_peak(edaa_ctx* c, double* tflops) {
  if (!c || !tflops) return EDAA_ERR_INVALID;
  EDAA_CUDA(c, cudaSetDevice(c->device));
  int sms = 0;
  EDAA_CUDA(c, cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, c->device));
  double* out = nullptr;
  EDAA_CUDA(c, cudaMalloc(&out, static_cast<size_t>(sms) * 2 * 256 * 8));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int iters = 20000;
  double best = 0.0;
  for (int rep = 0; rep < 4; ++rep) {
    cudaEventRecord(e0, c->stream);
    k_dmma_peak<<<sms * 2, 256, 0, c->stream>>>(out, rep == 0 ? 100 : iters);
    cudaEventRecord(e1, c->stream);
    cudaError_t e = cudaEventSynchronize(e1);
    if (e != cudaSuccess) {
      cudaFree(out);
      return cuda_fail(c, e, "k_dmma_peak");
    }
    float ms = 0.f;
    cudaEventElapsedTime(&ms, e0, e1);
    const double flop = 2.0 * 256 * 4 * static_cast<double>(iters) * sms * 2 * 256 / 32;
    if (rep > 0) best = std::max(best, flop / (ms * 1e-3) / 1e12);
  }
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaFree(out);
  *tflops = best;
  return EDAA_OK;
}

int edaa_nccl_unique_id(void* out, size_t bytes) {
  if (!out || bytes < sizeof(ncclUniqueId)) return EDAA_ERR_INVALID;
  const NcclApi& n = nccl();
  if (!n.ok) return EDAA_ERR_UNSUPPORTED;
  ncclUniqueId id;
  if (n.GetUniqueId(&id) != ncclSuccess) return EDAA_ERR_CUDA;
  std::memcpy(out, &id, sizeof id);
  return EDAA_OK;
}

int edaa_set_pixel_shard(edaa_ctx* c, const void* id, size_t bytes, int rank, int world) {
  if (!c) return EDAA_ERR_INVALID;
  EDAA_CUDA(c, cudaSetDevice(c->device));
  EDAA_CUDA(c, cudaStreamSynchronize(c->stream));
  if (c->comm) {
    nccl().CommDestroy(c->comm);
    c->comm = nullptr;
  }
  c->shard_rank = 0;
  c->shard_world = 1;
  ++c->image_gen;  // captured schedules hold the old communicator
  c->solved = false;
  if (world <= 1 && id == nullptr) return EDAA_OK;  // sharding off
  // (world == 1 with an id: a one-rank communicator — the exchange runs, as a check)
  if (!id || bytes < sizeof(ncclUniqueId) || world < 1 || rank < 0 || rank >= world)
    return set_err(c, EDAA_ERR_INVALID, "pixel shard: bad unique id, rank or world size");
  const NcclApi& n = nccl();
  if (!n.ok) return set_err(c, EDAA_ERR_UNSUPPORTED, "pixel shard: " + n.why);
  ncclUniqueId uid;
  std::memcpy(&uid, id, sizeof uid);
  EDAA_NCCL(c, n.CommInitRank(&c->comm, world, uid, rank));
  c->shard_rank = rank;
  c->shard_world = world;
  return EDAA_OK;
}

int edaa_set_shard_emulation(edaa_ctx* c, int world) {
  if (!c || world < 0) return EDAA_ERR_INVALID;
  if (c->comm) return set_err(c, EDAA_ERR_STATE, "shard emulation with a live communicator");
  c->shard_emulate = world;
  ++c->image_gen;
  return EDAA_OK;
}

int edaa_set_shard_exchange(edaa_ctx* c, int mode) {
  if (!c || (mode != 0 && mode != 1)) return EDAA_ERR_INVALID;
  c->shard_exchange = mode;
  ++c->image_gen;
  return EDAA_OK;
}

int edaa_shard_pixels(edaa_ctx* c, size_t* first, size_t* end) {
  if (!c || !first || !end) return EDAA_ERR_INVALID;
  if (!c->solved && c->d.nslices == 0) return set_err(c, EDAA_ERR_STATE, "no solve yet");
  int j0 = 0, j1 = 0;
  slice_pixels(c->d, c->d.sl0, c->d.sl1, &j0, &j1);
  *first = static_cast<size_t>(std::min(j0, c->N));
  *end = static_cast<size_t>(std::min(j1, c->N));
  return EDAA_OK;
}

int edaa_solve(edaa_ctx* c, const edaa_solve_params* prm) {
  int rc = edaa_solve_async(c, prm);
  if (rc) return rc;
  return edaa_finish(c);
}

int edaa_run_record_get(edaa_ctx* c, size_t run, edaa_run_record* out) {
  if (!c || !out) return EDAA_ERR_INVALID;
  if (!c->solved) return set_err(c, EDAA_ERR_STATE, "no finished solve");
  if (run >= static_cast<size_t>(c->d.M)) return set_err(c, EDAA_ERR_INVALID, "run index out of range");
  std::memset(out, 0, sizeof *out);
  out->fit_l1 = c->h_fit[run];
  out->coherence = c->h_mu[run];
  out->eta_a = c->h_eta_a[run];
  out->eta_b = c->h_eta_b[run];
  int code = c->h_fail_code[run];
  size_t outer = 0;
  if (code == EDAA_RUN_OK && c->h_fail_key[run] != ~0ull) {
    code = fail_key_code(c->h_fail_key[run], &outer);
  }
  out->fail_code = code;
  out->fail_outer = outer;
  out->ok = code == EDAA_RUN_OK;
  const std::string msg = run_message(code, outer, c->h_fail_value[run]);
  std::snprintf(out->message, sizeof out->message, "%s", msg.c_str());
  return EDAA_OK;
}

int edaa_traces(edaa_ctx* c, double* out) {
  if (!c || !out) return EDAA_ERR_INVALID;
  if (!c->solved) return set_err(c, EDAA_ERR_STATE, "no finished solve");
  std::memcpy(out, c->h_trace.data(), c->h_trace.size() * 8);
  return EDAA_OK;
}

int edaa_factors(edaa_ctx* c, size_t run, double* a, double* b, double* e) {
  if (!c) return EDAA_ERR_INVALID;
  if (!c->solved) return set_err(c, EDAA_ERR_STATE, "no finished solve");
  const Dims& d = c->d;
  if (run >= static_cast<size_t>(d.M)) return set_err(c, EDAA_ERR_INVALID, "run index out of range");
  const size_t pN = static_cast<size_t>(d.p) * d.Npad;
  if (a) {
    EDAA_CUDA(c, cudaMemcpy2D(a, d.N * 8, P<double>(c->A) + run * pN, d.Npad * 8, d.N * 8, d.p,
                              cudaMemcpyDeviceToHost));
  }
  if (b) {  // device keeps B column-major per run; the reference layout is N×p
    std::vector<double> tmp(pN);
    EDAA_CUDA(c, cudaMemcpy(tmp.data(), P<double>(c->Bv) + run * pN, pN * 8, cudaMemcpyDeviceToHost));
    for (int j = 0; j < d.N; ++j)
      for (int i = 0; i < d.p; ++i) b[static_cast<size_t>(j) * d.p + i] = tmp[static_cast<size_t>(i) * d.Npad + j];
  }
  if (e) {
    EDAA_CUDA(c, cudaMemcpy(e, P<double>(c->E) + run * d.Lpad * d.p, static_cast<size_t>(d.L) * d.p * 8,
                            cudaMemcpyDeviceToHost));
  }
  return EDAA_OK;
}

int edaa_select(edaa_ctx* c, double fit_slack, uint8_t* cand, size_t* selected, double* fit_min) {
  if (!c || !cand || !selected || !fit_min) return EDAA_ERR_INVALID;
  if (!c->solved) return set_err(c, EDAA_ERR_STATE, "no finished solve");
  if (!std::isfinite(fit_slack) || fit_slack < 1.0)
    return set_err(c, EDAA_ERR_INVALID, "fit slack must be at least 1");
  const Dims& d = c->d;
  EDAA_LAUNCH(c, edaa::launch_select(P<double>(c->fit), P<double>(c->mu), P<int>(c->fail_code),
                                     P<unsigned long long>(c->fail_key), d.M, fit_slack,
                                     P<unsigned char>(c->cand), P<long long>(c->selected),
                                     P<double>(c->fit_min), c->stream));
  long long sel = -1;
  EDAA_CUDA(c, cudaMemcpyAsync(cand, c->cand.p, d.M, cudaMemcpyDeviceToHost, c->stream));
  EDAA_CUDA(c, cudaMemcpyAsync(&sel, c->selected.p, 8, cudaMemcpyDeviceToHost, c->stream));
  EDAA_CUDA(c, cudaMemcpyAsync(fit_min, c->fit_min.p, 8, cudaMemcpyDeviceToHost, c->stream));
  EDAA_CUDA(c, cudaStreamSynchronize(c->stream));
  if (sel < 0) return set_err(c, EDAA_ERR_ALL_FAILED, "every run failed");
  *selected = static_cast<size_t>(sel);
  return EDAA_OK;
}

int edaa_solve_observed(edaa_ctx* c, const edaa_solve_params* prm, edaa_observer_fn fn, void* user) {
  if (!c || !fn) return set_err(c, EDAA_ERR_INVALID, "null argument");
  if (!prm || prm->runs != 1) return set_err(c, EDAA_ERR_INVALID, "observed mode takes exactly one run");
  EDAA_CUDA(c, cudaSetDevice(c->device));
  ObserveHook hook;
  hook.fn = fn;
  hook.user = user;
  int rc = solve_impl(c, prm, &hook);
  if (rc) return rc;
  return edaa_finish(c);
}

}  // extern "C"

// ---------------------------------------------------------------------------
// Single-evaluation primitives on the image set in the context.
namespace {

Dims prim_dims(edaa_ctx* c, size_t p) {
  Dims d{};
  d.L = c->L;
  d.Lpad = (c->L + 7) / 8 * 8;
  d.N = c->N;
  d.Npad = c->Npad;
  d.M = 1;
  d.p = static_cast<int>(p);
  d.xbytes = c->xbytes;
  return d;
}

// Upload a host p×N (row-major) matrix as [p][Npad] with zero padding.
int upload_pn(edaa_ctx* c, edaa_ctx::Buf& buf, const double* a, size_t p) {
  const size_t pitch = static_cast<size_t>(c->Npad) * 8;
  EDAA_CUDA(c, ensure(buf, p * pitch));
  EDAA_CUDA(c, cudaMemsetAsync(buf.p, 0, p * pitch, c->stream));
  EDAA_CUDA(c, cudaMemcpy2DAsync(buf.p, pitch, a, c->N * 8, c->N * 8, p, cudaMemcpyHostToDevice, c->stream));
  return EDAA_OK;
}

// Y = X·B (L×p, reference order) from a host N×p B; Y stays in c->pr_y as [L][p].
int device_xb(edaa_ctx* c, const double* b, size_t p) {
  std::vector<double> bt(p * c->N);
  for (int j = 0; j < c->N; ++j)
    for (size_t i = 0; i < p; ++i) bt[i * c->N + j] = b[static_cast<size_t>(j) * p + i];
  int rc = upload_pn(c, c->pr_b, bt.data(), p);
  if (rc) return rc;
  const Dims d = prim_dims(c, p);
  EDAA_CUDA(c, ensure(c->pr_y, static_cast<size_t>(d.Lpad) * p * 8));
  EDAA_LAUNCH(c, edaa::launch_strict_e(c->X, P<double>(c->pr_b), P<double>(c->pr_y), d, c->stream));
  return EDAA_OK;
}

int residual_from(edaa_ctx* c, const double* a, size_t p) {
  int rc = upload_pn(c, c->pr_a, a, p);
  if (rc) return rc;
  EDAA_CUDA(c, ensure(c->pr_r, static_cast<size_t>(c->L) * c->Npad * 8));
  EDAA_LAUNCH(c, edaa::launch_residual(c->X, c->xbytes, P<double>(c->pr_y), P<double>(c->pr_a),
                                       P<double>(c->pr_r), c->L, c->N, c->Npad, static_cast<int>(p), c->stream));
  return EDAA_OK;
}

int reduce_r(edaa_ctx* c, int mode, double scale, double* out) {
  const int parts = 256;
  EDAA_CUDA(c, ensure(c->pr_part, parts * 8));
  EDAA_CUDA(c, ensure(c->pr_out, 8));
  EDAA_LAUNCH_N(c, edaa::launch_reduce(P<double>(c->pr_r), static_cast<size_t>(c->L) * c->Npad, mode,
                                       scale, P<double>(c->pr_part), parts, P<double>(c->pr_out), c->stream), 2);
  EDAA_CUDA(c, cudaMemcpyAsync(out, c->pr_out.p, 8, cudaMemcpyDeviceToHost, c->stream));
  EDAA_CUDA(c, cudaStreamSynchronize(c->stream));
  return EDAA_OK;
}

int prim_check(edaa_ctx* c, size_t p, const void* a, const void* b) {
  if (!c || !a || !b) return set_err(c, EDAA_ERR_INVALID, "null argument");
  if (c->X == nullptr) return set_err(c, EDAA_ERR_STATE, "no image set");
  if (p < 1) return set_err(c, EDAA_ERR_INVALID, "need at least one endmember");
  EDAA_CUDA(c, cudaSetDevice(c->device));
  return EDAA_OK;
}

}  // namespace

extern "C" {

int edaa_xb(edaa_ctx* c, const double* b, size_t p, double* y) {
  int rc = prim_check(c, p, b, y);
  if (rc) return rc;
  rc = device_xb(c, b, p);
  if (rc) return rc;
  EDAA_CUDA(c, cudaMemcpyAsync(y, c->pr_y.p, static_cast<size_t>(c->L) * p * 8, cudaMemcpyDeviceToHost, c->stream));
  EDAA_CUDA(c, cudaStreamSynchronize(c->stream));
  return EDAA_OK;
}

int edaa_objective(edaa_ctx* c, const double* b, const double* a, size_t p, double* out) {
  int rc = prim_check(c, p, b, a);
  if (!rc) rc = device_xb(c, b, p);
  if (!rc) rc = residual_from(c, a, p);
  if (!rc) rc = reduce_r(c, 0, 0.5, out);
  return rc;
}

int edaa_fit_l1(edaa_ctx* c, const double* e, const double* a, size_t p, double* out) {
  int rc = prim_check(c, p, e, a);
  if (rc) return rc;
  EDAA_CUDA(c, ensure(c->pr_y, static_cast<size_t>(c->L) * p * 8));
  EDAA_CUDA(c, cudaMemcpyAsync(c->pr_y.p, e, static_cast<size_t>(c->L) * p * 8, cudaMemcpyHostToDevice, c->stream));
  rc = residual_from(c, a, p);
  if (!rc) rc = reduce_r(c, 1, 1.0, out);
  return rc;
}

int edaa_grad_abundances(edaa_ctx* c, const double* b, const double* a, size_t p, double* g) {
  int rc = prim_check(c, p, b, a);
  if (!rc) rc = device_xb(c, b, p);
  if (!rc) rc = residual_from(c, a, p);
  if (rc) return rc;
  EDAA_CUDA(c, ensure(c->pr_g, p * c->N * 8));
  EDAA_LAUNCH(c, edaa::launch_grad_a(P<double>(c->pr_y), P<double>(c->pr_r), P<double>(c->pr_g), c->L,
                                     c->N, c->Npad, static_cast<int>(p), c->stream));
  EDAA_CUDA(c, cudaMemcpyAsync(g, c->pr_g.p, p * c->N * 8, cudaMemcpyDeviceToHost, c->stream));
  EDAA_CUDA(c, cudaStreamSynchronize(c->stream));
  return EDAA_OK;
}

int edaa_grad_contributions(edaa_ctx* c, const double* b, const double* a, size_t p, double* g) {
  int rc = prim_check(c, p, b, a);
  if (!rc) rc = device_xb(c, b, p);
  if (!rc) rc = residual_from(c, a, p);
  if (rc) return rc;
  EDAA_CUDA(c, ensure(c->pr_g, p * c->N * 8));
  EDAA_CUDA(c, ensure(c->pr_rat, static_cast<size_t>(c->L) * p * 8));
  EDAA_LAUNCH_N(c, edaa::launch_grad_b(c->X, c->xbytes, P<double>(c->pr_r), P<double>(c->pr_a),
                                       P<double>(c->pr_rat), P<double>(c->pr_g), c->L, c->N, c->Npad,
                                       static_cast<int>(p), c->stream), 2);
  EDAA_CUDA(c, cudaMemcpyAsync(g, c->pr_g.p, p * c->N * 8, cudaMemcpyDeviceToHost, c->stream));
  EDAA_CUDA(c, cudaStreamSynchronize(c->stream));
  return EDAA_OK;
}

int edaa_check_iterate(edaa_ctx* c, const double* m, size_t rows, size_t cols, size_t outer,
                       int contribution, int* code, char* message, size_t message_len) {
  if (!c || !m || !code || rows == 0 || cols == 0) return c ? set_err(c, EDAA_ERR_INVALID, "check_iterate: bad argument") : EDAA_ERR_INVALID;
  if (rows >= (1ull << 34) - 1 || cols >= (1ull << 28))
    return set_err(c, EDAA_ERR_UNSUPPORTED, "check_iterate: matrix too large");
  EDAA_CUDA(c, cudaSetDevice(c->device));
  EDAA_CUDA(c, ensure(c->pr_g, rows * cols * 8 + 8));
  unsigned long long* key = reinterpret_cast<unsigned long long*>(P<double>(c->pr_g) + rows * cols);
  EDAA_CUDA(c, cudaMemcpyAsync(c->pr_g.p, m, rows * cols * 8, cudaMemcpyHostToDevice, c->stream));
  EDAA_CUDA(c, cudaMemsetAsync(key, 0xFF, 8, c->stream));
  EDAA_LAUNCH(c, edaa::launch_check_iterate(P<double>(c->pr_g), static_cast<int>(rows), static_cast<int>(cols),
                                            key, c->stream));
  unsigned long long h = 0;
  EDAA_CUDA(c, cudaMemcpyAsync(&h, key, 8, cudaMemcpyDeviceToHost, c->stream));
  EDAA_CUDA(c, cudaStreamSynchronize(c->stream));
  *code = EDAA_RUN_OK;
  if (h != ~0ull) {
    switch (static_cast<unsigned>(h & 3ull)) {
      case edaa::kFailNonFinite: *code = contribution ? EDAA_RUN_NONFINITE_B : EDAA_RUN_NONFINITE_A; break;
      case edaa::kFailNegative: *code = contribution ? EDAA_RUN_SIMPLEX_B : EDAA_RUN_SIMPLEX_A; break;
      default: *code = contribution ? EDAA_RUN_DRIFT_B : EDAA_RUN_DRIFT_A; break;
    }
  }
  if (message && message_len) std::snprintf(message, message_len, "%s", run_message(*code, outer, 0.0).c_str());
  return EDAA_OK;
}

int edaa_estimate_abundances(edaa_ctx* c, const double* e, size_t p, size_t iters, double eta,
                             double* a) {
  int rc = prim_check(c, p, e, a);
  if (rc) return rc;
  if (p > static_cast<size_t>(edaa::kMaxP))
    return set_err(c, EDAA_ERR_UNSUPPORTED, "endmember count above the compiled maximum (16)");
  EDAA_CUDA(c, ensure(c->pr_y, static_cast<size_t>(c->L) * p * 8));
  EDAA_CUDA(c, cudaMemcpyAsync(c->pr_y.p, e, static_cast<size_t>(c->L) * p * 8, cudaMemcpyHostToDevice, c->stream));
  EDAA_CUDA(c, ensure(c->pr_g, p * c->N * 8));
  EDAA_LAUNCH(c, edaa::launch_estimate(c->X, c->xbytes, P<double>(c->pr_y), P<double>(c->pr_g), c->L, c->N,
                                       c->Npad, static_cast<int>(p), static_cast<int>(iters), eta, c->stream));
  EDAA_CUDA(c, cudaMemcpyAsync(a, c->pr_g.p, p * c->N * 8, cudaMemcpyDeviceToHost, c->stream));
  EDAA_CUDA(c, cudaStreamSynchronize(c->stream));
  return EDAA_OK;
}

}  // extern "C"
