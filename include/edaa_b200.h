/* edaa_b200.h — the C-ABI of the B200-native EDAA hot path.
 *
 * This is the drop-in boundary: plain pointers and sizes, status codes, no
 * exceptions and no CUDA/torch types in the signatures.  The C++ drop-in
 * layer (include/archetype/*.hpp, implemented in
 * paper_2209_11002_b200/csrc/host/) and the Python surface
 * (paper_2209_11002_b200/edaa.py) are both thin callers of it.
 *
 * Reference interfaces replaced (paths under /root/reference/proj):
 *   edaa_set_image*    the X argument of run()/run_ensemble()
 *                      (solver.hpp:81, ensemble.hpp:68-69; HsiImage image.hpp:18-28)
 *   edaa_solve*        run() — Algorithm 1 (solver.cpp:190-238) for a BATCH of
 *                      runs (seeds/gammas per run, ensemble.cpp:117-139)
 *   edaa_run_record    RunRecord / RunResult scalars (ensemble.hpp:31-40,
 *                      solver.hpp:29-38) incl. the archetype::Error message of a
 *                      failed run (ensemble.cpp:133-136)
 *   edaa_traces        RunResult::objective_trace (solver.hpp:37)
 *   edaa_factors       RunResult::{abundances, contributions, endmembers}
 *   edaa_select        select_runs() (ensemble.hpp:63, ensemble.cpp:71-94)
 *   edaa_solve_observed the StepObserver hook (solver.hpp:69-77,81)
 *
 * Threading: one context per device; a context is not thread-safe (the
 * C++ layer serialises).  All device memory is owned by the context.
 *
 * Precision contract: X is stored as fp32 (or fp64 via edaa_set_image_host_f64);
 * every contraction with X, every per-pixel update and every reduction is fp64.
 */
#ifndef EDAA_B200_H
#define EDAA_B200_H

#include <stddef.h>
#include <stdint.h>

#if defined(__GNUC__)
#define EDAA_API __attribute__((visibility("default")))
#else
#define EDAA_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

typedef struct edaa_ctx edaa_ctx;

enum {
  EDAA_OK = 0,
  EDAA_ERR_INVALID = 1,     /* bad argument */
  EDAA_ERR_CUDA = 2,        /* CUDA runtime failure (message in edaa_last_error) */
  EDAA_ERR_UNSUPPORTED = 3, /* shape outside the compiled kernels (p > 16, L > 320) */
  EDAA_ERR_STATE = 4,       /* call out of order (no image / no solve) */
  EDAA_ERR_ALL_FAILED = 5   /* edaa_select: "every run failed" (ensemble.cpp:79-80) */
};

/* Per-run failure codes (RunRecord.ok == false), see edaa_run_record. */
enum {
  EDAA_RUN_OK = 0,
  EDAA_RUN_NONFINITE_A = 1,    /* solver.cpp:72-75 on the abundance block */
  EDAA_RUN_NONFINITE_B = 2,    /* solver.cpp:72-75 on the contribution block */
  EDAA_RUN_DEGENERATE = 3,     /* solver.cpp:141 */
  EDAA_RUN_SPECTRAL_BAD = 4,   /* matrix.cpp:151-152 */
  EDAA_RUN_SPECTRAL_NOCONV = 5, /* matrix.cpp:186-189 */
  EDAA_RUN_SIMPLEX_A = 6,      /* "abundance iterate left the simplex ..."      solver.cpp:77-81 */
  EDAA_RUN_SIMPLEX_B = 7,      /* "contribution iterate left the simplex ..."   solver.cpp:77-81 */
  EDAA_RUN_DRIFT_A = 8,        /* "abundance column sum drifted from 1 ..."     solver.cpp:84-88 */
  EDAA_RUN_DRIFT_B = 9         /* "contribution column sum drifted from 1 ..."  solver.cpp:84-88 */
};

typedef struct {
  size_t endmembers;     /* p  (SolverConfig::endmembers, solver.hpp:16) */
  size_t outer_iters;    /* T  (solver.hpp:17) */
  size_t inner_iters_a;  /* K1 (solver.hpp:18) */
  size_t inner_iters_b;  /* K2 (solver.hpp:19) */
  size_t runs;           /* M runs batched on this device */
  const uint64_t* seeds; /* [runs] host: SolverConfig::seed of each run */
  const double* gammas;  /* [runs] host: SolverConfig::gamma of each run */
} edaa_solve_params;

typedef struct {
  double fit_l1;      /* RunResult::fit_l1 */
  double coherence;   /* RunResult::coherence */
  double eta_a;       /* StepSizes::eta_a (solver.hpp:48-51) */
  double eta_b;
  int ok;             /* 1 if the run finished (RunRecord::ok) */
  int fail_code;      /* EDAA_RUN_* */
  size_t fail_outer;  /* outer iteration named in the message (when applicable) */
  char message[192];  /* the reference's archetype::Error text, "" when ok */
} edaa_run_record;

/* Context lifetime. device = CUDA ordinal. */
EDAA_API int edaa_create(int device, edaa_ctx** out);
EDAA_API int edaa_destroy(edaa_ctx* ctx);
EDAA_API const char* edaa_last_error(const edaa_ctx* ctx);
/* The cudaStream_t all work is enqueued on (as void*), for event timing. */
EDAA_API void* edaa_stream(edaa_ctx* ctx);

/* Image X (L×N row-major, bands × pixels, already ℓ2-normalised and
 * validated by the caller).  _host copies from host memory (pinned or
 * pageable); _device copies from a device pointer with row pitch ld (floats).
 * _host_f64 keeps X in fp64 on the device (for inputs that are not exactly
 * representable in fp32: results then track the reference on ANY fp64 input;
 * one CTA per SM instead of two). */
EDAA_API int edaa_set_image_host(edaa_ctx* ctx, const float* x, size_t bands, size_t pixels);
EDAA_API int edaa_set_image_host_f64(edaa_ctx* ctx, const double* x, size_t bands, size_t pixels);
/* _host_checked: as _host, then HsiImage::validate (image.cpp:10-27) on the
 * device — EDAA_ERR_INVALID with the reference's message ("image: non-finite
 * reflectance" / "image: negative reflectance", whichever element comes first
 * in row-major order) when the image is not finite and non-negative. */
EDAA_API int edaa_set_image_host_checked(edaa_ctx* ctx, const float* x, size_t bands, size_t pixels);
/* _device: x must be device memory of the context's GPU (else EDAA_ERR_INVALID);
 * the copy is ordered after all work already enqueued on that device (any
 * stream) and complete when the call returns, so the caller may free x; the
 * image is validated like _host_checked. */
EDAA_API int edaa_set_image_device(edaa_ctx* ctx, const float* x, size_t bands, size_t pixels, size_t ld);

/* Ingest on the device: HsiImage::validate + l2_normalize
 * (image.cpp:10-47) fused into the upload.  x: the RAW L×N image (fp64,
 * row-major).  Errors carry the reference's messages ("image: non-finite
 * reflectance" / "image: negative reflectance" for the first offending element
 * in scan order, "degenerate input: all pixels are zero"); zero pixels are
 * listed ascending (the first zero_cap of them; *n_zero = their count) and left
 * unnormalised, as NormalizeResult::zero_pixels.  The normalised values are
 * bitwise the reference's; when all are exactly representable in fp32 the
 * solve uses the fp32 image, else the fp64 one.  edaa_image_get returns the
 * context's image as L×N fp64 (and its storage width, 4 or 8 bytes). */
EDAA_API int edaa_ingest_host(edaa_ctx* ctx, const double* x, size_t bands, size_t pixels,
                              size_t* zero_pixels, size_t zero_cap, size_t* n_zero);
/* The same ingest from an fp32 payload as stored in the file, without the
 * host widening and reorder: pixel_major = 0 for an L×N band-major image,
 * 1 for an N×L pixel-major one (an (H, W, L) NPY cube, npy_to_image's pixel
 * index r·W + c).  Results, zero list and messages are those of
 * edaa_ingest_host on npy_to_image's fp64 image (fp32 widens exactly); the
 * upload is half the bytes. */
EDAA_API int edaa_ingest_host_f32(edaa_ctx* ctx, const float* x, size_t bands, size_t pixels,
                                  int pixel_major, size_t* zero_pixels, size_t zero_cap, size_t* n_zero);
EDAA_API int edaa_image_get(edaa_ctx* ctx, double* out, int* xbytes);

/* Batched Algorithm 1 over all runs.  _async only enqueues on edaa_stream();
 * edaa_finish waits and fetches the per-run records.  edaa_solve = both. */
EDAA_API int edaa_solve_async(edaa_ctx* ctx, const edaa_solve_params* params);
EDAA_API int edaa_finish(edaa_ctx* ctx);
EDAA_API int edaa_solve(edaa_ctx* ctx, const edaa_solve_params* params);

/* Results of the last solve. */
EDAA_API int edaa_run_record_get(edaa_ctx* ctx, size_t run, edaa_run_record* out);
EDAA_API int edaa_traces(edaa_ctx* ctx, double* out /* [runs][T+1] */);
/* Any pointer may be NULL. a: p×N, b: N×p, e: L×p (reference layouts). */
EDAA_API int edaa_factors(edaa_ctx* ctx, size_t run, double* a, double* b, double* e);
/* Model selection on device over the last solve's records (ensemble.cpp:71-94).
 * cand: [runs] bytes; returns EDAA_ERR_ALL_FAILED when no run is ok. */
EDAA_API int edaa_select(edaa_ctx* ctx, double fit_slack, uint8_t* cand, size_t* selected,
                double* fit_min);

/* Observed mode (StepObserver): a single run (runs == 1) whose every inner
 * iterate is delivered, in order, to the callback as host arrays
 * (a: p×N, b: N×p).  block is 'A' or 'B'. */
typedef void (*edaa_observer_fn)(size_t outer, char block, size_t inner, const double* a,
                                 const double* b, size_t p, size_t n, void* user);
EDAA_API int edaa_solve_observed(edaa_ctx* ctx, const edaa_solve_params* params, edaa_observer_fn fn,
                        void* user);

/* Pixel sharding of one solve over the GPUs of a node (no
 * reference counterpart — the reference runs a solve on one host thread,
 * solver.cpp:190-238).  One context per GPU, one process (or thread) per
 * context.  Rank 0 makes a communicator id with edaa_nccl_unique_id and sends
 * its bytes to every rank out of band (torch.distributed in
 * paper_2209_11002_b200/distributed.py); every rank then calls
 * edaa_set_pixel_shard with the same id (collective: blocks until all world
 * ranks joined).  From then on each solve on the context processes only the
 * rank's pixel slices and exchanges the slice partials after every pass
 * (NCCL broadcasts, inside the captured CUDA graph), so every rank ends with
 * the full result, bitwise equal to the one-device solve.  id == NULL turns
 * sharding off (world == 1 with an id makes a one-rank communicator whose
 * exchanges run as a self-check).  NCCL (libnccl.so.2) is resolved at run time.
 * edaa_shard_pixels: the pixel range [first, end) this rank owns in the last
 * solve.  edaa_set_shard_emulation(ctx, W): development/test mode on ONE
 * device — every pass is launched as W consecutive slice-range launches (no
 * collective), which checks the sharded decomposition without more GPUs. */
EDAA_API int edaa_nccl_unique_id(void* out, size_t bytes /* >= 128 */);
EDAA_API int edaa_set_pixel_shard(edaa_ctx* ctx, const void* id, size_t bytes, int rank, int world);
EDAA_API int edaa_shard_pixels(edaa_ctx* ctx, size_t* first, size_t* end);
EDAA_API int edaa_set_shard_emulation(edaa_ctx* ctx, int world);
/* What the ranks exchange after every pass.
 *   0 (default): ALLREDUCE — BASELINE north_star's shape.  Every rank reduces
 *     the partial sums of its own pixel slices to one block (Y or XAᵀ: L×Q;
 *     AAᵀ: Q×Q on the run diagonal; the 2·Q softmax normaliser terms (m, S);
 *     the M objective terms), the column maxima are max-allreduced, the blocks
 *     rescaled to them and sum-allreduced: ~(L+24)·Q·8 bytes per pass and rank
 *     (cfg4 single run: 47.6 KB).  Equal to the single-device solve to
 *     rounding (the cross-rank sum order is NCCL's).
 *   1: BROADCAST of every slice partial (nslices·(L+24)·Q·8 bytes per pass:
 *     7 MB at cfg4) followed by the single-device fixed-order combine on every
 *     rank: bitwise the single-device result. */
EDAA_API int edaa_set_shard_exchange(edaa_ctx* ctx, int mode);

/* Order of the pass kernels' (pixel slice, run chunk) work items (no reference
 * counterpart: a scheduling knob of this implementation).  0 = auto (chunk-major
 * when X fits in L2, else slice-major interleaved over the CTAs when the items
 * divide evenly), 1 = chunk-major, 2 = plain slice-major, 3 = slice-major
 * interleaved (CTA b takes items b, b+G, …, so X slices are shared in L2: ~1/3
 * of the HBM traffic on images far larger than L2, at about the same speed;
 * plain slice-major if uneven).  The
 * per-(slice, chunk) partials, and so every result, are bitwise the same for
 * all orders; only the speed differs. */
EDAA_API int edaa_set_pass_order(edaa_ctx* ctx, int order);

/* Single-evaluation primitives on the image of the context (reference
 * solver.hpp:52-67,85-86 and ensemble.hpp:50).  Host arrays in the
 * reference layouts (b: N×p, a: p×N, e: L×p); entries follow the reference's
 * accumulation order.
 *   edaa_xb                   y = X·B (L×p)               — matmul(x, b), solver.cpp:140
 *   edaa_objective            ½‖X − XB·A‖²               — objective_l2, solver.cpp:184-188
 *   edaa_grad_abundances      g = −(XB)ᵀ(X − XBA)  (p×N)  — solver.cpp:166-172
 *   edaa_grad_contributions   g = −Xᵀ((X − XBA)Aᵀ) (N×p)  — solver.cpp:174-182
 *   edaa_fit_l1               Σ|X − E·A|                  — ensemble.cpp:29-39
 *   edaa_estimate_abundances  A for fixed E, `iters` entropic steps from 1/p
 *                                                          — solver.cpp:240-259 */
EDAA_API int edaa_xb(edaa_ctx* ctx, const double* b, size_t p, double* y);
EDAA_API int edaa_objective(edaa_ctx* ctx, const double* b, const double* a, size_t p, double* out);
EDAA_API int edaa_grad_abundances(edaa_ctx* ctx, const double* b, const double* a, size_t p, double* g);
EDAA_API int edaa_grad_contributions(edaa_ctx* ctx, const double* b, const double* a, size_t p,
                                     double* g);
EDAA_API int edaa_fit_l1(edaa_ctx* ctx, const double* e, const double* a, size_t p, double* out);
EDAA_API int edaa_estimate_abundances(edaa_ctx* ctx, const double* e, size_t p, size_t iters,
                                      double eta, double* a);

/* check_iterate (reference solver.cpp:65-90: the simplex / finiteness check the
 * solver applies after every inner update) on a host row-major rows×cols
 * matrix whose COLUMNS are the simplex vectors, evaluated on the device by the
 * per-column check the solve's kernels use.  *code = EDAA_RUN_OK, or the code of
 * the first failing check in the reference's scan order (column by column; per
 * entry finite then >= 0; then |Σ − 1| <= 1e-9) for the abundance block
 * (contribution = 0) or the contribution block (contribution != 0); `message`
 * receives the reference's text for it with `outer` as the iteration index. */
EDAA_API int edaa_check_iterate(edaa_ctx* ctx, const double* m, size_t rows, size_t cols, size_t outer,
                                int contribution, int* code, char* message, size_t message_len);

/* Instrumentation.  With profiling on, every pass launch is bracketed by CUDA
 * events on edaa_stream(); edaa_profile_read returns, per pass kind, the
 * summed device time (ms) and launch count of the last finished solve
 * (kind 0 = init pass, 1 = A pass, 2 = B pass, 3 = objective pass, 4 = the
 * combine kernels between the passes).
 * edaa_launch_count: kernels launched by this context since creation. */
typedef struct {
  double ms[5];
  uint64_t launches[5];
} edaa_profile;
EDAA_API int edaa_profile_enable(edaa_ctx* ctx, int on);
EDAA_API int edaa_profile_read(edaa_ctx* ctx, edaa_profile* out);
EDAA_API uint64_t edaa_launch_count(const edaa_ctx* ctx);
/* Measures the fp64 tensor-pipe (DMMA) peak of this device in TFLOP/s with
 * a register-resident microkernel (the roofline denominator for the passes). */
EDAA_API int edaa_probe_fp64_peak(edaa_ctx* ctx, double* tflops);

/* Version / capability probe. */
EDAA_API const char* edaa_version(void);
EDAA_API size_t edaa_max_endmembers(void);
EDAA_API size_t edaa_max_bands(void);

#ifdef __cplusplus
}
#endif
#endif /* EDAA_B200_H */
