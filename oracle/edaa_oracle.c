/* TEST INFRASTRUCTURE ONLY — see edaa_oracle.h.
 *
 * Plain-C restatement of the reference EDAA hot path.  Each function names
 * the reference lines it follows; the floating-point operation ORDER of every
 * reduction is kept (ascending inner index, separate multiply and add,
 * compiled with -ffp-contract=off) so results match the reference bitwise.
 */
#include "edaa_oracle.h"

#include <math.h>
#include <pthread.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#define ORC_LOG_FLOOR 1e-30 /* solver.cpp:15 */

static int fail(char* err, size_t errlen, const char* msg) {
  if (err && errlen) {
    strncpy(err, msg, errlen - 1);
    err[errlen - 1] = '\0';
  }
  return 1;
}

/* ---- PRNG: prng.hpp:15-26 ------------------------------------------------ */
uint64_t orc_splitmix_next(uint64_t* state) {
  *state += 0x9E3779B97F4A7C15ULL;
  uint64_t z = *state;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}

double orc_splitmix_unit(uint64_t* state) {
  return (double)(orc_splitmix_next(state) >> 11) * 0x1.0p-53;
}

/* ---- dense products in the reference's accumulation order ---------------- */
/* c(m×q) = a(m×k)·b(k×q); matrix.cpp:64-73,77-95 (k ascending per row). */
static void mat_ab(const double* a, size_t m, size_t k, const double* b, size_t q, double* c) {
  for (size_t i = 0; i < m; ++i) {
    double* cr = c + i * q;
    for (size_t j = 0; j < q; ++j) cr[j] = 0.0;
    for (size_t kk = 0; kk < k; ++kk) {
      const double aik = a[i * k + kk];
      const double* br = b + kk * q;
      for (size_t j = 0; j < q; ++j) cr[j] += aik * br[j];
    }
  }
}

/* c(m×q) = aᵀ·b with a(k×m), b(k×q); matrix.cpp:97-112. */
static void mat_atb(const double* a, size_t k, size_t m, const double* b, size_t q, double* c) {
  for (size_t i = 0; i < m * q; ++i) c[i] = 0.0;
  for (size_t i = 0; i < m; ++i) {
    double* cr = c + i * q;
    for (size_t kk = 0; kk < k; ++kk) {
      const double aki = a[kk * m + i];
      const double* br = b + kk * q;
      for (size_t j = 0; j < q; ++j) cr[j] += aki * br[j];
    }
  }
}

/* c(m×q) = a·bᵀ with a(m×k), b(q×k); matrix.cpp:114-131. */
static void mat_abt(const double* a, size_t m, size_t k, const double* b, size_t q, double* c) {
  for (size_t i = 0; i < m; ++i)
    for (size_t j = 0; j < q; ++j) {
      double s = 0.0;
      for (size_t kk = 0; kk < k; ++kk) s += a[i * k + kk] * b[j * k + kk];
      c[i * q + j] = s;
    }
}

/* r = x − y·a, the materialised residual of solver.cpp:53-55 (matmul then
 * subtract, matrix.cpp:140-148). tmp holds y·a. */
static void residual(const double* x, const double* y, const double* a, size_t l, size_t n,
                     size_t p, double* tmp, double* r) {
  mat_ab(y, l, p, a, n, tmp);
  for (size_t i = 0; i < l * n; ++i) r[i] = x[i] - tmp[i];
}

static double half_sq(const double* r, size_t count) { /* solver.cpp:57-61 */
  double s = 0.0;
  for (size_t i = 0; i < count; ++i) s += r[i] * r[i];
  return 0.5 * s;
}

static double frob(const double* m, size_t count) { /* matrix.cpp:20-24 */
  double s = 0.0;
  for (size_t i = 0; i < count; ++i) s += m[i] * m[i];
  return sqrt(s);
}

/* ---- spectral norm: matrix.cpp:150-190 ------------------------------------ */
int orc_spectral_norm(const double* m, size_t rows, size_t cols, double tol, size_t max_iters,
                      double* out, char* err, size_t errlen) {
  const char* bad = "spectral_norm: matrix must be finite and nonzero";
  if (rows * cols == 0) return fail(err, errlen, bad);
  for (size_t i = 0; i < rows * cols; ++i)
    if (!isfinite(m[i])) return fail(err, errlen, bad);
  if (frob(m, rows * cols) == 0.0) return fail(err, errlen, bad);
  const size_t p = cols;
  double* gram = malloc(sizeof(double) * p * p);
  double* v = malloc(sizeof(double) * p);
  double* gv = malloc(sizeof(double) * p);
  mat_atb(m, rows, p, m, p, gram);
  for (size_t i = 0; i < p; ++i) v[i] = 1.0 / sqrt((double)p);
  double lambda = 0.0;
  const double stop = tol / 16.0;
  int rc = 1;
  for (size_t it = 0; it < max_iters; ++it) {
    for (size_t i = 0; i < p; ++i) {
      double s = 0.0;
      for (size_t j = 0; j < p; ++j) s += gram[i * p + j] * v[j];
      gv[i] = s;
    }
    double next = 0.0;
    for (size_t i = 0; i < p; ++i) next += v[i] * gv[i];
    double norm = 0.0;
    for (size_t i = 0; i < p; ++i) norm += gv[i] * gv[i];
    norm = sqrt(norm);
    if (norm == 0.0) { /* all-ones start in the null space: unit vector it%p */
      for (size_t i = 0; i < p; ++i) v[i] = 0.0;
      v[it % p] = 1.0;
      continue;
    }
    for (size_t i = 0; i < p; ++i) v[i] = gv[i] / norm;
    if (it > 0 && fabs(next - lambda) <= stop * fabs(next)) {
      *out = sqrt(next);
      rc = 0;
      break;
    }
    lambda = next;
  }
  if (rc) {
    char msg[160];
    snprintf(msg, sizeof msg, "spectral_norm: no convergence after %zu iterations; best estimate %g",
             max_iters, sqrt(fabs(lambda)));
    fail(err, errlen, msg);
  }
  free(gram);
  free(v);
  free(gv);
  return rc;
}

/* ---- initialisation: solver.cpp:113-136 ----------------------------------- */
int orc_init_contributions(size_t n, size_t p, uint64_t* state, double* b) {
  double* sc = malloc(sizeof(double) * n);
  for (size_t j = 0; j < p; ++j) { /* column j consumes draws j·n .. j·n+n-1 */
    double top = -INFINITY;
    for (size_t i = 0; i < n; ++i) {
      sc[i] = 0.1 * orc_splitmix_unit(state);
      top = (top < sc[i]) ? sc[i] : top;
    }
    double total = 0.0;
    for (size_t i = 0; i < n; ++i) {
      sc[i] = exp(sc[i] - top);
      total += sc[i];
    }
    for (size_t i = 0; i < n; ++i) b[i * p + j] = sc[i] / total;
  }
  free(sc);
  return 0;
}

int orc_step_sizes(const double* x, size_t l, size_t n, const double* b0, size_t p, double gamma,
                   double* eta_a, double* eta_b, char* err, size_t errlen) {
  if (!(gamma > 0.0)) return fail(err, errlen, "step_sizes: gamma must be positive");
  double* xb = malloc(sizeof(double) * l * p);
  mat_ab(x, l, n, b0, p, xb);
  int rc = 0;
  double sigma = 0.0;
  if (frob(xb, l * p) == 0.0)
    rc = fail(err, errlen, "degenerate initialization: X\xc2\xb7" "B0 is zero");
  else
    rc = orc_spectral_norm(xb, l, p, 1e-6, 1000, &sigma, err, errlen);
  free(xb);
  if (rc) return rc;
  *eta_a = gamma / (sigma * sigma);
  *eta_b = sqrt((double)p / (double)n) * *eta_a;
  return 0;
}

/* ---- entropic update: solver.cpp:20-46,151-164 ----------------------------- */
static void entropic_apply(double* z, size_t zs, const double* step, size_t ss, size_t d,
                           double* scratch) {
  double top = -INFINITY;
  for (size_t i = 0; i < d; ++i) {
    const double zi = z[i * zs] > ORC_LOG_FLOOR ? z[i * zs] : ORC_LOG_FLOOR;
    const double s = log(zi) + step[i * ss];
    scratch[i] = s;
    top = (top < s) ? s : top; /* std::max(top, s) */
  }
  double total = 0.0;
  for (size_t i = 0; i < d; ++i) {
    scratch[i] = exp(scratch[i] - top);
    total += scratch[i];
  }
  for (size_t i = 0; i < d; ++i) z[i * zs] = scratch[i] / total;
}

int orc_entropic_step(const double* z, const double* g, size_t d, double eta, double* out,
                      char* err, size_t errlen) {
  if (d == 0) return fail(err, errlen, "entropic_step: size mismatch");
  if (!(eta > 0.0) || !isfinite(eta)) return fail(err, errlen, "entropic_step: eta must be positive");
  double* step = malloc(sizeof(double) * d * 2);
  for (size_t i = 0; i < d; ++i) {
    if (!isfinite(g[i])) {
      free(step);
      return fail(err, errlen, "entropic_step: non-finite gradient");
    }
    step[i] = -eta * g[i];
  }
  memcpy(out, z, sizeof(double) * d);
  entropic_apply(out, 1, step, 1, d, step + d);
  free(step);
  return 0;
}

/* check_iterate, solver.cpp:65-90: columns of the d×cols matrix m. */
static int check_iterate(const double* m, size_t d, size_t cols, size_t outer, const char* which,
                         char* err, size_t errlen) {
  char msg[160];
  for (size_t j = 0; j < cols; ++j) {
    double sum = 0.0;
    for (size_t i = 0; i < d; ++i) {
      const double v = m[i * cols + j];
      if (!isfinite(v)) {
        snprintf(msg, sizeof msg, "non-finite %s iterate at outer iteration %zu", which, outer);
        return fail(err, errlen, msg);
      }
      if (v < 0.0) {
        snprintf(msg, sizeof msg, "%s iterate left the simplex at outer iteration %zu", which, outer);
        return fail(err, errlen, msg);
      }
      sum += v;
    }
    if (fabs(sum - 1.0) > 1e-9) {
      snprintf(msg, sizeof msg, "%s column sum drifted from 1 at outer iteration %zu", which, outer);
      return fail(err, errlen, msg);
    }
  }
  return 0;
}

/* ---- ingest: image.cpp:10-47 ------------------------------------------------ */
int orc_l2_normalize(const double* x, size_t l, size_t n, double* out, size_t* zero, size_t* n_zero,
                     char* err, size_t errlen) {
  /* HsiImage::validate: the first offending value in row-major order decides */
  if (l < 1 || n < 1) return fail(err, errlen, "image: needs at least one band and one pixel");
  for (size_t k = 0; k < l * n; ++k) {
    if (!isfinite(x[k])) return fail(err, errlen, "image: non-finite reflectance");
    if (x[k] < 0.0) return fail(err, errlen, "image: negative reflectance");
  }
  size_t nz = 0;
  int any = 0;
  for (size_t j = 0; j < n; ++j) {
    double s = 0.0; /* Matrix::column_norm, matrix.cpp:44-51 */
    for (size_t i = 0; i < l; ++i) {
      const double v = x[i * n + j];
      s += v * v;
    }
    const double norm = sqrt(s);
    if (norm == 0.0) {
      zero[nz++] = j;
      for (size_t i = 0; i < l; ++i) out[i * n + j] = x[i * n + j];
      continue;
    }
    any = 1;
    for (size_t i = 0; i < l; ++i) out[i * n + j] = x[i * n + j] / norm;
  }
  *n_zero = nz;
  if (!any) return fail(err, errlen, "degenerate input: all pixels are zero");
  return 0;
}

/* ---- Algorithm 1: solver.cpp:190-238 -------------------------------------- */
int orc_run(const double* x, size_t l, size_t n, size_t p, size_t t_outer, size_t k1, size_t k2,
            double gamma, uint64_t seed, double* trace, double* a_out, double* b_out,
            double* e_out, double* fit, double* mu, char* err, size_t errlen) {
  /* SolverConfig::validate, solver.cpp:103-111 */
  if (p < 2) return fail(err, errlen, "solver config: endmember count must be at least 2");
  if (t_outer < 1 || k1 < 1 || k2 < 1)
    return fail(err, errlen, "solver config: iteration counts must be at least 1");
  if (!(gamma > 0.0) || !isfinite(gamma))
    return fail(err, errlen, "solver config: step factor gamma must be positive");
  /* HsiImage::validate, image.cpp:10-27 (matrix part) */
  if (l < 1 || n < 1) return fail(err, errlen, "image: needs at least one band and one pixel");
  for (size_t i = 0; i < l * n; ++i) {
    if (!isfinite(x[i])) return fail(err, errlen, "image: non-finite reflectance");
    if (x[i] < 0.0) return fail(err, errlen, "image: negative reflectance");
  }
  double* a = malloc(sizeof(double) * p * n);
  double* b = malloc(sizeof(double) * n * p);
  double* xb = malloc(sizeof(double) * l * p);
  double* tmp = malloc(sizeof(double) * l * n);
  double* r = malloc(sizeof(double) * l * n);
  double* ga = malloc(sizeof(double) * p * n);
  double* gb = malloc(sizeof(double) * n * p);
  double* rat = malloc(sizeof(double) * l * p);
  double* scratch = malloc(sizeof(double) * (n > p ? n : p));
  int rc = 0;
  for (size_t i = 0; i < p * n; ++i) a[i] = 1.0 / (double)p;
  uint64_t st = seed;
  orc_init_contributions(n, p, &st, b);
  double eta_a = 0.0, eta_b = 0.0;
  rc = orc_step_sizes(x, l, n, b, p, gamma, &eta_a, &eta_b, err, errlen);
  if (rc) goto done;
  mat_ab(x, l, n, b, p, xb);
  residual(x, xb, a, l, n, p, tmp, r);
  if (trace) trace[0] = half_sq(r, l * n);
  for (size_t t = 1; t <= t_outer; ++t) {
    for (size_t k = 1; k <= k1; ++k) { /* A block, xb fixed: solver.cpp:212-218 */
      residual(x, xb, a, l, n, p, tmp, r);
      mat_atb(xb, l, p, r, n, ga);
      for (size_t i = 0; i < p * n; ++i) ga[i] *= eta_a;
      for (size_t j = 0; j < n; ++j) entropic_apply(a + j, n, ga + j, n, p, scratch);
      rc = check_iterate(a, p, n, t, "abundance", err, errlen);
      if (rc) goto done;
    }
    for (size_t k = 1; k <= k2; ++k) { /* B block: solver.cpp:219-227 */
      if (k > 1) mat_ab(x, l, n, b, p, xb);
      residual(x, xb, a, l, n, p, tmp, r);
      mat_abt(r, l, n, a, p, rat);
      mat_atb(x, l, n, rat, p, gb);
      for (size_t i = 0; i < n * p; ++i) gb[i] *= eta_b;
      for (size_t j = 0; j < p; ++j) entropic_apply(b + j, p, gb + j, p, n, scratch);
      rc = check_iterate(b, n, p, t, "contribution", err, errlen);
      if (rc) goto done;
    }
    mat_ab(x, l, n, b, p, xb);
    residual(x, xb, a, l, n, p, tmp, r);
    if (trace) trace[t] = half_sq(r, l * n);
  }
  if (a_out) memcpy(a_out, a, sizeof(double) * p * n);
  if (b_out) memcpy(b_out, b, sizeof(double) * n * p);
  if (e_out) memcpy(e_out, xb, sizeof(double) * l * p);
  if (fit) *fit = orc_fit_l1(x, l, n, xb, p, a);
  if (mu) *mu = orc_coherence(xb, l, p, 0);
done:
  free(a); free(b); free(xb); free(tmp); free(r); free(ga); free(gb); free(rat); free(scratch);
  return rc;
}

/* ---- model-selection primitives: ensemble.cpp:29-94 ----------------------- */
double orc_fit_l1(const double* x, size_t l, size_t n, const double* e, size_t p, const double* a) {
  double* recon = malloc(sizeof(double) * l * n);
  mat_ab(e, l, p, a, n, recon);
  double total = 0.0;
  for (size_t i = 0; i < l * n; ++i) total += fabs(x[i] - recon[i]);
  free(recon);
  return total;
}

double orc_coherence(const double* e, size_t l, size_t p, int normalized) {
  if (p < 2) return 0.0;
  double best = -INFINITY;
  for (size_t i = 0; i < p; ++i)
    for (size_t j = i + 1; j < p; ++j) {
      double dot = 0.0;
      for (size_t r = 0; r < l; ++r) dot += e[r * p + i] * e[r * p + j];
      if (normalized) {
        double ni = 0.0, nj = 0.0;
        for (size_t r = 0; r < l; ++r) ni += e[r * p + i] * e[r * p + i];
        for (size_t r = 0; r < l; ++r) nj += e[r * p + j] * e[r * p + j];
        ni = sqrt(ni);
        nj = sqrt(nj);
        if (ni == 0.0 || nj == 0.0) continue;
        dot /= ni * nj;
      }
      if (dot > best) best = dot;
    }
  return best == -INFINITY ? 0.0 : best;
}

double orc_sample_gamma(uint64_t* state, const double* set, size_t n_set) {
  size_t idx = (size_t)(orc_splitmix_unit(state) * (double)n_set);
  if (idx > n_set - 1) idx = n_set - 1;
  return set[idx];
}

int orc_select_runs(size_t m, const double* fit, const double* mu, const uint8_t* ok,
                    double fit_slack, uint8_t* cand, size_t* selected, double* fit_min,
                    char* err, size_t errlen) {
  double fmin = INFINITY;
  for (size_t i = 0; i < m; ++i)
    if (ok[i] && fit[i] < fmin) fmin = fit[i];
  if (fmin == INFINITY) return fail(err, errlen, "every run failed");
  *fit_min = fmin;
  const double cutoff = fit_slack * fmin;
  size_t best = (size_t)-1;
  for (size_t i = 0; i < m; ++i) {
    cand[i] = (uint8_t)(ok[i] && fit[i] <= cutoff);
    if (cand[i] && (best == (size_t)-1 || mu[i] < mu[best])) best = i;
  }
  *selected = best;
  return 0;
}

/* ---- Algorithm 2: ensemble.cpp:108-167 ------------------------------------ */
typedef struct {
  const double* x;
  size_t l, n, p, t_outer, k1, k2, runs;
  uint64_t base_seed;
  const double* gamma_set;
  size_t n_gamma;
  double* fits;
  double* mus;
  double* gammas;
  uint8_t* oks;
  double* traces; /* runs × (T+1) */
  double* as;     /* runs × p×N */
  double* bs;     /* runs × N×p */
  double* es;     /* runs × L×p */
  size_t next;
  pthread_mutex_t lock;
} ens_job;

static void ens_one(ens_job* J, size_t m) {
  uint64_t st = J->base_seed + m;
  const double gamma = orc_sample_gamma(&st, J->gamma_set, J->n_gamma);
  J->gammas[m] = gamma;
  char err[256];
  const int rc = orc_run(J->x, J->l, J->n, J->p, J->t_outer, J->k1, J->k2, gamma, J->base_seed + m,
                         J->traces + m * (J->t_outer + 1), J->as + m * J->p * J->n,
                         J->bs + m * J->n * J->p, J->es + m * J->l * J->p, &J->fits[m], &J->mus[m],
                         err, sizeof err);
  J->oks[m] = rc == 0;
}

static void* ens_worker(void* arg) {
  ens_job* J = arg;
  for (;;) {
    pthread_mutex_lock(&J->lock);
    const size_t m = J->next++;
    pthread_mutex_unlock(&J->lock);
    if (m >= J->runs) return NULL;
    ens_one(J, m);
  }
}

int orc_run_ensemble(const double* x, size_t l, size_t n, size_t p, size_t t_outer, size_t k1,
                     size_t k2, size_t runs, uint64_t base_seed, const double* gamma_set,
                     size_t n_gamma, double fit_slack, unsigned workers, uint64_t* rec_seed,
                     double* rec_gamma, double* rec_fit, double* rec_mu, uint8_t* rec_ok,
                     uint8_t* cand, size_t* selected, double* fit_min, double* trace, double* a,
                     double* b, double* e, char* err, size_t errlen) {
  /* EnsembleConfig::validate, ensemble.cpp:17-27 */
  if (runs == 0) return fail(err, errlen, "ensemble needs at least one run");
  if (n_gamma == 0) return fail(err, errlen, "step factor set is empty");
  for (size_t i = 0; i < n_gamma; ++i)
    if (!isfinite(gamma_set[i]) || gamma_set[i] <= 0.0)
      return fail(err, errlen, "step factors must be finite and positive");
  if (!isfinite(fit_slack) || fit_slack < 1.0) return fail(err, errlen, "fit slack must be at least 1");
  if (p < 2) return fail(err, errlen, "solver config: endmember count must be at least 2");
  if (t_outer < 1 || k1 < 1 || k2 < 1)
    return fail(err, errlen, "solver config: iteration counts must be at least 1");
  /* solver.gamma of the template is overwritten per run; its default 1.0 passes */
  if (l < 1 || n < 1) return fail(err, errlen, "image: needs at least one band and one pixel");
  for (size_t i = 0; i < l * n; ++i) {
    if (!isfinite(x[i])) return fail(err, errlen, "image: non-finite reflectance");
    if (x[i] < 0.0) return fail(err, errlen, "image: negative reflectance");
  }
  ens_job J = {x, l, n, p, t_outer, k1, k2, runs, base_seed, gamma_set, n_gamma};
  J.fits = calloc(runs, sizeof(double));
  J.mus = calloc(runs, sizeof(double));
  J.gammas = calloc(runs, sizeof(double));
  J.oks = calloc(runs, 1);
  J.traces = malloc(sizeof(double) * runs * (t_outer + 1));
  J.as = malloc(sizeof(double) * runs * p * n);
  J.bs = malloc(sizeof(double) * runs * n * p);
  J.es = malloc(sizeof(double) * runs * l * p);
  pthread_mutex_init(&J.lock, NULL);
  if (workers == 0) workers = 1;
  if (workers > runs) workers = (unsigned)runs;
  if (workers <= 1) {
    for (size_t m = 0; m < runs; ++m) ens_one(&J, m);
  } else {
    pthread_t* th = malloc(sizeof(pthread_t) * workers);
    for (unsigned w = 0; w < workers; ++w) pthread_create(&th[w], NULL, ens_worker, &J);
    for (unsigned w = 0; w < workers; ++w) pthread_join(th[w], NULL);
    free(th);
  }
  uint8_t* cmask = cand ? cand : calloc(runs, 1);
  size_t sel = 0;
  double fmin = 0.0;
  int rc = orc_select_runs(runs, J.fits, J.mus, J.oks, fit_slack, cmask, &sel, &fmin, err, errlen);
  if (rc == 0) {
    for (size_t m = 0; m < runs; ++m) {
      if (rec_seed) rec_seed[m] = base_seed + m;
      if (rec_gamma) rec_gamma[m] = J.gammas[m];
      if (rec_fit) rec_fit[m] = J.oks[m] ? J.fits[m] : 0.0;
      if (rec_mu) rec_mu[m] = J.oks[m] ? J.mus[m] : 0.0;
      if (rec_ok) rec_ok[m] = J.oks[m];
    }
    if (selected) *selected = sel;
    if (fit_min) *fit_min = fmin;
    if (trace) memcpy(trace, J.traces + sel * (t_outer + 1), sizeof(double) * (t_outer + 1));
    if (a) memcpy(a, J.as + sel * p * n, sizeof(double) * p * n);
    if (b) memcpy(b, J.bs + sel * n * p, sizeof(double) * n * p);
    if (e) memcpy(e, J.es + sel * l * p, sizeof(double) * l * p);
  }
  if (!cand) free(cmask);
  free(J.fits); free(J.mus); free(J.gammas); free(J.oks);
  free(J.traces); free(J.as); free(J.bs); free(J.es);
  pthread_mutex_destroy(&J.lock);
  return rc;
}
