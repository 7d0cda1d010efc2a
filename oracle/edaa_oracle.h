/* TEST INFRASTRUCTURE ONLY — the CPU oracle for the EDAA hot path.
 *
 * A plain-C restatement of the reference's Algorithm 1 (solver) and
 * Algorithm 2 (ensemble + model selection), written to reproduce the
 * reference's floating-point operation order exactly so that, on the same
 * fp64 inputs, it agrees BITWISE with the reference built from source
 * (oracle/_ref/liboracle_ref.so).  That bitwise agreement is checked in
 * tests/test_oracle.py, together with the golden vectors of the
 * reference's own unit tests (test_core.cpp, test_solver.cpp,
 * test_ensemble.cpp).
 *
 * Only tests/, __graft_entry__.smoke() and bench.py (cpu_baseline and the
 * --impl reference arm) may load this library.  It is never part of the
 * product path: the product fails loudly without its CUDA library.
 *
 * All matrices are dense row-major fp64, shapes as in the reference:
 * X L×N, A p×N, B N×p, E L×p.  Return value: 0 ok, else an error code and
 * the reference's message in err.
 */
#ifndef EDAA_ORACLE_H
#define EDAA_ORACLE_H
#include <stddef.h>
#include <stdint.h>
#ifdef __cplusplus
extern "C" {
#endif

/* HsiImage::validate + l2_normalize, image.cpp:10-47 (zero pixels listed, left as is) */
int orc_l2_normalize(const double* x, size_t l, size_t n, double* out, size_t* zero, size_t* n_zero,
                     char* err, size_t errlen);

/* SplitMix64, prng.hpp:15-26 */
uint64_t orc_splitmix_next(uint64_t* state);
double orc_splitmix_unit(uint64_t* state);

/* solver.cpp:118-136 */
int orc_init_contributions(size_t n, size_t p, uint64_t* state, double* b);
/* matrix.cpp:150-190 */
int orc_spectral_norm(const double* m, size_t rows, size_t cols, double tol, size_t max_iters,
                      double* out, char* err, size_t errlen);
/* solver.cpp:138-149 */
int orc_step_sizes(const double* x, size_t l, size_t n, const double* b0, size_t p, double gamma,
                   double* eta_a, double* eta_b, char* err, size_t errlen);
/* solver.cpp:151-164 (with the strided apply of solver.cpp:20-36) */
int orc_entropic_step(const double* z, const double* g, size_t d, double eta, double* out,
                      char* err, size_t errlen);
/* solver.cpp:190-238 */
int orc_run(const double* x, size_t l, size_t n, size_t p, size_t t_outer, size_t k1, size_t k2,
            double gamma, uint64_t seed, double* trace, double* a, double* b, double* e,
            double* fit, double* mu, char* err, size_t errlen);
/* ensemble.cpp:29-39 */
double orc_fit_l1(const double* x, size_t l, size_t n, const double* e, size_t p, const double* a);
/* ensemble.cpp:41-60 */
double orc_coherence(const double* e, size_t l, size_t p, int normalized);
/* ensemble.cpp:62-69 */
double orc_sample_gamma(uint64_t* state, const double* set, size_t n_set);
/* ensemble.cpp:71-94 */
int orc_select_runs(size_t m, const double* fit, const double* mu, const uint8_t* ok,
                    double fit_slack, uint8_t* cand, size_t* selected, double* fit_min,
                    char* err, size_t errlen);
/* ensemble.cpp:108-167; workers threads claim runs from a shared counter. */
int orc_run_ensemble(const double* x, size_t l, size_t n, size_t p, size_t t_outer, size_t k1,
                     size_t k2, size_t runs, uint64_t base_seed, const double* gamma_set,
                     size_t n_gamma, double fit_slack, unsigned workers, uint64_t* rec_seed,
                     double* rec_gamma, double* rec_fit, double* rec_mu, uint8_t* rec_ok,
                     uint8_t* cand, size_t* selected, double* fit_min, double* trace, double* a,
                     double* b, double* e, char* err, size_t errlen);

#ifdef __cplusplus
}
#endif
#endif
