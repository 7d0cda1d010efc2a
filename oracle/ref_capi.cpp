// TEST INFRASTRUCTURE ONLY — never linked into the product.
//
// extern "C" veneer over the UNMODIFIED reference C++ sources
// (/root/reference/proj/src/{matrix,image,types,solver,ensemble}.cpp), compiled
// by oracle/Makefile into oracle/_ref/liboracle_ref.so with
// -Darchetype=archetype_ref so its symbols cannot collide with the drop-in
// shim that re-implements the same C++ API on the GPU.
//
// Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
// --impl reference legs may load this library (as the checker / the CPU
// baseline), never the product path.
//
// Every entry point returns 0 on success and 1 when the reference threw
// archetype::Error (message copied into err[0..errlen)).
#include <algorithm>
#include <cstdint>
#include <cstring>
#include <exception>
#include <string>
#include <vector>

#include "archetype/ensemble.hpp"
#include "archetype/error.hpp"
#include "archetype/image.hpp"
#include "archetype/matrix.hpp"
#include "archetype/prng.hpp"
#include "archetype/solver.hpp"

// solver.cpp is compiled as part of THIS translation unit (included in place
// from /root/reference by the Makefile's -DREF_SOLVER_CPP, never copied), so
// the veneer can also reach its anonymous-namespace helpers — check_iterate
// (solver.cpp:65-90), the per-iterate simplex check that the drop-in's device
// checks must reproduce message for message.
#include REF_SOLVER_CPP

namespace ar = archetype;  // renamed to archetype_ref by the Makefile

namespace {

void put_err(const std::exception& e, char* err, size_t errlen) {
  if (!err || errlen == 0) return;
  std::strncpy(err, e.what(), errlen - 1);
  err[errlen - 1] = '\0';
}

ar::HsiImage make_image(const double* x, size_t l, size_t n) {
  ar::HsiImage img;
  img.data = ar::Matrix(l, n);
  std::copy(x, x + l * n, img.data.values().begin());
  return img;
}

void copy_out(const ar::Matrix& m, double* dst) {
  if (dst) std::copy(m.values().begin(), m.values().end(), dst);
}

void copy_result(const ar::RunResult& r, double* trace, double* a, double* b, double* e,
                 double* fit, double* mu) {
  if (trace) std::copy(r.objective_trace.begin(), r.objective_trace.end(), trace);
  copy_out(r.abundances.data, a);
  copy_out(r.contributions.data, b);
  copy_out(r.endmembers.data, e);
  if (fit) *fit = r.fit_l1;
  if (mu) *mu = r.coherence;
}

}  // namespace

extern "C" {

// l2_normalize (image.cpp:29-47), validation included. out: L×N; zero: up to n entries.
int oref_l2_normalize(const double* x, size_t l, size_t n, double* out, size_t* zero, size_t* n_zero,
                      char* err, size_t errlen) {
  try {
    ar::HsiImage img = make_image(x, l, n);
    const ar::NormalizeResult r = ar::l2_normalize(img);
    copy_out(r.image.data, out);
    *n_zero = r.zero_pixels.size();
    std::copy(r.zero_pixels.begin(), r.zero_pixels.end(), zero);
    return 0;
  } catch (const std::exception& e) {
    put_err(e, err, errlen);
    return 1;
  }
}

int oref_prng_u64(uint64_t seed, size_t count, uint64_t* out) {
  ar::Prng rng(seed);
  for (size_t i = 0; i < count; ++i) out[i] = rng.next_u64();
  return 0;
}

int oref_prng_unit(uint64_t seed, size_t count, double* out) {
  ar::Prng rng(seed);
  for (size_t i = 0; i < count; ++i) out[i] = rng.next_unit();
  return 0;
}

// run(): solver.cpp:190-238. trace has T+1 entries; a p×N, b N×p, e L×p.
int oref_run(const double* x, size_t l, size_t n, size_t p, size_t t_outer, size_t k1,
             size_t k2, double gamma, uint64_t seed, double* trace, double* a, double* b,
             double* e, double* fit, double* mu, char* err, size_t errlen) {
  try {
    ar::SolverConfig cfg;
    cfg.endmembers = p;
    cfg.outer_iters = t_outer;
    cfg.inner_iters_a = k1;
    cfg.inner_iters_b = k2;
    cfg.gamma = gamma;
    cfg.seed = seed;
    const ar::RunResult r = ar::run(make_image(x, l, n), cfg);
    copy_result(r, trace, a, b, e, fit, mu);
    return 0;
  } catch (const std::exception& ex) {
    put_err(ex, err, errlen);
    return 1;
  }
}

// Same as oref_run but records every inner iterate through the reference's
// StepObserver: snapshots laid out [T·(K1+K2)][p·N + N·p] (A then B).
int oref_run_observed(const double* x, size_t l, size_t n, size_t p, size_t t_outer, size_t k1,
                      size_t k2, double gamma, uint64_t seed, double* snaps, char* blocks,
                      double* trace, char* err, size_t errlen) {
  try {
    ar::SolverConfig cfg;
    cfg.endmembers = p;
    cfg.outer_iters = t_outer;
    cfg.inner_iters_a = k1;
    cfg.inner_iters_b = k2;
    cfg.gamma = gamma;
    cfg.seed = seed;
    size_t idx = 0;
    const size_t stride = 2 * p * n;
    const ar::RunResult r = ar::run(make_image(x, l, n), cfg, [&](const ar::InnerStep& s) {
      double* dst = snaps + idx * stride;
      std::copy(s.abundances.values().begin(), s.abundances.values().end(), dst);
      std::copy(s.contributions.values().begin(), s.contributions.values().end(), dst + p * n);
      if (blocks) blocks[idx] = s.block;
      ++idx;
    });
    if (trace) std::copy(r.objective_trace.begin(), r.objective_trace.end(), trace);
    return 0;
  } catch (const std::exception& ex) {
    put_err(ex, err, errlen);
    return 1;
  }
}

// run_ensemble(): ensemble.cpp:108-167. Per-run records go to the rec_* arrays
// (length M); the selected run's factors to trace/a/b/e. cand is an M-byte
// mask of the candidate set.
int oref_run_ensemble(const double* x, size_t l, size_t n, size_t p, size_t t_outer, size_t k1,
                      size_t k2, size_t runs, uint64_t base_seed, const double* gamma_set,
                      size_t n_gamma, double fit_slack, unsigned workers, uint64_t* rec_seed,
                      double* rec_gamma, double* rec_fit, double* rec_mu, uint8_t* rec_ok,
                      uint8_t* cand, size_t* selected, double* fit_min, double* trace, double* a,
                      double* b, double* e, char* err, size_t errlen) {
  try {
    ar::EnsembleConfig cfg;
    cfg.runs = runs;
    cfg.base_seed = base_seed;
    cfg.gamma_set.assign(gamma_set, gamma_set + n_gamma);
    cfg.fit_slack = fit_slack;
    cfg.solver.endmembers = p;
    cfg.solver.outer_iters = t_outer;
    cfg.solver.inner_iters_a = k1;
    cfg.solver.inner_iters_b = k2;
    cfg.workers = workers;
    const auto [res, rep] = ar::run_ensemble(make_image(x, l, n), cfg);
    for (size_t m = 0; m < runs; ++m) {
      const ar::RunRecord& rr = rep.per_run[m];
      if (rec_seed) rec_seed[m] = rr.seed;
      if (rec_gamma) rec_gamma[m] = rr.gamma;
      if (rec_fit) rec_fit[m] = rr.fit_l1;
      if (rec_mu) rec_mu[m] = rr.coherence;
      if (rec_ok) rec_ok[m] = rr.ok ? 1 : 0;
      if (cand) cand[m] = 0;
    }
    if (cand)
      for (size_t c : rep.candidate_set) cand[c] = 1;
    if (selected) *selected = rep.selected;
    if (fit_min) *fit_min = rep.fit_min;
    copy_result(res, trace, a, b, e, nullptr, nullptr);
    return 0;
  } catch (const std::exception& ex) {
    put_err(ex, err, errlen);
    return 1;
  }
}

int oref_select_runs(size_t m, const double* fit, const double* mu, const uint8_t* ok,
                     double fit_slack, uint8_t* cand, size_t* selected, double* fit_min,
                     char* err, size_t errlen) {
  try {
    std::vector<ar::RunRecord> recs(m);
    for (size_t i = 0; i < m; ++i) {
      recs[i].index = i;
      recs[i].fit_l1 = fit[i];
      recs[i].coherence = mu[i];
      recs[i].ok = ok[i] != 0;
    }
    const ar::SelectionReport rep = ar::select_runs(recs, fit_slack);
    for (size_t i = 0; i < m; ++i) cand[i] = 0;
    for (size_t c : rep.candidate_set) cand[c] = 1;
    *selected = rep.selected;
    *fit_min = rep.fit_min;
    return 0;
  } catch (const std::exception& ex) {
    put_err(ex, err, errlen);
    return 1;
  }
}

int oref_init_contributions(size_t n, size_t p, uint64_t seed, double* b, char* err,
                            size_t errlen) {
  try {
    ar::Prng rng(seed);
    copy_out(ar::init_contributions(n, p, rng).data, b);
    return 0;
  } catch (const std::exception& ex) {
    put_err(ex, err, errlen);
    return 1;
  }
}

int oref_step_sizes(const double* x, size_t l, size_t n, const double* b0, size_t p,
                    double gamma, double* eta_a, double* eta_b, char* err, size_t errlen) {
  try {
    ar::ContributionMatrix b{ar::Matrix(n, p)};
    std::copy(b0, b0 + n * p, b.data.values().begin());
    const ar::StepSizes s = ar::step_sizes(make_image(x, l, n), b, gamma);
    *eta_a = s.eta_a;
    *eta_b = s.eta_b;
    return 0;
  } catch (const std::exception& ex) {
    put_err(ex, err, errlen);
    return 1;
  }
}

int oref_spectral_norm(const double* m, size_t rows, size_t cols, double tol, size_t max_iters,
                       double* out, char* err, size_t errlen) {
  try {
    ar::Matrix mm(rows, cols);
    std::copy(m, m + rows * cols, mm.values().begin());
    *out = ar::spectral_norm(mm, tol, max_iters);
    return 0;
  } catch (const std::exception& ex) {
    put_err(ex, err, errlen);
    return 1;
  }
}

int oref_entropic_step(const double* z, const double* g, size_t d, double eta, double* out,
                       char* err, size_t errlen) {
  try {
    const std::vector<double> r =
        ar::entropic_step(std::span<const double>(z, d), std::span<const double>(g, d), eta);
    std::copy(r.begin(), r.end(), out);
    return 0;
  } catch (const std::exception& ex) {
    put_err(ex, err, errlen);
    return 1;
  }
}

int oref_fit_l1(const double* x, size_t l, size_t n, const double* e, size_t p, const double* a,
                double* out, char* err, size_t errlen) {
  try {
    ar::EndmemberMatrix em{ar::Matrix(l, p)};
    std::copy(e, e + l * p, em.data.values().begin());
    ar::AbundanceMatrix am{ar::Matrix(p, n)};
    std::copy(a, a + p * n, am.data.values().begin());
    *out = ar::fit_l1(make_image(x, l, n), em, am);
    return 0;
  } catch (const std::exception& ex) {
    put_err(ex, err, errlen);
    return 1;
  }
}

int oref_coherence(const double* e, size_t l, size_t p, int normalized, double* out) {
  ar::EndmemberMatrix em{ar::Matrix(l, p)};
  std::copy(e, e + l * p, em.data.values().begin());
  *out = ar::coherence(em, normalized != 0);
  return 0;
}

int oref_sample_gamma(uint64_t seed, const double* set, size_t n_set, size_t draws,
                      double* out, char* err, size_t errlen) {
  try {
    ar::Prng rng(seed);
    const std::vector<double> s(set, set + n_set);
    for (size_t i = 0; i < draws; ++i) out[i] = ar::sample_gamma(rng, s);
    return 0;
  } catch (const std::exception& ex) {
    put_err(ex, err, errlen);
    return 1;
  }
}

// grad_abundances / grad_contributions / objective_l2 (solver.cpp:166-188):
// b N×p, a p×N; ga p×N, gb N×p.
int oref_grad_abundances(const double* x, size_t l, size_t n, const double* b, size_t p,
                         const double* a, double* g, char* err, size_t errlen) {
  try {
    ar::ContributionMatrix bm{ar::Matrix(n, p)};
    std::copy(b, b + n * p, bm.data.values().begin());
    ar::AbundanceMatrix am{ar::Matrix(p, n)};
    std::copy(a, a + p * n, am.data.values().begin());
    copy_out(ar::grad_abundances(make_image(x, l, n), bm, am), g);
    return 0;
  } catch (const std::exception& ex) {
    put_err(ex, err, errlen);
    return 1;
  }
}

int oref_grad_contributions(const double* x, size_t l, size_t n, const double* b, size_t p,
                            const double* a, double* g, char* err, size_t errlen) {
  try {
    ar::ContributionMatrix bm{ar::Matrix(n, p)};
    std::copy(b, b + n * p, bm.data.values().begin());
    ar::AbundanceMatrix am{ar::Matrix(p, n)};
    std::copy(a, a + p * n, am.data.values().begin());
    copy_out(ar::grad_contributions(make_image(x, l, n), bm, am), g);
    return 0;
  } catch (const std::exception& ex) {
    put_err(ex, err, errlen);
    return 1;
  }
}

int oref_objective_l2(const double* x, size_t l, size_t n, const double* b, size_t p,
                      const double* a, double* out, char* err, size_t errlen) {
  try {
    ar::ContributionMatrix bm{ar::Matrix(n, p)};
    std::copy(b, b + n * p, bm.data.values().begin());
    ar::AbundanceMatrix am{ar::Matrix(p, n)};
    std::copy(a, a + p * n, am.data.values().begin());
    *out = ar::objective_l2(make_image(x, l, n), bm, am);
    return 0;
  } catch (const std::exception& ex) {
    put_err(ex, err, errlen);
    return 1;
  }
}

// estimate_abundances (solver.cpp:240-259): e L×p → a p×N.
int oref_estimate_abundances(const double* x, size_t l, size_t n, const double* e, size_t p,
                             size_t iters, double eta, double* a, char* err, size_t errlen) {
  try {
    ar::EndmemberMatrix em{ar::Matrix(l, p)};
    std::copy(e, e + l * p, em.data.values().begin());
    copy_out(ar::estimate_abundances(make_image(x, l, n), em, iters, eta).data, a);
    return 0;
  } catch (const std::exception& ex) {
    put_err(ex, err, errlen);
    return 1;
  }
}

// check_iterate (solver.cpp:65-90) on a rows×cols matrix: 0 if it passes, 1 with
// the reference's message otherwise. which: "abundance" or "contribution".
int oref_check_iterate(const double* m, size_t rows, size_t cols, size_t outer, const char* which,
                       char* err, size_t errlen) {
  try {
    ar::Matrix mm(rows, cols);
    std::copy(m, m + rows * cols, mm.values().begin());
    ar::check_iterate(mm, outer, which);
    return 0;
  } catch (const std::exception& ex) {
    put_err(ex, err, errlen);
    return 1;
  }
}

}  // extern "C"
