// Drop-in test of the archetype:: C++ API served by libarchetype_b200.so (GPU).
//
// The cases restate, against this library, the behaviour the reference's own
// hot-path unit tests pin (cited per case, paths under /root/reference/proj/
// tests/), plus an A/B comparison with the reference solver itself when
// oracle/_ref/liboracle_ref.so is present.  Exit status = failed cases.
#include <dlfcn.h>

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstdlib>
#include <string>
#include <vector>

#include "archetype/ensemble.hpp"
#include "archetype/error.hpp"
#include "archetype/image.hpp"
#include "archetype/matrix.hpp"
#include "archetype/prng.hpp"
#include "archetype/solver.hpp"
#include "archetype/types.hpp"
#include "mini_test.hpp"

using namespace archetype;
using mini::Approx;

namespace {

HsiImage uniform_image(std::size_t l, std::size_t n, std::uint64_t seed) {
  Prng rng(seed);
  HsiImage img;
  img.data = Matrix(l, n);
  for (double& v : img.data.values()) v = rng.next_unit();
  return img;
}

double col_sum(const Matrix& m, std::size_t c) {
  double s = 0.0;
  for (std::size_t r = 0; r < m.rows(); ++r) s += m(r, c);
  return s;
}

// Random point of the d-simplex (normalised exponentials of uniforms).
std::vector<double> simplex_point(Prng& rng, std::size_t d) {
  std::vector<double> v(d);
  double s = 0.0;
  for (double& x : v) {
    x = -std::log(1.0 - rng.next_unit());
    s += x;
  }
  for (double& x : v) x /= s;
  return v;
}

// Three separated smooth unit spectra over 12 bands and interior mixtures.
struct Mixture {
  EndmemberMatrix e;
  AbundanceMatrix a;
  HsiImage x;
};
Mixture three_bumps(std::size_t pixels) {
  Mixture m;
  m.e.data = Matrix(12, 3);
  const double centre[3] = {2.0, 6.0, 10.0};
  for (std::size_t k = 0; k < 3; ++k) {
    for (std::size_t i = 0; i < 12; ++i) {
      const double z = (static_cast<double>(i) - centre[k]) / 1.5;
      m.e.data(i, k) = std::exp(-0.5 * z * z) + 0.02;
    }
    const double nrm = m.e.data.column_norm(k);
    for (std::size_t i = 0; i < 12; ++i) m.e.data(i, k) /= nrm;
  }
  Prng rng(11);
  m.a.data = Matrix(3, pixels);
  for (std::size_t j = 0; j < pixels; ++j) {
    std::vector<double> c = simplex_point(rng, 3);
    for (std::size_t k = 0; k < 3; ++k) c[k] = 0.6 * c[k] + 0.4 / 3.0;  // keep it interior
    for (std::size_t k = 0; k < 3; ++k) m.a.data(k, j) = c[k];
  }
  m.x.data = matmul(m.e.data, m.a.data);
  return m;
}

}  // namespace

// ---- core (test_core.cpp) ----------------------------------------------------
TEST_CASE("prng stream and unit mapping are the published SplitMix64") {
  Prng r0(0);
  CHECK(r0.next_u64() == 0xe220a8397b1dcdafULL);
  CHECK(r0.next_u64() == 0x6e789e6aa1b965f4ULL);
  CHECK(r0.next_u64() == 0x06c45d188009454fULL);
  Prng u0(0);
  CHECK(u0.next_unit() == 0.8833108082136426);
  CHECK(u0.next_unit() == 0.43152799704850997);
  Prng u1(1);
  CHECK(u1.next_unit() == 0.5665615751722809);
}

TEST_CASE("matmul hand product, transposed forms, thread independence") {
  Matrix a(2, 3), b(3, 2);
  const double av[] = {1, 2, 3, 4, 5, 6}, bv[] = {7, 8, 9, 10, 11, 12};
  std::copy(av, av + 6, a.values().begin());
  std::copy(bv, bv + 6, b.values().begin());
  const Matrix c = matmul(a, b);
  CHECK(c(0, 0) == 58.0);
  CHECK(c(1, 1) == 154.0);
  CHECK(matmul_tn(a, a) == matmul(transpose(a), a));
  CHECK(matmul_nt(a, a) == matmul(a, transpose(a)));
  Prng rng(7);
  Matrix p(17, 23), q(23, 11);
  for (double& v : p.values()) v = rng.next_unit() - 0.5;
  for (double& v : q.values()) v = rng.next_unit() - 0.5;
  CHECK(matmul(p, q, 1) == matmul(p, q, 4));
  CHECK(matmul(p, q, 1) == matmul(p, q, 9));
}

TEST_CASE("spectral norm known values") {
  Matrix m(3, 4);
  const double mv[] = {1.0, 2.0, 0.5, -1.0, 0.0, 3.0, 1.5, 2.0, -2.0, 0.25, 1.0, 0.0};
  std::copy(mv, mv + 12, m.values().begin());
  CHECK(spectral_norm(m) == Approx(4.185922592173704).eps(1e-6));
  CHECK(spectral_norm(Matrix::identity(5)) == Approx(1.0).eps(1e-9));
}

TEST_CASE("image validation and l2 normalisation") {
  HsiImage img;
  img.data = Matrix(2, 3, 0.5);
  CHECK_NOTHROW(img.validate());
  img.data(1, 2) = -0.1;
  CHECK_THROWS_AS(img.validate(), Error);
  img.data(1, 2) = 0.5;
  img.spatial = Shape2d{2, 2};
  CHECK_THROWS_AS(img.validate(), Error);
  HsiImage z;
  z.data = Matrix(3, 2, 0.0);
  CHECK_THROWS_WITH(l2_normalize(z), "degenerate input: all pixels are zero");
}

TEST_CASE("simplex column validation") {
  Matrix good(3, 2, 1.0 / 3.0);
  CHECK_NOTHROW(validate_simplex_columns(good, 1e-9, "t"));
  Matrix drift = good;
  drift(0, 0) += 1e-6;
  CHECK_THROWS_AS(validate_simplex_columns(drift, 1e-9, "t"), Error);
  CHECK_NOTHROW(validate_simplex_columns(drift, 1e-5, "t"));
}

// ---- solver (test_solver.cpp) -----------------------------------------------
TEST_CASE("initialisations: uniform A, seeded near-uniform B") {
  const AbundanceMatrix a = init_abundances(4, 7);
  for (double v : a.data.values()) CHECK(v == 0.25);
  Prng rng(0);
  const ContributionMatrix b = init_contributions(3, 2, rng);
  const double u[] = {0.8833108082136426, 0.43152799704850997, 0.026433771592597743};
  double s[3], t = 0.0;
  for (int i = 0; i < 3; ++i) t += (s[i] = std::exp(0.1 * u[i] - 0.1 * u[0]));
  for (int i = 0; i < 3; ++i) CHECK(b.data(i, 0) == Approx(s[i] / t).eps(1e-15));
  CHECK_NOTHROW(b.validate(1e-12));
}

TEST_CASE("step sizes: γ/σ² and √(p/N) scaling, linear in γ (GPU X·B⁰)") {
  const HsiImage x = uniform_image(5, 40, 3);
  Prng rng(9);
  const ContributionMatrix b0 = init_contributions(40, 4, rng);
  const StepSizes e = step_sizes(x, b0, 2.0);
  const double sigma = spectral_norm(matmul(x.data, b0.data));
  CHECK(e.eta_a == Approx(2.0 / (sigma * sigma)).eps(1e-12));
  CHECK(e.eta_b == Approx(std::sqrt(4.0 / 40.0) * e.eta_a).eps(1e-12));
  const StepSizes e2 = step_sizes(x, b0, 4.0);
  CHECK(e2.eta_a == Approx(2.0 * e.eta_a).eps(1e-12));
}

TEST_CASE("entropic step closed forms and the 1e-30 floor") {
  const std::vector<double> out = entropic_step(std::vector<double>{0.5, 0.5}, std::vector<double>{1.0, 0.0}, 1.0);
  CHECK(out[0] == Approx(0.2689414213699951).eps(1e-15));
  const std::vector<double> o3 =
      entropic_step(std::vector<double>{0.2, 0.3, 0.5}, std::vector<double>{0.1, -0.2, 0.3}, 2.0);
  CHECK(o3[1] == Approx(0.5053039670477497).eps(1e-14));
  const std::vector<double> fl = entropic_step(std::vector<double>{0.0, 1.0}, std::vector<double>{-100.0, 0.0}, 1.0);
  CHECK(std::isfinite(fl[0]) && fl[0] > 0.0);
  CHECK_THROWS_AS(entropic_step(std::vector<double>{0.5}, std::vector<double>{1.0}, 0.0), Error);
}

TEST_CASE("gradients match central finite differences of the objective (GPU)") {
  const HsiImage x = uniform_image(4, 6, 21);
  Prng rng(22);
  AbundanceMatrix a{Matrix(2, 6)};
  for (std::size_t j = 0; j < 6; ++j) {
    const std::vector<double> c = simplex_point(rng, 2);
    a.data(0, j) = c[0];
    a.data(1, j) = c[1];
  }
  const ContributionMatrix b = init_contributions(6, 2, rng);
  const double h = 1e-6;
  const Matrix ga = grad_abundances(x, b, a);
  for (std::size_t i = 0; i < 2; ++i)
    for (std::size_t j = 0; j < 6; ++j) {
      AbundanceMatrix ap = a, am = a;
      ap.data(i, j) += h;
      am.data(i, j) -= h;
      const double fd = (objective_l2(x, b, ap) - objective_l2(x, b, am)) / (2 * h);
      CHECK(ga(i, j) == Approx(fd).eps(1e-5));
    }
  const Matrix gb = grad_contributions(x, b, a);
  for (std::size_t i = 0; i < 6; ++i)
    for (std::size_t j = 0; j < 2; ++j) {
      ContributionMatrix bp = b, bm = b;
      bp.data(i, j) += h;
      bm.data(i, j) -= h;
      const double fd = (objective_l2(x, bp, a) - objective_l2(x, bm, a)) / (2 * h);
      CHECK(gb(i, j) == Approx(fd).eps(1e-5));
    }
}

TEST_CASE("run: simplex iterates, observer count, Ê = X·B̂ bitwise, determinism") {
  const HsiImage x = uniform_image(6, 30, 5);
  SolverConfig cfg;
  cfg.endmembers = 3;
  cfg.outer_iters = 8;
  cfg.seed = 17;
  std::size_t seen = 0;
  const RunResult r = run(x, cfg, [&](const InnerStep& s) {
    ++seen;
    for (std::size_t j = 0; j < s.abundances.cols(); ++j) CHECK(col_sum(s.abundances, j) == Approx(1.0).eps(1e-9));
    for (std::size_t j = 0; j < s.contributions.cols(); ++j)
      CHECK(col_sum(s.contributions, j) == Approx(1.0).eps(1e-9));
  });
  CHECK(seen == 8 * 10);
  CHECK_NOTHROW(r.abundances.validate());
  CHECK_NOTHROW(r.contributions.validate());
  REQUIRE(r.objective_trace.size() == 9);
  CHECK(r.objective_trace.back() < r.objective_trace.front());
  CHECK(r.endmembers.data == matmul(x.data, r.contributions.data));
  CHECK(r.seed == 17);
  const RunResult r2 = run(x, cfg);
  CHECK(r.abundances.data == r2.abundances.data);
  CHECK(r.contributions.data == r2.contributions.data);
  CHECK(r.fit_l1 == r2.fit_l1);
  SolverConfig other = cfg;
  other.seed = 18;
  CHECK(!(run(x, other).contributions.data == r.contributions.data));
}

TEST_CASE("run rejects invalid configs") {
  const HsiImage x = uniform_image(4, 10, 1);
  SolverConfig cfg;
  cfg.endmembers = 1;
  CHECK_THROWS_WITH(run(x, cfg), "solver config: endmember count must be at least 2");
  cfg.endmembers = 2;
  cfg.gamma = 0.0;
  CHECK_THROWS_AS(run(x, cfg), Error);
  cfg.gamma = 1.0;
  cfg.outer_iters = 0;
  CHECK_THROWS_AS(run(x, cfg), Error);
}

TEST_CASE("estimate_abundances recovers known mixtures and decreases the residual (GPU)") {
  const Mixture m = three_bumps(80);
  const double sigma = spectral_norm(m.e.data);
  const double eta = 1.0 / (sigma * sigma);
  const AbundanceMatrix est = estimate_abundances(m.x, m.e, 4000, eta);
  CHECK_NOTHROW(est.validate(1e-9));
  double worst = 0.0;
  for (std::size_t i = 0; i < 3; ++i)
    for (std::size_t j = 0; j < 80; ++j) worst = std::max(worst, std::fabs(est.data(i, j) - m.a.data(i, j)));
  CHECK(worst <= 1e-3);
  auto resid = [&](std::size_t it) {
    const Matrix d = subtract(m.x.data, matmul(m.e.data, estimate_abundances(m.x, m.e, it, eta).data));
    return 0.5 * d.frobenius_norm() * d.frobenius_norm();
  };
  double prev = resid(40);
  for (std::size_t it = 41; it <= 45; ++it) {
    const double next = resid(it);
    CHECK(next <= prev + 1e-12);
    prev = next;
  }
  EndmemberMatrix one{Matrix(12, 1)};
  for (std::size_t i = 0; i < 12; ++i) one.data(i, 0) = m.e.data(i, 0);
  const AbundanceMatrix lone = estimate_abundances(three_bumps(6).x, one, 3, 0.5);
  for (std::size_t j = 0; j < 6; ++j) CHECK(lone.data(0, j) == 1.0);
}

// ---- ensemble (test_ensemble.cpp) --------------------------------------------
namespace {
RunRecord rec(std::size_t i, double fit, double mu, bool ok = true) {
  RunRecord r;
  r.index = i;
  r.seed = i;
  r.fit_l1 = fit;
  r.coherence = mu;
  r.ok = ok;
  return r;
}
}  // namespace

TEST_CASE("selection: cutoff, least coherent, ties low, failed runs skipped") {
  SelectionReport r = select_runs({rec(0, 10.0, 0.9), rec(1, 10.4, 0.8), rec(2, 11.0, 0.1)}, 1.05);
  CHECK(r.fit_min == 10.0);
  CHECK((r.candidate_set == std::vector<std::size_t>{0, 1}));
  CHECK(r.selected == 1);
  r = select_runs({rec(0, 10.0, 0.5), rec(1, 10.1, 0.5), rec(2, 10.2, 0.5)}, 1.05);
  CHECK(r.selected == 0);
  r = select_runs({rec(0, 1.0, 0.0, false), rec(1, 10.0, 0.9), rec(2, 10.2, 0.3)}, 1.05);
  CHECK((r.candidate_set == std::vector<std::size_t>{1, 2}) && r.selected == 2);
  CHECK_THROWS_WITH(select_runs({rec(0, 1.0, 0.0, false)}, 1.05), "every run failed");
}

TEST_CASE("gamma sampling: goldens and uniformity") {
  const std::vector<double> set{0.125, 0.25, 0.5, 1.0, 2.0, 4.0, 8.0};
  Prng rng(0);
  CHECK(sample_gamma(rng, set) == 8.0);
  CHECK(sample_gamma(rng, set) == 1.0);
  Prng mc(123);
  std::vector<int> counts(7, 0);
  for (int i = 0; i < 70000; ++i)
    ++counts[std::find(set.begin(), set.end(), sample_gamma(mc, set)) - set.begin()];
  for (int c : counts) CHECK(c > 10000 - 600 && c < 10000 + 600);
}

TEST_CASE("coherence and fit_l1 (fit on the GPU)") {
  Matrix e(3, 3, 0.0);
  e(0, 0) = e(1, 1) = 1.0;
  e(0, 2) = 0.6;
  e(1, 2) = 0.8;
  CHECK(coherence({e}) == Approx(0.8).eps(1e-12));
  Matrix s = e;
  for (std::size_t i = 0; i < 3; ++i) s(i, 2) *= 2.0;
  CHECK(coherence({s}) == Approx(1.6).eps(1e-12));
  CHECK(coherence({s}, true) == Approx(0.8).eps(1e-12));
  HsiImage x;
  x.data = Matrix(2, 2);
  x.data(0, 0) = x.data(1, 1) = 1.0;
  CHECK(fit_l1(x, {Matrix::identity(2)}, {Matrix(2, 2, 0.5)}) == Approx(2.0).eps(1e-12));
}

TEST_CASE("ensemble: seeds base+m, worker-count independent, replay bitwise") {
  const HsiImage x = uniform_image(6, 40, 77);
  EnsembleConfig cfg;
  cfg.runs = 4;
  cfg.base_seed = 5;
  cfg.solver.endmembers = 2;
  cfg.solver.outer_iters = 6;
  cfg.workers = 1;
  auto [r1, rep1] = run_ensemble(x, cfg);
  REQUIRE(rep1.per_run.size() == 4);
  for (std::size_t m = 0; m < 4; ++m) {
    CHECK(rep1.per_run[m].seed == 5 + m);
    CHECK(rep1.per_run[m].ok);
    CHECK(rep1.per_run[m].fit_l1 > 0.0);
  }
  CHECK(r1.seed == rep1.per_run[rep1.selected].seed);
  cfg.workers = 3;
  auto [r2, rep2] = run_ensemble(x, cfg);
  CHECK(r1.abundances.data == r2.abundances.data);
  CHECK(r1.endmembers.data == r2.endmembers.data);
  CHECK(rep1.selected == rep2.selected);
  SolverConfig replay = cfg.solver;
  replay.seed = rep1.per_run[rep1.selected].seed;
  replay.gamma = rep1.per_run[rep1.selected].gamma;
  const RunResult again = run(x, replay);
  CHECK(again.abundances.data == r1.abundances.data);
  CHECK(again.contributions.data == r1.contributions.data);
  CHECK(again.endmembers.data == r1.endmembers.data);
  CHECK(again.fit_l1 == r1.fit_l1);
  CHECK(again.coherence == r1.coherence);
}

TEST_CASE("worker resolution and ensemble config validation") {
  CHECK(resolve_workers(3) == 3);
  ::setenv("ARCHETYPE_THREADS", "5", 1);
  CHECK(resolve_workers(0) == 5);
  ::unsetenv("ARCHETYPE_THREADS");
  CHECK(resolve_workers(0) >= 1);
  EnsembleConfig cfg;
  cfg.solver.endmembers = 2;
  CHECK_NOTHROW(cfg.validate());
  cfg.runs = 0;
  CHECK_THROWS_AS(cfg.validate(), Error);
  cfg.runs = 1;
  cfg.gamma_set = {0.5, -1.0};
  CHECK_THROWS_AS(cfg.validate(), Error);
  cfg.gamma_set = {0.5};
  cfg.fit_slack = 0.9;
  CHECK_THROWS_AS(cfg.validate(), Error);
}

// ---- acceptance-style (acceptance.cpp:70-89) --------------------------------
TEST_CASE("simplex preserved over 1000 inner steps") {
  const Mixture m = three_bumps(500);
  SolverConfig cfg;
  cfg.endmembers = 3;
  std::size_t steps = 0, bad = 0;
  run(l2_normalize(m.x).image, cfg, [&](const InnerStep& s) {
    ++steps;
    for (const Matrix* mm : {&s.abundances, &s.contributions})
      for (std::size_t j = 0; j < mm->cols(); ++j) {
        bool neg = false;
        for (std::size_t i = 0; i < mm->rows(); ++i) neg |= (*mm)(i, j) < 0.0;
        if (neg || std::fabs(col_sum(*mm, j) - 1.0) > 1e-9) ++bad;
      }
  });
  CHECK(steps == 1000);
  CHECK(bad == 0);
}

// ---- A/B against the reference solver itself ---------------------------------
TEST_CASE("A/B: run() and run_ensemble() against the reference build") {
  const char* path = std::getenv("EDAA_ORACLE_REF");
  void* h = dlopen(path ? path : "oracle/_ref/liboracle_ref.so", RTLD_NOW | RTLD_LOCAL);
  if (!h) {
    std::printf("  (skipped: reference oracle library not found)\n");
    return;
  }
  using run_fn = int (*)(const double*, size_t, size_t, size_t, size_t, size_t, size_t, double, uint64_t,
                         double*, double*, double*, double*, double*, double*, char*, size_t);
  auto oref_run = reinterpret_cast<run_fn>(dlsym(h, "oref_run"));
  REQUIRE(oref_run != nullptr);
  const HsiImage x = l2_normalize(uniform_image(24, 600, 42)).image;
  for (double gamma : {1.0, 8.0}) {
    SolverConfig cfg;
    cfg.endmembers = 4;
    cfg.outer_iters = 60;
    cfg.gamma = gamma;
    cfg.seed = 3;
    const RunResult got = run(x, cfg);
    std::vector<double> tr(61), a(4 * 600), b(600 * 4), e(24 * 4);
    double fit = 0.0, mu = 0.0;
    char err[256];
    REQUIRE(oref_run(x.data.values().data(), 24, 600, 4, 60, 5, 5, gamma, 3, tr.data(), a.data(),
                     b.data(), e.data(), &fit, &mu, err, sizeof err) == 0);
    double obj = 0.0, fa = 0.0, fb = 0.0;
    for (std::size_t t = 0; t <= 50; ++t) obj = std::max(obj, std::fabs(got.objective_trace[t] - tr[t]) / tr[t]);
    for (std::size_t i = 0; i < a.size(); ++i) fa = std::max(fa, std::fabs(got.abundances.data.values()[i] - a[i]));
    for (std::size_t i = 0; i < b.size(); ++i) fb = std::max(fb, std::fabs(got.contributions.data.values()[i] - b[i]));
    std::printf("  gamma %.1f: objective rel %.2e, A %.2e, B %.2e\n", gamma, obj, fa, fb);
    CHECK(obj <= 1e-4);
    CHECK(fa <= 1e-3);
    CHECK(fb <= 1e-3);
    CHECK(got.fit_l1 == Approx(fit).eps(1e-9));
    CHECK(got.coherence == Approx(mu).eps(1e-9));
  }
  dlclose(h);
}

int main(int argc, char** argv) { return mini::run_all(argc > 1 ? argv[1] : nullptr); }
