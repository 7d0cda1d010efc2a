// archetype:: solver API on the GPU (reference contract: solver.hpp:15-86,
// solver.cpp:103-259).  run() is a one-run batch of the device solver; the
// image-sized primitives call the device primitives of include/edaa_b200.h.
#include "archetype/solver.hpp"

#include <algorithm>
#include <cmath>
#include <exception>
#include <limits>
#include <sstream>

#include "archetype/ensemble.hpp"
#include "archetype/error.hpp"
#include "device.hpp"

namespace archetype {

namespace {

constexpr double kFloor = 1e-30;  // solver.cpp:15

void shapes_agree(const HsiImage& x, const Matrix& b, const Matrix& a, const char* op) {
  if (b.rows() == x.pixels() && a.cols() == x.pixels() && b.cols() == a.rows()) return;
  std::ostringstream msg;
  msg << op << ": shape mismatch (X " << x.bands() << "x" << x.pixels() << ", B " << b.rows()
      << "x" << b.cols() << ", A " << a.rows() << "x" << a.cols() << ")";
  throw Error(msg.str());
}

struct ObserverBridge {
  const StepObserver* observer = nullptr;
  std::exception_ptr error;
};

void observe_cb(size_t outer, char block, size_t inner, const double* a, const double* b, size_t p,
                size_t n, void* user) {
  auto* br = static_cast<ObserverBridge*>(user);
  if (br->error) return;  // an observer already threw: stay quiet until the solve returns
  try {
    Matrix am(p, n), bm(n, p);
    std::copy(a, a + p * n, am.values().begin());
    std::copy(b, b + n * p, bm.values().begin());
    (*br->observer)(InnerStep{outer, block, inner, am, bm});
  } catch (...) {
    br->error = std::current_exception();
  }
}

}  // namespace

void SolverConfig::validate() const {
  if (endmembers < 2) throw Error("solver config: endmember count must be at least 2");
  if (outer_iters < 1 || inner_iters_a < 1 || inner_iters_b < 1)
    throw Error("solver config: iteration counts must be at least 1");
  if (!(gamma > 0.0) || !std::isfinite(gamma))
    throw Error("solver config: step factor gamma must be positive");
}

AbundanceMatrix init_abundances(std::size_t p, std::size_t n) {
  if (p < 2 || n < 1) throw Error("init_abundances: need p >= 2 and n >= 1");
  return {Matrix(p, n, 1.0 / static_cast<double>(p))};
}

ContributionMatrix init_contributions(std::size_t n, std::size_t p, Prng& rng) {
  if (n < 1 || p < 2) throw Error("init_contributions: need n >= 1 and p >= 2");
  Matrix b(n, p);
  std::vector<double> w(n);
  for (std::size_t c = 0; c < p; ++c) {
    double top = -std::numeric_limits<double>::infinity();
    for (std::size_t j = 0; j < n; ++j) {
      w[j] = 0.1 * rng.next_unit();
      top = std::max(top, w[j]);
    }
    double total = 0.0;
    for (std::size_t j = 0; j < n; ++j) {
      w[j] = std::exp(w[j] - top);
      total += w[j];
    }
    for (std::size_t j = 0; j < n; ++j) b(j, c) = w[j] / total;
  }
  return {b};
}

StepSizes step_sizes(const HsiImage& x, const ContributionMatrix& b0, double gamma) {
  if (!(gamma > 0.0)) throw Error("step_sizes: gamma must be positive");
  const std::size_t p = b0.endmember_count();
  Matrix xb(x.bands(), p);
  {
    detail::Device& d = detail::device(0);
    std::lock_guard<std::mutex> lock(d.mu);
    detail::upload_image(d, x.data);
    if (edaa_xb(d.ctx, b0.data.values().data(), p, xb.values().data()) != EDAA_OK)
      detail::fail(d, "step_sizes");
  }
  if (xb.frobenius_norm() == 0.0) throw Error("degenerate initialization: X\xc2\xb7" "B0 is zero");
  const double sigma = spectral_norm(xb);
  StepSizes eta;
  eta.eta_a = gamma / (sigma * sigma);
  eta.eta_b = std::sqrt(static_cast<double>(p) / static_cast<double>(b0.pixel_count())) * eta.eta_a;
  return eta;
}

std::vector<double> entropic_step(std::span<const double> z, std::span<const double> grad,
                                  double eta) {
  if (z.size() != grad.size() || z.empty()) throw Error("entropic_step: size mismatch");
  if (!(eta > 0.0) || !std::isfinite(eta)) throw Error("entropic_step: eta must be positive");
  const std::size_t d = z.size();
  std::vector<double> s(d), out(d);
  double top = -std::numeric_limits<double>::infinity();
  for (std::size_t i = 0; i < d; ++i) {
    if (!std::isfinite(grad[i])) throw Error("entropic_step: non-finite gradient");
    s[i] = std::log(std::max(z[i], kFloor)) + (-eta * grad[i]);
    top = std::max(top, s[i]);
  }
  double total = 0.0;
  for (std::size_t i = 0; i < d; ++i) {
    s[i] = std::exp(s[i] - top);
    total += s[i];
  }
  for (std::size_t i = 0; i < d; ++i) out[i] = s[i] / total;
  return out;
}

Matrix grad_abundances(const HsiImage& x, const ContributionMatrix& b, const AbundanceMatrix& a) {
  shapes_agree(x, b.data, a.data, "grad_abundances");
  Matrix g(a.data.rows(), x.pixels());
  detail::Device& d = detail::device(0);
  std::lock_guard<std::mutex> lock(d.mu);
  detail::upload_image(d, x.data);
  if (edaa_grad_abundances(d.ctx, b.data.values().data(), a.data.values().data(), a.data.rows(),
                           g.values().data()) != EDAA_OK)
    detail::fail(d, "grad_abundances");
  return g;
}

Matrix grad_contributions(const HsiImage& x, const ContributionMatrix& b,
                          const AbundanceMatrix& a) {
  shapes_agree(x, b.data, a.data, "grad_contributions");
  Matrix g(x.pixels(), b.data.cols());
  detail::Device& d = detail::device(0);
  std::lock_guard<std::mutex> lock(d.mu);
  detail::upload_image(d, x.data);
  if (edaa_grad_contributions(d.ctx, b.data.values().data(), a.data.values().data(),
                              a.data.rows(), g.values().data()) != EDAA_OK)
    detail::fail(d, "grad_contributions");
  return g;
}

double objective_l2(const HsiImage& x, const ContributionMatrix& b, const AbundanceMatrix& a) {
  shapes_agree(x, b.data, a.data, "objective_l2");
  double out = 0.0;
  detail::Device& d = detail::device(0);
  std::lock_guard<std::mutex> lock(d.mu);
  detail::upload_image(d, x.data);
  if (edaa_objective(d.ctx, b.data.values().data(), a.data.values().data(), a.data.rows(), &out) !=
      EDAA_OK)
    detail::fail(d, "objective_l2");
  return out;
}

RunResult run(const HsiImage& x, const SolverConfig& config, const StepObserver& observer) {
  config.validate();
  x.validate();
  const std::size_t p = config.endmembers, n = x.pixels(), l = x.bands();
  const std::uint64_t seed = config.seed;
  const double gamma = config.gamma;
  const edaa_solve_params prm{p, config.outer_iters, config.inner_iters_a, config.inner_iters_b,
                              1, &seed, &gamma};
  RunResult result;
  result.seed = seed;
  result.gamma = gamma;
  result.endmembers.data = Matrix(l, p);
  result.abundances.data = Matrix(p, n);
  result.contributions.data = Matrix(n, p);
  result.objective_trace.resize(config.outer_iters + 1);
  ObserverBridge bridge;
  edaa_run_record rec{};
  {
    detail::Device& d = detail::device(0);
    std::lock_guard<std::mutex> lock(d.mu);
    detail::upload_image(d, x.data);
    int rc;
    if (observer) {
      bridge.observer = &observer;
      rc = edaa_solve_observed(d.ctx, &prm, observe_cb, &bridge);
    } else {
      rc = edaa_solve(d.ctx, &prm);
    }
    if (rc != EDAA_OK) detail::fail(d, "run");
    if (edaa_run_record_get(d.ctx, 0, &rec) != EDAA_OK) detail::fail(d, "run");
    if (rec.ok) {
      if (edaa_traces(d.ctx, result.objective_trace.data()) != EDAA_OK ||
          edaa_factors(d.ctx, 0, result.abundances.data.values().data(),
                       result.contributions.data.values().data(),
                       result.endmembers.data.values().data()) != EDAA_OK)
        detail::fail(d, "run");
    }
  }
  if (bridge.error) std::rethrow_exception(bridge.error);
  if (!rec.ok) throw Error(rec.message);
  result.fit_l1 = rec.fit_l1;
  result.coherence = rec.coherence;
  return result;
}

AbundanceMatrix estimate_abundances(const HsiImage& x, const EndmemberMatrix& e, std::size_t iters,
                                    double eta) {
  if (!x.data.all_finite() || !e.data.all_finite())
    throw Error("estimate_abundances: non-finite input");
  if (e.bands() != x.bands()) throw Error("estimate_abundances: band count mismatch");
  if (e.count() < 1) throw Error("estimate_abundances: need at least one endmember");
  if (!(eta > 0.0) || !std::isfinite(eta)) throw Error("estimate_abundances: eta must be positive");
  AbundanceMatrix a{Matrix(e.count(), x.pixels())};
  detail::Device& d = detail::device(0);
  std::lock_guard<std::mutex> lock(d.mu);
  detail::upload_image(d, x.data);
  if (edaa_estimate_abundances(d.ctx, e.data.values().data(), e.count(), iters, eta,
                               a.data.values().data()) != EDAA_OK)
    detail::fail(d, "estimate_abundances");
  return a;
}

}  // namespace archetype
