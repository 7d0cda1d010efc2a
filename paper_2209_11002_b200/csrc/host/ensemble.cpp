// archetype:: ensemble + model selection on the GPU (reference contract:
// ensemble.hpp:15-73, ensemble.cpp:17-167).  All M runs are one batched device
// solve; with several devices the runs are split into contiguous blocks, one
// host thread per device.  A run's bits do not depend on its batch or device,
// so the result equals the single-device result (and the reference's
// worker-count independence, test_ensemble.cpp:118-148, holds).
#include "archetype/ensemble.hpp"

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdlib>
#include <exception>
#include <functional>
#include <limits>
#include <thread>

#include "archetype/error.hpp"
#include "device.hpp"

namespace archetype {

void EnsembleConfig::validate() const {
  if (runs == 0) throw Error("ensemble needs at least one run");
  if (gamma_set.empty()) throw Error("step factor set is empty");
  for (double g : gamma_set)
    if (!std::isfinite(g) || g <= 0.0) throw Error("step factors must be finite and positive");
  if (!std::isfinite(fit_slack) || fit_slack < 1.0) throw Error("fit slack must be at least 1");
  solver.validate();
}

double fit_l1(const HsiImage& x, const EndmemberMatrix& e, const AbundanceMatrix& a) {
  if (e.bands() != x.bands() || a.pixel_count() != x.pixels() || e.count() != a.endmember_count())
    throw Error("fit: dimension mismatch");
  double out = 0.0;
  detail::Device& d = detail::device(0);
  std::lock_guard<std::mutex> lock(d.mu);
  detail::upload_image(d, x.data);
  if (edaa_fit_l1(d.ctx, e.data.values().data(), a.data.values().data(), e.count(), &out) != EDAA_OK)
    detail::fail(d, "fit_l1");
  return out;
}

double coherence(const EndmemberMatrix& e, bool normalized) {
  const std::size_t p = e.count();
  if (p < 2) return 0.0;
  double best = -std::numeric_limits<double>::infinity();
  for (std::size_t i = 0; i < p; ++i)
    for (std::size_t j = i + 1; j < p; ++j) {
      double dot = 0.0;
      for (std::size_t r = 0; r < e.bands(); ++r) dot += e.data(r, i) * e.data(r, j);
      if (normalized) {
        const double ni = e.data.column_norm(i), nj = e.data.column_norm(j);
        if (ni == 0.0 || nj == 0.0) continue;
        dot /= ni * nj;
      }
      best = std::max(best, dot);
    }
  return best == -std::numeric_limits<double>::infinity() ? 0.0 : best;
}

double sample_gamma(Prng& rng, const std::vector<double>& gamma_set) {
  if (gamma_set.empty()) throw Error("step factor set is empty");
  const std::size_t n = gamma_set.size();
  const auto idx = static_cast<std::size_t>(rng.next_unit() * static_cast<double>(n));
  return gamma_set[std::min(idx, n - 1)];
}

SelectionReport select_runs(std::vector<RunRecord> per_run, double fit_slack) {
  SelectionReport rep;
  rep.per_run = std::move(per_run);
  double fmin = std::numeric_limits<double>::infinity();
  for (const RunRecord& r : rep.per_run)
    if (r.ok) fmin = std::min(fmin, r.fit_l1);
  if (fmin == std::numeric_limits<double>::infinity()) throw Error("every run failed");
  rep.fit_min = fmin;
  const double cutoff = fit_slack * fmin;
  for (const RunRecord& r : rep.per_run)
    if (r.ok && r.fit_l1 <= cutoff) rep.candidate_set.push_back(r.index);
  std::size_t best = rep.candidate_set.front();
  for (std::size_t idx : rep.candidate_set)
    if (rep.per_run[idx].coherence < rep.per_run[best].coherence) best = idx;
  rep.selected = best;
  return rep;
}

unsigned resolve_workers(unsigned requested) {
  if (requested != 0) return requested;
  if (const char* env = std::getenv("ARCHETYPE_THREADS")) {
    char* end = nullptr;
    const unsigned long v = std::strtoul(env, &end, 10);
    if (end != env && *end == '\0' && v > 0) return static_cast<unsigned>(std::min<unsigned long>(v, 1024));
  }
  const unsigned hw = std::thread::hardware_concurrency();
  return hw == 0 ? 1 : hw;
}

namespace {

struct Shard {
  std::size_t first = 0, count = 0;
  detail::Device* dev = nullptr;
  std::vector<edaa_run_record> recs;
  double wall_ms = 0.0;
  std::exception_ptr error;
};

using Uploader = std::function<void(detail::Device&)>;

void solve_shard(Shard& sh, const Uploader& upload, const EnsembleConfig& cfg,
                 const std::vector<std::uint64_t>& seeds, const std::vector<double>& gammas) {
  try {
    detail::Device& d = *sh.dev;  // locked by ensemble_on_devices for the whole call
    upload(d);
    const edaa_solve_params prm{cfg.solver.endmembers, cfg.solver.outer_iters,
                                cfg.solver.inner_iters_a, cfg.solver.inner_iters_b, sh.count,
                                seeds.data() + sh.first, gammas.data() + sh.first};
    const auto t0 = std::chrono::steady_clock::now();
    if (edaa_solve(d.ctx, &prm) != EDAA_OK) detail::fail(d, "run_ensemble");
    sh.wall_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    sh.recs.resize(sh.count);
    for (std::size_t m = 0; m < sh.count; ++m)
      if (edaa_run_record_get(d.ctx, m, &sh.recs[m]) != EDAA_OK) detail::fail(d, "run_ensemble");
  } catch (...) {
    sh.error = std::current_exception();
  }
}

}  // namespace

namespace {

// The batched solve behind run_ensemble, for an image the uploader puts on
// every device (host-normalised X, or the raw cube through the device ingest).
// The reference's run_ensemble is a reentrant pure function: every device this
// call uses stays locked from the upload through the solve, the selection and
// the factor / trace download, so a concurrent run(), primitive or
// run_ensemble() on another thread cannot swap the image or the results in
// between.  Locks are taken in ascending ordinal (deadlock-free); `held` is
// device 0's lock when the caller already holds it (ingest → solve).
std::pair<RunResult, SelectionReport> ensemble_on_devices(const Uploader& upload, std::size_t l,
                                                          std::size_t n, const EnsembleConfig& config,
                                                          std::unique_lock<std::mutex>* held = nullptr) {
  const std::size_t M = config.runs;
  std::vector<std::uint64_t> seeds(M);
  std::vector<double> gammas(M);
  for (std::size_t m = 0; m < M; ++m) {  // seed = base + m, γ from its first draw (ensemble.cpp:123-127)
    seeds[m] = config.base_seed + m;
    Prng rng(seeds[m]);
    gammas[m] = sample_gamma(rng, config.gamma_set);
  }
  const std::size_t ndev = std::min<std::size_t>(static_cast<std::size_t>(detail::device_count()), M);
  std::vector<std::unique_lock<std::mutex>> locks;
  for (std::size_t g = 0; g < ndev; ++g)
    if (!(g == 0 && held != nullptr)) locks.emplace_back(detail::device(static_cast<int>(g)).mu);
  std::vector<Shard> shards(ndev);
  for (std::size_t g = 0; g < ndev; ++g) {
    shards[g].first = g * M / ndev;
    shards[g].count = (g + 1) * M / ndev - shards[g].first;
    shards[g].dev = &detail::device(static_cast<int>(g));
  }
  if (ndev == 1) {
    solve_shard(shards[0], upload, config, seeds, gammas);
  } else {
    std::vector<std::thread> pool;
    for (auto& sh : shards) pool.emplace_back([&, ptr = &sh] { solve_shard(*ptr, upload, config, seeds, gammas); });
    for (auto& t : pool) t.join();
  }
  for (auto& sh : shards)
    if (sh.error) std::rethrow_exception(sh.error);

  std::vector<RunRecord> records(M);
  for (const Shard& sh : shards)
    for (std::size_t k = 0; k < sh.count; ++k) {
      const std::size_t m = sh.first + k;
      const edaa_run_record& r = sh.recs[k];
      RunRecord& rec = records[m];
      rec.index = m;
      rec.seed = seeds[m];
      rec.gamma = gammas[m];
      rec.ok = r.ok != 0;
      rec.fit_l1 = rec.ok ? r.fit_l1 : 0.0;
      rec.coherence = rec.ok ? r.coherence : 0.0;
      rec.error = rec.ok ? std::string() : std::string(r.message);
      rec.wall_ms = sh.wall_ms;  // runs of one device are solved together
    }

  SelectionReport report;
  if (ndev == 1) {  // Algorithm 2's rule on the device (k_select)
    detail::Device& d = *shards[0].dev;
    std::vector<std::uint8_t> cand(M);
    std::size_t sel = 0;
    double fmin = 0.0;
    const int rc = edaa_select(d.ctx, config.fit_slack, cand.data(), &sel, &fmin);
    if (rc == EDAA_ERR_ALL_FAILED) throw Error("every run failed");
    if (rc != EDAA_OK) detail::fail(d, "run_ensemble");
    report.per_run = std::move(records);
    for (std::size_t m = 0; m < M; ++m)
      if (cand[m]) report.candidate_set.push_back(m);
    report.selected = sel;
    report.fit_min = fmin;
  } else {
    report = select_runs(std::move(records), config.fit_slack);
  }

  const std::size_t s = report.selected;
  Shard* owner = nullptr;
  for (auto& sh : shards)
    if (s >= sh.first && s < sh.first + sh.count) owner = &sh;
  const std::size_t p = config.solver.endmembers;
  RunResult res;
  res.seed = seeds[s];
  res.gamma = gammas[s];
  res.fit_l1 = report.per_run[s].fit_l1;
  res.coherence = report.per_run[s].coherence;
  res.endmembers.data = Matrix(l, p);
  res.abundances.data = Matrix(p, n);
  res.contributions.data = Matrix(n, p);
  {
    detail::Device& d = *owner->dev;
    std::vector<double> traces(owner->count * (config.solver.outer_iters + 1));
    if (edaa_traces(d.ctx, traces.data()) != EDAA_OK ||
        edaa_factors(d.ctx, s - owner->first, res.abundances.data.values().data(),
                     res.contributions.data.values().data(), res.endmembers.data.values().data()) != EDAA_OK)
      detail::fail(d, "run_ensemble");
    const std::size_t stride = config.solver.outer_iters + 1;
    res.objective_trace.assign(traces.begin() + (s - owner->first) * stride,
                               traces.begin() + (s - owner->first + 1) * stride);
  }
  return {std::move(res), std::move(report)};
}

}  // namespace

std::pair<RunResult, SelectionReport> run_ensemble(const HsiImage& x,
                                                   const EnsembleConfig& config) {
  config.validate();
  x.validate();
  return ensemble_on_devices([&x](detail::Device& d) { detail::upload_image(d, x.data); }, x.bands(),
                             x.pixels(), config);
}

namespace detail {

// HsiImage::validate's non-value checks (image.cpp:15-26), in its order.
static void check_shape(const HsiImage& raw) {
  if (raw.spatial && raw.spatial->height * raw.spatial->width != raw.pixels()) {
    HsiImage probe;  // the reference's message, built by the host validate
    probe.data = Matrix(1, raw.pixels());
    probe.spatial = raw.spatial;
    probe.validate();
  }
  if (!raw.wavelengths.empty() && raw.wavelengths.size() != raw.bands())
    throw Error("image: wavelength list length differs from band count");
}

// Ingest (validate + ℓ2-normalise on the device) then the batched solve, in
// the reference's order of messages: a bad value, then the shape checks, then
// "degenerate input" — all before the config is looked at, as `unmix`
// validates and normalises the image before run_ensemble (cli.cpp:75-78).
// `upload` runs edaa_ingest_host[_f32] on one device and returns its status.
static std::pair<RunResult, SelectionReport> ingest_and_solve(const std::function<int(Device&, std::size_t&)>& upload,
                                                              const std::function<void()>& shape_check,
                                                              std::size_t l, std::size_t n,
                                                              const EnsembleConfig& config,
                                                              std::size_t& zero_pixels) {
  const auto ingest = [&](Device& d) {
    std::size_t nz = 0;
    if (upload(d, nz) != EDAA_OK) {
      const std::string what = edaa_last_error(d.ctx);
      if (what.rfind("degenerate", 0) == 0) shape_check();
      throw Error(what);
    }
    return nz;
  };
  Device& first = device(0);
  std::unique_lock<std::mutex> lock(first.mu);  // held from the ingest through the solve
  zero_pixels = ingest(first);
  shape_check();
  config.validate();
  // Device 0 already holds the normalised image; further devices ingest their own copy.
  return ensemble_on_devices([&](Device& d) { if (&d != &first) ingest(d); }, l, n, config, &lock);
}

std::pair<RunResult, SelectionReport> run_ensemble_raw(const HsiImage& raw, const EnsembleConfig& config,
                                                       std::size_t& zero_pixels) {
  if (raw.bands() < 1 || raw.pixels() < 1) raw.validate();  // the reference's size message
  return ingest_and_solve(
      [&raw](Device& d, std::size_t& nz) {
        return edaa_ingest_host(d.ctx, raw.data.values().data(), raw.bands(), raw.pixels(), nullptr, 0, &nz);
      },
      [&raw] { check_shape(raw); }, raw.bands(), raw.pixels(), config, zero_pixels);
}

std::pair<RunResult, SelectionReport> run_ensemble_raw_f32(const float* x, std::size_t bands, std::size_t pixels,
                                                           bool pixel_major, const EnsembleConfig& config,
                                                           std::size_t& zero_pixels) {
  if (bands < 1 || pixels < 1) {
    HsiImage empty;
    empty.data = Matrix(bands, pixels);
    empty.validate();
  }
  return ingest_and_solve(
      [&](Device& d, std::size_t& nz) {
        return edaa_ingest_host_f32(d.ctx, x, bands, pixels, pixel_major ? 1 : 0, nullptr, 0, &nz);
      },
      [] {}, bands, pixels, config, zero_pixels);  // an NPY cube has a consistent shape, no wavelengths
}

}  // namespace detail

}  // namespace archetype
