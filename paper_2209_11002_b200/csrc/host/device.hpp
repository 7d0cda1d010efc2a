// Internal: the process-wide device contexts behind the archetype:: API.
#pragma once

#include <mutex>
#include <string>

#include <utility>

#include "archetype/ensemble.hpp"
#include "archetype/error.hpp"
#include "archetype/image.hpp"
#include "archetype/matrix.hpp"
#include "archetype/solver.hpp"
#include "edaa_b200.h"

namespace archetype::detail {

struct Device {
  int ordinal = 0;
  edaa_ctx* ctx = nullptr;
  std::mutex mu;  // a context is not thread-safe; callers hold this lock
};

/// Number of CUDA devices usable by the library (≥ 1) — throws Error if none.
int device_count();
/// Lazily created context for device `i`.
Device& device(int i);
/// Throws Error carrying the context's last error text.
[[noreturn]] void fail(const Device& d, const std::string& what);
/// Copies X to the device: fp32 when every entry is exactly an fp32 (fast
/// path), fp64 otherwise.
void upload_image(Device& d, const Matrix& x);

/// run_ensemble(l2_normalize(raw).image, config) with the validate + ℓ2
/// normalisation done by the device ingest (edaa_ingest_host: same bits, same
/// messages in the same order) instead of host fp64 passes; `zero_pixels`
/// receives NormalizeResult::zero_pixels.size(). The CLI's `unmix` path.
std::pair<RunResult, SelectionReport> run_ensemble_raw(const HsiImage& raw, const EnsembleConfig& config,
                                                       std::size_t& zero_pixels);

}  // namespace archetype::detail
