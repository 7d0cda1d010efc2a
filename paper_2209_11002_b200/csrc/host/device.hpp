// Internal: the process-wide device contexts behind the archetype:: API.
#pragma once

#include <mutex>
#include <string>

#include <utility>

#include "archetype/ensemble.hpp"
#include "archetype/error.hpp"
#include "archetype/image.hpp"
#include "archetype/matrix.hpp"
#include "archetype/npy.hpp"
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
/// The same from an fp32 NPY payload as stored (L×N band-major, or the N×L
/// pixel-major payload of an (H, W, L) cube): no host widening or reorder,
/// half the upload (edaa_ingest_host_f32).
std::pair<RunResult, SelectionReport> run_ensemble_raw_f32(const float* x, std::size_t bands, std::size_t pixels,
                                                           bool pixel_major, const EnsembleConfig& config,
                                                           std::size_t& zero_pixels);

/// NPY payload without widening: shape, dtype and the raw little-endian bytes.
struct NpyPayload {
  std::vector<std::size_t> shape;
  NpyDtype dtype = NpyDtype::f8;
  std::vector<float> f32;    // when dtype == f4
  std::vector<double> f64;   // when dtype == f8
};
/// read_npy's parsing and messages, keeping an f4 payload in fp32.
NpyPayload read_npy_payload(const std::string& path);

}  // namespace archetype::detail
