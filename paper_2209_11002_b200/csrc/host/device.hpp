// Internal: the process-wide device contexts behind the archetype:: API.
#pragma once

#include <mutex>
#include <string>

#include "archetype/error.hpp"
#include "archetype/matrix.hpp"
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

}  // namespace archetype::detail
