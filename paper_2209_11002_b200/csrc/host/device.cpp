#include "device.hpp"

#include <algorithm>
#include <cstdlib>
#include <memory>
#include <vector>

namespace archetype::detail {

namespace {

struct Registry {
  std::mutex mu;
  int count = -1;
  std::vector<std::unique_ptr<Device>> devices;
};

Registry& registry() {
  static Registry r;
  return r;
}

}  // namespace

int device_count() {
  Registry& r = registry();
  std::lock_guard<std::mutex> lock(r.mu);
  if (r.count < 0) {
    // Probe by creating contexts until one fails; EDAA_DEVICES caps the count.
    int cap = 64;
    if (const char* env = std::getenv("EDAA_DEVICES")) cap = std::max(1, std::atoi(env));
    while (static_cast<int>(r.devices.size()) < cap) {
      auto d = std::make_unique<Device>();
      d->ordinal = static_cast<int>(r.devices.size());
      if (edaa_create(d->ordinal, &d->ctx) != EDAA_OK) break;
      r.devices.push_back(std::move(d));
    }
    // EDAA_VIRTUAL_DEVICES=K (K > visible GPUs): K contexts placed round-robin on
    // the visible GPUs, each with its own stream and buffers.  run_ensemble then
    // takes its multi-device branch (one host thread and one shard of the runs
    // per context, host-side select_runs) on a single GPU — how the tests cover
    // that branch on a one-GPU box.
    if (const char* env = std::getenv("EDAA_VIRTUAL_DEVICES")) {
      const int real = static_cast<int>(r.devices.size());
      const int want = std::min(64, std::atoi(env));
      while (real > 0 && static_cast<int>(r.devices.size()) < want) {
        auto d = std::make_unique<Device>();
        d->ordinal = static_cast<int>(r.devices.size());
        if (edaa_create(d->ordinal % real, &d->ctx) != EDAA_OK) break;
        r.devices.push_back(std::move(d));
      }
    }
    r.count = static_cast<int>(r.devices.size());
  }
  if (r.count == 0)
    throw Error("edaa: no usable CUDA device (this library has no CPU fallback)");
  return r.count;
}

Device& device(int i) {
  const int n = device_count();
  if (i < 0 || i >= n) throw Error("edaa: device index out of range");
  return *registry().devices[static_cast<std::size_t>(i)];
}

void fail(const Device& d, const std::string& what) {
  throw Error(what + ": " + edaa_last_error(d.ctx));
}

void upload_image(Device& d, const Matrix& x) {
  const auto v = x.values();
  bool exact = true;
  for (double e : v) {
    if (static_cast<double>(static_cast<float>(e)) != e) {
      exact = false;
      break;
    }
  }
  int rc;
  if (exact) {
    std::vector<float> f(v.begin(), v.end());
    rc = edaa_set_image_host(d.ctx, f.data(), x.rows(), x.cols());
  } else {
    rc = edaa_set_image_host_f64(d.ctx, v.data(), x.rows(), x.cols());
  }
  if (rc != EDAA_OK) fail(d, "edaa: image upload failed");
}

}  // namespace archetype::detail
