// Pass-kernel instantiations: double image, kModeA (p buckets 6-16).
// (One translation unit per mode so the kernels compile in parallel.)
#include "edaa_pass.cuh"

namespace edaa {
cudaError_t launch_pass_f64_ahi(const PassArgs& a, cudaStream_t st) {
  return pass_impl::launch_pass_mode<kModeA, double, pass_impl::kPtHi>(a, st);
}
}  // namespace edaa
