// Pass-kernel instantiations: float image, kModeA (p buckets 6-16).
// (One translation unit per mode so the kernels compile in parallel.)
#include "edaa_pass.cuh"

namespace edaa {
cudaError_t launch_pass_f32_ahi(const PassArgs& a, cudaStream_t st) {
  return pass_impl::launch_pass_mode<kModeA, float, pass_impl::kPtHi>(a, st);
}
}  // namespace edaa
