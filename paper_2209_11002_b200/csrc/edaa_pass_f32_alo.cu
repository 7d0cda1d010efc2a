// Pass-kernel instantiations: float image, kModeA (p buckets 2-5).
// (One translation unit per mode so the kernels compile in parallel.)
#include "edaa_pass.cuh"

namespace edaa {
cudaError_t launch_pass_f32_alo(const PassArgs& a, cudaStream_t st) {
  return pass_impl::launch_pass_mode<kModeA, float, pass_impl::kPtLo>(a, st);
}
}  // namespace edaa
