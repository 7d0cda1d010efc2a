// Pass-kernel instantiations: float image, kModeObj.
// (One translation unit per mode so the kernels compile in parallel.)
#include "edaa_pass.cuh"

namespace edaa {
cudaError_t launch_pass_f32_obj(const PassArgs& a, cudaStream_t st) {
  return pass_impl::launch_pass_mode<kModeObj, float>(a, st);
}
}  // namespace edaa
