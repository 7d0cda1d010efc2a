// Pass-kernel instantiations for a float image (split for parallel compilation).
#include "edaa_pass.cuh"

namespace edaa {
cudaError_t launch_pass_f32(int mode, const PassArgs& a, cudaStream_t st) {
  return pass_impl::launch_pass_xt<float>(mode, a, st);
}
}  // namespace edaa
