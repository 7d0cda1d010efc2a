// Pass-kernel instantiations for a double image (split for parallel compilation).
#include "edaa_pass.cuh"

namespace edaa {
cudaError_t launch_pass_f64(int mode, const PassArgs& a, cudaStream_t st) {
  return pass_impl::launch_pass_xt<double>(mode, a, st);
}
}  // namespace edaa
