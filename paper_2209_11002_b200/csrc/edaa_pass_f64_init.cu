// Pass-kernel instantiations: double image, kModeInit.
// (One translation unit per mode so the kernels compile in parallel.)
#include "edaa_pass.cuh"

namespace edaa {
cudaError_t launch_pass_f64_init(const PassArgs& a, cudaStream_t st) {
  return pass_impl::launch_pass_mode<kModeInit, double>(a, st);
}
}  // namespace edaa
