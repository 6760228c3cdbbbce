// Step-kernel instantiations for mode 0 (Poisson), policy 3.
#include "engine_impl.cuh"

namespace bfsim {
int launch_family_0_3(int wpl, int small, int all_smem, const KParams& kp, int grid, int wpc,
                          cudaStream_t s, int* occ) {
  return detail::launch_family<0, 3>(wpl, small, all_smem, kp, grid, wpc, s, occ);
}
}  // namespace bfsim
