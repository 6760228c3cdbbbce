// Step-kernel instantiations for mode 1 (overloaded), policy 0.
#include "engine_impl.cuh"

namespace bfsim {
int launch_family_1_0(int wpl, int small, int all_smem, const KParams& kp, int grid, int wpc,
                          cudaStream_t s, int* occ) {
  return detail::launch_family<1, 0>(wpl, small, all_smem, kp, grid, wpc, s, occ);
}
}  // namespace bfsim
