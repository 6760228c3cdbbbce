// Dispatch from (mode, policy, class-set kind, noisy) to the instantiation units.
#include <cuda_runtime.h>

#include "engine_impl.cuh"

namespace bfsim {

int launch_step_kernel(int mode, int policy, int wpl, int small_classes, int noisy, int hr,
                       const KParams& kp, int grid, int wpc, void* stream, int* occupancy) {
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const bool ovl = mode == BFSIM_MODE_OVERLOADED;
  switch (policy) {
    case BFSIM_POLICY_FCFS:
      return ovl ? launch_overloaded_fcfs(wpl, hr, kp, grid, wpc, s, occupancy)
                 : launch_poisson_fcfs(wpl, hr, kp, grid, wpc, s, occupancy);
    case BFSIM_POLICY_JSQ:
      return ovl ? launch_overloaded_jsq(wpl, hr, kp, grid, wpc, s, occupancy)
                 : launch_poisson_jsq(wpl, hr, kp, grid, wpc, s, occupancy);
    case BFSIM_POLICY_BFIO_GREEDY:
      if (hr == 1)  // wide trajectories (G > 128 with a lookahead window): a CTA of wpc warps each
        return ovl ? (small_classes ? launch_overloaded_greedy_wide_small(wpl, kp, grid, wpc, s, occupancy)
                                    : launch_overloaded_greedy_wide_large(wpl, kp, grid, wpc, s, occupancy))
                   : (small_classes ? launch_poisson_greedy_wide_small(wpl, kp, grid, wpc, s, occupancy)
                                    : launch_poisson_greedy_wide_large(wpl, kp, grid, wpc, s, occupancy));
      if (ovl)
        return small_classes ? launch_overloaded_greedy_small(wpl, hr, kp, grid, wpc, s, occupancy)
                             : launch_overloaded_greedy_large(wpl, hr, kp, grid, wpc, s, occupancy);
      if (noisy)
        return small_classes ? launch_poisson_greedy_noisy_small(wpl, hr, kp, grid, wpc, s, occupancy)
                             : launch_poisson_greedy_noisy_large(wpl, hr, kp, grid, wpc, s, occupancy);
      return small_classes ? launch_poisson_greedy_small(wpl, hr, kp, grid, wpc, s, occupancy)
                           : launch_poisson_greedy_large(wpl, hr, kp, grid, wpc, s, occupancy);
  }
  return static_cast<int>(cudaErrorInvalidValue);
}

}  // namespace bfsim
