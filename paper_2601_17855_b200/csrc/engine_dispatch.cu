// Dispatch from (mode, policy) to the per-family instantiation units.
#include <cuda_runtime.h>

#include "engine_impl.cuh"

namespace bfsim {

int launch_step_kernel(int mode, int policy, int wpl, int small_classes, const KParams& kp,
                       int grid, int wpc, void* stream, int* occupancy) {
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const bool ovl = mode == BFSIM_MODE_OVERLOADED;
  switch (policy) {
    case BFSIM_POLICY_FCFS:
      return ovl ? launch_family_1_0(wpl, small_classes, kp.plan.all_smem, kp, grid, wpc, s, occupancy)
                 : launch_family_0_0(wpl, small_classes, kp.plan.all_smem, kp, grid, wpc, s, occupancy);
    case BFSIM_POLICY_JSQ:
      return ovl ? launch_family_1_1(wpl, small_classes, kp.plan.all_smem, kp, grid, wpc, s, occupancy)
                 : launch_family_0_1(wpl, small_classes, kp.plan.all_smem, kp, grid, wpc, s, occupancy);
    case BFSIM_POLICY_BFIO_GREEDY:
      return ovl ? launch_family_1_3(wpl, small_classes, kp.plan.all_smem, kp, grid, wpc, s, occupancy)
                 : launch_family_0_3(wpl, small_classes, kp.plan.all_smem, kp, grid, wpc, s, occupancy);
  }
  return static_cast<int>(cudaErrorInvalidValue);
}

}  // namespace bfsim
