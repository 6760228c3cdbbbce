// Step-kernel instantiation unit: launch_poisson_greedy_noisy_large (mode 0, policy 3,
// small class set = false, noisy lookahead = true). One unit per variant so nvcc
// compiles them in parallel.
#include "engine_impl.cuh"

namespace bfsim {
BFSIM_DEFINE_UNIT(launch_poisson_greedy_noisy_large, 0, 3, false, true)
}  // namespace bfsim
