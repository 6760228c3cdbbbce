// Step-kernel instantiation unit: launch_poisson_greedy_noisy_small (mode 0, policy 3,
// small class set = true, noisy lookahead = true). One unit per variant so nvcc
// compiles them in parallel.
#include "engine_impl.cuh"

namespace bfsim {
BFSIM_DEFINE_UNIT(launch_poisson_greedy_noisy_small, 0, 3, true, true)
}  // namespace bfsim
