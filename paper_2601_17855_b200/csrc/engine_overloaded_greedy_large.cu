// Step-kernel instantiation unit: launch_overloaded_greedy_large (mode 1, policy 3,
// small class set = false, noisy lookahead = false). One unit per variant so nvcc
// compiles them in parallel.
#include "engine_impl.cuh"

namespace bfsim {
BFSIM_DEFINE_UNIT(launch_overloaded_greedy_large, 1, 3, false, false)
}  // namespace bfsim
