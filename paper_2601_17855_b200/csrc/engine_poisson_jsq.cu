// Step-kernel instantiation unit: launch_poisson_jsq (mode 0, policy 1,
// small class set = true, noisy lookahead = false). One unit per variant so nvcc
// compiles them in parallel.
#include "engine_impl.cuh"

namespace bfsim {
BFSIM_DEFINE_UNIT(launch_poisson_jsq, 0, 1, true, false)
}  // namespace bfsim
