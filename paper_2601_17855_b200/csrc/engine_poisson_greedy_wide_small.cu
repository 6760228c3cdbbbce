// Step-kernel instantiation unit: launch_poisson_greedy_wide_small (mode 0, bfio-greedy with a
// lookahead window on G > 128 workers, small class set = true): the
// wide CTA of ceil(G / 128) warps that share the placement chain.
#include "engine_impl.cuh"

namespace bfsim {
BFSIM_DEFINE_WIDE_UNIT(launch_poisson_greedy_wide_small, 0, true)
}  // namespace bfsim
