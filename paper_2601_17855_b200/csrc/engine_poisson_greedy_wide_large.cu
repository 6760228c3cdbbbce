// Step-kernel instantiation unit: launch_poisson_greedy_wide_large (mode 0, bfio-greedy with a
// lookahead window on G > 128 workers, small class set = false): the
// wide CTA of ceil(G / 128) warps that share the placement chain.
#include "engine_impl.cuh"

namespace bfsim {
BFSIM_DEFINE_WIDE_UNIT(launch_poisson_greedy_wide_large, 0, false)
}  // namespace bfsim
