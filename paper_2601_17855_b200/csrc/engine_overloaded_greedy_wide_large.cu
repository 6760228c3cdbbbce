// Step-kernel instantiation unit: launch_overloaded_greedy_wide_large (mode 1, bfio-greedy with a
// lookahead window on G > 128 workers, small class set = false): the
// wide CTA of ceil(G / 128) warps that share the placement chain.
#include "engine_impl.cuh"

namespace bfsim {
BFSIM_DEFINE_WIDE_UNIT(launch_overloaded_greedy_wide_large, 1, false)
}  // namespace bfsim
