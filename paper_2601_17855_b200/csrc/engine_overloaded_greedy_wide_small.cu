// Step-kernel instantiation unit: launch_overloaded_greedy_wide_small (mode 1, bfio-greedy with a
// lookahead window on G > 128 workers, small class set = true): the
// wide CTA of ceil(G / 128) warps that share the placement chain.
#include "engine_impl.cuh"

namespace bfsim {
BFSIM_DEFINE_WIDE_UNIT(launch_overloaded_greedy_wide_small, 1, true)
}  // namespace bfsim
