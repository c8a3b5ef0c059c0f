// Instantiation: stress_tma_kernel<Q, 3, KIND> -- loss differences of two trial steps over
// fp32 storage (Engine::loss_diff).
#include "stress_tma.cuh"

namespace gmds {
GMDS_INSTANTIATE_TMA_DIFF
GMDS_INSTANTIATE_TMA_DIFF1
}  // namespace gmds
