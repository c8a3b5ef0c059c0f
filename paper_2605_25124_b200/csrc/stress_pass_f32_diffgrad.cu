// Instantiation: stress_tma_kernel<Q, 6 | 7, kruskal> -- the device loop's tiny-phase pass:
// loss differences of the trial steps plus the gradient at the first trial point.
#include "stress_tma.cuh"

namespace gmds {
GMDS_INSTANTIATE_TMA_DG
}  // namespace gmds
