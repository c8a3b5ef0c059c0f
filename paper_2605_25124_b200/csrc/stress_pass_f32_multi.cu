// Instantiation: the device loop's merged pass launches (stress_tma.cuh,
// stress_tma_multi_kernel): kruskal, q <= 3.
#include "stress_tma.cuh"

namespace gmds {
GMDS_INSTANTIATE_TMA_MULTI
}  // namespace gmds
