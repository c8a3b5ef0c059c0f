// Instantiation: fp32-storage fused trial pass (stress_tma.cuh, MODE 2): the
// losses of two Armijo trial points and the gradient at the first.
#include "stress_tma.cuh"

namespace gmds {
GMDS_INSTANTIATE_TMA_FUSED
}  // namespace gmds
