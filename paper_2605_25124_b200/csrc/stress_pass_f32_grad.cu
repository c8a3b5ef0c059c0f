// Instantiation: stress_pass_kernel<Q, float, true, KIND> for Q in 1..4, every kind.
#include "stress_pass.cuh"

namespace gmds {
GMDS_INSTANTIATE_PASS(float, true)
}  // namespace gmds
