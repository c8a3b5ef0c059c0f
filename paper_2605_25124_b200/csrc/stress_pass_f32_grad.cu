// Instantiation: fp32-storage stress pass (TMA-streamed, stress_tma.cuh), GRAD=true.
#include "stress_tma.cuh"

namespace gmds {
GMDS_INSTANTIATE_TMA(true)
GMDS_INSTANTIATE_TMA_SOLO
}  // namespace gmds
