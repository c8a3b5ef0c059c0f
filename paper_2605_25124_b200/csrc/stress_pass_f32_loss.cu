// Instantiation: fp32-storage stress pass (TMA-streamed, stress_tma.cuh), GRAD=false.
#include "stress_tma.cuh"

namespace gmds {
GMDS_INSTANTIATE_TMA(false)
}  // namespace gmds
