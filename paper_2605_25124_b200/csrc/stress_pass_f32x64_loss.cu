// Instantiation: stress_pass_kernel<Q, float, false, KIND, double> -- loss passes over
// fp32-stored D in fp64 arithmetic (Engine::loss_raw_precise).
#include "stress_pass.cuh"

namespace gmds {
void launch_pass_precise(const PassArgs& a, int Q, cudaStream_t st) {
  const unsigned g = static_cast<unsigned>(a.nchunks);
  switch (Q) {
    GMDS_PRECISE_Q(1) GMDS_PRECISE_Q(2) GMDS_PRECISE_Q(3) GMDS_PRECISE_Q(4)
    default: fail(GMDS_ERROR, "stress pass: unsupported padded dimension");
  }
  count_launch();
  check_launch("stress_pass_kernel (precise)");
}
}  // namespace gmds
