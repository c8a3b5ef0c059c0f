// Instantiations + launcher of the linear-weight Gini kernel (gini_gmd.cuh).
#include "gini_gmd.cuh"

namespace gmds {

template <typename TO, int NW>
static void launch_one(const GmdArgs& ga, TO* out, size_t smem, unsigned blocks, cudaStream_t st) {
  GMDS_CUDA(cudaFuncSetAttribute(gini_gmd_kernel<TO, NW>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 static_cast<int>(smem)));
  gini_gmd_kernel<TO, NW><<<blocks, NW * 32, smem, st>>>(ga, out);
}

template <typename TO>
static void launch_t(const GmdArgs& ga, TO* out, size_t smem, unsigned blocks, int nwarps, cudaStream_t st) {
  switch (nwarps) {
    case 32: launch_one<TO, 32>(ga, out, smem, blocks, st); break;
    case 28: launch_one<TO, 28>(ga, out, smem, blocks, st); break;
    default: launch_one<TO, 24>(ga, out, smem, blocks, st); break;
  }
}

void launch_gini_gmd(const GmdArgs& ga, void* dout, gmds_dtype ot, size_t smem, unsigned blocks, int nwarps,
                     cudaStream_t st) {
  if (ot == GMDS_F32)
    launch_t(ga, static_cast<float*>(dout), smem, blocks, nwarps, st);
  else
    launch_t(ga, static_cast<double*>(dout), smem, blocks, nwarps, st);
}

}  // namespace gmds
