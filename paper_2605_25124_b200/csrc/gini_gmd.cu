// Instantiation + launcher of the linear-weight Gini kernel (gini_gmd.cuh).
#include "gini_gmd.cuh"

namespace gmds {

void launch_gini_gmd(const GmdArgs& ga, void* dout, gmds_dtype ot, size_t smem, unsigned blocks, cudaStream_t st) {
  if (ot == GMDS_F32) {
    GMDS_CUDA(cudaFuncSetAttribute(gini_gmd_kernel<float>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   static_cast<int>(smem)));
    gini_gmd_kernel<float><<<blocks, gmd_detail::kThreads, smem, st>>>(ga, static_cast<float*>(dout));
  } else {
    GMDS_CUDA(cudaFuncSetAttribute(gini_gmd_kernel<double>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   static_cast<int>(smem)));
    gini_gmd_kernel<double><<<blocks, gmd_detail::kThreads, smem, st>>>(ga, static_cast<double*>(dout));
  }
}

}  // namespace gmds
