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

template <typename TO, int NW, int NNU>
static void launch_gen_one(const GmdArgs& ga, TO* out, size_t smem, unsigned blocks, cudaStream_t st) {
  GMDS_CUDA(cudaFuncSetAttribute(gini_gen_kernel<TO, NW, NNU>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 static_cast<int>(smem)));
  gini_gen_kernel<TO, NW, NNU><<<blocks, NW * 32, smem, st>>>(ga, out);
}

template <typename TO>
static void launch_gen_t(const GmdArgs& ga, TO* out, size_t smem, unsigned blocks, int nwarps, cudaStream_t st) {
  const bool one = ga.s.g.nnu == 1;
  if (nwarps >= 28) {
    if (one) launch_gen_one<TO, 28, 1>(ga, out, smem, blocks, st);
    else launch_gen_one<TO, 28, 4>(ga, out, smem, blocks, st);
  } else {
    if (one) launch_gen_one<TO, 24, 1>(ga, out, smem, blocks, st);
    else launch_gen_one<TO, 24, 4>(ga, out, smem, blocks, st);
  }
}

void launch_gini_gen(const GmdArgs& ga, void* dout, gmds_dtype ot, size_t smem, unsigned blocks, int nwarps,
                     cudaStream_t st) {
  if (ga.s.g.nnu > 4) fail(GMDS_ERROR, "gini_gen_kernel: at most 4 nu per launch");
  if (ot == GMDS_F32)
    launch_gen_t(ga, static_cast<float*>(dout), smem, blocks, nwarps, st);
  else
    launch_gen_t(ga, static_cast<double*>(dout), smem, blocks, nwarps, st);
}

}  // namespace gmds
