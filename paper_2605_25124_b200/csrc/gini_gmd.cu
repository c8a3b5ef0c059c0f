// Instantiations + launcher of the linear-weight Gini kernel (gini_gmd.cuh).
#include <algorithm>

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

template <typename TO, int NW>
static void launch2_one(const GmdArgs& ga, TO* out, size_t smem, unsigned blocks, cudaStream_t st) {
  GMDS_CUDA(cudaFuncSetAttribute(gini_gmd2_kernel<TO, NW>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 static_cast<int>(smem)));
  gini_gmd2_kernel<TO, NW><<<blocks, NW * 32, smem, st>>>(ga, out);
}

void launch_gini_gmd2(const GmdArgs& ga, void* dout, gmds_dtype ot, size_t smem, unsigned blocks, int nwarps,
                      cudaStream_t st) {
  if (ot == GMDS_F32) {
    if (nwarps >= 28) launch2_one<float, 28>(ga, static_cast<float*>(dout), smem, blocks, st);
    else launch2_one<float, 24>(ga, static_cast<float*>(dout), smem, blocks, st);
  } else {
    if (nwarps >= 28) launch2_one<double, 28>(ga, static_cast<double*>(dout), smem, blocks, st);
    else launch2_one<double, 24>(ga, static_cast<double*>(dout), smem, blocks, st);
  }
}

// bkt[row][b] = #{k : bucket(v_(k)) < b}, bucket(v) = min(255, int(v * bscale[row])) -- the same
// float expression gini_gmd2_kernel evaluates for its query; rows of more than 255 nonzeros are
// never searched (they take the overflow list)
__global__ void row_bucket_kernel(const float* __restrict__ svs, const int64_t* __restrict__ rowptr, int64_t n,
                                  uint8_t* __restrict__ bkt, float* __restrict__ bscale) {
  for (int64_t row = blockIdx.x; row < n; row += gridDim.x) {
    const int64_t b0 = rowptr[row];
    const int cnt = static_cast<int>(min(rowptr[row + 1] - b0, static_cast<int64_t>(255)));
    const float* sv = svs + b0;
    const float scale = (cnt > 0 && sv[cnt - 1] > 0.f) ? 256.f / sv[cnt - 1] : 0.f;
    const int b = threadIdx.x;  // 256 threads: one bucket each
    int lo = 0, hi = cnt;       // smallest k with bucket(sv[k]) >= b
    while (lo < hi) {
      const int mid = (lo + hi) >> 1;
      if (min(255, __float2int_rz(sv[mid] * scale)) < b) lo = mid + 1; else hi = mid;
    }
    bkt[row * 256 + b] = static_cast<uint8_t>(lo);
    if (b == 0) bscale[row] = scale;
  }
}

void launch_row_buckets(const float* svs, const int64_t* rowptr, int64_t n, uint8_t* bkt, float* bscale,
                        cudaStream_t st) {
  if (n <= 0) return;
  row_bucket_kernel<<<static_cast<unsigned>(std::min<int64_t>(n, 148 * 16)), 256, 0, st>>>(svs, rowptr, n, bkt, bscale);
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

template <typename TO, int NW, int NNU>
static void launch_gen2_one(const GmdArgs& ga, TO* out, size_t smem, unsigned blocks, cudaStream_t st) {
  GMDS_CUDA(cudaFuncSetAttribute(gini_gen2_kernel<TO, NW, NNU>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 static_cast<int>(smem)));
  gini_gen2_kernel<TO, NW, NNU><<<blocks, NW * 32, smem, st>>>(ga, out);
}

template <typename TO>
static void launch_gen2_t(const GmdArgs& ga, TO* out, size_t smem, unsigned blocks, int nwarps, cudaStream_t st) {
  const bool one = ga.s.g.nnu == 1;
  if (nwarps >= 28) {
    if (one) launch_gen2_one<TO, 28, 1>(ga, out, smem, blocks, st);
    else launch_gen2_one<TO, 28, 4>(ga, out, smem, blocks, st);
  } else {
    if (one) launch_gen2_one<TO, 24, 1>(ga, out, smem, blocks, st);
    else launch_gen2_one<TO, 24, 4>(ga, out, smem, blocks, st);
  }
}

void launch_gini_gen2(const GmdArgs& ga, void* dout, gmds_dtype ot, size_t smem, unsigned blocks, int nwarps,
                      cudaStream_t st) {
  if (ga.s.g.nnu > 4) fail(GMDS_ERROR, "gini_gen2_kernel: at most 4 nu per launch");
  if (ot == GMDS_F32)
    launch_gen2_t(ga, static_cast<float*>(dout), smem, blocks, nwarps, st);
  else
    launch_gen2_t(ga, static_cast<double*>(dout), smem, blocks, nwarps, st);
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
