// C-ABI: the remaining metrics.hpp / embed.hpp entry points of the drop-in
// (directed distance, Gini norm / pseudo-distance, Hazen survival,
// double-centring).  Ranks come from the exact warp midrank kernel; the
// per-term factors are tabulated on the host with the reference's own
// expressions and std::pow, and the reductions run on the device.
#include <cmath>
#include <cstring>
#include <string>
#include <vector>

#include "common.cuh"
#include "dmat_kernels.cuh"
#include "kernels.cuh"
#include "lib_internal.h"

namespace gmds {

namespace {

// out = scale * sum_k z_k * L[2 R_k - 1], z = x - y (fp64), one block.
__global__ void dot_lut_kernel(const double* __restrict__ x, const double* __restrict__ y, int d,
                               const double* __restrict__ ranks, const double* __restrict__ L, double scale,
                               double* __restrict__ out) {
  __shared__ double red[256];
  double s = 0.0;
  for (int k = threadIdx.x; k < d; k += blockDim.x) {
    const double z = y ? x[k] - y[k] : x[k];
    const int h = static_cast<int>(2.0 * ranks[k] - 1.0);
    s += z * L[h];
  }
  red[threadIdx.x] = s;
  __syncthreads();
  for (int w = blockDim.x / 2; w > 0; w >>= 1) {
    if (threadIdx.x < w) red[threadIdx.x] += red[threadIdx.x + w];
    __syncthreads();
  }
  if (threadIdx.x == 0) *out = scale * red[0];
}

__global__ void survival_kernel(const double* __restrict__ ranks, int d, double* __restrict__ out) {
  const double inv_d = 1.0 / static_cast<double>(d);
  for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < d; k += gridDim.x * blockDim.x)
    out[k] = __dsub_rn(1.0, __dmul_rn(ranks[k] - 0.5, inv_d));  // metrics.cpp:142 (no FMA contraction)
}

void check_len_finite(const double* x, int64_t dx, const double* y, int64_t dy, const char* who) {
  if (y && dx != dy)
    fail(GMDS_INVALID_INPUT,
         std::string(who) + ": length mismatch (" + std::to_string(dx) + " vs " + std::to_string(dy) + ")");
  if (dx < 1) fail(GMDS_INVALID_INPUT, std::string(who) + ": input vector is empty");
  check_finite_host(x, GMDS_F64, dx, who);
  if (y) check_finite_host(y, GMDS_F64, dy, who);
}

// ranks of z (= x - y, or x) on the device; returns the device buffers
struct DeviceRanks {
  DevBuf<double> xy, ranks;
};

DeviceRanks ranks_of(const double* x, const double* y, int64_t d, cudaStream_t st) {
  DeviceRanks r;
  r.xy.alloc(static_cast<size_t>(2 * d));
  r.ranks.alloc(static_cast<size_t>(d));
  GMDS_CUDA(cudaMemcpyAsync(r.xy.get(), x, sizeof(double) * d, cudaMemcpyHostToDevice, st));
  if (y) {
    GMDS_CUDA(cudaMemcpyAsync(r.xy.get() + d, y, sizeof(double) * d, cudaMemcpyHostToDevice, st));
    DevBuf<int64_t> pr(2);
    const int64_t hp[2] = {0, 1};
    GMDS_CUDA(cudaMemcpyAsync(pr.get(), hp, sizeof hp, cudaMemcpyHostToDevice, st));
    launch_midrank(nullptr, r.xy.get(), GMDS_F64, pr.get(), 1, static_cast<int>(d), r.ranks.get(), st);
    GMDS_CUDA(cudaStreamSynchronize(st));
  } else {
    launch_midrank(r.xy.get(), nullptr, GMDS_F64, nullptr, 1, static_cast<int>(d), r.ranks.get(), st);
  }
  return r;
}

double dot_lut(const DeviceRanks& r, int64_t d, bool diff, const std::vector<double>& L, double scale, cudaStream_t st) {
  DevBuf<double> dL(L.size()), out(1);
  GMDS_CUDA(cudaMemcpyAsync(dL.get(), L.data(), L.size() * sizeof(double), cudaMemcpyHostToDevice, st));
  dot_lut_kernel<<<1, 256, 0, st>>>(r.xy.get(), diff ? r.xy.get() + d : nullptr, static_cast<int>(d), r.ranks.get(),
                                    dL.get(), scale, out.get());
  count_launch();
  check_launch("dot_lut_kernel");
  double h = 0.0;
  GMDS_CUDA(cudaMemcpyAsync(&h, out.get(), sizeof h, cudaMemcpyDeviceToHost, st));
  GMDS_CUDA(cudaStreamSynchronize(st));
  return h;
}

// gini_norm_impl (metrics.cpp:58-66): L[h] = R - (d+1)/2
std::vector<double> centered_rank_table(int64_t d) {
  std::vector<double> L(static_cast<size_t>(2 * d), 0.0);
  const double center = 0.5 * static_cast<double>(d + 1);
  for (int64_t h = 1; h < 2 * d; ++h) L[h] = 0.5 * static_cast<double>(h + 1) - center;
  return L;
}

// gen_gini_directed_impl (metrics.cpp:73-79): L[h] = pow(S(R), nu-1) - pow(0.5, nu-1), scale -d
std::vector<double> survival_pow_table(int64_t d, double nu) {
  std::vector<double> L(static_cast<size_t>(2 * d), 0.0);
  const double exponent = nu - 1.0;
  const double inv_d = 1.0 / static_cast<double>(d);
  const double c = std::pow(0.5, exponent);
  for (int64_t h = 1; h < 2 * d; ++h) {
    const double rank = 0.5 * static_cast<double>(h + 1);
    L[h] = std::pow(1.0 - (rank - 0.5) * inv_d, exponent) - c;
  }
  return L;
}

}  // namespace

}  // namespace gmds

using namespace gmds;

extern "C" {

gmds_status gmds_gen_gini_directed(const double* x, int64_t dx, const double* y, int64_t dy, double nu, double* out) {
  return guard([&] {
    check_nu(nu);
    check_len_finite(x, dx, y, dy, "gen_gini_directed");
    require_device();
    Stream st;
    const DeviceRanks r = ranks_of(x, y, dx, st.s);
    *out = dot_lut(r, dx, true, survival_pow_table(dx, nu), -static_cast<double>(dx), st.s);
  });
}

gmds_status gmds_gini_norm(const double* x, int64_t d, double* out) {
  return guard([&] {
    check_len_finite(x, d, nullptr, 0, "gini_norm");
    require_device();
    Stream st;
    const DeviceRanks r = ranks_of(x, nullptr, d, st.s);
    *out = dot_lut(r, d, false, centered_rank_table(d), 1.0, st.s);
  });
}

gmds_status gmds_gini_pseudo_distance(const double* x, int64_t dx, const double* y, int64_t dy, double* out) {
  return guard([&] {
    check_len_finite(x, dx, y, dy, "gini_pseudo_distance");
    require_device();
    Stream st;
    const DeviceRanks r = ranks_of(x, y, dx, st.s);
    *out = dot_lut(r, dx, true, centered_rank_table(dx), 1.0, st.s);
  });
}

gmds_status gmds_empirical_survival(const double* z, int64_t d, double* out) {
  return guard([&] {
    check_len_finite(z, d, nullptr, 0, "empirical_survival");
    require_device();
    Stream st;
    const DeviceRanks r = ranks_of(z, nullptr, d, st.s);
    DevBuf<double> dout(static_cast<size_t>(d));
    survival_kernel<<<static_cast<unsigned>(std::min<int64_t>(ceil_div(d, 256), 1024)), 256, 0, st.s>>>(
        r.ranks.get(), static_cast<int>(d), dout.get());
    count_launch();
    check_launch("survival_kernel");
    GMDS_CUDA(cudaMemcpyAsync(out, dout.get(), sizeof(double) * d, cudaMemcpyDeviceToHost, st.s));
    GMDS_CUDA(cudaStreamSynchronize(st.s));
  });
}

gmds_status gmds_double_center(const double* S, int64_t n, double* B) {
  return guard([&] {
    // validation of double_center (embed.cpp:382-397), in the reference's order
    if (n < 1) fail(GMDS_INVALID_INPUT, "double_center: matrix is not square");
    double scale = 0.0;
    for (int64_t k = 0; k < n * n; ++k) {
      if (!std::isfinite(S[k])) fail(GMDS_INVALID_INPUT, "double_center: non-finite entry");
      scale = std::max(scale, std::abs(S[k]));
    }
    scale = std::max(scale, 1.0);
    const double tol = 1e-9 * scale;
    for (int64_t i = 0; i < n; ++i) {
      if (std::abs(S[i * n + i]) > tol) fail(GMDS_INVALID_INPUT, "double_center: nonzero diagonal");
      for (int64_t j = i + 1; j < n; ++j) {
        if (std::abs(S[j * n + i] - S[i * n + j]) > tol)
          fail(GMDS_INVALID_INPUT, "double_center: asymmetric input beyond tolerance");
        if (S[j * n + i] < -tol) fail(GMDS_INVALID_INPUT, "double_center: negative squared distance");
      }
    }
    require_device();
    Stream st;
    DevBuf<double> d(static_cast<size_t>(n * n));
    // column-major S: transpose on upload so row i of the device image is S(i, :)
    std::vector<double> rm(static_cast<size_t>(n * n));
    for (int64_t i = 0; i < n; ++i)
      for (int64_t j = 0; j < n; ++j) rm[i * n + j] = S[j * n + i];
    GMDS_CUDA(cudaMemcpyAsync(d.get(), rm.data(), rm.size() * sizeof(double), cudaMemcpyHostToDevice, st.s));
    double_center_dev(d.get(), n, st.s);  // symmetric output: row-/column-major images coincide
    GMDS_CUDA(cudaMemcpyAsync(B, d.get(), sizeof(double) * n * n, cudaMemcpyDeviceToHost, st.s));
    GMDS_CUDA(cudaStreamSynchronize(st.s));
  });
}

}  // extern "C"
