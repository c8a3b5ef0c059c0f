// Device-side DistanceMatrix utilities: packing, unpacking, statistics,
// median extraction and the double-centred Gram matrix of classical MDS.
#include <cub/cub.cuh>
#include <vector>
#include <math.h>

#include "common.cuh"
#include "dmat_kernels.cuh"
#include "kernels.cuh"

namespace gmds {

namespace {

__device__ __forceinline__ void unpack_index(int64_t e, int64_t nb, int64_t& i, int64_t& j) {
  // packed element -> (i, j) (row-major upper triangle of kPT blocks)
  const int64_t blk = e / (kPT * kPT), w = e % (kPT * kPT);
  const double b = 2.0 * static_cast<double>(nb) + 1.0;
  int64_t I = static_cast<int64_t>((b - sqrt(b * b - 8.0 * static_cast<double>(blk))) * 0.5);
  if (I < 0) I = 0;
  auto start = [nb](int64_t r) { return r * nb - (r * (r - 1)) / 2; };
  while (I > 0 && start(I) > blk) --I;
  while (start(I + 1) <= blk) ++I;
  const int64_t J = I + (blk - start(I));
  i = I * kPT + w / kPT;
  j = J * kPT + w % kPT;
}

}  // namespace

template <typename TD>
__global__ void pack_kernel(const double* __restrict__ full, int64_t n, int64_t nb, int64_t total, TD* __restrict__ out) {
  for (int64_t e = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; e < total;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    int64_t i, j;
    unpack_index(e, nb, i, j);
    out[e] = (i < j && j < n) ? static_cast<TD>(full[i * n + j]) : TD(0);
  }
}

template <typename TD>
__global__ void unpack_kernel(const TD* __restrict__ packed, int64_t n, int64_t nb, double* __restrict__ full, int square) {
  // full[i][j] = D_ij (or D_ij^2 when square) for all i, j (zero diagonal)
  const int64_t total = n * n;
  for (int64_t e = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; e < total;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t i = e / n, j = e % n;
    double v = 0.0;
    if (i != j) {
      const int64_t lo = i < j ? i : j, hi = i < j ? j : i;
      v = static_cast<double>(packed[packed_offset(lo, hi, nb)]);
      if (square) v = v * v;
    }
    full[e] = v;
  }
}

// Per-CTA partials over valid entries: [sum D^2, sum D, min D, max D].
template <typename TD>
__global__ void stats_kernel(const TD* __restrict__ packed, int64_t n, int64_t nb, int64_t ebeg, int64_t total,
                             double* __restrict__ part) {
  double s2 = 0.0, s1 = 0.0, mn = INFINITY, mx = -INFINITY;
  const int64_t per = (total - ebeg + gridDim.x - 1) / gridDim.x;
  const int64_t e0 = ebeg + blockIdx.x * per, e1 = min(total, e0 + per);
  for (int64_t e = e0 + threadIdx.x; e < e1; e += blockDim.x) {
    int64_t i, j;
    unpack_index(e, nb, i, j);
    if (i < j && j < n) {
      const double v = static_cast<double>(packed[e]);
      s2 += v * v;
      s1 += v;
      mn = fmin(mn, v);
      mx = fmax(mx, v);
    }
  }
  __shared__ double r[4][256];
  r[0][threadIdx.x] = s2;
  r[1][threadIdx.x] = s1;
  r[2][threadIdx.x] = mn;
  r[3][threadIdx.x] = mx;
  __syncthreads();
  for (int w = blockDim.x / 2; w > 0; w >>= 1) {
    if (threadIdx.x < w) {
      r[0][threadIdx.x] += r[0][threadIdx.x + w];
      r[1][threadIdx.x] += r[1][threadIdx.x + w];
      r[2][threadIdx.x] = fmin(r[2][threadIdx.x], r[2][threadIdx.x + w]);
      r[3][threadIdx.x] = fmax(r[3][threadIdx.x], r[3][threadIdx.x + w]);
    }
    __syncthreads();
  }
  if (threadIdx.x == 0)
    for (int k = 0; k < 4; ++k) part[blockIdx.x * 4 + k] = r[k][0];
}

template <typename TD>
__global__ void extract_upper_kernel(const TD* __restrict__ packed, int64_t n, double* __restrict__ out) {
  // out[k] for k-th pair in row-major strict-upper order
  const int64_t npairs = n * (n - 1) / 2;
  const int64_t nb = (n + kPT - 1) / kPT;
  for (int64_t k = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; k < npairs;
       k += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    // row i: pairs before = i*n - i*(i+1)/2
    const double b = 2.0 * static_cast<double>(n) - 1.0;
    int64_t i = static_cast<int64_t>((b - sqrt(b * b - 8.0 * static_cast<double>(k))) * 0.5);
    if (i < 0) i = 0;
    auto start = [n](int64_t r) { return r * n - (r * (r + 1)) / 2; };
    while (i > 0 && start(i) > k) --i;
    while (start(i + 1) <= k) ++i;
    const int64_t j = i + 1 + (k - start(i));
    out[k] = static_cast<double>(packed[packed_offset(i, j, nb)]);
  }
}

__global__ void row_mean_kernel(const double* __restrict__ S, int64_t n, double* __restrict__ r) {
  // r_i = (sum_j S_ij) / n, one warp per row
  const int lane = threadIdx.x & 31;
  for (int64_t i = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5; i < n;
       i += (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5) {
    double s = 0.0;
    for (int64_t j = lane; j < n; j += 32) s += S[i * n + j];
    for (int d = 16; d > 0; d >>= 1) s += __shfl_xor_sync(0xffffffffu, s, d);
    if (lane == 0) r[i] = s / static_cast<double>(n);
  }
}

__global__ void center_kernel(double* __restrict__ S, int64_t n, const double* __restrict__ r, double g) {
  // B = -1/2 (S - r_i - r_j + g), computed from the (i <= j) entry and mirrored (embed.cpp:399-411)
  const int64_t total = n * n;
  for (int64_t e = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; e < total;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t i = e / n, j = e % n;
    const int64_t a = i < j ? i : j, b = i < j ? j : i;
    S[e] = -0.5 * (S[e] - r[a] - r[b] + g);
  }
}

// ---------------------------------------------------------------------------
namespace {
unsigned grid_for(int64_t m) {
  return static_cast<unsigned>(std::max<int64_t>(1, std::min<int64_t>(ceil_div(m, 256), 148 * 64)));
}
}  // namespace

void pack_full(const double* dfull, int64_t n, gmds_dtype storage, void* dpacked, cudaStream_t st) {
  const int64_t nb = ceil_div(n, kPT), total = packed_elems(n);
  if (storage == GMDS_F32)
    pack_kernel<float><<<grid_for(total), 256, 0, st>>>(dfull, n, nb, total, static_cast<float*>(dpacked));
  else
    pack_kernel<double><<<grid_for(total), 256, 0, st>>>(dfull, n, nb, total, static_cast<double*>(dpacked));
  count_launch();
  check_launch("pack_kernel");
}

// rows [r0, r1) of the full matrix (zero diagonal) into out[(i - r0) * n + j]
template <typename TD>
__global__ void unpack_rows_kernel(const TD* __restrict__ packed, int64_t n, int64_t nb, int64_t r0, int64_t r1,
                                   double* __restrict__ out) {
  const int64_t total = (r1 - r0) * n;
  for (int64_t e = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; e < total;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t i = r0 + e / n, j = e % n;
    double v = 0.0;
    if (i != j) {
      const int64_t lo = i < j ? i : j, hi = i < j ? j : i;
      v = static_cast<double>(packed[packed_offset(lo, hi, nb)]);
    }
    out[e] = v;
  }
}

void unpack_rows(const void* dpacked, gmds_dtype storage, int64_t n, int64_t r0, int64_t r1, double* dout,
                 cudaStream_t st) {
  const int64_t nb = ceil_div(n, kPT);
  const unsigned g = grid_for((r1 - r0) * n);
  if (storage == GMDS_F32)
    unpack_rows_kernel<float><<<g, 256, 0, st>>>(static_cast<const float*>(dpacked), n, nb, r0, r1, dout);
  else
    unpack_rows_kernel<double><<<g, 256, 0, st>>>(static_cast<const double*>(dpacked), n, nb, r0, r1, dout);
  count_launch();
  check_launch("unpack_rows_kernel");
}

void unpack_full(const void* dpacked, gmds_dtype storage, int64_t n, double* dfull, bool square, cudaStream_t st) {
  const int64_t nb = ceil_div(n, kPT);
  if (storage == GMDS_F32)
    unpack_kernel<float><<<grid_for(n * n), 256, 0, st>>>(static_cast<const float*>(dpacked), n, nb, dfull, square);
  else
    unpack_kernel<double><<<grid_for(n * n), 256, 0, st>>>(static_cast<const double*>(dpacked), n, nb, dfull, square);
  count_launch();
  check_launch("unpack_kernel");
}

DStats packed_stats(const void* dpacked, gmds_dtype storage, int64_t n, cudaStream_t st, int64_t blk_lo,
                    int64_t blk_hi) {
  const int64_t nb = ceil_div(n, kPT);
  const int64_t ebeg = blk_lo * kPT * kPT;
  const int64_t total = blk_hi < 0 ? packed_elems(n) : blk_hi * kPT * kPT;  // elements [ebeg, total)
  const int blocks = static_cast<int>(std::min<int64_t>(1024, std::max<int64_t>(1, ceil_div(total - ebeg, 4096))));
  DevBuf<double> part(static_cast<size_t>(blocks) * 4);
  if (storage == GMDS_F32)
    stats_kernel<float><<<blocks, 256, 0, st>>>(static_cast<const float*>(dpacked), n, nb, ebeg, total, part.get());
  else
    stats_kernel<double><<<blocks, 256, 0, st>>>(static_cast<const double*>(dpacked), n, nb, ebeg, total, part.get());
  count_launch();
  check_launch("stats_kernel");
  std::vector<double> h(static_cast<size_t>(blocks) * 4);
  GMDS_CUDA(cudaMemcpyAsync(h.data(), part.get(), h.size() * sizeof(double), cudaMemcpyDeviceToHost, st));
  GMDS_CUDA(cudaStreamSynchronize(st));
  DStats s{0.0, 0.0, INFINITY, -INFINITY};
  for (int b = 0; b < blocks; ++b) {
    s.sum_sq += h[b * 4 + 0];
    s.sum += h[b * 4 + 1];
    s.min_off = std::min(s.min_off, h[b * 4 + 2]);
    s.max_off = std::max(s.max_off, h[b * 4 + 3]);
  }
  return s;
}

double packed_median(const void* dpacked, gmds_dtype storage, int64_t n, cudaStream_t st) {
  // median_offdiag (embed.cpp:36-46): sort all strict-upper entries, take the middle (mean of two if even)
  const int64_t m = n * (n - 1) / 2;
  DevBuf<double> vals(static_cast<size_t>(m)), sorted(static_cast<size_t>(m));
  if (storage == GMDS_F32)
    extract_upper_kernel<float><<<grid_for(m), 256, 0, st>>>(static_cast<const float*>(dpacked), n, vals.get());
  else
    extract_upper_kernel<double><<<grid_for(m), 256, 0, st>>>(static_cast<const double*>(dpacked), n, vals.get());
  count_launch();
  check_launch("extract_upper_kernel");
  size_t tmp_bytes = 0;
  GMDS_CUDA(cub::DeviceRadixSort::SortKeys(nullptr, tmp_bytes, vals.get(), sorted.get(), static_cast<int>(m), 0, 64, st));
  DevBuf<unsigned char> tmp(tmp_bytes);
  GMDS_CUDA(cub::DeviceRadixSort::SortKeys(tmp.get(), tmp_bytes, vals.get(), sorted.get(), static_cast<int>(m), 0, 64,
                                           st));
  count_launch();
  double mid[2] = {0, 0};
  if (m % 2 == 1) {
    GMDS_CUDA(cudaMemcpyAsync(mid, sorted.get() + m / 2, sizeof(double), cudaMemcpyDeviceToHost, st));
    GMDS_CUDA(cudaStreamSynchronize(st));
    return mid[0];
  }
  GMDS_CUDA(cudaMemcpyAsync(mid, sorted.get() + m / 2 - 1, 2 * sizeof(double), cudaMemcpyDeviceToHost, st));
  GMDS_CUDA(cudaStreamSynchronize(st));
  return 0.5 * (mid[0] + mid[1]);
}

void double_center_dev(double* dS, int64_t n, cudaStream_t st) {
  DevBuf<double> r(static_cast<size_t>(n));
  row_mean_kernel<<<grid_for(n * 32), 256, 0, st>>>(dS, n, r.get());
  count_launch();
  check_launch("row_mean_kernel");
  std::vector<double> hr(static_cast<size_t>(n));
  GMDS_CUDA(cudaMemcpyAsync(hr.data(), r.get(), n * sizeof(double), cudaMemcpyDeviceToHost, st));
  GMDS_CUDA(cudaStreamSynchronize(st));
  double g = 0.0;
  for (double v : hr) g += v;
  g /= static_cast<double>(n);
  center_kernel<<<grid_for(n * n), 256, 0, st>>>(dS, n, r.get(), g);
  count_launch();
  check_launch("center_kernel");
  GMDS_CUDA(cudaStreamSynchronize(st));
}

}  // namespace gmds
