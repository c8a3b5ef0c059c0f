// classical_mds at large n: the top-q eigenpairs of the
// double-centred Gram matrix B = -1/2 J (D o D) J (embed.cpp:382-413) without
// forming B and without a dense O(n^3) eigensolver (embed.cpp:415-460 calls
// SelfAdjointEigenSolver on all of B).
//
//   B v        = -1/2 J S J v,  S = D o D, J = I - 11'/n:  v' = v - mean(v),
//                z = S v' streamed from the packed triangle of D (one read of
//                n(n-1)/2 entries, squared in fp64 on the fly -- exact for fp32
//                storage -- each entry used for its row and its column), then
//                B v = -1/2 (z - mean(z)).  HBM-bound; fixed-order reductions.
//   Lanczos    with full reorthogonalisation (classical Gram-Schmidt, twice) on
//              the device; the tridiagonal T_m on the host (implicit QL with
//              Wilkinson shifts); converged when every top-q Ritz residual
//              |beta_m s_{m,c}| <= tol max|theta|.  Lanczos resolves the
//              algebraically largest eigenvalues directly (both ends of the
//              spectrum converge), so no magnitude/sign separation test is
//              needed.  Breakdown (an invariant Krylov space) restarts from a
//              fresh seeded vector orthogonal to the basis.
//   Ritz       u_c = V s_c; the reference's sign rule and clamp
//              (embed.cpp:440-458).  The full spectrum is never formed, so
//              clamped_mass is not available here.
//
// No cuBLAS / cuSOLVER: every device operation below is a kernel of this file
// or the shared two-level row reduction (stress_kernels.cu).
#include <algorithm>
#include <cmath>
#include <random>
#include <string>
#include <vector>

#include "classical_topq.h"
#include "common.cuh"
#include "dmat.cuh"
#include "fit.h"
#include "kernels.cuh"
#include "stress.cuh"

namespace gmds {

namespace {

constexpr int kSvRows = 16;  // rows of a block per warp (8 warps x 16 = kPT)

// z-partials of S v' over one chunk (block row I, blocks J0..J1): warp w owns rows
// I*kPT + 16w .. +15, lane l columns 4l..4l+3 of every block (one float4 / double
// pair per row: coalesced).  Row sums stay in registers over the chunk and leave once
// (xor-tree over the lanes); column sums leave per block (warps added in order).
template <typename TD>
__global__ void __launch_bounds__(256, 2) sv_chunk_kernel(const TD* __restrict__ D, const int64_t* __restrict__ chunk_I,
                                                       const int64_t* __restrict__ chunk_J0, int64_t chunk_len,
                                                       int64_t nb, const double* __restrict__ v,
                                                       double* __restrict__ rowpart, double* __restrict__ colpart) {
  __shared__ double scol[8][kPT];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t chunk = blockIdx.x;
  const int64_t I = chunk_I[chunk], J0 = chunk_J0[chunk];
  const int64_t J1 = min(J0 + chunk_len, nb);
  double vi[kSvRows], racc[kSvRows];
#pragma unroll
  for (int x = 0; x < kSvRows; ++x) {
    vi[x] = v[I * kPT + warp * kSvRows + x];
    racc[x] = 0.0;
  }
  for (int64_t J = J0; J < J1; ++J) {
    const TD* blk = D + (I * nb - (I * (I - 1)) / 2 + (J - I)) * (kPT * kPT);
    double vj[4], cacc[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
    for (int c = 0; c < 4; ++c) vj[c] = v[J * kPT + 4 * lane + c];
    TD dv[kSvRows][4];  // the storage type (fp32: half the registers)
#pragma unroll
    for (int x = 0; x < kSvRows; ++x) {  // all 16 rows' loads in flight first
      const TD* row = blk + (warp * kSvRows + x) * kPT + 4 * lane;
      if constexpr (sizeof(TD) == 4) {
        const float4 f = *reinterpret_cast<const float4*>(row);
        dv[x][0] = f.x, dv[x][1] = f.y, dv[x][2] = f.z, dv[x][3] = f.w;
      } else {
        const double2 a = reinterpret_cast<const double2*>(row)[0], b = reinterpret_cast<const double2*>(row)[1];
        dv[x][0] = a.x, dv[x][1] = a.y, dv[x][2] = b.x, dv[x][3] = b.y;
      }
    }
#pragma unroll
    for (int x = 0; x < kSvRows; ++x)
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        const double d = static_cast<double>(dv[x][c]);
        const double s = d * d;  // (D o D) entry: exact from fp32
        racc[x] = fma(s, vj[c], racc[x]);
        cacc[c] = fma(s, vi[x], cacc[c]);
      }
#pragma unroll
    for (int c = 0; c < 4; ++c) scol[warp][4 * lane + c] = cacc[c];
    __syncthreads();
    if (threadIdx.x < kPT) {
      double t = 0.0;
#pragma unroll
      for (int w = 0; w < 8; ++w) t += scol[w][threadIdx.x];
      colpart[(I * nb - (I * (I - 1)) / 2 + (J - I)) * kPT + threadIdx.x] = t;
    }
    __syncthreads();
  }
#pragma unroll
  for (int x = 0; x < kSvRows; ++x) {
    double t = racc[x];
#pragma unroll
    for (int m = 16; m > 0; m >>= 1) t += __shfl_xor_sync(0xffffffffu, t, m);
    if (lane == 0) rowpart[chunk * kPT + warp * kSvRows + x] = t;
  }
}

// out = (in - mean(in)) * scale over the first n entries (the rest stay 0); one CTA,
// fixed-order sum
__global__ void center_scale_kernel(const double* __restrict__ in, int64_t n, double scale, double* __restrict__ out) {
  __shared__ double red[1024];
  double s = 0.0;
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) s += in[i];
  red[threadIdx.x] = s;
  __syncthreads();
  for (int w = blockDim.x / 2; w > 0; w >>= 1) {
    if (static_cast<int>(threadIdx.x) < w) red[threadIdx.x] += red[threadIdx.x + w];
    __syncthreads();
  }
  const double mean = red[0] / static_cast<double>(n);
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) out[i] = (in[i] - mean) * scale;
}

// c[t] = V_t . w for t < m (one CTA per t, fixed-order tree): V row-major [m][n]
__global__ void dots_kernel(const double* __restrict__ V, int64_t n, const double* __restrict__ w,
                            double* __restrict__ c) {
  __shared__ double red[256];
  const double* vt = V + static_cast<int64_t>(blockIdx.x) * n;
  double s = 0.0;
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) s = fma(vt[i], w[i], s);
  red[threadIdx.x] = s;
  __syncthreads();
  for (int k = blockDim.x / 2; k > 0; k >>= 1) {
    if (static_cast<int>(threadIdx.x) < k) red[threadIdx.x] += red[threadIdx.x + k];
    __syncthreads();
  }
  if (threadIdx.x == 0) c[blockIdx.x] = red[0];
}

// w -= sum_t V_t c[t] (t < m)
__global__ void sub_combo_kernel(const double* __restrict__ V, int64_t n, int m, const double* __restrict__ c,
                                 double* __restrict__ w) {
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    double s = 0.0;
    for (int t = 0; t < m; ++t) s = fma(V[static_cast<int64_t>(t) * n + i], c[t], s);
    w[i] -= s;
  }
}

// out_c = sum_t V_t S[c][t] for c < q (Ritz vectors; S row c = the c-th Ritz coefficients)
__global__ void combo_kernel(const double* __restrict__ V, int64_t n, int m, const double* __restrict__ S, int q,
                             double* __restrict__ out) {
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    for (int c = 0; c < q; ++c) {
      double s = 0.0;
      for (int t = 0; t < m; ++t) s = fma(V[static_cast<int64_t>(t) * n + i], S[c * m + t], s);
      out[static_cast<int64_t>(c) * n + i] = s;
    }
}

__global__ void scale_copy_kernel(const double* __restrict__ in, int64_t n, double s, double* __restrict__ out) {
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    out[i] = in[i] * s;
}

unsigned grid_n(int64_t n) { return static_cast<unsigned>(std::max<int64_t>(1, std::min<int64_t>(ceil_div(n, 256), 148 * 8))); }

// Symmetric tridiagonal eigenproblem by implicit QL with Wilkinson shifts; d (diagonal,
// m) and e (sub-diagonal, e[i] couples i and i+1) in; d = eigenvalues, Z (row-major
// m x m, Z[k][j] = component k of eigenvector j) out.  false: no convergence.
bool tridiag_ql(std::vector<double>& d, std::vector<double> e, std::vector<double>& Z) {
  const int m = static_cast<int>(d.size());
  Z.assign(static_cast<size_t>(m) * m, 0.0);
  for (int i = 0; i < m; ++i) Z[static_cast<size_t>(i) * m + i] = 1.0;
  e.resize(static_cast<size_t>(m), 0.0);
  for (int l = 0; l < m; ++l) {
    for (int iter = 0;; ++iter) {
      int mm = l;
      for (; mm < m - 1; ++mm) {
        const double dd = std::abs(d[mm]) + std::abs(d[mm + 1]);
        if (std::abs(e[mm]) <= 2.2e-16 * dd) break;
      }
      if (mm == l) break;
      if (iter == 60) return false;
      double g = (d[l + 1] - d[l]) / (2.0 * e[l]);
      double r = std::hypot(g, 1.0);
      g = d[mm] - d[l] + e[l] / (g + std::copysign(r, g));  // Wilkinson shift folded in
      double s = 1.0, c = 1.0, p = 0.0;
      int i = mm - 1;
      for (; i >= l; --i) {
        const double f = s * e[i], b = c * e[i];
        r = std::hypot(f, g);
        e[i + 1] = r;
        if (r == 0.0) {  // split: deflate and restart this l
          d[i + 1] -= p;
          e[mm] = 0.0;
          break;
        }
        s = f / r;
        c = g / r;
        g = d[i + 1] - p;
        r = (d[i] - g) * s + 2.0 * c * b;
        p = s * r;
        d[i + 1] = g + p;
        g = c * r - b;
        for (int k = 0; k < m; ++k) {  // rotate eigenvector columns i, i+1
          double& zi = Z[static_cast<size_t>(k) * m + i];
          double& zj = Z[static_cast<size_t>(k) * m + i + 1];
          const double t = zj;
          zj = s * zi + c * t;
          zi = c * zi - s * t;
        }
      }
      if (r == 0.0 && i >= l) continue;
      d[l] -= p;
      e[l] = g;
      e[mm] = 0.0;
    }
  }
  return true;
}

struct PackedSv {  // z = S v' over the packed triangle, reduced to n entries
  const gmds_dmat* D;
  int64_t n, nb, len, nchunks;
  DevBuf<int64_t> cI, cJ, sf;
  DevBuf<double> rowpart, colpart, gpart;
  cudaStream_t st;

  PackedSv(const gmds_dmat* D_, cudaStream_t st_) : D(D_), n(D_->n), st(st_) {
    nb = ceil_div(n, kPT);
    len = chunk_blocks(nb);
    std::vector<int64_t> hI, hJ, hs;
    chunk_list(nb, len, hI, hJ);
    for (int64_t I = 0, c = 0; I <= nb; ++I) {
      while (c < static_cast<int64_t>(hI.size()) && hI[c] < I) ++c;
      hs.push_back(c);
    }
    nchunks = static_cast<int64_t>(hI.size());
    cI.alloc(hI.size());
    cJ.alloc(hJ.size());
    sf.alloc(hs.size());
    GMDS_CUDA(cudaMemcpyAsync(cI.get(), hI.data(), hI.size() * 8, cudaMemcpyHostToDevice, st));
    GMDS_CUDA(cudaMemcpyAsync(cJ.get(), hJ.data(), hJ.size() * 8, cudaMemcpyHostToDevice, st));
    GMDS_CUDA(cudaMemcpyAsync(sf.get(), hs.data(), hs.size() * 8, cudaMemcpyHostToDevice, st));
    rowpart.alloc(static_cast<size_t>(nchunks) * kPT);
    colpart.alloc(static_cast<size_t>(nb * (nb + 1) / 2) * kPT);
    gpart.alloc(reduce_rows_scratch(nb, 1));
  }
  // vpad: nb * kPT entries, zero beyond n
  void apply(const double* vpad, double* z) {
    const unsigned g = static_cast<unsigned>(nchunks);
    if (D->storage == GMDS_F32)
      sv_chunk_kernel<float><<<g, 256, 0, st>>>(static_cast<const float*>(D->ptr()), cI.get(), cJ.get(), len, nb, vpad,
                                                rowpart.get(), colpart.get());
    else
      sv_chunk_kernel<double><<<g, 256, 0, st>>>(static_cast<const double*>(D->ptr()), cI.get(), cJ.get(), len, nb,
                                                 vpad, rowpart.get(), colpart.get());
    count_launch();
    check_launch("sv_chunk_kernel");
    launch_reduce_rows(rowpart.get(), colpart.get(), sf.get(), n, nb, 1, z, st, gpart.get());
  }
};

}  // namespace

void classical_topq_dev(const gmds_dmat* D, int q, double tol, int max_iters, double* coords, double* eigvals,
                        int* clamped_count, int* iterations, cudaStream_t st) {
  const int64_t n = D->n;
  if (q < 1 || q > n - 1)
    fail(GMDS_INVALID_INPUT, "classical_mds: target dimension must satisfy 1 <= p <= n-1, got p=" +
                                 std::to_string(q) + " with n=" + std::to_string(n));
  if (!(tol > 0.0)) fail(GMDS_INVALID_CONFIG, "classical_mds_topq: tol must be > 0");
  if (max_iters < 1) fail(GMDS_INVALID_CONFIG, "classical_mds_topq: max_iters must be >= 1");
  PackedSv S(D, st);
  const int m_max = static_cast<int>(std::min<int64_t>({n, static_cast<int64_t>(max_iters) + 1, int64_t(2000)}));
  DevBuf<double> V(static_cast<size_t>(m_max + 1) * n);  // Lanczos basis, row t = v_t
  DevBuf<double> vpad(static_cast<size_t>(S.nb) * kPT), z(static_cast<size_t>(n)), w(static_cast<size_t>(n));
  DevBuf<double> coef(static_cast<size_t>(m_max + 1)), dS(static_cast<size_t>(q) * m_max), U(static_cast<size_t>(q) * n);
  GMDS_CUDA(cudaMemsetAsync(vpad.get(), 0, vpad.n * sizeof(double), st));
  std::mt19937_64 rng(0x9e3779b97f4a7c15ull);  // seeded: reproducible runs
  std::normal_distribution<double> nd(0.0, 1.0);
  const unsigned gn = grid_n(n);
  auto orthogonalize = [&](int m) {  // w -= V_{<m} (V_{<m}' w), twice (CGS2)
    for (int pass = 0; pass < 2 && m > 0; ++pass) {
      dots_kernel<<<m, 256, 0, st>>>(V.get(), n, w.get(), coef.get());
      sub_combo_kernel<<<gn, 256, 0, st>>>(V.get(), n, m, coef.get(), w.get());
      count_launch(2);
    }
    check_launch("lanczos orthogonalisation");
  };
  auto norm_of_w = [&]() {
    dots_kernel<<<1, 256, 0, st>>>(w.get(), n, w.get(), coef.get());
    count_launch();
    double h = 0.0;
    GMDS_CUDA(cudaMemcpyAsync(&h, coef.get(), sizeof h, cudaMemcpyDeviceToHost, st));
    GMDS_CUDA(cudaStreamSynchronize(st));
    return std::sqrt(h);
  };
  // a fresh seeded start vector orthogonal to the first m basis vectors, normalised into V_m
  auto fresh = [&](int m) {
    std::vector<double> h(static_cast<size_t>(n));
    for (auto& x : h) x = nd(rng);
    GMDS_CUDA(cudaMemcpyAsync(w.get(), h.data(), n * sizeof(double), cudaMemcpyHostToDevice, st));
    orthogonalize(m);
    const double nv = norm_of_w();
    if (!(nv > 0.0)) return false;
    scale_copy_kernel<<<gn, 256, 0, st>>>(w.get(), n, 1.0 / nv, V.get() + static_cast<int64_t>(m) * n);
    count_launch();
    return true;
  };
  if (!fresh(0)) fail(GMDS_NUMERIC_FAILURE, "classical_mds_topq: start vector vanished");
  std::vector<double> alpha, beta;  // T: diagonal alpha, off-diagonal beta (beta[j] couples j, j+1)
  std::vector<double> th, Z;
  double bnorm = 0.0;  // ||T|| estimate (max |Ritz value|)
  bool conv = false;
  int m = 0;
  std::vector<int> top;
  for (int j = 0; j < m_max; ++j) {
    const double* vj = V.get() + static_cast<int64_t>(j) * n;
    // w = B v_j = -1/2 J S J v_j
    center_scale_kernel<<<1, 1024, 0, st>>>(vj, n, 1.0, vpad.get());
    count_launch();
    S.apply(vpad.get(), z.get());
    center_scale_kernel<<<1, 1024, 0, st>>>(z.get(), n, -0.5, w.get());
    count_launch();
    // alpha_j = v_j . w, then full reorthogonalisation against v_0..v_j (removes the
    // alpha / beta terms of the three-term recurrence with them)
    dots_kernel<<<1, 256, 0, st>>>(vj, n, w.get(), coef.get());
    count_launch();
    double a = 0.0;
    GMDS_CUDA(cudaMemcpyAsync(&a, coef.get(), sizeof a, cudaMemcpyDeviceToHost, st));
    GMDS_CUDA(cudaStreamSynchronize(st));
    alpha.push_back(a);
    orthogonalize(j + 1);
    const double b = norm_of_w();
    m = j + 1;
    bnorm = std::max({bnorm, std::abs(a), b});
    // Ritz values of T_m: check the top q every few steps (and at the end).  At m = n the
    // basis spans everything and the Ritz pairs are exact; a breakdown before that only
    // means the Krylov space is invariant, so it restarts from a fresh orthogonal vector
    // (T splits) instead of stopping -- a missed repeated eigenvalue is picked up then.
    const bool full = (m == n);
    const bool last = full || (m == m_max);
    const bool breakdown = !(b > 1e-13 * bnorm);
    if (m >= q && (full || (!breakdown && (m % 4 == 0 || last)))) {
      th = alpha;
      std::vector<double> off(beta.begin(), beta.end());
      if (!tridiag_ql(th, off, Z)) fail(GMDS_NUMERIC_FAILURE, "classical_mds_topq: tridiagonal QL did not converge");
      top.resize(static_cast<size_t>(m));
      for (int i = 0; i < m; ++i) top[i] = i;
      std::stable_sort(top.begin(), top.end(), [&](int x, int y) { return th[x] > th[y]; });
      double scale = 0.0;
      for (double t : th) scale = std::max(scale, std::abs(t));
      double worst = 0.0;
      for (int c = 0; c < q; ++c)  // residual of Ritz pair c: beta_m |s_{m-1, c}|
        worst = std::max(worst, (full ? 0.0 : b) * std::abs(Z[static_cast<size_t>(m - 1) * m + top[c]]));
      if (worst <= tol * std::max(scale, 1e-300)) {
        conv = true;
        break;
      }
    }
    if (last) break;
    if (breakdown) {
      beta.push_back(0.0);
      if (!fresh(m)) break;
      continue;
    }
    beta.push_back(b);
    scale_copy_kernel<<<gn, 256, 0, st>>>(w.get(), n, 1.0 / b, V.get() + static_cast<int64_t>(m) * n);
    count_launch();
  }
  if (!conv) fail(GMDS_NUMERIC_FAILURE, "classical_mds_topq: no convergence within max_iters");
  // Ritz vectors of the top q (descending) and the reference's sign rule / clamp
  std::vector<double> hs(static_cast<size_t>(q) * m);
  for (int c = 0; c < q; ++c)
    for (int t = 0; t < m; ++t) hs[static_cast<size_t>(c) * m + t] = Z[static_cast<size_t>(t) * m + top[c]];
  GMDS_CUDA(cudaMemcpyAsync(dS.get(), hs.data(), hs.size() * 8, cudaMemcpyHostToDevice, st));
  combo_kernel<<<gn, 256, 0, st>>>(V.get(), n, m, dS.get(), q, U.get());
  count_launch();
  check_launch("combo_kernel");
  std::vector<double> Uq(static_cast<size_t>(n) * q);
  GMDS_CUDA(cudaMemcpyAsync(Uq.data(), U.get(), Uq.size() * 8, cudaMemcpyDeviceToHost, st));
  GMDS_CUDA(cudaStreamSynchronize(st));
  *clamped_count = 0;
  for (int c = 0; c < q; ++c) {
    const double lambda = th[top[c]];
    eigvals[c] = lambda;
    const double* v = Uq.data() + static_cast<size_t>(c) * n;
    int64_t arg = 0;
    double best = std::abs(v[0]);
    for (int64_t i = 1; i < n; ++i)
      if (std::abs(v[i]) > best) {
        best = std::abs(v[i]);
        arg = i;
      }
    const double sgn = (v[arg] < 0.0) ? -1.0 : 1.0;
    if (lambda < 0.0) ++*clamped_count;
    const double sc = std::sqrt(std::max(lambda, 0.0));
    for (int64_t i = 0; i < n; ++i) coords[static_cast<size_t>(c) * n + i] = (sgn * v[i]) * sc;
  }
  *iterations = m;
}

}  // namespace gmds
