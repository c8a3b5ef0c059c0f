// classical_mds at large n: the top-q eigenpairs of the
// double-centred Gram matrix B = -1/2 J (D o D) J by block subspace iteration
// with Rayleigh-Ritz, instead of a dense O(n^3) eigensolver
// (embed.cpp:415-460 calls SelfAdjointEigenSolver on all of B).
//
//   B          dense n x n fp64 in HBM, built once (unpack + double_center_dev,
//              the same kernels as the dense path; 3.2 GB at n = 20k)
//   W = B V    cuBLAS DGEMM, n x n by n x k (a plain library GEMM, HBM-bound)
//   H = V'W    k x k Rayleigh quotient; its eigenpairs (host cyclic Jacobi,
//              k <= 32) give Ritz values theta and vectors U = V Y, BU = W Y
//   stop       when || BU_c - theta_c U_c || <= tol |theta_0| for c < q
//   next V     orth(BU) by Cholesky QR, twice (CholQR2)
//
// Subspace iteration finds the k eigenvalues of largest MAGNITUDE; the
// reference wants the q largest algebraically.  They coincide when the q-th
// largest Ritz value exceeds the magnitude of every Ritz value outside the
// top q (an uncaptured eigenvalue is no larger in magnitude than the
// smallest captured one); otherwise the call reports NumericFailure and the
// caller uses the dense path.  The sign rule and clamp are the reference's
// (embed.cpp:440-458).  The full spectrum is never formed, so the clamped
// mass of the dense path is not available here.
#include <cublas_v2.h>

#include <algorithm>
#include <cmath>
#include <map>
#include <random>
#include <string>
#include <vector>

#include "classical_topq.h"
#include "common.cuh"
#include "dmat.cuh"
#include "dmat_kernels.cuh"
#include "kernels.cuh"

namespace gmds {

namespace {

cublasHandle_t blas_handle(cudaStream_t st) {
  static thread_local std::map<int, cublasHandle_t> handles;
  int dev = 0;
  GMDS_CUDA(cudaGetDevice(&dev));
  cublasHandle_t& h = handles[dev];
  if (!h && cublasCreate(&h) != CUBLAS_STATUS_SUCCESS) {
    h = nullptr;
    fail(GMDS_CUDA_ERROR, "cublasCreate failed");
  }
  cublasSetStream(h, st);
  return h;
}

void gemm(cublasHandle_t h, cublasOperation_t ta, cublasOperation_t tb, int m, int n, int k, const double* A, int lda,
          const double* B, int ldb, double* C, int ldc) {
  const double one = 1.0, zero = 0.0;
  if (cublasDgemm(h, ta, tb, m, n, k, &one, A, lda, B, ldb, &zero, C, ldc) != CUBLAS_STATUS_SUCCESS)
    fail(GMDS_CUDA_ERROR, "classical_mds: cublasDgemm failed");
  count_launch();
}

// Symmetric k x k eigen-decomposition, cyclic Jacobi (column-major A, in place).
// w ascending-unsorted; V columns are the eigenvectors.
void jacobi_eig(int k, std::vector<double>& A, std::vector<double>& w, std::vector<double>& V) {
  V.assign(static_cast<size_t>(k) * k, 0.0);
  for (int i = 0; i < k; ++i) V[i * k + i] = 1.0;
  auto a = [&](int i, int j) -> double& { return A[static_cast<size_t>(j) * k + i]; };
  for (int sweep = 0; sweep < 100; ++sweep) {
    double off = 0.0, diag = 0.0;
    for (int j = 0; j < k; ++j)
      for (int i = 0; i < k; ++i) (i == j ? diag : off) += a(i, j) * a(i, j);
    if (off <= 1e-32 * diag || off == 0.0) break;
    for (int p = 0; p < k - 1; ++p)
      for (int q = p + 1; q < k; ++q) {
        const double apq = a(p, q);
        if (apq == 0.0) continue;
        const double theta = (a(q, q) - a(p, p)) / (2.0 * apq);
        const double t = (theta >= 0 ? 1.0 : -1.0) / (std::abs(theta) + std::sqrt(theta * theta + 1.0));
        const double c = 1.0 / std::sqrt(t * t + 1.0), s = t * c;
        for (int r = 0; r < k; ++r) {  // A <- A J
          const double arp = a(r, p), arq = a(r, q);
          a(r, p) = c * arp - s * arq;
          a(r, q) = s * arp + c * arq;
        }
        for (int r = 0; r < k; ++r) {  // A <- J' A
          const double apr = a(p, r), aqr = a(q, r);
          a(p, r) = c * apr - s * aqr;
          a(q, r) = s * apr + c * aqr;
        }
        for (int r = 0; r < k; ++r) {
          double& vp = V[static_cast<size_t>(p) * k + r];
          double& vq = V[static_cast<size_t>(q) * k + r];
          const double x = vp, y = vq;
          vp = c * x - s * y;
          vq = s * x + c * y;
        }
      }
  }
  w.resize(k);
  for (int i = 0; i < k; ++i) w[i] = a(i, i);
}

// X (n x k, column-major, device) <- X R^{-1} with X'X = R'R (Cholesky QR).
// Returns false when the Gram matrix is not numerically positive definite.
bool chol_qr(cublasHandle_t h, double* X, double* T, double* dK, int64_t n, int k, cudaStream_t st) {
  gemm(h, CUBLAS_OP_T, CUBLAS_OP_N, k, k, static_cast<int>(n), X, static_cast<int>(n), X, static_cast<int>(n), dK, k);
  std::vector<double> C(static_cast<size_t>(k) * k);
  GMDS_CUDA(cudaMemcpyAsync(C.data(), dK, C.size() * 8, cudaMemcpyDeviceToHost, st));
  GMDS_CUDA(cudaStreamSynchronize(st));
  // C = L L' (lower), then Rinv = L'^{-1} (upper)
  std::vector<double> L(static_cast<size_t>(k) * k, 0.0);
  for (int j = 0; j < k; ++j) {
    double s = C[static_cast<size_t>(j) * k + j];
    for (int m = 0; m < j; ++m) s -= L[static_cast<size_t>(m) * k + j] * L[static_cast<size_t>(m) * k + j];
    if (!(s > 0.0)) return false;
    const double ljj = std::sqrt(s);
    L[static_cast<size_t>(j) * k + j] = ljj;
    for (int i = j + 1; i < k; ++i) {
      double t = C[static_cast<size_t>(j) * k + i];
      for (int m = 0; m < j; ++m) t -= L[static_cast<size_t>(m) * k + i] * L[static_cast<size_t>(m) * k + j];
      L[static_cast<size_t>(j) * k + i] = t / ljj;
    }
  }
  // Linv (lower) by forward substitution, then Rinv = Linv'
  std::vector<double> Li(static_cast<size_t>(k) * k, 0.0);
  for (int c = 0; c < k; ++c) {
    for (int i = c; i < k; ++i) {
      double t = (i == c) ? 1.0 : 0.0;
      for (int m = c; m < i; ++m) t -= L[static_cast<size_t>(m) * k + i] * Li[static_cast<size_t>(c) * k + m];
      Li[static_cast<size_t>(c) * k + i] = t / L[static_cast<size_t>(i) * k + i];
    }
  }
  std::vector<double> Ri(static_cast<size_t>(k) * k);
  for (int i = 0; i < k; ++i)
    for (int j = 0; j < k; ++j) Ri[static_cast<size_t>(j) * k + i] = Li[static_cast<size_t>(i) * k + j];
  GMDS_CUDA(cudaMemcpyAsync(dK, Ri.data(), Ri.size() * 8, cudaMemcpyHostToDevice, st));
  gemm(h, CUBLAS_OP_N, CUBLAS_OP_N, static_cast<int>(n), k, k, X, static_cast<int>(n), dK, k, T, static_cast<int>(n));
  GMDS_CUDA(cudaMemcpyAsync(X, T, sizeof(double) * n * k, cudaMemcpyDeviceToDevice, st));
  return true;
}

// out[c] = || BU[:, c] - theta[c] U[:, c] ||^2 for c < q (one block per column, fixed-order tree)
__global__ void resid_kernel(const double* __restrict__ U, const double* __restrict__ BU, const double* __restrict__ theta,
                             int64_t n, double* __restrict__ out) {
  const int c = blockIdx.x;
  const double th = theta[c];
  double s = 0.0;
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) {
    const double r = BU[c * n + i] - th * U[c * n + i];
    s += r * r;
  }
  __shared__ double red[256];
  red[threadIdx.x] = s;
  __syncthreads();
  for (int d = blockDim.x / 2; d > 0; d >>= 1) {
    if (static_cast<int>(threadIdx.x) < d) red[threadIdx.x] += red[threadIdx.x + d];
    __syncthreads();
  }
  if (threadIdx.x == 0) out[c] = red[0];
}

}  // namespace

void classical_topq_dev(const gmds_dmat* D, int q, double tol, int max_iters, double* coords, double* eigvals,
                        int* clamped_count, int* iterations, cudaStream_t st) {
  const int64_t n = D->n;
  if (q < 1 || q > n - 1)
    fail(GMDS_INVALID_INPUT, "classical_mds: target dimension must satisfy 1 <= p <= n-1, got p=" +
                                 std::to_string(q) + " with n=" + std::to_string(n));
  if (!(tol > 0.0)) fail(GMDS_INVALID_CONFIG, "classical_mds_topq: tol must be > 0");
  if (max_iters < 1) fail(GMDS_INVALID_CONFIG, "classical_mds_topq: max_iters must be >= 1");
  // W = B V is bound by reading B (n^2 doubles), so a wide block costs little
  // per iteration and converges as (lambda_{k+1} / lambda_q)^t
  const int k = static_cast<int>(std::min<int64_t>(n, std::max(32, 2 * q)));
  cublasHandle_t h = blas_handle(st);
  DevBuf<double> B(static_cast<size_t>(n * n));
  unpack_full(D->ptr(), D->storage, n, B.get(), true, st);  // S = D o D
  double_center_dev(B.get(), n, st);                        // B = -1/2 J S J
  const size_t nk = static_cast<size_t>(n) * k;
  DevBuf<double> V(nk), W(nk), U(nk), BU(nk), T(nk), dK(static_cast<size_t>(k) * k), dth(k), dres(k);
  // seeded Gaussian start (fixed seed: runs are reproducible)
  {
    std::mt19937_64 rng(0x9e3779b97f4a7c15ull);
    std::normal_distribution<double> nd(0.0, 1.0);
    std::vector<double> h0(nk);
    for (auto& x : h0) x = nd(rng);
    GMDS_CUDA(cudaMemcpyAsync(V.get(), h0.data(), nk * 8, cudaMemcpyHostToDevice, st));
    if (!chol_qr(h, V.get(), T.get(), dK.get(), n, k, st) || !chol_qr(h, V.get(), T.get(), dK.get(), n, k, st))
      fail(GMDS_NUMERIC_FAILURE, "classical_mds_topq: start basis is rank deficient");
  }
  const int N = static_cast<int>(n);
  std::vector<double> H(static_cast<size_t>(k) * k), w, Y, th(k), Ys(static_cast<size_t>(k) * k), res(q);
  int it = 0;
  bool conv = false;
  for (; it < max_iters; ++it) {
    gemm(h, CUBLAS_OP_N, CUBLAS_OP_N, N, k, N, B.get(), N, V.get(), N, W.get(), N);       // W = B V
    gemm(h, CUBLAS_OP_T, CUBLAS_OP_N, k, k, N, V.get(), N, W.get(), N, dK.get(), k);     // H = V' W
    GMDS_CUDA(cudaMemcpyAsync(H.data(), dK.get(), H.size() * 8, cudaMemcpyDeviceToHost, st));
    GMDS_CUDA(cudaStreamSynchronize(st));
    for (int i = 0; i < k; ++i)
      for (int j = i + 1; j < k; ++j) {
        const double s = 0.5 * (H[static_cast<size_t>(j) * k + i] + H[static_cast<size_t>(i) * k + j]);
        H[static_cast<size_t>(j) * k + i] = H[static_cast<size_t>(i) * k + j] = s;
      }
    jacobi_eig(k, H, w, Y);
    // Ritz pairs sorted by descending value
    std::vector<int> ord(k);
    for (int i = 0; i < k; ++i) ord[i] = i;
    std::stable_sort(ord.begin(), ord.end(), [&](int x, int y) { return w[x] > w[y]; });
    for (int c = 0; c < k; ++c) {
      th[c] = w[ord[c]];
      for (int r = 0; r < k; ++r) Ys[static_cast<size_t>(c) * k + r] = Y[static_cast<size_t>(ord[c]) * k + r];
    }
    GMDS_CUDA(cudaMemcpyAsync(dK.get(), Ys.data(), Ys.size() * 8, cudaMemcpyHostToDevice, st));
    GMDS_CUDA(cudaMemcpyAsync(dth.get(), th.data(), k * 8, cudaMemcpyHostToDevice, st));
    gemm(h, CUBLAS_OP_N, CUBLAS_OP_N, N, k, k, V.get(), N, dK.get(), k, U.get(), N);    // U = V Y
    gemm(h, CUBLAS_OP_N, CUBLAS_OP_N, N, k, k, W.get(), N, dK.get(), k, BU.get(), N);   // BU = W Y
    resid_kernel<<<q, 256, 0, st>>>(U.get(), BU.get(), dth.get(), n, dres.get());
    count_launch();
    check_launch("resid_kernel");
    GMDS_CUDA(cudaMemcpyAsync(res.data(), dres.get(), q * 8, cudaMemcpyDeviceToHost, st));
    GMDS_CUDA(cudaStreamSynchronize(st));
    double scale = 0.0;
    for (int c = 0; c < k; ++c) scale = std::max(scale, std::abs(th[c]));
    double worst = 0.0;
    for (int c = 0; c < q; ++c) worst = std::max(worst, std::sqrt(res[c]));
    if (worst <= tol * std::max(scale, 1e-300)) {
      conv = true;
      ++it;
      break;
    }
    // next basis: orth(B U) (the Ritz-rotated W)
    GMDS_CUDA(cudaMemcpyAsync(V.get(), BU.get(), nk * 8, cudaMemcpyDeviceToDevice, st));
    if (!chol_qr(h, V.get(), T.get(), dK.get(), n, k, st) || !chol_qr(h, V.get(), T.get(), dK.get(), n, k, st))
      fail(GMDS_NUMERIC_FAILURE, "classical_mds_topq: subspace collapsed (B has rank < k)");
  }
  if (!conv) fail(GMDS_NUMERIC_FAILURE, "classical_mds_topq: no convergence within max_iters");
  // the q largest must also be the q largest in magnitude among the captured ones
  double outside = 0.0;
  for (int c = q; c < k; ++c) outside = std::max(outside, std::abs(th[c]));
  if (k < n && !(th[q - 1] > outside))
    fail(GMDS_NUMERIC_FAILURE, "classical_mds_topq: top eigenvalues not separated from the rest of the spectrum");
  // coords: sign rule (largest |v| entry positive, first index wins) and sqrt(max(lambda, 0))
  std::vector<double> Uq(static_cast<size_t>(n) * q);
  GMDS_CUDA(cudaMemcpyAsync(Uq.data(), U.get(), Uq.size() * 8, cudaMemcpyDeviceToHost, st));
  GMDS_CUDA(cudaStreamSynchronize(st));
  *clamped_count = 0;
  for (int c = 0; c < q; ++c) {
    const double lambda = th[c];
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
  *iterations = it;
}

}  // namespace gmds
