// Top-q classical MDS by subspace iteration (classical_topq.cu).
#pragma once

#include <cuda_runtime.h>

#include "dmat.cuh"

namespace gmds {

// n above which minimize_stress's classical init uses the subspace path
constexpr int64_t kDenseEigMaxN = 4096;

// coords n x q column-major (host), eigvals q; throws GMDS_NUMERIC_FAILURE when
// the iteration does not converge or the top q are not separated.
void classical_topq_dev(const gmds_dmat* D, int q, double tol, int max_iters, double* coords, double* eigvals,
                        int* clamped_count, int* iterations, cudaStream_t st);

}  // namespace gmds
