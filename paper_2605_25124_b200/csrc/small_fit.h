// Persistent (cooperative, all-SM) stress fit for small n (small_fit.cu).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

#include "gmds.h"

namespace gmds {

constexpr int64_t kSmallFitMaxN = 2048;

struct SmallFitArgs {
  const double* D;   // dense n x n row-major fp64 copy of the distance matrix
  double* buf[4];    // two coordinate slots (buf[0] = Y0 on entry) + two gradient slots, n x q row-major
  double* lossp;     // [2][grid][4] per-CTA partials (losses of two configurations, |g|^2; double-buffered)
  double* Yout;      // n x q row-major
  double* history;   // max_iters + 1 entries
  double* out;       // [0] final loss
  int* iout;         // [0] iterations, [1] converged, [2] history length, [3] passes over D
  int n;
  int kind;
  double delta;
  double sum, sum_sq;  // D statistics (loss normalisers)
  int max_iters;
  double rel_tol;
};

bool small_fit_supported(int64_t n, int q);
int small_fit_grid(int64_t n);  // CTAs for a cooperative launch, 0 if the device is too small
void launch_small_fit(const SmallFitArgs& a, int q, int grid, cudaStream_t st);

}  // namespace gmds
