// bench.py's second e2e leg: the reference API exactly as a C++ caller uses it,
//   const Matrix& D = ginimds::pairwise_matrix(X, MetricSpec::gini(nu)).matrix();
// (tools/main.cpp:168, tune.cpp:132), through the ginimds:: facade (libginimds_b200.so):
// host column-major X in, host n x n fp64 D out, timed on the host clock around the call.
// Built by paper_2605_25124_b200/csrc/Makefile into lib/libfacade_e2e.so (ctypes).
#include <chrono>
#include <cstdint>
#include <cstring>
#include <exception>

#include "ginimds/ginimds.hpp"

extern "C" int facade_e2e(const double* X_colmajor, int64_t n, int64_t p, double nu, double* seconds,
                          double* checksum) {
  try {
    ginimds::Matrix X(n, p);
    std::memcpy(X.data(), X_colmajor, sizeof(double) * static_cast<size_t>(n * p));
    const auto t0 = std::chrono::steady_clock::now();
    const ginimds::DistanceMatrix D = ginimds::pairwise_matrix(X, ginimds::MetricSpec::gini(nu));
    const ginimds::Matrix& M = D.matrix();
    const auto t1 = std::chrono::steady_clock::now();
    *seconds = std::chrono::duration<double>(t1 - t0).count();
    double s = 0.0;
    for (int64_t k = 0; k < n; k += std::max<int64_t>(1, n / 97)) s += M(k, n - 1 - k) + M(n - 1 - k, k);
    *checksum = s;
    return 0;
  } catch (const std::exception&) {
    return 1;
  }
}
