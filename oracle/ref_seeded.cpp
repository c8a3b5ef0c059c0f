// TEST INFRASTRUCTURE ONLY.  Seeded-init entry into the UNMODIFIED reference
// iterate loops.
//
// The reference's minimize_stress always starts from classical_mds (embed.cpp:495,
// SURVEY F4); its iterate loops gradient_descent (embed.cpp:222-272) and
// smacof_iterate (embed.cpp:296-347) take the start coordinates by value but sit
// in an anonymous namespace.  This translation unit #includes embed.cpp itself
// (by path, from /root/reference, via -I in oracle/Makefile), so those loops and
// resolve_params (embed.cpp:54-109) are called exactly as minimize_stress calls
// them (embed.cpp:518-522), with Y0 in place of the classical init.  It is built
// into its own library (oracle/_ref/libginimds_ref_seeded.so) so embed.cpp's
// public symbols are not defined twice in one link.
//
// Also: ref_gini_pairs, the reference's gen_gini_distance (metrics.cpp:157-167)
// over an arbitrary list of pairs under its own parallel_for, for sampled
// golden entries at sizes where the full matrix is not stored.
#include "embed.cpp"  // NOLINT: the reference source, unmodified

#include <cstdint>
#include <cstring>
#include <span>
#include <string>

#include "ginimds/error.hpp"
#include "ginimds/parallel.hpp"

namespace {

thread_local std::string g_seeded_err;

template <typename F>
int seeded_guard(F&& f) {
  try {
    f();
    return 0;
  } catch (const ginimds::InvalidInput& e) {
    g_seeded_err = e.what();
    return 1;
  } catch (const ginimds::InvalidConfig& e) {
    g_seeded_err = e.what();
    return 2;
  } catch (const ginimds::DegenerateInput& e) {
    g_seeded_err = e.what();
    return 3;
  } catch (const ginimds::NumericFailure& e) {
    g_seeded_err = e.what();
    return 4;
  } catch (const std::exception& e) {
    g_seeded_err = e.what();
    return 5;
  }
}

ginimds::StressKind seeded_kind(int k) {
  switch (k) {
    case 0: return ginimds::StressKind::kruskal;
    case 1: return ginimds::StressKind::huber;
    case 2: return ginimds::StressKind::sammon;
    default: return ginimds::StressKind::smacof;
  }
}

}  // namespace

extern "C" {

const char* ref_seeded_last_error() { return g_seeded_err.c_str(); }

// D column-major n x n fp64 (validated by DistanceMatrix::from_matrix), Y0
// column-major n x q.  kind: 0 kruskal, 1 huber (explicit delta), 2 sammon,
// 3 smacof (uniform weights).
int ref_seeded_fit(const double* D, int64_t n, int q, int kind, double huber_delta, int max_iters, double rel_tol,
                   const double* Y0, double* coords, double* history, int64_t hist_cap, int64_t* hist_len,
                   int* iterations, int* converged, double* loss) {
  return seeded_guard([&] {
    using namespace ginimds;
    Matrix Dm(n, n);
    std::memcpy(Dm.data(), D, sizeof(double) * static_cast<std::size_t>(n * n));
    const DistanceMatrix Dd = DistanceMatrix::from_matrix(Dm);
    Dm = Matrix();
    Matrix init(n, q);
    std::memcpy(init.data(), Y0, sizeof(double) * static_cast<std::size_t>(n * q));
    StressConfig cfg;
    cfg.loss = seeded_kind(kind);
    if (cfg.loss == StressKind::huber) cfg.huber_delta = huber_delta;
    cfg.max_iters = max_iters;
    cfg.rel_tol = rel_tol;
    const LossParams params = resolve_params(cfg.loss, Dd, cfg, "minimize_stress");
    IterativeResult r = (cfg.loss == StressKind::smacof)
                            ? smacof_iterate(init, Dd, params, cfg.max_iters, cfg.rel_tol)
                            : gradient_descent(cfg.loss, init, Dd, params, cfg.max_iters, cfg.rel_tol);
    std::memcpy(coords, r.coords.data(), sizeof(double) * static_cast<std::size_t>(n * q));
    const int64_t m = static_cast<int64_t>(r.history.size());
    *hist_len = m;
    for (int64_t t = 0; t < std::min(m, hist_cap); ++t) history[t] = r.history[static_cast<std::size_t>(t)];
    *iterations = r.iterations;
    *converged = r.converged ? 1 : 0;
    *loss = r.loss;
  });
}

// out[k] = gen_gini_distance(X[I[k]], X[J[k]], nu), X row-major n x p.
int ref_gini_pairs(const double* X, int64_t n, int64_t p, double nu, const int64_t* I, const int64_t* J, int64_t m,
                   double* out) {
  return seeded_guard([&] {
    using namespace ginimds;
    const GiniParams params(nu);
    const int64_t chunk = 4096;
    parallel_for((m + chunk - 1) / chunk, [&](std::int64_t c) {
      for (int64_t k = c * chunk; k < std::min(m, (c + 1) * chunk); ++k) {
        if (I[k] < 0 || I[k] >= n || J[k] < 0 || J[k] >= n) throw InvalidInput("ref_gini_pairs: index out of range");
        const std::span<const double> xi(X + I[k] * p, static_cast<std::size_t>(p));
        const std::span<const double> xj(X + J[k] * p, static_cast<std::size_t>(p));
        out[k] = gen_gini_distance(xi, xj, params);
      }
    });
  });
}

}  // extern "C"
