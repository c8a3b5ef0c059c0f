// TEST INFRASTRUCTURE ONLY.  extern "C" shims over the UNMODIFIED reference
// library (proj/core/src/*.cpp compiled by path from /root/reference by
// oracle/Makefile against oracle/eigen_shim).  Loaded by tests/, by
// oracle/make_golden.py and by bench.py's cpu_baseline / --impl reference
// arm through ctypes; never by the product library.
//
// Status codes mirror the reference exception classes (error.hpp:9-53) and the
// product's gmds_status enum: 0 ok, 1 InvalidInput, 2 InvalidConfig,
// 3 DegenerateInput, 4 NumericFailure, 5 other Error.
#include <cmath>
#include <cstdint>
#include <cstring>
#include <span>
#include <string>
#include <vector>

#include "ginimds/embed.hpp"
#include "ginimds/error.hpp"
#include "ginimds/metrics.hpp"
#include "ginimds/parallel.hpp"
#include "ginimds/rng.hpp"
#include "ginimds/tune.hpp"

using namespace ginimds;

namespace {

thread_local std::string g_err;

template <typename F>
int guard(F&& f) {
  try {
    f();
    return 0;
  } catch (const InvalidInput& e) {
    g_err = e.what();
    return 1;
  } catch (const InvalidConfig& e) {
    g_err = e.what();
    return 2;
  } catch (const DegenerateInput& e) {
    g_err = e.what();
    return 3;
  } catch (const NumericFailure& e) {
    g_err = e.what();
    return 4;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 5;
  }
}

Matrix colmajor(const double* p, int64_t rows, int64_t cols) {
  Matrix m(rows, cols);
  std::memcpy(m.data(), p, sizeof(double) * static_cast<std::size_t>(rows * cols));
  return m;
}

void put(const Matrix& m, double* out) {
  std::memcpy(out, m.data(), sizeof(double) * static_cast<std::size_t>(m.size()));
}

StressKind kind_of(int k) {
  switch (k) {
    case 0: return StressKind::kruskal;
    case 1: return StressKind::huber;
    case 2: return StressKind::sammon;
    default: return StressKind::smacof;
  }
}

StressConfig make_cfg(int kind, double huber_delta, const double* weights, int64_t n, int max_iters,
                      double rel_tol) {
  StressConfig c;
  c.loss = kind_of(kind);
  if (!std::isnan(huber_delta)) c.huber_delta = huber_delta;
  if (weights) c.smacof_weights = colmajor(weights, n, n);
  c.max_iters = max_iters;
  c.rel_tol = rel_tol;
  return c;
}

void put_embedding(const Embedding& e, double* coords, double* history, int64_t hist_cap,
                   int64_t* hist_len, int* iterations, int* converged, double* stress,
                   double* huber_delta) {
  put(e.coords, coords);
  const int64_t m = static_cast<int64_t>(e.stress_history.size());
  if (hist_len) *hist_len = m;
  if (history)
    for (int64_t t = 0; t < std::min(m, hist_cap); ++t) history[t] = e.stress_history[static_cast<std::size_t>(t)];
  if (iterations) *iterations = e.iterations;
  if (converged) *converged = e.converged ? 1 : 0;
  if (stress) *stress = e.stress;
  if (huber_delta) *huber_delta = e.huber_delta;
}

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

void ref_set_max_threads(int n) { set_max_threads(n); }
int ref_max_threads() { return max_threads(); }

// ---- rank / distance (metrics.cpp) ----
int ref_midrank(const double* v, int64_t d, double* out) {
  return guard([&] {
    const RankVector r = midrank(std::span<const double>(v, static_cast<std::size_t>(d)));
    put(r.ranks, out);
  });
}

int ref_gini_norm(const double* x, int64_t d, double* out) {
  return guard([&] { *out = gini_norm(std::span<const double>(x, static_cast<std::size_t>(d))); });
}

int ref_gini_pseudo_distance(const double* x, int64_t dx, const double* y, int64_t dy, double* out) {
  return guard([&] {
    *out = gini_pseudo_distance(std::span<const double>(x, static_cast<std::size_t>(dx)),
                                std::span<const double>(y, static_cast<std::size_t>(dy)));
  });
}

int ref_empirical_survival(const double* z, int64_t d, double* out) {
  return guard([&] {
    const SurvivalVector s = empirical_survival(std::span<const double>(z, static_cast<std::size_t>(d)));
    put(s.values, out);
  });
}

int ref_gen_gini_directed(const double* x, int64_t dx, const double* y, int64_t dy, double nu, double* out) {
  return guard([&] {
    *out = gen_gini_directed(std::span<const double>(x, static_cast<std::size_t>(dx)),
                             std::span<const double>(y, static_cast<std::size_t>(dy)), GiniParams(nu));
  });
}

int ref_gen_gini_distance(const double* x, int64_t dx, const double* y, int64_t dy, double nu, double* out) {
  return guard([&] {
    *out = gen_gini_distance(std::span<const double>(x, static_cast<std::size_t>(dx)),
                             std::span<const double>(y, static_cast<std::size_t>(dy)), GiniParams(nu));
  });
}

// X column-major n x p.  nu <= 0 selects the Euclidean branch.
int ref_pairwise_matrix(const double* X, int64_t n, int64_t p, double nu, int euclidean, double* D_out) {
  return guard([&] {
    const Matrix Xm = colmajor(X, n, p);
    const DistanceMatrix D = pairwise_matrix(Xm, euclidean ? MetricSpec::euclidean() : MetricSpec::gini(nu));
    put(D.matrix(), D_out);
  });
}

// Rows [r0, r1) of the Gini matrix only: the bounded CPU-baseline sample.
// Same per-pair call as pairwise_matrix (metrics.cpp:213-219) with the same
// parallel_for over rows; entries j <= i are left untouched.
int ref_gini_rows(const double* X_rowmajor, int64_t n, int64_t p, double nu, int64_t r0, int64_t r1,
                  double* out_rows) {
  return guard([&] {
    const GiniParams params(nu);
    parallel_for(r1 - r0, [&](std::int64_t t) {
      const int64_t i = r0 + t;
      const std::span<const double> xi(X_rowmajor + i * p, static_cast<std::size_t>(p));
      for (int64_t j = i + 1; j < n; ++j) {
        const std::span<const double> xj(X_rowmajor + j * p, static_cast<std::size_t>(p));
        out_rows[t * n + j] = gen_gini_distance(xi, xj, params);
      }
    });
  });
}

int ref_distance_matrix_validate(const double* M, int64_t n, double* out) {
  return guard([&] { put(DistanceMatrix::from_matrix(colmajor(M, n, n)).matrix(), out); });
}

// ---- stress (embed.cpp) ----
int ref_double_center(const double* S, int64_t n, double* out) {
  return guard([&] { put(double_center(colmajor(S, n, n)), out); });
}

int ref_classical_mds(const double* D, int64_t n, int q, double* coords, double* eigvals, int* clamped_count,
                      double* clamped_mass, double* stress) {
  return guard([&] {
    const DistanceMatrix Dm = DistanceMatrix::from_matrix(colmajor(D, n, n));
    const Embedding e = classical_mds(Dm, q);
    put(e.coords, coords);
    put(e.eigenvalues, eigvals);
    *clamped_count = e.clamped_count;
    *clamped_mass = e.clamped_mass;
    *stress = e.stress;
  });
}

int ref_kruskal_stress(const double* coords, int64_t n, int q, const double* D, double* out) {
  return guard([&] {
    *out = kruskal_stress(colmajor(coords, n, q), DistanceMatrix::from_matrix(colmajor(D, n, n)));
  });
}

int ref_stress_loss(int kind, const double* coords, int64_t n, int q, const double* D, double huber_delta,
                    const double* weights, double* out) {
  return guard([&] {
    const StressConfig c = make_cfg(kind, huber_delta, weights, n, 300, 1e-6);
    *out = stress_loss(c.loss, colmajor(coords, n, q), DistanceMatrix::from_matrix(colmajor(D, n, n)), c);
  });
}

int ref_stress_gradient(int kind, const double* coords, int64_t n, int q, const double* D, double huber_delta,
                        const double* weights, double* grad_out) {
  return guard([&] {
    const StressConfig c = make_cfg(kind, huber_delta, weights, n, 300, 1e-6);
    put(stress_gradient(c.loss, colmajor(coords, n, q), DistanceMatrix::from_matrix(colmajor(D, n, n)), c),
        grad_out);
  });
}

int ref_minimize_stress(const double* D, int64_t n, int q, int kind, double huber_delta, const double* weights,
                        int max_iters, double rel_tol, double* coords, double* history, int64_t hist_cap,
                        int64_t* hist_len, int* iterations, int* converged, double* stress,
                        double* huber_delta_out) {
  return guard([&] {
    const StressConfig c = make_cfg(kind, huber_delta, weights, n, max_iters, rel_tol);
    const Embedding e = minimize_stress(DistanceMatrix::from_matrix(colmajor(D, n, n)), q, c);
    put_embedding(e, coords, history, hist_cap, hist_len, iterations, converged, stress, huber_delta_out);
  });
}

// ---- tune (tune.cpp) ----
int ref_nugrid_linspace(double lo, double hi, int count, double* out, int64_t cap, int64_t* len) {
  return guard([&] {
    const NuGrid g = NuGrid::linspace(lo, hi, count);
    *len = static_cast<int64_t>(g.size());
    for (std::size_t k = 0; k < g.size() && static_cast<int64_t>(k) < cap; ++k) out[k] = g.values()[k];
  });
}

int ref_nugrid_validate(const double* v, int64_t m) {
  return guard([&] { (void)NuGrid::from_values(std::vector<double>(v, v + m)); });
}

// method: 0 classical, 1 kruskal, 2 huber, 3 sammon, 4 smacof (EmbeddingMethod order)
int ref_tune_nu(const double* X, int64_t n, int64_t p, int q, const double* grid, int64_t m, int k_folds,
                int method, uint64_t seed, double* mean_stress, double* nu_star, double* coords,
                double* best_stress) {
  return guard([&] {
    const NuGrid g = NuGrid::from_values(std::vector<double>(grid, grid + m));
    const TuneReport r = tune_nu(colmajor(X, n, p), q, g, k_folds, static_cast<EmbeddingMethod>(method), seed);
    for (std::size_t k = 0; k < r.mean_stress.size(); ++k) mean_stress[k] = r.mean_stress[k];
    *nu_star = r.nu_star;
    put(r.best_embedding.coords, coords);
    *best_stress = r.best_embedding.stress;
  });
}

int ref_alternating_tune(const double* X, int64_t n, int64_t p, int q, int outer, const double* grid, int64_t m,
                         uint64_t seed, double* nu_path, double* nu_star, double* coords, double* stress) {
  return guard([&] {
    const NuGrid g = NuGrid::from_values(std::vector<double>(grid, grid + m));
    const AlternatingResult r = alternating_tune(colmajor(X, n, p), q, outer, g, seed);
    for (std::size_t k = 0; k < r.nu_path.size(); ++k) nu_path[k] = r.nu_path[k];
    *nu_star = r.nu_star;
    put(r.embedding.coords, coords);
    *stress = r.embedding.stress;
  });
}

// ---- rng (rng.cpp), used to regenerate the reference tests' own inputs ----
struct RefRng {
  Rng rng;
};
void* ref_rng_new(uint64_t seed) { return new RefRng{Rng(seed)}; }
void ref_rng_free(void* r) { delete static_cast<RefRng*>(r); }
double ref_rng_uniform01(void* r) { return static_cast<RefRng*>(r)->rng.uniform01(); }
uint64_t ref_rng_uniform_below(void* r, uint64_t b) { return static_cast<RefRng*>(r)->rng.uniform_below(b); }
double ref_rng_normal(void* r) { return static_cast<RefRng*>(r)->rng.normal(); }
double ref_rng_log_normal(void* r, double s) { return static_cast<RefRng*>(r)->rng.log_normal(s); }
uint64_t ref_mix_seed(uint64_t base, uint64_t a, uint64_t b) { return mix_seed(base, a, b); }
void ref_shuffle(void* r, int* idx, int64_t m) {
  std::vector<int> v(idx, idx + m);
  shuffle_indices(v, static_cast<RefRng*>(r)->rng);
  std::memcpy(idx, v.data(), sizeof(int) * static_cast<std::size_t>(m));
}

}  // extern "C"
