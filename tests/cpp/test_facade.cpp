// The reference's own unit-test cases (proj/tests/unit/test_metrics.cpp,
// test_embed.cpp, test_tune.cpp), re-expressed against the B200 engine's
// ginimds:: drop-in facade -- the same calls a reference caller makes.
// Built and run by tests/test_cpp_facade.py.  Minimal CHECK harness (the
// reference uses doctest, absent here).
#include <cmath>
#include <cstdio>
#include <functional>
#include <limits>
#include <string>
#include <vector>

#include "ginimds/ginimds.hpp"

using namespace ginimds;

static int g_fail = 0, g_checks = 0;
#define CHECK(c)                                                         \
  do {                                                                   \
    ++g_checks;                                                          \
    if (!(c)) {                                                          \
      ++g_fail;                                                          \
      std::printf("CHECK failed %s:%d: %s\n", __FILE__, __LINE__, #c);  \
    }                                                                    \
  } while (0)
#define CHECK_THROWS_AS(expr, T)      \
  do {                                \
    bool ok = false;                  \
    try {                             \
      (void)(expr);                   \
    } catch (const T&) {              \
      ok = true;                      \
    } catch (...) {                   \
    }                                 \
    CHECK(ok);                        \
  } while (0)
static bool approx(double a, double b, double rel) { return std::abs(a - b) <= rel * std::max(1.0, std::abs(b)); }

static Vector vec(std::initializer_list<double> v) {
  Vector out(static_cast<Eigen::Index>(v.size()));
  Eigen::Index i = 0;
  for (double x : v) out(i++) = x;
  return out;
}

static void metrics_tests() {
  // test_metrics.cpp:94-119
  Vector r = midrank(vec({3.0, 1.0, 2.0})).ranks;
  CHECK(r(0) == 3.0 && r(1) == 1.0 && r(2) == 2.0);
  r = midrank(vec({0.0, 0.0, 0.0, 0.0})).ranks;
  for (int i = 0; i < 4; ++i) CHECK(r(i) == 2.5);
  r = midrank(vec({1.0, 2.0, 2.0, 4.0})).ranks;
  CHECK(r(0) == 1.0 && r(1) == 2.5 && r(2) == 2.5 && r(3) == 4.0);
  CHECK_THROWS_AS(midrank(vec({1.0, std::numeric_limits<double>::quiet_NaN()})), InvalidInput);
  CHECK_THROWS_AS(midrank(Vector{}), InvalidInput);
  // gini_norm (151-160), worked example (180-182), survival (216-226)
  CHECK(gini_norm(vec({5.0, 5.0, 5.0})) == 0.0);
  CHECK(approx(gini_norm(vec({1.0, 2.0, 3.0})), 2.0, 1e-14));
  CHECK(approx(gini_norm(vec({-2.0, -4.0, -6.0})), 4.0, 1e-14));
  CHECK(gini_pseudo_distance(vec({10.0, 1200.0}), vec({10.0, 12.0})) == 594.0);
  CHECK_THROWS_AS(gini_pseudo_distance(vec({1.0, 2.0}), vec({1.0})), InvalidInput);
  SurvivalVector s = empirical_survival(vec({0.0, 1188.0}));
  CHECK(s.values(0) == 0.75 && s.values(1) == 0.25 && s.at_zero == 0.5);
  // directed 445.5 / 742.5 (245-252), GiniParams (254-258), symmetrised (273-279)
  const Vector x = vec({10.0, 1200.0}), y = vec({10.0, 12.0});
  CHECK(approx(gen_gini_directed(x, y, GiniParams(2.0)), 594.0, 1e-12));
  CHECK(approx(gen_gini_directed(x, y, GiniParams(3.0)), 445.5, 1e-12));
  CHECK(approx(gen_gini_directed(y, x, GiniParams(3.0)), 742.5, 1e-12));
  CHECK_THROWS_AS(GiniParams(1.0), InvalidConfig);
  CHECK_THROWS_AS(GiniParams(0.5), InvalidConfig);
  CHECK(approx(gen_gini_distance(x, y, GiniParams(3.0)), 594.0, 1e-12));
  CHECK(gen_gini_distance(x, x, GiniParams(3.5)) == 0.0);
  // pairwise_matrix (302-354)
  Matrix X(2, 3);
  X << 1.0, 2.0, 3.0, 1.0, 2.0, 3.0;
  CHECK(pairwise_matrix(X, MetricSpec::gini(2.5))(0, 1) == 0.0);
  Matrix X2(2, 2);
  X2 << 10.0, 1200.0, 10.0, 12.0;
  const DistanceMatrix D = pairwise_matrix(X2, MetricSpec::gini(2.0));
  CHECK(approx(D(0, 1), 594.0, 1e-12) && D(1, 0) == D(0, 1) && D(0, 0) == 0.0);
  Matrix X1(1, 3);
  X1 << 1.0, 2.0, 3.0;
  CHECK_THROWS_AS(pairwise_matrix(X1, MetricSpec::euclidean()), InvalidInput);
  // DistanceMatrix validation (356-372)
  Matrix ok(2, 2), asym(2, 2), diag(2, 2), neg(2, 2);
  ok << 0.0, 1.0, 1.0, 0.0;
  asym << 0.0, 1.0, 2.0, 0.0;
  diag << 1.0, 1.0, 1.0, 0.0;
  neg << 0.0, -1.0, -1.0, 0.0;
  (void)DistanceMatrix::from_matrix(ok);
  CHECK_THROWS_AS(DistanceMatrix::from_matrix(asym), InvalidInput);
  CHECK_THROWS_AS(DistanceMatrix::from_matrix(diag), InvalidInput);
  CHECK_THROWS_AS(DistanceMatrix::from_matrix(neg), InvalidInput);
}

static DistanceMatrix unit_square() {
  Matrix pts(4, 2);
  pts << 0, 0, 1, 0, 1, 1, 0, 1;
  return pairwise_matrix(pts, MetricSpec::euclidean());
}

static void embed_tests() {
  // double_center (test_embed.cpp:41-79)
  Matrix S(2, 2);
  S << 0.0, 4.0, 4.0, 0.0;
  const Matrix B = double_center(S);
  CHECK(approx(B(0, 0), 1.0, 1e-14) && approx(B(0, 1), -1.0, 1e-14));
  Matrix asym(2, 2);
  asym << 0.0, 1.0, 3.0, 0.0;
  CHECK_THROWS_AS(double_center(asym), InvalidInput);
  // classical (81-128)
  const DistanceMatrix sq = unit_square();
  const Embedding e = classical_mds(sq, 2);
  CHECK(kruskal_stress(e.coords, sq) < 1e-8 && e.stress < 1e-8 && e.clamped_count == 0);
  Matrix D0(2, 2);
  D0 << 0.0, 2.0, 2.0, 0.0;
  const Embedding e2 = classical_mds(DistanceMatrix::from_matrix(D0), 1);
  CHECK(approx(e2.coords(0, 0), 1.0, 1e-12) && approx(e2.coords(1, 0), -1.0, 1e-12));
  CHECK(approx(e2.eigenvalues(0), 2.0, 1e-12));
  CHECK_THROWS_AS(classical_mds(sq, 0), InvalidInput);
  CHECK_THROWS_AS(classical_mds(sq, 4), InvalidInput);
  // kruskal_stress (148-157)
  Matrix pts(4, 2);
  pts << 0, 0, 1, 0, 1, 1, 0, 1;
  CHECK(kruskal_stress(pts, sq) < 1e-15);
  CHECK(kruskal_stress(Matrix::Zero(4, 2), sq) == 1.0);
  CHECK_THROWS_AS(kruskal_stress(Matrix::Zero(2, 1), DistanceMatrix::from_matrix(Matrix::Zero(2, 2))),
                  DegenerateInput);
  // stress_loss hand values (185-203)
  Matrix D5(2, 2);
  D5 << 0.0, 5.0, 5.0, 0.0;
  Matrix c1(2, 1);
  c1 << 0.0, 2.0;
  StressConfig cfg;
  cfg.huber_delta = 1.0;
  CHECK(approx(stress_loss(StressKind::huber, c1, DistanceMatrix::from_matrix(D5), cfg), 2.5, 1e-14));
  Matrix D2(2, 2);
  D2 << 0.0, 2.0, 2.0, 0.0;
  Matrix c2(2, 1);
  c2 << 0.0, 1.0;
  CHECK(approx(stress_loss(StressKind::sammon, c2, DistanceMatrix::from_matrix(D2), cfg), 0.25, 1e-14));
  // error paths (205-215)
  Matrix Dd(3, 3);
  Dd << 0, 0, 1, 0, 0, 1, 1, 1, 0;
  StressConfig plain;
  CHECK_THROWS_AS(stress_loss(StressKind::sammon, Matrix::Zero(3, 2), DistanceMatrix::from_matrix(Dd), plain),
                  DegenerateInput);
  CHECK_THROWS_AS(stress_loss(StressKind::huber, Matrix::Zero(3, 2), DistanceMatrix::from_matrix(Dd), plain),
                  InvalidConfig);
  // every kind reaches the optimum on the unit square (272-284)
  for (const StressKind kind : {StressKind::kruskal, StressKind::huber, StressKind::sammon, StressKind::smacof}) {
    StressConfig c;
    c.loss = kind;
    if (kind == StressKind::huber) c.huber_delta = 1.0;
    const Embedding f = minimize_stress(sq, 2, c);
    CHECK(f.stress < 1e-6 && f.converged && f.method != EmbeddingMethod::classical);
  }
  // non-convergence flag (343-358)
  StressConfig sc;
  sc.loss = StressKind::sammon;
  sc.max_iters = 1;
  sc.rel_tol = 1e-14;
  Matrix Xr(14, 4);
  for (int i = 0; i < 14; ++i)
    for (int j = 0; j < 4; ++j) Xr(i, j) = std::sin(1.0 + i * 0.7 + j * 1.3) * 2.0;
  const DistanceMatrix Dr = pairwise_matrix(Xr, MetricSpec::gini(2.0));
  const Embedding t = minimize_stress(Dr, 2, sc);
  CHECK(!t.converged && t.iterations == 1);
  CHECK_THROWS_AS(minimize_stress(Dr, 2, StressConfig{StressKind::kruskal, std::nullopt, std::nullopt, 0, 1e-6, 0}),
                  InvalidConfig);
}

static void tune_tests() {
  // NuGrid (test_tune.cpp:9-28)
  const NuGrid g = NuGrid::linspace();
  CHECK(g.size() == 30 && g.values().front() == 1.1 && g.values().back() == 5.0);
  CHECK_THROWS_AS(NuGrid::from_values({}), InvalidConfig);
  CHECK_THROWS_AS(NuGrid::from_values({2.0, 2.0}), InvalidConfig);
  CHECK_THROWS_AS(NuGrid::from_values({1.0, 2.0}), InvalidConfig);
  // ties to the smaller nu on constant data (85-93)
  Matrix X = Matrix::Ones(12, 3) * 4.2;
  const TuneReport r = tune_nu(X, 1, NuGrid::linspace(1.5, 3.5, 4), 3, EmbeddingMethod::classical, 5);
  CHECK(r.nu_star == 1.5);
  for (double s : r.mean_stress) CHECK(s == 0.0);
  // one fold + singleton grid == direct pipeline (36-46)
  Matrix X2(15, 4);
  for (int i = 0; i < 15; ++i)
    for (int j = 0; j < 4; ++j) X2(i, j) = std::cos(0.3 + i * 1.1 + j * 0.4) * 2.0;
  const TuneReport r2 = tune_nu(X2, 2, NuGrid::linspace(2.4, 2.4, 1), 1, EmbeddingMethod::classical, 9);
  const DistanceMatrix D = pairwise_matrix(X2, MetricSpec::gini(2.4));
  const Embedding direct = classical_mds(D, 2);
  CHECK(approx(r2.mean_stress[0], kruskal_stress(direct.coords, D), 1e-12));
  // alternating_tune T=1, grid {2} == one Sammon fit (112-124)
  const AlternatingResult alt = alternating_tune(X2, 2, 1, NuGrid::linspace(2.0, 2.0, 1), 3);
  StressConfig sam;
  sam.loss = StressKind::sammon;
  const Embedding fit = minimize_stress(pairwise_matrix(X2, MetricSpec::gini(2.0)), 2, sam);
  CHECK(alt.nu_star == 2.0 && approx(alt.embedding.stress, fit.stress, 1e-12));
  // the returned embeddings carry every Embedding field of the direct pipeline
  // (tools/main.cpp's embedding_diagnostics reads them for tune_report.json)
  CHECK(r2.best_embedding.method == EmbeddingMethod::classical);
  CHECK(r2.best_embedding.eigenvalues.size() == 2 && direct.eigenvalues.size() == 2);
  for (int k = 0; k < 2; ++k) CHECK(approx(r2.best_embedding.eigenvalues(k), direct.eigenvalues(k), 1e-12));
  CHECK(r2.best_embedding.clamped_count == direct.clamped_count);
  CHECK(approx(r2.best_embedding.clamped_mass, direct.clamped_mass, 1e-12));
  CHECK(r2.best_embedding.converged == direct.converged && r2.best_embedding.iterations == direct.iterations);
  CHECK(alt.embedding.method == EmbeddingMethod::sammon && alt.embedding.eigenvalues.size() == 0);
  CHECK(alt.embedding.iterations == fit.iterations && alt.embedding.converged == fit.converged);
  CHECK(alt.embedding.stress_history.size() == fit.stress_history.size() && fit.stress_history.size() > 1);
  for (std::size_t t = 0; t < fit.stress_history.size(); ++t)
    CHECK(approx(alt.embedding.stress_history[t], fit.stress_history[t], 1e-12));
  const TuneReport r3 = tune_nu(X2, 2, NuGrid::linspace(2.0, 2.0, 1), 1, EmbeddingMethod::kruskal, 9);
  StressConfig kr;
  kr.loss = StressKind::kruskal;
  const Embedding kfit = minimize_stress(pairwise_matrix(X2, MetricSpec::gini(2.0)), 2, kr);
  CHECK(r3.best_embedding.method == EmbeddingMethod::kruskal && r3.best_embedding.eigenvalues.size() == 0);
  CHECK(r3.best_embedding.iterations == kfit.iterations && r3.best_embedding.converged == kfit.converged);
  CHECK(r3.best_embedding.stress_history.size() == kfit.stress_history.size());
  CHECK(approx(r3.best_embedding.stress, kfit.stress, 1e-12));
  CHECK_THROWS_AS(alternating_tune(X2, 2, 0, NuGrid::linspace(2.0, 2.0, 1), 1), InvalidConfig);
}

int main() {
  for (auto& [name, fn] : std::vector<std::pair<const char*, std::function<void()>>>{
           {"metrics", metrics_tests}, {"embed", embed_tests}, {"tune", tune_tests}}) {
    try {
      fn();
    } catch (const std::exception& e) {
      ++g_fail;
      std::printf("%s: unexpected exception: %s\n", name, e.what());
    }
  }
  std::printf("%d checks, %d failed\n", g_checks, g_fail);
  return g_fail == 0 ? 0 : 1;
}
