// ginimds:: drop-in facade over the libgmds C-ABI (include/gmds.h).  Pure
// host glue: argument marshalling, status -> exception mapping, and the
// DistanceMatrix host/device dual representation.  All arithmetic of the
// path runs in libgmds's CUDA kernels.
#include <atomic>
#include <cmath>
#include <cstring>
#include <limits>
#include <mutex>
#include <string>

#include "ginimds/ginimds.hpp"
#include "gmds.h"

namespace ginimds {

namespace {

void check(gmds_status s) {
  if (s == GMDS_OK) return;
  const std::string msg = gmds_last_error();
  switch (s) {
    case GMDS_INVALID_INPUT: throw InvalidInput(msg);
    case GMDS_INVALID_CONFIG: throw InvalidConfig(msg);
    case GMDS_DEGENERATE_INPUT: throw DegenerateInput(msg);
    case GMDS_NUMERIC_FAILURE: throw NumericFailure(msg);
    case GMDS_CUDA_ERROR:
    case GMDS_NCCL_ERROR: throw DeviceError(msg);
    default: throw Error(msg);
  }
}

std::span<const double> as_span(const Vector& v) { return {v.data(), static_cast<std::size_t>(v.size())}; }

int kind_code(StressKind k) { return static_cast<int>(k); }

}  // namespace

// ---------------------------------------------------------------------------
// DistanceMatrix: host image (reference semantics) and/or device handle.

struct DistanceMatrix::Impl {
  int n = 0;
  mutable std::mutex mu;
  mutable std::optional<Matrix> host;
  mutable std::shared_ptr<gmds_dmat> dev;
};

namespace {
std::shared_ptr<gmds_dmat> own(gmds_dmat* h) { return std::shared_ptr<gmds_dmat>(h, [](gmds_dmat* p) { gmds_dmat_free(p); }); }
}  // namespace

DistanceMatrix DistanceMatrix::from_matrix(Matrix m) {
  if (m.rows() != m.cols()) throw InvalidInput("DistanceMatrix: matrix is not square");
  if (m.rows() < 1) throw InvalidInput("DistanceMatrix: matrix is empty");
  // validation + clamp on the upload path (gmds_dmat_from_host applies from_matrix's rules)
  gmds_dmat* h = nullptr;
  check(gmds_dmat_from_host(m.data(), m.rows(), GMDS_F64, &h));
  auto impl = std::make_shared<Impl>();
  impl->n = static_cast<int>(m.rows());
  impl->dev = own(h);
  return DistanceMatrix(impl);
}

int DistanceMatrix::n() const noexcept { return impl_ ? impl_->n : 0; }

const Matrix& DistanceMatrix::matrix() const {
  std::lock_guard<std::mutex> g(impl_->mu);
  if (!impl_->host) {
    Matrix m(impl_->n, impl_->n);
    check(gmds_dmat_download(impl_->dev.get(), m.data()));
    impl_->host = std::move(m);
  }
  return *impl_->host;
}

const gmds_dmat* DistanceMatrix::device() const {
  std::lock_guard<std::mutex> g(impl_->mu);
  if (!impl_->dev) {
    gmds_dmat* h = nullptr;
    check(gmds_dmat_from_host(impl_->host->data(), impl_->n, GMDS_F64, &h));
    impl_->dev = own(h);
  }
  return impl_->dev.get();
}

DistanceMatrix make_device_distance(gmds_dmat* handle, int n) {
  auto impl = std::make_shared<DistanceMatrix::Impl>();
  impl->n = n;
  impl->dev = own(handle);
  return DistanceMatrix(impl);
}

// ---------------------------------------------------------------------------
// metrics

RankVector midrank(std::span<const double> v) {
  RankVector out;
  out.ranks.resize(static_cast<Eigen::Index>(v.size()));
  check(gmds_midrank_batch(v.data(), 1, static_cast<int64_t>(v.size()), out.ranks.data()));
  return out;
}
RankVector midrank(const Vector& v) { return midrank(as_span(v)); }

double gini_norm(std::span<const double> x) {
  double r = 0.0;
  check(gmds_gini_norm(x.data(), static_cast<int64_t>(x.size()), &r));
  return r;
}
double gini_norm(const Vector& x) { return gini_norm(as_span(x)); }

double gini_pseudo_distance(std::span<const double> x, std::span<const double> y) {
  double r = 0.0;
  check(gmds_gini_pseudo_distance(x.data(), static_cast<int64_t>(x.size()), y.data(), static_cast<int64_t>(y.size()),
                                  &r));
  return r;
}
double gini_pseudo_distance(const Vector& x, const Vector& y) { return gini_pseudo_distance(as_span(x), as_span(y)); }

SurvivalVector empirical_survival(std::span<const double> z) {
  SurvivalVector out;
  out.values.resize(static_cast<Eigen::Index>(z.size()));
  check(gmds_empirical_survival(z.data(), static_cast<int64_t>(z.size()), out.values.data()));
  return out;
}
SurvivalVector empirical_survival(const Vector& z) { return empirical_survival(as_span(z)); }

double gen_gini_directed(std::span<const double> x, std::span<const double> y, const GiniParams& params) {
  double r = 0.0;
  check(gmds_gen_gini_directed(x.data(), static_cast<int64_t>(x.size()), y.data(), static_cast<int64_t>(y.size()),
                               params.nu(), &r));
  return r;
}
double gen_gini_directed(const Vector& x, const Vector& y, const GiniParams& params) {
  return gen_gini_directed(as_span(x), as_span(y), params);
}

double gen_gini_distance(std::span<const double> x, std::span<const double> y, const GiniParams& params) {
  double r = 0.0;
  check(gmds_gen_gini_distance(x.data(), static_cast<int64_t>(x.size()), y.data(), static_cast<int64_t>(y.size()),
                               params.nu(), &r));
  return r;
}
double gen_gini_distance(const Vector& x, const Vector& y, const GiniParams& params) {
  return gen_gini_distance(as_span(x), as_span(y), params);
}

DistanceMatrix pairwise_matrix(const Matrix& X, const MetricSpec& spec) {
  const int64_t n = X.rows(), p = X.cols();
  if (spec.is_gini()) {
    gmds_dmat* h = nullptr;
    check(gmds_dmat_gini(X.data(), GMDS_F64, GMDS_COL_MAJOR, n, p, spec.params->nu(), GMDS_F64, &h));
    return make_device_distance(h, static_cast<int>(n));
  }
  Matrix D(n, n);
  check(gmds_pairwise_euclidean(X.data(), GMDS_F64, GMDS_COL_MAJOR, n, p, D.data()));
  auto impl = std::make_shared<DistanceMatrix::Impl>();
  impl->n = static_cast<int>(n);
  impl->host = std::move(D);
  return DistanceMatrix(impl);
}

// ---------------------------------------------------------------------------
// embed

const char* to_string(EmbeddingMethod m) {
  switch (m) {
    case EmbeddingMethod::classical: return "classical";
    case EmbeddingMethod::kruskal: return "kruskal";
    case EmbeddingMethod::huber: return "huber";
    case EmbeddingMethod::sammon: return "sammon";
    case EmbeddingMethod::smacof: return "smacof";
  }
  return "?";
}

const char* to_string(StressKind k) {
  switch (k) {
    case StressKind::kruskal: return "kruskal";
    case StressKind::huber: return "huber";
    case StressKind::sammon: return "sammon";
    case StressKind::smacof: return "smacof";
  }
  return "?";
}

Matrix double_center(const Matrix& S) {
  if (S.rows() != S.cols() || S.rows() < 1) throw InvalidInput("double_center: matrix is not square");
  Matrix B(S.rows(), S.cols());
  check(gmds_double_center(S.data(), S.rows(), B.data()));
  return B;
}

namespace {
void check_coords(const Matrix& coords, const DistanceMatrix& D, const char* who) {
  if (coords.rows() != D.n())
    throw InvalidInput(std::string(who) + ": coords rows (" + std::to_string(coords.rows()) +
                       ") do not match distance matrix size (" + std::to_string(D.n()) + ")");
  if (!coords.allFinite()) throw InvalidInput(std::string(who) + ": non-finite coordinates");
}
double delta_of(const StressConfig& c) {
  return c.huber_delta ? *c.huber_delta : std::numeric_limits<double>::quiet_NaN();
}
const double* weights_of(const StressConfig& c, const DistanceMatrix& D) {
  if (!c.smacof_weights) return nullptr;
  if (c.smacof_weights->rows() != D.n() || c.smacof_weights->cols() != D.n())
    throw InvalidConfig("minimize_stress: smacof_weights size mismatch");
  return c.smacof_weights->data();
}
EmbeddingMethod method_of(StressKind k) {
  switch (k) {
    case StressKind::kruskal: return EmbeddingMethod::kruskal;
    case StressKind::huber: return EmbeddingMethod::huber;
    case StressKind::sammon: return EmbeddingMethod::sammon;
    case StressKind::smacof: return EmbeddingMethod::smacof;
  }
  return EmbeddingMethod::smacof;
}
}  // namespace

Embedding classical_mds(const DistanceMatrix& D, int p) {
  const int n = D.n();
  if (p < 1 || p > n - 1)
    throw InvalidInput("classical_mds: target dimension must satisfy 1 <= p <= n-1, got p=" + std::to_string(p) +
                       " with n=" + std::to_string(n));
  Embedding out;
  out.method = EmbeddingMethod::classical;
  out.coords.resize(n, p);
  out.eigenvalues.resize(p);
  int32_t cc = 0;
  check(gmds_classical_mds(D.device(), p, out.coords.data(), out.eigenvalues.data(), &cc, &out.clamped_mass,
                           &out.stress));
  out.clamped_count = cc;
  return out;
}

double kruskal_stress(const Matrix& coords, const DistanceMatrix& D) {
  check_coords(coords, D, "kruskal_stress");
  double r = 0.0;
  check(gmds_kruskal_stress(D.device(), coords.data(), static_cast<int32_t>(coords.cols()), &r));
  return r;
}

double stress_loss(StressKind kind, const Matrix& coords, const DistanceMatrix& D, const StressConfig& config) {
  check_coords(coords, D, "stress_loss");
  double r = 0.0;
  check(gmds_stress_loss(kind_code(kind), D.device(), coords.data(), static_cast<int32_t>(coords.cols()),
                         delta_of(config), weights_of(config, D), &r));
  return r;
}

Matrix stress_gradient(StressKind kind, const Matrix& coords, const DistanceMatrix& D, const StressConfig& config) {
  check_coords(coords, D, "stress_gradient");
  Matrix g(coords.rows(), coords.cols());
  check(gmds_stress_gradient(kind_code(kind), D.device(), coords.data(), static_cast<int32_t>(coords.cols()),
                             delta_of(config), weights_of(config, D), g.data()));
  return g;
}

namespace {
Embedding fit(const DistanceMatrix& D, int p, const StressConfig& config, const Matrix* init) {
  gmds_stress_cfg c{};
  c.kind = kind_code(config.loss);
  c.huber_delta = delta_of(config);
  c.smacof_weights = weights_of(config, D);
  c.max_iters = config.max_iters;
  c.rel_tol = config.rel_tol;
  c.seed = config.seed;
  Embedding out;
  out.coords.resize(D.n(), p);
  std::vector<double> hist(static_cast<std::size_t>(std::max(config.max_iters, 1)) + 2);
  gmds_fit_result r{};
  r.coords = out.coords.data();
  r.history = hist.data();
  r.history_cap = static_cast<int64_t>(hist.size());
  check(gmds_minimize_stress(D.device(), p, &c, init ? init->data() : nullptr, &r));
  hist.resize(static_cast<std::size_t>(std::min<int64_t>(r.history_len, r.history_cap)));
  out.stress = r.stress;
  out.method = method_of(config.loss);
  out.converged = r.converged != 0;
  out.iterations = r.iterations;
  out.huber_delta = r.huber_delta;
  out.stress_history = std::move(hist);
  return out;
}
}  // namespace

Embedding minimize_stress(const DistanceMatrix& D, int p, const StressConfig& config) {
  return fit(D, p, config, nullptr);
}

Embedding minimize_stress_from(const DistanceMatrix& D, const Matrix& init, const StressConfig& config) {
  check_coords(init, D, "minimize_stress");
  return fit(D, static_cast<int>(init.cols()), config, &init);
}

// ---------------------------------------------------------------------------
// tune

NuGrid NuGrid::linspace(double lo, double hi, int count) {
  if (count < 1) throw InvalidConfig("NuGrid: count must be >= 1");
  std::vector<double> values;
  if (count == 1) {
    values.push_back(lo);
  } else {
    const double step = (hi - lo) / static_cast<double>(count - 1);
    for (int i = 0; i < count; ++i) values.push_back(lo + step * i);
    values.back() = hi;
  }
  return from_values(std::move(values));
}

NuGrid NuGrid::from_values(std::vector<double> values) {
  if (values.empty()) throw InvalidConfig("NuGrid: empty grid");
  for (std::size_t i = 0; i < values.size(); ++i) {
    if (!(values[i] > 1.0)) throw InvalidConfig("NuGrid: every value must be > 1");
    if (i > 0 && !(values[i] > values[i - 1]))
      throw InvalidConfig("NuGrid: values must be strictly increasing (no duplicates)");
  }
  return NuGrid(std::move(values));
}

namespace {
// Embedding by value from a gmds_embedding filled by the library (every field of embed.hpp:28-40)
struct EmbeddingOut {
  gmds_embedding raw{};
  Embedding e;
  std::vector<double> hist;
  EmbeddingOut(Eigen::Index n, int p) {
    e.coords.resize(n, p);
    e.eigenvalues.resize(p);
    hist.resize(302);  // embed_distances' default StressConfig: max_iters 300 -> <= 301 entries
    raw.coords = e.coords.data();
    raw.eigenvalues = e.eigenvalues.data();
    raw.history = hist.data();
    raw.history_cap = static_cast<int64_t>(hist.size());
  }
  Embedding finish() {
    if (raw.n_eigenvalues != e.eigenvalues.size()) e.eigenvalues.resize(raw.n_eigenvalues);  // 0: stress fits
    hist.resize(static_cast<std::size_t>(std::min<int64_t>(raw.history_len, raw.history_cap)));
    e.stress_history = std::move(hist);
    e.method = static_cast<EmbeddingMethod>(raw.method);
    e.stress = raw.stress;
    e.clamped_count = raw.clamped_count;
    e.clamped_mass = raw.clamped_mass;
    e.converged = raw.converged != 0;
    e.iterations = raw.iterations;
    e.huber_delta = raw.huber_delta;
    return std::move(e);
  }
};
}  // namespace

TuneReport tune_nu(const Matrix& X, int p, const NuGrid& grid, int k_folds, EmbeddingMethod method,
                   std::uint64_t seed) {
  TuneReport r;
  r.grid = grid.values();
  r.mean_stress.resize(grid.size());
  r.folds = k_folds;
  r.seed = seed;
  EmbeddingOut out(X.rows(), p);
  check(gmds_tune_nu_ex(X.data(), GMDS_F64, GMDS_COL_MAJOR, X.rows(), X.cols(), p, grid.values().data(),
                        static_cast<int32_t>(grid.size()), k_folds, static_cast<int32_t>(method), seed,
                        r.mean_stress.data(), &r.nu_star, &out.raw));
  r.best_embedding = out.finish();
  return r;
}

AlternatingResult alternating_tune(const Matrix& X, int p, int outer_iters, const NuGrid& grid, std::uint64_t seed) {
  AlternatingResult r;
  r.nu_path.resize(static_cast<std::size_t>(std::max(outer_iters, 0)));
  EmbeddingOut out(X.rows(), p);
  check(gmds_alternating_tune_ex(X.data(), GMDS_F64, GMDS_COL_MAJOR, X.rows(), X.cols(), p, outer_iters,
                                 grid.values().data(), static_cast<int32_t>(grid.size()), seed, r.nu_path.data(),
                                 &r.nu_star, &out.raw));
  r.embedding = out.finish();
  return r;
}

// ---------------------------------------------------------------------------
// parallel knobs (recorded; device work does not depend on them)

namespace {
std::atomic<int>& cap() {
  static std::atomic<int> c{0};
  return c;
}
}  // namespace

int max_threads() {
  const int c = cap().load();
  if (c > 0) return c;
  const unsigned h = std::thread::hardware_concurrency();
  return h == 0 ? 1 : static_cast<int>(h);
}
void set_max_threads(int n) { cap().store(n > 0 ? n : 0); }

}  // namespace ginimds
