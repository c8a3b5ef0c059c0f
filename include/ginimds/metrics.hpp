// ginimds:: rank / distance API of the B200 engine -- drop-in for
// /root/reference/proj/core/include/ginimds/metrics.hpp (same names,
// signatures, exceptions).  Every call runs on the GPU through libgmds's
// C-ABI (include/gmds.h); there is no CPU implementation behind it.
//
// Difference in representation (not in results): a DistanceMatrix built by
// pairwise_matrix lives in HBM as a packed upper triangle; its n x n host
// image is materialised on first use of matrix() / operator(), so pipelines
// like minimize_stress(pairwise_matrix(X, spec), ...) never copy D to the host.
#pragma once

#include <Eigen/Dense>

#include <memory>
#include <optional>
#include <span>
#include <string>

#include "ginimds/error.hpp"

struct gmds_dmat;

namespace ginimds {

using Matrix = Eigen::MatrixXd;
using Vector = Eigen::VectorXd;

struct RankVector {
  Vector ranks;
};

struct SurvivalVector {
  Vector values;
  double at_zero = 0.5;
};

class GiniParams {
public:
  explicit GiniParams(double nu) : nu_(nu) {
    if (!(nu > 1.0)) throw InvalidConfig("GiniParams: nu must be > 1, got " + std::to_string(nu));
  }
  double nu() const noexcept { return nu_; }

private:
  double nu_;
};

class DistanceMatrix {
public:
  /// Validates symmetry (to 1e-12 relative), nonnegativity and zero diagonal.
  static DistanceMatrix from_matrix(Matrix m);

  int n() const noexcept;
  double operator()(int i, int j) const { return matrix()(i, j); }
  const Matrix& matrix() const;

  /// Engine extension: the device-resident packed matrix (created on demand).
  const gmds_dmat* device() const;

  struct Impl;

private:
  explicit DistanceMatrix(std::shared_ptr<Impl> impl) : impl_(std::move(impl)) {}
  std::shared_ptr<Impl> impl_;
  friend DistanceMatrix pairwise_matrix(const Matrix& X, const struct MetricSpec& spec);
  friend DistanceMatrix make_device_distance(gmds_dmat* handle, int n);
};

struct MetricSpec {
  static MetricSpec euclidean() { return MetricSpec{}; }
  static MetricSpec gini(double nu) { return MetricSpec{GiniParams(nu)}; }
  bool is_gini() const noexcept { return params.has_value(); }
  std::optional<GiniParams> params;
};

RankVector midrank(const Vector& v);
RankVector midrank(std::span<const double> v);

double gini_norm(const Vector& x);
double gini_norm(std::span<const double> x);

double gini_pseudo_distance(const Vector& x, const Vector& y);
double gini_pseudo_distance(std::span<const double> x, std::span<const double> y);

SurvivalVector empirical_survival(const Vector& z);
SurvivalVector empirical_survival(std::span<const double> z);

double gen_gini_directed(const Vector& x, const Vector& y, const GiniParams& params);
double gen_gini_directed(std::span<const double> x, std::span<const double> y, const GiniParams& params);

double gen_gini_distance(const Vector& x, const Vector& y, const GiniParams& params);
double gen_gini_distance(std::span<const double> x, std::span<const double> y, const GiniParams& params);

DistanceMatrix pairwise_matrix(const Matrix& X, const MetricSpec& spec);

/// Engine extension: wrap a device handle produced through the C-ABI.
DistanceMatrix make_device_distance(gmds_dmat* handle, int n);

}  // namespace ginimds
