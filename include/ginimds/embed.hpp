// ginimds:: stress / embedding API of the B200 engine -- drop-in for
// /root/reference/proj/core/include/ginimds/embed.hpp.
#pragma once

#include <cstdint>
#include <optional>
#include <vector>

#include "ginimds/metrics.hpp"

namespace ginimds {

enum class StressKind { kruskal, huber, sammon, smacof };
enum class EmbeddingMethod { classical, kruskal, huber, sammon, smacof };

const char* to_string(EmbeddingMethod m);
const char* to_string(StressKind k);

struct StressConfig {
  StressKind loss = StressKind::smacof;
  std::optional<double> huber_delta{};
  std::optional<Matrix> smacof_weights{};
  int max_iters = 300;
  double rel_tol = 1e-6;
  std::uint64_t seed = 0;
};

struct Embedding {
  Matrix coords;
  Vector eigenvalues;
  double stress = 0.0;
  EmbeddingMethod method = EmbeddingMethod::classical;
  int clamped_count = 0;
  double clamped_mass = 0.0;
  bool converged = true;
  int iterations = 0;
  double huber_delta = 0.0;
  std::vector<double> stress_history;
};

Matrix double_center(const Matrix& squared_distances);
Embedding classical_mds(const DistanceMatrix& D, int p);
double kruskal_stress(const Matrix& coords, const DistanceMatrix& D);
double stress_loss(StressKind kind, const Matrix& coords, const DistanceMatrix& D, const StressConfig& config);
Matrix stress_gradient(StressKind kind, const Matrix& coords, const DistanceMatrix& D, const StressConfig& config);
Embedding minimize_stress(const DistanceMatrix& D, int p, const StressConfig& config);

/// Engine extension: the same minimiser started from a given
/// layout instead of classical_mds(D, p).coords.
Embedding minimize_stress_from(const DistanceMatrix& D, const Matrix& init, const StressConfig& config);

}  // namespace ginimds
