// Stress engine bound to one device DistanceMatrix (host side).
#pragma once

#include <cuda_runtime.h>

#include <memory>
#include <vector>

#include "comm.h"
#include "common.cuh"
#include "dmat.cuh"
#include "stress.cuh"

namespace gmds {

// The tiled passes' work list: chunks of up to chunk_len blocks of one block row,
// in packed (row-major) order.  A row-sharded D holds the blocks of a contiguous
// chunk range balanced by block count (shard_blocks), so shard edges are chunk edges.
int64_t chunk_blocks(int64_t nb);
void chunk_list(int64_t nb, int64_t len, std::vector<int64_t>& cI, std::vector<int64_t>& cJ);
void shard_blocks(int64_t n, int rank, int size, int64_t& blk_lo, int64_t& blk_hi);

struct Engine {
  const gmds_dmat* D;
  int q, Q;
  bool rows_mode;
  cudaStream_t st;
  int64_t n = 0, nb = 0, nchunks = 0;
  int64_t chunk_len = 1;  // 128x128 blocks per CTA of a tiled pass (set from chunk_blocks(nb): up to 8)
  int64_t passes = 0;  // passes over D issued by this engine
  int64_t stride_row = 0, stride_col = 0;
  const void* W = nullptr;
  DevBuf<int64_t> chunk_I, chunk_J0, strip_first;
  DevBuf<double> rowpart, colpart, losspart, graw, scal, Y, sqpart;
  DevBuf<double> cand[kMaxCand];

  Comm* comm = nullptr;  // row-sharded engine: this rank's chunks, sums all-reduced after every pass
  DevBuf<double> xred, dsum, rawy;  // sharded device loop payload, difference-pass sums, raw loss at Y
  Engine(const gmds_dmat* D, int q, cudaStream_t st, Comm* comm = nullptr);
  void allreduce(double* d, size_t count);  // no-op unless sharded
  void upload(const double* coords_colmajor, double* dst);
  void download(const double* src, double* coords_colmajor);
  PassArgs args(int kind, double delta) const;
  // raw loss sums at up to kMaxCand configurations (one pass)
  std::vector<double> loss_raw(int kind, double delta, const double* const* Ys, int nc);
  // the same in fp64 arithmetic over fp32 storage (stress_pass_kernel<.., float, .., double>)
  std::vector<double> loss_raw_precise(int kind, double delta, const double* const* Ys, int nc);
  // e^2 kinds over fp32 storage: raw losses at Y and at Y - s0 g, Y - s1 g (g = graw, scaled),
  // the trial values as Y's plus accurately summed differences (difference pass)
  std::vector<double> loss_diff(int kind, double s0, double s1);
  // raw gradient sums into graw, returns the raw loss at Yd (one pass)
  double grad_raw(int kind, double delta, const double* Yd);
  // raw sums over one shard's chunks (sharded fits; summed across ranks)
  double grad_raw_shard(int kind, double delta, const double* Yd, int shard, int nshards);
  // graw *= scale, returns |graw|^2
  double scale_grad(double scale);
  // One round trip per gradient-descent iteration: gradient pass at Y, the
  // kind's scale applied on the device, trial points Y - s0 g -> cand[0] and
  // Y - s1 g -> cand[1], and their loss pass.  Returns raw loss at Y, |g|^2
  // (scaled g) and the two raw trial losses.
  struct GradTrials {
    double raw, gsq, trial[2];
  };
  GradTrials grad_and_trials(int kind, double delta, double s0, double s1);
  // Speculative variant (fp32 storage, q <= 4): with graw holding the raw
  // gradient at Y (and losspart column 0 the raw loss at Y), scale it, form
  // cand[0] = Y - s0 g and cand[1] = Y - s1 g, and in ONE pass over D get both
  // trial losses plus the raw gradient at cand[0] (into gnext; losspart column
  // 0 then holds the raw loss at cand[0]).
  bool fused_ok() const { return D->storage == GMDS_F32 && !rows_mode; }
  // the tiled passes over fp32 storage (TMA kernels) leave fp32 row/column partials
  bool f32parts() const { return D->storage == GMDS_F32 && !rows_mode; }
  GradTrials fused_trials(int kind, double delta, double s0, double s1);
  DevBuf<double> gnext;
  DevBuf<double> gpart;  // two-level row reduction scratch
  // Device-resident gradient descent (gd_step_kernel): from a state where graw
  // holds the raw gradient at Y and losspart column 0 the raw loss at Y, run
  // iterations on the device until one finishes the fit (stop 1) or needs the
  // host (stop 2: that iteration's trial losses and |g|^2 are in the state).
  // Appends the accepted losses to history.
  GdState device_gd(int kind, double delta, double f, double step, int it, int pred, int max_iters, double rel_tol,
                    std::vector<double>& history, double precise_rel, bool need_grad = false, bool init = false);
  DevBuf<double> sq2, hist;
  DevBuf<GdState> gdst;
  double loss_of(int kind, double raw) const;
};

// Engine for (D, q) on stream st: a cached workspace when free, else a fresh one.
struct EngineLease {
  std::shared_ptr<Engine> e;
  const gmds_dmat* D = nullptr;
  int slot = -1;
  Engine* operator->() const { return e.get(); }
  Engine& operator*() const { return *e; }
  EngineLease() = default;
  EngineLease(const EngineLease&) = delete;
  EngineLease(EngineLease&& o) noexcept : e(std::move(o.e)), D(o.D), slot(o.slot) {
    o.D = nullptr;
    o.slot = -1;
  }
  EngineLease& operator=(const EngineLease&) = delete;
  ~EngineLease();
};
EngineLease acquire_engine(const gmds_dmat* D, int q, cudaStream_t st);

void dmat_finish(gmds_dmat* d, cudaStream_t st);
void classical_mds_dev(const gmds_dmat* D, int q, double* coords, double* eigvals, int* clamped_count,
                       double* clamped_mass, double* stress, cudaStream_t st);
bool classical_mds_batch_dev(const std::vector<const gmds_dmat*>& Ds, int q, std::vector<std::vector<double>>& coords,
                             std::vector<double>& stress, cudaStream_t st);
void minimize_stress_dev(const gmds_dmat* D, int q, const gmds_stress_cfg& cfg, const double* Y0, gmds_fit_result* res,
                         cudaStream_t st, const double* init_cache);

}  // namespace gmds
