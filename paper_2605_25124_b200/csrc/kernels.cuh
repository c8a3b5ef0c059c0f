// Internal kernel launch interface of libgmds (host side).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "gmds.h"

namespace gmds {

// Packed upper-triangle tile image used for every device-resident D:
// kPT x kPT blocks (I <= J), each stored row-major, blocks in row-major
// upper-triangle order.  Entries with i >= j or j >= n are zero.
constexpr int kPT = 128;

__host__ __device__ int64_t packed_offset(int64_t i, int64_t j, int64_t nb);
int64_t packed_elems(int64_t n);

struct GiniTileArgs {
  int64_t n;           // rows
  int d;               // features (p)
  int tile;            // pairs tile edge (rows per panel)
  int64_t nbt;         // tile rows = ceil(n / tile)
  int64_t tile_begin;  // [begin, end) of this launch's tiles (pairs for p > 1024)
  int64_t tile_end;
  const double* lut;   // nnu x 2d, device
  int nnu;
  int packed;          // 0: full n x n per nu; 1: packed tile image per nu
  int64_t nb_packed;   // ceil(n / kPT)
  int64_t out_stride;  // elements between consecutive nu outputs
  int* flag;           // device: bit0 = non-finite distance produced, bit1 = pair not scored
  // score mode (fused nu-sweep scorer): instead of storing D_nu, accumulate
  // sum (|y_i - y_j| - D_nu)^2 and sum D_nu^2 for every nu (kruskal_stress of
  // a fixed embedding against every grid value).
  const double* Y;     // n x q row-major fp64 (nullptr: store mode)
  int q;
  double* score_part;  // [gridDim][nnu][2] per-CTA partials (fixed-order sums)
  // row-sharded packed builds (gmds_dmat_gini_sharded): only tiles inside packed
  // blocks [blk_lo, blk_hi) are computed (blk_hi <= blk_lo: every tile); needs kPT % tile == 0
  int64_t blk_lo, blk_hi;
};

__host__ __device__ inline bool tile_in_blocks(const GiniTileArgs& a, int64_t I, int64_t J) {
  if (a.blk_hi <= a.blk_lo) return true;
  const int64_t bI = I * a.tile / kPT, bJ = J * a.tile / kPT;
  const int64_t b = bI * a.nb_packed - (bI * (bI - 1)) / 2 + (bJ - bI);
  return b >= a.blk_lo && b < a.blk_hi;
}

constexpr int kMaxScoreNu = 64;

void count_launch(int64_t k = 1);
int64_t launch_count();

int gini_tile_size(int d, gmds_dtype xt, int nnu);
void launch_midrank(const double* dv, const void* dX, gmds_dtype xt, const int64_t* dpairs, int64_t nseg, int d,
                    double* dranks, cudaStream_t st);
void launch_gini(GiniTileArgs a, const void* dX, gmds_dtype xt, void* dout, gmds_dtype ot, cudaStream_t st,
                 int64_t max_blocks = 0);
void launch_euclid(const void* dX, gmds_dtype xt, int64_t n, int d, double* dout, cudaStream_t st);
// tcgen05 path (euclid_tc.cu): full n x n fp64 out; used when euclid_tc_enabled (GMDS_EUCLID=exact|tc overrides)
bool euclid_tc_enabled(int64_t n, int64_t p);
void launch_euclid_tc(const void* dX, gmds_dtype xt, int64_t n, int p, double* dout, cudaStream_t st);
void launch_transpose(const void* din, gmds_dtype t, int64_t rows, int64_t cols, void* dout, cudaStream_t st);

}  // namespace gmds
