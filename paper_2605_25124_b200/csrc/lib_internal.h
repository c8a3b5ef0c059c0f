// Host helpers shared by the C-ABI translation units.
#pragma once

#include <cuda_runtime.h>

#include <vector>

#include "common.cuh"

namespace gmds {

void call_stream_push(cudaStream_t s, cudaStream_t* prev);
void call_stream_pop(cudaStream_t prev);

// The stream of one library call (the caller's, via gmds_set_stream, or a
// private one).  While it lives, DevBufs released on this thread return to
// the pool ordered after this stream's work (pool.cu).
// A call on a caller-provided stream (the *_device entry points).
struct CallScope {
  cudaStream_t prev = nullptr;
  explicit CallScope(cudaStream_t s) { call_stream_push(s, &prev); }
  ~CallScope() { call_stream_pop(prev); }
  CallScope(const CallScope&) = delete;
  CallScope& operator=(const CallScope&) = delete;
};

struct Stream {
  cudaStream_t s = nullptr;
  cudaStream_t prev = nullptr;
  bool owned = true;
  Stream();
  ~Stream();
  Stream(const Stream&) = delete;
  Stream& operator=(const Stream&) = delete;
};

void require_device();
void check_nu(double nu);
void check_finite_host(const void* X, gmds_dtype xt, int64_t count, const char* who);
std::vector<double> build_lut(int d, const double* nus, int nnu);
DevBuf<unsigned char> upload_rows(const void* X, gmds_dtype xt, gmds_layout lx, int64_t n, int64_t p,
                                  cudaStream_t st);
// fp64 host input exactly representable in fp32 -> fp32 copy in buf (xt updated), else X unchanged
const void* narrow_exact_f32(const void* X, gmds_dtype& xt, int64_t m, std::vector<float>& buf);
// Fused nu-sweep scoring request: instead of storing D_nu, return per nu
// num = sum (|y_i - y_j| - D_nu)^2 and den = sum D_nu^2 over i < j (host arrays).
struct ScoreSpec {
  const double* dY = nullptr;  // n x q row-major fp64, device
  int q = 0;
  double* num = nullptr;
  double* den = nullptr;
  bool ok = false;  // out: false when a pair needed the overflow path (caller falls back)
};

// Progress of a full-layout (unpacked) distance run: tiles are enumerated
// block row by block row, and a tile (I, J) writes block (I, J) and its mirror
// (J, I), so once the tiles of block rows [0, R) are done, output rows
// [0, R * tile) are final.  run_gini then calls rows_done(rows, st) (after the
// launch on st); a caller may start copying those rows out.  late_writes is
// set when a pass over overflow pairs rewrote arbitrary entries afterwards.
struct RowSink {
  virtual ~RowSink() = default;
  virtual void rows_done(int64_t rows, cudaStream_t st) = 0;
  bool late_writes = false;
  int chunks = 12;
};

void run_gini(const void* dX, gmds_dtype xt, int64_t n, int64_t p, const double* nus, int nnu, gmds_dtype ot,
              int packed, void* dD, int shard, int nshards, cudaStream_t st, int* dflag, ScoreSpec* score = nullptr,
              RowSink* sink = nullptr, const int64_t* blk_range = nullptr);
void check_flag(int* dflag, cudaStream_t st);
// flag |= 4 when any of the m input entries is not finite
void launch_finite_check(const void* dX, gmds_dtype xt, int64_t m, int* dflag, cudaStream_t st);

}  // namespace gmds
