// Collectives of the multi-GPU path: one rank per GPU, the
// collective enqueued on the rank's stream so it is ordered with the passes it
// connects (no host round trip per iteration).
//
//   NcclComm        -- ncclAllReduce over NVLink / NVSwitch (production: one
//                      process per GPU, the unique id shared by the caller's
//                      own plumbing, e.g. torch.distributed).
//   LocalGroupComm  -- N ranks in ONE process on one device, each driven by its
//                      own host thread and stream: the reduction is one kernel
//                      over every rank's buffer in rank order, ordered by CUDA
//                      events and host barriers at enqueue time (no kernel ever
//                      waits on another).  For testing the sharded path with fewer
//                      GPUs than ranks (B200_PROFILING.md: emulate ranks as one
//                      kernel over all ranks' data).
#pragma once

#include <cuda_runtime.h>

#include <condition_variable>
#include <memory>
#include <mutex>
#include <vector>

#include "gmds.h"

namespace gmds {

enum class RedOp { kSum, kMin, kMax };

struct Comm {
  int rank = 0, size = 1;
  virtual ~Comm() = default;
  // in place, enqueued on st; every rank receives bit-identical results
  virtual void allreduce(double* buf, size_t count, RedOp op, cudaStream_t st) = 0;
  // several sum all-reduces issued as one group (NCCL: one fused launch)
  virtual void allreduce_group(double* const* bufs, const size_t* counts, int k, cudaStream_t st) {
    for (int i = 0; i < k; ++i) allreduce(bufs[i], counts[i], RedOp::kSum, st);
  }
  virtual const char* kind() const = 0;
};

// Contiguous share [lo, hi) of `units` for `rank` of `size` (the partition every sharded
// entry uses: packed blocks of D, grid values of a sweep).
inline void share_of(int64_t units, int rank, int size, int64_t& lo, int64_t& hi) {
  lo = units * rank / size;
  hi = units * (rank + 1) / size;
}

}  // namespace gmds

// The C-ABI handle (include/gmds.h) owns one rank's collective.
struct gmds_comm {
  std::unique_ptr<gmds::Comm> impl;
  int device = 0;
};
