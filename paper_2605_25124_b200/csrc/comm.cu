// Collectives (comm.h): NCCL ranks and the single-device local rank group, and
// their C-ABI (gmds_comm_*, include/gmds.h).
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <string>

#include "comm.h"
#include "common.cuh"
#include "kernels.cuh"

namespace gmds {

namespace {

// NCCL is bound at run time, on first use: a process that loads libgmds before torch must
// not pin a libnccl.so.2 other than torch's (torch's libtorch_cuda needs symbols of its own,
// newer NCCL).  Preference: the libnccl.so.2 already in the process (torch's), else torch's
// bundled copy (GMDS_NCCL_PATH, fixed at build time), else the system one.  The API used is
// the stable subset every NCCL 2.x exports.
struct NcclApi {
  ncclResult_t (*GetUniqueId)(ncclUniqueId*);
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int);
  ncclResult_t (*CommDestroy)(ncclComm_t);
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t, cudaStream_t);
  ncclResult_t (*GroupStart)();
  ncclResult_t (*GroupEnd)();
  const char* (*GetErrorString)(ncclResult_t);
};

const NcclApi& nccl() {
  static NcclApi api = [] {
    NcclApi a{};
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
#ifdef GMDS_NCCL_PATH
    if (!h) h = dlopen(GMDS_NCCL_PATH, RTLD_NOW | RTLD_GLOBAL);
#endif
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) return a;
    auto sym = [h](const char* name) { return dlsym(h, name); };
    a.GetUniqueId = reinterpret_cast<decltype(a.GetUniqueId)>(sym("ncclGetUniqueId"));
    a.CommInitRank = reinterpret_cast<decltype(a.CommInitRank)>(sym("ncclCommInitRank"));
    a.CommDestroy = reinterpret_cast<decltype(a.CommDestroy)>(sym("ncclCommDestroy"));
    a.AllReduce = reinterpret_cast<decltype(a.AllReduce)>(sym("ncclAllReduce"));
    a.GroupStart = reinterpret_cast<decltype(a.GroupStart)>(sym("ncclGroupStart"));
    a.GroupEnd = reinterpret_cast<decltype(a.GroupEnd)>(sym("ncclGroupEnd"));
    a.GetErrorString = reinterpret_cast<decltype(a.GetErrorString)>(sym("ncclGetErrorString"));
    return a;
  }();
  if (!api.GetUniqueId || !api.CommInitRank || !api.CommDestroy || !api.AllReduce || !api.GroupStart ||
      !api.GroupEnd || !api.GetErrorString)
    fail(GMDS_NCCL_ERROR, "NCCL (libnccl.so.2) could not be loaded");
  return api;
}

void nccl_check(ncclResult_t r, const char* what) {
  if (r != ncclSuccess) fail(GMDS_NCCL_ERROR, std::string(what) + ": " + nccl().GetErrorString(r));
}

ncclRedOp_t nccl_op(RedOp op) {
  switch (op) {
    case RedOp::kMin: return ncclMin;
    case RedOp::kMax: return ncclMax;
    default: return ncclSum;
  }
}

struct NcclComm final : Comm {
  ncclComm_t c = nullptr;
  ~NcclComm() override {
    if (c) nccl().CommDestroy(c);
  }
  void allreduce(double* buf, size_t count, RedOp op, cudaStream_t st) override {
    nccl_check(nccl().AllReduce(buf, buf, count, ncclDouble, nccl_op(op), c, st), "ncclAllReduce");
  }
  void allreduce_group(double* const* bufs, const size_t* counts, int k, cudaStream_t st) override {
    nccl_check(nccl().GroupStart(), "ncclGroupStart");
    for (int i = 0; i < k; ++i)
      nccl_check(nccl().AllReduce(bufs[i], bufs[i], counts[i], ncclDouble, ncclSum, c, st), "ncclAllReduce");
    nccl_check(nccl().GroupEnd(), "ncclGroupEnd");
  }
  const char* kind() const override { return "nccl"; }
};

constexpr int kMaxLocalRanks = 16;
struct RankPtrs {
  double* p[kMaxLocalRanks];
};

// v = buf_0 op buf_1 op ... op buf_{N-1} (rank order), written back to every rank's buffer
__global__ void local_allreduce_kernel(RankPtrs b, int nranks, size_t count, int op) {
  for (size_t k = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x; k < count;
       k += static_cast<size_t>(gridDim.x) * blockDim.x) {
    double v = b.p[0][k];
    for (int r = 1; r < nranks; ++r) {
      const double x = b.p[r][k];
      v = (op == 0) ? v + x : (op == 1 ? fmin(v, x) : fmax(v, x));
    }
    for (int r = 0; r < nranks; ++r) b.p[r][k] = v;
  }
}

struct LocalGroup {
  int size = 0;
  std::mutex mu;
  std::condition_variable cv;
  int arrived = 0;
  uint64_t gen = 0;
  RankPtrs bufs{};
  std::vector<cudaEvent_t> ev;
  cudaEvent_t done = nullptr;

  void barrier() {
    std::unique_lock<std::mutex> lk(mu);
    const uint64_t g = gen;
    if (++arrived == size) {
      arrived = 0;
      ++gen;
      cv.notify_all();
    } else {
      cv.wait(lk, [&] { return gen != g; });
    }
  }
  ~LocalGroup() {
    for (cudaEvent_t e : ev) cudaEventDestroy(e);
    if (done) cudaEventDestroy(done);
  }
};

struct LocalGroupComm final : Comm {
  std::shared_ptr<LocalGroup> g;
  void allreduce(double* buf, size_t count, RedOp op, cudaStream_t st) override {
    g->bufs.p[rank] = buf;
    GMDS_CUDA(cudaEventRecord(g->ev[rank], st));
    g->barrier();  // every rank's partial is enqueued before its event
    if (rank == 0) {
      for (int r = 0; r < size; ++r) GMDS_CUDA(cudaStreamWaitEvent(st, g->ev[r], 0));
      const unsigned blocks = static_cast<unsigned>(std::max<size_t>(1, std::min<size_t>((count + 255) / 256, 1184)));
      local_allreduce_kernel<<<blocks, 256, 0, st>>>(g->bufs, size, count, op == RedOp::kSum ? 0 : (op == RedOp::kMin ? 1 : 2));
      count_launch();
      check_launch("local_allreduce_kernel");
      GMDS_CUDA(cudaEventRecord(g->done, st));
    }
    g->barrier();  // the reduction is enqueued before anyone waits on it
    if (rank != 0) GMDS_CUDA(cudaStreamWaitEvent(st, g->done, 0));
  }
  const char* kind() const override { return "local"; }
};

}  // namespace

}  // namespace gmds

using namespace gmds;

extern "C" {

gmds_status gmds_comm_unique_id(unsigned char* id) {
  return guard([&] {
    static_assert(sizeof(ncclUniqueId) == GMDS_COMM_ID_BYTES, "ncclUniqueId size");
    ncclUniqueId u;
    nccl_check(nccl().GetUniqueId(&u), "ncclGetUniqueId");
    std::memcpy(id, &u, sizeof u);
  });
}

gmds_status gmds_comm_init_nccl(const unsigned char* id, int32_t nranks, int32_t rank, gmds_comm** out) {
  return guard([&] {
    *out = nullptr;
    if (nranks < 1 || rank < 0 || rank >= nranks) fail(GMDS_INVALID_CONFIG, "comm: bad rank / size");
    auto c = std::make_unique<NcclComm>();
    c->rank = rank;
    c->size = nranks;
    ncclUniqueId u;
    std::memcpy(&u, id, sizeof u);
    nccl_check(nccl().CommInitRank(&c->c, nranks, u, rank), "ncclCommInitRank");
    auto* h = new gmds_comm();
    GMDS_CUDA(cudaGetDevice(&h->device));
    h->impl = std::move(c);
    *out = h;
  });
}

gmds_status gmds_comm_init_local(int32_t nranks, gmds_comm** comms) {
  return guard([&] {
    if (nranks < 1 || nranks > kMaxLocalRanks) fail(GMDS_INVALID_CONFIG, "comm: local groups hold 1..16 ranks");
    auto g = std::make_shared<LocalGroup>();
    g->size = nranks;
    g->ev.resize(static_cast<size_t>(nranks));
    for (auto& e : g->ev) GMDS_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    GMDS_CUDA(cudaEventCreateWithFlags(&g->done, cudaEventDisableTiming));
    int dev = 0;
    GMDS_CUDA(cudaGetDevice(&dev));
    for (int r = 0; r < nranks; ++r) {
      auto c = std::make_unique<LocalGroupComm>();
      c->rank = r;
      c->size = nranks;
      c->g = g;
      comms[r] = new gmds_comm();
      comms[r]->device = dev;
      comms[r]->impl = std::move(c);
    }
  });
}

int32_t gmds_comm_rank(const gmds_comm* c) { return c ? c->impl->rank : -1; }
int32_t gmds_comm_size(const gmds_comm* c) { return c ? c->impl->size : 0; }

gmds_status gmds_comm_allreduce_device(gmds_comm* c, double* dbuf, int64_t count, int32_t op, void* stream) {
  return guard([&] {
    if (!c) fail(GMDS_INVALID_INPUT, "comm: null handle");
    if (op < 0 || op > 2) fail(GMDS_INVALID_CONFIG, "comm: op must be 0 (sum), 1 (min) or 2 (max)");
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    c->impl->allreduce(dbuf, static_cast<size_t>(count), op == 0 ? RedOp::kSum : (op == 1 ? RedOp::kMin : RedOp::kMax),
                       st);
    GMDS_CUDA(cudaStreamSynchronize(st));
  });
}

void gmds_comm_free(gmds_comm* c) { delete c; }

}  // extern "C"
