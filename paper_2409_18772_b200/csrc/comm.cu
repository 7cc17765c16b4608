// Transports of the row-sharded path (comm.h).
#include <nccl.h>

#include <chrono>
#include <condition_variable>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>

#include "comm.h"
#include "kernels.h"

namespace lrqmm {

// ------------------------------------------------------------------ NCCL
namespace {

class NcclComm final : public Comm {
 public:
  ncclComm_t c = nullptr;
  ~NcclComm() override {
    if (c) ncclCommDestroy(c);
  }
  int allreduce(void* buf, size_t n, int dtype, cudaStream_t st) override {
    return ncclAllReduce(buf, buf, n, dtype == kCommF64 ? ncclFloat64 : ncclFloat32, ncclSum, c, st) == ncclSuccess ? 0 : 1;
  }
  int allgather(void* full, size_t bytes, cudaStream_t st) override {
    char* base = reinterpret_cast<char*>(full);
    return ncclAllGather(base + bytes * rank, base, bytes, ncclInt8, c, st) == ncclSuccess ? 0 : 1;
  }
  // NCCL collectives are stream-capturable: the RSVD graph of a multi-rank handle contains them
  bool capturable() const override { return true; }
  int async_error() override {
    ncclResult_t ar = ncclSuccess;
    if (ncclCommGetAsyncError(c, &ar) != ncclSuccess) return 1;
    return ar == ncclSuccess ? 0 : 1;
  }
};

// --------------------------------------------------------------- loopback
// Sum of the ranks' buffers in rank order 0..world-1 (the same order, hence the same bits, on every
// rank); every rank reads all peers' buffers (same device) and writes its private scratch.
struct SumArgs {
  const void* src[8];
  int nsrc;
  void* dst;
  size_t n;
};

template <typename T>
__global__ void k_loopback_sum(SumArgs a) {
  const T* const* s = reinterpret_cast<const T* const*>(a.src);
  T* d = reinterpret_cast<T*>(a.dst);
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < a.n; i += (size_t)gridDim.x * blockDim.x) {
    T v = s[0][i];
    for (int r = 1; r < a.nsrc; ++r) v += s[r][i];
    d[i] = v;
  }
}

struct Group {
  int world = 0, device = -1, members = 0;
  std::mutex m;
  std::condition_variable cv;
  int arrived = 0;
  long generation = 0;
  bool broken = false;
  void* slot[8] = {};
  // returns false on timeout (a rank that never arrives) -- the group is then broken for good
  bool barrier() {
    std::unique_lock<std::mutex> l(m);
    if (broken) return false;
    const long gen = generation;
    if (++arrived == world) {
      arrived = 0;
      ++generation;
      cv.notify_all();
      return true;
    }
    const bool ok = cv.wait_for(l, std::chrono::seconds(120), [&] { return generation != gen || broken; });
    if (!ok || broken) {
      broken = true;
      cv.notify_all();
      return false;
    }
    return true;
  }
};

std::mutex g_groups_m;
std::map<int, std::shared_ptr<Group>> g_groups;

class LoopbackComm final : public Comm {
 public:
  std::shared_ptr<Group> g;
  int group_id = 0;
  void* scratch = nullptr;
  size_t scratch_bytes = 0;
  int err = 0;
  ~LoopbackComm() override {
    cudaFree(scratch);
    std::lock_guard<std::mutex> l(g_groups_m);
    if (--g->members == 0) g_groups.erase(group_id);
  }
  int fail() {
    err = 1;
    return 1;
  }
  int allreduce(void* buf, size_t n, int dtype, cudaStream_t st) override {
    if (err) return 1;
    const size_t bytes = n * (dtype == kCommF64 ? 8 : 4);
    if (bytes > scratch_bytes) {
      cudaFree(scratch);
      scratch = nullptr;
      if (cudaMalloc(&scratch, bytes) != cudaSuccess) return fail();
      scratch_bytes = bytes;
    }
    // every rank's contribution is complete before anyone reads it
    if (cudaStreamSynchronize(st) != cudaSuccess) return fail();
    g->slot[rank] = buf;
    if (!g->barrier()) return fail();
    SumArgs a{};
    for (int r = 0; r < world; ++r) a.src[r] = g->slot[r];
    a.nsrc = world;
    a.dst = scratch;
    a.n = n;
    const int grid = (int)((n + 255) / 256 < 1024 ? (n + 255) / 256 : 1024);
    if (n > 0) {
      if (dtype == kCommF64) k_loopback_sum<double><<<grid, 256, 0, st>>>(a);
      else k_loopback_sum<float><<<grid, 256, 0, st>>>(a);
      ++launch_counter();
    }
    if (cudaStreamSynchronize(st) != cudaSuccess) return fail();
    // nobody still reads buf once every rank passed this barrier
    if (!g->barrier()) return fail();
    if (n > 0 && cudaMemcpyAsync(buf, scratch, bytes, cudaMemcpyDeviceToDevice, st) != cudaSuccess) return fail();
    return 0;
  }
  int allgather(void* full, size_t bytes, cudaStream_t st) override {
    if (err) return 1;
    if (cudaStreamSynchronize(st) != cudaSuccess) return fail();
    g->slot[rank] = full;
    if (!g->barrier()) return fail();
    for (int r = 0; r < world; ++r)
      if (r != rank && bytes > 0 &&
          cudaMemcpyAsync(reinterpret_cast<char*>(full) + r * bytes, reinterpret_cast<const char*>(g->slot[r]) + r * bytes,
                          bytes, cudaMemcpyDeviceToDevice, st) != cudaSuccess)
        return fail();
    if (cudaStreamSynchronize(st) != cudaSuccess) return fail();
    // a rank may overwrite its own block (next quantize) only after every peer copied it
    if (!g->barrier()) return fail();
    return 0;
  }
  bool capturable() const override { return false; }  // host-synchronised
  int async_error() override { return err; }
};

}  // namespace

Comm* comm_create_nccl(int world, int rank, const unsigned char id[128]) {
  ncclUniqueId uid;
  static_assert(sizeof(uid.internal) == 128, "ncclUniqueId size");
  memcpy(uid.internal, id, 128);
  NcclComm* c = new NcclComm();
  c->world = world;
  c->rank = rank;
  if (ncclCommInitRank(&c->c, world, uid, rank) != ncclSuccess) {
    c->c = nullptr;
    delete c;
    return nullptr;
  }
  return c;
}

Comm* comm_create_loopback(int group, int world, int rank, int device) {
  if (world < 2 || world > 8 || rank < 0 || rank >= world) return nullptr;
  std::shared_ptr<Group> g;
  {
    std::lock_guard<std::mutex> l(g_groups_m);
    auto it = g_groups.find(group);
    if (it == g_groups.end()) {
      g = std::make_shared<Group>();
      g->world = world;
      g->device = device;
      g_groups[group] = g;
    } else {
      g = it->second;
      if (g->world != world || g->device != device || g->members >= world) return nullptr;
    }
    ++g->members;
  }
  LoopbackComm* c = new LoopbackComm();
  c->g = g;
  c->group_id = group;
  c->world = world;
  c->rank = rank;
  return c;
}

}  // namespace lrqmm
