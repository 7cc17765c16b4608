// Collectives of the row-sharded path, behind one interface:
//   NCCL      — the product transport (one process per GPU, NVLink/NVSwitch);
//   loopback  — a TEST transport (include/lrqmm_debug.h): several handles of ONE process, one host
//               thread per rank, all on one device, so that liblrqmm's own sharded schedule runs on
//               a single GPU.  Its collectives are host-synchronised (stream sync + host barrier +
//               a plain reduce / copy of the peers' buffers on the caller's stream): no kernel ever
//               waits on another rank's kernel.
#pragma once
#include <cuda_runtime.h>

#include <cstddef>

namespace lrqmm {

enum { kCommF32 = 0, kCommF64 = 1 };

struct Comm {
  int world = 1, rank = 0;
  virtual ~Comm() = default;
  // in-place elementwise sum over the ranks of n elements (kCommF32 / kCommF64) at buf, enqueued on
  // st; identical bits on every rank.  0 on success.
  virtual int allreduce(void* buf, size_t n, int dtype, cudaStream_t st) = 0;
  // in-place allgather: rank i contributes the `bytes` at full + i * bytes; afterwards every rank's
  // full[0 .. world * bytes) holds every block.  0 on success.
  virtual int allgather(void* full, size_t bytes, cudaStream_t st) = 0;
  // whether the collectives may be captured into a CUDA graph
  virtual bool capturable() const = 0;
  // 0 while healthy (NCCL async errors, loopback barrier timeouts)
  virtual int async_error() = 0;
};

// nullptr on failure
Comm* comm_create_nccl(int world, int rank, const unsigned char id[128]);
// all ranks of `group` must use the same world and device; nullptr on a mismatch
Comm* comm_create_loopback(int group, int world, int rank, int device);

}  // namespace lrqmm
