// Collective interface of the row-sharded estimate (comm.cu): NCCL in production, host-barrier
// "virtual shards" for G ranks in one process (single-GPU testing of the world > 1 paths).
#pragma once

#include <memory>
#include <string>

#include "rld_internal.cuh"

namespace rld {

struct Comm {
  int rank = 0, world = 1;
  virtual ~Comm() = default;
  // in place, fixed rank order
  virtual void allreduce_sum(double* buf, int64_t count, cudaStream_t st) = 0;
  virtual void allreduce_max(int* buf, int64_t count, cudaStream_t st) = 0;
  // recv = [world][count], rank g's `send` at g * count
  virtual void allgather(const double* send, double* recv, int64_t count, cudaStream_t st) = 0;
  // a rank failed: make the other ranks' pending / next collectives fail instead of hang
  virtual void abort(const std::string&) {}
  virtual const char* name() const = 0;
};

std::unique_ptr<Comm> make_nccl_comm(const void* nccl_id, int rank, int world);
std::unique_ptr<Comm> make_thread_comm(rld_vgroup* group, int rank);

}  // namespace rld
