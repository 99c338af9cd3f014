// Collectives of the row-sharded estimate behind one interface.
//
//   * NcclComm: the production backend -- one process (or thread) per GPU, NCCL over
//     NVLink / NVSwitch, every collective stream-ordered on the handle's stream.
//   * ThreadComm ("virtual shards"): G handles in ONE process, each driven by its own host
//     thread, exchanging through device staging slots with host barriers between the steps.
//     No kernel ever waits on another rank: a rank synchronises its own stream, then the host
//     barrier orders the ranks.  This is how the world > 1 branches of rld_api.cu run -- and are
//     checked against world = 1 and the oracle -- on a single GPU (tests/test_gpu_sharded.py),
//     and it works across devices of one process too (staging copies use UVA).
//
// Both backends reduce in a fixed order, so repeated runs are bit-identical for a fixed world.
#include <nccl.h>

#include <chrono>
#include <condition_variable>
#include <cstring>
#include <memory>
#include <mutex>

#include "comm.cuh"

struct rld_vgroup {
  int world = 1;
  std::mutex mu;
  std::condition_variable cv;
  int arrived = 0;
  uint64_t generation = 0;
  bool aborted = false;
  std::string why;
  std::vector<const void*> slot;   // per-rank published device pointers

  // All ranks arrive, or an abort / 300 s timeout fails every waiter.
  void barrier() {
    std::unique_lock<std::mutex> lk(mu);
    if (aborted) throw rld::Error{RLD_ERR_NCCL, "virtual group aborted: " + why};
    const uint64_t gen = generation;
    if (++arrived == world) {
      arrived = 0;
      ++generation;
      cv.notify_all();
      return;
    }
    const bool ok = cv.wait_for(lk, std::chrono::seconds(300), [&] { return generation != gen || aborted; });
    if (aborted) throw rld::Error{RLD_ERR_NCCL, "virtual group aborted: " + why};
    if (!ok) {
      aborted = true;
      why = "barrier timeout";
      cv.notify_all();
      throw rld::Error{RLD_ERR_NCCL, "virtual group barrier timed out"};
    }
  }

  void abort(const std::string& msg) {
    std::lock_guard<std::mutex> lk(mu);
    if (!aborted) {
      aborted = true;
      why = msg;
    }
    cv.notify_all();
  }
};

namespace rld {

namespace {

template <typename T, bool MAX>
__global__ void combine_kernel(const T* __restrict__ stage, int world, int64_t count, T* __restrict__ out) {
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < count; e += (int64_t)gridDim.x * blockDim.x) {
    T v = stage[e];
    for (int g = 1; g < world; ++g) {
      const T x = stage[(int64_t)g * count + e];
      v = MAX ? (x > v ? x : v) : v + x;   // rank order 0, 1, ..., G-1
    }
    out[e] = v;
  }
}

void nccl_check(ncclResult_t r, const char* what) {
  if (r != ncclSuccess) fail(RLD_ERR_NCCL, std::string(what) + ": " + ncclGetErrorString(r));
}

class NcclComm final : public Comm {
 public:
  NcclComm(const void* id, int rank, int world) {
    this->rank = rank;
    this->world = world;
    ncclUniqueId uid;
    memcpy(&uid, id, sizeof uid);
    nccl_check(ncclCommInitRank(&comm_, world, uid, rank), "ncclCommInitRank");
  }
  ~NcclComm() override {
    if (comm_) ncclCommDestroy(comm_);
  }
  void allreduce_sum(double* buf, int64_t count, cudaStream_t st) override {
    if (count > 0) nccl_check(ncclAllReduce(buf, buf, (size_t)count, ncclDouble, ncclSum, comm_, st), "ncclAllReduce");
  }
  void allreduce_max(int* buf, int64_t count, cudaStream_t st) override {
    if (count > 0) nccl_check(ncclAllReduce(buf, buf, (size_t)count, ncclInt32, ncclMax, comm_, st), "ncclAllReduce");
  }
  void allgather(const double* send, double* recv, int64_t count, cudaStream_t st) override {
    nccl_check(ncclAllGather(send, recv, (size_t)count, ncclDouble, comm_, st), "ncclAllGather");
  }
  const char* name() const override { return "nccl"; }

 private:
  ncclComm_t comm_ = nullptr;
};

class ThreadComm final : public Comm {
 public:
  ThreadComm(rld_vgroup* g, int rank) : g_(g) {
    this->rank = rank;
    this->world = g->world;
  }
  void abort(const std::string& why) override { g_->abort(why); }
  void allreduce_sum(double* buf, int64_t count, cudaStream_t st) override { reduce<double, false>(buf, count, st); }
  void allreduce_max(int* buf, int64_t count, cudaStream_t st) override { reduce<int, true>(buf, count, st); }
  void allgather(const double* send, double* recv, int64_t count, cudaStream_t st) override {
    publish(send, sizeof(double) * count, st);
    for (int g = 0; g < world; ++g)
      RLD_CUDA(cudaMemcpyAsync(recv + (int64_t)g * count, g_->slot[g], sizeof(double) * count, cudaMemcpyDefault, st));
    RLD_CUDA(cudaStreamSynchronize(st));
    g_->barrier();   // nobody refills a slot before every rank has read it
  }
  const char* name() const override { return "threads"; }

 private:
  // copy `bytes` of `src` into this rank's slot, wait for it, publish the slot, meet everyone
  void publish(const void* src, size_t bytes, cudaStream_t st) {
    mine_.reserve(std::max<size_t>(bytes, 8));
    if (bytes) RLD_CUDA(cudaMemcpyAsync(mine_.ptr, src, bytes, cudaMemcpyDefault, st));
    RLD_CUDA(cudaStreamSynchronize(st));
    {
      std::lock_guard<std::mutex> lk(g_->mu);
      if ((int)g_->slot.size() < world) g_->slot.resize(world, nullptr);
      g_->slot[rank] = mine_.ptr;
    }
    g_->barrier();
  }

  template <typename T, bool MAX>
  void reduce(T* buf, int64_t count, cudaStream_t st) {
    if (count <= 0) return;
    publish(buf, sizeof(T) * count, st);
    stage_.reserve(sizeof(T) * count * world);
    for (int g = 0; g < world; ++g)
      RLD_CUDA(cudaMemcpyAsync(stage_.as<T>() + (int64_t)g * count, g_->slot[g], sizeof(T) * count,
                               cudaMemcpyDefault, st));
    const int blocks = (int)std::min<int64_t>(ceil_div(count, 256), 1024);
    combine_kernel<T, MAX><<<blocks, 256, 0, st>>>(stage_.as<T>(), world, count, buf);
    RLD_LAUNCH_CHECK();
    RLD_CUDA(cudaStreamSynchronize(st));
    g_->barrier();
  }

  rld_vgroup* g_;
  DevBuf mine_, stage_;
};

}  // namespace

std::unique_ptr<Comm> make_nccl_comm(const void* id, int rank, int world) {
  return std::unique_ptr<Comm>(new NcclComm(id, rank, world));
}

std::unique_ptr<Comm> make_thread_comm(rld_vgroup* g, int rank) {
  if (!g) fail(RLD_ERR_INVALID_ARGUMENT, "virtual group is NULL");
  return std::unique_ptr<Comm>(new ThreadComm(g, rank));
}

}  // namespace rld

extern "C" {

int rld_vgroup_create(int32_t world_size, rld_vgroup** out) {
  if (!out || world_size < 1) return RLD_ERR_INVALID_ARGUMENT;
  rld_vgroup* g = new (std::nothrow) rld_vgroup();
  if (!g) return RLD_ERR_OUT_OF_MEMORY;
  g->world = world_size;
  g->slot.assign(world_size, nullptr);
  *out = g;
  return RLD_OK;
}

void rld_vgroup_destroy(rld_vgroup* g) { delete g; }

}  // extern "C"
