// Collectives for the hot path: the reference Communicator's all_reduce_sum
// and barrier (comm.hpp:28-52, comm.cpp:420-432) over NCCL on the context's
// CUDA stream. NCCL is dlopen'ed ("libnccl.so.2"), so the library has no
// link-time NCCL dependency and, inside a torch process, shares the NCCL
// torch already loaded. CollectiveStats are counted exactly like the
// reference (scalar = length 1, vector otherwise), also for world == 1.
#include <dlfcn.h>

#include <chrono>
#include <cstring>
#include <thread>
#include <mutex>
#include <set>
#include <tuple>

#include "sf_internal.hpp"

namespace sfb {

void set_max_dynamic_smem(const void* kernel, int bytes) {
  static std::mutex mu;
  static std::set<std::tuple<const void*, int, int>> done;
  int dev = 0;
  SF_CUDA(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> g(mu);
  if (done.count({kernel, dev, bytes})) return;
  SF_CUDA(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
  done.insert({kernel, dev, bytes});
}

namespace {
// nccl.h (2.27/2.28): ncclUniqueId is 128 bytes, ncclFloat64 = 8, ncclSum = 0
struct UniqueId {
  char internal[128];
};
using ncclComm_t = void*;
using GetUniqueId = int (*)(UniqueId*);
using CommInitRank = int (*)(ncclComm_t*, int, UniqueId, int);
using AllReduce = int (*)(const void*, void*, size_t, int, int, ncclComm_t, cudaStream_t);
using CommDestroy = int (*)(ncclComm_t);
using CommAbort = int (*)(ncclComm_t);
using CommGetAsyncError = int (*)(ncclComm_t, int*);
using GetErrorString = const char* (*)(int);
constexpr int kFloat64 = 8;
constexpr int kSum = 0;

void* open_nccl() {
  static void* lib = nullptr;
  if (lib) return lib;
  for (const char* name : {"libnccl.so.2", "libnccl.so"}) {
    lib = dlopen(name, RTLD_NOW | RTLD_GLOBAL);
    if (lib) return lib;
  }
  throw ProtocolError(std::string("cannot load NCCL (libnccl.so.2): ") + dlerror());
}

template <typename F>
F sym(void* lib, const char* name) {
  void* p = dlsym(lib, name);
  if (!p) throw ProtocolError(std::string("NCCL symbol missing: ") + name);
  return reinterpret_cast<F>(p);
}
}  // namespace

struct Nccl {
  ncclComm_t comm = nullptr;
  AllReduce all_reduce = nullptr;
  CommDestroy destroy = nullptr;
  CommAbort abort = nullptr;
  CommGetAsyncError async_error = nullptr;
  GetErrorString err = nullptr;
  bool aborted = false;
  ~Nccl() {
    if (comm && destroy && !aborted) destroy(comm);
  }
  void check(int rc, const char* what) const {
    if (rc != 0)
      throw ProtocolError(std::string(what) + ": " + (err ? err(rc) : "nccl error"));
  }
};

void nccl_unique_id(void* out128) {
  void* lib = open_nccl();
  auto get = sym<GetUniqueId>(lib, "ncclGetUniqueId");
  UniqueId id;
  const int rc = get(&id);
  if (rc != 0) throw ProtocolError("ncclGetUniqueId failed");
  std::memcpy(out128, id.internal, 128);
}

void nccl_join(Ctx& ctx, const void* id128, int rank, int world) {
  if (world < 1 || rank < 0 || rank >= world)
    throw DataError("invalid worker rank " + std::to_string(rank) + " of " +
                    std::to_string(world));
  ctx.rank = rank;
  ctx.world = world;
  ctx.nccl.reset();
  if (world == 1) return;
  void* lib = open_nccl();
  auto n = std::make_unique<Nccl>();
  n->all_reduce = sym<AllReduce>(lib, "ncclAllReduce");
  n->destroy = sym<CommDestroy>(lib, "ncclCommDestroy");
  n->abort = sym<CommAbort>(lib, "ncclCommAbort");
  n->async_error = sym<CommGetAsyncError>(lib, "ncclCommGetAsyncError");
  n->err = sym<GetErrorString>(lib, "ncclGetErrorString");
  auto init = sym<CommInitRank>(lib, "ncclCommInitRank");
  UniqueId id;
  std::memcpy(id.internal, id128, 128);
  SF_CUDA(cudaSetDevice(ctx.device));
  n->check(init(&n->comm, world, id, rank), "ncclCommInitRank");
  ctx.nccl = std::move(n);
}

void comm_drop_nccl(Ctx& ctx) { ctx.nccl.reset(); }

void comm_sync(Ctx& ctx) {
  if (!(ctx.world > 1 && ctx.nccl)) {
    SF_CUDA(cudaStreamSynchronize(ctx.stream));
    return;
  }
  const auto t0 = std::chrono::steady_clock::now();
  for (uint64_t spin = 0;; ++spin) {
    const cudaError_t q = cudaStreamQuery(ctx.stream);
    if (q == cudaSuccess) return;
    if (q != cudaErrorNotReady) SF_CUDA(q);
    int async = 0;
    if (ctx.nccl->async_error(ctx.nccl->comm, &async) == 0 && async != 0 && async != 7 /* ncclInProgress */) {
      ctx.nccl->abort(ctx.nccl->comm);
      ctx.nccl->aborted = true;
      throw ProtocolError(std::string("collective failed: ") + (ctx.nccl->err ? ctx.nccl->err(async) : "nccl error"));
    }
    const auto waited = std::chrono::duration_cast<std::chrono::milliseconds>(std::chrono::steady_clock::now() - t0);
    if (waited.count() > ctx.comm_timeout_ms) {
      // a peer never entered the collective: abort so the pending NCCL
      // kernel exits, then fail like the reference's rendezvous timeout
      ctx.nccl->abort(ctx.nccl->comm);
      ctx.nccl->aborted = true;
      cudaStreamSynchronize(ctx.stream);
      throw ProtocolError("collective timed out after " + std::to_string(ctx.comm_timeout_ms) +
                          " ms (rank " + std::to_string(ctx.rank) + " of " + std::to_string(ctx.world) + ")");
    }
    if (spin > 1000) std::this_thread::yield();
  }
}

void comm_allreduce_sum(Ctx& ctx, double* dev_buf, size_t count) {
  if (count == 1)
    ++ctx.stats.scalar_allreduce;
  else
    ++ctx.stats.vector_allreduce;
  ctx.stats.doubles_reduced += count;
  if (ctx.world == 1 && ctx.host_comm.all_reduce) {
    // one worker: the sum is the identity; the caller's Communicator still
    // sees (and counts) the collective, like the reference's LocalComm
    if (ctx.host_comm.all_reduce(ctx.host_comm.user, nullptr, count) != 0)
      throw ProtocolError("host communicator all_reduce_sum failed");
    return;
  }
  if (ctx.world == 1 || count == 0) return;
  if (ctx.host_comm.all_reduce) {
    ctx.comm_stage.reserve(count);
    SF_CUDA(cudaMemcpyAsync(ctx.comm_stage.p, dev_buf, count * 8, cudaMemcpyDeviceToHost, ctx.stream));
    SF_CUDA(cudaStreamSynchronize(ctx.stream));
    if (ctx.host_comm.all_reduce(ctx.host_comm.user, ctx.comm_stage.p, count) != 0)
      throw ProtocolError("host communicator all_reduce_sum failed");
    SF_CUDA(cudaMemcpyAsync(dev_buf, ctx.comm_stage.p, count * 8, cudaMemcpyHostToDevice, ctx.stream));
    SF_CUDA(cudaStreamSynchronize(ctx.stream));  // the staging buffer is reused
    ctx.d2h_bytes += count * 8;
    ctx.h2d_bytes += count * 8;
    return;
  }
  if (!ctx.nccl) throw ProtocolError("multi-rank context without a communicator");
  if (ctx.nccl->aborted) throw ProtocolError("communicator aborted after an earlier failure");
  ctx.nccl->check(ctx.nccl->all_reduce(dev_buf, dev_buf, count, kFloat64, kSum,
                                       ctx.nccl->comm, ctx.stream),
                  "ncclAllReduce");
}

void comm_barrier(Ctx& ctx) {
  ++ctx.stats.barriers;
  if (ctx.host_comm.barrier) {
    SF_CUDA(cudaStreamSynchronize(ctx.stream));
    if (ctx.host_comm.barrier(ctx.host_comm.user) != 0) throw ProtocolError("host communicator barrier failed");
    return;
  }
  if (ctx.world > 1) {
    if (!ctx.nccl) throw ProtocolError("multi-rank context without a communicator");
    if (ctx.nccl->aborted) throw ProtocolError("communicator aborted after an earlier failure");
    DevBuf<double>& one = ctx.barrier_buf;
    one.reserve(1);
    SF_CUDA(cudaMemsetAsync(one.p, 0, sizeof(double), ctx.stream));
    ctx.nccl->check(ctx.nccl->all_reduce(one.p, one.p, 1, kFloat64, kSum, ctx.nccl->comm,
                                         ctx.stream),
                    "ncclAllReduce(barrier)");
  }
  comm_sync(ctx);
}

Ctx::Ctx() = default;

Ctx::~Ctx() {
  if (stream) cudaStreamSynchronize(stream);
  for (cudaEvent_t& e : events)
    if (e) cudaEventDestroy(e);
  if (plan_ready) cudaEventDestroy(plan_ready);
  for (auto& pr : dom_events) {
    cudaEventDestroy(pr.first);
    cudaEventDestroy(pr.second);
  }
  nccl.reset();
  if (stream) cudaStreamDestroy(stream);
}

}  // namespace sfb
