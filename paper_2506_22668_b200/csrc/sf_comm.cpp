// Collectives for the hot path: the reference Communicator's all_reduce_sum
// and barrier (comm.hpp:28-52, comm.cpp:420-432) over NCCL on the context's
// CUDA stream. NCCL is dlopen'ed ("libnccl.so.2"), so the library has no
// link-time NCCL dependency and, inside a torch process, shares the NCCL
// torch already loaded. CollectiveStats are counted exactly like the
// reference (scalar = length 1, vector otherwise), also for world == 1.
#include <dlfcn.h>

#include <cstring>
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
  GetErrorString err = nullptr;
  ~Nccl() {
    if (comm && destroy) destroy(comm);
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
  n->err = sym<GetErrorString>(lib, "ncclGetErrorString");
  auto init = sym<CommInitRank>(lib, "ncclCommInitRank");
  UniqueId id;
  std::memcpy(id.internal, id128, 128);
  SF_CUDA(cudaSetDevice(ctx.device));
  n->check(init(&n->comm, world, id, rank), "ncclCommInitRank");
  ctx.nccl = std::move(n);
}

void comm_allreduce_sum(Ctx& ctx, double* dev_buf, size_t count) {
  if (count == 1)
    ++ctx.stats.scalar_allreduce;
  else
    ++ctx.stats.vector_allreduce;
  ctx.stats.doubles_reduced += count;
  if (ctx.world == 1 || count == 0) return;
  if (!ctx.nccl) throw ProtocolError("multi-rank context without a communicator");
  ctx.nccl->check(ctx.nccl->all_reduce(dev_buf, dev_buf, count, kFloat64, kSum,
                                       ctx.nccl->comm, ctx.stream),
                  "ncclAllReduce");
}

void comm_barrier(Ctx& ctx) {
  ++ctx.stats.barriers;
  if (ctx.world > 1) {
    if (!ctx.nccl) throw ProtocolError("multi-rank context without a communicator");
    DevBuf<double>& one = ctx.barrier_buf;
    one.reserve(1);
    SF_CUDA(cudaMemsetAsync(one.p, 0, sizeof(double), ctx.stream));
    ctx.nccl->check(ctx.nccl->all_reduce(one.p, one.p, 1, kFloat64, kSum, ctx.nccl->comm,
                                         ctx.stream),
                    "ncclAllReduce(barrier)");
  }
  SF_CUDA(cudaStreamSynchronize(ctx.stream));
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
