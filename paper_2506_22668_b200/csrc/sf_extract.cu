// Computational-graph extraction on the device (graph.cpp:195-261), for large
// graphs / balls: the reference's sequential BFS ball, induced player list and
// local CSR, byte-identical to it (and to the host version in sf_host.cpp).
//
//  * BFS, level-synchronous. The reference assigns local ids in discovery
//    order: frontier nodes in order, each one's neighbours in CSR order,
//    first sighting wins. Level l's candidate positions p (the concatenation
//    of the frontier's neighbour lists, an exclusive scan of their degrees)
//    are exactly that order, so a new node's id is decided by the smallest p
//    at which it appears (atomicMin per node), and ids are assigned by a scan
//    over the winning positions.
//  * Local CSR: row lu = the ball neighbours of lu in ascending local id
//    (the reference fills rows in player order, which is that order), built
//    by a count / scan / fill / segmented radix sort.
//  * Players: the upper part (lv > lu) of each row, in row order, is the
//    lexicographically sorted player list; edge_player of an upper entry is
//    its position there, of a lower entry (lw < lu) the position of lu in
//    row lw's upper part (binary search).
// The graph's CSR is uploaded once per context and graph (like its features).
#include <cuda_runtime.h>

#include <cub/cub.cuh>
#include <vector>

#include "sf_internal.hpp"

namespace sfb {

namespace {

constexpr uint32_t kNone = 0xFFFFFFFFu;

inline unsigned nblk(uint64_t n, unsigned t = 256) { return unsigned((n + t - 1) / t); }

__global__ void frontier_deg_kernel(const uint64_t* __restrict__ rp, const uint32_t* __restrict__ l2g, uint32_t fb,
                                    uint32_t fe, uint64_t* __restrict__ deg) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= fe - fb) return;
  const uint32_t g = l2g[fb + i];
  deg[i] = rp[g + 1] - rp[g];
}

// position p -> (frontier index i, neighbour) ; off: exclusive scan of the degrees
__device__ __forceinline__ uint32_t frontier_of(const uint64_t* off, uint32_t nf, uint64_t p) {
  uint32_t lo = 0, hi = nf;  // last i with off[i] <= p
  while (hi - lo > 1) {
    const uint32_t mid = (lo + hi) >> 1;
    if (off[mid] <= p) lo = mid; else hi = mid;
  }
  return lo;
}

__global__ void candidate_kernel(const uint64_t* __restrict__ rp, const uint32_t* __restrict__ col,
                                 const uint32_t* __restrict__ l2g, uint32_t fb, uint32_t nf,
                                 const uint64_t* __restrict__ off, uint64_t total,
                                 const uint32_t* __restrict__ local_of, unsigned long long* __restrict__ first) {
  const uint64_t p = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x;
  if (p >= total) return;
  const uint32_t i = frontier_of(off, nf, p);
  const uint32_t nb = col[rp[l2g[fb + i]] + (p - off[i])];
  if (local_of[nb] == kNone) atomicMin(&first[nb], (unsigned long long)p);
}

__global__ void winner_kernel(const uint64_t* __restrict__ rp, const uint32_t* __restrict__ col,
                              const uint32_t* __restrict__ l2g, uint32_t fb, uint32_t nf,
                              const uint64_t* __restrict__ off, uint64_t total,
                              const uint32_t* __restrict__ local_of, const unsigned long long* __restrict__ first,
                              uint32_t* __restrict__ flag) {
  const uint64_t p = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x;
  if (p >= total) return;
  const uint32_t i = frontier_of(off, nf, p);
  const uint32_t nb = col[rp[l2g[fb + i]] + (p - off[i])];
  flag[p] = (local_of[nb] == kNone && first[nb] == p) ? 1u : 0u;
}

__global__ void assign_kernel(const uint64_t* __restrict__ rp, const uint32_t* __restrict__ col,
                              uint32_t* __restrict__ l2g, uint32_t fb, uint32_t nf, const uint64_t* __restrict__ off,
                              uint64_t total, const uint32_t* __restrict__ flag, const uint32_t* __restrict__ pos,
                              uint32_t fe, uint32_t* __restrict__ local_of) {
  const uint64_t p = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x;
  if (p >= total || !flag[p]) return;
  const uint32_t i = frontier_of(off, nf, p);
  const uint32_t nb = col[rp[l2g[fb + i]] + (p - off[i])];
  const uint32_t id = fe + pos[p];
  l2g[id] = nb;
  local_of[nb] = id;
}

// warp per local node: number of its neighbours inside the ball
__global__ void ball_deg_kernel(const uint64_t* __restrict__ rp, const uint32_t* __restrict__ col,
                                const uint32_t* __restrict__ l2g, uint32_t V, const uint32_t* __restrict__ local_of,
                                uint64_t* __restrict__ cnt) {
  const uint32_t lu = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (lu >= V) return;
  const uint32_t g = l2g[lu];
  uint32_t c = 0;
  for (uint64_t k = rp[g] + lane; k < rp[g + 1]; k += 32) c += local_of[col[k]] != kNone;
  for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
  if (lane == 0) cnt[lu] = c;
}

__global__ void ball_fill_kernel(const uint64_t* __restrict__ rp, const uint32_t* __restrict__ col,
                                 const uint32_t* __restrict__ l2g, uint32_t V, const uint32_t* __restrict__ local_of,
                                 const uint64_t* __restrict__ lrp, uint32_t* __restrict__ lcol) {
  const uint32_t lu = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (lu >= V) return;
  const uint32_t g = l2g[lu];
  uint64_t base = lrp[lu];
  for (uint64_t k0 = rp[g]; k0 < rp[g + 1]; k0 += 32) {
    const uint64_t k = k0 + lane;
    const uint32_t lv = k < rp[g + 1] ? local_of[col[k]] : kNone;
    const unsigned keep = __ballot_sync(0xffffffffu, lv != kNone);
    if (lv != kNone) lcol[base + __popc(keep & ((1u << lane) - 1u))] = lv;
    base += __popc(keep);
  }
}

// first upper entry (lv > lu) of each sorted row and the upper counts
__global__ void upper_kernel(const uint64_t* __restrict__ lrp, const uint32_t* __restrict__ lcol, uint32_t V,
                             uint64_t* __restrict__ ufirst, uint64_t* __restrict__ ucnt) {
  const uint32_t lu = blockIdx.x * blockDim.x + threadIdx.x;
  if (lu >= V) return;
  uint64_t lo = lrp[lu], hi = lrp[lu + 1];
  while (lo < hi) {  // first entry > lu
    const uint64_t mid = (lo + hi) >> 1;
    if (lcol[mid] <= lu) lo = mid + 1; else hi = mid;
  }
  ufirst[lu] = lo;
  ucnt[lu] = lrp[lu + 1] - lo;
}

// edge_player per entry and the players list (u, v) in lexicographic order
__global__ void player_kernel(const uint64_t* __restrict__ lrp, const uint32_t* __restrict__ lcol, uint32_t V,
                              const uint64_t* __restrict__ ufirst, const uint64_t* __restrict__ pstart,
                              uint32_t* __restrict__ ep, uint32_t* __restrict__ players) {
  const uint32_t lu = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (lu >= V) return;
  const uint64_t b = lrp[lu], e = lrp[lu + 1], uf = ufirst[lu];
  for (uint64_t k = b + lane; k < e; k += 32) {
    const uint32_t lv = lcol[k];
    uint64_t id;
    if (k >= uf) {
      id = pstart[lu] + (k - uf);
      players[2 * id] = lu;
      players[2 * id + 1] = lv;
    } else {  // (lv, lu): position of lu in row lv's upper part
      uint64_t lo = ufirst[lv], hi = lrp[lv + 1];
      while (lo < hi) {
        const uint64_t mid = (lo + hi) >> 1;
        if (lcol[mid] < lu) lo = mid + 1; else hi = mid;
      }
      id = pstart[lv] + (lo - ufirst[lv]);
    }
    ep[k] = uint32_t(id);
  }
}

__global__ void reset_kernel(const uint32_t* __restrict__ l2g, uint32_t V, uint32_t* __restrict__ local_of,
                             unsigned long long* __restrict__ first) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= V) return;
  const uint32_t g = l2g[i];
  local_of[g] = kNone;
  first[g] = ~0ull;
}

__global__ void init_kernel(uint32_t* __restrict__ local_of, unsigned long long* __restrict__ first, uint32_t n) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  local_of[i] = kNone;
  first[i] = ~0ull;
}

template <typename T>
void exclusive_scan(Ctx& ctx, const T* in, T* out, uint64_t n, DevBuf<unsigned char>& tmp) {
  size_t bytes = 0;
  SF_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, bytes, in, out, n, ctx.stream));
  tmp.reserve(bytes + 16);
  SF_CUDA(cub::DeviceScan::ExclusiveSum(tmp.p, bytes, in, out, n, ctx.stream));
}

}  // namespace

Subgraph extract_device(Ctx& ctx, const Graph& g, uint32_t target, int hops) {
  if (target >= g.num_nodes) throw DataError("target node " + std::to_string(target) + " out of range");
  if (hops < 0) throw DataError("hop count must be nonnegative");
  cudaStream_t st = ctx.stream;
  ExtractState& x = ctx.extract;
  DebugTimer dt("extract (device)");
  if (x.graph_id != g.id) {  // graph CSR and per-node state, once per graph
    x.rp.upload(g.row_ptr.data(), g.row_ptr.size(), st);
    x.col.upload(g.col.data(), std::max<size_t>(g.col.size(), 1), st);
    x.local_of.reserve(std::max<uint32_t>(g.num_nodes, 1));
    x.first.reserve(std::max<uint32_t>(g.num_nodes, 1));
    if (g.num_nodes) {
      init_kernel<<<nblk(g.num_nodes), 256, 0, st>>>(x.local_of.p, reinterpret_cast<unsigned long long*>(x.first.p),
                                                     g.num_nodes);
      SF_LAUNCHED(ctx);
    }
    ctx.h2d_bytes += g.row_ptr.size() * 8 + g.col.size() * 4;
    x.graph_id = g.id;
  }
  auto* first = reinterpret_cast<unsigned long long*>(x.first.p);
  x.l2g.reserve(std::max<uint32_t>(g.num_nodes, 1));
  const uint32_t t32 = target, zero = 0;
  SF_CUDA(cudaMemcpyAsync(x.l2g.p, &t32, 4, cudaMemcpyHostToDevice, st));
  SF_CUDA(cudaMemcpyAsync(x.local_of.p + target, &zero, 4, cudaMemcpyHostToDevice, st));
  uint32_t fb = 0, fe = 1;
  for (int hop = 0; hop < hops && fb < fe; ++hop) {
    const uint32_t nf = fe - fb;
    x.off.reserve(nf + 1);
    x.deg.reserve(nf + 1);
    frontier_deg_kernel<<<nblk(nf), 256, 0, st>>>(x.rp.p, x.l2g.p, fb, fe, x.deg.p);
    SF_LAUNCHED(ctx);
    SF_CUDA(cudaMemsetAsync(x.deg.p + nf, 0, 8, st));
    exclusive_scan(ctx, x.deg.p, x.off.p, nf + 1, x.tmp);
    uint64_t total = 0;
    SF_CUDA(cudaMemcpyAsync(&total, x.off.p + nf, 8, cudaMemcpyDeviceToHost, st));
    SF_CUDA(cudaStreamSynchronize(st));
    if (total == 0) break;
    x.flag.reserve(total + 1);
    x.pos.reserve(total + 1);
    candidate_kernel<<<nblk(total), 256, 0, st>>>(x.rp.p, x.col.p, x.l2g.p, fb, nf, x.off.p, total, x.local_of.p,
                                                  first);
    SF_LAUNCHED(ctx);
    winner_kernel<<<nblk(total), 256, 0, st>>>(x.rp.p, x.col.p, x.l2g.p, fb, nf, x.off.p, total, x.local_of.p, first,
                                               x.flag.p);
    SF_LAUNCHED(ctx);
    SF_CUDA(cudaMemsetAsync(x.flag.p + total, 0, 4, st));
    exclusive_scan(ctx, x.flag.p, x.pos.p, total + 1, x.tmp);
    uint32_t added = 0;
    SF_CUDA(cudaMemcpyAsync(&added, x.pos.p + total, 4, cudaMemcpyDeviceToHost, st));
    assign_kernel<<<nblk(total), 256, 0, st>>>(x.rp.p, x.col.p, x.l2g.p, fb, nf, x.off.p, total, x.flag.p, x.pos.p,
                                               fe, x.local_of.p);
    SF_LAUNCHED(ctx);
    SF_CUDA(cudaStreamSynchronize(st));
    fb = fe;
    fe += added;
  }
  const uint32_t V = fe;
  dt.lap("bfs");
  // local CSR: ball neighbours per row, then each row sorted by local id
  x.lrp.reserve(uint64_t(V) + 1);
  x.cnt.reserve(uint64_t(V) + 1);
  ball_deg_kernel<<<nblk(uint64_t(V) * 32), 256, 0, st>>>(x.rp.p, x.col.p, x.l2g.p, V, x.local_of.p, x.cnt.p);
  SF_LAUNCHED(ctx);
  SF_CUDA(cudaMemsetAsync(x.cnt.p + V, 0, 8, st));
  exclusive_scan(ctx, x.cnt.p, x.lrp.p, uint64_t(V) + 1, x.tmp);
  uint64_t nnz = 0;
  SF_CUDA(cudaMemcpyAsync(&nnz, x.lrp.p + V, 8, cudaMemcpyDeviceToHost, st));
  SF_CUDA(cudaStreamSynchronize(st));
  x.lcol_raw.reserve(std::max<uint64_t>(nnz, 1));
  x.lcol.reserve(std::max<uint64_t>(nnz, 1));
  ball_fill_kernel<<<nblk(uint64_t(V) * 32), 256, 0, st>>>(x.rp.p, x.col.p, x.l2g.p, V, x.local_of.p, x.lrp.p,
                                                          x.lcol_raw.p);
  SF_LAUNCHED(ctx);
  if (nnz) {
    size_t bytes = 0;
    int bits = 1;
    while (bits < 32 && (uint64_t(1) << bits) < V) ++bits;
    SF_CUDA(cub::DeviceSegmentedRadixSort::SortKeys(nullptr, bytes, x.lcol_raw.p, x.lcol.p, int64_t(nnz), int64_t(V),
                                                    x.lrp.p, x.lrp.p + 1, 0, bits, st));
    x.tmp.reserve(bytes + 16);
    SF_CUDA(cub::DeviceSegmentedRadixSort::SortKeys(x.tmp.p, bytes, x.lcol_raw.p, x.lcol.p, int64_t(nnz), int64_t(V),
                                                    x.lrp.p, x.lrp.p + 1, 0, bits, st));
  }
  // players and edge_player
  x.ufirst.reserve(uint64_t(V) + 1);
  x.pstart.reserve(uint64_t(V) + 1);
  upper_kernel<<<nblk(V), 256, 0, st>>>(x.lrp.p, x.lcol.p, V, x.ufirst.p, x.cnt.p);
  SF_LAUNCHED(ctx);
  SF_CUDA(cudaMemsetAsync(x.cnt.p + V, 0, 8, st));
  exclusive_scan(ctx, x.cnt.p, x.pstart.p, uint64_t(V) + 1, x.tmp);
  const uint64_t n = nnz / 2;
  x.ep.reserve(std::max<uint64_t>(nnz, 1));
  x.players.reserve(std::max<uint64_t>(2 * n, 1));
  player_kernel<<<nblk(uint64_t(V) * 32), 256, 0, st>>>(x.lrp.p, x.lcol.p, V, x.ufirst.p, x.pstart.p, x.ep.p,
                                                       x.players.p);
  SF_LAUNCHED(ctx);
  Subgraph sg;
  sg.target_global = target;
  sg.feature_dim = g.feature_dim;
  sg.local_to_global.resize(V);
  sg.row_ptr.resize(uint64_t(V) + 1);
  sg.col.resize(nnz);
  sg.edge_player.resize(nnz);
  sg.players.resize(n);
  static_assert(sizeof(std::pair<uint32_t, uint32_t>) == 8, "pair layout");
  SF_CUDA(cudaMemcpyAsync(sg.local_to_global.data(), x.l2g.p, uint64_t(V) * 4, cudaMemcpyDeviceToHost, st));
  SF_CUDA(cudaMemcpyAsync(sg.row_ptr.data(), x.lrp.p, (uint64_t(V) + 1) * 8, cudaMemcpyDeviceToHost, st));
  if (nnz) {
    SF_CUDA(cudaMemcpyAsync(sg.col.data(), x.lcol.p, nnz * 4, cudaMemcpyDeviceToHost, st));
    SF_CUDA(cudaMemcpyAsync(sg.edge_player.data(), x.ep.p, nnz * 4, cudaMemcpyDeviceToHost, st));
    SF_CUDA(cudaMemcpyAsync(sg.players.data(), x.players.p, n * 8, cudaMemcpyDeviceToHost, st));
  }
  ctx.d2h_bytes += uint64_t(V) * 12 + 8 + nnz * 8 + n * 8;
  // leave the per-node state clean for the next target
  reset_kernel<<<nblk(V), 256, 0, st>>>(x.l2g.p, V, x.local_of.p, first);
  SF_LAUNCHED(ctx);
  SF_CUDA(cudaStreamSynchronize(st));
  dt.lap("csr + players");
  sg.source = &g;
  return sg;
}

}  // namespace sfb
