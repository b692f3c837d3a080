// Coalition sampler for sm_100a: counter-based Philox-4x32-10 + Floyd's
// subset sampler, one warp per complement pair, bit-exact with the
// reference generate_masks (sampler.cpp:153-210).
//
// Layout: rows are u64 words, bit e = player e, row-major,
// words_for_bits(n) words per row; local pair j owns rows 2j (kept-set,
// size s <= n/2) and 2j+1 (complement, tail bits cleared). Pair j of rank r
// is global pair g = r + j * world (sampler.cpp:177-178), so its Philox
// stream is (seed, g) and the layout of any world reproduces the
// single-worker rows at the same global index.
#include <cuda_runtime.h>

#include <cstdlib>

#include <cstring>

#include "sf_device.cuh"
#include "sf_internal.hpp"

namespace sfb {

namespace {

constexpr int kSamplerWarps = 4;  // warps per CTA

struct ClassTable {
  const uint32_t* size;
  const uint64_t* first;
  const uint64_t* pairs;
  uint32_t count;
};

__device__ __forceinline__ uint32_t find_class(const ClassTable& ct,
                                               uint64_t g) {
  // classes are contiguous and ascending in g (sampler.cpp:144-149)
  uint32_t lo = 0, hi = ct.count;  // first[lo] <= g < first[hi]
  while (hi - lo > 1) {
    const uint32_t mid = (lo + hi) >> 1;
    if (ct.first[mid] <= g)
      lo = mid;
    else
      hi = mid;
  }
  return lo;
}

// Bitset accessors for the two storage variants: shared memory (one row per
// warp, fast path) or the output row itself in global memory (large n).
// (shared memory has native 32-bit atomics only; 64-bit ones are CAS loops.
// Bit t of u64 word t/64 is bit t%32 of u32 word t/32 on little-endian.)
struct SmemSet {
  uint64_t* w;
  __device__ uint32_t* w32() const { return reinterpret_cast<uint32_t*>(w); }
  __device__ bool test(uint32_t t) const { return (w32()[t >> 5] >> (t & 31)) & 1u; }
  __device__ bool test_and_set(uint32_t t) const {
    const uint32_t b = 1u << (t & 31);
    return atomicOr(&w32()[t >> 5], b) & b;
  }
  __device__ void set(uint32_t t) const { test_and_set(t); }
  __device__ void clear(uint32_t t) const { atomicAnd(&w32()[t >> 5], ~(1u << (t & 31))); }
};
struct GmemSet {
  uint64_t* w;
  __device__ bool test(uint32_t t) const { return (__ldcg(&w[t >> 6]) >> (t & 63)) & 1ull; }
  __device__ bool test_and_set(uint32_t t) const {
    const unsigned long long b = 1ull << (t & 63);
    return atomicOr(reinterpret_cast<unsigned long long*>(&w[t >> 6]), b) & b;
  }
  __device__ void set(uint32_t t) const { test_and_set(t); }
  __device__ void clear(uint32_t t) const {
    atomicAnd(reinterpret_cast<unsigned long long*>(&w[t >> 6]), ~(1ull << (t & 63)));
  }
};

// Floyd (sampler.cpp:55-63): for m = n-s .. n-1 draw t = u64 % (m+1) and
// insert t, or m when t is already present. The warp draws 64 consecutive
// values at once (lane i owns Philox block base/2 + i, i.e. draws base+2i
// and base+2i+1), tests them against the set as it stood before the chunk,
// inserts the provisional picks (t, or m when t was already present). The
// sequential loop picks something else only when a draw hits an earlier
// pick of the same chunk, and then two provisional picks coincide (a
// provisional pick is never in the pre-chunk set: t only when absent, m
// above every earlier pick). So a clash seen by the atomic inserts is
// exactly the case that needs the in-order replay: the chunk's inserts are
// undone and the chunk is replayed with shuffles.
template <typename Set>
__device__ void floyd_warp(const Set& set, uint32_t n, uint32_t s,
                           uint64_t seed, uint64_t g, int lane) {
  const uint32_t m0 = n - s;
  for (uint32_t base = 0; base < s; base += 64) {
    uint64_t x0, x1;
    philox_block(seed, g, (base >> 1) + lane, x0, x1);
    const uint32_t i0 = base + 2 * lane, i1 = i0 + 1;
    const bool v0 = i0 < s, v1 = i1 < s;
    const uint32_t mm0 = m0 + i0, mm1 = m0 + i1;
    const uint32_t t0 = v0 ? mod_u64_u32(x0, mm0 + 1) : 0xffffffffu;
    const uint32_t t1 = v1 ? mod_u64_u32(x1, mm1 + 1) : 0xffffffffu;
    // (the set is ordered for this chunk by the previous chunk's trailing
    // __syncwarp, or by the caller's before the first chunk)
    bool hit0 = v0 && set.test(t0);
    bool hit1 = v1 && set.test(t1);
    __syncwarp();
    bool clash = false;
    if (v0) clash |= set.test_and_set(hit0 ? mm0 : t0);
    if (v1) clash |= set.test_and_set(hit1 ? mm1 : t1);
    if (__any_sync(kFull, clash)) {
      __syncwarp();
      if (v0) set.clear(hit0 ? mm0 : t0);
      if (v1) set.clear(hit1 ? mm1 : t1);
      __syncwarp();
      const uint32_t chunk = min(64u, s - base);
      for (uint32_t k = 0; k < chunk; ++k) {
        const int owner = k >> 1;
        uint32_t pk = (k & 1) ? (hit1 ? mm1 : t1) : (hit0 ? mm0 : t0);
        pk = __shfl_sync(kFull, pk, owner);
        // later draws of this chunk that drew the value just picked
        if (i0 > base + k && t0 == pk) hit0 = true;
        if (i1 > base + k && t1 == pk) hit1 = true;
      }
      if (v0) set.set(hit0 ? mm0 : t0);
      if (v1) set.set(hit1 ? mm1 : t1);
    }
    __syncwarp();
  }
}

// Exhaustive plans (sampler.cpp:38-51, 106-114, 192-199): lexicographic
// unranking, n <= 62 so a row is one word.
__device__ uint64_t binom_dev(uint32_t n, uint32_t s) {
  if (s > n) return 0;
  if (n - s < s) s = n - s;
  unsigned __int128 r = 1;
  for (uint32_t i = 1; i <= s; ++i) {
    r = r * (n - s + i) / i;
    if (r > (unsigned __int128)0xffffffffffffffffull) return 0xffffffffffffffffull;
  }
  return static_cast<uint64_t>(r);
}

__device__ uint64_t unrank(uint64_t idx, uint32_t m, uint32_t t,
                           uint32_t offset) {
  uint64_t row = 0;
  uint32_t x = 0;
  for (uint32_t i = 0; i < t; ++i) {
    for (;;) {
      const uint64_t c = binom_dev(m - 1 - x, t - 1 - i);
      if (idx < c) break;
      idx -= c;
      ++x;
    }
    row |= 1ull << (x + offset);
    ++x;
  }
  return row;
}

__global__ void exhaustive_kernel(ClassTable ct, uint32_t n, int rank,
                                  int world, uint64_t local_pairs,
                                  uint64_t* rows, int kept_only) {
  const uint64_t j = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x;
  if (j >= local_pairs) return;
  const uint64_t g = rank + j * uint64_t(world);
  const uint32_t ci = find_class(ct, g);
  const uint32_t s = ct.size[ci];
  const uint64_t idx = g - ct.first[ci];
  uint64_t sub;
  if (2 * s == n)
    sub = 1ull | unrank(idx, n - 1, s - 1, 1);
  else
    sub = unrank(idx, n, s, 0);
  const uint64_t tail = (n % 64) ? ((1ull << (n % 64)) - 1) : ~0ull;
  if (kept_only) {
    rows[j] = sub;
    return;
  }
  rows[2 * j] = sub;
  rows[2 * j + 1] = ~sub & tail;
}

template <bool kSmem>
__global__ void __launch_bounds__(kSamplerWarps * 32)
    floyd_kernel(ClassTable ct, uint32_t n, uint32_t W, uint64_t seed,
                 int rank, int world, uint64_t local_pairs, uint64_t* rows, int kept_only) {
  extern __shared__ uint64_t smem_sets[];
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  const uint64_t tail = (n % 64) ? ((1ull << (n % 64)) - 1) : ~0ull;
  const uint64_t warps_total = uint64_t(gridDim.x) * kSamplerWarps;
  for (uint64_t j = blockIdx.x * uint64_t(kSamplerWarps) + warp; j < local_pairs;
       j += warps_total) {
    const uint64_t g = rank + j * uint64_t(world);
    const uint32_t ci = find_class(ct, g);
    const uint32_t s = ct.size[ci];
    // kept-only layout: row j = the kept-set of local pair j (the odd row is
    // its complement, derived by the consumers); full layout: rows 2j, 2j+1
    uint64_t* even = rows + (kept_only ? j : 2 * j) * W;
    uint64_t* odd = even + W;
    uint64_t* bits = kSmem ? smem_sets + size_t(warp) * W : even;
    for (uint32_t w = lane; w < W; w += 32) bits[w] = 0;
    __syncwarp();
    if (kSmem)
      floyd_warp(SmemSet{bits}, n, s, seed, g, lane);
    else
      floyd_warp(GmemSet{bits}, n, s, seed, g, lane);
    __syncwarp();
    for (uint32_t w = lane; w < W; w += 32) {
      const uint64_t v = kSmem ? bits[w] : __ldcg(&bits[w]);
      if (kSmem) even[w] = v;
      if (!kept_only) odd[w] = (w == W - 1) ? (~v & tail) : ~v;
    }
    __syncwarp();
  }
}

template <bool kSmem>
__global__ void __launch_bounds__(kSamplerWarps * 32)
    floyd_jobs_kernel(uint32_t n, uint32_t W, uint64_t seed,
                      const uint64_t* __restrict__ streams,
                      const uint32_t* __restrict__ sizes,
                      const uint8_t* __restrict__ invert, uint64_t jobs,
                      uint64_t* __restrict__ rows) {
  extern __shared__ uint64_t smem_sets[];
  const int lane = threadIdx.x & 31;
  const uint64_t j = blockIdx.x * uint64_t(kSamplerWarps) + (threadIdx.x >> 5);
  if (j >= jobs) return;
  const uint64_t tail = n == 0 ? 0ull : (n % 64) ? ((1ull << (n % 64)) - 1) : ~0ull;
  uint64_t* row = rows + j * W;
  uint64_t* bits = kSmem ? smem_sets + size_t(threadIdx.x >> 5) * W : row;
  for (uint32_t w = lane; w < W; w += 32) bits[w] = 0;
  __syncwarp();
  if (kSmem)
    floyd_warp(SmemSet{bits}, n, sizes[j], seed, streams[j], lane);
  else
    floyd_warp(GmemSet{bits}, n, sizes[j], seed, streams[j], lane);
  __syncwarp();
  const bool inv = invert[j] != 0;
  for (uint32_t w = lane; w < W; w += 32) {
    uint64_t v = kSmem ? bits[w] : __ldcg(&bits[w]);
    if (inv) v = (w == W - 1) ? (~v & tail) : ~v;
    row[w] = v;
  }
}

__global__ void philox_stream_kernel(uint64_t seed, uint64_t stream,
                                     uint64_t count, uint64_t* out) {
  const uint64_t b = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x;
  if (2 * b >= count) return;
  uint64_t f, s;
  philox_block(seed, stream, b, f, s);
  out[2 * b] = f;
  if (2 * b + 1 < count) out[2 * b + 1] = s;
}

// Rows -> tile layout: out[t][e] bit i = bit e of row t*64+i (rows past
// `rows` read as zero). One CTA per (tile, kTWords-word chunk) stages the
// 64 x kTWords words coalesced in shared memory; each warp then transposes
// kTWords/8 words, each a 64 x 64 bit block, as four 32 x 32 butterfly transposes
// (5 shuffle stages each) and writes 256 contiguous bytes per output half.
// (bfly_step: sf_device.cuh)

constexpr int kTWords = 32;  // words per CTA (a multiple of 8: one or more per warp)

__global__ void __launch_bounds__(256)
    transpose_tiles_kernel(const uint64_t* __restrict__ in, uint64_t rows,
                           uint32_t W, uint64_t stride, uint64_t* __restrict__ out) {
  __shared__ uint64_t sm[64][kTWords + 1];
  const uint64_t t = blockIdx.y;
  const uint32_t w0 = blockIdx.x * kTWords;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (int i = tid; i < 64 * kTWords; i += 256) {
    const int r = i / kTWords, w = i % kTWords;
    const uint64_t row = t * 64 + r;
    sm[r][w] = (row < rows && w0 + w < W) ? in[row * stride + w0 + w] : 0ull;
  }
  __syncthreads();
  const uint64_t Wp = uint64_t(W) * 64;  // players per tile, padded
#pragma unroll 1
  for (int w = warp * (kTWords / 8); w < (warp + 1) * (kTWords / 8); ++w) {
    if (w0 + w >= W) break;
    const uint64_t r0 = sm[lane][w], r1 = sm[lane + 32][w];
    uint32_t a = uint32_t(r0), b = uint32_t(r0 >> 32), c = uint32_t(r1), d = uint32_t(r1 >> 32);
#pragma unroll
    for (int s = 16; s >= 1; s >>= 1) {
      const uint32_t m = s == 16 ? 0x0000FFFFu : s == 8 ? 0x00FF00FFu : s == 4 ? 0x0F0F0F0Fu
                       : s == 2 ? 0x33333333u : 0x55555555u;
      const uint32_t keep = (lane & s) ? ~m : m, amt = (lane & s) ? 32 - s : s;
      a = bfly_step(a, s, keep, amt);
      b = bfly_step(b, s, keep, amt);
      c = bfly_step(c, s, keep, amt);
      d = bfly_step(d, s, keep, amt);
    }
    uint64_t* o = out + t * Wp + uint64_t(w0 + w) * 64;
    o[lane] = (uint64_t(c) << 32) | a;
    o[lane + 32] = (uint64_t(d) << 32) | b;
  }
}

// Kept-only rows -> tile layout: tile t covers local pairs 32t..32t+31;
// out[t][e] bit 2i = bit e of pair (32t+i)'s kept-set row, bit 2i+1 = its
// complement (players e < n only; rows past `pairs` are zero). One CTA per
// (tile, kTWords-word chunk): 32 rows x kTWords words staged in shared
// memory; per word two 32 x 32 butterfly transposes give, for each player,
// the 32 pair bits, which are spread to the even bit positions and their
// complement to the odd ones.
__device__ __forceinline__ uint64_t spread_even(uint32_t x) {
  uint64_t v = x;
  v = (v | (v << 16)) & 0x0000FFFF0000FFFFull;
  v = (v | (v << 8)) & 0x00FF00FF00FF00FFull;
  v = (v | (v << 4)) & 0x0F0F0F0F0F0F0F0Full;
  v = (v | (v << 2)) & 0x3333333333333333ull;
  v = (v | (v << 1)) & 0x5555555555555555ull;
  return v;
}

__global__ void __launch_bounds__(256)
    transpose_pairs_kernel(const uint64_t* __restrict__ in, uint64_t pairs, uint32_t W, uint32_t n,
                           uint64_t* __restrict__ out) {
  __shared__ uint64_t sm[32][kTWords + 1];
  const uint64_t t = blockIdx.y;
  const uint32_t w0 = blockIdx.x * kTWords;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (int i = tid; i < 32 * kTWords; i += 256) {
    const int r = i / kTWords, w = i % kTWords;
    const uint64_t j = t * 32 + r;
    sm[r][w] = (j < pairs && w0 + w < W) ? in[j * W + w0 + w] : 0ull;
  }
  __syncthreads();
  const uint64_t Wp = uint64_t(W) * 64;
  const uint64_t left = pairs > t * 32 ? pairs - t * 32 : 0;
  const uint32_t npairs = left > 32 ? 32u : uint32_t(left);
  const uint32_t valid = npairs == 32 ? 0xFFFFFFFFu : ((1u << npairs) - 1u);
#pragma unroll 1
  for (int w = warp * (kTWords / 8); w < (warp + 1) * (kTWords / 8); ++w) {
    if (w0 + w >= W) break;
    const uint64_t r0 = sm[lane][w];
    uint32_t a = uint32_t(r0), b = uint32_t(r0 >> 32);
#pragma unroll
    for (int s = 16; s >= 1; s >>= 1) {
      const uint32_t m = s == 16 ? 0x0000FFFFu : s == 8 ? 0x00FF00FFu : s == 4 ? 0x0F0F0F0Fu
                       : s == 2 ? 0x33333333u : 0x55555555u;
      const uint32_t keep = (lane & s) ? ~m : m, amt = (lane & s) ? 32 - s : s;
      a = bfly_step(a, s, keep, amt);
      b = bfly_step(b, s, keep, amt);
    }
    const uint32_t ea = (w0 + w) * 64 + lane, eb = ea + 32;
    const uint32_t ca = ea < n ? (~a & valid) : 0u, cb = eb < n ? (~b & valid) : 0u;
    uint64_t* o = out + t * Wp + uint64_t(w0 + w) * 64;
    o[lane] = spread_even(a) | (spread_even(ca) << 1);
    o[lane + 32] = spread_even(b) | (spread_even(cb) << 1);
  }
}

}  // namespace

void launch_philox_stream(Ctx& ctx, uint64_t seed, uint64_t stream,
                          uint64_t count, uint64_t* dev_out) {
  if (count == 0) return;
  const uint64_t blocks = (count + 1) / 2;
  philox_stream_kernel<<<unsigned((blocks + 255) / 256), 256, 0, ctx.stream>>>(
      seed, stream, count, dev_out);
  SF_LAUNCHED(ctx);
}

void launch_generate_masks(Ctx& ctx, const SizePlan& plan, uint64_t seed,
                           int rank, int world, uint64_t* dev_rows, bool kept_only) {
  const uint64_t pairs = local_pair_count(plan.total_pairs(), rank, world);
  if (pairs == 0) return;
  const uint32_t n = plan.n;
  const uint32_t W = (n + 63) / 64;
  const size_t C = plan.classes.size();
  std::vector<uint32_t> sizes(C);
  std::vector<uint64_t> first(C), cnt(C);
  for (size_t i = 0; i < C; ++i) {
    sizes[i] = plan.classes[i].size;
    first[i] = plan.classes[i].first_pair;
    cnt[i] = plan.classes[i].pairs;
  }
  // class table: context-owned device buffers, filled from pinned staging
  // (no per-call allocation, no host synchronization)
  if (ctx.plan_ready) SF_CUDA(cudaEventSynchronize(ctx.plan_ready));  // staging free again
  else SF_CUDA(cudaEventCreateWithFlags(&ctx.plan_ready, cudaEventDisableTiming));
  ctx.plan_host.reserve(2 * C + 1);
  uint64_t* h = ctx.plan_host.p;
  for (size_t i = 0; i < C; ++i) {
    h[i] = first[i];
    h[C + i] = cnt[i];
  }
  ctx.plan_dev64.reserve(2 * C + 1);
  ctx.plan_dev32.reserve(C + 1);
  SF_CUDA(cudaMemcpyAsync(ctx.plan_dev64.p, h, 2 * C * 8, cudaMemcpyHostToDevice, ctx.stream));
  ctx.plan_host32.reserve(C + 1);
  std::memcpy(ctx.plan_host32.p, sizes.data(), C * 4);
  SF_CUDA(cudaMemcpyAsync(ctx.plan_dev32.p, ctx.plan_host32.p, C * 4, cudaMemcpyHostToDevice, ctx.stream));
  ctx.h2d_bytes += C * 20;
  ClassTable ct{ctx.plan_dev32.p, ctx.plan_dev64.p, ctx.plan_dev64.p + C, static_cast<uint32_t>(C)};
  if (plan.exhaustive) {
    exhaustive_kernel<<<unsigned((pairs + 127) / 128), 128, 0, ctx.stream>>>(
        ct, n, rank, world, pairs, dev_rows, kept_only ? 1 : 0);
    SF_LAUNCHED(ctx);
  } else {
    int sms = 148;
    SF_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, ctx.device));
    const size_t smem = size_t(kSamplerWarps) * W * 8;
    const uint64_t want = (pairs + kSamplerWarps - 1) / kSamplerWarps;
    if (smem <= 200 * 1024) {
      auto k = floyd_kernel<true>;
      // a fixed ceiling, set once per device: launches on several streams
      // (explain_nodes workers) must not race on a per-call value
      set_max_dynamic_smem(k, 200 * 1024);
      int per_sm = 1;
      SF_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k, kSamplerWarps * 32, smem));
      const uint64_t grid = std::min<uint64_t>(want, uint64_t(sms) * std::max(per_sm, 1) * 4);
      k<<<unsigned(grid), kSamplerWarps * 32, smem, ctx.stream>>>(
          ct, n, W, seed, rank, world, pairs, dev_rows, kept_only ? 1 : 0);
    } else {
      // rows whose set does not fit in shared memory build it in place in
      // the output row (L2 atomics). SF_FLOYD_GBLOCKS CTAs per SM (default
      // 4: 592 rows in flight keep more of the sets in L2; C4 sampling
      // 453 -> 369 ms vs 16 per SM, 407 at 2, 552 at 1)
      static const uint64_t gblocks = std::getenv("SF_FLOYD_GBLOCKS")
                                          ? std::max<uint64_t>(1, std::strtoull(std::getenv("SF_FLOYD_GBLOCKS"), nullptr, 10))
                                          : 4;
      const uint64_t grid = std::min<uint64_t>(want, uint64_t(sms) * gblocks);
      floyd_kernel<false><<<unsigned(grid), kSamplerWarps * 32, 0, ctx.stream>>>(
          ct, n, W, seed, rank, world, pairs, dev_rows, kept_only ? 1 : 0);
    }
    SF_LAUNCHED(ctx);
  }
  // the pinned staging copies are reused by the next call: order it after
  // this launch's uploads
  SF_CUDA(cudaEventRecord(ctx.plan_ready, ctx.stream));
}

void launch_floyd_jobs(Ctx& ctx, uint32_t n, uint64_t seed,
                       const uint64_t* dev_streams, const uint32_t* dev_sizes,
                       const uint8_t* dev_invert, uint64_t jobs,
                       uint64_t* dev_rows) {
  if (jobs == 0) return;
  // same row stride as the caller's mask layout (one word even when n == 0)
  const uint32_t W = std::max<uint32_t>((n + 63) / 64, 1);
  const unsigned grid = unsigned((jobs + kSamplerWarps - 1) / kSamplerWarps);
  const size_t smem = size_t(kSamplerWarps) * W * 8;
  if (smem <= 200 * 1024) {  // the set in shared memory (one row per warp)
    auto k = floyd_jobs_kernel<true>;
    set_max_dynamic_smem(k, 200 * 1024);
    k<<<grid, kSamplerWarps * 32, smem, ctx.stream>>>(n, W, seed, dev_streams, dev_sizes, dev_invert, jobs,
                                                      dev_rows);
  } else {
    floyd_jobs_kernel<false><<<grid, kSamplerWarps * 32, 0, ctx.stream>>>(n, W, seed, dev_streams, dev_sizes,
                                                                          dev_invert, jobs, dev_rows);
  }
  SF_LAUNCHED(ctx);
}

void launch_transpose_pairs(Ctx& ctx, const uint64_t* dev_kept, uint64_t pairs, uint32_t W, uint32_t n,
                            uint64_t tiles, uint64_t* dev_maskt) {
  if (tiles == 0) return;
  dim3 grid((W + kTWords - 1) / kTWords, unsigned(tiles));
  transpose_pairs_kernel<<<grid, 256, 0, ctx.stream>>>(dev_kept, pairs, W, n, dev_maskt);
  SF_LAUNCHED(ctx);
}

void launch_transpose_tiles(Ctx& ctx, const uint64_t* dev_rows, uint64_t rows,
                            uint32_t W, uint64_t tiles, uint64_t* dev_maskt, uint64_t stride) {
  if (tiles == 0) return;
  dim3 grid((W + kTWords - 1) / kTWords, unsigned(tiles));
  transpose_tiles_kernel<<<grid, 256, 0, ctx.stream>>>(dev_rows, rows, W, stride ? stride : W, dev_maskt);
  SF_LAUNCHED(ctx);
}

}  // namespace sfb
