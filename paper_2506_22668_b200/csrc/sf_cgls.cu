// Weighted least squares on the bit-packed coalition matrix, sm_100a.
// Replaces assemble_problem + solve_cgls (solver.cpp:95-362) and the Gram
// build of solve_direct (solver.cpp:364-428).
//
// The system is sqrt(W) M phi ~ sqrt(W) t plus one pinned all-ones row of
// weight constraint_weight and target constraint_target. M stays bit-packed
// in HBM in two layouts:
//   rows   row-major u64 words (the sampler's output) -> M u  (forward)
//   mte    tiles of 64 pairs over the even rows (odd rows of non-complement
//          pairs in a second layout), u64 per player, bit i = pair t*64+i -> M^T r
// Complement pairs (row 2j+1 = ~row 2j) take the reference's shortcut
// (solver.cpp:188-198, 209-223, 261-263): the odd dot is sum(u) - dot and
// the odd row contributes a constant plus a difference on the even row, so
// only kept-set bits are visited. All n-vectors and row vectors are FP64.
// Reductions use fixed-shape trees, so a run is bitwise reproducible for a
// given layout (the reference's cross-world bitwise property comes from its
// PairwiseFolder; here the parity bar is 1e-3 relative L2).
#include <cuda_runtime.h>

#include <type_traits>

#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>

#include <algorithm>
#include <cmath>
#include <cstdlib>

#include "sf_device.cuh"
#include "sf_internal.hpp"

namespace sfb {

namespace {

constexpr int kRedBlocks = 256;
constexpr int kRedThreads = 256;

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(kFull, v, o);
  return v;
}

// ---------------------------------------------------------------- reductions
// Fixed-shape two-stage sum: kRedBlocks grid-strided partials, then one
// block folds them in order. mode 0: sum x, 1: sum x^2, 2: sum (x - c)^2.
__global__ void __launch_bounds__(kRedThreads)
    reduce_stage1(const double* __restrict__ x, uint64_t n, int mode, double c,
                  double* __restrict__ part) {
  __shared__ double sh[kRedThreads / 32];
  double acc = 0.0;
  for (uint64_t i = blockIdx.x * uint64_t(kRedThreads) + threadIdx.x; i < n;
       i += uint64_t(kRedBlocks) * kRedThreads) {
    const double v = x[i];
    acc += mode == 0 ? v : (mode == 1 ? v * v : (v - c) * (v - c));
  }
  acc = warp_sum(acc);
  if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x < 32) {
    double v = threadIdx.x < kRedThreads / 32 ? sh[threadIdx.x] : 0.0;
    v = warp_sum(v);
    if (threadIdx.x == 0) part[blockIdx.x] = v;
  }
}

__global__ void reduce_stage2(const double* __restrict__ part, int count,
                              double* __restrict__ out) {
  __shared__ double sh[kRedBlocks];
  sh[threadIdx.x] = threadIdx.x < count ? part[threadIdx.x] : 0.0;
  __syncthreads();
  for (int h = kRedBlocks / 2; h > 0; h >>= 1) {
    if (int(threadIdx.x) < h) sh[threadIdx.x] += sh[threadIdx.x + h];
    __syncthreads();
  }
  if (threadIdx.x == 0) *out = sh[0];
}

// ---------------------------------------------------------------- setup
// warp per pair, one read of both rows: set bits per row (load-balancing
// weights, list sizes) and is_comp[j] = (row 2j+1 == ~row 2j, tail cleared)
// (solver.cpp:188-198)
__global__ void pair_scan_kernel(const uint64_t* __restrict__ rows, uint32_t W, uint32_t n, uint64_t pairs,
                                 uint32_t* __restrict__ pop, uint8_t* __restrict__ is_comp, int kept_only) {
  const uint64_t j = (blockIdx.x * uint64_t(blockDim.x) + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (j >= pairs) return;
  const uint64_t tail = (n % 64) ? ((1ull << (n % 64)) - 1) : ~0ull;
  const uint64_t* e = rows + (kept_only ? j : 2 * j) * W;
  const uint64_t* o = e + W;
  uint32_t pe = 0, po = 0;
  bool ok = true;
  for (uint32_t w = lane; w < W; w += 32) {
    const uint64_t x = e[w];
    pe += __popcll(x);
    if (!kept_only) {
      const uint64_t y = o[w];
      po += __popcll(y);
      ok &= (y == ((w == W - 1) ? (~x & tail) : ~x));
    }
  }

#pragma unroll
  for (int d = 16; d > 0; d >>= 1) {
    pe += __shfl_xor_sync(kFull, pe, d);
    po += __shfl_xor_sync(kFull, po, d);
  }
  ok = __all_sync(kFull, ok);
  if (kept_only) po = n - pe;
  if (lane == 0) {
    pop[2 * j] = pe;
    pop[2 * j + 1] = po;
    is_comp[j] = ok ? 1 : 0;
  }
}

__global__ void init_r_kernel(const double* __restrict__ sw,
                              const double* __restrict__ tgt, uint64_t rows,
                              double* __restrict__ r) {
  const uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x;
  if (i < rows) r[i] = sw[i] * tgt[i];
}

// ---------------------------------------------------------------- M u
// acc += su[base + b] over the set bits b of a 32-bit half word (FLO from
// the top: one instruction per bit instead of a 64-bit find-first-set)
__device__ __forceinline__ void add_bits(uint32_t x, const double* __restrict__ su, int base,
                                         double& acc) {
  while (x) {
    const int b = 31 - __clz(x);
    x ^= 1u << b;
    acc += su[base + b];
  }
}

// One CTA (32 warps) per block of rows (whole complement pairs; block
// boundaries balance the set-bit count, rows are ordered by coalition size).
// The player axis is walked in word-aligned chunks of up to kFwdChunk
// doubles of u staged in shared memory (one chunk when n <= kFwdChunk);
// every needed row of the block adds the u values of its set bits in the
// chunk (warp per row, dynamic fetch, largest coalitions first), so each
// mask word is read exactly once. Odd rows of complement pairs are skipped:
// the epilogue applies the complement shortcut (solver.cpp:261-263), writes
// v and leaves the block's partial sum of v^2 for a fixed-order reduction.
constexpr uint32_t kFwdRows = 1024;
constexpr int kFwdThreads = 1024;
constexpr uint32_t kFwdChunk = 24576;  // doubles (192 KB), a multiple of 64
constexpr int kFwdWordsPerLane = kFwdChunk / 64 / 32;  // 12

__global__ void __launch_bounds__(kFwdThreads)
    forward_kernel(const uint64_t* __restrict__ rows, uint32_t W, const uint32_t* __restrict__ row_start,
                   const uint8_t* __restrict__ is_comp, const double* __restrict__ u,
                   uint32_t n, const double* __restrict__ sw,
                   const double* __restrict__ sum_u, double* __restrict__ v,
                   double* __restrict__ dsq_part, int kept_only) {
  extern __shared__ double su[];  // min(n, kFwdChunk) doubles
  __shared__ double rowsum[kFwdRows];
  __shared__ double red[kFwdThreads / 32];
  __shared__ unsigned next_row;
  const uint64_t r0 = row_start[blockIdx.x];
  const uint32_t nr = row_start[blockIdx.x + 1] - uint32_t(r0);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (uint32_t i = threadIdx.x; i < nr; i += blockDim.x) rowsum[i] = 0.0;
  for (uint32_t e0 = 0; e0 < n; e0 += kFwdChunk) {
    const uint32_t ce = min(n - e0, kFwdChunk);
    __syncthreads();  // the previous chunk's lookups are done
    if (threadIdx.x == 0) next_row = 0;
#pragma unroll 4
    for (uint32_t i = threadIdx.x; i < ce; i += blockDim.x) su[i] = u[e0 + i];
    __syncthreads();
    const uint32_t w0 = e0 / 64, w1 = min(W, (e0 + ce + 63) / 64);
    for (;;) {
      unsigned f = 0;
      if (lane == 0) f = atomicAdd(&next_row, 1u);
      f = __shfl_sync(kFull, f, 0);
      if (f >= nr) break;
      const uint32_t rl = nr - 1 - f;
      const uint64_t row = r0 + rl;
      if ((row & 1) && is_comp[row >> 1]) continue;
      const uint64_t* rp = rows + (kept_only ? (row >> 1) : row) * W;
      double acc0 = 0.0, acc1 = 0.0;
      // all of this lane's words of the chunk are loaded before any is used
      uint64_t xs[kFwdWordsPerLane];
#pragma unroll
      for (int q = 0; q < kFwdWordsPerLane; ++q) {
        const uint32_t w = w0 + lane + 32 * q;
        xs[q] = w < w1 ? __ldcs(rp + w) : 0ull;
      }
#pragma unroll
      for (int q = 0; q < kFwdWordsPerLane; ++q) {
        const int base = int((w0 + lane + 32 * q) * 64 - e0);
        add_bits(uint32_t(xs[q]), su, base, acc0);
        add_bits(uint32_t(xs[q] >> 32), su, base + 32, acc1);
      }
      double acc = warp_sum(acc0 + acc1);
      if (lane == 0) rowsum[rl] += acc;
    }
  }
  __syncthreads();
  double dsq = 0.0;
  for (uint32_t jl = threadIdx.x; 2 * jl < nr; jl += blockDim.x) {
    const uint64_t e = r0 + 2 * jl;
    const double de = rowsum[2 * jl];
    const double ve = sw[e] * de;
    const double vo = is_comp[e >> 1] ? sw[e + 1] * (*sum_u - de) : sw[e + 1] * rowsum[2 * jl + 1];
    v[e] = ve;
    v[e + 1] = vo;
    dsq += ve * ve + vo * vo;
  }
  dsq = warp_sum(dsq);
  if (lane == 0) red[warp] = dsq;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int i = 0; i < kFwdThreads / 32; ++i) t += red[i];
    dsq_part[blockIdx.x] = t;
  }
}

// ---------------------------------------------------------------- nibble tables
// When every pair is a complement pair (the sampler's layout), both passes
// run dense over the mask words instead of looping over set bits: each
// 4-bit nibble of a word indexes a 16-entry table of subset sums (the 16
// sums of 4 coefficients, 128 bytes = one row of shared-memory banks). All
// lanes of a warp read the same table row at the same time (lanes own rows
// in M u and players in M^T r), so every lookup is a conflict-free shared
// load, there is no per-bit loop and no divergence except skipping all-zero
// 32-bit half words. 16 lookups per word replace ~4 set bits at ~25
// issued instructions each.

// The 16 subset sums of (a, b, c, d), nibble bit i <-> element i. Table
// rows are XOR-swizzled by the nibble group's index within its word
// (key = j in 0..15, entry v stored at v ^ key): the builder's lanes own
// different groups, so unswizzled rows would put a whole warp's stores in
// one bank pair; the lookups (one table row per warp at a time) stay
// conflict-free since the key is warp-uniform and folds into the mask op.
__device__ __forceinline__ void subset_sums(double a, double b, double c, double d, uint32_t key,
                                            double* __restrict__ t) {
  const double ab = a + b, cd = c + d;
  const double lo[4] = {0.0, a, b, ab};
  const double hi[4] = {0.0, c, d, cd};
#pragma unroll
  for (int h = 0; h < 4; ++h)
#pragma unroll
    for (int l = 0; l < 4; ++l) t[uint32_t(h * 4 + l) ^ key] = (h == 0) ? lo[l] : (l == 0 ? hi[h] : hi[h] + lo[l]);
}

// acc += sum over the 8 nibbles of x of tab[j][nibble_j ^ (kbase + j)] (8
// swizzled rows of 16 at base + wb + kImm). The keys are XORed into x with
// one constant first; each lookup is then one shift and one LOP3 ((x >> s)
// & 0x78 | wb, wb a multiple of 2048 with the low bits free) in front of
// the LDS, whose immediate carries kImm + 128 j.
template <uint32_t kbase, uint32_t kImm>
__device__ __forceinline__ void nib8(uint32_t x, const char* __restrict__ base, uint32_t wb, double& acc) {
  if (x == 0u) return;
  const uint32_t xk = x ^ (kbase == 0 ? 0x76543210u : 0xFEDCBA98u);
  double t[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    const uint32_t off = ((j == 0 ? (xk << 3) : (xk >> (4 * j - 3))) & 0x78u) | wb;
    t[j] = *reinterpret_cast<const double*>(base + off + kImm + j * 128);
  }
  acc += ((t[0] + t[1]) + (t[2] + t[3])) + ((t[4] + t[5]) + (t[6] + t[7]));
}

// M^T (coef) over the transposed pair tiles: CTA = kNbPlayers players x one
// split of tiles; per step kNbTT tiles' tables (16 per tile) are built from
// the coefficients (double-buffered, one barrier per step).
constexpr int kNbTT = 8;
constexpr int kNbPer = 2;  // players per thread
constexpr int kNbPlayers = 256 * kNbPer;

template <int kMinBlocks>
__global__ void __launch_bounds__(256, kMinBlocks)
    nib_transpose_kernel(const uint64_t* __restrict__ mt, uint64_t Wp, uint32_t n, uint64_t ptiles,
                         const uint32_t* __restrict__ split_start, const double* __restrict__ coef,
                         double* __restrict__ s_part) {
  __shared__ __align__(16) double tab[2][kNbTT][16][16];  // 32 KB
  const int tid = threadIdx.x;
  const uint32_t e0 = blockIdx.x * kNbPlayers + tid;
  const uint64_t t0 = split_start[blockIdx.y], t1 = split_start[blockIdx.y + 1];
  double acc[kNbPer];
#pragma unroll
  for (int p = 0; p < kNbPer; ++p) acc[p] = 0.0;
  int buf = 0;
  for (uint64_t tb = t0; tb < t1; tb += kNbTT, buf ^= 1) {
    const int nt = (t1 - tb) < uint64_t(kNbTT) ? int(t1 - tb) : kNbTT;
    uint64_t w[kNbTT][kNbPer];
#pragma unroll
    for (int q = 0; q < kNbTT; ++q)
#pragma unroll
      for (int p = 0; p < kNbPer; ++p) {
        const uint32_t e = e0 + p * 256;
        w[q][p] = (q < nt && e < n) ? __ldcs(mt + (tb + q) * Wp + e) : 0ull;
      }
    if (tid < kNbTT * 16) {  // one (tile, nibble group) per thread
      const int q = tid >> 4, j = tid & 15;
      double a = 0.0, b = 0.0, c = 0.0, d = 0.0;
      if (q < nt && tb + q < ptiles) {
        const double2* cp = reinterpret_cast<const double2*>(coef + (tb + q) * 64 + 4 * j);
        const double2 x = cp[0], y = cp[1];
        a = x.x, b = x.y, c = y.x, d = y.y;
      }
      subset_sums(a, b, c, d, uint32_t(j), &tab[buf][q][j][0]);
    }
    __syncthreads();
    const char* tbase = reinterpret_cast<const char*>(&tab[0][0][0][0]);
    const uint32_t wb = uint32_t(buf) * uint32_t(sizeof(tab[0]));
    static_assert(sizeof(tab[0]) % 2048 == 0, "table halves on 2048-byte boundaries");
    auto tile = [&](auto qc) {
      constexpr int q = decltype(qc)::value;
#pragma unroll
      for (int p = 0; p < kNbPer; ++p) {
        nib8<0, q * 2048>(uint32_t(w[q][p]), tbase, wb, acc[p]);
        nib8<8, q * 2048 + 1024>(uint32_t(w[q][p] >> 32), tbase, wb, acc[p]);
      }
    };
    static_assert(kNbTT == 8, "unrolled over 8 tiles");
    tile(std::integral_constant<int, 0>{});
    tile(std::integral_constant<int, 1>{});
    tile(std::integral_constant<int, 2>{});
    tile(std::integral_constant<int, 3>{});
    tile(std::integral_constant<int, 4>{});
    tile(std::integral_constant<int, 5>{});
    tile(std::integral_constant<int, 6>{});
    tile(std::integral_constant<int, 7>{});
  }
  double* out = s_part + uint64_t(blockIdx.y) * n;
#pragma unroll
  for (int p = 0; p < kNbPer; ++p) {
    const uint32_t e = e0 + p * 256;
    if (e < n) out[e] = acc[p];
  }
}

// The dense pairs' even rows, word-major (rT[w][jl], jl = j - pd, padded with
// zero rows to a whole number of 256-pair blocks), so the forward pass reads
// one coalesced 8-byte word per lane. Built once per solve.
__global__ void __launch_bounds__(256)
    rows_word_major_kernel(const uint64_t* __restrict__ rows, uint32_t W, uint64_t row_step, uint64_t pd,
                           uint64_t pairs, uint64_t pstride, uint64_t* __restrict__ rT) {
  __shared__ uint64_t t[32][33];
  const uint32_t w0 = blockIdx.x * 32;
  const uint64_t jl0 = blockIdx.y * 32ull;
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  for (int r = ty; r < 32; r += 8) {  // r: pair within the tile, tx: word
    const uint64_t j = pd + jl0 + r;
    t[r][tx] = (j < pairs && w0 + tx < W) ? rows[j * row_step + w0 + tx] : 0ull;
  }
  __syncthreads();
  for (int r = ty; r < 32; r += 8)  // r: word, tx: pair
    if (w0 + r < W) rT[uint64_t(w0 + r) * pstride + jl0 + tx] = t[tx][r];
}

// The same word-major rows from the tile-transposed layout: per (dense tile
// t, word w) one warp transposes the 64 x 64 bit block (64 players' pair
// words -> 64 pairs' player words; a 64 x 64 bit transpose is its own
// inverse, the butterfly of transpose_tiles_kernel). Tiles past ptiles give
// the zero pad rows. Lets the rows buffer be overwritten by rT.
__global__ void __launch_bounds__(256)
    tiles_word_major_kernel(const uint64_t* __restrict__ mt, uint64_t Wp, uint32_t W, uint64_t tiles_b,
                            uint64_t ptiles, uint64_t pstride, uint64_t* __restrict__ rT) {
  const int lane = threadIdx.x & 31;
  const uint64_t blk = blockIdx.x * 8ull + (threadIdx.x >> 5);
  const uint64_t nt = pstride / 64;  // tile slots of rT (dense tiles + zero pad)
  if (blk >= nt * W) return;
  const uint32_t w = uint32_t(blk / nt);
  const uint64_t tl = blk % nt, t = tiles_b + tl;
  uint64_t* o = rT + uint64_t(w) * pstride + tl * 64;
  if (t >= ptiles) {
    o[lane] = 0ull;
    o[lane + 32] = 0ull;
    return;
  }
  const uint64_t* src = mt + t * Wp + uint64_t(w) * 64;
  const uint64_t r0 = src[lane], r1 = src[lane + 32];
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
  o[lane] = (uint64_t(c) << 32) | a;
  o[lane + 32] = (uint64_t(d) << 32) | b;
}

// M u over the dense pairs, lane per pair: CTA = 256 pairs x one part of
// the player axis, walked in chunks of kNbChunk players whose tables (built
// from u) fill 64 KB of shared memory. Writes the even-row dots per part.
constexpr uint32_t kNbChunk = 2048;  // players per table chunk (a multiple of 64)

template <uint32_t kChunk>
__global__ void __launch_bounds__(256)
    nib_forward_kernel(const uint64_t* __restrict__ rT, uint64_t pstride, uint64_t pairs_n,
                       const double* __restrict__ u, uint32_t n, uint32_t part_players,
                       double* __restrict__ vpart) {
  extern __shared__ __align__(16) double ftab[];  // [kChunk / 4][16]
  const int tid = threadIdx.x;
  const uint64_t jl = blockIdx.x * 256ull + tid;
  const uint32_t p0 = blockIdx.y * part_players, p1 = min(n, p0 + part_players);
  const uint64_t* col = rT + jl;
  double acc0 = 0.0, acc1 = 0.0;
  for (uint32_t c0 = p0; c0 < p1; c0 += kChunk) {
    const uint32_t cp = min(kChunk, p1 - c0);
    __syncthreads();  // the previous chunk's lookups are done
    for (uint32_t g = tid; g < kChunk / 4; g += 256) {
      const uint32_t e = c0 + 4 * g;
      double a = 0.0, b = 0.0, c = 0.0, d = 0.0;
      if (4 * g < cp) {  // n need not be a multiple of 4
        a = u[e];
        if (e + 1 < p1) b = u[e + 1];
        if (e + 2 < p1) c = u[e + 2];
        if (e + 3 < p1) d = u[e + 3];
      }
      subset_sums(a, b, c, d, g & 15u, ftab + g * 16);
    }
    __syncthreads();
    const uint32_t w0 = c0 / 64, nw = (cp + 63) / 64;
    for (uint32_t k = 0; k < nw; k += 8) {
      uint64_t x[8];
#pragma unroll
      for (int q = 0; q < 8; ++q) x[q] = (k + q < nw) ? __ldcs(col + uint64_t(w0 + k + q) * pstride) : 0ull;
      const char* tbase = reinterpret_cast<const char*>(ftab);
      const uint32_t wb = k * 2048u;  // k is a multiple of 8: bits below 2^14 free
      auto word = [&](auto qc) {
        constexpr int q = decltype(qc)::value;
        nib8<0, q * 2048>(uint32_t(x[q]), tbase, wb, (q & 1) ? acc1 : acc0);
        nib8<8, q * 2048 + 1024>(uint32_t(x[q] >> 32), tbase, wb, (q & 1) ? acc1 : acc0);
      };
      word(std::integral_constant<int, 0>{});
      word(std::integral_constant<int, 1>{});
      word(std::integral_constant<int, 2>{});
      word(std::integral_constant<int, 3>{});
      word(std::integral_constant<int, 4>{});
      word(std::integral_constant<int, 5>{});
      word(std::integral_constant<int, 6>{});
      word(std::integral_constant<int, 7>{});
    }
  }
  if (jl < pairs_n) vpart[uint64_t(blockIdx.y) * pairs_n + jl] = acc0 + acc1;
}

// v (complement shortcut, solver.cpp:261-263) and per-block sums of v^2
__global__ void __launch_bounds__(256)
    nib_forward_finish(const double* __restrict__ vpart, uint32_t parts, uint64_t j0, uint64_t pairs,
                       const double* __restrict__ sw, const double* __restrict__ sum_u,
                       double* __restrict__ v, double* __restrict__ dsq_part) {
  __shared__ double red[8];
  const uint64_t j = j0 + blockIdx.x * 256ull + threadIdx.x;
  double dsq = 0.0;
  if (j < pairs) {
    double de = 0.0;
    for (uint32_t k = 0; k < parts; ++k) de += vpart[uint64_t(k) * (pairs - j0) + (j - j0)];
    const double ve = sw[2 * j] * de, vo = sw[2 * j + 1] * (*sum_u - de);
    v[2 * j] = ve;
    v[2 * j + 1] = vo;
    dsq = ve * ve + vo * vo;
  }
  dsq = warp_sum(dsq);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = dsq;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int i = 0; i < 8; ++i) t += red[i];
    dsq_part[blockIdx.x] = t;
  }
}

// ---------------------------------------------------------------- kept-set lists
// The sparse pairs [0, pd) (small coalitions: most of the mask bytes, few of
// the bits) are expanded once per solve into u32 index lists, so their
// passes cost per kept player instead of per mask word:
//   rows     per pair j, the even row's players, ascending      (M u)
//   players  per player e, the pairs j < pd containing e, ascending (M^T r)
// Lists are ascending and reduced in a fixed order (bitwise reproducible).
constexpr uint32_t kListTiles = 128;  // pair tiles per counting segment

__global__ void even_pop_kernel(const uint32_t* __restrict__ pop, uint64_t pd, uint64_t* __restrict__ cnt) {
  const uint64_t j = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x;
  if (j <= pd) cnt[j] = j < pd ? pop[2 * j] : 0;
}

// warp per pair: the even row's set bits in ascending order
__global__ void row_list_fill_kernel(const uint64_t* __restrict__ rows, uint32_t W, uint64_t row_step,
                                     uint64_t pd, const uint64_t* __restrict__ off, uint32_t* __restrict__ idx) {
  const uint64_t j = (blockIdx.x * uint64_t(blockDim.x) + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (j >= pd) return;
  const uint64_t* rp = rows + j * row_step;
  uint64_t base = off[j];
  for (uint32_t wb = 0; wb < W; wb += 32) {
    const uint32_t w = wb + lane;
    uint64_t x = w < W ? rp[w] : 0ull;
    const uint32_t k = __popcll(x);
    uint32_t incl = k;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t t = __shfl_up_sync(kFull, incl, o);
      if (lane >= o) incl += t;
    }
    uint64_t pos = base + incl - k;
    while (x) {
      const int b = __ffsll(static_cast<long long>(x)) - 1;
      x &= x - 1;
      idx[pos++] = w * 64 + uint32_t(b);
    }
    base += __shfl_sync(kFull, incl, 31);
  }
}

// thread per (segment g, player e) over the transposed tiles [0, tiles_b):
// counts in player-major order so a player's list is contiguous
__global__ void player_list_count_kernel(const uint64_t* __restrict__ mt, uint64_t Wp, uint32_t n,
                                         uint64_t tiles_b, uint32_t segs, uint64_t* __restrict__ cnt) {
  const uint32_t e = blockIdx.x * blockDim.x + threadIdx.x, g = blockIdx.y;
  if (e >= n) return;
  const uint64_t t0 = uint64_t(g) * kListTiles, t1 = min(tiles_b, t0 + kListTiles);
  uint32_t k = 0;
  for (uint64_t t = t0; t < t1; ++t) k += __popcll(mt[t * Wp + e]);
  cnt[uint64_t(e) * segs + g] = k;
}

__global__ void player_list_fill_kernel(const uint64_t* __restrict__ mt, uint64_t Wp, uint32_t n,
                                        uint64_t tiles_b, uint32_t segs, const uint64_t* __restrict__ off,
                                        uint32_t* __restrict__ idx) {
  const uint32_t e = blockIdx.x * blockDim.x + threadIdx.x, g = blockIdx.y;
  if (e >= n) return;
  const uint64_t t0 = uint64_t(g) * kListTiles, t1 = min(tiles_b, t0 + kListTiles);
  uint64_t pos = off[uint64_t(e) * segs + g];
  for (uint64_t t = t0; t < t1; ++t) {
    uint64_t x = mt[t * Wp + e];
    while (x) {
      const int b = __ffsll(static_cast<long long>(x)) - 1;
      x &= x - 1;
      idx[pos++] = uint32_t(t * 64 + b);
    }
  }
}

// sum over list entries [a, b) of val[idx[i]], warp-strided, fixed order
__device__ __forceinline__ double list_sum(const uint32_t* __restrict__ idx, uint64_t a, uint64_t b,
                                           const double* __restrict__ val, int lane) {
  double acc0 = 0.0, acc1 = 0.0;
  uint64_t i = a + lane;
  for (; i + 96 < b; i += 128) {
    const uint32_t i0 = idx[i], i1 = idx[i + 32], i2 = idx[i + 64], i3 = idx[i + 96];
    const double x0 = __ldg(val + i0), x1 = __ldg(val + i1), x2 = __ldg(val + i2), x3 = __ldg(val + i3);
    acc0 += x0 + x2;
    acc1 += x1 + x3;
  }
  for (; i < b; i += 32) acc0 += __ldg(val + idx[i]);
  return warp_sum(acc0 + acc1);
}

// M u over the sparse pairs: CTA = 64 pairs (8 per warp); v by the
// complement shortcut and the CTA's sum of v^2
__global__ void __launch_bounds__(256)
    list_forward_kernel(const uint64_t* __restrict__ off, const uint32_t* __restrict__ idx, uint64_t pd,
                        const double* __restrict__ u, const double* __restrict__ sw,
                        const double* __restrict__ sum_u, double* __restrict__ v,
                        double* __restrict__ dsq_part) {
  __shared__ double red[8];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  double dsq = 0.0;
  for (int q = 0; q < 8; ++q) {
    const uint64_t j = blockIdx.x * 64ull + warp * 8 + q;
    if (j >= pd) break;
    const double de = list_sum(idx, off[j], off[j + 1], u, lane);
    const double ve = sw[2 * j] * de, vo = sw[2 * j + 1] * (*sum_u - de);
    if (lane == 0) {
      v[2 * j] = ve;
      v[2 * j + 1] = vo;
    }
    dsq += ve * ve + vo * vo;
  }
  if (lane == 0) red[warp] = dsq;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int i = 0; i < 8; ++i) t += red[i];
    dsq_part[blockIdx.x] = t;
  }
}

// M^T coef over the sparse pairs: warp per player
__global__ void __launch_bounds__(256)
    list_transpose_kernel(const uint64_t* __restrict__ off, const uint32_t* __restrict__ idx, uint32_t n,
                          uint32_t segs, const double* __restrict__ coef, double* __restrict__ out) {
  const int lane = threadIdx.x & 31;
  const uint32_t e = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (e >= n) return;
  const double acc = list_sum(idx, off[uint64_t(e) * segs], off[uint64_t(e + 1) * segs], coef, lane);
  if (lane == 0) out[e] = acc;
}

// ---------------------------------------------------------------- updates
__global__ void axpy_kernel(double* __restrict__ y, const double* __restrict__ x,
                            const double* __restrict__ alpha_num,
                            const double* __restrict__ alpha_den, double sign,
                            uint64_t n) {
  const uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x;
  if (i >= n) return;
  const double a = sign * (*alpha_num / *alpha_den);
  y[i] += a * x[i];
}

// One CGLS step's scalars on the device (solver.cpp:282-296): delta =
// ||v||^2 (all-reduced, scal[1]) + v_c^2 with v_c = sqrt(cw) sum_u
// (scal[0]); stop flag scal[12] = 2 non-finite, 1 delta <= 0; theta =
// gamma / delta applied through scal[8] / scal[9]; r_c (scal[7]) -= theta v_c.
// (scal[gslot] = scal[nslot] first: the previous iteration's gamma_next
// becomes this iteration's gamma, so every iteration runs the same kernels
// with the same arguments — one CUDA graph replays them)
__global__ void step_kernel(double* __restrict__ scal, double scw, int gslot, int nslot) {
  scal[gslot] = scal[nslot];
  const double v_c = scw * scal[0];
  const double delta = scal[1] + v_c * v_c;
  const double stop = !isfinite(delta) ? 2.0 : (delta <= 0.0 ? 1.0 : 0.0);
  scal[9] = delta;
  scal[12] = stop;
  if (stop == 0.0) {
    const double gamma = scal[gslot];
    scal[8] = gamma;
    scal[7] -= (gamma / delta) * v_c;
  }
}

// y += sign (num / den) x unless *stop is set
__global__ void axpy_stop_kernel(double* __restrict__ y, const double* __restrict__ x,
                                 const double* __restrict__ scal, double sign, uint64_t n) {
  const uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x;
  if (i >= n || scal[12] != 0.0) return;
  y[i] += sign * (scal[8] / scal[9]) * x[i];
}

// s += sqrt(cw) r_c (the pin row), r_c on the device
__global__ void add_pin_kernel(double* __restrict__ s, double scw, const double* __restrict__ r_c, uint32_t n) {
  const uint32_t e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e < n) s[e] += scw * (*r_c);
}

// u = s + beta u, beta = gamma_next / gamma (solver.cpp:357-358)
__global__ void direction_kernel(double* __restrict__ u, const double* __restrict__ s,
                                 const double* __restrict__ g_next,
                                 const double* __restrict__ g, uint64_t n) {
  const uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x;
  if (i >= n) return;
  const double beta = *g_next / *g;
  u[i] = s[i] + beta * u[i];
}

// ---------------------------------------------------------------- M^T r
// Pair coefficients (solver.cpp:209-217): a complement pair contributes
// c_o to every player (kconst) plus (c_e - c_o) on the even row's bits; a
// non-complement pair contributes c_e on the even row and c_o on the odd
// row (second tile layout). Entries past `pairs` are zero.
__global__ void coef_kernel(const double* __restrict__ sw, const double* __restrict__ r,
                            const uint8_t* __restrict__ is_comp, uint64_t pairs, uint64_t padded,
                            double* __restrict__ coef_e, double* __restrict__ coef_o,
                            double* __restrict__ kconst) {
  const uint64_t j = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x;
  if (j >= padded) return;
  double ce = 0.0, co = 0.0, kc = 0.0;
  if (j < pairs) {
    const double e = sw[2 * j] * r[2 * j], o = sw[2 * j + 1] * r[2 * j + 1];
    if (is_comp[j]) {
      ce = e - o;
      kc = o;
    } else {
      ce = e;
      co = o;
    }
    kconst[j] = kc;
  }
  coef_e[j] = ce;
  coef_o[j] = co;
}

// s_part[split][e] (+)= sum over the split's pair tiles, over set bits i of
// mt[t][e], of coef[t*64+i]. Each thread owns two players; kTT tiles per
// step: their coefficients are staged in shared memory while all 2*kTT
// mask words are in flight.
constexpr int kTT = 8;

__global__ void __launch_bounds__(256)
    transpose_partial_kernel(const uint64_t* __restrict__ mt, uint64_t Wp,
                             uint32_t n, const uint32_t* __restrict__ split_start,
                             const double* __restrict__ coef, int accumulate,
                             double* __restrict__ s_part) {
  __shared__ double sc[kTT][64];
  const uint32_t ea = blockIdx.x * 512 + threadIdx.x, eb = ea + 256;
  const uint64_t t0 = split_start[blockIdx.y], t1 = split_start[blockIdx.y + 1];
  double acc_a = 0.0, acc_b = 0.0, acc_a2 = 0.0, acc_b2 = 0.0;
  for (uint64_t tb = t0; tb < t1; tb += kTT) {
    const int nt = (t1 - tb) < uint64_t(kTT) ? int(t1 - tb) : kTT;
    uint64_t wa[kTT], wb[kTT];
#pragma unroll
    for (int q = 0; q < kTT; ++q) {
      wa[q] = (q < nt && ea < n) ? mt[(tb + q) * Wp + ea] : 0ull;
      wb[q] = (q < nt && eb < n) ? mt[(tb + q) * Wp + eb] : 0ull;
    }
    __syncthreads();  // the previous step's coefficients are consumed
    for (int idx = threadIdx.x; idx < nt * 64; idx += blockDim.x) sc[idx >> 6][idx & 63] = coef[tb * 64 + idx];
    __syncthreads();
#pragma unroll
    for (int q = 0; q < kTT; ++q) {
      add_bits(uint32_t(wa[q]), sc[q], 0, acc_a);
      add_bits(uint32_t(wa[q] >> 32), sc[q], 32, acc_a2);
      add_bits(uint32_t(wb[q]), sc[q], 0, acc_b);
      add_bits(uint32_t(wb[q] >> 32), sc[q], 32, acc_b2);
    }
  }
  acc_a += acc_a2;
  acc_b += acc_b2;
  double* pa = s_part + uint64_t(blockIdx.y) * n;
  if (ea < n) pa[ea] = (accumulate ? pa[ea] : 0.0) + acc_a;
  if (eb < n) pa[eb] = (accumulate ? pa[eb] : 0.0) + acc_b;
}

// s_e = K + sum_split s_part[split][e]
__global__ void transpose_finish_kernel(const double* __restrict__ s_part,
                                        uint32_t splits, uint32_t n,
                                        const double* __restrict__ kconst,
                                        double* __restrict__ s) {
  const uint32_t e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= n) return;
  double acc = *kconst;
  for (uint32_t k = 0; k < splits; ++k) acc += s_part[uint64_t(k) * n + e];
  s[e] = acc;
}

// ---------------------------------------------------------------- fixed order
// Reproducible summation (fixed-order mode). A value x with |x| <= 2^E that
// enters a sum of at most 2^(H-1) terms is split into three parts on fixed
// grids q1 = 2^(E+H-52), q2 = q1 2^(H-53), q3 = q2 2^(H-53): x1 = rint(x/q1)
// q1, x2 = rint((x-x1)/q2) q2, x3 = rint((x-x1-x2)/q3) q3 (every step exact).
// Any sum of same-level parts is then exact in FP64 in any order and
// grouping, so the level sums — and ((S1 + S2) + S3) — do not depend on how
// rows are split across ranks, tiles, CTAs or NCCL's reduction order. The
// grids come from bounds that every rank computes identically.
__device__ __forceinline__ void split3(double x, const double* g, double& a, double& b, double& c) {
  a = rint(x * (1.0 / g[0])) * g[0];
  const double r1 = x - a;
  b = rint(r1 * (1.0 / g[1])) * g[1];
  const double r2 = r1 - b;
  c = rint(r2 * (1.0 / g[2])) * g[2];
}

// out[k * stride + i] = part k of x[i] (0 past count)
__global__ void split3_kernel(const double* __restrict__ x, uint64_t count, uint64_t padded,
                              const double* __restrict__ grid, double* __restrict__ out, uint64_t stride) {
  const uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x;
  if (i >= padded) return;
  double a = 0.0, b = 0.0, c = 0.0;
  if (i < count) split3(x[i], grid, a, b, c);
  out[i] = a;
  out[stride + i] = b;
  out[2 * stride + i] = c;
}

// max_i |x_i * (y ? y_i : 1)|, one CTA
__global__ void __launch_bounds__(1024) absmax_kernel(const double* __restrict__ x, const double* __restrict__ y,
                                                      uint64_t count, double* __restrict__ out) {
  __shared__ double red[32];
  double m = 0.0;
  for (uint64_t i = threadIdx.x; i < count; i += blockDim.x) m = fmax(m, fabs(x[i] * (y ? y[i] : 1.0)));
  for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = m;
  __syncthreads();
  if (threadIdx.x < 32) {
    m = red[threadIdx.x];
    for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
    if (threadIdx.x == 0) *out = m;
  }
}

__device__ __forceinline__ void make_grid(int E, int H, double* g) {
  g[0] = ldexp(1.0, E + H - 52);
  g[1] = ldexp(g[0], H - 53);
  g[2] = ldexp(g[1], H - 53);
}

// per-iteration grids from the replicated direction u: gU for the parts of
// u (row dots of <= n terms, complements sum_u - dot), gD for v^2 (rows)
__global__ void iter_grids_kernel(const double* __restrict__ umax, int e_sw, int log_n, int h_u, int h_rows,
                                  double* __restrict__ gU, double* __restrict__ gD) {
  int e = 0;
  frexp(*umax, &e);  // umax < 2^e
  if (*umax == 0.0) e = -1000;
  make_grid(e, h_u, gU);
  // |v| <= max sw * n * umax
  make_grid(2 * (e_sw + e + log_n), h_rows, gD);
}

// s = (((L0 + L1) + L2) + ((K0 + K1) + K2)) + pin
__global__ void combine_s_kernel(const double* __restrict__ lev, uint32_t n, double pin, double* __restrict__ s) {
  const uint32_t e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= n) return;
  const double* k = lev + 3ull * n;
  s[e] = (((lev[e] + lev[n + e]) + lev[2ull * n + e]) + ((k[0] + k[1]) + k[2])) + pin;
}

// v = sw ((V0 + V1) + V2) per row, and the parts of v^2 for delta
__global__ void combine_v_kernel(const double* __restrict__ vl, uint64_t rows, const double* __restrict__ sw,
                                 const double* __restrict__ gD, double* __restrict__ v,
                                 double* __restrict__ dparts) {
  const uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x;
  if (i >= rows) return;
  const double x = sw[i] * ((vl[i] + vl[rows + i]) + vl[2 * rows + i]);
  v[i] = x;
  double a, b, c;
  split3(x * x, gD, a, b, c);
  dparts[i] = a;
  dparts[rows + i] = b;
  dparts[2 * rows + i] = c;
}

__global__ void sq_parts_kernel(const double* __restrict__ r, uint64_t rows, const double* __restrict__ g,
                                double* __restrict__ parts) {
  const uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x;
  if (i >= rows) return;
  double a, b, c;
  split3(r[i] * r[i], g, a, b, c);
  parts[i] = a;
  parts[rows + i] = b;
  parts[2 * rows + i] = c;
}

// ---------------------------------------------------------------- fixed order, small systems
// The reference's own order (PairwiseFolder, solver.cpp:31-61, 227-237,
// 270-279): leaves are pushed in bit-reversed local pair order and folded
// in a binary tree; with the Communicator folding ranks by halves this is
// one tree over the global pairs, the same for every worker count. Used when
// padded pairs x players is small (the leaves are dense n-vectors).
__device__ __forceinline__ uint64_t bitrev_n(uint64_t x, int bits) {
  return bits ? (__brevll(x) >> (64 - bits)) : 0ull;
}

// thread per player: s_local[e] = folded leaves, leaf_j[e] = c_o + (c_e - c_o)
// bit (complement pair, solver.cpp:209-217) or c_e bit_e + c_o bit_o
__global__ void __launch_bounds__(128) tree_transpose_kernel(const uint64_t* __restrict__ mte,
                                                             const uint64_t* __restrict__ mto, uint64_t Wp,
                                                             uint32_t n, uint64_t pairs, const uint8_t* __restrict__ is_comp,
                                                             const double* __restrict__ sw, const double* __restrict__ r,
                                                             uint64_t padded, int log_local, double* __restrict__ out) {
  const uint32_t e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= n) return;
  double slot[40];
  double carry = 0.0;
  for (uint64_t t = 0; t < padded; ++t) {
    const uint64_t j = bitrev_n(t, log_local);
    double leaf = 0.0;
    if (j < pairs) {
      const double ce = sw[2 * j] * r[2 * j], co = sw[2 * j + 1] * r[2 * j + 1];
      const double be = double((mte[(j >> 6) * Wp + e] >> (j & 63)) & 1ull);
      if (is_comp[j]) {
        leaf = co + (ce - co) * be;
      } else {
        const double bo = double((mto[(j >> 6) * Wp + e] >> (j & 63)) & 1ull);
        leaf = ce * be + co * bo;
      }
    }
    carry = leaf;
    int level = 0;
    for (uint64_t c = t; c & 1; c >>= 1, ++level) carry = slot[level] + carry;
    slot[level] = carry;
  }
  int top = 0;
  while (!((padded >> top) & 1)) ++top;
  out[e] = slot[top];
}

// x[0] = fold by halves of x[0, padded) (x[j] += x[j + h], h = padded/2 ... 1):
// the same tree as pushing x in bit-reversed order through the folder
__global__ void fold_level_kernel(double* __restrict__ x, uint64_t h) {
  const uint64_t j = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x;
  if (j < h) x[j] = x[j] + x[j + h];
}
__global__ void __launch_bounds__(1024) fold_small_kernel(double* __restrict__ x, uint64_t padded, double* out) {
  __shared__ double sm[2048];
  for (uint64_t j = threadIdx.x; j < padded; j += blockDim.x) sm[j] = x[j];
  __syncthreads();
  for (uint64_t h = padded / 2; h >= 1; h /= 2) {
    for (uint64_t j = threadIdx.x; j < h; j += blockDim.x) sm[j] = sm[j] + sm[j + h];
    __syncthreads();
  }
  if (threadIdx.x == 0) *out = sm[0];
}
// leaves of the scalar sums: d_j = a[2j]^2 + a[2j+1]^2 for j < pairs, 0 up to padded
__global__ void pair_sq_kernel(const double* __restrict__ a, uint64_t pairs, uint64_t padded, double* __restrict__ d) {
  const uint64_t j = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x;
  if (j >= padded) return;
  d[j] = j < pairs ? a[2 * j] * a[2 * j] + a[2 * j + 1] * a[2 * j + 1] : 0.0;
}

// x <- r - x (exact row residual sqrt(W) t - sqrt(W) M phi for the fused protocol)
__global__ void residual_kernel(const double* __restrict__ r, double* __restrict__ x, uint64_t rows) {
  const uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x;
  if (i < rows) x[i] = r[i] - x[i];
}

__global__ void fill_kernel(double* __restrict__ x, double value, uint64_t count) {
  const uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x;
  if (i < count) x[i] = value;
}

__global__ void add_scalar_kernel(double* __restrict__ s, double c, uint32_t n) {
  const uint32_t e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e < n) s[e] += c;
}

// ---------------------------------------------------------------- assemble
// per row: size = popcount; sw = sqrt(weight_of_size[size]);
// target = double(value) - base (solver.cpp:140-154)
__global__ void assemble_kernel(const uint64_t* __restrict__ rows, uint64_t nrows,
                                uint32_t W, uint32_t n,
                                const double* __restrict__ wsize,
                                const float* __restrict__ values, double base,
                                double* __restrict__ sw, double* __restrict__ tgt,
                                int* __restrict__ bad) {
  const uint64_t row = (blockIdx.x * uint64_t(blockDim.x) + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (row >= nrows) return;
  uint32_t cnt = 0;
  for (uint32_t w = lane; w < W; w += 32) cnt += __popcll(rows[row * W + w]);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) cnt += __shfl_xor_sync(kFull, cnt, o);
  if (lane == 0) {
    if (cnt == 0 || cnt >= n) {
      atomicMin(bad, row < 0x7fffffffull ? int(row) : 0x7fffffff);
      sw[row] = 0.0;
    } else {
      sw[row] = sqrt(wsize[cnt]);
    }
    tgt[row] = double(values[row]) - base;
  }
}

// warp per pair: assemble_kernel for rows 2j and 2j+1 plus pair_scan_kernel
// (set bits per row, complement flag), one read of both rows
__global__ void assemble_pairs_kernel(const uint64_t* __restrict__ rows, uint64_t pairs, uint32_t W,
                                      uint32_t n, const double* __restrict__ wsize,
                                      const float* __restrict__ values, double base,
                                      double* __restrict__ sw, double* __restrict__ tgt,
                                      int* __restrict__ bad, uint32_t* __restrict__ pop,
                                      uint8_t* __restrict__ is_comp, int kept_only) {
  const uint64_t j = (blockIdx.x * uint64_t(blockDim.x) + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (j >= pairs) return;
  const uint64_t tail = (n % 64) ? ((1ull << (n % 64)) - 1) : ~0ull;
  const uint64_t* e = rows + (kept_only ? j : 2 * j) * W;
  const uint64_t* o = e + W;
  uint32_t pe = 0, po = 0;
  bool ok = true;
  for (uint32_t w = lane; w < W; w += 32) {
    const uint64_t x = e[w];
    pe += __popcll(x);
    if (!kept_only) {
      const uint64_t y = o[w];
      po += __popcll(y);
      ok &= (y == ((w == W - 1) ? (~x & tail) : ~x));
    }
  }
#pragma unroll
  for (int d = 16; d > 0; d >>= 1) {
    pe += __shfl_xor_sync(kFull, pe, d);
    po += __shfl_xor_sync(kFull, po, d);
  }
  ok = __all_sync(kFull, ok);
  if (kept_only) po = n - pe;  // the complement row
  if (lane < 2) {
    const uint64_t row = 2 * j + lane;
    const uint32_t cnt = lane ? po : pe;
    if (cnt == 0 || cnt >= n) {
      atomicMin(bad, row < 0x7fffffffull ? int(row) : 0x7fffffff);
      sw[row] = 0.0;
    } else {
      sw[row] = sqrt(wsize[cnt]);
    }
    tgt[row] = double(values[row]) - base;
    pop[row] = cnt;
    if (lane == 0) is_comp[j] = ok ? 1 : 0;
  }
}


// order-preserving key of -phi (+0 and -0 share a key: they compare equal)
__global__ void rank_keys_kernel(const double* __restrict__ phi, uint32_t n, uint64_t* __restrict__ key,
                                 uint32_t* __restrict__ idx) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double v = phi[i] == 0.0 ? 0.0 : phi[i];
  uint64_t b = uint64_t(__double_as_longlong(v));
  b = (b >> 63) ? ~b : (b | (1ull << 63));  // ascending in v
  key[i] = ~b;                              // descending
  idx[i] = i;
}

inline unsigned blocks_for(uint64_t n, unsigned t = 256) {
  return unsigned((n + t - 1) / t);
}

// device scratch for one solve
struct Scratch {
  unsigned char* base = nullptr;
  uint64_t off = 0;
  template <typename T>
  T* take(uint64_t count) {
    off = (off + 255) & ~uint64_t(255);
    T* p = reinterpret_cast<T*>(base + off);
    off += sizeof(T) * std::max<uint64_t>(count, 1);
    return p;
  }
};

}  // namespace

void launch_assemble(Ctx& ctx, const uint64_t* dev_rows, uint64_t rows,
                     uint32_t W, uint32_t n, const double* dev_wsize,
                     const float* dev_values, double base, double* dev_sw,
                     double* dev_targets, int* dev_bad_row) {
  if (rows == 0) return;
  assemble_kernel<<<blocks_for(rows * 32), 256, 0, ctx.stream>>>(
      dev_rows, rows, W, n, dev_wsize, dev_values, base, dev_sw, dev_targets, dev_bad_row);
  SF_LAUNCHED(ctx);
}

void launch_assemble_pairs(Ctx& ctx, const uint64_t* dev_rows, uint64_t rows, uint32_t W, uint32_t n,
                           const double* dev_wsize, const float* dev_values, double base, double* dev_sw,
                           double* dev_targets, int* dev_bad_row, uint32_t* dev_pop, uint8_t* dev_is_comp,
                           bool kept_only) {
  if (rows == 0) return;
  if (rows % 2) throw DataError("assemble_pairs needs adjacent row pairs");
  assemble_pairs_kernel<<<blocks_for(rows / 2 * 32), 256, 0, ctx.stream>>>(
      dev_rows, rows / 2, W, n, dev_wsize, dev_values, base, dev_sw, dev_targets, dev_bad_row, dev_pop,
      dev_is_comp, kept_only ? 1 : 0);
  SF_LAUNCHED(ctx);
}

CglsResult cgls_solve(Ctx& ctx, const CglsInput& in, double tol,
                      uint64_t max_iter, int mode, bool trace) {
  if (mode != 0 && mode != 1) throw DataError("solver mode must be 0 (reference protocol) or 1 (fused)");
  CglsResult res;
  const uint32_t n = in.n;
  if (n == 0) {
    res.converged = true;
    return res;
  }
  if (in.rows % 2) throw DataError("local rows must come in adjacent pairs");
  const uint64_t rows = in.rows, pairs = rows / 2;
  const uint32_t W = in.W;
  const uint64_t ptiles = (pairs + 63) / 64;  // tiles of 64 pairs (even / odd row layouts)
  const uint64_t Wp = uint64_t(W) * 64;
  int sms = 148;
  SF_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, ctx.device));
  const uint64_t pblocks = (n + 511) / 512;  // transpose: 512 players per CTA
  const uint64_t max_splits = std::max<uint64_t>(1, (8ull * sms) / pblocks);
  const uint64_t nib_pblocks = (n + kNbPlayers - 1) / kNbPlayers;
  // nibble kernels run 3 CTAs per SM; ~8 waves keep the tail wave small
  const uint64_t nib_ctas = 24ull * sms;
  // tensor-core (i8) passes: 128 lanes per item, splits of <= 16384 tiles
  // (2^20 elements: the S32 accumulators stay exact), >= 2 items per SM
  const bool i8 = cgls_i8_enabled();
  const uint64_t i8_pb = (n + 127) / 128;
  const uint64_t i8_max_nsplits = std::max<uint64_t>((2ull * sms + i8_pb - 1) / i8_pb, (ptiles + 16383) / 16384);
  const uint64_t i8_max_parts = std::min<uint64_t>((W + 3) / 4, std::max<uint64_t>(2ull * sms, (W + 16383) / 16384));
  const uint64_t max_nsplits =
      i8 ? i8_max_nsplits : (nib_ctas + nib_pblocks - 1) / nib_pblocks;
  const uint64_t fblocks_max = (rows + 63) / 64 + 8ull * sms + 2 + (pairs + 255) / 256 + 1;
  // nibble forward: the player axis in parts so the grid covers the SMs
  const uint32_t nb_parts_max =
      i8 ? uint32_t(i8_max_parts) : uint32_t(std::min<uint64_t>((n + kNbChunk - 1) / kNbChunk, nib_ctas));
  const uint64_t i8_bytes =
      i8 ? cgls_i8_digit_bytes(uint64_t(W) * 64) + cgls_i8_digit_bytes(ptiles * 64) + cgls_i8_scratch_doubles() * 8 + 64
         : 0;
  const uint64_t bytes = (in.kept_only ? 1 : 2) * ptiles * Wp * 8 + pairs + rows * 8 * 2 + fblocks_max * 8 + rows * 4 +
                         (fblocks_max + max_splits + max_nsplits + 4) * 4 + 2 * ptiles * 64 * 8 + pairs * 8 +
                         (max_splits + max_nsplits + 1) * n * 8 + uint64_t(nb_parts_max) * pairs * 8 + i8_bytes + 5 * 256 +
                         uint64_t(n) * 8 * 6 + 16 + rows * 8 + kRedBlocks * 8 + 64 * 8 + 32 * 8 + 18 * 256;
  const bool repro_req = in.fixed_order;
  // fixed order: the reference's folder tree when the dense leaves are small
  // (and the cross-rank sum is the caller's fold-by-halves or a 2-rank sum),
  // exact level sums otherwise
  auto ceil2 = [](uint64_t x) {
    uint64_t p = 1;
    while (p < x) p <<= 1;
    return p;
  };
  const uint64_t tree_global = ceil2(std::max<uint64_t>(in.global_pair_count, 64));
  const uint64_t tree_local = ceil2(std::max<uint64_t>({tree_global / uint64_t(ctx.world), pairs, 1}));
  int tree_log = 0;
  while ((uint64_t(1) << tree_log) < tree_local) ++tree_log;
  const bool tree = repro_req && tree_local * uint64_t(n) <= (uint64_t(1) << 27) &&
                    (ctx.world <= 2 || ctx.host_comm.all_reduce != nullptr);
  const bool repro = repro_req && !tree;
  if (repro && mode != 0) throw DataError("fixed-order summation runs the reference protocol (solver mode 0)");
  constexpr int kBins = 2201;  // frexp exponents -1100..1100
  const uint64_t repro_bytes =
      repro ? (2 * (3ull * n + 3) + 3 * rows * 2 + 3 * ptiles * 64 * 2 + 3 * std::max<uint64_t>(pairs, 1) + rows +
               (2ull * kBins + 8) + 64) * 8 + 16 * 256
            : 0;
  const uint64_t tree_bytes = tree ? (tree_local + 2) * 8 + 256 : 0;
  ctx.solver_work.reserve(bytes + repro_bytes + tree_bytes);
  Scratch sc{ctx.solver_work.p, 0};
  uint64_t* mte = sc.take<uint64_t>(ptiles * Wp);  // even rows, 64 pairs per tile
  // odd rows (non-complement pairs only; kept-only rows are all complement pairs)
  uint64_t* mto = in.kept_only ? nullptr : sc.take<uint64_t>(ptiles * Wp);
  uint8_t* is_comp = in.dev_is_comp ? const_cast<uint8_t*>(in.dev_is_comp) : sc.take<uint8_t>(pairs);
  double* r = sc.take<double>(rows);
  double* v = sc.take<double>(rows);
  double* coef_e = sc.take<double>(ptiles * 64);
  double* coef_o = sc.take<double>(ptiles * 64);
  double* dsq = sc.take<double>(fblocks_max);
  uint32_t* pop = in.dev_pop ? const_cast<uint32_t*>(in.dev_pop) : sc.take<uint32_t>(rows);
  uint32_t* d_bounds = sc.take<uint32_t>(fblocks_max + max_splits + max_nsplits + 4);
  double* kc = sc.take<double>(pairs);
  double* s_part = sc.take<double>((max_splits + max_nsplits + 1) * n);
  double* vpart = sc.take<double>(uint64_t(nb_parts_max) * pairs);
  uint8_t* i8_udig = i8 ? sc.take<uint8_t>(cgls_i8_digit_bytes(uint64_t(W) * 64)) : nullptr;  // digits of u
  uint8_t* i8_cdig = i8 ? sc.take<uint8_t>(cgls_i8_digit_bytes(ptiles * 64)) : nullptr;      // of the coefficients
  double* i8_abs = i8 ? sc.take<double>(cgls_i8_scratch_doubles()) : nullptr;
  int* i8_exp = i8 ? sc.take<int>(2) : nullptr;
  double* s = sc.take<double>(n);
  double* tv = sc.take<double>(2ull * n + 2);  // fused mode: [A^T v ; ||v||^2 ; A^T r_exact]
  double* vphi = mode == 1 ? sc.take<double>(std::max<uint64_t>(rows, 1)) : nullptr;  // fused: sw M phi
  double* u = sc.take<double>(n);
  double* phi = sc.take<double>(n);
  double* tleaf = tree ? sc.take<double>(tree_local + 2) : nullptr;  // scalar tree leaves
  // fixed-order mode buffers
  double *lev = nullptr, *ul = nullptr, *vl = nullptr, *dparts = nullptr, *cel = nullptr, *col = nullptr,
         *kcl = nullptr, *ones = nullptr, *flags = nullptr, *grids = nullptr;
  if (repro) {
    lev = sc.take<double>(3ull * n + 3);     // all-reduced: 3 level sums of M^T r, 3 of the pair constants
    ul = sc.take<double>(3ull * n + 3);      // parts of u, then their 3 sums
    vl = sc.take<double>(3 * rows);          // per-level row dots
    dparts = sc.take<double>(3 * rows);      // parts of v^2 (or r^2 for the trace)
    cel = sc.take<double>(3 * ptiles * 64);  // parts of the even-row coefficients
    col = sc.take<double>(3 * ptiles * 64);  // parts of the odd-row coefficients
    kcl = sc.take<double>(3 * std::max<uint64_t>(pairs, 1));
    ones = sc.take<double>(rows);
    flags = sc.take<double>(2 * kBins + 8);
    grids = sc.take<double>(64);  // gT[0..3) gU[8..11) gD[16..19) gR[24..27) zero[32] maxes[40..42) dsum[48..51)
  }
  double* red = sc.take<double>(kRedBlocks);
  // device scalars: 0 sum_u, 1 delta, 2 gamma, 3 gamma_next, 4 kconst,
  // 5 sse, 6 data0
  double* scal = sc.take<double>(32);

  cudaStream_t st = ctx.stream;
  auto reduce = [&](const double* x, uint64_t count, int md, double c, double* out) {
    reduce_stage1<<<kRedBlocks, kRedThreads, 0, st>>>(x, count, md, c, red);
    SF_LAUNCHED(ctx);
    reduce_stage2<<<1, kRedBlocks, 0, st>>>(red, kRedBlocks, out);
    SF_LAUNCHED(ctx);
  };
  ctx.solver_host.reserve(32);
  double* host = ctx.solver_host.p;
  auto fetch = [&](int idx, int count) {
    ctx.d2h_bytes += uint64_t(count) * sizeof(double);
    SF_CUDA(cudaMemcpyAsync(host + idx, scal + idx, count * sizeof(double),
                            cudaMemcpyDeviceToHost, st));
    comm_sync(ctx);
  };

  DebugTimer dt("cgls");
  const uint64_t pair_step = in.kept_only ? uint64_t(W) : 2ull * W;  // words between even rows
  launch_transpose_tiles(ctx, in.dev_rows, pairs, W, ptiles, mte, pair_step);
  if (pairs) {
    if (!in.dev_pop || !in.dev_is_comp) {
      pair_scan_kernel<<<blocks_for(pairs * 32), 256, 0, st>>>(in.dev_rows, W, n, pairs, pop, is_comp,
                                                                in.kept_only ? 1 : 0);
      SF_LAUNCHED(ctx);
    }
    init_r_kernel<<<blocks_for(rows), 256, 0, st>>>(in.dev_sw, in.dev_targets, rows, r);
    SF_LAUNCHED(ctx);
  }
  // per-row set-bit counts and complement flags on the host (pinned: the
  // copies run at full PCIe rate and overlap nothing else anyway)
  ctx.cgls_hpop.reserve(std::max<uint64_t>(rows, 1));
  ctx.cgls_hcomp.reserve(std::max<uint64_t>(pairs, 1));
  uint32_t* const h_pop = ctx.cgls_hpop.p;
  uint8_t* const h_comp = ctx.cgls_hcomp.p;
  if (rows) {
    SF_CUDA(cudaMemcpyAsync(h_pop, pop, rows * 4, cudaMemcpyDeviceToHost, st));
    SF_CUDA(cudaMemcpyAsync(h_comp, is_comp, pairs, cudaMemcpyDeviceToHost, st));
    SF_CUDA(cudaStreamSynchronize(st));
    ctx.d2h_bytes += rows * 4 + pairs;
  }
  dt.lap("tiles + pair scan");
  auto needed = [&](uint64_t row) { return !((row & 1) && h_comp[row >> 1]); };
  bool any_noncomp = false;
  for (uint64_t j = 0; j < pairs; ++j) any_noncomp |= !h_comp[j];
  if (any_noncomp && in.kept_only) throw std::logic_error("kept-only rows are complement pairs");
  if (any_noncomp) launch_transpose_tiles(ctx, in.dev_rows + W, pairs, W, ptiles, mto, 2ull * W);

  // Dense tiles (pairs from pd on) take the nibble-table passes, sparse
  // tiles the set-bit loops: with every pair a complement pair, the first
  // tile whose mean kept-set size reaches n * density (SF_CGLS_NIB_DENSITY,
  // default 1/64; the sampler orders pairs by size, so that is a suffix).
  // SF_CGLS_NIBBLE=0 keeps every tile on the set-bit loops.
  uint64_t pd = pairs;
  {
    bool nibble = pairs > 0 && !any_noncomp && !tree;
    if (const char* env = std::getenv("SF_CGLS_NIBBLE")) nibble = nibble && std::atoi(env) != 0;
    double density = 1.0 / 64;
    if (const char* env = std::getenv("SF_CGLS_NIB_DENSITY")) density = std::atof(env);
    if (nibble) {
      const double thr = density * n * 64;
      for (uint64_t t = 0; t < ptiles; ++t) {
        uint64_t c = 0;
        for (uint64_t j = t * 64; j < std::min(pairs, t * 64 + 64); ++j) c += h_pop[2 * j];
        if (double(c) >= thr) {
          pd = t * 64;
          break;
        }
      }
    }
  }
  const uint64_t tiles_b = (pd + 63) / 64, pairs_n = pairs - pd;
  // the sparse pairs as kept-set lists (SF_CGLS_LISTS=0: set-bit loops)
  bool lists = pd > 0 && pd < pairs + 1 && !any_noncomp && !tree;
  if (const char* env = std::getenv("SF_CGLS_LISTS")) lists = lists && std::atoi(env) != 0;
  const uint32_t lsegs = uint32_t(std::max<uint64_t>(1, (tiles_b + kListTiles - 1) / kListTiles));
  const uint64_t* row_off = nullptr;
  const uint32_t* row_idx = nullptr;
  const uint64_t* pl_off = nullptr;
  const uint32_t* pl_idx = nullptr;
  if (lists) {
    uint64_t entries = 0;
    for (uint64_t j = 0; j < pd; ++j) entries += h_pop[2 * j];
    const uint64_t nr = pd + 1, np = uint64_t(n) * lsegs + 1;
    size_t tmp_r = 0, tmp_p = 0;
    SF_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tmp_r, static_cast<const uint64_t*>(nullptr),
                                          static_cast<uint64_t*>(nullptr), nr, st));
    SF_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tmp_p, static_cast<const uint64_t*>(nullptr),
                                          static_cast<uint64_t*>(nullptr), np, st));
    const uint64_t tmp = std::max(tmp_r, tmp_p);
    const uint64_t need = 2 * (nr + np) * 8 + tmp + 2 * entries * 4 + 8 * 256;
    // (no cudaMemGetInfo: it measured 0.15-45 ms per call; an allocation
    // that fails falls back to the set-bit loops instead)
    if (need > ctx.solver_lists.n) {
      try {
        ctx.solver_lists.reserve(need);
      } catch (const std::exception&) {
        cudaGetLastError();
        ctx.solver_lists.release();
        lists = false;
      }
    }
    if (lists) {
      Scratch sp{ctx.solver_lists.p, 0};
      uint64_t* r_cnt = sp.take<uint64_t>(nr);
      uint64_t* r_off = sp.take<uint64_t>(nr);
      uint64_t* p_cnt = sp.take<uint64_t>(np);
      uint64_t* p_off = sp.take<uint64_t>(np);
      void* tmp_buf = sp.take<unsigned char>(tmp);
      uint32_t* r_idx = sp.take<uint32_t>(entries);
      uint32_t* p_idx = sp.take<uint32_t>(entries);
      even_pop_kernel<<<blocks_for(nr), 256, 0, st>>>(pop, pd, r_cnt);
      SF_LAUNCHED(ctx);
      SF_CUDA(cudaMemsetAsync(p_cnt + np - 1, 0, 8, st));
      player_list_count_kernel<<<dim3(blocks_for(n), lsegs), 256, 0, st>>>(mte, Wp, n, tiles_b, lsegs, p_cnt);
      SF_LAUNCHED(ctx);
      if (dt.on) {
        SF_CUDA(cudaStreamSynchronize(st));
        dt.lap("lists: counts");
      }
      size_t tb = tmp;
      SF_CUDA(cub::DeviceScan::ExclusiveSum(tmp_buf, tb, r_cnt, r_off, nr, st));
      tb = tmp;
      SF_CUDA(cub::DeviceScan::ExclusiveSum(tmp_buf, tb, p_cnt, p_off, np, st));
      if (dt.on) {
        SF_CUDA(cudaStreamSynchronize(st));
        dt.lap("lists: scans");
      }
      row_list_fill_kernel<<<blocks_for(pd * 32), 256, 0, st>>>(in.dev_rows, W, pair_step, pd, r_off, r_idx);
      SF_LAUNCHED(ctx);
      player_list_fill_kernel<<<dim3(blocks_for(n), lsegs), 256, 0, st>>>(mte, Wp, n, tiles_b, lsegs, p_off,
                                                                         p_idx);
      SF_LAUNCHED(ctx);
      row_off = r_off;
      row_idx = r_idx;
      pl_off = p_off;
      pl_idx = p_idx;
    }
  }
  if (lists) {
    SF_CUDA(cudaStreamSynchronize(st));
    dt.lap("lists");
  }
  const uint64_t rows_b = lists ? 0 : 2 * pd;
  const uint64_t lblocks = lists ? (pd + 63) / 64 : 0;
  // Load balance (rows are ordered by coalition size, so uniform splits put
  // every dense row in the last blocks): forward row blocks and transpose
  // tile splits of the set-bit part are cut at equal cumulative set-bit
  // cost, once per solve.
  std::vector<uint32_t> bounds{0};
  if (rows_b) {
    const uint64_t wcost = (W + 31) / 32 * 4 + 16;  // word loads + row overhead per needed row
    uint64_t total = 0;
    for (uint64_t i = 0; i < rows_b; ++i) total += needed(i) ? h_pop[i] + wcost : 1;
    const uint64_t target = std::max<uint64_t>(1, total / (4ull * sms));
    uint64_t acc = 0;
    for (uint64_t i = 0; i < rows_b; i += 2) {
      acc += (needed(i) ? h_pop[i] + wcost : 1) + (needed(i + 1) ? h_pop[i + 1] + wcost : 1);
      const uint64_t cur = i + 2 - bounds.back();
      if (acc >= target || cur >= kFwdRows) {
        bounds.push_back(uint32_t(i + 2));
        acc = 0;
      }
    }
    if (bounds.back() != rows_b) bounds.push_back(uint32_t(rows_b));
  }
  const uint64_t fblocks = bounds.size() - 1;
  std::vector<uint32_t> sbounds{0};
  if (tiles_b && !lists) {
    std::vector<uint64_t> tcost(tiles_b, (any_noncomp ? 2 : 1) * (n / 8 + 64));
    for (uint64_t i = 0; i < std::min(rows, tiles_b * 128); ++i)
      if (needed(i)) tcost[i / 128] += h_pop[i];
    uint64_t total = 0;
    for (uint64_t c : tcost) total += c;
    const uint64_t target = std::max<uint64_t>(1, (total + max_splits - 1) / max_splits);
    uint64_t acc = 0;
    for (uint64_t t = 0; t < tiles_b; ++t) {
      acc += tcost[t];
      if (acc >= target && sbounds.size() < max_splits) {
        sbounds.push_back(uint32_t(t + 1));
        acc = 0;
      }
    }
    if (sbounds.back() != tiles_b) sbounds.push_back(uint32_t(tiles_b));
  }
  const uint32_t splits = uint32_t(sbounds.size() - 1);
  // nibble part: uniform tile splits (every dense tile costs the same)
  std::vector<uint32_t> nbounds{uint32_t(tiles_b)};
  if (ptiles > tiles_b && i8) {
    // i8 passes: split boundaries on whole digit groups (4 tiles)
    const uint64_t nt = ptiles - tiles_b;
    uint64_t ns = std::max<uint64_t>((2ull * sms + i8_pb - 1) / i8_pb, (nt + 16383) / 16384);
    ns = std::max<uint64_t>(1, std::min<uint64_t>({ns, max_nsplits, (nt + 15) / 16}));
    for (uint64_t k = 1; k < ns; ++k) {
      const uint64_t b = (tiles_b + nt * k / ns) & ~uint64_t(3);
      if (b > nbounds.back()) nbounds.push_back(uint32_t(b));
    }
    nbounds.push_back(uint32_t(ptiles));
  } else if (ptiles > tiles_b) {
    const uint64_t nt = ptiles - tiles_b;
    const uint64_t ns = std::max<uint64_t>(1, std::min<uint64_t>(max_nsplits, (nt + kNbTT - 1) / kNbTT));
    for (uint64_t k = 1; k <= ns; ++k) nbounds.push_back(uint32_t(tiles_b + nt * k / ns));
  }
  const uint32_t nsplits = uint32_t(nbounds.size() - 1);
  const uint64_t nb_rowblocks = (pairs_n + 255) / 256;
  const uint32_t nb_parts = uint32_t(std::max<uint64_t>(
      1, std::min<uint64_t>({uint64_t(nb_parts_max), nib_ctas,
                             (nib_ctas + nb_rowblocks - 1) / std::max<uint64_t>(nb_rowblocks, 1)})));
  const uint32_t nb_part_players = uint32_t(((uint64_t(n) + nb_parts - 1) / nb_parts + 63) / 64 * 64);
  // i8 forward: parts of the word axis (whole digit groups, <= 16384 words)
  // so that >= 2 items per SM
  uint32_t i8_parts = 1, i8_part_words = ((W + 3) / 4) * 4;
  if (i8 && pairs_n) {
    const uint64_t lb = (pairs_n + 127) / 128;
    uint64_t parts = std::max<uint64_t>((2ull * sms + lb - 1) / lb, (W + 16383) / 16384);
    parts = std::max<uint64_t>(1, std::min<uint64_t>(parts, nb_parts_max));
    i8_part_words = uint32_t(((W + parts - 1) / parts + 3) / 4 * 4);
    i8_parts = uint32_t((W + i8_part_words - 1) / i8_part_words);
  }
  const uint64_t pstride = nb_rowblocks * 256;
  uint64_t* rT = nullptr;
  // rT in the caller's rows buffer when it may be overwritten and nothing
  // reads the rows during the iterations (kept-set lists on the sparse
  // pairs, the row lists already built): saves W x pstride words (C4: the
  // dense pairs' share of the mask bytes)
  const bool rt_in_rows = pairs_n && lists && rows_b == 0 && pd % 64 == 0 &&
                          in.rows_scratch_words >= uint64_t(W) * pstride;
  if (rt_in_rows) {
    rT = const_cast<uint64_t*>(in.dev_rows);
    const uint64_t blocks = (pstride / 64) * W;
    tiles_word_major_kernel<<<unsigned((blocks + 7) / 8), 256, 0, st>>>(mte, Wp, W, tiles_b, ptiles, pstride, rT);
    SF_LAUNCHED(ctx);
  } else if (pairs_n) {
    ctx.solver_dense.reserve(uint64_t(W) * pstride);
    rT = ctx.solver_dense.p;
    rows_word_major_kernel<<<dim3((W + 31) / 32, unsigned(pstride / 32)), 256, 0, st>>>(in.dev_rows, W, pair_step, pd, pairs,
                                                                                      pstride, rT);
    SF_LAUNCHED(ctx);
  }
  if (pairs_n) {
    set_max_dynamic_smem(nib_forward_kernel<kNbChunk>, int(kNbChunk / 4 * 16 * 8));
    set_max_dynamic_smem(nib_forward_kernel<kNbChunk / 2>, int(kNbChunk / 8 * 16 * 8));
  }
  const uint32_t* row_start = d_bounds;
  const uint32_t* split_start = d_bounds + bounds.size();
  const uint32_t* nsplit_start = split_start + sbounds.size();
  SF_CUDA(cudaMemcpyAsync(d_bounds, bounds.data(), bounds.size() * 4, cudaMemcpyHostToDevice, st));
  SF_CUDA(cudaMemcpyAsync(d_bounds + bounds.size(), sbounds.data(), sbounds.size() * 4,
                          cudaMemcpyHostToDevice, st));
  SF_CUDA(cudaMemcpyAsync(d_bounds + bounds.size() + sbounds.size(), nbounds.data(), nbounds.size() * 4,
                          cudaMemcpyHostToDevice, st));
  ctx.h2d_bytes += (bounds.size() + sbounds.size() + nbounds.size()) * 4;
  SF_CUDA(cudaStreamSynchronize(st));
  const double scw = std::sqrt(in.constraint_weight);
  int rp_esw = 0, rp_logn = 0, rp_hu = 0, rp_hrows = 0;  // fixed-order bounds (set at init)
  double r_c = scw * in.constraint_target;

  // out = M^T (sw x) (+ the pair constants); x = r (reference protocol) or
  // v (fused mode, coefficients sw * v). Local: no collective here.
  auto coefs = [&](const double* x) {
    SF_CUDA(cudaMemsetAsync(kc, 0, std::max<uint64_t>(pairs, 1) * 8, st));
    if (pairs) {
      coef_kernel<<<blocks_for(ptiles * 64), 256, 0, st>>>(in.dev_sw, x, is_comp, pairs, ptiles * 64,
                                                          coef_e, coef_o, kc);
      SF_LAUNCHED(ctx);
    }
  };
  // out = sum over pairs of the coefficients on their set bits + *kconst
  // The sparse-pair list passes run on a side stream beside the dense-pair
  // passes (they write disjoint partials; SF_CGLS_OVERLAP=0 serialises).
  static const bool overlap_env = [] {
    const char* v = std::getenv("SF_CGLS_OVERLAP");
    return v == nullptr || std::strcmp(v, "0") != 0;
  }();
  auto ensure_side = [&]() {
    SideStream& sd = ctx.side;
    if (!sd.s) {
      SF_CUDA(cudaStreamCreateWithFlags(&sd.s, cudaStreamNonBlocking));
      SF_CUDA(cudaEventCreateWithFlags(&sd.fork, cudaEventDisableTiming));
      SF_CUDA(cudaEventCreateWithFlags(&sd.join, cudaEventDisableTiming));
    }
  };
  auto fork = [&]() {
    SideStream& sd = ctx.side;
    ensure_side();
    SF_CUDA(cudaEventRecord(sd.fork, st));
    SF_CUDA(cudaStreamWaitEvent(sd.s, sd.fork, 0));
    return sd.s;
  };
  auto join = [&]() {
    SF_CUDA(cudaEventRecord(ctx.side.join, ctx.side.s));
    SF_CUDA(cudaStreamWaitEvent(st, ctx.side.join, 0));
  };
  auto passes = [&](const double* ce, const double* co, const double* kconst, double* out) {
    if (splits) {
      dim3 grid(unsigned(pblocks), splits);
      transpose_partial_kernel<<<grid, 256, 0, st>>>(mte, Wp, n, split_start, ce, 0, s_part);
      SF_LAUNCHED(ctx);
      if (any_noncomp) {
        transpose_partial_kernel<<<grid, 256, 0, st>>>(mto, Wp, n, split_start, co, 1, s_part);
        SF_LAUNCHED(ctx);
      }
    }
    const bool ov = overlap_env && lists && nsplits;
    if (lists) {
      cudaStream_t ls = ov ? fork() : st;
      list_transpose_kernel<<<blocks_for(uint64_t(n) * 32), 256, 0, ls>>>(
          pl_off, pl_idx, n, lsegs, ce, s_part + uint64_t(splits + nsplits) * n);
      SF_LAUNCHED(ctx);
    }
    if (nsplits && i8) {
      launch_cgls_digits(ce, tiles_b * 64, ptiles * 64, i8_abs, i8_cdig, i8_exp + 1, st);
      SF_LAUNCHED(ctx);
      ctx.launches++;
      launch_bitmat_i8(mte, Wp, n, n, nsplits, nsplit_start, 0, uint32_t(ptiles), i8_cdig, i8_exp + 1,
                       s_part + uint64_t(splits) * n, n, sms, st);
      SF_LAUNCHED(ctx);
    } else if (nsplits) {
      // register-capped to 64 for 4 CTAs per SM (SF_NIB_T4=0: uncapped, 3)
      static const bool t4 = !(std::getenv("SF_NIB_T4") && std::atoi(std::getenv("SF_NIB_T4")) == 0);
      if (t4)
        nib_transpose_kernel<4><<<dim3(unsigned(nib_pblocks), nsplits), 256, 0, st>>>(
            mte, Wp, n, ptiles, nsplit_start, ce, s_part + uint64_t(splits) * n);
      else
        nib_transpose_kernel<1><<<dim3(unsigned(nib_pblocks), nsplits), 256, 0, st>>>(
            mte, Wp, n, ptiles, nsplit_start, ce, s_part + uint64_t(splits) * n);
      SF_LAUNCHED(ctx);
    }
    if (ov) join();
    transpose_finish_kernel<<<blocks_for(n), 256, 0, st>>>(s_part, splits + nsplits + (lists ? 1 : 0), n,
                                                           kconst, out);
    SF_LAUNCHED(ctx);
  };
  // out = M^T (sw x) (+ the pair constants); x = r (reference protocol) or
  // v (fused mode, coefficients sw * v). Local: no collective here.
  auto transpose_local = [&](const double* x, double* out) {
    coefs(x);
    reduce(kc, pairs, 0, 0.0, scal + 4);
    passes(coef_e, coef_o, scal + 4, out);
  };
  // fixed-order mode: the three level sums of M^T (sw r) and of the pair
  // constants into lev[0, 3n + 3), exact on every rank
  auto transpose_levels = [&](const double* x) {
    coefs(x);
    const uint64_t P = ptiles * 64;
    if (P) {
      split3_kernel<<<blocks_for(P), 256, 0, st>>>(coef_e, P, P, grids + 0, cel, P);
      SF_LAUNCHED(ctx);
      if (any_noncomp) {
        split3_kernel<<<blocks_for(P), 256, 0, st>>>(coef_o, P, P, grids + 0, col, P);
        SF_LAUNCHED(ctx);
      }
    }
    const uint64_t KP = std::max<uint64_t>(pairs, 1);
    split3_kernel<<<blocks_for(KP), 256, 0, st>>>(kc, pairs, KP, grids + 0, kcl, KP);
    SF_LAUNCHED(ctx);
    for (int k = 0; k < 3; ++k) {
      passes(cel + k * P, col + k * P, grids + 32, lev + uint64_t(k) * n);
      reduce(kcl + k * KP, pairs, 0, 0.0, lev + 3ull * n + k);
    }
  };
  // s = M^T (sw r) all-reduced, then the pin row (solver.cpp:226-248)
  // scalar fold over pair leaves d_j = x[2j]^2 + x[2j+1]^2 into *out
  auto tree_scalar = [&](const double* x, double* out) {
    pair_sq_kernel<<<blocks_for(tree_local), 256, 0, st>>>(x, pairs, tree_local, tleaf);
    SF_LAUNCHED(ctx);
    uint64_t h = tree_local;
    while (h > 2048) {
      h /= 2;
      fold_level_kernel<<<blocks_for(h), 256, 0, st>>>(tleaf, h);
      SF_LAUNCHED(ctx);
    }
    fold_small_kernel<<<1, 1024, 0, st>>>(tleaf, h, out);
    SF_LAUNCHED(ctx);
  };
  auto transpose_product = [&]() {
    if (tree) {
      tree_transpose_kernel<<<unsigned((n + 127) / 128), 128, 0, st>>>(mte, mto, Wp, n, pairs, is_comp, in.dev_sw, r,
                                                                       tree_local, tree_log, s);
      SF_LAUNCHED(ctx);
      comm_allreduce_sum(ctx, s, n);
      add_scalar_kernel<<<blocks_for(n), 256, 0, st>>>(s, scw * r_c, n);
      SF_LAUNCHED(ctx);
      return;
    }
    if (repro) {
      transpose_levels(r);
      comm_allreduce_sum(ctx, lev, 3ull * n + 3);
      combine_s_kernel<<<blocks_for(n), 256, 0, st>>>(lev, n, scw * r_c, s);
      SF_LAUNCHED(ctx);
      return;
    }
    transpose_local(r, s);
    comm_allreduce_sum(ctx, s, n);
    add_scalar_kernel<<<blocks_for(n), 256, 0, st>>>(s, scw * r_c, n);
    SF_LAUNCHED(ctx);
  };
  // v (set-bit rows [0, rows_b), nibble pairs [pd, pairs)) and the per-block
  // sums of v^2 in dsq[0, fwd_blocks)
  const uint64_t fwd_blocks = fblocks + lblocks + nb_rowblocks;
  auto forward_v = [&](const double* x, const double* swp, const double* sum_u, double* vout) {
    const bool ov = overlap_env && lblocks && nb_rowblocks;
    // 1024-player table chunks (32 KB: 4 CTAs per SM) unless SF_NIB_CHUNK=2048
    // (64 KB, 3 per SM); with the 4-CTA transpose: C2 solve 24.5 -> 23.4 ms
    static const bool nib_half = !(std::getenv("SF_NIB_CHUNK") && std::atoi(std::getenv("SF_NIB_CHUNK")) == 2048);
    if (lblocks) {
      cudaStream_t ls = ov ? fork() : st;
      list_forward_kernel<<<unsigned(lblocks), 256, 0, ls>>>(row_off, row_idx, pd, x, swp, sum_u, vout,
                                                              dsq + fblocks);
      SF_LAUNCHED(ctx);
    }
    if (fblocks) {
      forward_kernel<<<unsigned(fblocks), kFwdThreads, size_t(std::min<uint32_t>(n, kFwdChunk)) * 8, st>>>(
          in.dev_rows, W, row_start, is_comp, x, n, swp, sum_u, vout, dsq, in.kept_only ? 1 : 0);
      SF_LAUNCHED(ctx);
    }
    if (nb_rowblocks && i8) {
      launch_cgls_digits(x, 0, n, i8_abs, i8_udig, i8_exp, st);
      SF_LAUNCHED(ctx);
      ctx.launches++;
      launch_bitmat_i8(rT, pstride, pstride, pairs_n, i8_parts, nullptr, i8_part_words, W, i8_udig, i8_exp, vpart,
                       pairs_n, sms, st);
      SF_LAUNCHED(ctx);
      nib_forward_finish<<<unsigned(nb_rowblocks), 256, 0, st>>>(vpart, i8_parts, pd, pairs, swp, sum_u, vout,
                                                                   dsq + fblocks + lblocks);
      SF_LAUNCHED(ctx);
    } else if (nb_rowblocks) {
      if (nib_half)
        nib_forward_kernel<kNbChunk / 2><<<dim3(unsigned(nb_rowblocks), nb_parts), 256, kNbChunk / 8 * 16 * 8, st>>>(
            rT, pstride, pairs_n, x, n, nb_part_players, vpart);
      else
        nib_forward_kernel<kNbChunk><<<dim3(unsigned(nb_rowblocks), nb_parts), 256, kNbChunk / 4 * 16 * 8, st>>>(
            rT, pstride, pairs_n, x, n, nb_part_players, vpart);
      SF_LAUNCHED(ctx);
      nib_forward_finish<<<unsigned(nb_rowblocks), 256, 0, st>>>(vpart, nb_parts, pd, pairs, swp,
                                                                   sum_u, vout, dsq + fblocks + lblocks);
      SF_LAUNCHED(ctx);
    }
    if (ov) join();
  };
  set_max_dynamic_smem(forward_kernel, int(kFwdChunk * 8));
  // v = sqrt(W) M u; delta = ||v||^2 all-reduced + v_c^2 (solver.cpp:252-287)
  auto forward_product = [&](double& delta, double& v_c) {
    if (tree) {
      reduce(u, n, 0, 0.0, scal + 0);  // sum_u
      if (rows) forward_v(u, in.dev_sw, scal + 0, v);
      tree_scalar(v, scal + 1);
      comm_allreduce_sum(ctx, scal + 1, 1);
      fetch(0, 2);
      delta = host[1];
      v_c = scw * host[0];
      delta += v_c * v_c;
      return;
    }
    if (repro) {
      // parts of u on a grid from max|u| (u is replicated: same grid on
      // every rank), exact per-level row dots, v = sw ((V0 + V1) + V2),
      // delta from the parts of v^2
      reduce(u, n, 0, 0.0, scal + 0);  // sum_u for the pin row
      absmax_kernel<<<1, 1024, 0, st>>>(u, nullptr, n, grids + 40);
      SF_LAUNCHED(ctx);
      iter_grids_kernel<<<1, 1, 0, st>>>(grids + 40, rp_esw, rp_logn, rp_hu, rp_hrows, grids + 8, grids + 16);
      SF_LAUNCHED(ctx);
      split3_kernel<<<blocks_for(n), 256, 0, st>>>(u, n, n, grids + 8, ul, n);
      SF_LAUNCHED(ctx);
      for (int k = 0; k < 3; ++k) reduce(ul + uint64_t(k) * n, n, 0, 0.0, ul + 3ull * n + k);
      if (rows) {
        for (int k = 0; k < 3; ++k) forward_v(ul + uint64_t(k) * n, ones, ul + 3ull * n + k, vl + k * rows);
        combine_v_kernel<<<blocks_for(rows), 256, 0, st>>>(vl, rows, in.dev_sw, grids + 16, v, dparts);
        SF_LAUNCHED(ctx);
      }
      for (int k = 0; k < 3; ++k) reduce(dparts + k * rows, rows, 0, 0.0, grids + 48 + k);
      comm_allreduce_sum(ctx, grids + 48, 3);
      ctx.d2h_bytes += 4 * sizeof(double);
      SF_CUDA(cudaMemcpyAsync(host + 12, grids + 48, 3 * sizeof(double), cudaMemcpyDeviceToHost, st));
      fetch(0, 1);
      delta = (host[12] + host[13]) + host[14];
      v_c = scw * host[0];
      delta += v_c * v_c;
      return;
    }
    reduce(u, n, 0, 0.0, scal + 0);  // sum_u
    if (rows) forward_v(u, in.dev_sw, scal + 0, v);
    reduce(dsq, rows ? fwd_blocks : 0, 0, 0.0, scal + 1);
    comm_allreduce_sum(ctx, scal + 1, 1);
    fetch(0, 2);
    delta = host[1];
    v_c = scw * host[0];
    delta += v_c * v_c;
  };

  SF_CUDA(cudaStreamSynchronize(st));
  dt.lap("setup");
  SF_CUDA(cudaMemsetAsync(phi, 0, uint64_t(n) * 8, st));
  if (repro) {
    // Global bounds, identical on every rank: exponent flags of max |sw t|
    // and max sw plus the global pair count, summed over ranks (one extra
    // vector all-reduce at init; flags are 0/1 so the sum is exact).
    absmax_kernel<<<1, 1024, 0, st>>>(in.dev_sw, in.dev_targets, rows, grids + 40);
    SF_LAUNCHED(ctx);
    absmax_kernel<<<1, 1024, 0, st>>>(in.dev_sw, nullptr, rows, grids + 41);
    SF_LAUNCHED(ctx);
    SF_CUDA(cudaMemcpyAsync(host + 12, grids + 40, 2 * sizeof(double), cudaMemcpyDeviceToHost, st));
    SF_CUDA(cudaStreamSynchronize(st));
    std::vector<double> fl(2 * kBins + 1, 0.0);
    for (int q = 0; q < 2; ++q) {
      if (host[12 + q] > 0.0 && std::isfinite(host[12 + q])) {
        int e = 0;
        std::frexp(host[12 + q], &e);
        fl[q * kBins + std::clamp(e + 1100, 0, kBins - 1)] = 1.0;
      }
    }
    fl[2 * kBins] = double(pairs);
    SF_CUDA(cudaMemcpyAsync(flags, fl.data(), fl.size() * 8, cudaMemcpyHostToDevice, st));
    comm_allreduce_sum(ctx, flags, fl.size());
    SF_CUDA(cudaMemcpyAsync(fl.data(), flags, fl.size() * 8, cudaMemcpyDeviceToHost, st));
    comm_sync(ctx);
    ctx.h2d_bytes += fl.size() * 8;
    ctx.d2h_bytes += fl.size() * 8;
    auto top = [&](int q) {
      for (int b = kBins - 1; b >= 0; --b)
        if (fl[q * kBins + b] != 0.0) return b - 1100;
      return -1000;
    };
    const int e_b = top(0);  // max |sw t| < 2^e_b
    rp_esw = top(1);         // max sw < 2^rp_esw
    const double gpairs = fl[2 * kBins];
    const double grows = 2.0 * gpairs;
    auto clog2 = [](double x) { return int(std::ceil(std::log2(std::max(x, 1.0)))); };
    // ||[r; r_c]|| never exceeds its start (CGLS minimises it): |r_i| <= R
    const double rc0 = std::fabs(scw * in.constraint_target);
    const double R = 2.0 * std::sqrt(grows * std::ldexp(1.0, 2 * e_b) + rc0 * rc0);
    int e_r = 0;
    std::frexp(R, &e_r);
    const int h_pairs = clog2(gpairs + 1) + 1;
    rp_hrows = clog2(grows + 1) + 1;
    rp_logn = clog2(double(n) + 1);
    rp_hu = rp_logn + 2;
    // pair coefficients: |c_e - c_o| <= 2 max sw R
    double g[3];
    auto host_grid = [&](int E, int H) {
      g[0] = std::ldexp(1.0, E + H - 52);
      g[1] = std::ldexp(g[0], H - 53);
      g[2] = std::ldexp(g[1], H - 53);
    };
    host_grid(rp_esw + 1 + e_r, h_pairs);
    SF_CUDA(cudaMemcpyAsync(grids + 0, g, 3 * sizeof(double), cudaMemcpyHostToDevice, st));
    host_grid(2 * e_r, rp_hrows);  // r^2 for the trace
    SF_CUDA(cudaMemcpyAsync(grids + 24, g, 3 * sizeof(double), cudaMemcpyHostToDevice, st));
    SF_CUDA(cudaMemsetAsync(grids + 32, 0, sizeof(double), st));
    if (rows) {
      fill_kernel<<<blocks_for(rows), 256, 0, st>>>(ones, 1.0, rows);
      SF_LAUNCHED(ctx);
    }
    SF_CUDA(cudaStreamSynchronize(st));
  }
  transpose_product();
  reduce(s, n, 1, 0.0, scal + 2);                // gamma = ||s||^2
  reduce(s, n, 2, scw * r_c, scal + 6);          // data0 = ||s - pin||^2
  fetch(2, 5);
  double gamma = host[2];
  const double gamma0 = gamma;
  const double data0 = host[6];
  auto download_phi = [&]() {
    ctx.d2h_bytes += uint64_t(n) * 8;
    res.phi.resize(n);
    SF_CUDA(cudaMemcpyAsync(res.phi.data(), phi, uint64_t(n) * 8, cudaMemcpyDeviceToHost, st));
    SF_CUDA(cudaStreamSynchronize(st));
  };
  if (gamma0 == 0.0) {
    res.converged = true;
    download_phi();
    return res;
  }
  const double reference = data0 > 0.0 ? data0 : gamma0;
  res.relative_residual = std::sqrt(gamma0 / reference);
  SF_CUDA(cudaMemcpyAsync(u, s, uint64_t(n) * 8, cudaMemcpyDeviceToDevice, st));
  const double blowup = 1.0e12 * std::max(res.relative_residual, 1.0);
  const uint64_t maxit = max_iter ? max_iter : std::min<uint64_t>(n, 5000);
  if (mode == 1) {
    // Fused protocol: per iteration one (n+1)-double
    // all-reduce of [A^T v ; ||v||^2]; s follows the recurrence
    // s <- s - theta A^T A u instead of s = A^T r (same math, different
    // rounding; r is not formed). Stop rule and error semantics unchanged.
    // Residual replacement every `every` iterations: the exact gradient
    // A^T r(phi) (r = sqrt(W)(t - M phi), pin row sqrt(cw)(ct - sum phi))
    // rides in the same all-reduce, so the recurrence's drift stays
    // bounded and the collective count stays one per iteration.
    static const uint64_t every =
        std::getenv("SF_CGLS_RECOMPUTE") ? std::strtoull(std::getenv("SF_CGLS_RECOMPUTE"), nullptr, 10) : 10;
    while (res.iterations < maxit) {
      const bool exact = every && res.iterations > 0 && res.iterations % every == 0;
      if (exact) {
        reduce(phi, n, 0, 0.0, scal + 13);  // sum phi
        if (rows) {
          forward_v(phi, in.dev_sw, scal + 13, vphi);
          residual_kernel<<<blocks_for(rows), 256, 0, st>>>(r, vphi, rows);  // vphi <- sw t - sw M phi
          SF_LAUNCHED(ctx);
          transpose_local(vphi, tv + n + 1);
        } else {
          SF_CUDA(cudaMemsetAsync(tv + n + 1, 0, uint64_t(n) * 8, st));
        }
      }
      reduce(u, n, 0, 0.0, scal + 0);  // sum_u (pin row: v_c = scw sum_u)
      if (rows) {
        forward_v(u, in.dev_sw, scal + 0, v);
        transpose_local(v, tv);
      } else {
        SF_CUDA(cudaMemsetAsync(tv, 0, uint64_t(n) * 8, st));
      }
      reduce(dsq, rows ? fwd_blocks : 0, 0, 0.0, tv + n);
      comm_allreduce_sum(ctx, tv, exact ? 2ull * n + 1 : uint64_t(n) + 1);
      if (exact) {
        fetch(13, 1);
        r_c = scw * in.constraint_target - scw * host[13];
        // s <- exact gradient at phi (+ the pin row); the step below then
        // applies -theta (A^T v + scw v_c) as usual
        SF_CUDA(cudaMemcpyAsync(s, tv + n + 1, uint64_t(n) * 8, cudaMemcpyDeviceToDevice, st));
        add_scalar_kernel<<<blocks_for(n), 256, 0, st>>>(s, scw * r_c, n);
        SF_LAUNCHED(ctx);
      }
      fetch(0, 1);
      SF_CUDA(cudaMemcpyAsync(host + 1, tv + n, sizeof(double), cudaMemcpyDeviceToHost, st));
      comm_sync(ctx);
      ctx.d2h_bytes += sizeof(double);
      const double v_c = scw * host[0];
      const double delta = host[1] + v_c * v_c;
      if (!std::isfinite(delta))
        throw NumericalError("iterative solve diverged at iteration " +
                             std::to_string(res.iterations) + ": non-finite step norm");
      if (delta <= 0.0) break;
      const double theta = gamma / delta;
      host[8] = gamma;
      host[9] = delta;
      SF_CUDA(cudaMemcpyAsync(scal + 8, host + 8, 2 * sizeof(double), cudaMemcpyHostToDevice, st));
      axpy_kernel<<<blocks_for(n), 256, 0, st>>>(phi, u, scal + 8, scal + 9, 1.0, n);
      SF_LAUNCHED(ctx);
      // s -= theta (A^T v + scw v_c)
      add_scalar_kernel<<<blocks_for(n), 256, 0, st>>>(tv, scw * v_c, n);
      SF_LAUNCHED(ctx);
      axpy_kernel<<<blocks_for(n), 256, 0, st>>>(s, tv, scal + 8, scal + 9, -1.0, n);
      SF_LAUNCHED(ctx);
      r_c -= theta * v_c;
      reduce(s, n, 1, 0.0, scal + 3);
      fetch(3, 1);
      const double gamma_next = host[3];
      ++res.iterations;
      res.relative_residual = std::sqrt(gamma_next / reference);
      if (trace) res.trace.push_back(res.relative_residual);
      if (!std::isfinite(gamma_next) || res.relative_residual > blowup)
        throw NumericalError("iterative solve diverged at iteration " +
                             std::to_string(res.iterations) + ": residual exploded");
      if (res.relative_residual <= tol) {
        res.converged = true;
        break;
      }
      host[10] = gamma_next;
      host[11] = gamma;
      SF_CUDA(cudaMemcpyAsync(scal + 10, host + 10, 2 * sizeof(double), cudaMemcpyHostToDevice, st));
      direction_kernel<<<blocks_for(n), 256, 0, st>>>(u, s, scal + 10, scal + 11, n);
      SF_LAUNCHED(ctx);
      gamma = gamma_next;
    }
    download_phi();
    return res;
  }
  DebugTimer di("cgls iteration");
  if (!trace && !repro && !tree) {
    // One host round trip per iteration: delta, theta, r_c and beta stay on
    // the device; the host reads (delta, stop flag, gamma_next) once after
    // the transpose and applies the reference's stop rule and error
    // semantics. A stopped step (delta <= 0 or non-finite) leaves phi and
    // r untouched, like the reference's break before the update.
    host[7] = r_c;
    SF_CUDA(cudaMemcpyAsync(scal + 7, host + 7, sizeof(double), cudaMemcpyHostToDevice, st));
    // gamma in scal[2] (from the init reduce), gamma_next in scal[3]; the
    // step kernel moves gamma_next into gamma at the start of an iteration
    constexpr int g = 2, gn = 3;
    SF_CUDA(cudaMemcpyAsync(scal + gn, scal + g, sizeof(double), cudaMemcpyDeviceToDevice, st));
    auto body = [&]() {
      reduce(u, n, 0, 0.0, scal + 0);  // sum_u
      if (rows) forward_v(u, in.dev_sw, scal + 0, v);
      reduce(dsq, rows ? fwd_blocks : 0, 0, 0.0, scal + 1);
      comm_allreduce_sum(ctx, scal + 1, 1);
      step_kernel<<<1, 1, 0, st>>>(scal, scw, g, gn);
      SF_LAUNCHED(ctx);
      axpy_stop_kernel<<<blocks_for(n), 256, 0, st>>>(phi, u, scal, 1.0, n);
      SF_LAUNCHED(ctx);
      if (rows) {
        axpy_stop_kernel<<<blocks_for(rows), 256, 0, st>>>(r, v, scal, -1.0, rows);
        SF_LAUNCHED(ctx);
      }
      transpose_local(r, s);
      comm_allreduce_sum(ctx, s, n);
      add_pin_kernel<<<blocks_for(n), 256, 0, st>>>(s, scw, scal + 7, n);
      SF_LAUNCHED(ctx);
      reduce(s, n, 1, 0.0, scal + gn);  // gamma_next
      direction_kernel<<<blocks_for(n), 256, 0, st>>>(u, s, scal + gn, scal + g, n);
      SF_LAUNCHED(ctx);
      ctx.d2h_bytes += 16 * sizeof(double);
      SF_CUDA(cudaMemcpyAsync(host, scal, 16 * sizeof(double), cudaMemcpyDeviceToHost, st));
    };
    // One worker, no host communicator, not one of several concurrent
    // explain workers: the iteration body is captured once as a CUDA graph
    // and replayed — one graph launch instead of ~15 kernel launches per
    // iteration (C1 solve 2.8 -> 2.2 ms). Concurrent workers launch the
    // kernels directly (their short solves do not repay the capture, and
    // instantiation contends across threads: C5 -34% with graphs).
    // SF_CGLS_GRAPH=0 disables it.
    static const bool graphs_env = [] {
      const char* e = std::getenv("SF_CGLS_GRAPH");
      return e == nullptr || std::strcmp(e, "0") != 0;
    }();
    bool graph_ok = graphs_env && ctx.world == 1 && ctx.host_comm.all_reduce == nullptr && !i8 &&
                    !ctx.concurrent && maxit - res.iterations >= 3;
    struct GraphExec {
      cudaGraphExec_t e = nullptr;
      ~GraphExec() {
        if (e) cudaGraphExecDestroy(e);
      }
    } gexec;
    uint64_t glaunches = 0, gd2h = 0;
    CommStats gstats;
    if (graph_ok) {
      if (lists && overlap_env) ensure_side();
      const uint64_t l0 = ctx.launches, d0 = ctx.d2h_bytes;
      const CommStats s0 = ctx.stats;
      // a capture or instantiation failure falls back to direct launches
      // (nothing of the body has run: captured work is only recorded)
      cudaGraph_t gr = nullptr;
      bool captured = cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal) == cudaSuccess;
      if (captured) {
        try {
          body();
        } catch (...) {
          captured = false;
        }
        if (cudaStreamEndCapture(st, &gr) != cudaSuccess) captured = false;
        if (captured && gr && cudaGraphInstantiate(&gexec.e, gr, 0) != cudaSuccess) {
          gexec.e = nullptr;
          captured = false;
        }
        if (gr) cudaGraphDestroy(gr);
      }
      if (!captured || !gexec.e) {
        cudaGetLastError();  // clear the capture error
        if (gexec.e) cudaGraphExecDestroy(gexec.e);
        gexec.e = nullptr;
        graph_ok = false;
      }
      glaunches = ctx.launches - l0;
      gd2h = ctx.d2h_bytes - d0;
      gstats.scalar_allreduce = ctx.stats.scalar_allreduce - s0.scalar_allreduce;
      gstats.vector_allreduce = ctx.stats.vector_allreduce - s0.vector_allreduce;
      gstats.doubles_reduced = ctx.stats.doubles_reduced - s0.doubles_reduced;
      ctx.launches = l0;
      ctx.d2h_bytes = d0;
      ctx.stats = s0;
    }
    while (res.iterations < maxit) {
      if (graph_ok) {
        SF_CUDA(cudaGraphLaunch(gexec.e, st));
        ctx.launches += glaunches;
        ctx.d2h_bytes += gd2h;
        ctx.stats.scalar_allreduce += gstats.scalar_allreduce;
        ctx.stats.vector_allreduce += gstats.vector_allreduce;
        ctx.stats.doubles_reduced += gstats.doubles_reduced;
      } else {
        body();
      }
      comm_sync(ctx);
      if (host[12] == 2.0)
        throw NumericalError("iterative solve diverged at iteration " + std::to_string(res.iterations) +
                             ": non-finite step norm");
      if (host[12] == 1.0) break;
      const double gamma_next = host[gn];
      ++res.iterations;
      res.relative_residual = std::sqrt(gamma_next / reference);
      if (!std::isfinite(gamma_next) || res.relative_residual > blowup)
        throw NumericalError("iterative solve diverged at iteration " + std::to_string(res.iterations) +
                             ": residual exploded");
      if (res.relative_residual <= tol) {
        res.converged = true;
        break;
      }
      di.lap("");
    }
    download_phi();
    return res;
  }
  while (res.iterations < maxit) {
    di.lap("");
    double delta = 0.0, v_c = 0.0;
    forward_product(delta, v_c);
    if (!std::isfinite(delta))
      throw NumericalError("iterative solve diverged at iteration " +
                           std::to_string(res.iterations) + ": non-finite step norm");
    if (delta <= 0.0) break;
    const double theta = gamma / delta;
    host[8] = gamma;
    host[9] = delta;
    // theta on device: write (gamma, delta) into scal[8..9]
    SF_CUDA(cudaMemcpyAsync(scal + 8, host + 8, 2 * sizeof(double), cudaMemcpyHostToDevice, st));
    axpy_kernel<<<blocks_for(n), 256, 0, st>>>(phi, u, scal + 8, scal + 9, 1.0, n);
    SF_LAUNCHED(ctx);
    if (rows) {
      axpy_kernel<<<blocks_for(rows), 256, 0, st>>>(r, v, scal + 8, scal + 9, -1.0, rows);
      SF_LAUNCHED(ctx);
    }
    r_c -= theta * v_c;
    if (trace && tree) {
      tree_scalar(r, scal + 5);
      comm_allreduce_sum(ctx, scal + 5, 1);
      fetch(5, 1);
      res.row_residual_trace.push_back(std::sqrt(host[5] + r_c * r_c));
    } else if (trace && repro) {
      sq_parts_kernel<<<blocks_for(std::max<uint64_t>(rows, 1)), 256, 0, st>>>(r, rows, grids + 24, dparts);
      SF_LAUNCHED(ctx);
      for (int k = 0; k < 3; ++k) reduce(dparts + k * rows, rows, 0, 0.0, grids + 48 + k);
      comm_allreduce_sum(ctx, grids + 48, 3);
      SF_CUDA(cudaMemcpyAsync(host + 12, grids + 48, 3 * sizeof(double), cudaMemcpyDeviceToHost, st));
      comm_sync(ctx);
      res.row_residual_trace.push_back(std::sqrt(((host[12] + host[13]) + host[14]) + r_c * r_c));
    } else if (trace) {
      reduce(r, rows, 1, 0.0, scal + 5);
      comm_allreduce_sum(ctx, scal + 5, 1);
      fetch(5, 1);
      res.row_residual_trace.push_back(std::sqrt(host[5] + r_c * r_c));
    }
    transpose_product();
    reduce(s, n, 1, 0.0, scal + 3);
    fetch(3, 1);
    const double gamma_next = host[3];
    ++res.iterations;
    res.relative_residual = std::sqrt(gamma_next / reference);
    if (trace) res.trace.push_back(res.relative_residual);
    if (!std::isfinite(gamma_next) || res.relative_residual > blowup)
      throw NumericalError("iterative solve diverged at iteration " +
                           std::to_string(res.iterations) + ": residual exploded");
    if (res.relative_residual <= tol) {
      res.converged = true;
      break;
    }
    host[10] = gamma_next;
    host[11] = gamma;
    SF_CUDA(cudaMemcpyAsync(scal + 10, host + 10, 2 * sizeof(double), cudaMemcpyHostToDevice, st));
    direction_kernel<<<blocks_for(n), 256, 0, st>>>(u, s, scal + 10, scal + 11, n);
    SF_LAUNCHED(ctx);
    gamma = gamma_next;
  }
  download_phi();
  return res;
}

// solver.cpp:430-440: a stable LSD radix sort of the keys over the index
// order gives phi descending with ties by ascending index. NaN never gets
// here (the solver rejects non-finite values).
std::vector<uint32_t> rank_players(Ctx& ctx, const std::vector<double>& phi) {
  const uint32_t n = uint32_t(phi.size());
  std::vector<uint32_t> out(n);
  if (n == 0) return out;
  size_t tmp = 0;
  SF_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tmp, static_cast<const uint64_t*>(nullptr),
                                          static_cast<uint64_t*>(nullptr), static_cast<const uint32_t*>(nullptr),
                                          static_cast<uint32_t*>(nullptr), n, 0, 64, ctx.stream));
  ctx.rank_work.reserve(uint64_t(n) * (8 + 8 + 8 + 4 + 4) + tmp + 5 * 256);
  Scratch sc{ctx.rank_work.p, 0};
  double* d_phi = sc.take<double>(n);
  uint64_t* k0 = sc.take<uint64_t>(n);
  uint64_t* k1 = sc.take<uint64_t>(n);
  uint32_t* i0 = sc.take<uint32_t>(n);
  uint32_t* i1 = sc.take<uint32_t>(n);
  void* t = sc.take<unsigned char>(tmp);
  cudaStream_t st = ctx.stream;
  SF_CUDA(cudaMemcpyAsync(d_phi, phi.data(), uint64_t(n) * 8, cudaMemcpyHostToDevice, st));
  ctx.h2d_bytes += uint64_t(n) * 8;
  rank_keys_kernel<<<blocks_for(n), 256, 0, st>>>(d_phi, n, k0, i0);
  SF_LAUNCHED(ctx);
  SF_CUDA(cub::DeviceRadixSort::SortPairs(t, tmp, k0, k1, i0, i1, n, 0, 64, st));
  SF_CUDA(cudaMemcpyAsync(out.data(), i1, uint64_t(n) * 4, cudaMemcpyDeviceToHost, st));
  ctx.d2h_bytes += uint64_t(n) * 4;
  SF_CUDA(cudaStreamSynchronize(st));
  return out;
}

}  // namespace sfb
