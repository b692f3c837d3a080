// Direct weighted least squares on the device (solve_direct, solver.cpp:364-428):
// the Gram matrix G = M^T W M + cw 1 1^T on the tensor cores, then a blocked
// FP64 Cholesky and two triangular solves. No host arithmetic.
//
// Gram (gram_tc_kernel). Rows come in runs of equal weight (explain_node:
// one run per size class, both rows of a complement pair share the class
// weight w_s = w_{n-s}; solve_direct on caller rows: runs of equal weight).
// Within a run, G_run = w * (M_run^T M_run) and M_run^T M_run is an integer
// count matrix, so the 0/1 bits go through tcgen05.mma kind::f16 exactly
// (0/1 are exact in f16, FP32 accumulation is exact below 2^24 rows) and
// every run is folded into an FP64 tile accumulator in shared memory:
// G_tile += w * C_run. Only the run boundaries touch FP64; the rows never do.
// Operands are expanded from the tile-transposed mask words (one u64 per
// player per 64 rows) straight into the canonical K-major no-swizzle layout.
// Output tiles are 128 x 128 players (lower triangle of tiles); when there
// are few tiles the row axis is split across CTAs (deterministic: per-split
// FP64 partials summed in split order).
//
// Cholesky: right-looking, 64 x 64 blocks, lower, row-major, padded to a
// multiple of 128 with an identity tail. Per block column: the diagonal
// block in one CTA (shared memory), the panel below it (one CTA per block
// row, triangular solve against the diagonal block), the trailing update of
// the lower blocks (FP64 FMA tiles). A non-positive or non-finite pivot is
// reported with its index; the host then adds the reference's jitter
// (1e-10 trace / n, solver.cpp:398-400) and factors once more.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <vector>

#include "sf_internal.hpp"
#include "sf_tcgen05.cuh"

namespace sfb {

namespace {

using namespace tc;

constexpr int kGT = 128;         // players per output tile side
constexpr int kGThreads = 256;
constexpr int kOpBytes = kGT * 64 * 2;  // one operand: 128 players x 64 rows, f16
constexpr int kGSmem = 2 * 2 * kOpBytes + kGT * kGT * 8 + 64;
constexpr int kCB = 64;  // Cholesky block

__device__ __forceinline__ void mma_f16_ss(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                           uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}

// 8 bits -> 8 f16 (0 or 1.0 = 0x3C00), packed into 16 bytes
__device__ __forceinline__ uint4 expand8(uint32_t b) {
  uint32_t v[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const uint32_t lo = ((b >> (2 * i)) & 1u) * 0x3C00u;
    const uint32_t hi = ((b >> (2 * i + 1)) & 1u) * 0x3C00u;
    v[i] = lo | (hi << 16);
  }
  return make_uint4(v[0], v[1], v[2], v[3]);
}

// Work entry: rows [lo, hi) of 64-row tile t, weight run `run`; flag bit 0 =
// last entry of its run inside this split (fold into FP64 after it).
struct GramEntry {
  uint32_t tile;
  uint32_t lo, hi;
  uint32_t run_and_flag;
};

__global__ void __launch_bounds__(kGThreads, 1)
    gram_tc_kernel(const uint64_t* __restrict__ maskt, uint64_t Wp, uint32_t n, uint32_t T,
                   const GramEntry* __restrict__ ent, const uint32_t* __restrict__ split_start,
                   const double* __restrict__ run_w, double* __restrict__ Gp, uint64_t Np) {
  extern __shared__ __align__(1024) unsigned char smem[];
  unsigned char* ops = smem;                                         // [2 buf][A|B]
  double* acc = reinterpret_cast<double*>(smem + 4 * kOpBytes);      // [n][m] column-major
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + 4 * kOpBytes + kGT * kGT * 8);
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 2);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  // lower-triangular tile pair (ta >= tb) from blockIdx.x
  uint32_t ta = 0, rem = blockIdx.x;
  while (rem > ta) {
    rem -= ta + 1;
    ++ta;
  }
  const uint32_t tb = rem;
  const uint32_t e0 = split_start[blockIdx.y], e1 = split_start[blockIdx.y + 1];

  if (tid == 0) {
    mbar_init(&bars[0], 1);
    mbar_init(&bars[1], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  for (int i = tid; i < kGT * kGT; i += kGThreads) acc[i] = 0.0;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(su32(tmem_slot)),
                 "r"(128));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  // kind::f16: D f32, A/B f16, both K-major, N = 128, M = 128
  const uint32_t idesc = (1u << 4) | (uint32_t(kGT >> 3) << 17) | (uint32_t(kGT >> 4) << 24);
  constexpr uint32_t kLBO = (kGT / 8) * 128;  // k-unit (8 f16) stride
  // staging role: thread -> (operand, player)
  const int op = tid >> 7, p = tid & 127;
  const uint32_t player = (op == 0 ? ta : tb) * kGT + p;
  uint32_t uses[2] = {0, 0};
  uint32_t accumulate = 0;
  for (uint32_t e = e0; e < e1; ++e) {
    const GramEntry en = ent[e];
    const int buf = (e - e0) & 1;
    unsigned char* A = ops + buf * 2 * kOpBytes;
    if (uses[buf]) mbar_wait(&bars[buf], (uses[buf] - 1) & 1);  // the MMAs that read this buffer are done
    {
      uint64_t w = player < n ? __ldg(&maskt[uint64_t(en.tile) * Wp + player]) : 0ull;
      const uint64_t span = (en.hi - en.lo == 64) ? ~0ull : (((1ull << (en.hi - en.lo)) - 1) << en.lo);
      w &= span;
      unsigned char* dst = A + op * kOpBytes + (p >> 3) * 128 + (p & 7) * 16;
#pragma unroll
      for (int u = 0; u < 8; ++u)
        *reinterpret_cast<uint4*>(dst + u * kLBO) = expand8(uint32_t(w >> (8 * u)) & 0xFFu);
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    if (tid == 0) {
      const uint32_t a0 = su32(A), b0 = su32(A + kOpBytes);
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const uint64_t ad = smem_desc(a0 + j * 2 * kLBO, kLBO, 128);
        const uint64_t bd = smem_desc(b0 + j * 2 * kLBO, kLBO, 128);
        mma_f16_ss(tmem, ad, bd, idesc, (accumulate | uint32_t(j)) ? 1u : 0u);
      }
      tc_commit(&bars[buf]);
    }
    ++uses[buf];
    accumulate = 1;
    if (en.run_and_flag & 1u) {
      // fold the run: acc += w * C (C exact integer counts in f32)
      mbar_wait(&bars[buf], (uses[buf] - 1) & 1);
      tc_fence_after();
      const double wr = run_w[en.run_and_flag >> 1];
      const int q = warp & 3, half = warp >> 2;
      const int m = q * 32 + lane;
      uint32_t r[32];
#pragma unroll 1
      for (int c = 0; c < 2; ++c) {
        const int col0 = half * 64 + c * 32;
        TC_LD32(tmem + (uint32_t(q * 32) << 16) + col0, r);
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
        for (int j = 0; j < 32; ++j) acc[(col0 + j) * kGT + m] += wr * double(__uint_as_float(r[j]));
      }
      tc_fence_before();
      __syncthreads();  // TMEM reads done before the next run's first MMA overwrites it
      tc_fence_after();
      accumulate = 0;
    }
  }
  __syncthreads();
  // partial tile -> Gp[split][row = ta tile][col = tb tile]
  double* out = Gp + uint64_t(blockIdx.y) * Np * Np;
  for (int i = tid; i < kGT * kGT; i += kGThreads) {
    const int m = i / kGT, c = i % kGT;  // row-major walk of the tile
    out[(uint64_t(ta) * kGT + m) * Np + uint64_t(tb) * kGT + c] = acc[c * kGT + m];
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(128));
  }
}

// G (lower, row-major, Np x Np) = sum over splits (in order) + cw inside
// n x n; the padded tail is the identity.
__global__ void gram_finish_kernel(const double* __restrict__ Gp, uint32_t splits, uint32_t n, uint64_t Np,
                                   double cw, double* __restrict__ G) {
  const uint64_t idx = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x;
  if (idx >= Np * Np) return;
  const uint64_t i = idx / Np, j = idx % Np;
  double v = 0.0;
  if (j <= i) {
    if (i < n) {
      for (uint32_t s = 0; s < splits; ++s) v += Gp[s * Np * Np + idx];
      v += cw;
    } else {
      v = (i == j) ? 1.0 : 0.0;
    }
  }
  G[idx] = v;
}

// rhs partials: part[blockIdx.y][a] = sum over the block's 256 tiles t and
// the set bits i of maskt[t][a] of wt[t*64+i] (fixed tree per block);
// rhs[a] = sum of the parts in order + cw ct
__global__ void __launch_bounds__(256) gram_rhs_part_kernel(const uint64_t* __restrict__ maskt, uint64_t Wp,
                                                            uint64_t tiles, const double* __restrict__ wt,
                                                            double* __restrict__ part, uint32_t n) {
  __shared__ double red[256];
  const uint32_t a = blockIdx.x;
  const uint64_t t = uint64_t(blockIdx.y) * 256 + threadIdx.x;
  double acc = 0.0;
  if (t < tiles) {
    uint64_t x = maskt[t * Wp + a];
    const double* w = wt + t * 64;
    while (x) {
      const int i = __ffsll(static_cast<long long>(x)) - 1;
      x &= x - 1;
      acc += w[i];
    }
  }
  red[threadIdx.x] = acc;
  __syncthreads();
  for (int h = 128; h > 0; h >>= 1) {
    if (int(threadIdx.x) < h) red[threadIdx.x] += red[threadIdx.x + h];
    __syncthreads();
  }
  if (threadIdx.x == 0) part[uint64_t(blockIdx.y) * n + a] = red[0];
}

__global__ void gram_rhs_finish_kernel(const double* __restrict__ part, uint32_t parts, uint32_t n, double cwct,
                                       double* __restrict__ rhs) {
  const uint32_t a = blockIdx.x * blockDim.x + threadIdx.x;
  if (a >= n) return;
  double acc = 0.0;
  for (uint32_t k = 0; k < parts; ++k) acc += part[uint64_t(k) * n + a];
  rhs[a] = acc + cwct;
}

// wt[i] = w_run(i) * t_i over the runs (rows past `rows`: 0)
__global__ void run_targets_kernel(const uint32_t* __restrict__ run_of_row, const double* __restrict__ run_w,
                                   const double* __restrict__ tgt, uint64_t rows, uint64_t padded,
                                   double* __restrict__ wt) {
  const uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x;
  if (i >= padded) return;
  wt[i] = i < rows ? run_w[run_of_row[i]] * tgt[i] : 0.0;
}

// ---------------------------------------------------------------- Cholesky
// one warp factors the 64 x 64 diagonal block in shared memory (lane owns
// rows lane and lane + 32; __syncwarp only)
__global__ void __launch_bounds__(32) chol_diag_kernel(double* __restrict__ A, uint64_t Np, uint32_t k0,
                                                       int* __restrict__ info) {
  __shared__ double a[kCB][kCB + 1];
  const int lane = threadIdx.x;
  if (*info >= 0) return;  // an earlier block already failed
  for (int i = lane; i < kCB * kCB; i += 32) {
    const int r = i / kCB, c = i % kCB;
    a[r][c] = A[(uint64_t(k0) + r) * Np + k0 + c];
  }
  __syncwarp();
  for (int c = 0; c < kCB; ++c) {
    const double d = a[c][c];
    if (!(d > 0.0) || !isfinite(d)) {
      if (lane == 0) *info = int(k0) + c;
      return;
    }
    const double piv = sqrt(d);
    __syncwarp();
    if (lane == 0) a[c][c] = piv;
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int r = lane + 32 * h;
      if (r > c) a[r][c] /= piv;
    }
    __syncwarp();
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int r = lane + 32 * h;
      if (r > c) {
        const double lrc = a[r][c];
        for (int q = c + 1; q <= r; ++q) a[r][q] -= lrc * a[q][c];
      }
    }
    __syncwarp();
  }
  for (int i = lane; i < kCB * kCB; i += 32) {
    const int r = i / kCB, c = i % kCB;
    if (c <= r) A[(uint64_t(k0) + r) * Np + k0 + c] = a[r][c];
  }
}

// rows of block row (k0/64 + 1 + blockIdx.x): X L_kk^T = A_rk
__global__ void __launch_bounds__(64) chol_panel_kernel(double* __restrict__ A, uint64_t Np, uint32_t k0,
                                                        const int* __restrict__ info) {
  __shared__ double l[kCB][kCB + 1];
  if (*info >= 0) return;
  const int tid = threadIdx.x;
  for (int i = tid; i < kCB * kCB; i += blockDim.x) {
    const int r = i / kCB, c = i % kCB;
    l[r][c] = c <= r ? A[(uint64_t(k0) + r) * Np + k0 + c] : 0.0;
  }
  __syncthreads();
  const uint64_t row = uint64_t(k0) + kCB * (1 + blockIdx.x) + tid;
  double x[kCB];
  double* a = A + row * Np + k0;
#pragma unroll
  for (int j = 0; j < kCB; ++j) x[j] = a[j];
#pragma unroll
  for (int j = 0; j < kCB; ++j) {
    double t = x[j];
#pragma unroll
    for (int q = 0; q < j; ++q) t -= x[q] * l[j][q];
    x[j] = t / l[j][j];
  }
#pragma unroll
  for (int j = 0; j < kCB; ++j) a[j] = x[j];
}

// trailing update of the lower blocks (bi >= bj) right of column block kb:
// A_ij -= L_ik L_jk^T
__global__ void __launch_bounds__(256) chol_update_kernel(double* __restrict__ A, uint64_t Np, uint32_t k0,
                                                          const int* __restrict__ info) {
  constexpr int KH = kCB / 2;
  __shared__ double li[kCB][KH + 1];
  __shared__ double lj[kCB][KH + 1];
  if (*info >= 0) return;
  uint32_t bi = 0, rem = blockIdx.x;
  while (rem > bi) {
    rem -= bi + 1;
    ++bi;
  }
  const uint32_t bj = rem;
  const uint64_t r0 = uint64_t(k0) + kCB * (1 + bi), c0 = uint64_t(k0) + kCB * (1 + bj);
  const int tid = threadIdx.x;
  const int tr = (tid / 16) * 4, tc = (tid % 16) * 4;
  double s[4][4] = {};
  for (int kh = 0; kh < 2; ++kh) {
    for (int i = tid; i < kCB * KH; i += blockDim.x) {
      const int r = i / KH, c = i % KH;
      li[r][c] = A[(r0 + r) * Np + k0 + kh * KH + c];
      lj[r][c] = A[(c0 + r) * Np + k0 + kh * KH + c];
    }
    __syncthreads();
#pragma unroll 4
    for (int k = 0; k < KH; ++k) {
      double a[4], b[4];
#pragma unroll
      for (int x = 0; x < 4; ++x) {
        a[x] = li[tr + x][k];
        b[x] = lj[tc + x][k];
      }
#pragma unroll
      for (int x = 0; x < 4; ++x)
#pragma unroll
        for (int y = 0; y < 4; ++y) s[x][y] = fma(a[x], b[y], s[x][y]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int x = 0; x < 4; ++x)
#pragma unroll
    for (int y = 0; y < 4; ++y) {
      const uint64_t r = r0 + tr + x, c = c0 + tc + y;
      if (c <= r) A[r * Np + c] -= s[x][y];
    }
}

// L z = b then L^T phi = z, one CTA; 64-row blocks: the diagonal block is
// staged in shared memory, warp 0 solves it with shuffles, all threads then
// update the rest of z.
__global__ void __launch_bounds__(1024) chol_solve_kernel(const double* __restrict__ L, uint64_t Np,
                                                          double* __restrict__ z) {
  const int tid = threadIdx.x, lane = tid & 31;
  const uint32_t nb = uint32_t(Np / kCB);
  __shared__ double blk[kCB];
  __shared__ double d[kCB][kCB + 1];
  for (uint32_t kb = 0; kb < nb; ++kb) {
    const uint64_t k0 = uint64_t(kb) * kCB;
    for (int i = tid; i < kCB * kCB; i += blockDim.x) d[i / kCB][i % kCB] = L[(k0 + i / kCB) * Np + k0 + i % kCB];
    __syncthreads();
    if (tid < 32) {
      double z0 = z[k0 + lane], z1 = z[k0 + 32 + lane];
      for (int j = 0; j < kCB; ++j) {
        double zj = __shfl_sync(0xffffffffu, j < 32 ? z0 : z1, j & 31) / d[j][j];
        if (j == lane) z0 = zj;
        if (j == lane + 32) z1 = zj;
        if (lane > j) z0 -= d[lane][j] * zj;
        if (lane + 32 > j) z1 -= d[lane + 32][j] * zj;
      }
      blk[lane] = z0;
      blk[lane + 32] = z1;
      z[k0 + lane] = z0;
      z[k0 + 32 + lane] = z1;
    }
    __syncthreads();
    for (uint64_t i = k0 + kCB + tid; i < Np; i += blockDim.x) {
      double t = z[i];
      const double* li = L + i * Np + k0;
#pragma unroll 8
      for (int j = 0; j < kCB; ++j) t -= li[j] * blk[j];
      z[i] = t;
    }
    __syncthreads();
  }
  for (uint32_t kbb = nb; kbb > 0; --kbb) {
    const uint64_t k0 = uint64_t(kbb - 1) * kCB;
    for (int i = tid; i < kCB * kCB; i += blockDim.x) d[i / kCB][i % kCB] = L[(k0 + i / kCB) * Np + k0 + i % kCB];
    __syncthreads();
    if (tid < 32) {
      double z0 = z[k0 + lane], z1 = z[k0 + 32 + lane];
      for (int j = kCB - 1; j >= 0; --j) {
        double zj = __shfl_sync(0xffffffffu, j < 32 ? z0 : z1, j & 31) / d[j][j];
        if (j == lane) z0 = zj;
        if (j == lane + 32) z1 = zj;
        if (lane < j) z0 -= d[j][lane] * zj;
        if (lane + 32 < j) z1 -= d[j][lane + 32] * zj;
      }
      blk[lane] = z0;
      blk[lane + 32] = z1;
      z[k0 + lane] = z0;
      z[k0 + 32 + lane] = z1;
    }
    __syncthreads();
    for (uint64_t i = tid; i < k0; i += blockDim.x) {
      double t = z[i];
#pragma unroll 8
      for (int j = 0; j < kCB; ++j) t -= L[(k0 + j) * Np + i] * blk[j];
      z[i] = t;
    }
    __syncthreads();
  }
}

__global__ void diag_trace_kernel(const double* __restrict__ G, uint64_t Np, uint32_t n, double* __restrict__ out) {
  __shared__ double part[256];
  double s = 0.0;
  for (uint32_t i = threadIdx.x; i < n; i += blockDim.x) s += G[uint64_t(i) * Np + i];
  part[threadIdx.x] = s;
  __syncthreads();
  for (int h = 128; h > 0; h >>= 1) {
    if (int(threadIdx.x) < h) part[threadIdx.x] += part[threadIdx.x + h];
    __syncthreads();
  }
  if (threadIdx.x == 0) *out = part[0];
}

__global__ void add_diag_kernel(double* __restrict__ G, uint64_t Np, uint32_t n, const double* __restrict__ trace) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) G[uint64_t(i) * Np + i] += 1.0e-10 * (*trace) / n;
}

inline unsigned nblk(uint64_t n, unsigned t = 256) { return unsigned((n + t - 1) / t); }

}  // namespace

// Factors G (Np x Np, lower) in place; returns -1 or the failing pivot.
static int chol_factor(Ctx& ctx, double* G, uint64_t Np, int* d_info) {
  cudaStream_t st = ctx.stream;
  const int none = -1;
  SF_CUDA(cudaMemcpyAsync(d_info, &none, sizeof(int), cudaMemcpyHostToDevice, st));
  const uint32_t nb = uint32_t(Np / kCB);
  for (uint32_t kb = 0; kb < nb; ++kb) {
    const uint32_t k0 = kb * kCB;
    chol_diag_kernel<<<1, 32, 0, st>>>(G, Np, k0, d_info);
    SF_LAUNCHED(ctx);
    const uint32_t below = nb - kb - 1;
    if (below) {
      chol_panel_kernel<<<below, 64, 0, st>>>(G, Np, k0, d_info);
      SF_LAUNCHED(ctx);
      chol_update_kernel<<<below * (below + 1) / 2, 256, 0, st>>>(G, Np, k0, d_info);
      SF_LAUNCHED(ctx);
    }
  }
  int info = -1;
  SF_CUDA(cudaMemcpyAsync(&info, d_info, sizeof(int), cudaMemcpyDeviceToHost, st));
  SF_CUDA(cudaStreamSynchronize(st));
  return info;
}

std::vector<double> gram_solve(Ctx& ctx, const CglsInput& in, const std::vector<GramRun>& runs) {
  const uint32_t n = in.n;
  if (n == 0) return {};
  const uint64_t rows = in.rows;
  const uint32_t W = in.W;
  const uint64_t tiles = (rows + 63) / 64;
  const uint64_t Wp = uint64_t(W) * 64;
  const uint32_t T = (n + kGT - 1) / kGT;
  const uint64_t Np = uint64_t(T) * kGT;
  const uint32_t pairs_t = T * (T + 1) / 2;
  int sms = 148;
  SF_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, ctx.device));
  // work entries: (tile, row range, run), run ends flagged; split the row
  // axis when there are few output tiles
  std::vector<GramEntry> ent;
  std::vector<double> run_w(runs.size());
  std::vector<uint32_t> run_of_row(rows);
  for (size_t r = 0; r < runs.size(); ++r) {
    run_w[r] = runs[r].weight;
    for (uint64_t i = runs[r].begin; i < runs[r].end; ++i) run_of_row[i] = uint32_t(r);
    for (uint64_t i = runs[r].begin; i < runs[r].end;) {
      const uint64_t t = i / 64, hi = std::min<uint64_t>(runs[r].end, t * 64 + 64);
      ent.push_back(GramEntry{uint32_t(t), uint32_t(i - t * 64), uint32_t(hi - t * 64), uint32_t(r) << 1});
      i = hi;
    }
    if (!ent.empty()) ent.back().run_and_flag |= 1u;
  }
  const uint64_t want = std::max<uint64_t>(1, (2ull * sms + pairs_t - 1) / pairs_t);
  const uint64_t splits = std::max<uint64_t>(1, std::min<uint64_t>({want, 64, (ent.size() + 15) / 16}));
  std::vector<uint32_t> sstart;
  for (uint64_t s = 0; s <= splits; ++s) sstart.push_back(uint32_t(ent.size() * s / splits));
  for (uint64_t s = 1; s < splits; ++s)  // a split that ends inside a run folds its part of the run
    if (sstart[s] > 0) ent[sstart[s] - 1].run_and_flag |= 1u;

  cudaStream_t st = ctx.stream;
  DebugTimer dt("gram");
  auto lap = [&](const char* what) {
    if (!dt.on) return;
    SF_CUDA(cudaStreamSynchronize(st));
    dt.lap(what);
  };
  ctx.gram_maskt.reserve(std::max<uint64_t>(tiles * Wp, 1));
  if (in.kept_only)
    launch_transpose_pairs(ctx, in.dev_rows, rows / 2, W, n, tiles, ctx.gram_maskt.p);
  else
    launch_transpose_tiles(ctx, in.dev_rows, rows, W, tiles, ctx.gram_maskt.p);
  const uint64_t rhs_parts = std::max<uint64_t>(1, (tiles + 255) / 256);
  const uint64_t wbytes = ent.size() * sizeof(GramEntry) + (splits + 1) * 4 + run_w.size() * 8 +
                          rows * 4 + (tiles * 64 + 1) * 8 + rhs_parts * n * 8 + 16 * 256;
  ctx.gram_work.reserve(wbytes);
  unsigned char* base = ctx.gram_work.p;
  uint64_t off = 0;
  auto take = [&](uint64_t b) {
    off = (off + 255) & ~uint64_t(255);
    unsigned char* p = base + off;
    off += std::max<uint64_t>(b, 1);
    return p;
  };
  auto* d_ent = reinterpret_cast<GramEntry*>(take(ent.size() * sizeof(GramEntry)));
  auto* d_ss = reinterpret_cast<uint32_t*>(take((splits + 1) * 4));
  auto* d_rw = reinterpret_cast<double*>(take(run_w.size() * 8));
  auto* d_run = reinterpret_cast<uint32_t*>(take(rows * 4));
  auto* d_wt = reinterpret_cast<double*>(take((tiles * 64 + 1) * 8));
  auto* d_info = reinterpret_cast<int*>(take(16));
  auto* d_trace = reinterpret_cast<double*>(take(16));
  auto* d_part = reinterpret_cast<double*>(take(rhs_parts * n * 8));
  lap("plan + tiles");
  SF_CUDA(cudaMemcpyAsync(d_ent, ent.data(), ent.size() * sizeof(GramEntry), cudaMemcpyHostToDevice, st));
  SF_CUDA(cudaMemcpyAsync(d_ss, sstart.data(), sstart.size() * 4, cudaMemcpyHostToDevice, st));
  SF_CUDA(cudaMemcpyAsync(d_rw, run_w.data(), run_w.size() * 8, cudaMemcpyHostToDevice, st));
  SF_CUDA(cudaMemcpyAsync(d_run, run_of_row.data(), rows * 4, cudaMemcpyHostToDevice, st));
  ctx.h2d_bytes += ent.size() * sizeof(GramEntry) + sstart.size() * 4 + run_w.size() * 8 + rows * 4;
  ctx.gram_g.reserve(splits * Np * Np + 2 * Np * Np + Np);
  double* Gp = ctx.gram_g.p;
  double* G = Gp + splits * Np * Np;
  double* G0 = G + Np * Np;  // unfactored copy for the jitter retry
  double* z = G0 + Np * Np;
  set_max_dynamic_smem(gram_tc_kernel, kGSmem);
  if (!ent.empty()) {
    gram_tc_kernel<<<dim3(pairs_t, unsigned(splits)), kGThreads, kGSmem, st>>>(ctx.gram_maskt.p, Wp, n, T, d_ent,
                                                                              d_ss, d_rw, Gp, Np);
    SF_LAUNCHED(ctx);
  } else {
    SF_CUDA(cudaMemsetAsync(Gp, 0, splits * Np * Np * 8, st));
  }
  gram_finish_kernel<<<nblk(Np * Np), 256, 0, st>>>(Gp, unsigned(ent.empty() ? 1 : splits), n, Np,
                                                    in.constraint_weight, G);
  SF_LAUNCHED(ctx);
  run_targets_kernel<<<nblk(tiles * 64), 256, 0, st>>>(d_run, d_rw, in.dev_targets, rows, tiles * 64, d_wt);
  SF_LAUNCHED(ctx);
  SF_CUDA(cudaMemsetAsync(z, 0, Np * 8, st));
  {
    const uint32_t parts = uint32_t(std::max<uint64_t>(1, (tiles + 255) / 256));
    if (tiles) {
      gram_rhs_part_kernel<<<dim3(n, parts), 256, 0, st>>>(ctx.gram_maskt.p, Wp, tiles, d_wt, d_part, n);
      SF_LAUNCHED(ctx);
    } else {
      SF_CUDA(cudaMemsetAsync(d_part, 0, uint64_t(n) * 8, st));
    }
    gram_rhs_finish_kernel<<<nblk(n), 256, 0, st>>>(d_part, parts, n, in.constraint_weight * in.constraint_target,
                                                    z);
    SF_LAUNCHED(ctx);
  }
  SF_CUDA(cudaMemcpyAsync(G0, G, Np * Np * 8, cudaMemcpyDeviceToDevice, st));
  lap("gram + rhs");
  int bad = chol_factor(ctx, G, Np, d_info);
  lap("cholesky");
  if (bad >= 0) {
    // the reference's one retry with diagonal jitter 1e-10 trace / n
    SF_CUDA(cudaMemcpyAsync(G, G0, Np * Np * 8, cudaMemcpyDeviceToDevice, st));
    diag_trace_kernel<<<1, 256, 0, st>>>(G, Np, n, d_trace);
    SF_LAUNCHED(ctx);
    add_diag_kernel<<<nblk(n), 256, 0, st>>>(G, Np, n, d_trace);
    SF_LAUNCHED(ctx);
    bad = chol_factor(ctx, G, Np, d_info);
    if (bad >= 0)
      throw NumericalError("normal equations are singular: factorization failed at pivot " + std::to_string(bad) +
                           " of " + std::to_string(n) + " even after diagonal jitter");
  }
  chol_solve_kernel<<<1, 1024, 0, st>>>(G, Np, z);
  SF_LAUNCHED(ctx);
  std::vector<double> phi(n);
  SF_CUDA(cudaMemcpyAsync(phi.data(), z, uint64_t(n) * 8, cudaMemcpyDeviceToHost, st));
  SF_CUDA(cudaStreamSynchronize(st));
  ctx.d2h_bytes += uint64_t(n) * 8 + 4;
  return phi;
}

}  // namespace sfb
