// Tensor-core passes of the bit-row CGLS over the dense pairs — the two
// products the nibble-table kernels in sf_cgls.cu compute (M u in
// solver.cpp:252-287, M^T c in solver.cpp:209-248) — as exact integer
// arithmetic on tcgen05 kind::i8:
//
//  * the FP64 vector x (u over players, or the pair coefficients) is cut
//    into 16 signed 7-bit digits on a fixed-point grid set by max|x|:
//    round(x 2^(61-e)) in 9 digits and the 48-bit remainder in 7
//    (digits_kernel, laid out as the MMA's B operand: K-major canonical,
//    one 4 KB group per 256 elements);
//  * each lane (a pair row, or a player) expands its 64-bit mask words in
//    registers: bit 8j+k of a 32-bit half becomes byte j of a TMEM column
//    with value 0 or 2^k (one LOP3 per column), stored with tcgen05.st —
//    the A operand, never in shared memory;
//  * one MMA per bit position k (M = 128 lanes, N = 16 digits, K = 32)
//    accumulates 2^k x (the sum of the masked digits) into its own S32
//    accumulator D_k; the epilogue takes sum_k D_k >> k per digit and
//    weighs the digits into one FP64 value.
// The integer sums are exact, so a pass result depends only on the grid
// values of x — not on the order, the split of the work or the rank layout.
// Against the nibble tables (one 64-bit shared-memory lookup per 4 mask
// bits, bound by shared-memory wavefronts) this moves the bits through
// registers and TMEM only; the kernel is bound by the mask words' HBM reads.
//
// Work items are (block of 128 lanes, part of the word axis); a persistent
// CTA per SM walks its items with a 14-stage bulk-copy ring (mask words +
// the digit group), 4 TMEM A slots and two TMEM accumulator sets, so the
// epilogue of one item overlaps the MMAs of the next.
#include <cuda_runtime.h>

#include <cfloat>
#include <climits>
#include <cstdlib>
#include <cstring>

#include "sf_device.cuh"
#include "sf_internal.hpp"
#include "sf_tcgen05.cuh"

namespace sfb {

namespace {

using namespace tc;

constexpr int kThreads = 192;  // warps 0-3 expand + epilogue, 4 bulk copies, 5 MMAs
constexpr uint32_t kRowBytes = 128 * 8;          // one u64 word per lane
constexpr uint32_t kStageA = 4 * kRowBytes;      // 4 words per lane
constexpr uint32_t kGroup = 256;                 // elements per digit group (4 words)
constexpr uint32_t kGroupBytes = kGroup * 16;    // 16 digits each
constexpr uint32_t kStageBytes = kStageA + kGroupBytes;
constexpr uint32_t kATile = 128 * 32;            // one MMA's A: 128 lanes x 32 bytes
// A in TMEM (ts): 14 stages, 4 TMEM A slots of 64 columns, D at [0, 256);
// 120 KB of shared memory keeps one CTA per SM (the TMEM allocation is 512).
// A in shared memory (ss): 10 stages, 4 A slots of 8 tiles (32 KB), TMEM 256.
template <bool kSS>
struct I8Cfg {
  static constexpr int kStages = kSS ? 10 : 14;
  static constexpr int kASlots = 4;
  static constexpr uint32_t kAOff = kStages * kStageBytes;
  static constexpr uint32_t kBarOff = kAOff + (kSS ? kASlots * 8 * kATile : 0);
  static constexpr uint32_t kSmem = kSS ? kBarOff + 512 : 120 * 1024;
  static constexpr uint32_t kTmemCols = kSS ? 256 : 512;
  static_assert(kBarOff + 512 <= kSmem && kSmem <= 227 * 1024, "shared memory budget");
};
constexpr int kAbsBlocks = 296;
constexpr uint32_t kIdesc = (2u << 4) |            // D: S32
                            (0u << 7) |            // A: U8 (0 or 2^k)
                            (1u << 10) |           // B: S8 digits
                            ((16u >> 3) << 17) |   // N = 16
                            ((128u >> 4) << 24);   // M = 128

#define I8_ST8(taddr, r)                                                                               \
  asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(taddr), \
               "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7])  \
               : "memory")

__device__ __forceinline__ void mma_i8_ss(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
      "l"(adesc), "l"(bdesc), "r"(kIdesc), "r"(accumulate)
      : "memory");
}
__device__ __forceinline__ void mma_i8_ts(uint32_t d_tmem, uint32_t a_tmem, uint64_t bdesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::i8 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d_tmem),
      "r"(a_tmem), "l"(bdesc), "r"(kIdesc), "r"(accumulate)
      : "memory");
}

__global__ void __launch_bounds__(256)
    absmax_partial_kernel(const double* __restrict__ x, uint64_t beg, uint64_t end, double* __restrict__ partial) {
  __shared__ double red[8];
  double m = 0.0;
  for (uint64_t i = beg + blockIdx.x * 256ull + threadIdx.x; i < end; i += uint64_t(gridDim.x) * 256ull) {
    const double a = fabs(x[i]);
    m = (a <= DBL_MAX) ? fmax(m, a) : __longlong_as_double(0x7ff0000000000000ll);  // non-finite -> inf
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) m = fmax(m, __shfl_xor_sync(kFullMask, m, o));
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = m;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = red[0];
    for (int i = 1; i < 8; ++i) t = fmax(t, red[i]);
    partial[blockIdx.x] = t;
  }
}

// 16 digits of x on the grid 2^(e-109), |x| < 2^e: x 2^(61-e) = hi + r,
// hi in 9 balanced base-128 digits (d0..d8), round(r 2^48) in 7 (d9..d15)
__device__ __forceinline__ void digits16(double x, int e, int d[16]) {
  const double xs = ldexp(x, 61 - e);
  long long hi = llrint(xs);
  const double r = xs - double(hi);
  long long lo = llrint(ldexp(r, 48));
#pragma unroll
  for (int s = 0; s < 9; ++s) {
    const long long t = ((hi + 64) & 127) - 64;
    d[s] = int(t);
    hi = (hi - t) >> 7;
  }
#pragma unroll
  for (int s = 0; s < 7; ++s) {
    const long long t = ((lo + 64) & 127) - 64;
    d[9 + s] = int(t);
    lo = (lo - t) >> 7;
  }
}

// Digit groups [g_lo, g_hi) of x[0, len): thread = (group, bit position k,
// K half qb): 16 elements, 16 digit rows of 16 bytes each.
__global__ void __launch_bounds__(256)
    digits_kernel(const double* __restrict__ x, uint64_t len, uint64_t g_lo, uint64_t g_hi,
                  const double* __restrict__ partial, uint8_t* __restrict__ out, int* __restrict__ exp_slot) {
  __shared__ double red[8];
  __shared__ int e_sh;
  double m = 0.0;
  for (int i = threadIdx.x; i < kAbsBlocks; i += 256) m = fmax(m, partial[i]);
#pragma unroll
  for (int o = 16; o; o >>= 1) m = fmax(m, __shfl_xor_sync(kFullMask, m, o));
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = m;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = red[0];
    for (int i = 1; i < 8; ++i) t = fmax(t, red[i]);
    int e = 0;
    if (!(t <= DBL_MAX))
      e = INT_MIN;  // a non-finite input: the pass returns NaN (the solver's blowup check)
    else if (t > 0.0)
      frexp(t, &e);  // t < 2^e
    e_sh = e;
    if (blockIdx.x == 0) *exp_slot = e;
  }
  __syncthreads();
  const int e = e_sh;
  const uint64_t unit = blockIdx.x * 256ull + threadIdx.x;
  const uint64_t g = g_lo + unit / 16;
  if (g >= g_hi) return;
  const uint32_t k = uint32_t(unit % 16) >> 1, qb = uint32_t(unit & 1);
  uint32_t row[16][4];
#pragma unroll
  for (int s = 0; s < 16; ++s)
#pragma unroll
    for (int w = 0; w < 4; ++w) row[s][w] = 0u;
#pragma unroll
  for (int qq = 0; qq < 16; ++qq) {
    const uint32_t q = qb * 16 + qq, cc = q >> 2, j = q & 3;
    const uint32_t l = (cc >> 1) * 64 + (cc & 1) * 32 + j * 8 + k;
    const uint64_t idx = g * kGroup + l;
    const double v = idx < len ? x[idx] : 0.0;
    int d[16];
    if (e == INT_MIN || v == 0.0) {
#pragma unroll
      for (int s = 0; s < 16; ++s) d[s] = 0;
    } else {
      digits16(v, e, d);
    }
#pragma unroll
    for (int s = 0; s < 16; ++s) row[s][qq >> 2] |= (uint32_t(d[s]) & 0xffu) << (8 * (qq & 3));
  }
  uint8_t* base = out + g * kGroupBytes + k * 512 + qb * 256;
#pragma unroll
  for (int s = 0; s < 16; ++s)
    *reinterpret_cast<uint4*>(base + (s >> 3) * 128 + (s & 7) * 16) = make_uint4(row[s][0], row[s][1], row[s][2],
                                                                                  row[s][3]);
}

__device__ __forceinline__ double combine_digits(const long long* S, int e) {
  if (e == INT_MIN) return __longlong_as_double(0x7ff8000000000000ll);
  double hi = 0.0, lo = 0.0;
#pragma unroll
  for (int s = 8; s >= 0; --s) hi = hi * 128.0 + double(S[s]);
#pragma unroll
  for (int s = 15; s >= 9; --s) lo = lo * 128.0 + double(S[s]);
  return ldexp(hi, e - 61) + ldexp(lo, e - 109);
}

// out[p][lane] = sum over the words a in part p of the lane's mask bits
// times x (digit groups), for every lane of every 128-lane block.
//   words   word a of lane L at words[a * stride + L]
//   parts   split_start ? [split_start[p], split_start[p+1]) : [p pw, min(A, (p+1) pw))
template <bool kSS>
__global__ void __launch_bounds__(kThreads, 1)
    bitmat_i8_kernel(const uint64_t* __restrict__ words, uint64_t stride, uint64_t lanes, uint64_t out_lanes,
                     uint64_t lane_blocks, uint32_t nparts, const uint32_t* __restrict__ split_start,
                     uint32_t part_words, uint32_t total_words, const uint8_t* __restrict__ digits,
                     const int* __restrict__ exp_slot, double* __restrict__ out, uint64_t out_stride) {
  using Cfg = I8Cfg<kSS>;
  constexpr int kStages = Cfg::kStages, kASlots = Cfg::kASlots;
  extern __shared__ __align__(1024) unsigned char smem[];
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + Cfg::kBarOff);
  uint64_t* full = bars;                       // [kStages] words + digits landed
  uint64_t* sdone = full + kStages;            // [kStages] the stage's MMAs done
  uint64_t* afull = sdone + kStages;           // [kASlots] A slot written (128 arrivals)
  uint64_t* tdone = afull + kASlots;           // [kASlots] the slot's MMAs done
  uint64_t* dfull = tdone + kASlots;           // [2] an item's accumulators final
  uint64_t* dfree = dfull + 2;                 // [2] accumulators read (128 arrivals)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(dfree + 2);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (tid == 0) {
    for (int i = 0; i < kStages; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&sdone[i], 1);
    }
    for (int i = 0; i < kASlots; ++i) {
      mbar_init(&afull[i], 128);
      mbar_init(&tdone[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&dfull[i], 1);
      mbar_init(&dfree[i], 128);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(su32(tmem_slot)),
                 "r"(Cfg::kTmemCols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;  // columns: D sets [0, 128) [128, 256); A slots 256 + 64 a

  const uint64_t items = lane_blocks * nparts;
  auto part_range = [&](uint32_t p, uint32_t& a0, uint32_t& a1) {
    if (split_start) {
      a0 = split_start[p];
      a1 = split_start[p + 1];
    } else {
      a0 = p * part_words;
      a1 = min(total_words, a0 + part_words);
    }
  };
  auto slots_of = [](uint32_t a0, uint32_t a1) { return a1 > a0 ? (a1 + 3) / 4 - a0 / 4 : 0u; };

  if (warp == 4) {
    if (lane == 0) {  // bulk copies: 4 word rows (128 lanes each) + the digit group
      uint32_t gs = 0;
      for (uint64_t id = blockIdx.x; id < items; id += gridDim.x) {
        const uint64_t lb = id % lane_blocks;
        uint32_t a0, a1;
        part_range(uint32_t(id / lane_blocks), a0, a1);
        const uint32_t ns = slots_of(a0, a1);
        const uint64_t lane0 = lb * 128;
        const uint32_t rowbytes = uint32_t((stride - lane0 < 128 ? stride - lane0 : 128) * 8);
        for (uint32_t i = 0; i < ns; ++i, ++gs) {
          const uint32_t st = gs % kStages;
          if (gs >= uint32_t(kStages)) mbar_wait(&sdone[st], ((gs / kStages) - 1) & 1u);
          const uint32_t g = a0 / 4 + i;
          uint32_t nv = 0;
          for (uint32_t c = 0; c < 4; ++c) nv += (4 * g + c >= a0 && 4 * g + c < a1) ? 1u : 0u;
          unsigned char* stage = smem + st * kStageBytes;
          mbar_arrive_expect_tx(&full[st], kGroupBytes + nv * rowbytes);
          for (uint32_t c = 0; c < 4; ++c) {
            const uint32_t a = 4 * g + c;
            if (a >= a0 && a < a1) bulk_g2s(stage + c * kRowBytes, words + uint64_t(a) * stride + lane0, rowbytes,
                                            &full[st]);
          }
          bulk_g2s(stage + kStageA, digits + uint64_t(g) * kGroupBytes, kGroupBytes, &full[st]);
        }
      }
    }
  } else if (warp == 5) {
    if (lane == 0) {  // MMA issue: 8 per slot (one per bit position k)
      uint32_t gs = 0, ii = 0;
      for (uint64_t id = blockIdx.x; id < items; id += gridDim.x) {
        uint32_t a0, a1;
        part_range(uint32_t(id / lane_blocks), a0, a1);
        const uint32_t ns = slots_of(a0, a1);
        if (ns == 0) continue;
        const uint32_t db = ii & 1u;
        if (ii >= 2) {
          mbar_wait(&dfree[db], ((ii / 2) - 1) & 1u);
          tc_fence_after();
        }
        for (uint32_t i = 0; i < ns; ++i, ++gs) {
          const uint32_t a = gs % kASlots, st = gs % kStages;
          mbar_wait(&afull[a], (gs / kASlots) & 1u);
          tc_fence_after();
          const uint32_t bbase = su32(smem + st * kStageBytes + kStageA);
          if constexpr (kSS) {
            const uint32_t abase = su32(smem + Cfg::kAOff + a * 8 * kATile);
#pragma unroll
            for (uint32_t k = 0; k < 8; ++k)
              mma_i8_ss(tmem + db * 128 + 16 * k, smem_desc(abase + k * kATile, 2048, 128),
                        smem_desc(bbase + k * 512, 256, 128), i > 0 ? 1u : 0u);
          } else {
#pragma unroll
            for (uint32_t k = 0; k < 8; ++k)
              mma_i8_ts(tmem + db * 128 + 16 * k, tmem + 256 + 64 * a + 8 * k, smem_desc(bbase + k * 512, 256, 128),
                        i > 0 ? 1u : 0u);
          }
          tc_commit(&tdone[a]);
          tc_commit(&sdone[st]);
        }
        tc_commit(&dfull[db]);
        ++ii;
      }
    }
  } else {  // warps 0-3: lane m of the block, TMEM lane quarter = warp
    const uint32_t m = uint32_t(tid);
    const uint32_t lane_base = uint32_t(warp * 32) << 16;
    uint32_t gs = 0, ii = 0;
    for (uint64_t id = blockIdx.x; id < items; id += gridDim.x) {
      const uint64_t lb = id % lane_blocks;
      const uint32_t p = uint32_t(id / lane_blocks);
      uint32_t a0, a1;
      part_range(p, a0, a1);
      const uint32_t ns = slots_of(a0, a1);
      const uint64_t L = lb * 128 + m;
      if (ns == 0) {
        if (L < out_lanes) out[uint64_t(p) * out_stride + L] = 0.0;
        continue;
      }
      const bool lv = L < lanes;
      for (uint32_t i = 0; i < ns; ++i, ++gs) {
        const uint32_t st = gs % kStages, a = gs % kASlots;
        mbar_wait(&full[st], (gs / kStages) & 1u);
        const uint64_t* sw = reinterpret_cast<const uint64_t*>(smem + st * kStageBytes);
        const uint32_t g = a0 / 4 + i;
        uint64_t x[4];
#pragma unroll
        for (uint32_t c = 0; c < 4; ++c) {
          const uint32_t aa = 4 * g + c;
          x[c] = (lv && aa >= a0 && aa < a1) ? sw[c * 128 + m] : 0ull;
        }
        if (gs >= uint32_t(kASlots)) {
          mbar_wait(&tdone[a], ((gs / kASlots) - 1) & 1u);
          tc_fence_after();
        }
        if constexpr (kSS) {
          // A tile k (K-major canonical, no swizzle): row m's 32 bytes in two
          // 16-byte core-matrix rows, K blocks 2048 bytes apart
          unsigned char* arow = smem + Cfg::kAOff + a * 8 * kATile + (m >> 3) * 128 + (m & 7) * 16;
#pragma unroll
          for (uint32_t k = 0; k < 8; ++k) {
            uint32_t v[8];
#pragma unroll
            for (int c = 0; c < 4; ++c) {
              v[2 * c] = uint32_t(x[c]) & (0x01010101u << k);
              v[2 * c + 1] = uint32_t(x[c] >> 32) & (0x01010101u << k);
            }
            *reinterpret_cast<uint4*>(arow + k * kATile) = make_uint4(v[0], v[1], v[2], v[3]);
            *reinterpret_cast<uint4*>(arow + k * kATile + 2048) = make_uint4(v[4], v[5], v[6], v[7]);
          }
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        } else {
          const uint32_t acol = tmem + lane_base + 256 + 64 * a;
#pragma unroll
          for (uint32_t k = 0; k < 8; ++k) {
            uint32_t v[8];
#pragma unroll
            for (int c = 0; c < 4; ++c) {
              v[2 * c] = uint32_t(x[c]) & (0x01010101u << k);
              v[2 * c + 1] = uint32_t(x[c] >> 32) & (0x01010101u << k);
            }
            I8_ST8(acol + 8 * k, v);
          }
          asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
        }
        tc_fence_before();
        mbar_arrive(&afull[a]);
      }
      const uint32_t db = ii & 1u;
      mbar_wait(&dfull[db], (ii / 2) & 1u);
      tc_fence_after();
      long long S[16];
#pragma unroll
      for (int s = 0; s < 16; ++s) S[s] = 0;
#pragma unroll
      for (uint32_t kk = 0; kk < 4; ++kk) {
        uint32_t r[32];
        TC_LD32(tmem + lane_base + db * 128 + 32 * kk, r);
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
        for (int s = 0; s < 16; ++s)
          S[s] += (long long)(int(r[s]) >> (2 * kk)) + (long long)(int(r[16 + s]) >> (2 * kk + 1));
      }
      tc_fence_before();
      mbar_arrive(&dfree[db]);
      const double val = combine_digits(S, *exp_slot);
      if (L < out_lanes) out[uint64_t(p) * out_stride + L] = val;
      ++ii;
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(Cfg::kTmemCols));
  }
}

}  // namespace

// SF_CGLS_I8: 0 off (nibble tables, the default: 24.6 vs 32.2 ms for the
// C2 solve), 1 A operand in TMEM, 2 A in shared memory
static int cgls_i8_mode() {
  static const int mode = [] {
    const char* v = std::getenv("SF_CGLS_I8");
    return v == nullptr ? 0 : std::atoi(v);
  }();
  return mode;
}
bool cgls_i8_enabled() { return cgls_i8_mode() != 0; }

uint64_t cgls_i8_digit_bytes(uint64_t elements) { return (elements + kGroup - 1) / kGroup * kGroupBytes; }
uint64_t cgls_i8_scratch_doubles() { return kAbsBlocks; }

void launch_cgls_digits(const double* x, uint64_t beg, uint64_t len, double* partial, uint8_t* digits, int* exp_slot,
                        cudaStream_t st) {
  const uint64_t g_lo = beg / kGroup, g_hi = (len + kGroup - 1) / kGroup;
  absmax_partial_kernel<<<kAbsBlocks, 256, 0, st>>>(x, g_lo * kGroup, len, partial);
  const uint64_t units = std::max<uint64_t>(g_hi - g_lo, 1) * 16;
  digits_kernel<<<unsigned((units + 255) / 256), 256, 0, st>>>(x, len, g_lo, g_hi, partial, digits, exp_slot);
}

void launch_bitmat_i8(const uint64_t* words, uint64_t stride, uint64_t lanes, uint64_t out_lanes, uint32_t nparts,
                      const uint32_t* split_start, uint32_t part_words, uint32_t total_words, const uint8_t* digits,
                      const int* exp_slot, double* out, uint64_t out_stride, int sms, cudaStream_t st) {
  const uint64_t lane_blocks = (out_lanes + 127) / 128;
  const uint64_t items = lane_blocks * nparts;
  if (items == 0) return;
  const unsigned grid = unsigned(std::min<uint64_t>(items, uint64_t(sms)));
  if (cgls_i8_mode() == 2) {
    set_max_dynamic_smem(bitmat_i8_kernel<true>, int(I8Cfg<true>::kSmem));
    bitmat_i8_kernel<true><<<grid, kThreads, I8Cfg<true>::kSmem, st>>>(words, stride, lanes, out_lanes, lane_blocks,
                                                                       nparts, split_start, part_words, total_words,
                                                                       digits, exp_slot, out, out_stride);
  } else {
    set_max_dynamic_smem(bitmat_i8_kernel<false>, int(I8Cfg<false>::kSmem));
    bitmat_i8_kernel<false><<<grid, kThreads, I8Cfg<false>::kSmem, st>>>(words, stride, lanes, out_lanes,
                                                                         lane_blocks, nparts, split_start, part_words,
                                                                         total_words, digits, exp_slot, out, out_stride);
  }
}

}  // namespace sfb
