// Tensor-core fused layer-0 -> layer-1 kernel, fp16x2 variant (the default
// for hidden widths 64 and 128; sf_fused_tc.cu is the 3xTF32 variant and
// documents the math). For a work item (u, segments v of {u} u N(u)) and two
// tiles (M = 128 coalitions):
//   H_v[m][:] = sum_{entries k of v} coef[k][m] * P[x_k][:]     (GEMM, K = entries)
//   A_u[m][:] += m_m(e_uv) isd_m(v) relu(isd_m(v) H_v[m][:] + b0)  (per segment)
// The GEMM runs as tcgen05.mma kind::f16 (fp16 in, f32 accumulate, K = 16)
// with both operands split into fp16 hi + lo parts and three products
// (a_hi b_hi + a_hi b_lo + a_lo b_hi), the same ~22-bit product precision as
// 3xTF32. Operands are pre-scaled by powers of two so the lo parts stay
// normal fp16 (coefficients by kCoefScale, P0 by a per-target scale); the
// epilogue folds the exact inverse into isd(v). 16-bit operands allow an
// MN-major B, so the producers gather the pre-split P0 rows straight into
// the swizzled B tile (no staging transpose), and a K = 16 MMA halves the
// MMA count of the tf32 kernel.
//
// Warp roles (768 threads, 1 CTA/SM):
//   warps 0-7    epilogue (two per TMEM lane quarter, column halves)
//   warps 8-11   staging (one per TMEM lane quarter): coefficients (mask
//                bit x 1/sqrt(deg) from the shared table) -> fp16 hi/lo
//                pairs in TMEM (A operand)
//   warps 12-22  producers: 16-byte cp.async gathers of the fp16 P0 planes
//                into the MN-major SWIZZLE_128B B tile, of the u16 degree
//                rows and of the mask words; each thread waits for its own
//                copies one chunk later, fences the async proxy and arrives
//   warp 23      MMA issuer (warp-converged, one elected lane issues)
// One ring of kStages stages: shared memory (B planes, degrees, masks) and
// TMEM (A) share the stage index. Layouts were verified exactly with
// csrc/tools/tc_f16_probe.cu (MN-major SW128 B: atoms of 64 n x 8 k = 1024
// B, LBO = n-atom stride, SBO = k-group stride; TMEM A: two fp16 per column,
// even k in the low half).
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>

#include "sf_device.cuh"
#include "sf_internal.hpp"
#include "sf_tcgen05.cuh"

namespace sfb {

namespace {

using namespace tc;

constexpr int kTile = 64;
constexpr unsigned kFull = 0xffffffffu;
constexpr uint32_t kSelf = 0xFFFFFFFFu;
constexpr uint32_t kPad = 0xFFFFFFFEu;
constexpr int kM = 128;     // coalitions per CTA (two tiles)
constexpr int kKC = 32;     // entries per chunk (two K = 16 k-steps)
constexpr int kStages = 4;  // shared-memory stages = TMEM A stages
constexpr int kMaxKsteps = 4096;
constexpr int kTabCap = 12288;
constexpr float kCoefScale = 256.f;  // coefficients are in (0, 1]: keep the fp16 lo parts normal
constexpr int kEpiWarps = 8, kStgWarps = 4, kProdWarps = 11;
constexpr int kProducerWarp = kEpiWarps + kStgWarps, kMmaWarp = kProducerWarp + kProdWarps;
constexpr int kThreads = (kMmaWarp + 1) * 32;

template <int D>
struct F16Cfg {
  static constexpr int NA = D / 64;                    // 128-byte atoms along n
  static constexpr int KSTRIDE = NA * 1024;            // bytes between 8-row k groups (SBO)
  static constexpr int PLANE = (kKC / 8) * KSTRIDE;    // one plane (hi or lo) of a chunk
  static constexpr int OFF_BHI = 0, OFF_BLO = PLANE;
  static constexpr int OFF_DEG = 2 * PLANE;            // u16 degrees [k][128]
  static constexpr int OFF_W = OFF_DEG + kKC * kM * 2; // mask words [k][2]
  static constexpr int STAGE = ((OFF_W + kKC * 2 * 8 + 1023) / 1024) * 1024;
  static constexpr int OFF_KFL = kStages * STAGE;      // the item's k-step flags
  static constexpr int OFF_BIAS = OFF_KFL + kMaxKsteps;
  static constexpr int NBARS = 3 * kStages + 4;
  static constexpr int OFF_BARS = OFF_BIAS + D * 4;
  static constexpr int OFF_TAB = ((OFF_BARS + 8 * NBARS + 16 + 15) / 16) * 16;
  static constexpr int SMEM = OFF_TAB;  // + the 1/sqrt(deg) table, sized at launch
  static constexpr uint32_t A_COL = 3 * D;  // TMEM: H0, H1, accumulator, A stages (hi 16 | lo 16)
  static constexpr uint32_t TMEM_COLS = 3 * D + kStages * 32 <= 256 ? 256 : 512;
  static_assert(D == 64 || D == 128, "fp16 kernel widths");
  static_assert(3 * D + kStages * 32 <= 512, "TMEM columns");
  static_assert(SMEM + kTabCap * 4 <= 227 * 1024, "shared memory");
};

#define TC_ST8(taddr, r)                                                                          \
  asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(taddr), \
               "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]) \
               : "memory")

__device__ __forceinline__ void tc_mma_f16_elect(uint32_t d_tmem, uint32_t a_tmem, uint64_t bdesc,
                                                 uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p, e;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d_tmem),
      "r"(a_tmem), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}

// fp16 hi/lo of a float, packed in pairs (even entry in the low half)
__device__ __forceinline__ void split2(float c0, float c1, uint32_t& hi, uint32_t& lo) {
  const __half h0 = __float2half_rn(c0), h1 = __float2half_rn(c1);
  const __half l0 = __float2half_rn(c0 - __half2float(h0)), l1 = __float2half_rn(c1 - __half2float(h1));
  hi = uint32_t(__half_as_ushort(h0)) | (uint32_t(__half_as_ushort(h1)) << 16);
  lo = uint32_t(__half_as_ushort(l0)) | (uint32_t(__half_as_ushort(l1)) << 16);
}

// entry: (x, e) — P / degree row x, mask player e (kSelf: always kept, kPad:
// coefficient 0). kflags[k-step of 16]: bit0 segment start, bit1 segment end.
constexpr int kProfSites = 16;
#define F16_WAIT(site, bar, par)                       \
  do {                                                 \
    if constexpr (PROF) {                              \
      const long long _t = clock64();                  \
      mbar_wait(bar, par);                             \
      pw[site] += uint64_t(clock64() - _t);            \
    } else {                                           \
      mbar_wait(bar, par);                             \
    }                                                  \
  } while (0)

template <int D, bool PROF>
__global__ void __launch_bounds__(kThreads, 1)
    fused_f16_kernel(const uint64_t* __restrict__ maskt, uint64_t Wp, const float* __restrict__ isd,
                     uint32_t V, const uint16_t* __restrict__ deg16, const float* __restrict__ tab,
                     uint32_t tab_n, const uint16_t* __restrict__ P16, const float* __restrict__ pscale,
                     const float* __restrict__ bias, const uint2* __restrict__ ent,
                     const uint8_t* __restrict__ kflags, const uint2* __restrict__ seg,
                     const uint32_t* __restrict__ item_ent, const uint32_t* __restrict__ item_seg,
                     const uint32_t* __restrict__ item_order, uint32_t items, uint32_t npairs,
                     const uint64_t* __restrict__ const_words, float* __restrict__ Apart,
                     unsigned long long* __restrict__ prof) {
  using Cfg = F16Cfg<D>;
  uint64_t pw[2] = {0, 0};
  const long long t_begin = PROF ? clock64() : 0;
  auto prof_flush = [&](int base, int n) {
    if constexpr (PROF) {
      if ((threadIdx.x & 31) == 0) {
        for (int k = 0; k < n; ++k) atomicAdd(&prof[base + k], (unsigned long long)pw[k]);
        atomicAdd(&prof[base + n], (unsigned long long)(clock64() - t_begin));
      }
    }
  };
  extern __shared__ __align__(1024) unsigned char smem[];
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + Cfg::OFF_BARS);
  uint64_t* full = bars;                  // producers (copies landed) -> staging
  uint64_t* staged = full + kStages;      // staging (A in TMEM) -> MMA
  uint64_t* empty = staged + kStages;     // MMA commit -> producers
  uint64_t* hfull = empty + kStages;      // MMA commit -> epilogue
  uint64_t* hfree = hfull + 2;            // epilogue -> MMA
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(hfree + 2);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  // One work unit (item in cost order, tile pair) per CTA: u = blockIdx.x.
  // (A persistent variant striding units over 148 CTAs measured slower: the
  // unit costs are uneven and static striding left SMs idle.)
  const uint32_t nunits = items * npairs;
  auto unit_of = [&](uint32_t u, uint32_t& item, uint64_t& t0, uint32_t& e0, uint32_t& e1) {
    item = item_order[u % items];
    t0 = uint64_t(u / items) * 2;
    e0 = item_ent[item];
    e1 = item_ent[item + 1];
  };

  if (tid == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&full[s], kProdWarps * 32);
      mbar_init(&staged[s], kStgWarps);
      mbar_init(&empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&hfull[b], 1);
      mbar_init(&hfree[b], kEpiWarps);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  for (int j = tid; j < D; j += kThreads) reinterpret_cast<float*>(smem + Cfg::OFF_BIAS)[j] = bias[j];
  const uint32_t tab_s = tab_n;  // the launch sizes shared memory for the whole table
  for (uint32_t j = tid; j < tab_s; j += kThreads) reinterpret_cast<float*>(smem + Cfg::OFF_TAB)[j] = tab[j];
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(su32(tmem_slot)),
                 "r"(Cfg::TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp >= kProducerWarp && warp < kMmaWarp) {
    // ------------------------------------------------------------ producers
    const int pt = tid - kProducerWarp * 32;
    const int pw_base = pt - lane;
    constexpr int kRowChunks = 2 * D / 8;  // 16-byte pieces of one hi|lo P16 row
    uint32_t g = 0;  // chunk counter across units
    for (uint32_t u = blockIdx.x; u < nunits; u += gridDim.x) {  // one unit per CTA
      uint32_t item, e0, e1;
      uint64_t t0;
      unit_of(u, item, t0, e0, e1);
      const uint32_t nchunks = (e1 - e0 + kKC - 1) / kKC;
      uint2 rec_next = make_uint2(0, kPad);
      if (lane < int(e1 - e0)) rec_next = ent[e0 + lane];
      for (uint32_t c = 0; c < nchunks; ++c, ++g) {
        const int s = g % kStages;
        const uint32_t base = e0 + c * kKC;
        const int cnt = int(min(uint32_t(kKC), e1 - base));
        const uint2 rec = lane < cnt ? rec_next : make_uint2(0, kPad);
        if (base + kKC + lane < e1) rec_next = ent[base + kKC + lane];
        if (g >= uint32_t(kStages)) F16_WAIT(0, &empty[s], ((g / kStages) - 1) & 1);
        unsigned char* st = smem + s * Cfg::STAGE;
        // P16 rows -> swizzled MN-major B planes (warp-uniform trip counts for the shuffles)
        for (int J0 = pw_base; J0 < cnt * kRowChunks; J0 += kProdWarps * 32) {
          const int J = J0 + lane, k = min(J / kRowChunks, 31), pc = J % kRowChunks;
          const uint32_t x = __shfl_sync(kFull, rec.x, k);
          if (J < cnt * kRowChunks) {
            const int plane = pc / (D / 8), nc = pc % (D / 8), an = nc >> 3, cc = nc & 7, r = k & 7;
            cp_async16(st + plane * Cfg::PLANE + (k >> 3) * Cfg::KSTRIDE + an * 1024 + r * 128 + ((cc ^ r) << 4),
                       P16 + uint64_t(x) * 2 * D + pc * 8);
          }
        }
        for (int J0 = pw_base; J0 < cnt * 16; J0 += kProdWarps * 32) {  // u16 degree rows, 2 tiles
          const int J = J0 + lane, k = min(J >> 4, 31), q = (J >> 3) & 1, ug = J & 7;
          const uint32_t x = __shfl_sync(kFull, rec.x, k);
          if (J < cnt * 16)
            cp_async16(st + Cfg::OFF_DEG + (k * kM + q * kTile + ug * 8) * 2,
                       deg16 + ((t0 + q) * uint64_t(V) + x) * kTile + ug * 8);
        }
        {  // mask words, one u64 per (entry, tile); self -> all ones, pad -> zero
          const int k = pt >> 1, q = pt & 1;
          const uint32_t y = __shfl_sync(kFull, rec.y, k & 31);
          if (k < cnt) {
            const uint64_t* src = y == kSelf ? const_words : (y == kPad ? const_words + 1 : maskt + (t0 + q) * Wp + y);
            cp_async8(st + Cfg::OFF_W + (k * 2 + q) * 8, src);
          }
        }
        asm volatile("cp.async.commit_group;" ::: "memory");
        if (g >= 1) {  // the previous chunk's copies of this thread have landed
          asm volatile("cp.async.wait_group 1;" ::: "memory");
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
          mbar_arrive(&full[(g - 1) % kStages]);
        }
      }
    }
    if (g) {
      asm volatile("cp.async.wait_group 0;" ::: "memory");
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      mbar_arrive(&full[(g - 1) % kStages]);
    }
    prof_flush(0, 1);  // producers: 0 wait empty, 1 total
  } else if (warp >= kEpiWarps && warp < kEpiWarps + kStgWarps) {
    // ------------------------------------------------------------ staging
    const int sw = warp - kEpiWarps, q = sw & 3;  // one warp per TMEM lane quarter
    const int m = q * 32 + lane, tq = m >> 6, i = m & 63;
    const float* stab = reinterpret_cast<const float*>(smem + Cfg::OFF_TAB);
    uint32_t g = 0;
    for (uint32_t u = blockIdx.x; u < nunits; u += gridDim.x) {  // one unit per CTA
      uint32_t item, e0, e1;
      uint64_t t0;
      unit_of(u, item, t0, e0, e1);
      const uint32_t nchunks = (e1 - e0 + kKC - 1) / kKC;
      for (uint32_t c = 0; c < nchunks; ++c, ++g) {
        const int s = g % kStages;
        F16_WAIT(0, &full[s], (g / kStages) & 1);
        tc_fence_after();  // TMEM A stage s: its previous MMAs completed before the producers refilled s
        const unsigned char* st = smem + s * Cfg::STAGE;
        const uint16_t* degs = reinterpret_cast<const uint16_t*>(st + Cfg::OFF_DEG);
        const uint64_t* ws = reinterpret_cast<const uint64_t*>(st + Cfg::OFF_W);
        const int cnt = int(min(uint32_t(kKC), e1 - (e0 + c * kKC)));
#pragma unroll 1
        for (int k0 = 0; k0 < cnt; k0 += 16) {
          uint32_t hv[8], lv[8];
#pragma unroll
          for (int w = 0; w < 16; w += 2) {
            float cf[2];
#pragma unroll
            for (int h = 0; h < 2; ++h) {
              const int k = k0 + w + h;
              const float iv = stab[min(uint32_t(degs[k * kM + m]), tab_s - 1)];
              cf[h] = ((ws[k * 2 + tq] >> i) & 1ull) ? iv * kCoefScale : 0.f;
            }
            split2(cf[0], cf[1], hv[w >> 1], lv[w >> 1]);
          }
          const uint32_t ta = tmem + (uint32_t(q * 32) << 16) + Cfg::A_COL + s * 32 + (k0 >> 1);
          TC_ST8(ta, hv);
          TC_ST8(ta + 16, lv);
        }
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&staged[s]);
      }
    }
    prof_flush(2, 1);  // staging: 2 wait full, 3 total
  } else if (warp == kMmaWarp) {
    // ------------------------------------------------------------ MMA issuer
    uint8_t* sfl = smem + Cfg::OFF_KFL;
    // kind::f16: f32 accumulate, a/b fp16, A K-major (TMEM), B MN-major (bit 16), N = D, M = 128
    const uint32_t idesc = (1u << 4) | (1u << 16) | (uint32_t(D >> 3) << 17) | (uint32_t(kM >> 4) << 24);
    auto bdesc = [](uint32_t addr) {
      uint64_t d = 0;
      d |= uint64_t((addr >> 4) & 0x3FFF);
      d |= uint64_t((1024u >> 4) & 0x3FFF) << 16;                  // LBO: n-atom stride
      d |= uint64_t((uint32_t(Cfg::KSTRIDE) >> 4) & 0x3FFF) << 32;  // SBO: k-group stride
      d |= uint64_t(1) << 46;
      d |= uint64_t(2) << 61;  // SWIZZLE_128B
      return d;
    };
    const uint16_t* sfl16 = reinterpret_cast<const uint16_t*>(sfl);
    uint32_t g = 0, sg = 0, b = 0, acc = 0;
    for (uint32_t u = blockIdx.x; u < nunits; u += gridDim.x) {  // one unit per CTA
      uint32_t item, e0, e1;
      uint64_t t0;
      unit_of(u, item, t0, e0, e1);
      (void)t0;
      const uint32_t nchunks = (e1 - e0 + kKC - 1) / kKC;
      __syncwarp();  // the previous unit's flags are consumed
      for (uint32_t j = lane; j < (e1 - e0) / 16; j += 32) sfl[j] = kflags[e0 / 16 + j];
      __syncwarp();
      for (uint32_t c = 0; c < nchunks; ++c, ++g) {
        const int s = g % kStages;
        F16_WAIT(0, &staged[s], (g / kStages) & 1);
        tc_fence_after();
        const int nk = int(min(uint32_t(kKC), e1 - (e0 + c * kKC))) / 16;
        const uint32_t fw = sfl16[c];
        const uint32_t sb = su32(smem + s * Cfg::STAGE);
        const uint32_t a0 = tmem + Cfg::A_COL + s * 32;
#pragma unroll
        for (int j = 0; j < kKC / 16; ++j) {
          if (j < nk) {
            const uint32_t f = (fw >> (8 * j)) & 0xFFu;
            if (f & 1u) {
              b = sg & 1u;
              if (sg >= 2) {
                F16_WAIT(1, &hfree[b], ((sg >> 1) - 1) & 1);
                tc_fence_after();
              }
              acc = 0;
            }
            const uint32_t d = tmem + b * D, ahi = a0 + j * 8;
            const uint64_t bh = bdesc(sb + Cfg::OFF_BHI + j * 2 * Cfg::KSTRIDE);
            const uint64_t bl = bdesc(sb + Cfg::OFF_BLO + j * 2 * Cfg::KSTRIDE);
            tc_mma_f16_elect(d, ahi, bh, idesc, acc);
            tc_mma_f16_elect(d, ahi, bl, idesc, 1);
            tc_mma_f16_elect(d, ahi + 16, bh, idesc, 1);
            acc = 1;
            if (f & 2u) {
              tc_commit_elect(&hfull[b]);
              ++sg;
            }
          }
        }
        tc_commit_elect(&empty[s]);
      }
    }
    prof_flush(4, 2);  // MMA: 4 wait staged, 5 wait hfree, 6 total
  } else if (warp < kEpiWarps) {
    // ------------------------------------------------------------ epilogue
    constexpr int HALF = D / 2, CW = 16, NCH = HALF / CW;
    const int q = warp & 3;
    const int hb = (warp >> 2) * HALF;
    const int m = q * 32 + lane;
    const int i = m & 63;
    const float* sbias = reinterpret_cast<const float*>(smem + Cfg::OFF_BIAS);
    const float unscale = pscale[1] * (1.f / kCoefScale);  // exact: powers of two
    const uint32_t lane_base = uint32_t(q * 32) << 16;
    const uint32_t acc_col = 2 * D + hb;
    uint32_t r[CW], a[CW];
    uint32_t sgi = 0;  // segment counter across units (H buffer protocol)
    for (uint32_t u = blockIdx.x; u < nunits; u += gridDim.x) {  // one unit per CTA
      uint32_t item, e0, e1;
      uint64_t t0;
      unit_of(u, item, t0, e0, e1);
      const uint64_t tile = t0 + (m >> 6);
      const uint64_t* mt = maskt + tile * Wp;
      const float* isd_t = isd + tile * uint64_t(V) * kTile;
#pragma unroll
      for (int j = 0; j < CW; ++j) a[j] = 0u;
#pragma unroll
      for (int cc = 0; cc < NCH; ++cc) TC_ST16(tmem + lane_base + acc_col + cc * CW, a);
      asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
      const uint32_t s0 = item_seg[item], s1 = item_seg[item + 1];
      auto factors = [&](uint32_t k, float& svk, float& dvk) {
        const uint2 se = seg[k];
        svk = __ldg(&isd_t[uint64_t(se.x) * kTile + i]);
        const bool muv = se.y == kSelf || ((__ldg(&mt[se.y]) >> i) & 1ull);
        dvk = muv ? svk : 0.f;
      };
      float sv, dv;
      factors(s0, sv, dv);
      for (uint32_t k = s0; k < s1; ++k, ++sgi) {
        float sv_next = 0.f, dv_next = 0.f;
        if (k + 1 < s1) factors(k + 1, sv_next, dv_next);
        const uint32_t b = sgi & 1u;
        F16_WAIT(0, &hfull[b], (sgi >> 1) & 1);
        tc_fence_after();
        const float svs = sv * unscale;
#pragma unroll 1
        for (int cc = 0; cc < NCH; ++cc) {
          const uint32_t hcol = tmem + lane_base + b * D + hb + cc * CW;
          const uint32_t acol = tmem + lane_base + acc_col + cc * CW;
          TC_LD16(hcol, r);
          TC_LD16(acol, a);
          asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
          const float4* b4 = reinterpret_cast<const float4*>(sbias + hb + cc * CW);
#pragma unroll
          for (int j4 = 0; j4 < CW / 4; ++j4) {
            const float4 bb = b4[j4];
            const int j = 4 * j4;
            float h0, h1, h2, h3;
            ffma2(h0, h1, svs, svs, __uint_as_float(r[j]), __uint_as_float(r[j + 1]), bb.x, bb.y);
            ffma2(h2, h3, svs, svs, __uint_as_float(r[j + 2]), __uint_as_float(r[j + 3]), bb.z, bb.w);
            h0 = fmaxf(h0, 0.f);
            h1 = fmaxf(h1, 0.f);
            h2 = fmaxf(h2, 0.f);
            h3 = fmaxf(h3, 0.f);
            float a0v, a1v, a2v, a3v;
            ffma2(a0v, a1v, dv, dv, h0, h1, __uint_as_float(a[j]), __uint_as_float(a[j + 1]));
            ffma2(a2v, a3v, dv, dv, h2, h3, __uint_as_float(a[j + 2]), __uint_as_float(a[j + 3]));
            a[j] = __float_as_uint(a0v);
            a[j + 1] = __float_as_uint(a1v);
            a[j + 2] = __float_as_uint(a2v);
            a[j + 3] = __float_as_uint(a3v);
          }
          TC_ST16(acol, a);
        }
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&hfree[b]);
        sv = sv_next;
        dv = dv_next;
      }
      prof_flush(7, 1);  // epilogue: 7 wait hfull, 8 loop total
      float* out = Apart + ((tile * items + item) * kTile + i) * uint64_t(D) + hb;
#pragma unroll 1
      for (int cc = 0; cc < NCH; ++cc) {
        TC_LD16(tmem + lane_base + acc_col + cc * CW, a);
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
        for (int j4 = 0; j4 < CW / 4; ++j4)
          reinterpret_cast<float4*>(out + cc * CW)[j4] =
              make_float4(__uint_as_float(a[4 * j4]), __uint_as_float(a[4 * j4 + 1]),
                          __uint_as_float(a[4 * j4 + 2]), __uint_as_float(a[4 * j4 + 3]));
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if constexpr (PROF) {
    if (tid == 0) {
      atomicAdd(&prof[12], 1ull);
      atomicAdd(&prof[13], (unsigned long long)(clock64() - t_begin));
    }
  }
  if (warp == 0) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(Cfg::TMEM_COLS));
  }
}

// max |P0| by a fixed-shape reduction (one CTA)
__global__ void absmax_kernel(const float* __restrict__ x, uint64_t n, float* __restrict__ out) {
  __shared__ float red[32];
  float m = 0.f;
  for (uint64_t i = threadIdx.x; i < n; i += blockDim.x) m = fmaxf(m, fabsf(x[i]));
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(kFull, m, o));
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = m;
  __syncthreads();
  if (threadIdx.x < 32) {
    m = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : 0.f;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(kFull, m, o));
    if (threadIdx.x == 0) {
      // scale = 2^(14 - e), e = exponent such that max |P0| < 2^e: scaled values stay below 2^14
      const int e = m > 0.f ? ilogbf(m) + 1 : 0;
      out[0] = ldexpf(1.f, 14 - e);
      out[1] = ldexpf(1.f, e - 14);
    }
  }
}

// P16[row] = fp16 hi (D) | fp16 lo (D) of scale * P0[row]
__global__ void split_p16_kernel(const float* __restrict__ P0, uint64_t rows, uint32_t D,
                                 const float* __restrict__ scale, uint16_t* __restrict__ P16) {
  const uint64_t idx = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x;
  if (idx >= rows * D) return;
  const uint64_t r = idx / D, d = idx % D;
  const float v = P0[idx] * scale[0];
  const __half h = __float2half_rn(v);
  const __half l = __float2half_rn(v - __half2float(h));
  P16[r * 2 * D + d] = __half_as_ushort(h);
  P16[r * 2 * D + D + d] = __half_as_ushort(l);
}

template <int D, bool PROF>
void launch_f16_impl(Ctx& ctx, const Engine& e, const uint64_t* maskt, uint64_t Wp, const float* isd,
                     const uint16_t* deg16, uint64_t ntp, float* apart, unsigned long long* prof) {
  using Cfg = F16Cfg<D>;
  set_max_dynamic_smem(fused_f16_kernel<D, PROF>, int(Cfg::SMEM + kTabCap * 4));
  const size_t smem = Cfg::SMEM + size_t(e.isd_tab_n) * 4;
  const uint32_t npairs = uint32_t(ntp / 2), units = e.tc_items * npairs;
  fused_f16_kernel<D, PROF><<<units, kThreads, smem, ctx.stream>>>(
      maskt, Wp, isd, e.V, deg16, e.isd_tab.p, e.isd_tab_n, e.p16.p, e.p16_scale.p, e.b[0]->p,
      reinterpret_cast<const uint2*>(e.tc_ent.p), e.tc_kflags.p, reinterpret_cast<const uint2*>(e.tc_seg.p),
      e.tc_item_ent.p, e.tc_item_seg.p, e.tc_item_order.p, e.tc_items, npairs,
      reinterpret_cast<const uint64_t*>(e.tc_const.p), apart, prof);
  SF_LAUNCHED(ctx);
}

// SF_TC_PROF=1: PROF instantiation, per-role wait breakdown every 100 launches
template <int D>
void launch_f16(Ctx& ctx, const Engine& e, const uint64_t* maskt, uint64_t Wp, const float* isd,
                const uint16_t* deg16, uint64_t ntp, float* apart) {
  static const bool prof_on = std::getenv("SF_TC_PROF") != nullptr;
  if (!prof_on) {
    launch_f16_impl<D, false>(ctx, e, maskt, Wp, isd, deg16, ntp, apart, nullptr);
    return;
  }
  static unsigned long long* dprof = nullptr;
  static uint64_t nlaunch = 0;
  if (!dprof) {
    SF_CUDA(cudaMalloc(&dprof, kProfSites * sizeof(unsigned long long)));
    SF_CUDA(cudaMemset(dprof, 0, kProfSites * sizeof(unsigned long long)));
  }
  launch_f16_impl<D, true>(ctx, e, maskt, Wp, isd, deg16, ntp, apart, dprof);
  if (++nlaunch % 100 == 0) {
    unsigned long long h[kProfSites];
    SF_CUDA(cudaMemcpy(h, dprof, sizeof(h), cudaMemcpyDeviceToHost));
    const double ctas = double(h[12] ? h[12] : 1);
    auto per = [&](int k, int warps) { return double(h[k]) / ctas / warps; };
    std::fprintf(stderr,
                 "[f16 prof] launches %llu CTAs %llu kernel %.0f cyc/CTA | producer wait empty %.0f total %.0f | "
                 "staging wait full %.0f total %.0f | mma wait staged %.0f hfree %.0f total %.0f | epilogue wait "
                 "hfull %.0f loop %.0f\n",
                 (unsigned long long)nlaunch, h[12], double(h[13]) / ctas, per(0, kProdWarps), per(1, kProdWarps),
                 per(2, kStgWarps), per(3, kStgWarps), per(4, 1), per(5, 1), per(6, 1), per(7, kEpiWarps),
                 per(8, kEpiWarps));
  }
}

}  // namespace

bool tc16_width(uint64_t d) { return d == 64 || d == 128; }
uint32_t tc16_max_table() { return uint32_t(kTabCap); }

void prepare_tc16(Ctx& ctx, Engine& e) {
  const uint64_t D = e.dims[1];
  e.p16_scale.reserve(2);
  e.p16.reserve(uint64_t(e.V) * 2 * D);
  absmax_kernel<<<1, 1024, 0, ctx.stream>>>(e.p0.p, uint64_t(e.V) * D, e.p16_scale.p);
  SF_LAUNCHED(ctx);
  const uint64_t n = uint64_t(e.V) * D;
  split_p16_kernel<<<unsigned((n + 255) / 256), 256, 0, ctx.stream>>>(e.p0.p, e.V, uint32_t(D), e.p16_scale.p,
                                                                      e.p16.p);
  SF_LAUNCHED(ctx);
}

bool launch_fused_tc16(Ctx& ctx, const Engine& e, const uint64_t* maskt, uint64_t Wp, const float* isd,
                       const uint16_t* deg16, uint64_t ntp, float* apart) {
  switch (e.dims[1]) {
    case 128: launch_f16<128>(ctx, e, maskt, Wp, isd, deg16, ntp, apart); return true;
    case 64: launch_f16<64>(ctx, e, maskt, Wp, isd, deg16, ntp, apart); return true;
    default: return false;
  }
}

}  // namespace sfb
