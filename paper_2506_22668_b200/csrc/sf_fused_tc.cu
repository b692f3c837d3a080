// Tensor-core (tcgen05) variant of the fused layer-0 -> layer-1 kernel
// (sf_gcn.cu "fused" documents the math). For a work item (u, segments
// v of {u} u N(u)) and two tiles (M = 128 coalitions):
//   H_v[m][:] = sum_{entries k of v} coef[k][m] * P[x_k][:]     (GEMM, K = entries)
//   A_u[m][:] += m_m(e_uv) isd_m(v) relu(isd_m(v) H_v[m][:] + b0)  (per segment)
// The GEMM runs as tcgen05.mma kind::tf32 in 3xTF32 form
// (A_hi B_hi + A_hi B_lo + A_lo B_hi, FP32-level accuracy; a single TF32
// product would miss the 1e-5 prediction bar), with the segment sums H_v
// accumulated in TMEM. Segments are padded to multiples of 8 entries in the
// plan (zero coefficients), so every segment is a whole number of MMA
// k-steps.
//
// Warp roles (640 threads):
//   warps 0-7   epilogue: per finished segment, tcgen05.ld H_v, fold it into
//               the TMEM accumulator A_u, release the H buffer; warps q and
//               q+4 share TMEM lane quarter q and split the columns
//   warps 8-14  staging: per 32-entry chunk build the A (coefficients) and
//               B (gathered P rows, transposed) operand tiles, hi/lo split,
//               both K-major in the canonical no-swizzle layout (MN-major
//               tf32 without swizzle produced no output on B200; see
//               csrc/tools/tc_probe.cu, which checks the layouts exactly)
//   warps 15-18 producers: cp.async gathers of entry records, P rows, isd
//               rows and mask words into a raw ring
//   warp 19     one elected thread issues the MMAs and the commits
// Pipelines: kStages smem stages (full/empty mbarriers), two TMEM H buffers
// (hfull/hfree mbarriers).
#include <cuda_runtime.h>

#include <algorithm>
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
constexpr uint32_t kSelf = 0xFFFFFFFFu;  // coefficient isd(x) (self loop)
constexpr uint32_t kPad = 0xFFFFFFFEu;   // padding entry: coefficient 0
constexpr int kM = 128;                  // coalitions per CTA (two tiles)
constexpr int kKC = 32;                  // entries per chunk (4 MMA k-steps)
#ifndef SF_RAW_STAGES
#define SF_RAW_STAGES 4
#endif
constexpr int kRawStages = SF_RAW_STAGES, kCanStages = 2;
constexpr int kMaxKsteps = 4096;  // per work item (host checks)
constexpr int kEpiWarps = 8, kStgWarps = 8, kProdWarps = 7;
constexpr int kProducerWarp = kEpiWarps + kStgWarps, kMmaWarp = kProducerWarp + kProdWarps;
constexpr int kBLoadWarp = kMmaWarp + 1;  // one warp, one lane: B tiles from the B bank
constexpr int kThreads = (kBLoadWarp + 1) * 32;

constexpr int kTabCap = 8192;  // 1/sqrt table entries in shared memory (u16-degree variant)

template <int D, bool DEG = false>
struct TcCfg {
  // smem stage: B (gathered P rows, K-major) hi | lo; A lives in TMEM
  static constexpr int B_LBO = (D / 8) * 128;          // k-unit stride (n-groups of 8 rows)
  static constexpr int B_BYTES = D * kKC * 4;
  static constexpr int OFF_BHI = 0;
  static constexpr int OFF_BLO = B_BYTES;
  static constexpr int STAGE = ((2 * B_BYTES + 1023) / 1024) * 1024;
  // raw stage: isd rows (2 tiles) | mask words (2 tiles); B tiles come
  // pre-transposed from the B bank straight into the stage
  // isd rows are f32 (4 B) or u16 degrees (2 B, DEG) per coalition
  static constexpr int ISD_ELEM = DEG ? 2 : 4;
  static constexpr int RAW_ISD = 0;
  static constexpr int RAW_W = RAW_ISD + kKC * kM * ISD_ELEM;
  static constexpr int RAW = ((RAW_W + kKC * 2 * 8 + 127) / 128) * 128;
  static constexpr int OFF_RAW = kCanStages * STAGE;
  static constexpr int OFF_KFL = OFF_RAW + kRawStages * RAW;  // the item's k-step flags
  static constexpr int OFF_BIAS = OFF_KFL + kMaxKsteps;      // b0 (D floats)
  static constexpr int OFF_BARS = OFF_BIAS + D * 4;
  static constexpr int OFF_TAB = ((OFF_BARS + 8 * (2 * kRawStages + 3 * kCanStages + 4) + 16 + 15) / 16) * 16;
  static constexpr int SMEM = OFF_TAB + (DEG ? kTabCap * 4 : 0);
  // TMEM columns: H buffers [0, 2D), accumulator [2D, 3D), A stages (hi 32 | lo 32) from 3D
  static constexpr uint32_t A_COL = 3 * D;
  static constexpr uint32_t TMEM_COLS = 3 * D + kCanStages * 2 * kKC <= 256 ? 256 : 512;
  static_assert(3 * D + kCanStages * 2 * kKC <= 512, "TMEM columns");
  static_assert(D % 32 == 0 && D <= 256, "width");
  static_assert(SMEM <= 227 * 1024, "shared memory");
};

__device__ __forceinline__ float tf32_hi(float x) {
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
  return __uint_as_float(r);
}

// entry: (x, e) — P / isd row x, mask player e (kSelf: always kept, kPad:
// coefficient 0). kflags[k-step]: bit0 segment start, bit1 segment end.
// seg: (v, e_uv) per segment in item order.
// PROF instantiation (env SF_TC_PROF): clock64 cycles spent in each
// mbarrier wait and per role, summed over warps into prof[kProfSites].
constexpr int kProfSites = 16;
#define TC_WAIT(site, bar, par)                        \
  do {                                                 \
    if constexpr (PROF) {                              \
      const long long _t = clock64();                  \
      mbar_wait(bar, par);                             \
      pw[site] += uint64_t(clock64() - _t);            \
    } else {                                           \
      mbar_wait(bar, par);                             \
    }                                                  \
  } while (0)

template <int D, bool PROF, bool DEG>
__global__ void __launch_bounds__(kThreads, 1)
    fused_tc_kernel(const uint64_t* __restrict__ maskt, uint64_t Wp, const float* __restrict__ isd,
                    const uint16_t* __restrict__ deg16, const float* __restrict__ tab, uint32_t tab_n,
                    uint32_t V, const float* __restrict__ bbank, const uint32_t* __restrict__ item_chunk,
                    const float* __restrict__ bias,
                    const uint2* __restrict__ ent, const uint8_t* __restrict__ kflags,
                    const uint2* __restrict__ seg, const uint32_t* __restrict__ item_ent,
                    const uint32_t* __restrict__ item_seg, const uint32_t* __restrict__ item_order,
                    uint32_t items, const uint64_t* __restrict__ const_words, float* __restrict__ Apart,
                    unsigned long long* __restrict__ prof) {
  using Cfg = TcCfg<D, DEG>;
  uint64_t pw[3] = {0, 0, 0};
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
  uint64_t* raw_full = bars;                   // producer (expect_tx) -> staging
  uint64_t* raw_empty = raw_full + kRawStages;  // staging -> producer
  uint64_t* can_full = raw_empty + kRawStages;  // staging -> MMA
  uint64_t* can_empty = can_full + kCanStages;  // MMA commit -> staging
  uint64_t* hfull = can_empty + kCanStages;     // MMA commit -> epilogue
  uint64_t* hfree = hfull + 2;                  // epilogue -> MMA
  uint64_t* b_full = hfree + 2;                 // B loader (bulk copy, expect_tx) -> MMA
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(b_full + kCanStages);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const uint32_t item = item_order[blockIdx.x];
  const uint64_t t0 = uint64_t(blockIdx.y) * 2;  // tiles t0, t0+1
  const uint32_t e0 = item_ent[item], e1 = item_ent[item + 1];
  const uint32_t nchunks = (e1 - e0 + kKC - 1) / kKC;

  if (tid == 0) {
    for (int s = 0; s < kRawStages; ++s) {
      mbar_init(&raw_full[s], kProdWarps * 32);
      mbar_init(&raw_empty[s], kStgWarps);
    }
    for (int s = 0; s < kCanStages; ++s) {
      mbar_init(&can_full[s], kStgWarps);
      mbar_init(&can_empty[s], 1);
      mbar_init(&b_full[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&hfull[b], 1);
      mbar_init(&hfree[b], kEpiWarps);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  for (int j = tid; j < D; j += kThreads) reinterpret_cast<float*>(smem + Cfg::OFF_BIAS)[j] = bias[j];
  if constexpr (DEG)
    for (uint32_t j = tid; j < tab_n; j += kThreads) reinterpret_cast<float*>(smem + Cfg::OFF_TAB)[j] = tab[j];
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
    // 16-byte cp.async gathers (LDGSTS) of the chunk's P rows, isd rows
    // (both tiles) and mask words; each producer thread arrives on raw_full
    // once its own copies have landed. (Lane-parallel cp.async.bulk from one
    // warp was measured 2x slower: bulk-copy issue serializes.)
    const int pt = tid - kProducerWarp * 32;
    const int pw_base = pt - lane;  // first J of this warp
    uint2 rec_next = make_uint2(0, kPad);
    if (lane < int(e1 - e0)) rec_next = ent[e0 + lane];
    for (uint32_t c = 0; c < nchunks; ++c) {
      const int r = c % kRawStages;
      const uint32_t base = e0 + c * kKC;
      const int cnt = int(min(uint32_t(kKC), e1 - base));
      const uint2 rec = lane < cnt ? rec_next : make_uint2(0, kPad);
      if (base + kKC + lane < e1) rec_next = ent[base + kKC + lane];
      if (c >= uint32_t(kRawStages)) TC_WAIT(0, &raw_empty[r], ((c / kRawStages) - 1) & 1);
      unsigned char* rw = smem + Cfg::OFF_RAW + r * Cfg::RAW;
      // trip counts are warp-uniform (J0 steps by whole warps), so every lane
      // takes part in the shuffles
      if constexpr (DEG) {
        for (int J0 = pw_base; J0 < cnt * 2 * 8; J0 += kProdWarps * 32) {  // u16 degree rows, 2 tiles
          const int J = J0 + lane, k = min(J >> 4, 31), q = (J >> 3) & 1, ug = J & 7;
          const uint32_t x = __shfl_sync(kFull, rec.x, k);
          if (J < cnt * 2 * 8)
            cp_async16(rw + Cfg::RAW_ISD + (k * kM + q * kTile + ug * 8) * 2,
                       deg16 + ((t0 + q) * uint64_t(V) + x) * kTile + ug * 8);
        }
      } else {
        for (int J0 = pw_base; J0 < cnt * 2 * 16; J0 += kProdWarps * 32) {  // isd rows, 2 tiles
          const int J = J0 + lane, k = min(J >> 5, 31), q = (J >> 4) & 1, ug = J & 15;
          const uint32_t x = __shfl_sync(kFull, rec.x, k);
          if (J < cnt * 2 * 16)
            cp_async16(rw + Cfg::RAW_ISD + (k * kM + q * kTile + ug * 4) * 4,
                       isd + ((t0 + q) * uint64_t(V) + x) * kTile + ug * 4);
        }
      }
      {  // mask words, one u64 per (entry, tile); self -> all ones, pad -> zero
        const int k = pt >> 1, q = pt & 1;
        const uint32_t y = __shfl_sync(kFull, rec.y, k & 31);
        if (k < cnt) {
          const uint64_t* src = y == kSelf ? const_words : (y == kPad ? const_words + 1 : maskt + (t0 + q) * Wp + y);
          cp_async8(rw + Cfg::RAW_W + (k * 2 + q) * 8, src);
        }
      }
      cp_async_arrive(&raw_full[r]);
    }
    prof_flush(0, 1);  // 0 wait raw_empty, 1 total
  } else if (warp >= kEpiWarps && warp < kEpiWarps + kStgWarps) {
    // ------------------------------------------------------------ staging
    const int st_tid = tid - kEpiWarps * 32;
    for (uint32_t c = 0; c < nchunks; ++c) {
      const int r = c % kRawStages, s = c % kCanStages;
      TC_WAIT(0, &raw_full[r], (c / kRawStages) & 1);
      if (c >= uint32_t(kCanStages)) TC_WAIT(1, &can_empty[s], ((c / kCanStages) - 1) & 1);
      tc_fence_after();  // the A stage in TMEM is rewritten after the MMAs that read it
      const unsigned char* rw = smem + Cfg::OFF_RAW + r * Cfg::RAW;
      const float* isds = reinterpret_cast<const float*>(rw + Cfg::RAW_ISD);
      const uint16_t* degs = reinterpret_cast<const uint16_t*>(rw + Cfg::RAW_ISD);
      const float* stab = reinterpret_cast<const float*>(smem + Cfg::OFF_TAB);
      const uint64_t* ws = reinterpret_cast<const uint64_t*>(rw + Cfg::RAW_W);
      unsigned char* st = smem + s * Cfg::STAGE;
      const int cnt = int(min(uint32_t(kKC), e1 - (e0 + c * kKC)));  // multiple of 8
      // A: coefficients m_m(e) isd_m(x) into TMEM (lane = coalition m, column
      // = entry k), hi/lo split. Warp sw covers lane quarter sw % 4 and
      // entries [16 (sw / 4), +16).
      {
        const int sw = warp - kEpiWarps, q = sw & 3, k0 = (sw >> 2) * 16;
        if (k0 < cnt) {
          const int m = q * 32 + lane, tq = m >> 6, i = m & 63;
          uint32_t hv[16], lv[16];
#pragma unroll
          for (int w = 0; w < 16; ++w) {
            const int k = k0 + w;
            float iv;
            // entries past the chunk's count hold stale stage data (their
            // k-steps are not issued): keep the table index in range
            if constexpr (DEG) iv = stab[degs[k * kM + m] & (kTabCap - 1)];
            else iv = isds[k * kM + m];
            const float cf = ((ws[k * 2 + tq] >> i) & 1ull) ? iv : 0.f;
            const float h = tf32_hi(cf);
            hv[w] = __float_as_uint(h);
            lv[w] = __float_as_uint(cf - h);
          }
          const uint32_t ta = tmem + (uint32_t(q * 32) << 16) + Cfg::A_COL + s * 2 * kKC + k0;
          TC_ST16(ta, hv);
          TC_ST16(ta + kKC, lv);
          asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
        }
      }
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      tc_fence_before();
      __syncwarp();
      if (lane == 0) {
        mbar_arrive(&raw_empty[r]);
        mbar_arrive(&can_full[s]);
      }
    }
    prof_flush(2, 2);  // 2 wait raw_full, 3 wait can_empty, 4 total
  } else if (warp == kMmaWarp) {
    // ------------------------------------------------------------ MMA issuer
    uint8_t* sfl = smem + Cfg::OFF_KFL;
    for (uint32_t j = lane; j < (e1 - e0) / 8; j += 32) sfl[j] = kflags[e0 / 8 + j];
    __syncwarp();
    {
      // The whole warp runs the loop (warp-uniform values), one elected lane
      // issues each MMA / commit. kind::tf32, D f32, A (TMEM) and B (smem) K-major, N = D, M = 128.
      // The issue loop is kept short (MMA issue latency, not the tensor
      // pipe, bounds a looped issuer; csrc/tools/tc_rate_probe.cu):
      // descriptors are per-stage bases plus constant k-step offsets, the
      // chunk's four k-step flags come from one 32-bit load.
      const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | (uint32_t(D >> 3) << 17) |
                             (uint32_t(kM >> 4) << 24);
      uint64_t bhi0[kCanStages], blo0[kCanStages];
#pragma unroll
      for (int st2 = 0; st2 < kCanStages; ++st2) {
        const uint32_t sa = su32(smem + st2 * Cfg::STAGE);
        bhi0[st2] = smem_desc(sa + Cfg::OFF_BHI, Cfg::B_LBO, 128);
        blo0[st2] = smem_desc(sa + Cfg::OFF_BLO, Cfg::B_LBO, 128);
      }
      constexpr uint64_t kStep = uint64_t(2 * Cfg::B_LBO) >> 4;  // descriptor address units per k-step
      const uint32_t* sfl32 = reinterpret_cast<const uint32_t*>(sfl);
      uint32_t sg = 0, b = 0, acc = 0;
      for (uint32_t c = 0; c < nchunks; ++c) {
        const int s = c % kCanStages;
        TC_WAIT(0, &can_full[s], (c / kCanStages) & 1);
        mbar_wait(&b_full[s], (c / kCanStages) & 1);
        tc_fence_after();
        const int nk = int(min(uint32_t(kKC), e1 - (e0 + c * kKC))) / 8;
        const uint32_t fw = sfl32[c];
        const uint32_t a0 = tmem + Cfg::A_COL + s * 2 * kKC;
        static_assert(kCanStages == 2, "stage select below");
        const uint64_t bhs = s ? bhi0[1] : bhi0[0], bls = s ? blo0[1] : blo0[0];
#pragma unroll
        for (int j = 0; j < kKC / 8; ++j) {
          if (j < nk) {
            const uint32_t f = (fw >> (8 * j)) & 0xFFu;
            if (f & 1u) {
              b = sg & 1u;
              if (sg >= 2) {
                TC_WAIT(1, &hfree[b], ((sg >> 1) - 1) & 1);
                tc_fence_after();
              }
              acc = 0;
            }
            const uint32_t d = tmem + b * D, ahi = a0 + j * 8;
            const uint64_t bh = bhs + j * kStep, bl = bls + j * kStep;
            tc_mma_ts_elect(d, ahi, bh, idesc, acc);
            tc_mma_ts_elect(d, ahi, bl, idesc, 1);
            tc_mma_ts_elect(d, ahi + kKC, bh, idesc, 1);
            acc = 1;
            if (f & 2u) {
              tc_commit_elect(&hfull[b]);
              ++sg;
            }
          }
        }
        tc_commit_elect(&can_empty[s]);
      }
      prof_flush(6, 2);  // 6 wait can_full, 7 wait hfree, 8 total
    }
  } else if (warp == kBLoadWarp) {
    // ------------------------------------------------------------ B loader
    // The chunk's B operand (P0 rows of its entries, K-major, tf32 hi | lo)
    // is the same for every tile pair: one bulk copy from the B bank.
    if (lane == 0) {
      const float* src = bbank + uint64_t(item_chunk[item]) * (2 * Cfg::B_BYTES / 4);
      for (uint32_t c = 0; c < nchunks; ++c) {
        const int s = c % kCanStages;
        if (c >= uint32_t(kCanStages)) mbar_wait(&can_empty[s], ((c / kCanStages) - 1) & 1);
        mbar_arrive_expect_tx(&b_full[s], 2 * Cfg::B_BYTES);
        bulk_g2s(smem + s * Cfg::STAGE, src + uint64_t(c) * (2 * Cfg::B_BYTES / 4), 2 * Cfg::B_BYTES, &b_full[s]);
      }
    }
  } else if (warp < kEpiWarps) {
    // ------------------------------------------------------------ epilogue
    // warp w: TMEM lane quarter w % 4 (coalitions), columns [hb, hb + D/2)
    constexpr int HALF = D / 2, CW = 16, NCH = HALF / CW;
    const int q = warp & 3;
    const int hb = (warp >> 2) * HALF;
    const int m = q * 32 + lane;
    const uint64_t tile = t0 + (m >> 6);
    const int i = m & 63;
    const uint64_t* mt = maskt + tile * Wp;
    const float* isd_t = DEG ? nullptr : isd + tile * uint64_t(V) * kTile;
    const uint16_t* deg_t = DEG ? deg16 + tile * uint64_t(V) * kTile : nullptr;
    const float* stab_e = reinterpret_cast<const float*>(smem + Cfg::OFF_TAB);
    const float* sbias = reinterpret_cast<const float*>(smem + Cfg::OFF_BIAS);
    const uint32_t lane_base = uint32_t(q * 32) << 16;
    const uint32_t acc_col = 2 * D + hb;
    uint32_t r[CW], a[CW];
#pragma unroll
    for (int j = 0; j < CW; ++j) a[j] = 0u;
#pragma unroll
    for (int cc = 0; cc < NCH; ++cc) {
      if constexpr (CW == 32) TC_ST32(tmem + lane_base + acc_col + cc * CW, a);
      else TC_ST16(tmem + lane_base + acc_col + cc * CW, a);
    }
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    const uint32_t s0 = item_seg[item], s1 = item_seg[item + 1];
    auto factors = [&](uint32_t k, float& svk, float& dvk) {
      const uint2 se = seg[k];
      if constexpr (DEG) svk = stab_e[__ldg(&deg_t[uint64_t(se.x) * kTile + i])];
      else svk = __ldg(&isd_t[uint64_t(se.x) * kTile + i]);
      const bool muv = se.y == kSelf || ((__ldg(&mt[se.y]) >> i) & 1ull);
      dvk = muv ? svk : 0.f;
    };
    float sv, dv;
    factors(s0, sv, dv);
    for (uint32_t sg = 0; sg < s1 - s0; ++sg) {
      float sv_next = 0.f, dv_next = 0.f;
      if (s0 + sg + 1 < s1) factors(s0 + sg + 1, sv_next, dv_next);  // in flight during the wait
      const uint32_t b = sg & 1u;
      TC_WAIT(0, &hfull[b], (sg >> 1) & 1);
      tc_fence_after();
#pragma unroll 1
      for (int cc = 0; cc < NCH; ++cc) {
        const uint32_t hcol = tmem + lane_base + b * D + hb + cc * CW;
        const uint32_t acol = tmem + lane_base + acc_col + cc * CW;
        if constexpr (CW == 32) {
          TC_LD32(hcol, r);
          TC_LD32(acol, a);
        } else {
          TC_LD16(hcol, r);
          TC_LD16(acol, a);
        }
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        const float4* b4 = reinterpret_cast<const float4*>(sbias + hb + cc * CW);
#pragma unroll
        for (int j4 = 0; j4 < CW / 4; ++j4) {
          const float4 bb = b4[j4];
          const int j = 4 * j4;
          float h0, h1, h2, h3;
          ffma2(h0, h1, sv, sv, __uint_as_float(r[j]), __uint_as_float(r[j + 1]), bb.x, bb.y);
          ffma2(h2, h3, sv, sv, __uint_as_float(r[j + 2]), __uint_as_float(r[j + 3]), bb.z, bb.w);
          h0 = fmaxf(h0, 0.f);
          h1 = fmaxf(h1, 0.f);
          h2 = fmaxf(h2, 0.f);
          h3 = fmaxf(h3, 0.f);
          float a0, a1, a2, a3;
          ffma2(a0, a1, dv, dv, h0, h1, __uint_as_float(a[j]), __uint_as_float(a[j + 1]));
          ffma2(a2, a3, dv, dv, h2, h3, __uint_as_float(a[j + 2]), __uint_as_float(a[j + 3]));
          a[j] = __float_as_uint(a0);
          a[j + 1] = __float_as_uint(a1);
          a[j + 2] = __float_as_uint(a2);
          a[j + 3] = __float_as_uint(a3);
        }
        if constexpr (CW == 32) TC_ST32(acol, a);
        else TC_ST16(acol, a);
      }
      asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&hfree[b]);
      sv = sv_next;
      dv = dv_next;
    }
    prof_flush(9, 1);  // 9 wait hfull, 10 total before the write-out
    // write the accumulator: Apart[tile][item][i][hb ..]
    float* out = Apart + ((tile * items + item) * kTile + i) * uint64_t(D) + hb;
#pragma unroll 1
    for (int cc = 0; cc < NCH; ++cc) {
      if constexpr (CW == 32) TC_LD32(tmem + lane_base + acc_col + cc * CW, a);
      else TC_LD16(tmem + lane_base + acc_col + cc * CW, a);
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
      for (int j4 = 0; j4 < CW / 4; ++j4)
        reinterpret_cast<float4*>(out + cc * CW)[j4] =
            make_float4(__uint_as_float(a[4 * j4]), __uint_as_float(a[4 * j4 + 1]),
                        __uint_as_float(a[4 * j4 + 2]), __uint_as_float(a[4 * j4 + 3]));
    }
  }
  if constexpr (PROF) {  // 11 epilogue incl. write-out, 12 CTAs, 13 kernel
    if (warp < kEpiWarps && lane == 0) atomicAdd(&prof[11], (unsigned long long)(clock64() - t_begin));
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


// B bank: for every chunk of every item, the K-major tf32 hi | lo B tile of
// the chunk's P0 rows (entries past the chunk end are zero). One CTA per
// chunk; thread = (feature n, 4 entries), the same layout the staging warps
// used to build per tile pair.
template <int D>
__global__ void __launch_bounds__(256)
    build_bbank_kernel(const float* __restrict__ P, const uint2* __restrict__ ent,
                       const uint32_t* __restrict__ chunk_ent, float* __restrict__ bank) {
  using Cfg = TcCfg<D>;
  const uint32_t ci = blockIdx.x, base = chunk_ent[2 * ci], cnt = chunk_ent[2 * ci + 1];
  unsigned char* out = reinterpret_cast<unsigned char*>(bank + uint64_t(ci) * (2 * Cfg::B_BYTES / 4));
  for (int J = threadIdx.x; J < D * (kKC / 4); J += blockDim.x) {
    const int n = J % D, u = J / D;
    float pv[4];
#pragma unroll
    for (int w = 0; w < 4; ++w) {
      const uint32_t k = 4 * u + w;
      pv[w] = k < cnt ? __ldg(&P[uint64_t(ent[base + k].x) * D + n]) : 0.f;
    }
    float4 hi;
    hi.x = tf32_hi(pv[0]);
    hi.y = tf32_hi(pv[1]);
    hi.z = tf32_hi(pv[2]);
    hi.w = tf32_hi(pv[3]);
    const float4 lo = make_float4(pv[0] - hi.x, pv[1] - hi.y, pv[2] - hi.z, pv[3] - hi.w);
    const uint32_t off = u * Cfg::B_LBO + (n >> 3) * 128 + (n & 7) * 16;
    *reinterpret_cast<float4*>(out + Cfg::OFF_BHI + off) = hi;
    *reinterpret_cast<float4*>(out + Cfg::OFF_BLO + off) = lo;
  }
}

template <int D, bool PROF, bool DEG>
void launch_tc_impl(Ctx& ctx, const Engine& e, const uint64_t* maskt, uint64_t Wp, const float* isd,
                    const uint16_t* deg16, uint64_t ntp, float* apart, unsigned long long* prof) {
  using Cfg = TcCfg<D, DEG>;
  set_max_dynamic_smem(fused_tc_kernel<D, PROF, DEG>, int(Cfg::SMEM));
  const size_t smem = Cfg::SMEM;
  dim3 grid(e.tc_items, unsigned(ntp / 2));
  fused_tc_kernel<D, PROF, DEG><<<grid, kThreads, smem, ctx.stream>>>(
      maskt, Wp, isd, deg16, e.isd_tab.p, e.isd_tab_n, e.V, e.tc_bbank.p, e.tc_item_chunk.p, e.b[0]->p,
      reinterpret_cast<const uint2*>(e.tc_ent.p), e.tc_kflags.p, reinterpret_cast<const uint2*>(e.tc_seg.p),
      e.tc_item_ent.p, e.tc_item_seg.p, e.tc_item_order.p, e.tc_items, reinterpret_cast<const uint64_t*>(e.tc_const.p),
      apart, prof);
  SF_LAUNCHED(ctx);
}

// SF_TC_PROF=1: run the PROF instantiation and print the per-role wait
// breakdown (cycles per warp per CTA) every 100 launches to stderr.
template <int D>
void launch_tc(Ctx& ctx, const Engine& e, const uint64_t* maskt, uint64_t Wp, const float* isd,
               const uint16_t* deg16, uint64_t ntp, float* apart) {
  static const bool prof_on = std::getenv("SF_TC_PROF") != nullptr;
  if (!prof_on) {
    if (deg16) launch_tc_impl<D, false, true>(ctx, e, maskt, Wp, isd, deg16, ntp, apart, nullptr);
    else launch_tc_impl<D, false, false>(ctx, e, maskt, Wp, isd, deg16, ntp, apart, nullptr);
    return;
  }
  static unsigned long long* dprof = nullptr;
  static uint64_t nlaunch = 0;
  if (!dprof) {
    SF_CUDA(cudaMalloc(&dprof, kProfSites * sizeof(unsigned long long)));
    SF_CUDA(cudaMemset(dprof, 0, kProfSites * sizeof(unsigned long long)));
  }
  if (deg16) launch_tc_impl<D, true, true>(ctx, e, maskt, Wp, isd, deg16, ntp, apart, dprof);
  else launch_tc_impl<D, true, false>(ctx, e, maskt, Wp, isd, deg16, ntp, apart, dprof);
  if (++nlaunch % 100 == 0) {
    unsigned long long h[kProfSites];
    SF_CUDA(cudaMemcpy(h, dprof, sizeof(h), cudaMemcpyDeviceToHost));
    const double ctas = double(h[12] ? h[12] : 1);
    auto per = [&](int k, int warps) { return double(h[k]) / ctas / warps; };
    std::fprintf(stderr,
                 "[tc prof] launches %llu CTAs %llu kernel %.0f cyc/CTA | producer wait raw_empty %.0f total %.0f | "
                 "staging wait raw_full %.0f can_empty %.0f total %.0f | mma wait can_full %.0f hfree %.0f total %.0f | "
                 "epilogue wait hfull %.0f loop %.0f with write %.0f\n",
                 (unsigned long long)nlaunch, h[12], double(h[13]) / ctas, per(0, kProdWarps), per(1, kProdWarps),
                 per(2, kStgWarps), per(3, kStgWarps), per(4, kStgWarps), per(6, 1), per(7, 1), per(8, 1),
                 per(9, kEpiWarps), per(10, kEpiWarps), per(11, kEpiWarps));
  }
}

}  // namespace

bool tc_width(uint64_t d) { return d == 32 || d == 64 || d == 128; }
uint32_t tc_deg_table_cap() { return uint32_t(kTabCap); }

// Padded entries / k-step flags / segments / items for the tensor-core path
// (segments padded to multiples of e.tc_kstep entries).
void build_tc_plan(Ctx& ctx, Engine& e, const Subgraph& sg) {
  const uint32_t U = uint32_t(e.ball[e.L - 2]);
  // padded entries per work item (per-CTA pipeline fill/drain and item
  // partials for the tail vs wave quantization). C2 value ms/step with the
  // B bank, 768 MB batches and the 16-coalition tail: 768: 51.3, 1024: 49.2,
  // 1536: 48.3, 2048: 47.4, 3072: 47.5, 4096: 48.4, 8192: 50.8.
  // SF_TC_ITEM overrides for experiments.
  static const uint64_t kItem =
      std::getenv("SF_TC_ITEM") ? std::strtoull(std::getenv("SF_TC_ITEM"), nullptr, 10) : 2048;
  std::vector<uint32_t> ent;        // 2 words per entry
  std::vector<uint8_t> kfl;         // per 8 entries
  std::vector<uint32_t> segs;       // 2 words per segment
  std::vector<uint32_t> item_ent{0}, item_seg{0}, u_items{0};
  std::vector<uint64_t> work;
  for (uint32_t u = 0; u < U; ++u) {
    uint64_t open = 0;
    auto close = [&]() {
      if (ent.size() / 2 > item_ent.back()) {
        item_ent.push_back(uint32_t(ent.size() / 2));
        item_seg.push_back(uint32_t(segs.size() / 2));
        work.push_back(open);
        open = 0;
      }
    };
    const uint64_t ks = e.tc_kstep;  // entries per MMA k-step (8 tf32, 16 fp16)
    auto segment = [&](uint32_t v, uint32_t euv) {
      const uint64_t w = sg.row_ptr[v + 1] - sg.row_ptr[v] + 1;
      const uint64_t padded = (w + ks - 1) / ks * ks;
      if (open && open + padded > kItem) close();
      const size_t k0 = ent.size() / 2;
      ent.insert(ent.end(), {v, kSelf});
      for (uint64_t k = sg.row_ptr[v]; k < sg.row_ptr[v + 1]; ++k)
        ent.insert(ent.end(), {sg.col[k], sg.edge_player[k]});
      for (uint64_t k = w; k < padded; ++k) ent.insert(ent.end(), {v, kPad});
      const size_t nk = padded / ks;
      for (size_t j = 0; j < nk; ++j) kfl.push_back(uint8_t((j == 0 ? 1 : 0) | (j + 1 == nk ? 2 : 0)));
      (void)k0;
      segs.insert(segs.end(), {v, euv});
      open += padded;
    };
    segment(u, kSelf);
    for (uint64_t k = sg.row_ptr[u]; k < sg.row_ptr[u + 1]; ++k) segment(sg.col[k], sg.edge_player[k]);
    close();
    u_items.push_back(uint32_t(item_ent.size() - 1));
  }
  for (size_t it = 0; it + 1 < item_ent.size(); ++it)
    if ((item_ent[it + 1] - item_ent[it]) / e.tc_kstep > uint32_t(kMaxKsteps)) {
      e.tc = false;  // a segment too long for the kernel's flag buffer: SIMT kernel
      return;
    }
  std::vector<uint32_t> order(work.size());
  for (uint32_t i = 0; i < order.size(); ++i) order[i] = i;
  std::stable_sort(order.begin(), order.end(), [&](uint32_t a, uint32_t b) { return work[a] > work[b]; });
  e.tc_items = uint32_t(work.size());
  e.tc_entries = ent.size() / 2;
  const uint32_t consts[4] = {0xFFFFFFFFu, 0xFFFFFFFFu, 0u, 0u};  // u64 all-ones, u64 zero
  e.tc_const.upload(consts, 4, ctx.stream);
  e.tc_ent.upload(ent.data(), ent.size(), ctx.stream);
  e.tc_kflags.upload(kfl.data(), kfl.size(), ctx.stream);
  e.tc_seg.upload(segs.data(), segs.size(), ctx.stream);
  e.tc_item_ent.upload(item_ent.data(), item_ent.size(), ctx.stream);
  e.tc_item_seg.upload(item_seg.data(), item_seg.size(), ctx.stream);
  e.tc_item_order.upload(order.data(), order.size(), ctx.stream);
  e.tc_u_items.upload(u_items.data(), u_items.size(), ctx.stream);
  ctx.h2d_bytes += ent.size() * 4 + kfl.size() + segs.size() * 4 +
                   (item_ent.size() + item_seg.size() + order.size() + u_items.size()) * 4;
  if (!e.tc16) {  // B bank for the 3xTF32 kernel: one pre-transposed B tile per chunk
    std::vector<uint32_t> item_chunk(work.size()), chunk_ent;
    uint32_t nch = 0;
    for (size_t it = 0; it + 1 < item_ent.size(); ++it) {
      item_chunk[it] = nch;
      for (uint32_t b0 = item_ent[it]; b0 < item_ent[it + 1]; b0 += kKC) {
        chunk_ent.push_back(b0);
        chunk_ent.push_back(std::min<uint32_t>(kKC, item_ent[it + 1] - b0));
        ++nch;
      }
    }
    e.tc_item_chunk.upload(item_chunk.data(), item_chunk.size(), ctx.stream);
    e.tc_chunk_ent.upload(chunk_ent.data(), chunk_ent.size(), ctx.stream);
    ctx.h2d_bytes += (item_chunk.size() + chunk_ent.size()) * 4;
    const uint32_t D = uint32_t(e.dims[1]);
    e.tc_bbank.reserve(uint64_t(nch) * 2 * D * kKC);
    if (nch) {
      switch (D) {
        case 128: build_bbank_kernel<128><<<nch, 256, 0, ctx.stream>>>(e.p0.p, reinterpret_cast<const uint2*>(e.tc_ent.p), e.tc_chunk_ent.p, e.tc_bbank.p); break;
        case 64: build_bbank_kernel<64><<<nch, 256, 0, ctx.stream>>>(e.p0.p, reinterpret_cast<const uint2*>(e.tc_ent.p), e.tc_chunk_ent.p, e.tc_bbank.p); break;
        case 32: build_bbank_kernel<32><<<nch, 256, 0, ctx.stream>>>(e.p0.p, reinterpret_cast<const uint2*>(e.tc_ent.p), e.tc_chunk_ent.p, e.tc_bbank.p); break;
        default: throw std::logic_error("B bank width");
      }
      SF_LAUNCHED(ctx);
    }
  }
  SF_CUDA(cudaStreamSynchronize(ctx.stream));
}

bool launch_fused_tc(Ctx& ctx, const Engine& e, const uint64_t* maskt, uint64_t Wp, const float* isd,
                     const uint16_t* deg16, uint64_t ntp, float* apart) {
  switch (e.dims[1]) {
    case 128: launch_tc<128>(ctx, e, maskt, Wp, isd, deg16, ntp, apart); return true;
    case 64: launch_tc<64>(ctx, e, maskt, Wp, isd, deg16, ntp, apart); return true;
    case 32: launch_tc<32>(ctx, e, maskt, Wp, isd, deg16, ntp, apart); return true;
    default: return false;
  }
}

}  // namespace sfb
