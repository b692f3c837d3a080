// Masked-GCN inference engine for sm_100a (replaces evaluate_masks,
// gcn.cpp:40-156, behind predict_batched / predict_probs).
//
// Coalitions are processed in tiles of 64 mask rows. Per tile the engine
// keeps ("data layout in HBM"):
//   maskt[t][e]      u64, bit i = row t*64+i keeps player e (transposed so
//                    one 8-byte load serves all 64 coalitions of a tile)
//   isd[t][u][i]     f32 1/sqrt(deg) of node u under coalition i
//   H_l[t][r][i][f]  f32 layer outputs for the rows each layer needs
// Layer 0 is evaluated transform-first, A_i (X W0) with X W0 computed once
// per target (the reference aggregates first; the reassociation is within
// ~1e-6 relative). Layer l produces only the rows of
// the (L-1-l)-hop ball, which is a prefix of the BFS-ordered local ids; the
// last layer produces only the target row (gcn.cpp:134-140).
//
// Arithmetic: FP32 (FFMA) in the SIMT kernels of this file; the default
// layer-0 path is the tcgen05 3xTF32 kernel in sf_fused_tc.cu.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>

#include "sf_device.cuh"
#include "sf_internal.hpp"

namespace sfb {

namespace {

constexpr int kTile = 64;  // coalitions per tile

// ---------------------------------------------------------------- degrees
// deg_i(u) = 1 + sum over u's CSR entries of bit_i(edge_player) (the
// self-loop counts, gcn.cpp:76-81), isd = 1/sqrt(deg) read from a table of
// the correctly rounded values (inv_sqrt_deg, bitwise equal to gcn.cpp:82).
// Nodes are taken in descending degree order (hubs first). A node with more
// than 32 incidences ("big", the first nbig in that order) gets one warp per
// tile and counts 32-incidence chunks; any other node gets one warp for all
// tiles, with G = next power of two >= degree incidence slots per tile and
// 32/G tiles per pass. Each pass loads one mask word per lane (row j = tile
// j/G, incidence j%G), transposes the 32 x 64 bit block with a butterfly so
// lane l holds coalitions l and l+32, and counts each tile's G-bit field
// with popc.
// 32x32 bit transpose across a warp: lane l ends with bit j = bit l of lane
// j's input. Per stage s each lane sends rot(x) & keep (rotate right by s,
// or by 32 - s on lanes with bit s set) and keeps x & keep; the per-lane
// rotate amounts and keep masks are computed once (Bfly).
struct Bfly {
  uint32_t keep[5], amt[5];
  __device__ __forceinline__ explicit Bfly(int lane) {
#pragma unroll
    for (int q = 0; q < 5; ++q) {
      const int sh = 16 >> q;
      const uint32_t m = sh == 16 ? 0x0000FFFFu : sh == 8 ? 0x00FF00FFu : sh == 4 ? 0x0F0F0F0Fu
                       : sh == 2 ? 0x33333333u : 0x55555555u;
      keep[q] = (lane & sh) ? ~m : m;
      amt[q] = (lane & sh) ? 32 - sh : sh;
    }
  }
  __device__ __forceinline__ uint32_t operator()(uint32_t x) const {
#pragma unroll
    for (int q = 0; q < 5; ++q) {
      const uint32_t send = __funnelshift_r(x, x, amt[q]) & keep[q];
      x = (x & keep[q]) | __shfl_xor_sync(kFull, send, 16 >> q);
    }
    return x;
  }
};

__global__ void __launch_bounds__(256)
    isd_kernel(const uint64_t* __restrict__ maskt, uint64_t Wp, uint32_t ntiles,
               const uint32_t* __restrict__ row_ptr,
               const uint32_t* __restrict__ ep, const uint32_t* __restrict__ order,
               uint32_t nbig, const float* __restrict__ tab, uint32_t V,
               float* __restrict__ isd, uint16_t* __restrict__ deg16,
               uint32_t tsplit, uint32_t tchunk, uint32_t f32_nodes, uint32_t f32_stride) {
  const int lane = threadIdx.x & 31;
  const Bfly bfly32(lane);
  const uint32_t w = blockIdx.x * 8 + (threadIdx.x >> 5);
  const uint32_t big_warps = nbig * ntiles;
  if (w < big_warps) {  // hub: one tile, 32-incidence chunks
    const uint32_t u = order[w / ntiles];
    const uint64_t t = w % ntiles;
    const uint64_t* mt = maskt + t * Wp;
    uint32_t clo = 1, chi = 1;
    const uint32_t beg = row_ptr[u], end = row_ptr[u + 1];
    uint32_t i = beg + lane;
    for (; i + 32 - lane < end; i += 64) {  // two chunks in flight
      const uint64_t x0 = __ldg(&mt[__ldg(&ep[i])]);
      const uint64_t x1 = i + 32 < end ? __ldg(&mt[__ldg(&ep[i + 32])]) : 0ull;
      clo += __popc(bfly32(uint32_t(x0))) + __popc(bfly32(uint32_t(x1)));
      chi += __popc(bfly32(uint32_t(x0 >> 32))) + __popc(bfly32(uint32_t(x1 >> 32)));
    }
    for (; i - lane < end; i += 32) {
      const uint64_t x = i < end ? __ldg(&mt[__ldg(&ep[i])]) : 0ull;
      clo += __popc(bfly32(uint32_t(x)));
      chi += __popc(bfly32(uint32_t(x >> 32)));
    }
    if (isd && u < f32_nodes) {
      float* out = isd + (t * f32_stride + u) * kTile;
      __stcs(&out[lane], __ldg(&tab[clo]));
      __stcs(&out[lane + 32], __ldg(&tab[chi]));
    }
    if (deg16) {
      uint16_t* o16 = deg16 + (t * V + u) * kTile;
      o16[lane] = uint16_t(min(clo, 0xFFFFu));
      o16[lane + 32] = uint16_t(min(chi, 0xFFFFu));
    }
    return;
  }
  // small nodes: warp per (node, chunk of tchunk tiles); tsplit chunks per
  // node so that few-node subgraphs still fill the GPU
  const uint32_t j = nbig + (w - big_warps) / tsplit;
  if (j >= V) return;
  const uint32_t tb0 = ((w - big_warps) % tsplit) * tchunk;
  const uint32_t te = min(ntiles, tb0 + tchunk);
  const uint32_t u = order[j];
  const uint32_t beg = row_ptr[u], deg = row_ptr[u + 1] - beg;
  if (deg == 0) {
    const float one = __ldg(&tab[1]);
    for (uint32_t t = tb0; t < te; ++t) {
      if (isd && u < f32_nodes) {
        float* out = isd + (uint64_t(t) * f32_stride + u) * kTile;
        out[lane] = one;
        out[lane + 32] = one;
      }
      if (deg16) {
        deg16[(uint64_t(t) * V + u) * kTile + lane] = 1;
        deg16[(uint64_t(t) * V + u) * kTile + lane + 32] = 1;
      }
    }
    return;
  }
  const int lg = deg <= 1 ? 0 : 32 - __clz(deg - 1);  // G = 1 << lg >= deg
  const uint32_t G = 1u << lg, per = 32u >> lg;
  const uint32_t slot = lane & (G - 1), sub = lane >> lg;
  const uint32_t p = slot < deg ? __ldg(&ep[beg + slot]) : 0u;
  const uint32_t fmask = G == 32 ? 0xFFFFFFFFu : (1u << G) - 1u;
  // kIsdAhead groups of `per` tiles per step: their mask words are all in
  // flight before the first transpose (the loop is latency-bound otherwise)
#ifndef SF_ISD_AHEAD
#define SF_ISD_AHEAD 4
#endif
  constexpr int kIsdAhead = SF_ISD_AHEAD;
  for (uint32_t t0 = tb0; t0 < te; t0 += kIsdAhead * per) {
    uint64_t xs[kIsdAhead];
#pragma unroll
    for (int k = 0; k < kIsdAhead; ++k) {
      const uint32_t t = t0 + k * per + sub;
      xs[k] = (slot < deg && t < te) ? __ldg(&maskt[uint64_t(t) * Wp + p]) : 0ull;
    }
#pragma unroll
    for (int k = 0; k < kIsdAhead; ++k) {
      const uint32_t tb = t0 + k * per;
      if (tb >= te) continue;  // warp-uniform (continue, not break: xs stays in registers)
      const uint32_t lo = bfly32(uint32_t(xs[k])), hi = bfly32(uint32_t(xs[k] >> 32));
      for (uint32_t q = 0; q < per && tb + q < te; ++q) {
        const uint32_t sh = q << lg;
        const uint32_t dlo = 1 + __popc((lo >> sh) & fmask), dhi = 1 + __popc((hi >> sh) & fmask);
        if (isd && u < f32_nodes) {
          float* out = isd + (uint64_t(tb + q) * f32_stride + u) * kTile;
          __stcs(&out[lane], __ldg(&tab[dlo]));
          __stcs(&out[lane + 32], __ldg(&tab[dhi]));
        }
        if (deg16) {
          uint16_t* o16 = deg16 + (uint64_t(tb + q) * V + u) * kTile;
          o16[lane] = uint16_t(dlo);
          o16[lane + 32] = uint16_t(dhi);
        }
      }
    }
  }
}

__global__ void isd_table_kernel(float* tab, uint32_t n) {
  const uint32_t d = blockIdx.x * blockDim.x + threadIdx.x;
  if (d < n) tab[d] = inv_sqrt_deg(d);
}

// ---------------------------------------------------------------- fused
// Layer 0 evaluated on the fly and aggregated straight into the next layer
// (DESIGN.md "fused engine"). For a work item (u, segments v_a..v_b of
// {u} u N(u)) and the 64 coalitions i of tile t:
//   h_i(v)   = relu(isd_i(v) * sum_{x in {v} u kept N(v)} isd_i(x) P[x] + b0)
//   Apart_i  = sum_v m_i(e_uv) isd_i(v) h_i(v)       (isd_i(u) applied later)
// P = X W0 is shared by all coalitions: each gathered P row is read once per
// tile and reused by the 64 coalitions; layer-0 rows never reach memory.
//
// Pipeline (per CTA = one item x one tile): warp 8 is a producer that
// streams, 32 entries per chunk, the entry records, the P rows, the isd rows
// and the mask words of the chunk into a kStages-deep shared-memory ring
// with cp.async.bulk (TMA bulk copies completing on an mbarrier). Warps 0-7
// consume: they turn (mask bit, isd) into coefficients in shared memory,
// then run the rank-1 updates h += coef (x) P from shared memory only.
// Thread (cg, fg) of the consumers owns features 4fg..4fg+3 of CB
// coalitions. Segment state (h, isd_i(v), m_i(e_uv) isd_i(v)) stays in
// registers across chunks.
constexpr uint32_t kSelf = 0xFFFFFFFFu;
constexpr int kChunkEntries = 32;
constexpr int kConsumers = 256;

template <int D>
struct FusedCfg {
  static constexpr int FG = D / 4;            // float4 lanes per row
  static constexpr int CGS = kConsumers / FG;  // coalition groups
  static constexpr int CB = kTile / CGS;       // coalitions per thread
  static constexpr int STAGES = D >= 256 ? 2 : 3;
  // stage layout (bytes): records | P rows | isd rows | mask words | coef
  static constexpr int OFF_P = kChunkEntries * 16;
  static constexpr int OFF_ISD = OFF_P + kChunkEntries * D * 4;
  static constexpr int OFF_W = OFF_ISD + kChunkEntries * kTile * 4;
  static constexpr int OFF_COEF = OFF_W + kChunkEntries * 32;
  static constexpr int OFF_FLAGS = OFF_COEF + kChunkEntries * kTile * 4;  // start / end bitmasks
  static constexpr int STAGE_BYTES = OFF_FLAGS + 16;
  static constexpr int SMEM = STAGES * STAGE_BYTES + 2 * STAGES * 8;
  static_assert(D % 4 == 0 && FG <= kConsumers && kTile % CGS == 0, "shape");
};

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n\t}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void consumer_sync() {
  asm volatile("bar.sync 1, %0;" ::"n"(kConsumers) : "memory");
}

// entry record: x (P / isd row), e (mask player of the (v, x) edge or kSelf),
// euv (mask player of the (u, v) edge, self entries only), flags bit0 =
// first entry of a segment (x = v), bit1 = last entry of a segment
template <int D>
__global__ void __launch_bounds__(kConsumers + 32) __maxnreg__(D >= 256 ? 224 : 96)
    fused_kernel(const uint64_t* __restrict__ maskt, uint64_t Wp,
                 const float* __restrict__ isd, uint32_t V,
                 const float* __restrict__ P, const float* __restrict__ bias,
                 const uint4* __restrict__ ent, const uint32_t* __restrict__ item_ent,
                 const uint32_t* __restrict__ item_order, uint32_t items,
                 float* __restrict__ Apart) {
  using Cfg = FusedCfg<D>;
  extern __shared__ __align__(128) unsigned char smem[];
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + Cfg::STAGES * Cfg::STAGE_BYTES);
  uint64_t* empty = full + Cfg::STAGES;
  const uint32_t item = item_order[blockIdx.x];
  const uint64_t t = blockIdx.y;
  const int tid = threadIdx.x;
  const uint32_t e0 = item_ent[item], e1 = item_ent[item + 1];
  const uint32_t nchunks = (e1 - e0 + kChunkEntries - 1) / kChunkEntries;
  if (tid == 0) {
    for (int s = 0; s < Cfg::STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], kConsumers / 32);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  if (tid >= kConsumers) {
    // ------------------------------------------------------------ producer
    const int lane = tid - kConsumers;
    uint4 rec_next = make_uint4(0, kSelf, kSelf, 0);
    if (e0 + lane < e1) rec_next = ent[e0 + lane];
    const uint64_t* mt = maskt + t * Wp;
    const float* isd_t = isd + t * uint64_t(V) * kTile;
    for (uint32_t c = 0; c < nchunks; ++c) {
      const int s = c % Cfg::STAGES;
      unsigned char* st = smem + s * Cfg::STAGE_BYTES;
      const uint32_t base = e0 + c * kChunkEntries;
      const bool on = base + lane < e1;
      const uint4 rec = on ? rec_next : make_uint4(0, kSelf, kSelf, 0);
      // prefetch the next chunk's records before waiting for a free stage
      if (base + kChunkEntries + lane < e1) rec_next = ent[base + kChunkEntries + lane];
      if (c >= uint32_t(Cfg::STAGES)) mbar_wait(&empty[s], ((c / Cfg::STAGES) - 1) & 1);
      uint32_t bytes = 0;
      if (on) {
        bytes = D * 4 + kTile * 4 + (rec.y != kSelf ? 16 : 0) + (rec.z != kSelf ? 16 : 0);
        reinterpret_cast<uint4*>(st)[lane] = rec;
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) bytes += __shfl_xor_sync(kFull, bytes, o);
      const uint32_t startm = __ballot_sync(kFull, on && (rec.w & 1u));
      const uint32_t endm = __ballot_sync(kFull, on && (rec.w & 2u));
      if (lane == 0) {
        reinterpret_cast<uint32_t*>(st + Cfg::OFF_FLAGS)[0] = startm;
        reinterpret_cast<uint32_t*>(st + Cfg::OFF_FLAGS)[1] = endm;
        mbar_arrive_expect_tx(&full[s], bytes);
      }
      __syncwarp();
      if (on) {
        bulk_g2s(st + Cfg::OFF_P + lane * D * 4, P + uint64_t(rec.x) * D, D * 4, &full[s]);
        bulk_g2s(st + Cfg::OFF_ISD + lane * kTile * 4, isd_t + uint64_t(rec.x) * kTile, kTile * 4, &full[s]);
        if (rec.y != kSelf)
          bulk_g2s(st + Cfg::OFF_W + lane * 32, mt + (rec.y & ~1u), 16, &full[s]);
        if (rec.z != kSelf)
          bulk_g2s(st + Cfg::OFF_W + lane * 32 + 16, mt + (rec.z & ~1u), 16, &full[s]);
      }
    }
    return;
  }

  // -------------------------------------------------------------- consumers
  const int fg = tid % Cfg::FG, cg = tid / Cfg::FG;
  const int ci = tid & (kTile - 1), ck = tid >> 6;  // coefficient pass: coalition ci, entries ck + 4r
  const float4 bv = reinterpret_cast<const float4*>(bias)[fg];
  float4 h[Cfg::CB], acc[Cfg::CB];
  float sv[Cfg::CB];
  uint32_t dmask = 0;  // bit j: m_i(e_uv) for coalition cg*CB+j of the open segment
#pragma unroll
  for (int j = 0; j < Cfg::CB; ++j) {
    h[j] = make_float4(0.f, 0.f, 0.f, 0.f);
    acc[j] = make_float4(0.f, 0.f, 0.f, 0.f);
    sv[j] = 0.f;
  }
  for (uint32_t c = 0; c < nchunks; ++c) {
    const int s = c % Cfg::STAGES;
    mbar_wait(&full[s], (c / Cfg::STAGES) & 1);
    unsigned char* st = smem + s * Cfg::STAGE_BYTES;
    const uint4* recs = reinterpret_cast<const uint4*>(st);
    const float* Ps = reinterpret_cast<const float*>(st + Cfg::OFF_P);
    const float* isds = reinterpret_cast<const float*>(st + Cfg::OFF_ISD);
    const uint64_t* ws = reinterpret_cast<const uint64_t*>(st + Cfg::OFF_W);
    float* coef = reinterpret_cast<float*>(st + Cfg::OFF_COEF);
    const int cnt = int(min(uint32_t(kChunkEntries), e1 - (e0 + c * kChunkEntries)));
    // coefficients m_i(e) isd_i(x); self entries additionally carry
    // m_i(e_uv) in the sign-free slot dv (kept as the raw bit below)
#pragma unroll
    for (int r = 0; r < kChunkEntries / 4; ++r) {
      const int k = ck + 4 * r;
      if (k < cnt) {
        const uint4 rec = recs[k];
        const bool kept = rec.y == kSelf || ((ws[k * 4 + (rec.y & 1u)] >> ci) & 1ull);
        coef[k * kTile + ci] = kept ? isds[k * kTile + ci] : 0.f;
      }
    }
    consumer_sync();
    // Runs of entries between segment boundaries: a segment starts at the
    // first entry of a run (chunk start or right after an end) and the run
    // stops at the next segment end, so the inner loop is branch-free.
    const uint32_t startm = reinterpret_cast<const uint32_t*>(st + Cfg::OFF_FLAGS)[0];
    const uint32_t endm = reinterpret_cast<const uint32_t*>(st + Cfg::OFF_FLAGS)[1];
    int k = 0;
    while (k < cnt) {
      if ((startm >> k) & 1u) {  // segment start: x = v; keep isd_i(v) and m_i(e_uv)
        const uint32_t z = recs[k].z;
        const uint64_t wv = z == kSelf ? ~0ull : ws[k * 4 + 2 + (z & 1u)];
        dmask = uint32_t(wv >> (cg * Cfg::CB));
#pragma unroll
        for (int j = 0; j < Cfg::CB; ++j) sv[j] = isds[k * kTile + cg * Cfg::CB + j];
      }
      const uint32_t rest = endm >> k;
      const int stop = rest ? k + __ffs(int(rest)) - 1 : cnt - 1;  // inclusive
#pragma unroll 2
      for (; k <= stop; ++k) {
        const float4 x = reinterpret_cast<const float4*>(Ps + k * D)[fg];
        const float* ckp = coef + k * kTile + cg * Cfg::CB;
#pragma unroll
        for (int j = 0; j < Cfg::CB; ++j) {
          const float cc = ckp[j];
          h[j].x = fmaf(cc, x.x, h[j].x);
          h[j].y = fmaf(cc, x.y, h[j].y);
          h[j].z = fmaf(cc, x.z, h[j].z);
          h[j].w = fmaf(cc, x.w, h[j].w);
        }
      }
      if (rest) {  // segment end: h_i(v) = relu(isd_i(v) h + b0); A += m isd_i(v) h_i(v)
#pragma unroll
        for (int j = 0; j < Cfg::CB; ++j) {
          const float dv = ((dmask >> j) & 1u) ? sv[j] : 0.f;
          acc[j].x = fmaf(dv, fmaxf(fmaf(sv[j], h[j].x, bv.x), 0.f), acc[j].x);
          acc[j].y = fmaf(dv, fmaxf(fmaf(sv[j], h[j].y, bv.y), 0.f), acc[j].y);
          acc[j].z = fmaf(dv, fmaxf(fmaf(sv[j], h[j].z, bv.z), 0.f), acc[j].z);
          acc[j].w = fmaf(dv, fmaxf(fmaf(sv[j], h[j].w, bv.w), 0.f), acc[j].w);
          h[j] = make_float4(0.f, 0.f, 0.f, 0.f);
        }
      }
    }
    __syncwarp();
    if ((tid & 31) == 0) mbar_arrive(&empty[s]);
  }
  float* out = Apart + (t * items + item) * uint64_t(kTile) * D;
#pragma unroll
  for (int j = 0; j < Cfg::CB; ++j)
    reinterpret_cast<float4*>(out + uint64_t(cg * Cfg::CB + j) * D)[fg] = acc[j];
}

// Softmax of z (float, max subtraction, sequential sum) as gcn.cpp:143-152.
__device__ __forceinline__ void softmax_row(float* zi, uint32_t C) {
  float mx = zi[0];
  for (uint32_t c = 1; c < C; ++c) mx = fmaxf(mx, zi[c]);
  float sum = 0.f;
  for (uint32_t c = 0; c < C; ++c) {
    zi[c] = expf(zi[c] - mx);
    sum += zi[c];
  }
  for (uint32_t c = 0; c < C; ++c) zi[c] = zi[c] / sum;
}

// The same float softmax with the warp's lanes over the classes: max and
// sum by butterfly reductions (sum order differs from the sequential
// reference loop by float rounding only), exp and divide per lane.

// A[t][u][i][:] = isd_i(u) * sum over the items of u of Apart[t][item][i][:]
// (fixed item order, deterministic), one float4 per thread.
__global__ void __launch_bounds__(256)
    reduce_partials_kernel(const float4* __restrict__ Apart, uint32_t items,
                           const uint32_t* __restrict__ u_items,
                           const float* __restrict__ isd, uint32_t V, uint32_t K4,
                           uint32_t U, float4* __restrict__ A) {
  const uint64_t idx = blockIdx.x * 256ull + threadIdx.x;
  const uint64_t per_u = uint64_t(kTile) * K4;
  if (idx >= U * per_u) return;
  const uint64_t t = blockIdx.y;
  const uint32_t u = uint32_t(idx / per_u);
  const uint64_t rem = idx % per_u;
  const uint32_t i = uint32_t(rem / K4);
  float4 s = make_float4(0.f, 0.f, 0.f, 0.f);
  for (uint32_t it = u_items[u]; it < u_items[u + 1]; ++it) {
    const float4 p = Apart[(t * items + it) * per_u + rem];
    s.x += p.x;
    s.y += p.y;
    s.z += p.z;
    s.w += p.w;
  }
  const float sc = isd[(t * V + u) * kTile + i];
  A[(t * U + u) * per_u + rem] = make_float4(sc * s.x, sc * s.y, sc * s.z, sc * s.w);
}

// Softmax of each logit row (warp per row), p[cls] and optionally all probs.
__global__ void softmax_rows_kernel(float* __restrict__ Z, uint32_t N, uint64_t row0,
                                    uint64_t nbatch, uint64_t rows, uint32_t cls,
                                    float* __restrict__ out, float* __restrict__ allprobs) {
  const uint64_t r = (blockIdx.x * uint64_t(blockDim.x) + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (r >= nbatch || row0 + r >= rows) return;
  float* z = Z + r * N;
  if (lane == 0) {
    softmax_row(z, N);
    out[row0 + r] = z[cls];
  }
  __syncwarp();
  if (allprobs)
    for (uint32_t c = lane; c < N; c += 32) allprobs[(row0 + r) * N + c] = z[c];
}

// ---------------------------------------------------------------- generic
// Any width. out[t][r][i][f] = act(isd_i(r) * sum_v isd_i(v) X(v,i,f) + b[f])
// with X = P[v][f] (shared) or Hin[t][v][i][f] (per coalition, Rin rows).
// bias may be null (hidden aggregation feeding a GEMM).
__global__ void agg_generic_kernel(const uint64_t* __restrict__ maskt,
                                   uint64_t Wp,
                                   const uint32_t* __restrict__ row_ptr,
                                   const uint32_t* __restrict__ col,
                                   const uint32_t* __restrict__ ep,
                                   const float* __restrict__ isd, uint32_t V,
                                   const float* __restrict__ X, int shared_x,
                                   uint32_t Rin, uint32_t D,
                                   const float* __restrict__ bias, int relu,
                                   uint32_t R, float* __restrict__ out) {
  const uint32_t r = blockIdx.x;
  const uint64_t t = blockIdx.y;
  const uint64_t* mt = maskt + t * Wp;
  const float* isd_t = isd + t * uint64_t(V) * kTile;
  const uint32_t beg = row_ptr[r], end = row_ptr[r + 1];
  for (uint32_t idx = threadIdx.x; idx < kTile * D; idx += blockDim.x) {
    const uint32_t i = idx / D, f = idx % D;
    auto x_at = [&](uint32_t v) {
      return shared_x ? X[uint64_t(v) * D + f]
                      : X[((t * Rin + v) * kTile + i) * D + f];
    };
    float acc = isd_t[uint64_t(r) * kTile + i] * x_at(r);
    for (uint32_t e = beg; e < end; ++e) {
      if (!((mt[ep[e]] >> i) & 1ull)) continue;
      const uint32_t v = col[e];
      acc = fmaf(isd_t[uint64_t(v) * kTile + i], x_at(v), acc);
    }
    float h = isd_t[uint64_t(r) * kTile + i] * acc;
    if (bias) h += bias[f];
    if (relu) h = fmaxf(h, 0.f);
    out[((t * R + r) * kTile + i) * D + f] = h;
  }
}

// ---------------------------------------------------------------- GEMM
// C[M x N] = act(A[M x K] B[K x N] + bias), row-major FP32, 64x64 tiles,
// 16-deep K slabs, 4x4 outputs per thread.
__global__ void __launch_bounds__(256)
    sgemm_kernel(const float* __restrict__ A, const float* __restrict__ B,
                 const float* __restrict__ bias, float* __restrict__ Cm,
                 uint64_t M, uint32_t N, uint32_t K, int relu, const uint32_t* __restrict__ arow) {
  __shared__ float As[16][64 + 4];
  __shared__ float Bs[16][64 + 4];
  const int tx = threadIdx.x % 16, ty = threadIdx.x / 16;
  const uint64_t m0 = uint64_t(blockIdx.y) * 64;
  const uint32_t n0 = blockIdx.x * 64;
  float acc[4][4] = {};
  for (uint32_t k0 = 0; k0 < K; k0 += 16) {
    for (int idx = threadIdx.x; idx < 64 * 16; idx += 256) {
      const int mm = idx / 16, kk = idx % 16;
      const uint64_t gm = m0 + mm;
      const uint32_t gk = k0 + kk;
      As[kk][mm] = (gm < M && gk < K) ? A[(arow ? uint64_t(arow[gm]) : gm) * K + gk] : 0.f;
      const int kb = idx / 64, nb = idx % 64;
      const uint32_t gkb = k0 + kb, gn = n0 + nb;
      Bs[kb][nb] = (gkb < K && gn < N) ? B[uint64_t(gkb) * N + gn] : 0.f;
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < 16; ++kk) {
      float a[4], b[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        a[q] = As[kk][ty * 4 + q];
        b[q] = Bs[kk][tx * 4 + q];
      }
#pragma unroll
      for (int p = 0; p < 4; ++p)
#pragma unroll
        for (int q = 0; q < 4; ++q) acc[p][q] = fmaf(a[p], b[q], acc[p][q]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int p = 0; p < 4; ++p) {
    const uint64_t gm = m0 + ty * 4 + p;
    if (gm >= M) continue;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const uint32_t gn = n0 + tx * 4 + q;
      if (gn >= N) continue;
      float v = acc[p][q] + (bias ? bias[gn] : 0.f);
      if (relu) v = fmaxf(v, 0.f);
      Cm[gm * N + gn] = v;
    }
  }
}

// ---------------------------------------------------------------- last layer
// Target row only (gcn.cpp:134-140) + softmax (143-152); one CTA per
// (tile, block of cpb coalitions).
// a_i = isd_i(0) sum_{v in {0} u kept N(0)} isd_i(v) X(v, i, :)
// z_i = bias + a_i W   (skipped when X is already transformed: L == 1)
// p_i = softmax(z_i) in float with max subtraction; out = p_i[cls].
__global__ void last_kernel(const uint64_t* __restrict__ maskt, uint64_t Wp,
                            const uint32_t* __restrict__ row_ptr,
                            const uint32_t* __restrict__ col,
                            const uint32_t* __restrict__ ep,
                            const float* __restrict__ isd, uint32_t V,
                            const float* __restrict__ X, int shared_x,
                            uint32_t Rin, uint32_t Din,
                            const float* __restrict__ Wt,
                            const float* __restrict__ bias, uint32_t C,
                            uint32_t cls, uint64_t row0, uint64_t rows, uint32_t cpb,
                            float* __restrict__ out,
                            float* __restrict__ allprobs) {
  extern __shared__ float sm[];
  float* a = sm;                // [cpb][Din]
  float* z = sm + cpb * Din;    // [cpb][C]
  const uint64_t t = blockIdx.x;
  const uint32_t i0 = blockIdx.y * cpb;
  const uint64_t* mt = maskt + t * Wp;
  const float* isd_t = isd + t * uint64_t(V) * kTile;
  const uint32_t beg = row_ptr[0], end = row_ptr[1];
  for (uint32_t idx = threadIdx.x; idx < cpb * Din; idx += blockDim.x) {
    const uint32_t i = i0 + idx / Din, f = idx % Din;
    auto x_at = [&](uint32_t v) {
      return shared_x ? X[uint64_t(v) * Din + f]
                      : X[((t * Rin + v) * kTile + i) * Din + f];
    };
    float acc = isd_t[i] * x_at(0);
    for (uint32_t e = beg; e < end; ++e) {
      if (!((mt[ep[e]] >> i) & 1ull)) continue;
      const uint32_t v = col[e];
      acc = fmaf(isd_t[uint64_t(v) * kTile + i], x_at(v), acc);
    }
    a[idx] = isd_t[i] * acc;
  }
  __syncthreads();
  for (uint32_t idx = threadIdx.x; idx < cpb * C; idx += blockDim.x) {
    const uint32_t il = idx / C, c = idx % C;
    float v = bias[c];
    if (Wt) {
      // bias-first sequential accumulation as in affine_row (gcn.cpp:116-123)
      for (uint32_t k = 0; k < Din; ++k)
        v = __fadd_rn(v, __fmul_rn(a[il * Din + k], Wt[uint64_t(k) * C + c]));
    } else {
      v = __fadd_rn(a[il * Din + c], v);
    }
    z[idx] = v;
  }
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int nwarps = blockDim.x >> 5;
  for (uint32_t il = warp; il < cpb; il += nwarps) {
    const uint64_t row = row0 + t * kTile + i0 + il;
    if (row >= rows) continue;
    if (lane == 0) {
      softmax_row(z + il * C, C);
      out[row] = z[il * C + cls];
    }
    __syncwarp();
    if (allprobs)
      for (uint32_t c = lane; c < C; c += 32) allprobs[row * C + c] = z[il * C + c];
  }
}

constexpr int kTailThreads = 512;

__device__ __forceinline__ void tf32_split(float x, uint32_t& hi, uint32_t& lo) {
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(hi) : "f"(x));
  const float r = x - __uint_as_float(hi);
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(lo) : "f"(r));
}

// d += a (16x8, row) * b (8x8, col), tf32 in, f32 accumulate
__device__ __forceinline__ void mma_tf32(float (&d)[4], const uint32_t (&a)[4], const uint32_t (&b)[2]) {
  asm volatile(
      "mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]));
}

// ---------------------------------------------------------------- fused tail
// Everything after the fused layer-0/1 kernel, for one tile t and cpb
// coalitions per CTA, in shared memory (replaces reduce_partials + sgemm +
// last_kernel / softmax_rows with the same arithmetic order):
//   A[u][i]  = isd_i(u) * sum over the items of u of Apart[t][item][i]
//   H[u][i]  = act(sum_k A[u][i][k] W1[k] + b1)   (k ascending, as sgemm)
//   L == 3:  a_i = isd_i(0)(isd_i(0) H[0][i] + sum_{kept v in N(0)} isd_i(v) H[v][i])
//            z_i = b2 + a_i W2 (bias-first, gcn.cpp:116-123)
//   L == 2:  z_i = H[0][i] (logits, no activation)
//   p_i = softmax(z_i) (gcn.cpp:143-152); out = p_i[cls].
// Rows of A and H are u-major: r = u * cpb + il.
__global__ void __launch_bounds__(kTailThreads, 2)
    tail_kernel(const float4* __restrict__ Apart, uint32_t items,
                const uint32_t* __restrict__ u_items, const uint64_t* __restrict__ maskt,
                uint64_t Wp, const uint32_t* __restrict__ row_ptr,
                const uint32_t* __restrict__ col, const uint32_t* __restrict__ ep,
                const float* __restrict__ isd, uint32_t V, uint32_t U, uint32_t K,
                uint32_t N, const float* __restrict__ W1, const float* __restrict__ b1,
                const float* __restrict__ W2, const float* __restrict__ b2, uint32_t C,
                int three_layer, uint32_t cls, uint64_t row0, uint64_t rows, uint32_t cpb,
                float* __restrict__ out, float* __restrict__ allprobs) {
  extern __shared__ float4 sm4[];
  const uint32_t R = U * cpb, K4 = K / 4;
  // padded row strides (floats): conflict-free mma.sync fragment loads
  const uint32_t SA = K + 4, SA4 = SA / 4, SW = (N % 4 == 0) ? N + 8 : N;
  float4* sA = sm4;                                    // [R][SA]
  float* sW1 = reinterpret_cast<float*>(sA + R * SA4); // [K][SW]
  float* sW2 = sW1 + K * SW;                           // [N][C] (three_layer)
  float* sH = sW2 + (three_layer ? N * C : 0);         // [R][N]
  float* sa = sH + R * N;                              // [cpb][N]
  float* sz = sa + cpb * N;                            // [cpb][C]
  const uint64_t t = blockIdx.x;
  const uint32_t i0 = blockIdx.y * cpb;
  const float* isd_t = isd + t * uint64_t(V) * kTile;
  const int tid = threadIdx.x;
  {  // weights -> shared memory with cp.async, overlapped with the partial sums below
    const uint32_t n1 = K * N / 4;
    if (SW != N) {  // padded rows
      const uint32_t rq = N / 4;
      for (uint32_t idx = tid; idx < n1; idx += blockDim.x)
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(
                         static_cast<uint32_t>(__cvta_generic_to_shared(sW1 + (idx / rq) * SW + 4 * (idx % rq)))),
                     "l"(W1 + 4 * idx) : "memory");
    } else {  // K * N is a multiple of 4 (K is)
      for (uint32_t idx = tid; idx < n1; idx += blockDim.x)
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(
                         static_cast<uint32_t>(__cvta_generic_to_shared(sW1 + 4 * idx))),
                     "l"(W1 + 4 * idx) : "memory");
    }
    if (three_layer) {
      const uint32_t n2 = N * C / 4;
      for (uint32_t idx = tid; idx < n2; idx += blockDim.x)
        asm volatile("cp.async.ca.shared.global [%0], [%1], 16;" ::"r"(
                         static_cast<uint32_t>(__cvta_generic_to_shared(sW2 + 4 * idx))),
                     "l"(W2 + 4 * idx) : "memory");
      for (uint32_t idx = 4 * n2 + tid; idx < N * C; idx += blockDim.x) sW2[idx] = __ldg(&W2[idx]);
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  }
  // A (partials in item order, then isd_i(u)); loads batched 8 items deep
  for (uint32_t idx = tid; idx < R * K4; idx += blockDim.x) {
    const uint32_t r = idx / K4, k4 = idx % K4, u = r / cpb, i = i0 + r % cpb;
    float4 s = make_float4(0.f, 0.f, 0.f, 0.f);
    const uint32_t ib = u_items[u], ie = u_items[u + 1];
    const float4* src = Apart + ((t * items) * kTile + i) * K4 + k4;
    const uint64_t stride = uint64_t(kTile) * K4;
    uint32_t it = ib;
    for (; it + 8 <= ie; it += 8) {
      float4 p[8];
#pragma unroll
      for (int q = 0; q < 8; ++q) p[q] = src[(it + q) * stride];
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        s.x += p[q].x;
        s.y += p[q].y;
        s.z += p[q].z;
        s.w += p[q].w;
      }
    }
    for (; it < ie; ++it) {
      const float4 p = src[it * stride];
      s.x += p.x;
      s.y += p.y;
      s.z += p.z;
      s.w += p.w;
    }
    const float sc = isd_t[uint64_t(u) * kTile + i];
    sA[r * SA4 + k4] = make_float4(sc * s.x, sc * s.y, sc * s.z, sc * s.w);
  }
  asm volatile("cp.async.wait_all;" ::: "memory");
  __syncthreads();
  // H = act(A W1 + b1)
  if (N % 16 == 0 && K % 8 == 0) {
    // warp tensor-core MMAs (mma.sync m16n8k8 tf32, 3xTF32 split in
    // registers: FP32-level products); warp job = 16 rows x 16 columns
    const int warp = tid >> 5, lane = tid & 31, g = lane >> 2, tq = lane & 3;
    const float* Af = reinterpret_cast<const float*>(sA);
    const uint32_t mtiles = (R + 15) / 16, npairs = N / 16;
    for (uint32_t job = warp; job < mtiles * npairs; job += blockDim.x / 32) {
      const uint32_t m0 = (job / npairs) * 16, n0 = (job % npairs) * 16;
      const uint32_t r0 = m0 + g, r1 = m0 + g + 8;
      float d[2][4] = {};
      for (uint32_t k0 = 0; k0 < K; k0 += 8) {
        const float af[4] = {r0 < R ? Af[r0 * SA + k0 + tq] : 0.f, r1 < R ? Af[r1 * SA + k0 + tq] : 0.f,
                             r0 < R ? Af[r0 * SA + k0 + tq + 4] : 0.f, r1 < R ? Af[r1 * SA + k0 + tq + 4] : 0.f};
        uint32_t ah[4], al[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) tf32_split(af[q], ah[q], al[q]);
#pragma unroll
        for (int nt = 0; nt < 2; ++nt) {
          const uint32_t n = n0 + nt * 8 + g;
          uint32_t bh[2], bl[2];
          tf32_split(sW1[(k0 + tq) * SW + n], bh[0], bl[0]);
          tf32_split(sW1[(k0 + tq + 4) * SW + n], bh[1], bl[1]);
          mma_tf32(d[nt], ah, bh);
          mma_tf32(d[nt], ah, bl);
          mma_tf32(d[nt], al, bh);
        }
      }
#pragma unroll
      for (int nt = 0; nt < 2; ++nt) {
        const uint32_t c0 = n0 + nt * 8 + 2 * tq;
        const float bb0 = b1[c0], bb1 = b1[c0 + 1];
        if (r0 < R) {
          const float v0 = d[nt][0] + bb0, v1 = d[nt][1] + bb1;
          sH[r0 * N + c0] = three_layer ? fmaxf(v0, 0.f) : v0;
          sH[r0 * N + c0 + 1] = three_layer ? fmaxf(v1, 0.f) : v1;
        }
        if (r1 < R) {
          const float v2 = d[nt][2] + bb0, v3 = d[nt][3] + bb1;
          sH[r1 * N + c0] = three_layer ? fmaxf(v2, 0.f) : v2;
          sH[r1 * N + c0 + 1] = three_layer ? fmaxf(v3, 0.f) : v3;
        }
      }
    }
  } else {
  // SIMT: thread = (column n, row group of up to kRB rows)
  // one job per thread when N * ceil(R / kRB) <= blockDim.x
  constexpr uint32_t kRB = 8;
  const uint32_t rgroups = max(1u, min(R, blockDim.x / N));
  const uint32_t RB = (R + rgroups - 1) / rgroups;
  for (uint32_t job = tid; job < N * rgroups; job += blockDim.x) {
    const uint32_t n = job % N, g = job / N;
    for (uint32_t rb0 = g * RB; rb0 < min(R, (g + 1) * RB); rb0 += kRB) {
      const uint32_t nr = min(kRB, min(R, (g + 1) * RB) - rb0);
      float acc[kRB];
#pragma unroll
      for (uint32_t j = 0; j < kRB; ++j) acc[j] = 0.f;
      for (uint32_t k4 = 0; k4 < K4; ++k4) {
        const float w0 = sW1[(4 * k4) * SW + n], w1 = sW1[(4 * k4 + 1) * SW + n];
        const float w2 = sW1[(4 * k4 + 2) * SW + n], w3 = sW1[(4 * k4 + 3) * SW + n];
#pragma unroll
        for (uint32_t j = 0; j < kRB; ++j) {
          if (j < nr) {
            const float4 a = sA[(rb0 + j) * SA4 + k4];
            acc[j] = fmaf(a.x, w0, acc[j]);
            acc[j] = fmaf(a.y, w1, acc[j]);
            acc[j] = fmaf(a.z, w2, acc[j]);
            acc[j] = fmaf(a.w, w3, acc[j]);
          }
        }
      }
      const float bn = b1[n];
#pragma unroll
      for (uint32_t j = 0; j < kRB; ++j) {
        if (j < nr) {
          const float v = acc[j] + bn;
          sH[(rb0 + j) * N + n] = three_layer ? fmaxf(v, 0.f) : v;
        }
      }
    }
  }
  }
  __syncthreads();
  if (three_layer) {
    const uint64_t* mt = maskt + t * Wp;
    const uint32_t beg = row_ptr[0], end = row_ptr[1];
    for (uint32_t idx = tid; idx < cpb * N; idx += blockDim.x) {
      const uint32_t il = idx / N, f = idx % N, i = i0 + il;
      float acc = isd_t[i] * sH[il * N + f];
      for (uint32_t e = beg; e < end; ++e) {
        if (!((mt[ep[e]] >> i) & 1ull)) continue;
        const uint32_t v = col[e];
        acc = fmaf(isd_t[uint64_t(v) * kTile + i], sH[(v * cpb + il) * N + f], acc);
      }
      sa[idx] = isd_t[i] * acc;
    }
    __syncthreads();
    for (uint32_t idx = tid; idx < cpb * C; idx += blockDim.x) {
      const uint32_t il = idx / C, c = idx % C;
      // bias-first (gcn.cpp:116-123), even and odd k in two chains
      float v0 = b2[c], v1 = 0.f;
      uint32_t k = 0;
      for (; k + 1 < N; k += 2) {
        v0 = __fadd_rn(v0, __fmul_rn(sa[il * N + k], sW2[k * C + c]));
        v1 = __fadd_rn(v1, __fmul_rn(sa[il * N + k + 1], sW2[(k + 1) * C + c]));
      }
      if (k < N) v0 = __fadd_rn(v0, __fmul_rn(sa[il * N + k], sW2[k * C + c]));
      sz[idx] = __fadd_rn(v0, v1);
    }
  } else {
    for (uint32_t idx = tid; idx < cpb * C; idx += blockDim.x) sz[idx] = sH[idx];  // U == 1: row il
  }
  __syncthreads();
  const int lane = tid & 31, warp = tid >> 5, nwarps = blockDim.x >> 5;
  for (uint32_t il = warp; il < cpb; il += nwarps) {
    const uint64_t row = row0 + t * kTile + i0 + il;
    if (row >= rows) continue;
    softmax_row_warp(sz + il * C, C, lane);
    if (lane == 0) out[row] = sz[il * C + cls];
    __syncwarp();
    if (allprobs)
      for (uint32_t c = lane; c < C; c += 32) allprobs[row * C + c] = sz[il * C + c];
  }
}

size_t tail_smem(uint32_t U, uint32_t K, uint32_t N, uint32_t C, uint32_t cpb, bool three_layer) {
  return (size_t(U) * cpb * (K + 4 + N) + size_t(cpb) * (N + C) + size_t(K) * (N + 8) +
          (three_layer ? size_t(N) * C : 0)) * 4;
}

// X W0 for the whole subgraph (once per target)
// (arow: row r of A is row arow[r] of the given matrix — the ball's rows
// of the graph's features)
void gemm(Ctx& ctx, const float* A, const float* B, const float* bias, float* Cm,
          uint64_t M, uint32_t N, uint32_t K, bool relu, const uint32_t* arow = nullptr) {
  if (M == 0 || N == 0) return;
  dim3 grid((N + 63) / 64, unsigned((M + 63) / 64));
  sgemm_kernel<<<grid, 256, 0, ctx.stream>>>(A, B, bias, Cm, M, N, K, relu ? 1 : 0, arow);
  SF_LAUNCHED(ctx);
}

}  // namespace

namespace {
constexpr uint32_t kItemEntries = 512;  // target staged entries per work item
constexpr size_t kTailSmem = 200 * 1024;  // fused tail kernel shared-memory cap

bool fused_width(uint64_t d) { return d == 16 || d == 32 || d == 64 || d == 128 || d == 256; }

template <int D>
bool try_fused(Ctx& ctx, const Engine& e, const uint64_t* maskt, uint64_t Wp, const float* isd,
               uint64_t nt, float* apart) {
  if (e.dims[1] != uint64_t(D)) return false;
  using Cfg = FusedCfg<D>;
  set_max_dynamic_smem(fused_kernel<D>, int(Cfg::SMEM));
  // two CTAs per SM need the maximum shared-memory carveout
  SF_CUDA(cudaFuncSetAttribute(fused_kernel<D>, cudaFuncAttributePreferredSharedMemoryCarveout,
                               int(cudaSharedmemCarveoutMaxShared)));
  dim3 grid(e.items, unsigned(nt));
  fused_kernel<D><<<grid, kConsumers + 32, Cfg::SMEM, ctx.stream>>>(
      maskt, Wp, isd, e.V, e.p0.p, e.b[0]->p, reinterpret_cast<const uint4*>(e.ent.p), e.item_ent.p,
      e.item_order.p, e.items, apart);
  SF_LAUNCHED(ctx);
  return true;
}

// Entry records and work items of the fused plan (see Engine / fused_kernel).
void build_fused_plan(Ctx& ctx, Engine& e, const Subgraph& sg) {
  const uint32_t U = uint32_t(e.ball[e.L - 2]);
  std::vector<uint32_t> ent;  // 4 words per entry: x, e, euv, flags
  std::vector<uint32_t> item_ent{0}, u_items{0};
  std::vector<uint64_t> item_work;
  auto entries = [&]() { return uint64_t(ent.size() / 4); };
  for (uint32_t u = 0; u < U; ++u) {
    uint64_t open_entries = 0;
    auto close_item = [&]() {
      if (entries() > item_ent.back()) {
        item_ent.push_back(uint32_t(entries()));
        item_work.push_back(open_entries);
        open_entries = 0;
      }
    };
    auto segment = [&](uint32_t v, uint32_t euv) {
      const uint64_t w = sg.row_ptr[v + 1] - sg.row_ptr[v] + 1;
      if (open_entries && open_entries + w > kItemEntries) close_item();
      ent.insert(ent.end(), {v, kSelf, euv, w == 1 ? 3u : 1u});
      for (uint64_t k = sg.row_ptr[v]; k < sg.row_ptr[v + 1]; ++k) {
        const bool last = (k + 1 == sg.row_ptr[v + 1]);
        ent.insert(ent.end(), {sg.col[k], sg.edge_player[k], kSelf, last ? 2u : 0u});
      }
      open_entries += w;
    };
    segment(u, kSelf);
    for (uint64_t k = sg.row_ptr[u]; k < sg.row_ptr[u + 1]; ++k) segment(sg.col[k], sg.edge_player[k]);
    close_item();
    u_items.push_back(uint32_t(item_ent.size() - 1));
  }
  if (entries() >= (1ull << 32)) throw DataError("fused plan too large");
  // heaviest items first (LPT); partial sums keep the item index, so the
  // reduction order stays fixed
  std::vector<uint32_t> order(item_work.size());
  for (uint32_t i = 0; i < order.size(); ++i) order[i] = i;
  std::stable_sort(order.begin(), order.end(),
                   [&](uint32_t a, uint32_t b) { return item_work[a] > item_work[b]; });
  e.U = U;
  e.items = uint32_t(item_work.size());
  e.entries = entries();
  e.ent.upload(ent.data(), ent.size(), ctx.stream);
  e.item_ent.upload(item_ent.data(), item_ent.size(), ctx.stream);
  e.item_order.upload(order.data(), order.size(), ctx.stream);
  e.u_items.upload(u_items.data(), u_items.size(), ctx.stream);
  ctx.h2d_bytes += (ent.size() + item_ent.size() + order.size() + u_items.size()) * 4;
  // (no sync: cudaMemcpyAsync from pageable memory returns once the source
  // is staged, so the vectors may go; the host builds the next plan while
  // the device copies)
}
}  // namespace

void engine_prepare(Ctx& ctx, const Subgraph& sg, const Model& m) {
  Engine& e = ctx.engine;
  if (e.sg_id == sg.id && e.model_id == m.id && e.kind == ctx.fused_kind) return;
  if (m.layers.empty()) throw DataError("model has no layers");
  if (m.layers.front().in != sg.feature_dim)
    throw DataError("model input dim " + std::to_string(m.layers.front().in) +
                    " does not match feature dim " + std::to_string(sg.feature_dim));
  DebugTimer dt("engine_prepare");
  e.sg_id = 0;
  e.V = sg.num_nodes();
  e.n = sg.num_players();
  e.W = std::max<uint32_t>(1, static_cast<uint32_t>((e.n + 63) / 64));  // n = 0: one zero word
  e.L = m.depth();
  e.dims.assign(1, m.layers.front().in);
  for (const Layer& l : m.layers) e.dims.push_back(l.out);
  e.ball = sg.ball_sizes(e.L);
  if (sg.col.size() >= (1ull << 32)) throw DataError("subgraph too large for u32 CSR");
  std::vector<uint32_t> rp(sg.row_ptr.begin(), sg.row_ptr.end());
  e.row_ptr.upload(rp.data(), rp.size(), ctx.stream);
  e.col.upload(sg.col.data(), sg.col.size(), ctx.stream);
  e.edge_player.upload(sg.edge_player.data(), sg.edge_player.size(), ctx.stream);
  dt.lap("csr upload");
  {  // isd_kernel: nodes by descending degree, 1/sqrt(deg) table
    std::vector<uint32_t> order(e.V);
    uint32_t maxdeg = 0;
    for (uint32_t v = 0; v < e.V; ++v) {
      order[v] = v;
      maxdeg = std::max(maxdeg, rp[v + 1] - rp[v]);
    }
    std::stable_sort(order.begin(), order.end(),
                     [&](uint32_t a, uint32_t b) { return rp[a + 1] - rp[a] > rp[b + 1] - rp[b]; });
    e.isd_order.upload(order.data(), order.size(), ctx.stream);
    e.isd_nbig = 0;
    while (e.isd_nbig < e.V && rp[order[e.isd_nbig] + 1] - rp[order[e.isd_nbig]] > 32) ++e.isd_nbig;
    e.isd_tab.reserve(maxdeg + 2);
    e.isd_tab_n = maxdeg + 2;
    isd_table_kernel<<<(maxdeg + 2 + 255) / 256, 256, 0, ctx.stream>>>(e.isd_tab.p, maxdeg + 2);
    SF_LAUNCHED(ctx);
  }
  // P0 = X W0 on the device
  DevBuf<float>& w0 = ctx.w0_dev;
  w0.upload(m.layers[0].weight.data(), m.layers[0].weight.size(), ctx.stream);
  e.p0.reserve(uint64_t(e.V) * e.dims[1]);
  if (sg.source) {  // X rows gathered from the graph's device-resident features
    const Graph& g = *sg.source;
    if (ctx.graph_feat_id != g.id) {
      ctx.graph_feat.upload(g.features.data(), g.features.size(), ctx.stream);
      ctx.graph_feat_id = g.id;
      ctx.h2d_bytes += g.features.size() * 4;
    }
    ctx.ball_rows.upload(sg.local_to_global.data(), sg.local_to_global.size(), ctx.stream);
    ctx.h2d_bytes += sg.local_to_global.size() * 4;
    gemm(ctx, ctx.graph_feat.p, w0.p, nullptr, e.p0.p, e.V, uint32_t(e.dims[1]), uint32_t(e.dims[0]), false,
         ctx.ball_rows.p);
  } else {
    DevBuf<float>& x = ctx.feat_dev;
    x.upload(sg.features.data(), sg.features.size(), ctx.stream);
    ctx.h2d_bytes += sg.features.size() * 4;
    gemm(ctx, x.p, w0.p, nullptr, e.p0.p, e.V, uint32_t(e.dims[1]), uint32_t(e.dims[0]), false);
  }
  while (int(e.w.size()) < e.L) {  // buffers are kept (and grown) across targets
    e.w.emplace_back(new DevBuf<float>);
    e.b.emplace_back(new DevBuf<float>);
  }
  for (int l = 0; l < e.L; ++l) {
    if (l > 0) e.w[l]->upload(m.layers[l].weight.data(), m.layers[l].weight.size(), ctx.stream);
    e.b[l]->upload(m.layers[l].bias.data(), m.layers[l].bias.size(), ctx.stream);
  }
  ctx.h2d_bytes += (rp.size() + sg.col.size() + sg.edge_player.size()) * 4;
  for (const Layer& l : m.layers) ctx.h2d_bytes += (l.weight.size() + l.bias.size()) * 4;
  // (no sync: the pageable sources are staged before cudaMemcpyAsync
  // returns; the host goes on with the plans while X W0 runs)
  dt.lap("p0 gemm + weights");
  e.fused = e.L >= 2 && fused_width(e.dims[1]) && e.n > 0;
  if (e.fused) build_fused_plan(ctx, e, sg);
  dt.lap("fused plan");
  // tcgen05 3xTF32 fused kernel by default; SF_FUSED_TC=0 selects the SIMT FP32 kernel
  static const bool use_tc = [] {
    const char* v = std::getenv("SF_FUSED_TC");
    return v == nullptr || std::strcmp(v, "0") != 0;
  }();
  const bool want_tc = ctx.fused_kind >= 2 || (ctx.fused_kind == 0 && use_tc);
  e.tc = e.fused && want_tc && tc_width(e.dims[1]);
  // fp16x2 variant (sf_fused_f16.cu: MN-major B gathered directly, K = 16,
  // u16 degree rows + a shared 1/sqrt table). Opt-in with SF_FUSED_TC16=1:
  // on C2 it measured level with 3xTF32 (its 16-entry segment padding adds
  // ~20% work items and its degree buffer shrinks the batch).
  static const bool use_tc16 = [] {
    const char* v = std::getenv("SF_FUSED_TC16");
    return v != nullptr && std::strcmp(v, "0") != 0;
  }();
  const bool want_tc16 = ctx.fused_kind == 3 || (ctx.fused_kind == 0 && use_tc16);
  e.tc16 = e.tc && want_tc16 && tc16_width(e.dims[1]) && e.isd_tab_n <= tc16_max_table();
  e.tc_kstep = e.tc16 ? 16 : 8;
  if (e.tc) build_tc_plan(ctx, e, sg);
  if (e.tc16 && !e.tc) e.tc16 = false;  // the plan may have rejected the tensor-core path
  if (e.tc16) prepare_tc16(ctx, e);
  // layer-1 GEMM + last layer on tcgen05 (SF_TAIL_TC=0: never, 1: always).
  // By default a call takes it when a full batch has >= 64 tile pairs (one
  // CTA per tile pair and B_1 share, one per SM): C2 (74 tile pairs per
  // batch) 11.20M vs 10.71M coalitions/s; C3 (28) 3.09M vs 3.16M and C4
  // (7) 467K vs 586K favour the mma.sync tail's many small CTAs.
  static const int use_tail_tc = [] {
    const char* v = std::getenv("SF_TAIL_TC");
    return v == nullptr ? 2 : std::atoi(v);
  }();
  e.tail_tc = use_tail_tc != 0 && tail_tc_supported(e);
  e.tail_tc_always = use_tail_tc == 1;
  if (e.tail_tc) build_tail_tc(ctx, e);
  // u16 degree rows + a shared-memory 1/sqrt table instead of f32 isd rows
  // for the fused kernel (f32 rows kept for B_1 when the mma.sync tail runs).
  // SF_ISD_U16: unset = with the mma.sync tail only (C3 +3.3%, C4 +4.7%;
  // with the tcgen05 tail, C2 -0.8%), 1 = always, 0 = never.
  static const int deg_mode = [] {
    const char* v = std::getenv("SF_ISD_U16");
    return v == nullptr ? 2 : std::atoi(v);
  }();
  e.deg_mode = deg_mode;
  e.deg_capable = e.tc && !e.tc16 && e.L == 3 && e.isd_tab_n <= tc_deg_table_cap();
  dt.lap("tc plan");
  e.sg_id = sg.id;
  e.model_id = m.id;
  e.kind = ctx.fused_kind;
}

void engine_predict(Ctx& ctx, const uint64_t* dev_rows, uint64_t rows,
                    uint32_t cls, float* dev_out, float* dev_allprobs,
                    float* dominant_ms, bool kept_only) {
  (void)dominant_ms;
  Engine& e = ctx.engine;
  if (rows == 0) return;
  const uint64_t tiles = (rows + kTile - 1) / kTile;
  const uint64_t Wp = uint64_t(e.W) * 64;
  const int L = e.L;
  const uint32_t C = uint32_t(e.dims[L]);
  // rows each layer produces: R_l = |B_{L-1-l}|
  std::vector<uint64_t> R(L);
  for (int l = 0; l < L; ++l) R[l] = e.ball[L - 1 - l];
  // per-tile bytes: masks + isd + activations. Fused: item partials and the
  // layer-1 outputs at U; generic: two activation buffers + aggregation.
  uint64_t hmax = 0, amax = 0, apart = 0;
  const int first_generic = e.fused ? 2 : 0;  // first layer the generic path runs
  uint64_t afused = 0;  // reduced layer-1 aggregation at U (fused path)
  if (e.fused) {
    apart = uint64_t(std::max(e.items, e.tc_items)) * kTile * e.dims[1];
    afused = uint64_t(e.U) * kTile * e.dims[1];
    hmax = uint64_t(e.U) * kTile * e.dims[2];  // H at U (L >= 3) or logits (L == 2)
  }
  for (int l = first_generic; l + 1 < L; ++l) hmax = std::max(hmax, R[l] * kTile * e.dims[l + 1]);
  for (int l = std::max(1, first_generic); l + 1 < L; ++l) amax = std::max(amax, R[l] * kTile * e.dims[l]);
  // batch sizing with f32 isd rows (the u16-degree choice below only shrinks
  // a batch's workspace)
  const uint64_t isd_b = e.tc16 ? 6 : 4;  // f32 isd and / or u16 degrees per (node, coalition)
  const uint64_t per_tile = Wp * 8 + uint64_t(e.V) * kTile * isd_b + (2 * hmax + amax + apart + afused) * 4;
  // per-batch workspace (masks tiles, isd, partials, activations). Larger
  // batches mean fewer launches and fuller waves for the fused kernel: C2
  // measured 74.0 ms/step at 96 MB, 62.0 at 448, 60.6 at 1024 (plateau);
  // SF_BATCH_MB overrides.
  static const uint64_t budget =
      (std::getenv("SF_BATCH_MB") ? std::strtoull(std::getenv("SF_BATCH_MB"), nullptr, 10) : 768ull) << 20;
  uint64_t T = std::max<uint64_t>(1, budget / std::max<uint64_t>(per_tile, 1));
  T = std::min<uint64_t>(T, tiles);
  T = std::min<uint64_t>(T, 65534);
  const bool wide = e.tc;  // the tensor-core kernels take tile pairs
  if (wide) T = (T + 1) & ~uint64_t(1);  // tile pairs: odd batches get an all-zero tile
  // one tail for every batch of the call (the same rounding for all rows):
  // tcgen05 when a full batch holds >= 64 tile pairs
  const bool tail_tc_call = e.tail_tc && (e.tail_tc_always || T / 2 >= 64);
  const bool deg = e.deg_capable && (e.deg_mode == 1 || (e.deg_mode == 2 && !tail_tc_call));
  // u16-degree mode: f32 isd rows only for B_1 (the mma.sync tail reads them)
  const uint64_t f32_stride = deg ? std::max<uint64_t>(e.U, 1) : e.V;
  const uint64_t off_isd = T * Wp * 8;
  const uint64_t off_h0 = off_isd + T * f32_stride * kTile * 4;
  const uint64_t off_h1 = off_h0 + T * hmax * 4;
  const uint64_t off_a = off_h1 + T * hmax * 4;
  const uint64_t off_p = off_a + T * amax * 4;
  const uint64_t off_af = off_p + T * apart * 4;
  const uint64_t off_d16 = (off_af + T * afused * 4 + 255) & ~uint64_t(255);
  const uint64_t d16_bytes = (e.tc16 || deg) ? T * uint64_t(e.V) * kTile * 2 : 0;  // u16 degrees
  ctx.work.reserve(off_d16 + d16_bytes + 256);
  unsigned char* base = ctx.work.p;
  uint64_t* maskt = reinterpret_cast<uint64_t*>(base);
  float* isd = reinterpret_cast<float*>(base + off_isd);
  float* hbuf[2] = {reinterpret_cast<float*>(base + off_h0), reinterpret_cast<float*>(base + off_h1)};
  float* abuf = reinterpret_cast<float*>(base + off_a);
  float* pbuf = reinterpret_cast<float*>(base + off_p);
  float* afbuf = reinterpret_cast<float*>(base + off_af);
  uint16_t* deg16 = (e.tc16 || deg) ? reinterpret_cast<uint16_t*>(base + off_d16) : nullptr;
  // f32 isd rows: every node, or (u16 degrees) B_1 for the mma.sync tail, or none
  const uint32_t f32_nodes = !deg ? uint32_t(e.V) : (tail_tc_call ? 0u : uint32_t(f32_stride));
  if (deg && tail_tc_call) isd = nullptr;
  for (uint64_t t0 = 0; t0 < tiles; t0 += T) {
    const uint64_t nt = std::min(T, tiles - t0);
    const uint64_t row0 = t0 * kTile;
    const uint64_t nrows = std::min<uint64_t>(rows - row0, nt * kTile);
    const uint64_t ntp = wide ? (nt + 1) & ~uint64_t(1) : nt;  // tiles the fused kernel covers
    if (kept_only)  // row0 is a multiple of 64: pairs from row0 / 2
      launch_transpose_pairs(ctx, dev_rows + (row0 / 2) * e.W, (nrows + 1) / 2, e.W, uint32_t(e.n), ntp, maskt);
    else
      launch_transpose_tiles(ctx, dev_rows + row0 * e.W, nrows, e.W, ntp, maskt);
    {
      // small-node warps: split the tiles when there are too few nodes to
      // fill 148 SMs x 64 warps (chunks of a multiple of 32 tiles)
      const uint64_t small = e.V - e.isd_nbig;
      uint64_t tchunk = ntp;
      if (small && small < 148ull * 64) {
        const uint64_t want = (148ull * 64 + small - 1) / small;
        tchunk = std::max<uint64_t>(32, ((ntp + want - 1) / want + 31) / 32 * 32);
        tchunk = std::min(tchunk, ntp);
      }
      const uint64_t tsplit = (ntp + tchunk - 1) / tchunk;
      const uint64_t warps = uint64_t(e.isd_nbig) * ntp + small * tsplit;
      isd_kernel<<<unsigned((warps + 7) / 8), 256, 0, ctx.stream>>>(
          maskt, Wp, uint32_t(ntp), e.row_ptr.p, e.edge_player.p, e.isd_order.p, e.isd_nbig,
          e.isd_tab.p, e.V, isd, deg16, uint32_t(tsplit), uint32_t(tchunk), f32_nodes, uint32_t(f32_stride));
      SF_LAUNCHED(ctx);
    }
    const float* X = e.p0.p;  // current layer input: P0 (shared) or per-coalition H
    bool shared_x = true;
    uint64_t Rin = e.V;
    int cur = 0;
    int l = 0;
    if (e.fused) {
      std::pair<cudaEvent_t, cudaEvent_t>* ev = nullptr;
      if (ctx.time_dominant) {
        if (ctx.dom_used == ctx.dom_events.size()) {
          std::pair<cudaEvent_t, cudaEvent_t> pr;
          SF_CUDA(cudaEventCreate(&pr.first));
          SF_CUDA(cudaEventCreate(&pr.second));
          ctx.dom_events.push_back(pr);
        }
        ev = &ctx.dom_events[ctx.dom_used++];
        ctx.dom_pairs += nrows / 2;
        SF_CUDA(cudaEventRecord(ev->first, ctx.stream));
      }
      const bool ok = (e.tc16 && launch_fused_tc16(ctx, e, maskt, Wp, isd, deg16, ntp, pbuf)) ||
                      (e.tc && launch_fused_tc(ctx, e, maskt, Wp, isd, deg ? deg16 : nullptr, ntp, pbuf)) ||
                      try_fused<128>(ctx, e, maskt, Wp, isd, nt, pbuf) ||
                      try_fused<64>(ctx, e, maskt, Wp, isd, nt, pbuf) ||
                      try_fused<32>(ctx, e, maskt, Wp, isd, nt, pbuf) ||
                      try_fused<16>(ctx, e, maskt, Wp, isd, nt, pbuf) ||
                      try_fused<256>(ctx, e, maskt, Wp, isd, nt, pbuf);
      if (!ok) throw std::logic_error("fused width not instantiated");
      if (ev) SF_CUDA(cudaEventRecord(ev->second, ctx.stream));
      const uint32_t K = uint32_t(e.dims[1]), N = uint32_t(e.dims[2]);
      if (tail_tc_call) {  // tcgen05 tail (sf_tail_tc.cu)
        launch_tail_tc(ctx, e, pbuf, maskt, Wp, isd, deg ? deg16 : nullptr, ntp, cls, row0, rows, dev_out,
                       dev_allprobs);
        continue;
      }
      if (L <= 3) {  // fused tail: reduce + layer 1 + last layer + softmax in one kernel
        // coalitions per CTA: 16 when the tile fits (the weights are staged
        // once per CTA; 16 measured 49.1 vs 50.5 ms/step for 4 at C2); the
        // whole tile when U == 1 (2-layer: little work per coalition, C5
        // 2.40 -> 2.28 s per 1,024-target batch)
        static const uint32_t cpb_env = std::getenv("SF_TAIL_CPB") ? uint32_t(std::atoi(std::getenv("SF_TAIL_CPB"))) : 0u;
        uint32_t cpb = cpb_env ? cpb_env : (e.U == 1 ? uint32_t(kTile) : 16u);
        while (cpb > 1 && tail_smem(e.U, K, N, C, cpb, L == 3) > kTailSmem) cpb /= 2;
        if (tail_smem(e.U, K, N, C, cpb, L == 3) <= kTailSmem) {
          const size_t smem = tail_smem(e.U, K, N, C, cpb, L == 3);
          set_max_dynamic_smem(tail_kernel, int(kTailSmem));
          dim3 grid(unsigned(nt), kTile / cpb);
          tail_kernel<<<grid, kTailThreads, smem, ctx.stream>>>(
              reinterpret_cast<const float4*>(pbuf), e.tc ? e.tc_items : e.items,
              e.tc ? e.tc_u_items.p : e.u_items.p, maskt, Wp, e.row_ptr.p, e.col.p,
              e.edge_player.p, isd, uint32_t(f32_stride), e.U, K, N, e.w[1]->p, e.b[1]->p,
              L == 3 ? e.w[2]->p : nullptr, L == 3 ? e.b[2]->p : nullptr, C, L == 3 ? 1 : 0, cls,
              row0, rows, cpb, dev_out, dev_allprobs);
          SF_LAUNCHED(ctx);
          continue;
        }
      }
      {
        const uint64_t work = uint64_t(e.U) * kTile * (K / 4);
        dim3 grid(unsigned((work + 255) / 256), unsigned(nt));
        reduce_partials_kernel<<<grid, 256, 0, ctx.stream>>>(
            reinterpret_cast<const float4*>(pbuf), e.tc ? e.tc_items : e.items,
            e.tc ? e.tc_u_items.p : e.u_items.p, isd, uint32_t(f32_stride), K / 4, e.U,
            reinterpret_cast<float4*>(afbuf));
        SF_LAUNCHED(ctx);
      }
      // layer 1: A W1 + b1 (ReLU for a hidden layer; logits when L == 2)
      gemm(ctx, afbuf, e.w[1]->p, e.b[1]->p, hbuf[0], nt * e.U * kTile, N, K, L >= 3);
      if (L == 2) {
        const uint64_t nb = nt * kTile;
        softmax_rows_kernel<<<unsigned((nb * 32 + 255) / 256), 256, 0, ctx.stream>>>(
            hbuf[0], N, row0, nb, rows, cls, dev_out, dev_allprobs);
        SF_LAUNCHED(ctx);
      }
      if (L == 2) continue;
      X = hbuf[0];
      shared_x = false;
      Rin = e.U;
      cur = 1;
      l = 2;
    }
    for (; l + 1 < L; ++l) {
      float* out = hbuf[cur];
      const uint32_t Rl = uint32_t(R[l]);
      const uint32_t Din = uint32_t(e.dims[l]), Dout = uint32_t(e.dims[l + 1]);
      dim3 grid(Rl, unsigned(nt));
      if (l == 0) {  // generic layer 0 (unsupported widths): aggregate P0, bias, ReLU
        agg_generic_kernel<<<grid, 256, 0, ctx.stream>>>(
            maskt, Wp, e.row_ptr.p, e.col.p, e.edge_player.p, isd, uint32_t(f32_stride), e.p0.p, 1, 0, Dout,
            e.b[0]->p, 1, Rl, out);
        SF_LAUNCHED(ctx);
      } else {
        agg_generic_kernel<<<grid, 256, 0, ctx.stream>>>(
            maskt, Wp, e.row_ptr.p, e.col.p, e.edge_player.p, isd, uint32_t(f32_stride), X, shared_x ? 1 : 0,
            uint32_t(Rin), Din, nullptr, 0, Rl, abuf);
        SF_LAUNCHED(ctx);
        gemm(ctx, abuf, e.w[l]->p, e.b[l]->p, out, nt * Rl * kTile, Dout, Din, true);
      }
      X = out;
      shared_x = false;
      Rin = Rl;
      cur ^= 1;
    }
    {
      const uint32_t Din = uint32_t(L == 1 ? C : e.dims[L - 1]);
      const float* Wt = (L == 1) ? nullptr : e.w[L - 1]->p;
      const uint32_t cpb = 8;  // coalitions per CTA
      const size_t smem = size_t(cpb) * (Din + C) * 4;
      if (smem > 48 * 1024)
        set_max_dynamic_smem(last_kernel, 227 * 1024);
      dim3 grid(unsigned(nt), kTile / cpb);
      last_kernel<<<grid, 256, smem, ctx.stream>>>(
          maskt, Wp, e.row_ptr.p, e.col.p, e.edge_player.p, isd, uint32_t(f32_stride), X, shared_x ? 1 : 0,
          uint32_t(Rin), Din, Wt, e.b[L - 1]->p, C, cls, row0, rows, cpb, dev_out, dev_allprobs);
      SF_LAUNCHED(ctx);
    }
  }
}

}  // namespace sfb
