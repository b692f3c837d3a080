// Tensor-core tail of the 3-layer fused engine (hidden widths 128 / 128):
// everything after fused_tc_kernel for one tile pair (M = 128 coalitions),
// replacing tail_kernel's mma.sync path (gcn.cpp:103-154):
//   A_u[m][:]  = isd_m(u) * sum over the items of u of Apart[t][item][i][:]
//   H_u[m][:]  = relu(A_u[m][:] W1 + b1)                 tcgen05 kind::tf32, 3xTF32
//   a[m][:]    = isd_m(0) (isd_m(0) H_0[m] + sum_{kept v in N(0)} isd_m(v) H_v[m])
//   z[m][c]    = b2[c] + a[m][:] W2[:, c];  p = softmax(z[m]); out = p[cls]
// (m = coalition in the tile pair, t = tile, i = m mod 64, u over U = B_1).
// A_u goes into TMEM (lane = coalition, column = k; hi | lo tf32 split) and
// multiplies the pre-split, K-major W1 image in shared memory (one bulk copy
// per CTA from the per-model image built at engine_prepare); H_u is
// double-buffered in TMEM, so the epilogue of u overlaps the MMAs of u+1.
// The layer-2 aggregation a[m] stays in registers (two warps per TMEM lane
// quarter, 64 columns each).
#include <cuda_runtime.h>

#include <cstdlib>

#include "sf_device.cuh"
#include "sf_internal.hpp"
#include "sf_tcgen05.cuh"

namespace sfb {

namespace {

using namespace tc;

constexpr int kTile = 64;
constexpr int kM = 128;       // coalitions per CTA (tile pair)
constexpr int kD = 128;       // K = N = hidden width
constexpr int kThreads = 256; // 8 warps: staging, epilogue; warp 0 lane 0 issues the MMAs
constexpr uint32_t kLBO = (kD / 8) * 128;        // k-unit (4 tf32) stride of the K-major B image
constexpr uint32_t kWBytes = kD * kD * 4;        // one of hi | lo
constexpr uint32_t kOffW = 0;                    // W1 hi | lo image (128 KB)
constexpr uint32_t kOffW2 = 2 * kWBytes;         // W2 (kD x C floats), then a (kM x (kD+1)), barriers
constexpr int kMaxC = 64;

__device__ __forceinline__ float tf32_hi(float x) {
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
  return __uint_as_float(r);
}

// W1 (in x out row-major) -> K-major canonical image: row n = output
// feature, k-units of 4 inputs; hi then lo (same layout as the B bank)
__global__ void w1_image_kernel(const float* __restrict__ W1, float* __restrict__ img) {
  const int idx = blockIdx.x * blockDim.x + threadIdx.x;  // over (n, k4)
  if (idx >= kD * kD / 4) return;
  const int n = idx % kD, u = idx / kD;
  float v[4], h[4];
#pragma unroll
  for (int w = 0; w < 4; ++w) {
    v[w] = W1[(4 * u + w) * kD + n];
    h[w] = tf32_hi(v[w]);
  }
  unsigned char* out = reinterpret_cast<unsigned char*>(img);
  const uint32_t off = u * kLBO + (n >> 3) * 128 + (n & 7) * 16;
  *reinterpret_cast<float4*>(out + off) = make_float4(h[0], h[1], h[2], h[3]);
  *reinterpret_cast<float4*>(out + kWBytes + off) =
      make_float4(v[0] - h[0], v[1] - h[1], v[2] - h[2], v[3] - h[3]);
}

__global__ void __launch_bounds__(kThreads, 1)
    tail_tc_kernel(const float4* __restrict__ Apart, uint32_t items, const uint32_t* __restrict__ u_items,
                   uint32_t U, const uint64_t* __restrict__ maskt, uint64_t Wp, const uint32_t* __restrict__ row_ptr,
                   const uint32_t* __restrict__ col, const uint32_t* __restrict__ ep, const float* __restrict__ isd,
                   const uint16_t* __restrict__ deg16, const float* __restrict__ tab,
                   uint32_t V, const float* __restrict__ w1img, const float* __restrict__ b1,
                   const float* __restrict__ W2, const float* __restrict__ b2, uint32_t C, uint32_t cls,
                   uint64_t row0, uint64_t rows, float* __restrict__ out, float* __restrict__ allprobs,
                   float* __restrict__ apart_out, uint32_t* __restrict__ counters) {
  extern __shared__ __align__(1024) unsigned char smem[];
  float* sW2 = reinterpret_cast<float*>(smem + kOffW2);
  float* sA = sW2 + kD * C;  // a[m][:] after the u loop
  float* sZ2 = reinterpret_cast<float*>(smem + kOffW);  // z[m][:]: reuses the W1 image once the MMAs are done
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + ((kOffW2 + (kD * C + kM * (kD + 1)) * 4 + 15) & ~15u));
  uint64_t* w_full = bars;       // W1 image landed
  uint64_t* h_full = bars + 1;   // [2] MMAs of a u committed
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 3);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const uint64_t tp = blockIdx.x, t0 = 2 * tp;
  if (tid == 0) {
    mbar_init(w_full, 1);
    mbar_init(&h_full[0], 1);
    mbar_init(&h_full[1], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(su32(tmem_slot)),
                 "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  // TMEM columns: H buffers [0, 128) and [128, 256); A hi [256, 384), lo [384, 512)
  constexpr uint32_t kAcol = 2 * kD;
  if (tid == 0) {
    mbar_arrive_expect_tx(w_full, 2 * kWBytes);
    for (uint32_t c = 0; c < 2 * kWBytes; c += 32768)
      bulk_g2s(smem + kOffW + c, reinterpret_cast<const unsigned char*>(w1img) + c, 32768, w_full);
  }
  for (uint32_t idx = tid; idx < kD * C; idx += kThreads) sW2[idx] = __ldg(&W2[idx]);

  // per-thread coalition and column half (TMEM lane quarter = warp % 4)
  const int q = warp & 3, half = warp >> 2;
  const int m = q * 32 + lane;
  const uint64_t tile = t0 + (m >> 6);
  const int i = m & 63;
  // isd of node x for this coalition: f32 rows or u16 degrees + table
  const float* isd_t = isd ? isd + tile * uint64_t(V) * kTile : nullptr;
  const uint16_t* deg_t = deg16 ? deg16 + tile * uint64_t(V) * kTile : nullptr;
  auto isd_of = [&](uint32_t x) {
    return deg_t ? __ldg(&tab[__ldg(&deg_t[uint64_t(x) * kTile + i])]) : __ldg(&isd_t[uint64_t(x) * kTile + i]);
  };
  const uint64_t* mt = maskt + tile * Wp;
  const uint32_t lane_base = uint32_t(q * 32) << 16;
  const int c0 = half * (kD / 2);
  const float isd0 = isd_of(0);
  const uint32_t e_beg = row_ptr[0], e_end = row_ptr[1];
  float acc[kD / 2];
#pragma unroll
  for (int j = 0; j < kD / 2; ++j) acc[j] = 0.f;
  const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | (uint32_t(kD >> 3) << 17) | (uint32_t(kM >> 4) << 24);
  const uint64_t K4 = kD / 4;

  // u range of this CTA: gridDim.y CTAs split B_1 (their partial a's are
  // summed in CTA order by tail_finish_kernel)
  const uint32_t S = gridDim.y, ub = U * blockIdx.y / S, ue = U * (blockIdx.y + 1) / S;
  for (uint32_t u = ub; u < ue; ++u) {
    const uint32_t b = (u - ub) & 1u, ul = u - ub;
    // (1) A_u: this thread's coalition, columns [c0, c0 + 64): partial sums
    // in item order, isd(u) scale, tf32 hi/lo into TMEM
    if (ul >= 1) {  // the previous u's MMAs read the A region: wait for them
      mbar_wait(&h_full[(ul - 1) & 1u], ((ul - 1) >> 1) & 1u);
      tc_fence_after();
    }
    const float su = isd_of(u);
    const uint32_t ib = u_items[u], ie = u_items[u + 1];
#pragma unroll 1
    for (int cc = 0; cc < 2; ++cc) {  // 32-column chunks
      float4 s[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) s[j] = make_float4(0.f, 0.f, 0.f, 0.f);
      const float4* src = Apart + ((tile * items) * kTile + i) * K4 + (c0 + 32 * cc) / 4;
      uint32_t it = ib;
      for (; it + 2 <= ie; it += 2) {  // two items' loads in flight, summed in item order
        const float4* p = src + uint64_t(it) * kTile * K4;
        float4 v[8], w[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          v[j] = __ldg(p + j);
          w[j] = __ldg(p + uint64_t(kTile) * K4 + j);
        }
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          s[j].x += v[j].x;
          s[j].y += v[j].y;
          s[j].z += v[j].z;
          s[j].w += v[j].w;
          s[j].x += w[j].x;
          s[j].y += w[j].y;
          s[j].z += w[j].z;
          s[j].w += w[j].w;
        }
      }
      if (it < ie) {
        const float4* p = src + uint64_t(it) * kTile * K4;
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const float4 v = __ldg(p + j);
          s[j].x += v.x;
          s[j].y += v.y;
          s[j].z += v.z;
          s[j].w += v.w;
        }
      }
      uint32_t hv[32], lv[32];
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const float a4[4] = {su * s[j].x, su * s[j].y, su * s[j].z, su * s[j].w};
#pragma unroll
        for (int w = 0; w < 4; ++w) {
          const float h = tf32_hi(a4[w]);
          hv[4 * j + w] = __float_as_uint(h);
          lv[4 * j + w] = __float_as_uint(a4[w] - h);
        }
      }
      const uint32_t ta = tmem + lane_base + kAcol + c0 + 32 * cc;
      TC_ST32(ta, hv);
      TC_ST32(ta + kD, lv);
    }
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    // (2) MMAs: H_u[b] = A_u W1, 3xTF32, 16 k-steps
    if (tid == 0) {
      if (ul == 0) mbar_wait(w_full, 0);
      const uint32_t sw = su32(smem + kOffW);
      const uint32_t d = tmem + b * kD;
#pragma unroll 1
      for (int j = 0; j < kD / 8; ++j) {
        const uint64_t bh = smem_desc(sw + j * 2 * kLBO, kLBO, 128);
        const uint64_t bl = smem_desc(sw + kWBytes + j * 2 * kLBO, kLBO, 128);
        const uint32_t ahi = tmem + kAcol + j * 8, alo = ahi + kD;
        tc_mma_ts(d, ahi, bh, idesc, j > 0 ? 1u : 0u);
        tc_mma_ts(d, ahi, bl, idesc, 1u);
        tc_mma_ts(d, alo, bh, idesc, 1u);
      }
      tc_commit(&h_full[b]);
    }
    // (3) epilogue of u: relu(H + b1) scaled by the target-row coefficient
    mbar_wait(&h_full[b], (ul >> 1) & 1u);
    tc_fence_after();
    float coef;
    if (u == 0) {
      coef = isd0;
    } else {  // u in N(0): kept edge (0, u) and isd(u)
      coef = 0.f;
      for (uint32_t e = e_beg; e < e_end; ++e)
        if (col[e] == u) {
          coef = ((mt[ep[e]] >> i) & 1ull) ? su : 0.f;
          break;
        }
    }
    coef *= isd0;
#pragma unroll
    for (int cc = 0; cc < 2; ++cc) {
      uint32_t r[32];
      TC_LD32(tmem + lane_base + b * kD + c0 + 32 * cc, r);
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
      for (int j = 0; j < 32; ++j) {
        const float h = fmaxf(__uint_as_float(r[j]) + __ldg(&b1[c0 + 32 * cc + j]), 0.f);
        acc[32 * cc + j] = fmaf(coef, h, acc[32 * cc + j]);
      }
    }
    tc_fence_before();
  }
  if (S > 1) {
    // partial a of this u range -> [tp][s][m][k]; the last of the S CTAs of
    // the tile pair sums the partials in s order (deterministic) and finishes
    float* o = apart_out + ((tp * S + blockIdx.y) * kM + m) * uint64_t(kD) + c0;
#pragma unroll
    for (int j = 0; j < kD / 2; j += 4)
      *reinterpret_cast<float4*>(o + j) = make_float4(acc[j], acc[j + 1], acc[j + 2], acc[j + 3]);
    __threadfence();
    __syncthreads();
    uint32_t* flag = reinterpret_cast<uint32_t*>(tmem_slot + 1);
    if (counters == nullptr) {  // tail_finish_kernel sums the partials
      tc_fence_before();
      if (warp == 0) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
      }
      return;
    }
    if (tid == 0) {
      const uint32_t prev = atomicAdd(&counters[tp], 1u);
      *flag = prev == S - 1 ? 1u : 0u;
      if (prev == S - 1) counters[tp] = 0u;  // ready for the next launch
    }
    __syncthreads();
    if (*flag == 0u) {
      tc_fence_before();
      if (warp == 0) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
      }
      return;
    }
    __threadfence();
    for (uint32_t idx = tid; idx < kM * kD; idx += kThreads) {
      const uint32_t mm = idx / kD, k = idx % kD;
      float a = 0.f;
      for (uint32_t sidx = 0; sidx < S; ++sidx) a += __ldcg(&apart_out[((tp * S + sidx) * kM + mm) * uint64_t(kD) + k]);
      sA[mm * (kD + 1) + k] = a;
    }
  } else {
    // (4) a -> shared memory, z = b2 + a W2, softmax, p[cls]
    __syncthreads();
#pragma unroll
    for (int j = 0; j < kD / 2; ++j) sA[m * (kD + 1) + c0 + j] = acc[j];
  }
  __syncthreads();
  for (uint32_t idx = tid; idx < kM * C; idx += kThreads) {
    const uint32_t mm = idx / C, c = idx % C;
    float v0 = b2[c], v1 = 0.f;
    const float* a = sA + mm * (kD + 1);
#pragma unroll 4
    for (int k = 0; k < kD; k += 2) {
      v0 = fmaf(a[k], sW2[k * C + c], v0);
      v1 = fmaf(a[k + 1], sW2[(k + 1) * C + c], v1);
    }
    sZ2[idx] = v0 + v1;
  }
  __syncthreads();
  for (uint32_t mm = warp; mm < kM; mm += kThreads / 32) {
    const uint64_t row = row0 + t0 * kTile + mm;  // tiles t0, t0 + 1 of this batch
    if (row >= rows) continue;
    softmax_row_warp(sZ2 + mm * C, C, lane);
    if (lane == 0) out[row] = sZ2[mm * C + cls];
    __syncwarp();
    if (allprobs)
      for (uint32_t c = lane; c < C; c += 32) allprobs[row * C + c] = sZ2[mm * C + c];
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
  }
}

// a = sum of the u-range partials (CTA order), z = b2 + a W2, softmax, p[cls]
__global__ void __launch_bounds__(kThreads)
    tail_finish_kernel(const float* __restrict__ apart, uint32_t S, const float* __restrict__ W2,
                       const float* __restrict__ b2, uint32_t C, uint32_t cls, uint64_t row0, uint64_t rows,
                       float* __restrict__ out, float* __restrict__ allprobs) {
  extern __shared__ float fsm[];
  float* sW2 = fsm;                 // [kD][C]
  float* sA = sW2 + kD * C;         // [32][kD + 1]: 32 coalitions per CTA
  float* sZ = sA + 32 * (kD + 1);   // [32][C]
  const uint64_t tp = blockIdx.x;
  const uint32_t m0 = blockIdx.y * 32;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  // 16-byte loads, all of a thread's in flight before the first use (the
  // kernel is load-latency bound: ~50 KB per CTA from L2)
  {
    const float4* w4 = reinterpret_cast<const float4*>(W2);
    float4* s4 = reinterpret_cast<float4*>(sW2);
    const uint32_t n4 = kD * C / 4;  // kD is a multiple of 4
#pragma unroll 6
    for (uint32_t idx = tid; idx < n4; idx += kThreads) s4[idx] = __ldg(&w4[idx]);
  }
  {
    constexpr uint32_t kQ = 32 * kD / 4 / kThreads;  // float4 of a per thread (4)
    static_assert(32 * kD / 4 % kThreads == 0, "partial sums: whole float4 per thread");
    float4 acc[kQ];
#pragma unroll
    for (uint32_t q = 0; q < kQ; ++q) acc[q] = make_float4(0.f, 0.f, 0.f, 0.f);
    for (uint32_t sidx = 0; sidx < S; ++sidx) {
      float4 v[kQ];
#pragma unroll
      for (uint32_t q = 0; q < kQ; ++q) {
        const uint32_t idx = tid + q * kThreads, ml = idx / (kD / 4), k4 = idx % (kD / 4);
        v[q] = __ldg(reinterpret_cast<const float4*>(apart + ((tp * S + sidx) * kM + m0 + ml) * uint64_t(kD)) + k4);
      }
#pragma unroll
      for (uint32_t q = 0; q < kQ; ++q) {
        acc[q].x += v[q].x;
        acc[q].y += v[q].y;
        acc[q].z += v[q].z;
        acc[q].w += v[q].w;
      }
    }
#pragma unroll
    for (uint32_t q = 0; q < kQ; ++q) {
      const uint32_t idx = tid + q * kThreads, ml = idx / (kD / 4), k = 4 * (idx % (kD / 4));
      float* d = sA + ml * (kD + 1) + k;
      d[0] = acc[q].x;
      d[1] = acc[q].y;
      d[2] = acc[q].z;
      d[3] = acc[q].w;
    }
  }
  __syncthreads();
  for (uint32_t idx = tid; idx < 32 * C; idx += kThreads) {
    const uint32_t ml = idx / C, c = idx % C;
    float v0 = b2[c], v1 = 0.f;
    const float* a = sA + ml * (kD + 1);
#pragma unroll 4
    for (int k = 0; k < kD; k += 2) {
      v0 = fmaf(a[k], sW2[k * C + c], v0);
      v1 = fmaf(a[k + 1], sW2[(k + 1) * C + c], v1);
    }
    sZ[idx] = v0 + v1;
  }
  __syncthreads();
  for (uint32_t ml = warp; ml < 32; ml += kThreads / 32) {
    const uint64_t row = row0 + 2 * tp * kTile + m0 + ml;
    if (row >= rows) continue;
    softmax_row_warp(sZ + ml * C, C, lane);
    if (lane == 0) out[row] = sZ[ml * C + cls];
    __syncwarp();
    if (allprobs)
      for (uint32_t c = lane; c < C; c += 32) allprobs[row * C + c] = sZ[ml * C + c];
  }
}

}  // namespace

size_t tail_tc_smem(uint32_t C) {
  return ((size_t(kOffW2) + (size_t(kD) * C + size_t(kM) * (kD + 1)) * 4 + 15) & ~size_t(15)) + 64;
}

bool tail_tc_supported(const Engine& e) {
  return e.tc && !e.tc16 && e.L == 3 && e.dims[1] == kD && e.dims[2] == kD && e.dims[3] <= kMaxC &&
         tail_tc_smem(uint32_t(e.dims[3])) <= 227 * 1024;
}

void build_tail_tc(Ctx& ctx, Engine& e) {
  e.tail_w1img.reserve(2 * kD * kD);
  w1_image_kernel<<<(kD * kD / 4 + 255) / 256, 256, 0, ctx.stream>>>(e.w[1]->p, e.tail_w1img.p);
  SF_LAUNCHED(ctx);
}

void launch_tail_tc(Ctx& ctx, const Engine& e, const float* apart, const uint64_t* maskt, uint64_t Wp,
                    const float* isd, const uint16_t* deg16, uint64_t ntp, uint32_t cls, uint64_t row0,
                    uint64_t rows, float* out, float* allprobs) {
  const uint32_t C = uint32_t(e.dims[3]);
  const size_t smem = tail_tc_smem(C);
  set_max_dynamic_smem(tail_tc_kernel, int(227 * 1024));
  // split B_1 over S CTAs per tile pair when the tile pairs alone do not
  // fill the SMs (one CTA per SM: 512 TMEM columns, ~218 KB smem)
  int sms = 148;
  SF_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, ctx.device));
  const uint64_t tps = ntp / 2;
  uint32_t S = 1;
  while (S < e.U && tps * S < uint64_t(sms)) ++S;
  float* apart_out = nullptr;
  uint32_t* counters = nullptr;
  if (S > 1) {
    ctx.tail_part.reserve(tps * S * kM * kD);
    apart_out = ctx.tail_part.p;
    // the last CTA of a tile pair finishes (SF_TAIL_LAST=1) or a second
    // kernel does (default)
    static const bool last = std::getenv("SF_TAIL_LAST") && std::atoi(std::getenv("SF_TAIL_LAST")) != 0;
    if (last) {
      if (ctx.tail_count.n < tps) {  // zeroed once; the finishing CTA resets its counter
        ctx.tail_count.reserve(tps);
        SF_CUDA(cudaMemsetAsync(ctx.tail_count.p, 0, tps * 4, ctx.stream));
      }
      counters = ctx.tail_count.p;
    }
  }
  tail_tc_kernel<<<dim3(unsigned(tps), S), kThreads, smem, ctx.stream>>>(
      reinterpret_cast<const float4*>(apart), e.tc_items, e.tc_u_items.p, e.U, maskt, Wp, e.row_ptr.p, e.col.p,
      e.edge_player.p, isd, deg16, e.isd_tab.p, e.V, e.tail_w1img.p, e.b[1]->p, e.w[2]->p, e.b[2]->p, C, cls, row0, rows, out, allprobs,
      apart_out, counters);
  SF_LAUNCHED(ctx);
  if (S > 1 && counters == nullptr) {
    const size_t fsmem = (size_t(kD) * C + 32 * (kD + 1) + 32 * size_t(C)) * 4;
    set_max_dynamic_smem(tail_finish_kernel, int(fsmem));
    tail_finish_kernel<<<dim3(unsigned(tps), kM / 32), kThreads, fsmem, ctx.stream>>>(
        ctx.tail_part.p, S, e.w[2]->p, e.b[2]->p, C, cls, row0, rows, out, allprobs);
    SF_LAUNCHED(ctx);
  }
}

}  // namespace sfb
