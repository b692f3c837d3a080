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
// Arithmetic: FP32 on the CUDA cores (SIMT FFMA), accuracy mode "FP32".
#include <cuda_runtime.h>

#include <algorithm>

#include "sf_device.cuh"
#include "sf_internal.hpp"

namespace sfb {

namespace {

constexpr int kTile = 64;  // coalitions per tile

// ---------------------------------------------------------------- degrees
// deg_i(u) = 1 + sum over u's CSR entries of bit_i(edge_player) (the
// self-loop counts, gcn.cpp:76-81). One warp per (tile, node); the warp
// loads 32 incidences at once and broadcasts them with shuffles.
__global__ void __launch_bounds__(256)
    isd_kernel(const uint64_t* __restrict__ maskt, uint64_t Wp,
               const uint32_t* __restrict__ row_ptr,
               const uint32_t* __restrict__ ep, uint32_t V,
               float* __restrict__ isd) {
  const int lane = threadIdx.x & 31;
  const uint32_t u = blockIdx.x * 8 + (threadIdx.x >> 5);
  const uint64_t t = blockIdx.y;
  if (u >= V) return;
  const uint64_t* mt = maskt + t * Wp;
  uint32_t d0 = 1, d1 = 1;
  const uint32_t beg = row_ptr[u], end = row_ptr[u + 1];
  for (uint32_t i0 = beg; i0 < end; i0 += 32) {
    const uint32_t i = i0 + lane;
    const uint64_t w = i < end ? __ldg(&mt[ep[i]]) : 0ull;
    const uint32_t cnt = min(32u, end - i0);
    for (uint32_t k = 0; k < cnt; ++k) {
      const uint64_t wk = __shfl_sync(kFull, w, k);
      d0 += (wk >> lane) & 1u;
      d1 += (wk >> (lane + 32)) & 1u;
    }
  }
  float* out = isd + (t * V + u) * kTile;
  out[lane] = inv_sqrt_deg(d0);
  out[lane + 32] = inv_sqrt_deg(d1);
}

// ---------------------------------------------------------------- layer 0
// H[t][r][i][f] = relu(isd_i(r) * sum_{v in {r} u kept N(r)} isd_i(v) P[v][f]
//                     + bias[f])        (P = X W0, shared by all coalitions)
// One CTA per (tile, row r). Thread (cg, fg) owns features 4fg..4fg+3 of
// CB coalitions; the per-(neighbor, coalition) coefficients
// bit_i(e) * isd_i(v) are staged in shared memory 32 neighbors at a time,
// so each P row is fetched once per tile and reused by 64 coalitions.
template <int D>
struct L0Cfg {
  static constexpr int FG = D / 4;               // float4 lanes per row
  static constexpr int THREADS = 256;
  static constexpr int CGS = THREADS / FG;        // coalition groups
  static constexpr int CB = kTile / CGS;          // coalitions per thread
  static_assert(D % 4 == 0 && FG <= THREADS && kTile % CGS == 0, "shape");
};

template <int D, bool kRelu>
__global__ void __launch_bounds__(256)
    layer0_kernel(const uint64_t* __restrict__ maskt, uint64_t Wp,
                  const uint32_t* __restrict__ row_ptr,
                  const uint32_t* __restrict__ col,
                  const uint32_t* __restrict__ ep,
                  const float* __restrict__ isd, uint32_t V,
                  const float* __restrict__ P, const float* __restrict__ bias,
                  uint32_t R, float* __restrict__ H) {
  using Cfg = L0Cfg<D>;
  constexpr int KC = 32;
  __shared__ __align__(16) float coef[KC][kTile];
  __shared__ uint32_t nbr[KC];
  const uint32_t r = blockIdx.x;
  const uint64_t t = blockIdx.y;
  const int tid = threadIdx.x;
  const int fg = tid % Cfg::FG, cg = tid / Cfg::FG;
  const uint64_t* mt = maskt + t * Wp;
  const float* isd_t = isd + t * uint64_t(V) * kTile;

  float4 acc[Cfg::CB];
#pragma unroll
  for (int j = 0; j < Cfg::CB; ++j) acc[j] = make_float4(0.f, 0.f, 0.f, 0.f);

  const uint32_t beg = row_ptr[r], end = row_ptr[r + 1];
  // entry -1 is the self-loop (always kept)
  for (int64_t c0 = int64_t(beg) - 1; c0 < int64_t(end); c0 += KC) {
    const int64_t left = int64_t(end) - c0;
    const int cnt = left < KC ? int(left) : KC;
    __syncthreads();
    for (int idx = tid; idx < cnt * kTile; idx += Cfg::THREADS) {
      const int k = idx / kTile, i = idx % kTile;
      const int64_t e = c0 + k;
      float c;
      uint32_t v;
      if (e < int64_t(beg)) {
        v = r;
        c = isd_t[uint64_t(r) * kTile + i];
      } else {
        v = col[e];
        const uint64_t w = mt[ep[e]];
        c = ((w >> i) & 1ull) ? isd_t[uint64_t(v) * kTile + i] : 0.f;
      }
      coef[k][i] = c;
      if (i == 0) nbr[k] = v;
    }
    __syncthreads();
    for (int k = 0; k < cnt; ++k) {
      const float4 x = __ldg(reinterpret_cast<const float4*>(P + uint64_t(nbr[k]) * D) + fg);
      const float* ck = &coef[k][cg * Cfg::CB];
#pragma unroll
      for (int j = 0; j < Cfg::CB; ++j) {
        const float c = ck[j];
        acc[j].x = fmaf(c, x.x, acc[j].x);
        acc[j].y = fmaf(c, x.y, acc[j].y);
        acc[j].z = fmaf(c, x.z, acc[j].z);
        acc[j].w = fmaf(c, x.w, acc[j].w);
      }
    }
  }
  const float4 bv = reinterpret_cast<const float4*>(bias)[fg];
#pragma unroll
  for (int j = 0; j < Cfg::CB; ++j) {
    const int i = cg * Cfg::CB + j;
    const float s = isd_t[uint64_t(r) * kTile + i];
    float4 h;
    h.x = fmaf(s, acc[j].x, bv.x);
    h.y = fmaf(s, acc[j].y, bv.y);
    h.z = fmaf(s, acc[j].z, bv.z);
    h.w = fmaf(s, acc[j].w, bv.w);
    if (kRelu) {
      h.x = fmaxf(h.x, 0.f);
      h.y = fmaxf(h.y, 0.f);
      h.z = fmaxf(h.z, 0.f);
      h.w = fmaxf(h.w, 0.f);
    }
    reinterpret_cast<float4*>(H + ((t * R + r) * kTile + i) * D)[fg] = h;
  }
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
                 uint64_t M, uint32_t N, uint32_t K, int relu) {
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
      As[kk][mm] = (gm < M && gk < K) ? A[gm * K + gk] : 0.f;
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
// Target row only (gcn.cpp:134-140) + softmax (143-152), one CTA per tile.
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
                            uint32_t cls, uint64_t row0, uint64_t rows,
                            float* __restrict__ out,
                            float* __restrict__ allprobs) {
  extern __shared__ float sm[];
  float* a = sm;                  // [64][Din]
  float* z = sm + kTile * Din;    // [64][C]
  const uint64_t t = blockIdx.x;
  const uint64_t* mt = maskt + t * Wp;
  const float* isd_t = isd + t * uint64_t(V) * kTile;
  const uint32_t beg = row_ptr[0], end = row_ptr[1];
  for (uint32_t idx = threadIdx.x; idx < kTile * Din; idx += blockDim.x) {
    const uint32_t i = idx / Din, f = idx % Din;
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
  for (uint32_t idx = threadIdx.x; idx < kTile * C; idx += blockDim.x) {
    const uint32_t i = idx / C, c = idx % C;
    float v = bias[c];
    if (Wt) {
      // bias-first sequential accumulation as in affine_row (gcn.cpp:116-123)
      for (uint32_t k = 0; k < Din; ++k)
        v = __fadd_rn(v, __fmul_rn(a[i * Din + k], Wt[uint64_t(k) * C + c]));
    } else {
      v = __fadd_rn(a[i * Din + c], v);
    }
    z[idx] = v;
  }
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int nwarps = blockDim.x >> 5;
  for (int i = warp; i < kTile; i += nwarps) {
    const uint64_t row = row0 + t * kTile + i;
    if (row >= rows) continue;
    if (lane == 0) {
      float* zi = z + i * C;
      float mx = zi[0];
      for (uint32_t c = 1; c < C; ++c) mx = fmaxf(mx, zi[c]);
      float sum = 0.f;
      for (uint32_t c = 0; c < C; ++c) {
        zi[c] = expf(zi[c] - mx);
        sum += zi[c];
      }
      for (uint32_t c = 0; c < C; ++c) zi[c] = zi[c] / sum;
      out[row] = zi[cls];
    }
    __syncwarp();
    if (allprobs)
      for (uint32_t c = lane; c < C; c += 32) allprobs[row * C + c] = z[i * C + c];
  }
}

// X W0 for the whole subgraph (once per target)
void gemm(Ctx& ctx, const float* A, const float* B, const float* bias, float* Cm,
          uint64_t M, uint32_t N, uint32_t K, bool relu) {
  if (M == 0 || N == 0) return;
  dim3 grid((N + 63) / 64, unsigned((M + 63) / 64));
  sgemm_kernel<<<grid, 256, 0, ctx.stream>>>(A, B, bias, Cm, M, N, K, relu ? 1 : 0);
  SF_LAUNCHED(ctx);
}

template <int D>
bool try_layer0(Ctx& ctx, const uint64_t* maskt, uint64_t Wp, const Engine& e,
                const float* isd, const float* bias, uint32_t R, uint64_t T,
                float* H, bool relu) {
  if (e.dims[1] != uint64_t(D)) return false;
  dim3 grid(R, unsigned(T));
  if (relu)
    layer0_kernel<D, true><<<grid, 256, 0, ctx.stream>>>(
        maskt, Wp, e.row_ptr.p, e.col.p, e.edge_player.p, isd, e.V, e.p0.p, bias, R, H);
  else
    layer0_kernel<D, false><<<grid, 256, 0, ctx.stream>>>(
        maskt, Wp, e.row_ptr.p, e.col.p, e.edge_player.p, isd, e.V, e.p0.p, bias, R, H);
  SF_LAUNCHED(ctx);
  return true;
}

}  // namespace

void engine_prepare(Ctx& ctx, const Subgraph& sg, const Model& m) {
  Engine& e = ctx.engine;
  if (e.sg_id == sg.id && e.model_id == m.id) return;
  if (m.layers.empty()) throw DataError("model has no layers");
  if (m.layers.front().in != sg.feature_dim)
    throw DataError("model input dim " + std::to_string(m.layers.front().in) +
                    " does not match feature dim " + std::to_string(sg.feature_dim));
  e.sg_id = 0;
  e.V = sg.num_nodes();
  e.n = sg.num_players();
  e.W = static_cast<uint32_t>((e.n + 63) / 64);
  e.L = m.depth();
  e.dims.assign(1, m.layers.front().in);
  for (const Layer& l : m.layers) e.dims.push_back(l.out);
  e.ball = sg.ball_sizes(e.L);
  if (sg.col.size() >= (1ull << 32)) throw DataError("subgraph too large for u32 CSR");
  std::vector<uint32_t> rp(sg.row_ptr.begin(), sg.row_ptr.end());
  e.row_ptr.upload(rp.data(), rp.size(), ctx.stream);
  e.col.upload(sg.col.data(), sg.col.size(), ctx.stream);
  e.edge_player.upload(sg.edge_player.data(), sg.edge_player.size(), ctx.stream);
  // P0 = X W0 on the device
  DevBuf<float> x, w0;
  x.upload(sg.features.data(), sg.features.size(), ctx.stream);
  w0.upload(m.layers[0].weight.data(), m.layers[0].weight.size(), ctx.stream);
  e.p0.reserve(uint64_t(e.V) * e.dims[1]);
  gemm(ctx, x.p, w0.p, nullptr, e.p0.p, e.V, uint32_t(e.dims[1]), uint32_t(e.dims[0]), false);
  e.w.clear();
  e.b.clear();
  for (int l = 0; l < e.L; ++l) {
    e.w.emplace_back(new DevBuf<float>);
    e.b.emplace_back(new DevBuf<float>);
    if (l > 0) e.w[l]->upload(m.layers[l].weight.data(), m.layers[l].weight.size(), ctx.stream);
    e.b[l]->upload(m.layers[l].bias.data(), m.layers[l].bias.size(), ctx.stream);
  }
  ctx.h2d_bytes += (rp.size() + sg.col.size() + sg.edge_player.size()) * 4 + sg.features.size() * 4;
  for (const Layer& l : m.layers) ctx.h2d_bytes += (l.weight.size() + l.bias.size()) * 4;
  SF_CUDA(cudaStreamSynchronize(ctx.stream));  // temporaries x, w0 die here
  e.sg_id = sg.id;
  e.model_id = m.id;
}

void engine_predict(Ctx& ctx, const uint64_t* dev_rows, uint64_t rows,
                    uint32_t cls, float* dev_out, float* dev_allprobs,
                    float* dominant_ms) {
  Engine& e = ctx.engine;
  if (rows == 0) return;
  const uint64_t tiles = (rows + kTile - 1) / kTile;
  const uint64_t Wp = uint64_t(e.W) * 64;
  const int L = e.L;
  const uint32_t C = uint32_t(e.dims[L]);
  // rows each layer produces: R_l = |B_{L-1-l}|
  std::vector<uint64_t> R(L);
  for (int l = 0; l < L; ++l) R[l] = e.ball[L - 1 - l];
  // per-tile bytes: masks + isd + two activation buffers + aggregation
  uint64_t hmax = 0, amax = 0;
  for (int l = 0; l + 1 < L; ++l) hmax = std::max(hmax, R[l] * kTile * e.dims[l + 1]);
  for (int l = 1; l + 1 < L; ++l) amax = std::max(amax, R[l] * kTile * e.dims[l]);
  const uint64_t per_tile = Wp * 8 + uint64_t(e.V) * kTile * 4 + (2 * hmax + amax) * 4;
  const uint64_t budget = 96ull << 20;  // keep a batch's intermediates L2-sized
  uint64_t T = std::max<uint64_t>(1, budget / std::max<uint64_t>(per_tile, 1));
  T = std::min<uint64_t>(T, tiles);
  T = std::min<uint64_t>(T, 65535);
  const uint64_t off_isd = T * Wp * 8;
  const uint64_t off_h0 = off_isd + T * uint64_t(e.V) * kTile * 4;
  const uint64_t off_h1 = off_h0 + T * hmax * 4;
  const uint64_t off_a = off_h1 + T * hmax * 4;
  ctx.work.reserve(off_a + T * amax * 4 + 256);
  unsigned char* base = ctx.work.p;
  uint64_t* maskt = reinterpret_cast<uint64_t*>(base);
  float* isd = reinterpret_cast<float*>(base + off_isd);
  float* hbuf[2] = {reinterpret_cast<float*>(base + off_h0), reinterpret_cast<float*>(base + off_h1)};
  float* abuf = reinterpret_cast<float*>(base + off_a);

  (void)dominant_ms;
  for (uint64_t t0 = 0; t0 < tiles; t0 += T) {
    const uint64_t nt = std::min(T, tiles - t0);
    const uint64_t row0 = t0 * kTile;
    const uint64_t nrows = std::min<uint64_t>(rows - row0, nt * kTile);
    launch_transpose_tiles(ctx, dev_rows + row0 * e.W, nrows, e.W, nt, maskt);
    {
      dim3 grid((e.V + 7) / 8, unsigned(nt));
      isd_kernel<<<grid, 256, 0, ctx.stream>>>(maskt, Wp, e.row_ptr.p, e.edge_player.p, e.V, isd);
      SF_LAUNCHED(ctx);
    }
    const float* X = e.p0.p;  // layer input: P0 (shared) or per-coalition H
    bool shared_x = true;
    uint64_t Rin = e.V;
    int cur = 0;
    for (int l = 0; l + 1 < L; ++l) {
      float* out = hbuf[cur];
      const uint32_t Rl = uint32_t(R[l]);
      if (l == 0) {
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
        const float* b0 = e.b[0]->p;
        bool done = try_layer0<128>(ctx, maskt, Wp, e, isd, b0, Rl, nt, out, true) ||
                    try_layer0<64>(ctx, maskt, Wp, e, isd, b0, Rl, nt, out, true) ||
                    try_layer0<32>(ctx, maskt, Wp, e, isd, b0, Rl, nt, out, true) ||
                    try_layer0<16>(ctx, maskt, Wp, e, isd, b0, Rl, nt, out, true) ||
                    try_layer0<256>(ctx, maskt, Wp, e, isd, b0, Rl, nt, out, true);
        if (!done) {
          dim3 grid(Rl, unsigned(nt));
          agg_generic_kernel<<<grid, 256, 0, ctx.stream>>>(
              maskt, Wp, e.row_ptr.p, e.col.p, e.edge_player.p, isd, e.V, e.p0.p, 1, 0,
              uint32_t(e.dims[1]), b0, 1, Rl, out);
          SF_LAUNCHED(ctx);
        }
        if (ev) SF_CUDA(cudaEventRecord(ev->second, ctx.stream));
      } else {
        const uint32_t Din = uint32_t(e.dims[l]), Dout = uint32_t(e.dims[l + 1]);
        dim3 grid(Rl, unsigned(nt));
        agg_generic_kernel<<<grid, 256, 0, ctx.stream>>>(
            maskt, Wp, e.row_ptr.p, e.col.p, e.edge_player.p, isd, e.V, X, 0, uint32_t(Rin), Din,
            nullptr, 0, Rl, abuf);
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
      const size_t smem = size_t(kTile) * (Din + C) * 4;
      if (smem > 48 * 1024)
        SF_CUDA(cudaFuncSetAttribute(last_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     int(std::min<size_t>(smem, 227 * 1024))));
      last_kernel<<<unsigned(nt), 256, smem, ctx.stream>>>(
          maskt, Wp, e.row_ptr.p, e.col.p, e.edge_player.p, isd, e.V, X, shared_x ? 1 : 0,
          uint32_t(Rin), Din, Wt, e.b[L - 1]->p, C, cls, row0, rows, dev_out - row0 + row0,
          dev_allprobs);
      SF_LAUNCHED(ctx);
    }
  }
}

}  // namespace sfb
