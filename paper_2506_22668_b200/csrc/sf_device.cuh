// Device helpers shared by the sm_100a kernels.
#pragma once

#include <cstdint>

namespace sfb {

constexpr unsigned kFull = 0xffffffffu;

// Philox-4x32-10 block (philox.hpp:39-66): key = (lo, hi) of seed, counter
// = (lo, hi) of the block index followed by (lo, hi) of the stream. The two
// u64 draws of a block, in the order the reference hands them out
// (philox.hpp:21-27), are first = (b3 << 32) | b2, second = (b1 << 32) | b0.
__device__ __forceinline__ void philox_block(uint64_t seed, uint64_t stream,
                                             uint64_t block, uint64_t& first,
                                             uint64_t& second) {
  uint32_t c0 = static_cast<uint32_t>(block), c1 = static_cast<uint32_t>(block >> 32);
  uint32_t c2 = static_cast<uint32_t>(stream), c3 = static_cast<uint32_t>(stream >> 32);
  uint32_t k0 = static_cast<uint32_t>(seed), k1 = static_cast<uint32_t>(seed >> 32);
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    const uint32_t lo0 = 0xD2511F53u * c0, hi0 = __umulhi(0xD2511F53u, c0);
    const uint32_t lo1 = 0xCD9E8D57u * c2, hi1 = __umulhi(0xCD9E8D57u, c2);
    const uint32_t n0 = hi1 ^ c1 ^ k0, n2 = hi0 ^ c3 ^ k1;
    c0 = n0;
    c1 = lo1;
    c2 = n2;
    c3 = lo0;
    k0 += 0x9E3779B9u;
    k1 += 0xBB67AE85u;
  }
  first = (static_cast<uint64_t>(c3) << 32) | c2;
  second = (static_cast<uint64_t>(c1) << 32) | c0;
}

// Exact x mod d for a u64 x and a 32-bit d > 0 (the reference takes
// next_u64() % (m + 1) in 64-bit arithmetic, sampler.cpp:59). Two 32-bit
// steps: (hi mod d) then ((r << 32) | lo) mod d, the second with a
// quotient that fits 32 bits.
__device__ __forceinline__ uint32_t mod_u64_u32(uint64_t x, uint32_t d) {
  // x % d exactly: r = hi % d, then y = r:lo < d * 2^32, so y / d < 2^32.
  // Both quotients come from the same FP64 reciprocal (53-bit: the
  // estimates are off by at most one, fixed below) — no integer division.
  const double rd = __drcp_rn(static_cast<double>(d));
  const uint32_t hi = static_cast<uint32_t>(x >> 32);
  const uint32_t q1 = __double2uint_rz(__dmul_rz(static_cast<double>(hi), rd));
  int64_t r = static_cast<int64_t>(hi) - static_cast<int64_t>(q1) * d;
  if (r < 0) r += d;
  if (r >= static_cast<int64_t>(d)) r -= d;
  const uint64_t y = (static_cast<uint64_t>(r) << 32) | static_cast<uint32_t>(x);
  const uint64_t q = static_cast<uint64_t>(__dmul_rz(__ull2double_rz(y), rd));
  int64_t rem = static_cast<int64_t>(y - q * d);
  if (rem < 0) rem += d;
  if (rem >= static_cast<int64_t>(d)) rem -= d;
  return static_cast<uint32_t>(rem);
}

__device__ __forceinline__ float inv_sqrt_deg(uint32_t deg) {
  // 1.0f / std::sqrt(static_cast<float>(deg)) with IEEE-rounded sqrt and
  // division, bitwise equal to the reference (gcn.cpp:82)
  return __fdiv_rn(1.0f, __fsqrt_rn(static_cast<float>(deg)));
}

// float softmax of one row in place (max subtraction, gcn.cpp:143-152), one warp
__device__ __forceinline__ void softmax_row_warp(float* zi, uint32_t C, int lane) {
  float mx = -INFINITY;
  for (uint32_t c = lane; c < C; c += 32) mx = fmaxf(mx, zi[c]);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  float sum = 0.f;
  for (uint32_t c = lane; c < C; c += 32) {
    const float e = expf(zi[c] - mx);
    zi[c] = e;
    sum += e;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
  for (uint32_t c = lane; c < C; c += 32) zi[c] = zi[c] / sum;
  __syncwarp();
}

// one 32 x 32 bit-transpose butterfly stage (see Bfly in sf_gcn.cu): send
// rot(x) & keep to the lane s away, keep x & keep
__device__ __forceinline__ uint32_t bfly_step(uint32_t x, int s, uint32_t keep, uint32_t amt) {
  const uint32_t send = __funnelshift_r(x, x, amt) & keep;
  return (x & keep) | __shfl_xor_sync(0xffffffffu, send, s);
}

}  // namespace sfb
