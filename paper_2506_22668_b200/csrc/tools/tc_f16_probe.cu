// Probe: tcgen05.mma kind::f16 (fp16 in, f32 accumulate), M = 128, N = 128,
// K = 32 (two K = 16 MMAs), A in TMEM (two fp16 per 32-bit column), B in
// shared memory MN-major (N contiguous) in candidate canonical layouts.
// Prints which (layout, LBO, SBO, A packing) combination is exact.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a tc_f16_probe.cu
#include <cuda_fp16.h>
#include <cstdint>
#include <cstdio>
#include <cmath>
#include <vector>

constexpr int M = 128, N = 128, K = 32;

__device__ __forceinline__ uint32_t su32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ uint64_t desc(uint32_t addr, uint32_t lbo, uint32_t sbo, uint32_t layout) {
  uint64_t d = 0;
  d |= uint64_t((addr >> 4) & 0x3FFF);
  d |= uint64_t((lbo >> 4) & 0x3FFF) << 16;
  d |= uint64_t((sbo >> 4) & 0x3FFF) << 32;
  d |= uint64_t(1) << 46;
  d |= uint64_t(layout) << 61;  // 0 none, 2 SWIZZLE_128B
  return d;
}

// B element (k, n) byte offset for the candidate layouts
__device__ uint32_t boff(int k, int n, int lay) {
  if (lay == 0) {  // SW128, atom = 64 n x 8 k (1024 B); n-atoms adjacent (1024), k-atoms 2048 apart
    const int an = n / 64, ak = k / 8, r = k % 8, c16 = (n % 64) / 8;
    return (ak * 2 + an) * 1024 + r * 128 + ((c16 ^ r) * 16) + (n % 8) * 2;
  }
  if (lay == 1) {  // SW128, k-atoms adjacent (1024), n-atoms 4096 apart (K = 32: 4 k-atoms)
    const int an = n / 64, ak = k / 8, r = k % 8, c16 = (n % 64) / 8;
    return (an * 4 + ak) * 1024 + r * 128 + ((c16 ^ r) * 16) + (n % 8) * 2;
  }
  // lay 2: no swizzle MN-major "interleave": core matrix = 8 n (16 B) x 8 k rows = 128 B;
  // core matrices: n-groups adjacent (128 B apart), k-groups (N/8)*128 apart
  const int gn = n / 8, gk = k / 8, r = k % 8;
  return gk * (N / 8) * 128 + gn * 128 + r * 16 + (n % 8) * 2;
}

__global__ void probe(const float* A, const float* B, float* D, int lay, uint32_t lbo, uint32_t sbo, int pack) {
  extern __shared__ __align__(1024) unsigned char sb[];
  __shared__ uint32_t tslot;
  __shared__ __align__(8) uint64_t bar;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  for (int i = tid; i < K * N * 2; i += blockDim.x) sb[i] = 0;
  __syncthreads();
  for (int idx = tid; idx < K * N; idx += blockDim.x) {
    const int k = idx / N, n = idx % N;
    *reinterpret_cast<__half*>(sb + boff(k, n, lay)) = __float2half(B[k * N + n]);
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"(su32(&tslot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = tslot;
  {  // A -> TMEM columns 128.., two fp16 per column
    const uint32_t lb = uint32_t(warp * 32) << 16;
    const int m = warp * 32 + lane;
    for (int c = 0; c < K / 2; ++c) {
      const __half a0 = __float2half(A[m * K + 2 * c]), a1 = __float2half(A[m * K + 2 * c + 1]);
      const uint32_t lo = __half_as_ushort(pack ? a1 : a0), hi = __half_as_ushort(pack ? a0 : a1);
      const uint32_t v = lo | (hi << 16);
      asm volatile("tcgen05.st.sync.aligned.32x32b.x1.b32 [%0], {%1};" ::"r"(tmem + lb + 128 + c), "r"(v) : "memory");
    }
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  if (tid == 0) {
    // kind::f16: c F32 (bit 4), a/b F16 (0), a K-major, b MN-major (bit 16)
    const uint32_t idesc = (1u << 4) | (1u << 16) | (uint32_t(N >> 3) << 17) | (uint32_t(M >> 4) << 24);
    for (int j = 0; j < K / 16; ++j) {
      // k-step j covers k = 16 j .. 16 j + 15
      uint32_t start;
      if (lay == 0) start = su32(sb) + j * 2 * 2048;       // two k-atoms per step, k-atoms 2048 apart
      else if (lay == 1) start = su32(sb) + j * 2 * 1024;  // k-atoms 1024 apart
      else start = su32(sb) + j * 2 * (N / 8) * 128;
      const uint64_t bd = desc(start, lbo, sbo, lay == 2 ? 0 : 2);
      asm volatile(
          "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
          "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(tmem), "r"(tmem + 128 + j * 8),
          "l"(bd), "r"(idesc), "r"(uint32_t(j > 0))
          : "memory");
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&bar))
                 : "memory");
  }
  __syncwarp();
  asm volatile(
      "{\n\t.reg .pred p;\n\tW:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n\t@!p bra W;\n\t}" ::"r"(su32(&bar))
      : "memory");
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  {
    const uint32_t lb = uint32_t(warp * 32) << 16;
    for (int c = 0; c < N; ++c) {
      uint32_t r;
      asm volatile("tcgen05.ld.sync.aligned.32x32b.x1.b32 {%0}, [%1];" : "=r"(r) : "r"(tmem + lb + c));
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
      D[(warp * 32 + lane) * N + c] = __uint_as_float(r);
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;" ::"r"(tmem));
  }
}

int main() {
  std::vector<float> A(M * K), B(K * N), D(M * N), R(M * N, 0.f);
  for (int i = 0; i < M * K; ++i) A[i] = float((i * 37) % 17) / 8.0f - 1.0f;
  for (int i = 0; i < K * N; ++i) B[i] = float((i * 29) % 13) / 4.0f - 1.5f;
  for (int m = 0; m < M; ++m)
    for (int n = 0; n < N; ++n)
      for (int k = 0; k < K; ++k) R[m * N + n] += A[m * K + k] * B[k * N + n];
  float *dA, *dB, *dD;
  cudaMalloc(&dA, A.size() * 4);
  cudaMalloc(&dB, B.size() * 4);
  cudaMalloc(&dD, D.size() * 4);
  cudaMemcpy(dA, A.data(), A.size() * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(dB, B.data(), B.size() * 4, cudaMemcpyHostToDevice);
  const int smem = 16384;
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const uint32_t cand[] = {16, 128, 256, 1024, 2048, 4096};
  for (int lay = 0; lay < 3; ++lay)
    for (int pack = 0; pack < 2; ++pack)
      for (uint32_t lbo : cand)
        for (uint32_t sbo : cand) {
          cudaMemset(dD, 0, D.size() * 4);
          probe<<<1, 128, smem>>>(dA, dB, dD, lay, lbo, sbo, pack);
          cudaError_t e = cudaDeviceSynchronize();
          if (e != cudaSuccess) {
            printf("lay %d pack %d lbo %u sbo %u: %s\n", lay, pack, lbo, sbo, cudaGetErrorString(e));
            return 1;
          }
          cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost);
          double err = 0;
          for (int i = 0; i < M * N; ++i) err = std::max(err, double(std::fabs(D[i] - R[i])));
          if (err < 1e-3) printf("EXACT: lay %d pack %d lbo %u sbo %u\n", lay, pack, lbo, sbo);
        }
  printf("done\n");
  return 0;
}
