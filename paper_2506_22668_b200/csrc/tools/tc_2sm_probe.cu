// Probe: tcgen05.mma.cta_group::2.kind::tf32, M = 256 (rows 0-127 in CTA
// rank 0's TMEM, 128-255 in rank 1's), N = 128 (columns 0-63 of B in rank
// 0's shared memory, 64-127 in rank 1's, same offsets), K = 32 (4 MMAs),
// A in TMEM, B K-major without swizzle. Rank 0 issues; the commit is
// multicast to both CTAs. Each CTA then reads its 128 rows x 128 columns.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a tc_2sm_probe.cu
#include <cstdint>
#include <cstdio>
#include <cmath>
#include <vector>

constexpr int M = 256, N = 128, K = 32, NH = N / 2;

__device__ __forceinline__ uint32_t su32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ uint64_t desc(uint32_t addr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= uint64_t((addr >> 4) & 0x3FFF);
  d |= uint64_t((lbo >> 4) & 0x3FFF) << 16;
  d |= uint64_t((sbo >> 4) & 0x3FFF) << 32;
  d |= uint64_t(1) << 46;
  return d;
}
__device__ __forceinline__ uint32_t cta_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

__global__ void __cluster_dims__(2, 1, 1) probe(const float* A, const float* B, float* D) {
  __shared__ __align__(1024) unsigned char sb[K * NH * 4];
  __shared__ uint32_t tslot;
  __shared__ __align__(8) uint64_t bar;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const uint32_t rank = cta_rank();
  // B half: this CTA's columns n = rank*64 .. +63, K-major: (k/4)*(NH/8*128) + (n/8)*128 + (n%8)*16 + (k%4)*4
  for (int idx = tid; idx < K * NH; idx += blockDim.x) {
    const int k = idx / NH, nl = idx % NH, n = int(rank) * NH + nl;
    *reinterpret_cast<float*>(sb + (k / 4) * (NH / 8 * 128) + (nl / 8) * 128 + (nl % 8) * 16 + (k % 4) * 4) =
        B[k * N + n];
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"(su32(&tslot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  cluster_sync();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = tslot;
  {  // A rows rank*128 + m -> TMEM lane m, columns 128 + k
    const uint32_t lb = uint32_t(warp * 32) << 16;
    const int m = int(rank) * 128 + warp * 32 + lane;
    for (int k = 0; k < K; ++k) {
      const uint32_t v = __float_as_uint(A[m * K + k]);
      asm volatile("tcgen05.st.sync.aligned.32x32b.x1.b32 [%0], {%1};" ::"r"(tmem + lb + 128 + k), "r"(v) : "memory");
    }
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  cluster_sync();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  if (rank == 0 && tid == 0) {
    const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | (uint32_t(N >> 3) << 17) | (uint32_t(M >> 4) << 24);
    for (int j = 0; j < K / 8; ++j) {
      const uint64_t bd = desc(su32(sb) + j * 2 * (NH / 8 * 128), NH / 8 * 128, 128);
      asm volatile(
          "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
          "tcgen05.mma.cta_group::2.kind::tf32 [%0], [%1], %2, %3, p;\n\t}" ::"r"(tmem), "r"(tmem + 128 + j * 8),
          "l"(bd), "r"(idesc), "r"(uint32_t(j > 0))
          : "memory");
    }
    asm volatile(
        "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
            su32(&bar)),
        "h"(uint16_t(3))
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
    const int m = int(rank) * 128 + warp * 32 + lane;
    for (int c = 0; c < N; ++c) {
      uint32_t r;
      asm volatile("tcgen05.ld.sync.aligned.32x32b.x1.b32 {%0}, [%1];" : "=r"(r) : "r"(tmem + lb + c));
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
      D[m * N + c] = __uint_as_float(r);
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  cluster_sync();
  if (warp == 0) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 256;" ::"r"(tmem));
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
  cudaMemset(dD, 0, D.size() * 4);
  probe<<<2, 128>>>(dA, dB, dD);
  cudaError_t e = cudaDeviceSynchronize();
  cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost);
  double err = 0, mx = 0;
  for (int i = 0; i < M * N; ++i) {
    err = std::max(err, double(std::fabs(D[i] - R[i])));
    mx = std::max(mx, double(std::fabs(R[i])));
  }
  printf("2SM TS: %s max_abs_err=%.3g max_ref=%.3g D[0]=%g R[0]=%g D[130*N+70]=%g R=%g\n", cudaGetErrorString(e),
         err, mx, D[0], R[0], D[130 * N + 70], R[130 * N + 70]);
  return 0;
}
