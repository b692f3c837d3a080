// Standalone probe for the tcgen05 operand layouts used by sf_fused_tc.cu:
// A (128 x 32, K-major, no swizzle), B (32 x N) as MN-major (modes 0/1) or
// K-major (mode 2), D (128 x N f32 in TMEM), 4 k-steps of kind::tf32.
// Prints the max error against a CPU product. On B200 (driver 580) modes
// 0/1 returned all zeros and mode 2 was exact, so sf_fused_tc.cu stages both
// operands K-major. Build: nvcc -gencode arch=compute_100a,code=sm_100a
#include <cstdio>
#include <cstdint>
#include <cmath>
#include <vector>

constexpr int M = 128, K = 32, N = 128;
constexpr int B_SBO = (K / 8) * 128 + 16;

__device__ __forceinline__ uint32_t su32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ uint64_t smem_desc(uint32_t addr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= uint64_t((addr >> 4) & 0x3FFF);
  d |= uint64_t((lbo >> 4) & 0x3FFF) << 16;
  d |= uint64_t((sbo >> 4) & 0x3FFF) << 32;
  d |= uint64_t(1) << 46;
  return d;
}

__global__ void probe(const float* A, const float* B, float* D, int mode) {
  extern __shared__ __align__(1024) unsigned char smem[];
  __shared__ uint32_t tslot;
  __shared__ __align__(8) uint64_t bar;
  unsigned char* sa = smem;
  unsigned char* sb = smem + M * K * 4;  // 16 KB offset: 1024-aligned
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  // A[m][k]: offset (k/4)*2048 + (m/8)*128 + (m%8)*16 + (k%4)*4
  for (int idx = tid; idx < M * K; idx += blockDim.x) {
    const int m = idx / K, k = idx % K;
    *reinterpret_cast<float*>(sa + (k / 4) * 2048 + (m / 8) * 128 + (m % 8) * 16 + (k % 4) * 4) = A[m * K + k];
  }
  for (int idx = tid; idx < K * N; idx += blockDim.x) {
    const int k = idx / N, n = idx % N;
    const float bv = mode >= 6 ? (n == k ? 1.f : 0.f) : B[k * N + n];
    uint32_t off;
    if (mode == 3 || mode == 4)  // MN-major SWIZZLE_128B: atom (32 n x 8 k) = 1024 B, [n/32][k/8][atom]
      off = (n / 32) * (K / 8 * 1024) + (k / 8) * 1024 + (k % 8) * 128 + ((((n % 32) / 4) ^ (k % 8)) * 16) + (n % 4) * 4;
    else if (mode == 2)  // K-major B (N x K): (k/4)*(N/8*128) + (n/8)*128 + (n%8)*16 + (k%4)*4
      off = (k / 4) * (N / 8 * 128) + (n / 8) * 128 + (n % 8) * 16 + (k % 4) * 4;
    else            // MN-major: (n/4)*B_SBO + (k/8)*128 + (k%8)*16 + (n%4)*4
      off = (n / 4) * B_SBO + (k / 8) * 128 + (k % 8) * 16 + (n % 4) * 4;
    *reinterpret_cast<float*>(sb + off) = bv;
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(su32(&tslot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = tslot;
  if (mode >= 5 && warp < 4) {  // A -> TMEM columns 256.. (lane m = row, column k)
    const uint32_t lb = uint32_t(warp * 32) << 16;
    for (int k = 0; k < K; ++k) {
      const float f = mode == 6 ? float(warp * 32 + lane + 1) : mode == 7 ? float(k + 1) : A[(warp * 32 + lane) * K + k];
      const uint32_t v = __float_as_uint(f);
      asm volatile("tcgen05.st.sync.aligned.32x32b.x1.b32 [%0], {%1};" ::"r"(tmem + lb + 256 + k), "r"(v) : "memory");
    }
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  if (tid == 0 && mode >= 5) {
    const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | (uint32_t(N >> 3) << 17) | (uint32_t(M >> 4) << 24);
    for (int j = 0; j < K / 8; ++j) {
      const uint64_t bd = smem_desc(su32(sb) + j * 2 * (N / 8 * 128), N / 8 * 128, 128);
      const uint32_t acc = j > 0;
      asm volatile(
          "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
          "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n\t}" ::"r"(tmem),
          "r"(tmem + 256 + j * 8), "l"(bd), "r"(idesc), "r"(acc)
          : "memory");
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&bar))
                 : "memory");
  } else if (tid == 0) {
    const uint32_t b_major = mode == 2 ? 0u : 1u;
    const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | (b_major << 16) | (uint32_t(N >> 3) << 17) |
                           (uint32_t(M >> 4) << 24);
    for (int j = 0; j < K / 8; ++j) {
      const uint64_t ad = smem_desc(su32(sa) + j * 4096, 2048, 128);
      uint64_t bd;
      if (mode == 0) bd = smem_desc(su32(sb) + j * 128, 128, B_SBO);
      else if (mode == 1) bd = smem_desc(su32(sb) + j * 128, B_SBO, 128);
      else if (mode == 2) bd = smem_desc(su32(sb) + j * 2 * (N / 8 * 128), N / 8 * 128, 128);
      else if (mode == 3) bd = smem_desc(su32(sb) + j * 1024, K / 8 * 1024, 1024) | (uint64_t(2) << 61);
      else bd = smem_desc(su32(sb) + j * 1024, 1024, K / 8 * 1024) | (uint64_t(2) << 61);
      const uint32_t acc = j > 0;
      asm volatile(
          "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
          "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem),
          "l"(ad), "l"(bd), "r"(idesc), "r"(acc)
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
  if (warp < 4) {
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
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
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
  const int smem = M * K * 4 + (N / 4) * B_SBO + 4096;
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  for (int mode = 5; mode < 8; ++mode) {
    cudaMemset(dD, 0, D.size() * 4);
    probe<<<1, 128, smem>>>(dA, dB, dD, mode);
    cudaError_t e = cudaDeviceSynchronize();
    cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost);
    double err = 0, mx = 0;
    for (int i = 0; i < M * N; ++i) {
      err = std::max(err, double(std::fabs(D[i] - R[i])));
      mx = std::max(mx, double(std::fabs(R[i])));
    }
    if (mode >= 6) {
      printf("mode %d (%s): D[m][k] for m in {0,1,2,31,32,64,127}, k = 0..31\n", mode, mode == 6 ? "TMEM lane+1" : "TMEM column+1");
      for (int m : {0, 1, 2, 31, 32, 64, 127}) {
        printf("  m=%3d:", m);
        for (int k = 0; k < K; ++k) printf(" %g", D[m * N + k]);
        printf("\n");
      }
      continue;
    }
    printf("mode %d (%s B): status=%s max_abs_err=%.3g max_ref=%.3g D[0]=%g R[0]=%g D[1]=%g R[1]=%g D[N]=%g R[N]=%g\n",
           mode, mode == 5 ? "A in TMEM, K-major" : mode == 4 ? "MN-major SW128 swapped" : mode == 3 ? "MN-major SW128" : mode == 2 ? "K-major" : (mode ? "MN-major swapped lbo/sbo" : "MN-major"), cudaGetErrorString(e), err, mx, D[0], R[0], D[1], R[1], D[N], R[N]);
  }
  return 0;
}
