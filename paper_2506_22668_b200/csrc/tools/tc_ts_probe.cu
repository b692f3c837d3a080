// Probe: tcgen05.mma kind::tf32 with A in TMEM (".ts"). A cell (lane m,
// column 256 + c) holds c + 1 (lane-independent); B (K-major smem) is the
// 8 x N identity; one MMA reads A at column 256 + aoff. D[0][n] for n < 8
// shows which TMEM column fed A[:, n]. Build: nvcc -gencode
// arch=compute_100a,code=sm_100a tc_ts_probe.cu
#include <cstdint>
#include <cstdio>

constexpr int M = 128, N = 128, K = 32;

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

__global__ void probe(float* D, int aoff, int stx, int nmma) {
  __shared__ __align__(1024) unsigned char sb[K * N * 4];
  __shared__ uint32_t tslot;
  __shared__ __align__(8) uint64_t bar;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  for (int idx = tid; idx < K * N; idx += blockDim.x) {
    const int k = idx / N, n = idx % N;
    const uint32_t off = (k / 4) * (N / 8 * 128) + (n / 8) * 128 + (n % 8) * 16 + (k % 4) * 4;
    *reinterpret_cast<float*>(sb + off) = n == k ? 1.f : 0.f;
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
  const uint32_t lb = uint32_t(warp * 32) << 16;
  if (stx == 1) {
    for (int c = 0; c < 64; ++c) {
      const uint32_t v = __float_as_uint(float(c + 1));
      asm volatile("tcgen05.st.sync.aligned.32x32b.x1.b32 [%0], {%1};" ::"r"(tmem + lb + 256 + c), "r"(v) : "memory");
    }
  } else {  // .x8 stores, 8 columns at a time
    for (int c0 = 0; c0 < 64; c0 += 8) {
      uint32_t v[8];
      for (int j = 0; j < 8; ++j) v[j] = __float_as_uint(float(c0 + j + 1));
      asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(tmem + lb + 256 + c0),
                   "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7])
                   : "memory");
    }
  }
  asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  if (tid == 0) {
    const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | (uint32_t(N >> 3) << 17) | (uint32_t(M >> 4) << 24);
    for (int j = 0; j < nmma; ++j) {
      const uint64_t bd = smem_desc(su32(sb) + j * 2 * (N / 8 * 128), N / 8 * 128, 128);
      asm volatile(
          "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
          "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n\t}" ::"r"(tmem),
          "r"(tmem + 256 + aoff + j * 8), "l"(bd), "r"(idesc), "r"(uint32_t(j > 0))
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
  for (int c = 0; c < 32; ++c) {
    uint32_t r;
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x1.b32 {%0}, [%1];" : "=r"(r) : "r"(tmem + lb + c));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
    D[(warp * 32 + lane) * 32 + c] = __uint_as_float(r);
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
  }
}

int main() {
  float* dD;
  cudaMalloc(&dD, M * 32 * 4);
  float h[M * 32];
  for (int nmma = 1; nmma <= 4; ++nmma)
    for (int aoff : {0, 8}) {
      const int stx = 8;
      cudaMemset(dD, 0, M * 32 * 4);
      probe<<<1, 128>>>(dD, aoff, stx, nmma);
      cudaError_t e = cudaDeviceSynchronize();
      cudaMemcpy(h, dD, sizeof(h), cudaMemcpyDeviceToHost);
      printf("nmma=%d aoff=%2d (%s): m=77:", nmma, aoff, cudaGetErrorString(e));
      for (int n = 0; n < 32; ++n) printf(" %g", h[77 * 32 + n]);
      printf("\n");
    }
  return 0;
}
