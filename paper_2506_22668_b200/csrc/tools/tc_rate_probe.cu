// Probe: issue and completion rate of tcgen05.mma kind::tf32, M = 128,
// K = 8, for N in {64, 128, 256}, A from TMEM (ts) or shared memory (ss),
// B K-major in shared memory (no swizzle). One CTA, one issuing thread,
// `count` back-to-back MMAs into one accumulator, then one commit.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a tc_rate_probe.cu
#include <cstdint>
#include <cstdio>

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

__global__ void rate(int N, int ts, int count, long long* out) {
  extern __shared__ __align__(1024) unsigned char sm[];
  __shared__ uint32_t tslot;
  __shared__ __align__(8) uint64_t bar;
  const int tid = threadIdx.x, warp = tid >> 5;
  for (int i = tid; i < 64 * 1024 / 4; i += blockDim.x) reinterpret_cast<float*>(sm)[i] = 0.5f;
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
  if (tid == 0) {
    const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | (uint32_t(N >> 3) << 17) | (uint32_t(128 >> 4) << 24);
    const uint32_t sa = su32(sm), sb = su32(sm + 32768);
    const long long t0 = clock64();
    for (int i = 0; i < count; ++i) {
      const int j = i & 3;
      const uint64_t bd = smem_desc(sb + j * 2 * (N / 8 * 128), N / 8 * 128, 128);
      if (ts) {
        asm volatile(
            "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
            "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n\t}" ::"r"(tmem),
            "r"(tmem + 256 + j * 8), "l"(bd), "r"(idesc), "r"(uint32_t(i > 0))
            : "memory");
      } else {
        const uint64_t ad = smem_desc(sa + j * 4096, 2048, 128);
        asm volatile(
            "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
            "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem),
            "l"(ad), "l"(bd), "r"(idesc), "r"(uint32_t(i > 0))
            : "memory");
      }
    }
    const long long t1 = clock64();
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&bar))
                 : "memory");
    asm volatile(
        "{\n\t.reg .pred p;\n\tW:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n\t@!p bra W;\n\t}" ::"r"(su32(&bar))
        : "memory");
    const long long t2 = clock64();
    out[0] = t1 - t0;
    out[1] = t2 - t0;
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
  }
}

int main() {
  long long* d;
  cudaMalloc(&d, 16);
  cudaFuncSetAttribute(rate, cudaFuncAttributeMaxDynamicSharedMemorySize, 96 * 1024);
  for (int ts = 0; ts < 2; ++ts)
    for (int N : {64, 128, 256}) {
      const int count = 1024;
      long long h[2] = {0, 0};
      for (int rep = 0; rep < 2; ++rep) rate<<<1, 128, 96 * 1024>>>(N, ts, count, d);
      cudaError_t e = cudaDeviceSynchronize();
      cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
      const double flops = 2.0 * 128 * N * 8 * count;
      printf("%s N=%3d: issue %.1f cyc/MMA, complete %.1f cyc/MMA (%.0f flop/cyc/SM) %s\n", ts ? "ts" : "ss", N,
             double(h[0]) / count, double(h[1]) / count, flops / double(h[1]), cudaGetErrorString(e));
    }
  return 0;
}
