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

__global__ void rate(int N, int ts, int count, long long* out, int pattern) {
  extern __shared__ __align__(1024) unsigned char sm[];
  __shared__ uint32_t tslot;
  __shared__ __align__(8) uint64_t bar, bar2;
  const int tid = threadIdx.x, warp = tid >> 5;
  for (int i = tid; i < 64 * 1024 / 4; i += blockDim.x) reinterpret_cast<float*>(sm)[i] = 0.5f;
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar)));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar2)));
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
    unsigned long long g0, g1;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g0));
    const long long t0 = clock64();
    if (pattern == 22 || pattern == 23) {  // unrolled TS (A in TMEM), fused-kernel term order
      uint64_t bds[8];
#pragma unroll
      for (int q = 0; q < 8; ++q) bds[q] = smem_desc(sb + (q & 1) * 16384 + (q >> 1) * 2 * (N / 8 * 128), N / 8 * 128, 128);
      for (int i = 0; i < count; i += 12) {
#pragma unroll
        for (int q = 0; q < 12; ++q) {
          const int ks = q / 3, term = q % 3;
          const uint32_t acol = 256 + ks * 8 + (term == 2 ? 32 : 0);
          const uint64_t bd = bds[ks * 2 + (term == 1 ? 1 : 0)];
          const uint32_t dcol = pattern == 23 ? ((i / 12) & 1) * 128 : 0;
          asm volatile(
              "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
              "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n\t}" ::"r"(tmem + dcol),
              "r"(tmem + acol), "l"(bd), "r"(idesc), "r"(1u)
              : "memory");
        }
      }
    } else if (pattern == 24) {  // unrolled SS, fused-kernel term order (A hi/lo in smem)
      uint64_t bds[8], ads[8];
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        bds[q] = smem_desc(sb + (q & 1) * 16384 + (q >> 1) * 2 * (N / 8 * 128), N / 8 * 128, 128);
        ads[q] = smem_desc(sa + (q & 1) * 16384 + (q >> 1) * 4096, 2048, 128);
      }
      for (int i = 0; i < count; i += 12) {
#pragma unroll
        for (int q = 0; q < 12; ++q) {
          const int ks = q / 3, term = q % 3;
          asm volatile(
              "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
              "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem),
              "l"(ads[ks * 2 + (term == 2 ? 1 : 0)]), "l"(bds[ks * 2 + (term == 1 ? 1 : 0)]), "r"(idesc), "r"(1u)
              : "memory");
        }
      }
    } else
    if (pattern == 20 || pattern == 21) {  // unrolled: 12 MMAs per iteration, descriptors precomputed
      uint64_t bds[4], ads[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        bds[q] = smem_desc(sb + q * 2 * (N / 8 * 128), N / 8 * 128, 128);
        ads[q] = smem_desc(sa + q * 4096, 2048, 128);
      }
      for (int i = 0; i < count; i += 12) {
#pragma unroll
        for (int q = 0; q < 12; ++q) {
          const uint32_t dcol = pattern == 21 ? (q / 6) * 128 : 0;
          asm volatile(
              "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
              "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem + dcol),
              "l"(ads[q & 3]), "l"(bds[(q >> 2) & 3]), "r"(idesc), "r"(1u)
              : "memory");
        }
      }
    } else
    for (int i = 0; i < count; ++i) {
      const int j = i & 3;
      uint64_t bd = smem_desc(sb + j * 2 * (N / 8 * 128), N / 8 * 128, 128);
      if (pattern >= 10) {  // round-robin over (pattern - 10) independent accumulators, SS, N=128
        const int nb = pattern - 10;
        const int b = i % nb;
        const uint64_t ad = smem_desc(sa + j * 4096, 2048, 128);
        asm volatile(
            "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
            "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem + b * 128),
            "l"(ad), "l"(bd), "r"(idesc), "r"(uint32_t(i >= nb))
            : "memory");
        continue;
      }
      if (pattern) {  // fused-kernel pattern: k-step = i/3, (a_hi b_hi, a_hi b_lo, a_lo b_hi)
        const int kstep = (i / 3) & 3, term = i % 3;
        const uint32_t blo = term == 1 ? 16384 : 0;
        bd = smem_desc(sb + blo + kstep * 2 * (N / 8 * 128), N / 8 * 128, 128);
        const uint32_t acol = 128 + ((i / 12) & 1) * 64 + kstep * 8 + (term == 2 ? 32 : 0);
        const uint32_t dcol = 0;
        asm volatile(
            "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
            "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n\t}" ::"r"(tmem + dcol),
            "r"(tmem + acol), "l"(bd), "r"(idesc), "r"(uint32_t(i % 6 > 0))
            : "memory");
        if (pattern == 2 && i % 12 == 11)
          asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                           su32(&bar2)) : "memory");
        continue;
      }
      if (ts == 2) {  // kind::f16 (bf16 in, f32 acc), K = 16, A in TMEM (2 bf16 per column)
        const uint32_t id16 = (1u << 4) | (1u << 7) | (1u << 10) | (uint32_t(N >> 3) << 17) | (uint32_t(128 >> 4) << 24);
        asm volatile(
            "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
            "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(tmem),
            "r"(tmem + 128 + j * 8), "l"(bd), "r"(id16), "r"(uint32_t(i > 0))
            : "memory");
      } else if (ts) {
        asm volatile(
            "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
            "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n\t}" ::"r"(tmem),
            "r"(tmem + 128 + j * 8), "l"(bd), "r"(idesc), "r"(uint32_t(i > 0))
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
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g1));
    out[0] = t1 - t0;
    out[1] = t2 - t0;
    out[2] = (long long)(g1 - g0);
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
  cudaMalloc(&d, 32);
  cudaFuncSetAttribute(rate, cudaFuncAttributeMaxDynamicSharedMemorySize, 96 * 1024);
  for (int w = 0; w < 200; ++w) rate<<<148, 128, 96 * 1024>>>(128, 0, 4096, d, 0);  // warm clocks
  cudaDeviceSynchronize();
  cudaFuncSetAttribute(rate, cudaFuncAttributeMaxDynamicSharedMemorySize, 96 * 1024);
  if (0) for (int ts = 0; ts < 2; ++ts)
    for (int N : {64, 128, 256}) {
      const int count = 1024;
      long long h[2] = {0, 0};
      for (int rep = 0; rep < 2; ++rep) rate<<<1, 128, 96 * 1024>>>(N, ts, count, d, 0);
      cudaError_t e = cudaDeviceSynchronize();
      cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
      const double flops = 2.0 * 128 * N * 8 * count;
      printf("%s N=%3d: issue %.1f cyc/MMA, complete %.1f cyc/MMA (%.0f flop/cyc/SM) %s\n", ts ? "ts" : "ss", N,
             double(h[0]) / count, double(h[1]) / count, flops / double(h[1]), cudaGetErrorString(e));
    }
  if (0) for (int N : {64, 128, 256}) {
    const int count = 1024;
    long long h[2] = {0, 0};
    for (int rep = 0; rep < 2; ++rep) rate<<<1, 128, 96 * 1024>>>(N, 2, count, d, 0);
    cudaError_t e = cudaDeviceSynchronize();
    cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
    const double flops = 2.0 * 128 * N * 16 * count;
    printf("bf16 ts N=%3d K=16: issue %.1f, complete %.1f cyc/MMA (%.0f flop/cyc/SM) %s\n", N, double(h[0]) / count,
           double(h[1]) / count, flops / double(h[1]), cudaGetErrorString(e));
  }
  if (0) for (int pattern = 1; pattern <= 2; ++pattern) {
    const int count = 1200;
    long long h[2] = {0, 0};
    for (int rep = 0; rep < 2; ++rep) rate<<<1, 128, 96 * 1024>>>(128, 1, count, d, pattern);
    cudaError_t e = cudaDeviceSynchronize();
    cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
    printf("fused pattern %d (ts, N=128, 3 hi/lo MMAs per k-step, D alternating per 6%s): issue %.1f, complete %.1f cyc/MMA %s\n",
           pattern, pattern == 2 ? ", commit per 12" : "", double(h[0]) / count, double(h[1]) / count, cudaGetErrorString(e));
  }
  for (int pat : {20, 22, 23, 24}) {
    const int count = 4800;
    long long h[3] = {0, 0, 0};
    for (int rep = 0; rep < 3; ++rep) rate<<<1, 128, 96 * 1024>>>(128, 0, count, d, pat);
    cudaError_t e = cudaDeviceSynchronize();
    cudaMemcpy(h, d, 24, cudaMemcpyDeviceToHost);
    printf("N=128 unrolled x12, %s: %.1f cyc/MMA, %.1f ns/MMA %s\n",
           pat == 20 ? "ss simple" : pat == 22 ? "ts fused order" : pat == 23 ? "ts fused order, D alternating" : "ss fused order",
           double(h[1]) / count, double(h[2]) / count, cudaGetErrorString(e));
  }
  for (int ts = 0; ts < 3; ++ts) {
    const int count = 4096;
    long long h[3] = {0, 0, 0};
    for (int rep = 0; rep < 3; ++rep) rate<<<1, 128, 96 * 1024>>>(128, ts, count, d, 0);
    cudaError_t e = cudaDeviceSynchronize();
    cudaMemcpy(h, d, 24, cudaMemcpyDeviceToHost);
    printf("%s N=128 single chain: %.1f cyc/MMA, %.1f ns/MMA %s\n", ts == 2 ? "bf16 ts K16" : ts ? "tf32 ts" : "tf32 ss",
           double(h[1]) / count, double(h[2]) / count, cudaGetErrorString(e));
  }
  {
    const int count = 4096;
    long long h[3] = {0, 0, 0};
    rate<<<148, 128, 96 * 1024>>>(128, 0, count, d, 12);
    rate<<<148, 128, 96 * 1024>>>(128, 0, count, d, 12);
    cudaError_t e = cudaDeviceSynchronize();
    cudaMemcpy(h, d, 24, cudaMemcpyDeviceToHost);
    printf("148 CTAs, 2 accumulators: %.1f cyc/MMA, %.1f ns/MMA %s\n", double(h[1]) / count, double(h[2]) / count,
           cudaGetErrorString(e));
  }
  return 0;
}
