// Probe: tcgen05.mma kind::i8 issue rate on one SM per CTA (148 CTAs):
// cycles per MMA for A in TMEM (ts) or shared memory (ss), N digits, the
// number of distinct accumulators the MMAs rotate over, and a commit+wait
// every `sync` MMAs (0 = none). Values are garbage (uninitialised
// operands); only the timing matters. Build: nvcc -gencode
// arch=compute_100a,code=sm_100a i8_rate_probe.cu
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

__global__ void probe(long long* out, int ts, int N, int nacc, int total, int sync, int kind) {
  __shared__ __align__(1024) unsigned char sb[40 * 1024];
  __shared__ uint32_t tslot;
  __shared__ __align__(8) uint64_t bar;
  const int tid = threadIdx.x, warp = tid >> 5;
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
    const uint32_t idesc = (kind == 0 ? (2u << 4) | (1u << 10) : (1u << 4)) | (uint32_t(N >> 3) << 17) |
                           (uint32_t(128 >> 4) << 24);
    uint32_t phase = 0;
    const long long t0 = clock64();
    for (int j = 0; j < total; ++j) {
      const int a = j % nacc;
      const uint32_t d = tmem + a * N;  // accumulators in columns [0, nacc N)
      const uint64_t bd = smem_desc(su32(sb) + (j % 8) * 1024, (N / 8) * 128, 128);
      if (ts) {
        if (kind == 0)
          asm volatile(
              "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
              "tcgen05.mma.cta_group::1.kind::i8 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d),
              "r"(tmem + 256 + (j % 32) * 8), "l"(bd), "r"(idesc), "r"(1u)
              : "memory");
        else if (kind == 1)
          asm volatile(
              "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
              "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d),
              "r"(tmem + 256 + (j % 32) * 8), "l"(bd), "r"(idesc), "r"(1u)
              : "memory");
        else
          asm volatile(
              "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
              "tcgen05.mma.cta_group::1.kind::f8f6f4 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d),
              "r"(tmem + 256 + (j % 32) * 8), "l"(bd), "r"(idesc), "r"(1u)
              : "memory");
      } else {
        const uint64_t ad = smem_desc(su32(sb) + 8192 + (j % 4) * 4096, 16 * 128, 128);
        asm volatile(
            "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
            "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
            "l"(ad), "l"(bd), "r"(idesc), "r"(1u)
            : "memory");
      }
      if (sync && (j + 1) % sync == 0) {
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&bar))
                     : "memory");
        asm volatile(
            "{\n\t.reg .pred p;\n\tW1:\n\t"
            "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@!p bra W1;\n\t}" ::"r"(su32(&bar)),
            "r"(phase)
            : "memory");
        phase ^= 1;
      }
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&bar))
                 : "memory");
    asm volatile(
        "{\n\t.reg .pred p;\n\tW2:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@!p bra W2;\n\t}" ::"r"(su32(&bar)),
        "r"(phase)
        : "memory");
    const long long t1 = clock64();
    out[blockIdx.x] = t1 - t0;
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
  cudaMalloc(&d, 148 * 8);
  long long h[148];
  struct C { int ts, N, nacc, sync, kind; };
  const C cs[] = {{1, 16, 8, 0, 0}, {1, 256, 1, 0, 0}, {0, 16, 8, 0, 0}, {1, 16, 8, 0, 1}, {1, 64, 4, 0, 1},
                  {1, 256, 1, 0, 1}, {0, 16, 8, 0, 1}, {0, 256, 1, 0, 1}, {1, 16, 8, 0, 2}, {1, 64, 4, 0, 2},
                  {1, 256, 1, 0, 2}, {0, 16, 8, 0, 2}, {0, 256, 1, 0, 2}};
  const int total = 8192;
  for (const C& c : cs) {
    probe<<<148, 128>>>(d, c.ts, c.N, c.nacc, total, c.sync, c.kind);
    cudaError_t e = cudaDeviceSynchronize();
    cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
    long long mx = 0;
    for (int i = 0; i < 148; ++i) mx = h[i] > mx ? h[i] : mx;
    printf("%s %s N=%3d nacc=%2d sync=%2d: %.1f cycles/MMA (%s)\n", c.kind == 0 ? "i8 " : c.kind == 1 ? "f16" : "f8 ",
           c.ts ? "ts" : "ss", c.N, c.nacc, c.sync,
           double(mx) / total, cudaGetErrorString(e));
  }
  return 0;
}
