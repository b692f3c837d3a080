// Probe: row-gather throughput into shared memory per SM (the fused
// kernel's producer pattern). Rows of 512 B at random indices of an
// L2-resident table are copied into a 2-stage ring by `warps` warps with
// 16-byte cp.async (LDGSTS), 4 rows of 512 B per ... ; reports bytes per
// SM cycle. Build: nvcc -gencode arch=compute_100a,code=sm_100a gather_probe.cu
#include <cstdint>
#include <cstdio>
#include <vector>

__device__ __forceinline__ uint32_t su32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// mode 0: cp.async 16 B per lane (row = 32 lanes x 16 B)
// mode 1: plain 16 B loads into registers, then st.shared (register staging)
// mode 2: cp.async 16 B, but each warp handles 2 rows per instruction (lanes 0-15 row a)
__global__ void gather(const float4* __restrict__ table, const uint32_t* __restrict__ idx, int rows_per_chunk,
                       int chunks, int warps, int mode, long long* out) {
  extern __shared__ __align__(16) unsigned char sm[];
  __shared__ uint32_t sidx[64 * 128];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  for (int i = tid; i < chunks * rows_per_chunk; i += blockDim.x)
    sidx[i] = idx[uint64_t(blockIdx.x) * chunks * rows_per_chunk + i];
  __syncthreads();
  const long long t0 = clock64();
  if (warp < warps) {
    for (int c = 0; c < chunks; ++c) {
      const uint32_t* ix = sidx + c * rows_per_chunk;
      unsigned char* dst = sm + (c & 1) * rows_per_chunk * 512;
      if (mode == 2) {  // one 512-byte cp.async.bulk per row, lane-parallel, completion on an mbarrier
        __shared__ __align__(8) uint64_t bar[16];
        if (c == 0 && lane == 0) {
          asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar[warp])));
        }
        __syncwarp();
        int mine = 0;
        for (int r = warp + lane * warps; r < rows_per_chunk; r += 32 * warps) ++mine;
        const int total = __reduce_add_sync(0xffffffffu, mine);
        if (lane == 0)
          asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&bar[warp])), "r"(total * 512)
                       : "memory");
        __syncwarp();
        for (int r = warp + lane * warps; r < rows_per_chunk; r += 32 * warps)
          asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], 512, [%2];" ::"r"(
                           su32(dst + r * 512)),
                       "l"(table + uint64_t(ix[r]) * 32), "r"(su32(&bar[warp]))
                       : "memory");
        asm volatile(
            "{\n\t.reg .pred p;\n\tW:\n\t"
            "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@!p bra W;\n\t}" ::"r"(su32(&bar[warp])),
            "r"(c & 1)
            : "memory");
      } else if (mode == 1) {
        for (int r = warp; r < rows_per_chunk; r += warps) {
          const float4 v = __ldg(table + uint64_t(ix[r]) * 32 + lane);
          *reinterpret_cast<float4*>(dst + r * 512 + lane * 16) = v;
        }
      } else {
        for (int r = warp; r < rows_per_chunk; r += warps) {
          const float4* src = table + uint64_t(ix[r]) * 32 + lane;
          asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(su32(dst + r * 512 + lane * 16)), "l"(src)
                       : "memory");
        }
        asm volatile("cp.async.commit_group;" ::: "memory");
        asm volatile("cp.async.wait_group 1;" ::: "memory");
      }
    }
    asm volatile("cp.async.wait_all;" ::: "memory");
  }
  __syncthreads();
  if (tid == 0) out[blockIdx.x] = clock64() - t0;
}

int main() {
  const int V = 9727, rows_per_chunk = 64, chunks = 128, ctas = 148;
  float4* table;
  uint32_t* idx;
  long long* out;
  cudaMalloc(&table, size_t(V) * 512);
  cudaMemset(table, 0, size_t(V) * 512);
  std::vector<uint32_t> h(size_t(ctas) * chunks * rows_per_chunk);
  uint64_t st = 88172645463325252ull;
  for (auto& x : h) {
    st ^= st << 13; st ^= st >> 7; st ^= st << 17;
    x = uint32_t(st % V);
  }
  cudaMalloc(&idx, h.size() * 4);
  cudaMemcpy(idx, h.data(), h.size() * 4, cudaMemcpyHostToDevice);
  cudaMalloc(&out, ctas * 8);
  cudaFuncSetAttribute(gather, cudaFuncAttributeMaxDynamicSharedMemorySize, 2 * rows_per_chunk * 512);
  cudaFuncSetAttribute(gather, cudaFuncAttributeMaxDynamicSharedMemorySize, 2 * rows_per_chunk * 512);
  for (int mode : {0, 2})
    for (int warps : {1, 2, 3, 4, 6, 8, 12, 16}) {
      for (int rep = 0; rep < 3; ++rep)
        gather<<<ctas, 512, 2 * rows_per_chunk * 512>>>(table, idx, rows_per_chunk, chunks, warps, mode, out);
      cudaError_t e = cudaDeviceSynchronize();
      std::vector<long long> cyc(ctas);
      cudaMemcpy(cyc.data(), out, ctas * 8, cudaMemcpyDeviceToHost);
      double mean = 0;
      for (auto c : cyc) mean += double(c) / ctas;
      const double bytes = double(chunks) * rows_per_chunk * 512;
      printf("%s warps=%2d: %.1f B/cycle/SM (%.0f cycles) %s\n", mode == 2 ? "bulk 512 B  " : mode ? "ld+st.shared" : "cp.async16  ", warps,
             bytes / mean, mean, cudaGetErrorString(e));
    }
  return 0;
}
