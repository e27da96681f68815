// tma_copy_size.cu -- cp.async.bulk global->shared throughput against the size of one copy.
// Every CTA stages `per_cta` bytes with copies of `csz` bytes (one mbarrier, one issuing thread),
// the grid covers `total` bytes of a buffer larger than L2.  Question: is the butterfly-apply stage
// kernel (one bulk copy per stored block column: 256-512 B in config 2) bound by the per-copy cost?
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o tma_copy_size tma_copy_size.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__global__ void __launch_bounds__(64) stage_copy(const char* __restrict__ src, int per_cta, int csz, unsigned long long* sink) {
  extern __shared__ __align__(128) unsigned char smem[];
  const uint32_t bar = (uint32_t)__cvta_generic_to_shared(smem);
  const uint32_t dst0 = bar + 128;
  const char* s = src + (size_t)blockIdx.x * per_cta;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bar));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("mbarrier.arrive.expect_tx.release.cta.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"((uint32_t)per_cta) : "memory");
  }
  __syncthreads();
  const int n = per_cta / csz;
  for (int c = threadIdx.x; c < n; c += blockDim.x)
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst0 + c * csz),
                 "l"(s + (size_t)c * csz), "r"((uint32_t)csz), "r"(bar) : "memory");
  asm volatile(
      "{\n\t.reg .pred done;\n\tW_%=:\n\tmbarrier.try_wait.parity.acquire.cta.shared::cta.b64 done, [%0], 0;\n\t@!done bra W_%=;\n\t}\n" ::"r"(bar)
      : "memory");
  if (threadIdx.x == 0 && smem[128 + (blockIdx.x & 255)] == 0x5a && sink) atomicAdd(sink, 1ull);
}

int main() {
  const size_t total = 1ull << 30;  // 1 GB > L2
  char* buf;
  cudaMalloc(&buf, total);
  cudaMemset(buf, 1, total);
  cudaFuncSetAttribute(stage_copy, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const int per_ctas[] = {8192, 16384, 65536};
  const int cszs[] = {128, 256, 512, 1024, 2048, 4096, 8192, 16384};
  for (int issuers : {1, 32}) {
    for (int pc : per_ctas) {
      for (int csz : cszs) {
        if (csz > pc) continue;
        const int grid = (int)(total / pc);
        stage_copy<<<grid, issuers, pc + 128>>>(buf, pc, csz, nullptr);
        cudaEventRecord(a);
        stage_copy<<<grid, issuers, pc + 128>>>(buf, pc, csz, nullptr);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        printf("issuing threads %2d  bytes/CTA %6d  copy %6d B  %8.1f GB/s  (%s)\n", issuers, pc, csz, total / ms / 1e6,
               cudaGetErrorString(cudaGetLastError()));
      }
    }
  }
  return 0;
}
