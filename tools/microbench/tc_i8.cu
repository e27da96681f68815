// tc_i8.cu -- tcgen05 kind::i8 feasibility check on sm_100a:
//   (1) correctness of hand-built smem/instruction descriptors (K-major,
//       no swizzle) for D[128 x N] (s32, TMEM) = A[128 x K] (u8/s8) * B[N x K]^T (s8);
//   (2) sustained MMA throughput from shared memory (N = 256, M = 128).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 tc_i8.cu -o tc_i8
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <algorithm>
#include <vector>

#define CK(x)                                                                      \
  do {                                                                             \
    cudaError_t e_ = (x);                                                          \
    if (e_ != cudaSuccess) {                                                       \
      printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e_), __FILE__, __LINE__); \
      exit(1);                                                                     \
    }                                                                              \
  } while (0)

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

// K-major, SWIZZLE_NONE canonical layout: core matrix = 8 rows x 16 B
// contiguous (128 B); LBO = byte step between the two 16-B K halves of one
// MMA K-step; SBO = byte step between 8-row groups.
__device__ __forceinline__ uint64_t smem_desc(uint32_t addr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((addr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;  // version (sm_100)
  return d;                // base_offset 0, lbo_mode 0, layout SWIZZLE_NONE (0)
}

// instruction descriptor, kind::i8: c = s32, a/b signedness, K-major both
__host__ __device__ constexpr uint32_t idesc_i8(int M, int N, bool a_signed, bool b_signed) {
  return (2u << 4) | ((a_signed ? 1u : 0u) << 7) | ((b_signed ? 1u : 0u) << 10) | ((uint32_t)(N >> 3) << 17) |
         ((uint32_t)(M >> 4) << 24);
}

__device__ __forceinline__ void mma_i8(uint32_t tmem_d, uint64_t da, uint64_t db, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem_d),
      "l"(da), "l"(db), "r"(idesc), "r"(acc));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
  asm volatile(
      "{\n\t.reg .pred done;\n\t"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 done, [%0], %1;\n\t"
      "@!done bra WAIT_%=;\n\t}\n" ::"r"(smem_u32(bar)),
      "r"(phase)
      : "memory");
}

// byte offset of element (row, k) in a K-major no-swizzle tile with `rows`
// rows: [k/16][row/8][row%8][k%16]
__device__ __forceinline__ int kmaj_off(int row, int k, int rows) {
  return ((k >> 4) * (rows >> 3) + (row >> 3)) * 128 + (row & 7) * 16 + (k & 15);
}

template <int N, int K>
__global__ void __launch_bounds__(128, 1) gemm_check(const uint8_t* A, const int8_t* B, int32_t* D, int a_signed) {
  constexpr int M = 128;
  __shared__ __align__(1024) uint8_t sA[M * K];
  __shared__ __align__(1024) uint8_t sB[N * K];
  __shared__ uint64_t bar;
  __shared__ uint32_t tmem_base;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  for (int i = tid; i < M * K; i += 128) sA[kmaj_off(i / K, i % K, M)] = A[i];
  for (int i = tid; i < N * K; i += 128) sB[kmaj_off(i / K, i % K, N)] = (uint8_t)B[i];
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tmem_base)),
                 "n"(N < 32 ? 32 : N));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) {
    mbar_init(&bar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = tmem_base;
  if (tid == 0) {
    const uint32_t idesc = idesc_i8(M, N, a_signed != 0, true);
    for (int ks = 0; ks < K / 32; ++ks) {
      uint64_t da = smem_desc(smem_u32(sA) + ks * 2 * (M / 8) * 128, (M / 8) * 128, 128);
      uint64_t db = smem_desc(smem_u32(sB) + ks * 2 * (N / 8) * 128, (N / 8) * 128, 128);
      mma_i8(tmem, da, db, idesc, ks > 0);
    }
    mma_commit(&bar);
  }
  mbar_wait(&bar, 0);
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  // warp w reads TMEM lanes [32w, 32w+32): row = 32w + lane
  for (int c0 = 0; c0 < N; c0 += 8) {
    uint32_t v[8];
    const uint32_t addr = tmem + ((uint32_t)(warp * 32) << 16) + c0;
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7])
                 : "r"(addr));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
    for (int j = 0; j < 8; ++j) D[(warp * 32 + lane) * N + c0 + j] = (int32_t)v[j];
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(N < 32 ? 32 : N));
}

// throughput: each CTA issues `iters` x (K/32) MMAs of 128 x N x 32 on resident tiles
template <int N, int K>
__global__ void __launch_bounds__(128, 1) gemm_rate(int iters, int32_t* sink) {
  constexpr int M = 128;
  extern __shared__ __align__(1024) uint8_t dyn[];
  uint8_t* sA = dyn;
  uint8_t* sB = dyn + M * K;
  __shared__ uint64_t bar;
  __shared__ uint32_t tmem_base;
  const int tid = threadIdx.x, warp = tid >> 5;
  for (int i = tid; i < (M + N) * K; i += 128) dyn[i] = (uint8_t)(i * 7 + 3);
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tmem_base)),
                 "n"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) {
    mbar_init(&bar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = tmem_base;
  if (tid == 0) {
    const uint32_t idesc = idesc_i8(M, N, false, true);
    for (int it = 0; it < iters; ++it)
      for (int ks = 0; ks < K / 32; ++ks) {
        uint64_t da = smem_desc(smem_u32(sA) + ks * 2 * (M / 8) * 128, (M / 8) * 128, 128);
        uint64_t db = smem_desc(smem_u32(sB) + ks * 2 * (N / 8) * 128, (N / 8) * 128, 128);
        mma_i8(tmem + (it & 1) * 256, da, db, idesc, 1);
      }
    mma_commit(&bar);
  }
  mbar_wait(&bar, 0);
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  uint32_t v;
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x1.b32 {%0}, [%1];" : "=r"(v) : "r"(tmem + ((uint32_t)(warp * 32) << 16)));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
  if (v == 0x12345) sink[0] = v;
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(512));
}

template <int N, int K>
bool check(int a_signed) {
  constexpr int M = 128;
  std::vector<uint8_t> A(M * K);
  std::vector<int8_t> B(N * K);
  srand(1234 + N + K + a_signed);
  for (auto& a : A) a = (uint8_t)(rand() & 255);
  for (auto& b : B) b = (int8_t)(rand() & 255);
  uint8_t* dA;
  int8_t* dB;
  int32_t* dD;
  CK(cudaMalloc(&dA, A.size()));
  CK(cudaMalloc(&dB, B.size()));
  CK(cudaMalloc(&dD, M * N * 4));
  CK(cudaMemcpy(dA, A.data(), A.size(), cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dB, B.data(), B.size(), cudaMemcpyHostToDevice));
  gemm_check<N, K><<<1, 128>>>(dA, dB, dD, a_signed);
  CK(cudaGetLastError());
  CK(cudaDeviceSynchronize());
  std::vector<int32_t> D(M * N);
  CK(cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost));
  int bad = 0;
  for (int i = 0; i < M; ++i)
    for (int j = 0; j < N; ++j) {
      int64_t s = 0;
      for (int k = 0; k < K; ++k) {
        int av = a_signed ? (int)(int8_t)A[i * K + k] : (int)A[i * K + k];
        s += (int64_t)av * B[j * K + k];
      }
      if (s != D[i * N + j] && bad++ < 5) printf("  mismatch (%d,%d): got %d want %lld\n", i, j, D[i * N + j], (long long)s);
    }
  printf("check N=%d K=%d a_%s: %s\n", N, K, a_signed ? "s8" : "u8", bad ? "FAIL" : "ok");
  cudaFree(dA);
  cudaFree(dB);
  cudaFree(dD);
  return bad == 0;
}

template <int N, int K>
void rate(int sms) {
  constexpr int M = 128;
  const int smem = (M + N) * K;
  CK(cudaFuncSetAttribute(gemm_rate<N, K>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  int32_t* sink;
  CK(cudaMalloc(&sink, 4));
  const int iters = 4000;
  gemm_rate<N, K><<<sms, 128, smem>>>(10, sink);
  CK(cudaDeviceSynchronize());
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaEventRecord(a);
  gemm_rate<N, K><<<sms, 128, smem>>>(iters, sink);
  cudaEventRecord(b);
  CK(cudaEventSynchronize(b));
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  const double ops = 2.0 * M * N * K * (double)iters * sms;
  printf("rate M=128 N=%d K/iter=%d: %.3f ms  %.1f TOPS (int8)\n", N, K, ms, ops / ms / 1e9);
  cudaFree(sink);
}


// overlap test: warp 0 issues int8 MMAs (as gemm_rate); warps 1..nw run
// independent DFMA chains for `fiters` iterations
template <int N, int K>
__global__ void __launch_bounds__(32 * 17, 1) mixed(int iters, int fiters, int nw, int32_t* sink, double* dsink) {
  constexpr int M = 128;
  extern __shared__ __align__(1024) uint8_t dyn[];
  uint8_t* sA = dyn;
  uint8_t* sB = dyn + M * K;
  __shared__ uint64_t bar;
  __shared__ uint32_t tmem_base;
  const int tid = threadIdx.x, warp = tid >> 5;
  for (int i = tid; i < (M + N) * K; i += blockDim.x) dyn[i] = (uint8_t)(i * 7 + 3);
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tmem_base)),
                 "n"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) {
    mbar_init(&bar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = tmem_base;
  if (warp == 0) {
    if (tid == 0) {
      const uint32_t idesc = idesc_i8(M, N, false, true);
      for (int it = 0; it < iters; ++it)
        for (int ks = 0; ks < K / 32; ++ks) {
          uint64_t da = smem_desc(smem_u32(sA) + ks * 2 * (M / 8) * 128, (M / 8) * 128, 128);
          uint64_t db = smem_desc(smem_u32(sB) + ks * 2 * (N / 8) * 128, (N / 8) * 128, 128);
          mma_i8(tmem + (it & 1) * 256, da, db, idesc, 1);
        }
      mma_commit(&bar);
    }
    mbar_wait(&bar, 0);
  } else if (warp <= nw) {
    double a[8];
    for (int j = 0; j < 8; ++j) a[j] = 1.0 + 1e-9 * (tid + j);
    const double b = 0.999999999, c = 1e-12;
    for (int i = 0; i < fiters; ++i)
#pragma unroll
      for (int j = 0; j < 8; ++j) a[j] = fma(a[j], b, c);
    double s = 0;
    for (int j = 0; j < 8; ++j) s += a[j];
    if (s == 12345.0) dsink[0] = s;
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(512));
  if (tid == 0 && iters < 0) sink[0] = 1;
}

void overlap(int sms) {
  constexpr int N = 256, K = 128, M = 128;
  const int smem = (M + N) * K;
  CK(cudaFuncSetAttribute(mixed<N, K>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  int32_t* sink;
  double* dsink;
  CK(cudaMalloc(&sink, 4));
  CK(cudaMalloc(&dsink, 8));
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  auto run = [&](int iters, int fiters, int nw) {
    mixed<N, K><<<sms, 32 * 17, smem>>>(iters, fiters, nw, sink, dsink);
    CK(cudaDeviceSynchronize());
    cudaEventRecord(a);
    mixed<N, K><<<sms, 32 * 17, smem>>>(iters, fiters, nw, sink, dsink);
    cudaEventRecord(b);
    CK(cudaEventSynchronize(b));
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    return (double)ms;
  };
  const int iters = 3000, fiters = 20000, nw = 16;
  const double t_mma = run(iters, 0, 0);
  const double t_fma = run(0, fiters, nw);
  const double t_both = run(iters, fiters, nw);
  const double iops = 2.0 * M * N * K * (double)iters * sms;
  const double flops = 2.0 * 8 * (double)fiters * 32 * nw * sms;
  printf("overlap: int8 MMA alone %.3f ms (%.0f TOPS); DFMA alone %.3f ms (%.1f TF/s); both %.3f ms\n", t_mma,
         iops / t_mma / 1e9, t_fma, flops / t_fma / 1e9, t_both);
  printf("  -> both/(mma+fma) = %.2f (1.0 = fully serialised, %.2f = perfect overlap)\n", t_both / (t_mma + t_fma),
         std::max(t_mma, t_fma) / (t_mma + t_fma));
}

int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  bool ok = true;
  ok &= check<64, 64>(0);
  ok &= check<64, 64>(1);
  ok &= check<32, 128>(0);
  ok &= check<256, 32>(0);
  ok &= check<16, 64>(1);
  rate<256, 128>(sms);
  rate<128, 128>(sms);
  rate<64, 128>(sms);
  rate<32, 128>(sms);
  overlap(sms);
  printf(ok ? "ALL OK\n" : "FAILURES\n");
  return ok ? 0 : 1;
}
