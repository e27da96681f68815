// tc_interf.cu -- what slows K2's MMAs down inside the kernel: one K2 stage's
// tcgen05 kind::i8 MMA schedule (M = 128, K = 32, NCB = 32; the round-2
// 20-MMA 7-diagonal schedule or the 18-MMA one with free windows) issued by
// warp 0, while warps 1..15 do one stage's worth of the evaluation's other
// work, paced per stage (a stage ends when both the MMAs and the work are
// done):
//   F: 4096 warp-level DFMAs (the ~32 FP64 instructions x 4096 entries of a stage)
//   L: 128 warp-level random LDS.128 gathers from a 32 KB table (the sin/cos table)
//   S: 48 KB of 8-byte shared stores (the A-slice images)
// Prints cycles per stage for each combination.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 --expt-relaxed-constexpr tc_interf.cu -o tc_interf
#include <cstdint>
#include <cstdio>
#include <cstdlib>

#define CK(x)                                                                                    \
  do {                                                                                           \
    cudaError_t e_ = (x);                                                                        \
    if (e_ != cudaSuccess) {                                                                     \
      printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e_), __FILE__, __LINE__);           \
      exit(1);                                                                                   \
    }                                                                                            \
  } while (0)

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t smem_desc(uint32_t addr, uint32_t lbo, uint32_t sbo) {
  return (uint64_t)((addr >> 4) & 0x3FFF) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) | ((uint64_t)1 << 46);
}
__host__ __device__ constexpr uint32_t idesc_i8(int M, int N, bool a_signed, bool b_signed) {
  return (2u << 4) | ((a_signed ? 1u : 0u) << 7) | ((b_signed ? 1u : 0u) << 10) | ((uint32_t)(N >> 3) << 17) |
         ((uint32_t)(M >> 4) << 24);
}
__device__ __forceinline__ void mma_ss(uint32_t d, uint64_t da, uint64_t db, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(d),
      "l"(da), "l"(db), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ void mma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
  asm volatile(
      "{\n\t.reg .pred done;\n\tWAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 done, [%0], %1;\n\t"
      "@!done bra WAIT_%=;\n\t}\n" ::"r"(smem_u32(bar)),
      "r"(phase)
      : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

constexpr int NSL = 6, BN2 = 64, BM = 128, KS = 32;
constexpr int ASLICE = BM * KS, APLANE = NSL * ASLICE, BROWS = NSL * BN2, BOPER = BROWS * KS;
struct Sched {
  int h[64], p[64], jlo[64], nb[64];
  int n;
};
constexpr Sched make_sched(int e0, bool split) {
  Sched s{};
  s.n = 0;
  const int T = NSL - 1, D = 2 * NSL - 1 - e0;
  for (int h = 0; h < 2; ++h) {
    if (split) {
      for (int j = 1; j <= D - 1; j += 4) { s.h[s.n] = h; s.p[s.n] = T; s.jlo[s.n] = j; s.nb[s.n] = (D - j) < 4 ? D - j : 4; ++s.n; }
      s.h[s.n] = h; s.p[s.n] = T - 1; s.jlo[s.n] = 0; s.nb[s.n] = 1; ++s.n;
      for (int j = 1; j <= T; j += 4) { s.h[s.n] = h; s.p[s.n] = T - 1; s.jlo[s.n] = j; s.nb[s.n] = (T + 1 - j) < 4 ? T + 1 - j : 4; ++s.n; }
      for (int p = T - 2; p >= 0; --p)
        for (int j = 0; j <= p + 1; j += 4) { s.h[s.n] = h; s.p[s.n] = p; s.jlo[s.n] = j; s.nb[s.n] = (p + 2 - j) < 4 ? p + 2 - j : 4; ++s.n; }
    } else {
      for (int p = T; p >= 0; --p) {
        const int jlo = p > e0 ? p - e0 : 0;
        const int jhi = (D - 1) < (T + p - e0) ? (D - 1) : (T + p - e0);
        for (int j = jlo; j <= jhi; j += 4) { s.h[s.n] = h; s.p[s.n] = p; s.jlo[s.n] = j; s.nb[s.n] = (jhi + 1 - j) < 4 ? jhi + 1 - j : 4; ++s.n; }
      }
    }
  }
  return s;
}

constexpr int SM_A = 0, SM_B = SM_A + 2 * APLANE, SM_TAB = SM_B + 2 * BOPER, SM_ST = SM_TAB + 32768;
constexpr int SMEM = SM_ST + 49152;

// work flags: 1 MMAs, 2 F, 4 L, 8 S
template <int E0, bool SPLIT>
__global__ void __launch_bounds__(512, 1) stage(int iters, int flags, double* sink) {
  extern __shared__ __align__(1024) uint8_t dyn[];
  __shared__ uint64_t mma_bar, work_bar;
  __shared__ uint32_t tmem_base;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  for (int i = tid; i < SMEM / 4; i += 512) reinterpret_cast<uint32_t*>(dyn)[i] = i * 2654435761u;
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tmem_base)),
                 "n"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(&mma_bar)), "r"(1));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(&work_bar)), "r"(15));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = tmem_base;
  constexpr Sched S = make_sched(E0, SPLIT);
  const bool mma = flags & 1;
  if (warp == 0) {
    const uint64_t da0 = smem_desc(smem_u32(dyn + SM_A), (BM / 8) * 128, 128);
    const uint64_t db0 = smem_desc(smem_u32(dyn + SM_B), (BROWS / 8) * 128, 128);
    for (int it = 0; it < iters; ++it) {
      if (mma) {
#pragma unroll
        for (int i = 0; i < S.n; ++i) {
          const int q0 = S.jlo[i] + E0 - S.p[i];
          const uint64_t db = db0 + (uint64_t)((S.h[i] * BOPER + q0 * BN2 * 16) >> 4);
          const uint64_t da = da0 + (uint64_t)((S.h[i] * APLANE + S.p[i] * ASLICE) >> 4);
          if (lane == 0) mma_ss(tmem + S.jlo[i] * BN2, da, db, idesc_i8(128, S.nb[i] * BN2, S.p[i] == NSL - 1, true), 1);
        }
        if (lane == 0) mma_commit(&mma_bar);
        __syncwarp();
        mbar_wait(&mma_bar, it & 1);
      }
      mbar_wait(&work_bar, it & 1);
    }
  } else {
    double acc[8];
#pragma unroll
    for (int c = 0; c < 8; ++c) acc[c] = 1.0 + 1e-9 * (tid + c);
    const double2* tab = reinterpret_cast<const double2*>(dyn + SM_TAB);
    uint32_t x = tid * 7919u;
    for (int it = 0; it < iters; ++it) {
      if (flags & 2) {
        // 4096 / 15 ~ 273 warp DFMAs: 8 chains x 34
#pragma unroll 2
        for (int r = 0; r < 34; ++r)
#pragma unroll
          for (int c = 0; c < 8; ++c) acc[c] = fma(acc[c], 0.999999999, 1e-12);
      }
      if (flags & 4) {
        // 128 / 15 ~ 9 random LDS.128 per warp
#pragma unroll
        for (int r = 0; r < 9; ++r) {
          x = x * 1664525u + 1013904223u;
          const double2 t = (flags & 16) ? tab[((x >> 24) << 3) | (lane & 7)]  // 256 entries x 8 lane copies
                                         : tab[x >> 21];                       // 2048 entries
          acc[r & 7] += t.x * 1e-30;
        }
      }
      if (flags & 8) {
        // 48 KB / 480 threads / 8 B ~ 13 STS.64 per thread
        uint8_t* st = dyn + SM_ST;
#pragma unroll
        for (int r = 0; r < 13; ++r) {
          x = x * 1664525u + 1013904223u;
          *reinterpret_cast<uint2*>(st + ((tid * 8 + r * 3840) % 49152)) = make_uint2(x, x ^ 5);
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&work_bar);
      if (mma) mbar_wait(&mma_bar, it & 1);
      mbar_wait(&work_bar, it & 1);
    }
    double s = 0;
#pragma unroll
    for (int c = 0; c < 8; ++c) s += acc[c];
    if (s == 12345.0) sink[0] = s;
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(512));
}

template <int E0, bool SPLIT>
void run(const char* tag, int sms, double* sink) {
  auto k = stage<E0, SPLIT>;
  CK(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM));
  const char* names[16] = {"none", "MMA", "F", "MMA+F", "L", "MMA+L", "F+L", "MMA+F+L",
                           "S", "MMA+S", "F+S", "MMA+F+S", "L+S", "MMA+L+S", "F+L+S", "MMA+F+L+S"};
  const int fl[] = {1, 2, 3, 4, 5, 8, 9, 6, 7, 14, 15, 20, 21, 23, 31};
  for (int f : fl) {
    const int iters = 2000;
    k<<<sms, 512, SMEM>>>(10, f, sink);
    CK(cudaDeviceSynchronize());
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaEventRecord(a);
    k<<<sms, 512, SMEM>>>(iters, f, sink);
    cudaEventRecord(b);
    CK(cudaEventSynchronize(b));
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    printf("%-22s %-10s%s %6.0f cycles/stage\n", tag, names[f & 15], (f & 16) ? " (L: 8 lane copies)" : "", ms / 1e3 * 1.965e9 / iters);
  }
}

int main() {
  double* sink;
  CK(cudaMalloc(&sink, 8));
  int sms = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  run<4, true>("e>=4, 20 MMAs (r2)", sms, sink);
  run<4, false>("e>=4, 18 MMAs", sms, sink);
  run<5, false>("e>=5, 16 MMAs", sms, sink);
  return 0;
}
