// tc_sched.cu -- tcgen05 kind::i8 throughput of the K2 slice-pair MMA schedule
// (k_matvec_oz.cu, 6 slices, NCB = 32: 20 MMAs per stage, M = 128, K = 32,
// N = 64..256 over 7 TMEM diagonal blocks whose windows overlap), against
// orderings of the same MMAs and the plain same-D K-loop.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 tc_sched.cu -o tc_sched
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>

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
__device__ __forceinline__ void mma_i8(uint32_t d, uint64_t da, uint64_t db, uint32_t idesc, uint32_t acc) {
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

constexpr int NSL = 6, E0 = 4, NDIAG = 7, BN2 = 64, BM = 128, KS = 32;
constexpr int ASLICE = BM * KS, APLANE = NSL * ASLICE, BROWS = NSL * BN2, BOPER = BROWS * KS;

struct Mma {
  int h, p, jlo, nb;
};

// variant 0: the kernel's order; 1: the two planes of each (p, window) back to back;
// 2: the kernel's MMAs all aimed at D block 0 (no partial window overlaps);
// 3: plain K-loop, N = 256 into one D (reference)
__constant__ Mma g_sched[64];
__constant__ int g_n;

// 4: variant 0 while 15 other warps spin on the completion mbarrier (try_wait loop);
// 5: variant 0 while 15 warps store to a scratch region (the A-slice write traffic);
// 6: variant 0 with a TMA bulk copy refilling the B image before every stage
__global__ void __launch_bounds__(512, 1) rate(int iters, int variant, int32_t* sink, const uint8_t* gsrc) {
  extern __shared__ __align__(1024) uint8_t dyn[];
  uint8_t* sA = dyn;
  uint8_t* sB = dyn + 2 * APLANE;
  uint8_t* scratch = dyn + 2 * APLANE + 2 * BOPER;
  __shared__ uint64_t bar, tbar;
  __shared__ volatile int done;
  __shared__ uint32_t tmem_base;
  const int tid = threadIdx.x, warp = tid >> 5;
  for (int i = tid; i < 2 * APLANE + 2 * BOPER; i += 512) dyn[i] = (uint8_t)(i * 7 + 3);
  if (tid == 0) done = 0;
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tmem_base)),
                 "n"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(&tbar)), "r"(1));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(&bar)), "r"(1));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = tmem_base;
  if (tid == 0) {
    const uint64_t da0 = smem_desc(smem_u32(sA), (BM / 8) * 128, 128);
    const uint64_t db0 = smem_desc(smem_u32(sB), (BROWS / 8) * 128, 128);
    for (int it = 0; it < iters; ++it) {
      if (variant == 3) {
        for (int k = 0; k < 13; ++k) {
          const uint64_t da = da0 + (uint64_t)((k % 12) * ASLICE >> 4);
          const uint64_t db = db0;
          mma_i8(tmem, da, db, idesc_i8(128, 256, false, true), 1);
        }
        continue;
      }
      if (variant == 6) {
        // refill B by TMA (24 KB) and wait for it, as a stage does
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&tbar)), "r"(2 * BOPER)
                     : "memory");
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                         smem_u32(sB)),
                     "l"(gsrc + (it & 63) * 2 * BOPER), "r"(2 * BOPER), "r"(smem_u32(&tbar))
                     : "memory");
        mbar_wait(&tbar, it & 1);
      }
      for (int i = 0; i < g_n; ++i) {
        const Mma m = g_sched[i];
        const int q0 = m.jlo + E0 - m.p;
        const uint64_t da = da0 + (uint64_t)((m.h * APLANE + m.p * ASLICE) >> 4);
        const uint64_t db = db0 + (uint64_t)((m.h * BOPER + q0 * BN2 * 16) >> 4);
        const uint32_t d = tmem + (variant == 2 ? 0 : m.jlo * BN2);
        mma_i8(d, da, db, idesc_i8(128, m.nb * BN2, m.p == NSL - 1, true), 1);
      }
    }
    mma_commit(&bar);
  } else if (variant == 5 && warp > 0) {
    // store traffic: 8-byte stores at the A-image rate until the MMAs are done
    uint32_t x = tid;
    while (!done) {
      for (int r = 0; r < 64; ++r) {
        x = x * 1664525u + 1013904223u;
        *reinterpret_cast<uint2*>(scratch + ((tid * 8 + r * 4096) & 49151)) = make_uint2(x, x ^ 7);
      }
    }
  }
  if (tid == 0) {
    mbar_wait(&bar, 0);
    done = 1;
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

static std::vector<Mma> kernel_sched(bool plane_pairs) {
  // the 6-slice schedule of k_matvec_oz.cu (make_sched, MAXB = 4)
  std::vector<Mma> per_plane;
  const int T = NSL - 1, D = NDIAG, maxb = 4;
  for (int j = 1; j <= D - 1; j += maxb) per_plane.push_back({0, T, j, (D - j) < maxb ? D - j : maxb});
  per_plane.push_back({0, T - 1, 0, 1});
  for (int j = 1; j <= T; j += maxb) per_plane.push_back({0, T - 1, j, (T + 1 - j) < maxb ? T + 1 - j : maxb});
  for (int p = T - 2; p >= 0; --p)
    for (int j = 0; j <= p + 1; j += maxb) per_plane.push_back({0, p, j, (p + 2 - j) < maxb ? p + 2 - j : maxb});
  std::vector<Mma> s;
  if (plane_pairs) {
    for (auto m : per_plane) {
      s.push_back(m);
      m.h = 1;
      s.push_back(m);
    }
  } else {
    for (int h = 0; h < 2; ++h)
      for (auto m : per_plane) {
        m.h = h;
        s.push_back(m);
      }
  }
  return s;
}

int main() {
  int32_t* sink;
  CK(cudaMalloc(&sink, 4));
  const int smem = 2 * APLANE + 2 * BOPER + 49152;
  uint8_t* gsrc;
  CK(cudaMalloc(&gsrc, 64 * 2 * BOPER));
  CK(cudaMemset(gsrc, 3, 64 * 2 * BOPER));
  CK(cudaFuncSetAttribute(rate, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  int sms = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  const char* names[7] = {"kernel order", "plane pairs", "all D at block 0", "K-loop N=256 (13 MMAs)",
                          "+ 15 warps spinning", "+ 15 warps storing", "+ TMA B refill"};
  for (int variant = 0; variant < 7; ++variant) {
    std::vector<Mma> s = kernel_sched(variant == 1);
    double macs_per_iter = 0;
    if (variant == 3) {
      macs_per_iter = 13.0 * 128 * 256 * 32;
    } else {
      for (auto& m : s) macs_per_iter += 128.0 * m.nb * BN2 * 32;
    }
    int n = (int)s.size();
    CK(cudaMemcpyToSymbol(g_sched, s.data(), s.size() * sizeof(Mma)));
    CK(cudaMemcpyToSymbol(g_n, &n, sizeof(int)));
    const int iters = 2000;
    rate<<<sms, 512, smem>>>(10, variant, sink, gsrc);
    CK(cudaDeviceSynchronize());
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaEventRecord(a);
    rate<<<sms, 512, smem>>>(iters, variant, sink, gsrc);
    cudaEventRecord(b);
    CK(cudaEventSynchronize(b));
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    const double tops = 2.0 * macs_per_iter * iters * sms / (ms / 1e3) / 1e12;
    printf("%-24s %2d MMAs/stage: %.3f ms  %.1f TOPS int8  (%.0f cycles/stage at 1.965 GHz)\n", names[variant],
           variant == 3 ? 13 : n, ms, tops, ms / 1e3 * 1.965e9 / iters);
  }
  return 0;
}
