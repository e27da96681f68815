// tc_tmem_a.cu -- tcgen05 kind::i8 with the A operand in tensor memory vs shared
// memory, for the K2 slice-pair schedules (k_matvec_oz.cu):
//  (1) layout check: D = A B^T with A stored in TMEM (lane = row, column c =
//      K bytes 4c..4c+3) equals the shared-memory-A MMA and a host reference;
//  (2) throughput of one stage's MMAs (M = 128, K = 32, NCB = 32) for
//      - the 6-slice, 7-diagonal schedule (20 MMAs, A in smem) = round 2,
//      - the 6-slice, 6-diagonal schedule (e >= 5: 16 MMAs) with A in smem,
//      - the 6-diagonal schedule with A in TMEM,
//      each alone and with 15 warps writing the next A stage concurrently
//      (shared-memory stores for smem A, tcgen05.st for TMEM A).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 --expt-relaxed-constexpr tc_tmem_a.cu -o tc_tmem_a
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
__device__ __forceinline__ void mma_ss(uint32_t d, uint64_t da, uint64_t db, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(d),
      "l"(da), "l"(db), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ void mma_ts(uint32_t d, uint32_t ta, uint64_t db, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::i8 [%0], [%1], %2, %3, p;\n\t}\n" ::"r"(d),
      "r"(ta), "l"(db), "r"(idesc), "r"(acc));
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
__device__ __forceinline__ void tmem_st2(uint32_t addr, uint32_t a, uint32_t b) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x2.b32 [%0], {%1, %2};" ::"r"(addr), "r"(a), "r"(b) : "memory");
}
__device__ __forceinline__ void tmem_st8(uint32_t addr, const uint32_t (&v)[8]) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};" ::"r"(addr), "r"(v[0]),
               "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7])
               : "memory");
}

// ------------------------------------------------------------ (1) layout check
// A: 128 x 32 int8 (row-major, signed), B: 64 x 32 int8 (N rows, signed)
__global__ void __launch_bounds__(128, 1) check(const int8_t* A, const int8_t* B, int32_t* Dss, int32_t* Dts) {
  __shared__ __align__(1024) uint8_t sA[128 * 32];
  __shared__ __align__(1024) uint8_t sB[64 * 32];
  __shared__ uint64_t bar;
  __shared__ uint32_t tmem_base;
  const int tid = threadIdx.x, warp = tid >> 5;
  // canonical K-major no-swizzle images: core matrix (8 rows x 16 B), LBO = K-direction step
  for (int i = tid; i < 128 * 32; i += 128) {
    const int r = i / 32, k = i % 32;
    sA[((k >> 4) * 16 + (r >> 3)) * 128 + (r & 7) * 16 + (k & 15)] = (uint8_t)A[i];
  }
  for (int i = tid; i < 64 * 32; i += 128) {
    const int r = i / 32, k = i % 32;
    sB[((k >> 4) * 8 + (r >> 3)) * 128 + (r & 7) * 16 + (k & 15)] = (uint8_t)B[i];
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tmem_base)),
                 "n"(256));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(&bar)), "r"(1));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = tmem_base;
  // A into TMEM columns 128..135: lane = row, column c = bytes 4c..4c+3 of the row
  {
    const int r = tid;
    uint32_t v[8];
    for (int c = 0; c < 8; ++c) {
      uint32_t w = 0;
      for (int b = 0; b < 4; ++b) w |= (uint32_t)(uint8_t)A[r * 32 + 4 * c + b] << (8 * b);
      v[c] = w;
    }
    tmem_st8(tmem + ((uint32_t)(warp * 32) << 16) + 128, v);
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  if (tid == 0) {
    const uint64_t da = smem_desc(smem_u32(sA), (128 / 8) * 128, 128);
    const uint64_t db = smem_desc(smem_u32(sB), (64 / 8) * 128, 128);
    mma_ss(tmem + 0, da, db, idesc_i8(128, 64, true, true), 0);
    mma_ts(tmem + 64, tmem + 128, db, idesc_i8(128, 64, true, true), 0);
    mma_commit(&bar);
  }
  mbar_wait(&bar, 0);
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  for (int c = 0; c < 128; ++c) {
    uint32_t v;
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x1.b32 {%0}, [%1];"
                 : "=r"(v)
                 : "r"(tmem + ((uint32_t)(warp * 32) << 16) + c));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
    if (c < 64)
      Dss[tid * 64 + c] = (int32_t)v;
    else
      Dts[tid * 64 + c - 64] = (int32_t)v;
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(256));
}

// ------------------------------------------------------------ (2) throughput
constexpr int NSL = 6, BN2 = 64, BM = 128, KS = 32;
constexpr int ASLICE = BM * KS, APLANE = NSL * ASLICE, BROWS = NSL * BN2, BOPER = BROWS * KS;
struct Sched {
  int h[64], p[64], jlo[64], nb[64];
  int n;
};
// slice-pair schedule: diagonals e = e0 .. 2 NSL - 2 kept, windows of <= 4 blocks per slice
constexpr Sched make_sched(int e0, bool split) {
  Sched s{};
  s.n = 0;
  const int T = NSL - 1, D = 2 * NSL - 1 - e0;
  for (int h = 0; h < 2; ++h) {
    if (split) {  // k_matvec_oz.cu make_sched (round 2)
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

// TMEM_A: A operand from TMEM; WRITERS: 15 warps write one A stage (48 KB:
// smem stores, or tcgen05.st for TMEM A) per MMA stage, paced by the stage's
// commit barrier
template <int E0, bool SPLIT, bool TMEM_A, bool WRITERS>
__global__ void __launch_bounds__(512, 1) rate(int iters, int32_t* sink) {
  extern __shared__ __align__(1024) uint8_t dyn[];
  uint8_t* sA = dyn;
  uint8_t* sB = dyn + 2 * APLANE;
  uint8_t* scratch = dyn + 2 * APLANE + 2 * BOPER;
  __shared__ uint64_t bar, stage_bar;
  __shared__ uint32_t tmem_base;
  const int tid = threadIdx.x, warp = tid >> 5;
  for (int i = tid; i < 2 * APLANE + 2 * BOPER; i += 512) dyn[i] = (uint8_t)(i * 7 + 3);
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tmem_base)),
                 "n"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(&bar)), "r"(1));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(&stage_bar)), "r"(1));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = tmem_base;
  const uint32_t tA = tmem + 384;  // TMEM A stage: 12 slice-planes x 8 columns
  constexpr Sched S = make_sched(E0, SPLIT);
  if (warp == 0) {
    const uint64_t da0 = smem_desc(smem_u32(sA), (BM / 8) * 128, 128);
    const uint64_t db0 = smem_desc(smem_u32(sB), (BROWS / 8) * 128, 128);
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int i = 0; i < S.n; ++i) {
        const int q0 = S.jlo[i] + E0 - S.p[i];
        const uint64_t db = db0 + (uint64_t)((S.h[i] * BOPER + q0 * BN2 * 16) >> 4);
        const uint32_t d = tmem + S.jlo[i] * BN2;
        constexpr uint32_t dummy = 0;
        (void)dummy;
        const uint32_t idesc = idesc_i8(128, S.nb[i] * BN2, S.p[i] == NSL - 1, true);
        if (threadIdx.x == 0) {
          if (TMEM_A)
            mma_ts(d, tA + (S.h[i] * NSL + S.p[i]) * 8, db, idesc, 1);
          else
            mma_ss(d, da0 + (uint64_t)((S.h[i] * APLANE + S.p[i] * ASLICE) >> 4), db, idesc, 1);
        }
      }
      if (threadIdx.x == 0) mma_commit(&stage_bar);
      __syncwarp();
      if (WRITERS) mbar_wait(&stage_bar, it & 1);  // one stage in flight, like the kernel's ring
    }
    if (threadIdx.x == 0) mma_commit(&bar);
  } else if (WRITERS) {
    // each of the 15 warps: 1/15 of an A stage per MMA stage
    uint32_t x = tid;
    for (int it = 0; it < iters; ++it) {
      if (!TMEM_A) {
        for (int r = 0; r < 13; ++r) {  // 13 x 8 B x 480 threads = 49 KB
          x = x * 1664525u + 1013904223u;
          *reinterpret_cast<uint2*>(scratch + ((tid * 8 + r * 4096) & 49151)) = make_uint2(x, x ^ 7);
        }
      } else {
        const uint32_t base = tmem + ((uint32_t)((warp & 3) * 32) << 16) + 480 + 8 * ((warp >> 2) & 3);
        for (int r = 0; r < 3; ++r) {  // 3 x 32 B x 480 threads = 45 KB
          x = x * 1664525u + 1013904223u;
          uint32_t v[8] = {x, x ^ 1, x ^ 2, x ^ 3, x ^ 4, x ^ 5, x ^ 6, x ^ 7};
          tmem_st8(base, v);
        }
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
      }
      mbar_wait(&stage_bar, it & 1);
    }
  }
  mbar_wait(&bar, 0);
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  uint32_t v;
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x1.b32 {%0}, [%1];" : "=r"(v) : "r"(tmem + ((uint32_t)((warp & 3) * 32) << 16)));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
  if (v == 0x12345) sink[0] = v;
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(512));
}

template <int E0, bool SPLIT, bool TMEM_A, bool WRITERS>
void run(const char* name, int sms, int32_t* sink) {
  constexpr Sched S = make_sched(E0, SPLIT);
  double ncols = 0;
  for (int i = 0; i < S.n; ++i) ncols += S.nb[i] * BN2;
  const int smem = 2 * APLANE + 2 * BOPER + 49152;
  auto k = rate<E0, SPLIT, TMEM_A, WRITERS>;
  CK(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  const int iters = 2000;
  k<<<sms, 512, smem>>>(10, sink);
  CK(cudaDeviceSynchronize());
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaEventRecord(a);
  k<<<sms, 512, smem>>>(iters, sink);
  cudaEventRecord(b);
  CK(cudaEventSynchronize(b));
  float ms = 0;
  cudaEventElapsedTime(&ms, a, b);
  const double tops = 2.0 * ncols * 128 * 32 * iters * sms / (ms / 1e3) / 1e12;
  printf("%-40s %2d MMAs, %5.0f N-cols/stage: %.3f ms  %.1f TOPS  %.0f cycles/stage\n", name, S.n, ncols, ms, tops,
         ms / 1e3 * 1.965e9 / iters);
}

int main() {
  // (1) layout check
  {
    std::vector<int8_t> A(128 * 32), B(64 * 32);
    uint32_t x = 12345;
    for (auto& a : A) { x = x * 1664525u + 1013904223u; a = (int8_t)(x >> 24); }
    for (auto& b : B) { x = x * 1664525u + 1013904223u; b = (int8_t)(x >> 24); }
    int8_t *dA, *dB;
    int32_t *dss, *dts;
    CK(cudaMalloc(&dA, A.size()));
    CK(cudaMalloc(&dB, B.size()));
    CK(cudaMalloc(&dss, 128 * 64 * 4));
    CK(cudaMalloc(&dts, 128 * 64 * 4));
    CK(cudaMemcpy(dA, A.data(), A.size(), cudaMemcpyHostToDevice));
    CK(cudaMemcpy(dB, B.data(), B.size(), cudaMemcpyHostToDevice));
    check<<<1, 128>>>(dA, dB, dss, dts);
    CK(cudaDeviceSynchronize());
    std::vector<int32_t> ss(128 * 64), ts(128 * 64);
    CK(cudaMemcpy(ss.data(), dss, ss.size() * 4, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(ts.data(), dts, ts.size() * 4, cudaMemcpyDeviceToHost));
    int bad_ss = 0, bad_ts = 0;
    for (int i = 0; i < 128; ++i)
      for (int j = 0; j < 64; ++j) {
        int32_t r = 0;
        for (int k = 0; k < 32; ++k) r += (int32_t)A[i * 32 + k] * (int32_t)B[j * 32 + k];
        bad_ss += ss[i * 64 + j] != r;
        bad_ts += ts[i * 64 + j] != r;
      }
    printf("layout check (128x64x32 i8): smem-A mismatches %d, TMEM-A mismatches %d of %d\n", bad_ss, bad_ts, 128 * 64);
  }
  // (2) throughput
  int32_t* sink;
  CK(cudaMalloc(&sink, 4));
  int sms = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  run<4, true, false, false>("7 diag, init split, smem A (round 2)", sms, sink);
  run<4, false, false, false>("7 diag, no split, smem A", sms, sink);
  run<4, false, true, false>("7 diag, no split, TMEM A", sms, sink);
  run<5, false, false, false>("6 diag (e>=5), smem A", sms, sink);
  run<5, false, true, false>("6 diag (e>=5), TMEM A", sms, sink);
  run<4, true, false, true>("7 diag split smem A, paced + A writes", sms, sink);
  run<4, true, false, false>("(same, no writers, unpaced)", sms, sink);
  run<4, false, true, true>("7 diag TMEM A, paced + tcgen05.st", sms, sink);
  run<5, false, false, true>("6 diag smem A, paced + A writes", sms, sink);
  run<5, false, true, true>("6 diag TMEM A, paced + tcgen05.st", sms, sink);
  return 0;
}
