// k_gemm.cu -- batched small complex GEMM (butterfly apply levels, partial
// chain projections; butterfly.hpp:71-193, 330-382).
//
// Every output block is C_e = sum_{s<S} op(A_s) B_s with uniform padded
// shapes per launch (zero padding contributes exact zeros).  One CTA computes
// a 32 x 32 tile of one block; A and B tiles are staged through shared memory.
#include <climits>
#include <cstdlib>
#include <type_traits>

#include "kernels.cuh"

namespace bfly {

namespace {

constexpr int TM = 32, TN = 32, TK = 16;

template <typename R, int OP, int S>
__global__ void __launch_bounds__(256) bgemm_kernel(const cx<R>* __restrict__ A, int64_t lda,
                                                    const cx<R>* __restrict__ B, int64_t ldb, cx<R>* __restrict__ C,
                                                    int64_t ldc, int M, int K, const GemmEnt* __restrict__ ents,
                                                    int accumulate, int ncols_all) {
  using V = cx<R>;
  __shared__ V As[TK][TM + 1];
  __shared__ V Bs[TK][TN + 1];
  const GemmEnt e = ents[blockIdx.x];
  const int ncols = ncols_all > 0 ? ncols_all : e.ncols;
  const int Me = min(M, e.mrows), Ke = min(K, e.krows);
  const int n0 = blockIdx.y * TN;
  const int m0 = blockIdx.z * TM;
  if (n0 >= ncols || m0 >= Me) return;
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  V acc[2][2];
#pragma unroll
  for (int i = 0; i < 2; ++i)
#pragma unroll
    for (int j = 0; j < 2; ++j) acc[i][j] = mkc<R>(0, 0);

#pragma unroll
  for (int s = 0; s < S; ++s) {
    const V* Ab = A + (s == 0 ? e.a0 : e.a1);
    const V* Bb = B + (s == 0 ? e.b0 : e.b1);
    for (int k0 = 0; k0 < K; k0 += TK) {
      // A tile: element (m, k) of op(A), m in [m0, m0+32), k in [k0, k0+16)
#pragma unroll
      for (int q = 0; q < 2; ++q) {
        int idx = threadIdx.x + q * 256;
        int mm, kk;
        if (OP == OP_N) {
          mm = idx & 31;
          kk = idx >> 5;
        } else {
          kk = idx & 15;
          mm = idx >> 4;
        }
        int gm = m0 + mm, gk = k0 + kk;
        V v = mkc<R>(0, 0);
        if (gm < Me && gk < K) {
          if (OP == OP_N) v = Ab[gm + (int64_t)gk * lda];
          else {
            v = Ab[gk + (int64_t)gm * lda];
            if (OP == OP_H) v = cconj(v);
          }
        }
        As[kk][mm] = v;
      }
#pragma unroll
      for (int q = 0; q < 2; ++q) {
        int idx = threadIdx.x + q * 256;
        int kk = idx & 15, nn = idx >> 4;
        int gk = k0 + kk, gn = n0 + nn;
        V v = mkc<R>(0, 0);
        if (gk < Ke && gn < ncols) v = Bb[gk + (int64_t)gn * ldb];
        Bs[kk][nn] = v;
      }
      __syncthreads();
#pragma unroll
      for (int kk = 0; kk < TK; ++kk) {
        V a0 = As[kk][ty], a1 = As[kk][ty + 16];
        V b0 = Bs[kk][tx], b1 = Bs[kk][tx + 16];
        cfma(acc[0][0], a0, b0);
        cfma(acc[0][1], a0, b1);
        cfma(acc[1][0], a1, b0);
        cfma(acc[1][1], a1, b1);
      }
      __syncthreads();
    }
  }
  V* Cb = C + e.c;
#pragma unroll
  for (int i = 0; i < 2; ++i)
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      int gm = m0 + ty + 16 * i, gn = n0 + tx + 16 * j;
      if (gm < Me && gn < ncols) {
        V* p = Cb + gm + (int64_t)gn * ldc;
        *p = accumulate ? cadd(*p, acc[i][j]) : acc[i][j];
      }
    }
}

// Small-k path (butterfly apply with few columns: HBM/latency bound).  One
// 128-thread CTA per output block: op(A_s) is staged in shared memory with
// coalesced reads for both N (down the columns) and H (along the rows of the
// stored block), the K x k input slice next to it; each thread then owns
// (row, column) outputs.  Every factor element is read exactly once.
template <typename R, int OP, int S>
__global__ void __launch_bounds__(128) bgemm_small_kernel(const cx<R>* __restrict__ A, int64_t lda,
                                                          const cx<R>* __restrict__ B, int64_t ldb,
                                                          cx<R>* __restrict__ C, int64_t ldc, int M, int K,
                                                          const GemmEnt* __restrict__ ents, int accumulate,
                                                          int ncols_all) {
  using V = cx<R>;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  V* As = reinterpret_cast<V*>(smem_raw);  // [S][K][M+1]: op(A)(m, kk) at m + kk*(M+1)
  const GemmEnt e = ents[blockIdx.x];
  const int ncols = ncols_all > 0 ? ncols_all : e.ncols;
  const int Me = min(M, e.mrows), Ke = min(K, e.krows);
  const int SMA = M + 1;
  V* Bs = As + S * K * SMA;                // [S][ncols][K]
  // A (a fixed factor level when launched with programmatic dependent launch,
  // see launch_bgemm's pdl flag) is staged first; B, the previous stage's
  // output, only after griddepcontrol.wait (a no-op for ordinary launches).
#pragma unroll
  for (int s = 0; s < S; ++s) {
    const V* Ab = A + (s == 0 ? e.a0 : e.a1);
    V* as = As + s * K * SMA;
    if (OP == OP_N) {
      for (int idx = threadIdx.x; idx < M * K; idx += 128) {
        const int m = idx % M, kk = idx / M;
        as[m + kk * SMA] = Ab[m + (int64_t)kk * lda];
      }
    } else {
      for (int idx = threadIdx.x; idx < M * K; idx += 128) {
        const int kk = idx % K, m = idx / K;
        V v = Ab[kk + (int64_t)m * lda];
        if (OP == OP_H) v = cconj(v);
        as[m + kk * SMA] = v;
      }
    }
  }
  asm volatile("griddepcontrol.wait;" ::: "memory");
#pragma unroll
  for (int s = 0; s < S; ++s) {
    const V* Bb = B + (s == 0 ? e.b0 : e.b1);
    V* bs = Bs + s * ncols * K;
    for (int idx = threadIdx.x; idx < K * ncols; idx += 128) {
      const int kk = idx % K, cc = idx / K;
      bs[kk + cc * K] = kk < Ke ? Bb[kk + (int64_t)cc * ldb] : mkc<R>(0, 0);
    }
  }
  __syncthreads();
  asm volatile("griddepcontrol.launch_dependents;");
  V* Cb = C + e.c;
  for (int idx = threadIdx.x; idx < Me * ncols; idx += 128) {
    const int m = idx % Me, cc = idx / Me;
    V acc = mkc<R>(0, 0);
#pragma unroll
    for (int s = 0; s < S; ++s) {
      const V* as = As + s * K * SMA + m;
      const V* bs = Bs + s * ncols * K + cc * K;
      for (int kk = 0; kk < K; ++kk) cfma(acc, as[kk * SMA], bs[kk]);
    }
    V* p = Cb + m + (int64_t)cc * ldc;
    *p = accumulate ? cadd(*p, acc) : acc;
  }
}

// Butterfly apply stages (programmatic dependent launch chains, k <= 16).
// WPE warps own one output block (a CTA holds up to 4 single-warp groups), so a k = 1
// stage grid needs ~14 warps per SM and three to four consecutive stage grids
// fit on the GPU at once.  Each grid triggers its dependents on entry; a
// launched-but-waiting grid queues its factor blocks (never written by the
// chain) as cp.async global->shared copies -- no register round trip, so a
// warp has its whole share of the block in flight at once -- and only then
// parks at griddepcontrol.wait.  The factor traffic of the next stages thus
// streams from HBM while this stage computes; the per-stage critical path is
// the previous stage's output (L2 resident) plus the small GEMV, which splits
// K over Q lanes per output (shuffle reduction) when the block has few
// outputs.  griddepcontrol.wait returns only once the prerequisite grid has
// completed and flushed, which transitively orders every earlier stage.
template <typename V>
__device__ __forceinline__ void cp_async_elem(V* dst, const V* src) {
  const uint32_t d = (uint32_t)__cvta_generic_to_shared(dst);
  if constexpr (sizeof(V) == 16)
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(d), "l"(src) : "memory");
  else
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(d), "l"(src) : "memory");
}

#ifdef BFLY_STAGE_TRACE
// per stage: [0] first group start, [1] last group start, [2] first wait return,
// [3] last wait return, [4] last group end (%globaltimer ns)
__device__ unsigned long long g_stage_trace[64][10];
__device__ __forceinline__ unsigned long long gtime() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
#define STAGE_TRACE(slot, v)                                                  \
  do {                                                                          \
    if (t == 0 && (ei & 31) == 0) {                                           \
      const unsigned long long now = gtime();                                   \
      if (v & 1) atomicMax(&g_stage_trace[slot][v >> 1], now);                  \
      else atomicMin(&g_stage_trace[slot][v >> 1], now);                        \
    }                                                                           \
  } while (0)
#else
#define STAGE_TRACE(slot, v) \
  do {                       \
  } while (0)
#endif

__device__ __forceinline__ void st_mbar_wait(uint32_t bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred done;\n\t"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.acquire.cta.shared::cta.b64 done, [%0], %1, %2;\n\t"
      "@!done bra WAIT_%=;\n\t}\n" ::"r"(bar),
      "r"(parity), "r"(1000000u)
      : "memory");
}

// Shared-memory image of one output block: per s, op(A_s) in the stored
// orientation -- OP_N: column kk of A_s (M entries) at kk*(M+1), lanes then
// read consecutive rows; OP_T/OP_H: stored column m (K entries) at m*P with
// an ODD pitch P (K+1 or K+2), so lanes reading one kk of different m hit
// distinct 16-byte bank groups -- then the K x ncols input slices; an
// mbarrier heads the group's region.
__host__ __device__ __forceinline__ int stage_pitch(int op, int M, int K) {
  return op == OP_N ? M + 1 : K + 1 + (K & 1);
}
__host__ __device__ __forceinline__ int64_t stage_group_elems(int op, int M, int K, int S, int ncols) {
  return (int64_t)S * ((int64_t)(op == OP_N ? K : M) * stage_pitch(op, M, K) + (int64_t)K * ncols);
}

__device__ __forceinline__ void dmma884(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

// DM = true (complex128, 8..32 columns): after the same staging, the warps of
// the group tile the output block in 8 x 8 DMMA tiles (m8n8k4 f64 fragments
// read from the shared-memory image; complex MAC = 4 real DMMAs, two
// interleaved accumulator sets per tile).
template <typename R, int OP, int S, bool DM = false>
__global__ void __launch_bounds__(256) bgemm_stage_kernel(const cx<R>* __restrict__ A, int64_t lda,
                                                          const cx<R>* __restrict__ B, int64_t ldb,
                                                          cx<R>* __restrict__ C, int64_t ldc, int M, int K,
                                                          const GemmEnt* __restrict__ ents, int nent, int accumulate,
                                                          int ncols, int wpe, L2Prefetch pf) {
  using V = cx<R>;
  constexpr bool kBulk = sizeof(V) == 16;  // TMA bulk copies need 16-byte granules
  asm volatile("griddepcontrol.launch_dependents;");
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int gthreads = 32 * wpe;
  const int grp = threadIdx.x / gthreads, t = threadIdx.x % gthreads;
  const int64_t ei = (int64_t)blockIdx.x * (blockDim.x / gthreads) + grp;
  if (ei >= nent) return;
  // DM groups stage only the factor image (B fragments go to registers)
  const int64_t gbytes = 16 + stage_group_elems(OP, M, K, S, DM ? 0 : ncols) * (int64_t)sizeof(V);
  unsigned char* gbase = smem_raw + grp * gbytes;
  const uint32_t bar = (uint32_t)__cvta_generic_to_shared(gbase);
  V* As = reinterpret_cast<V*>(gbase + 16);
  const int cpitch = stage_pitch(OP, M, K);
  const int64_t aelems = (int64_t)(OP == OP_N ? K : M) * cpitch;
  V* Bs = As + S * aelems;  // [S][ncols][K]
  const GemmEnt e = ents[ei];
  const int Me = min(M, e.mrows), Ke = min(K, e.krows);
  if (pf.base != nullptr && pf.len >= 16 && t == 0) {
    const char* p = static_cast<const char*>(pf.base) + ei * pf.stride;
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"((uint32_t)(pf.len & ~int64_t(15)))
                 : "memory");
  }
  const int slot = e.pad_ & 63;  // stage index (BFLY_STAGE_TRACE instrumentation)
  (void)slot;
  STAGE_TRACE(slot, 0);
  STAGE_TRACE(slot, 3);
  // op(A_s) columns: OP_N copies the K stored columns (M entries each), the
  // transposed ops the M stored columns (K entries each)
  const int ncopy = OP == OP_N ? K : M, clen = OP == OP_N ? M : K;
  if constexpr (kBulk) {
    // the tensor-memory-access engine moves the factor block, so the load/
    // store pipe stays free for the running stage's GEMV
    if (t == 0) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bar));
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
      asm volatile("mbarrier.arrive.expect_tx.release.cta.shared::cta.b64 _, [%0], %1;" ::"r"(bar),
                   "r"((uint32_t)(S * ncopy * clen * sizeof(V)))
                   : "memory");
    }
    if (wpe == 1) __syncwarp();
    else __syncthreads();
    for (int c = t; c < S * ncopy; c += gthreads) {
      const int s = c >= ncopy, j = c - s * ncopy;
      const V* src = A + (s == 0 ? e.a0 : e.a1) + (int64_t)j * lda;
      const uint32_t dst = (uint32_t)__cvta_generic_to_shared(As + s * aelems + (int64_t)j * cpitch);
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                       dst),
                   "l"(src), "r"((uint32_t)(clen * sizeof(V))), "r"(bar)
                   : "memory");
    }
  } else {
#pragma unroll
    for (int s = 0; s < S; ++s) {
      const V* Ab = A + (s == 0 ? e.a0 : e.a1);
      V* as = As + s * aelems;
      for (int idx = t; idx < ncopy * clen; idx += gthreads) {
        const int i = idx % clen, j = idx / clen;
        cp_async_elem(as + i + j * cpitch, Ab + i + (int64_t)j * lda);
      }
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  }
  asm volatile("griddepcontrol.wait;" ::: "memory");
  STAGE_TRACE(slot, 4);
  STAGE_TRACE(slot, 7);
#pragma unroll
  for (int s = 0; s < (DM ? 0 : S); ++s) {
    const V* Bb = B + (s == 0 ? e.b0 : e.b1);
    V* bs = Bs + s * ncols * K;
    for (int idx = t; idx < K * ncols; idx += gthreads) {
      const int kk = idx % K, cc = idx / K;
      if (kk < Ke) cp_async_elem(bs + kk + cc * K, Bb + kk + (int64_t)cc * ldb);
      else bs[kk + cc * K] = mkc<R>(0, 0);
    }
  }
  asm volatile("cp.async.commit_group;" ::: "memory");
  asm volatile("cp.async.wait_all;" ::: "memory");
  if constexpr (kBulk) st_mbar_wait(bar, 0);
  if (wpe == 1) __syncwarp();
  else __syncthreads();  // multi-warp groups run one per CTA
  STAGE_TRACE(slot, 11);
  STAGE_TRACE(slot, 12);
  if constexpr (DM) {
    // B fragments straight from L2 (the previous stage's output; .cg: never a
    // stale L1 line), 8 k-steps per batch of loads
    const int lane = t & 31, gq = lane >> 2, tq = lane & 3;
    const int mt = (Me + 7) / 8, ntiles = mt * ((ncols + 7) / 8);
    if (K <= 32) {
      // one batch per source: the next batch (next source, or the next tile's
      // first) is requested before the current one's DMMAs, so the L2 latency
      // of the B fragments overlaps them (config-4 k = 16 apply)
      const int nw = gthreads >> 5;
      auto load = [&](int tl, int s, V(&bf)[8]) {
        const int n = (tl / mt) * 8 + gq;
        const V* Bb = B + (s == 0 ? e.b0 : e.b1) + (int64_t)n * ldb;
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const int k = 4 * u + tq;
          bf[u] = (tl < ntiles && n < ncols && k < Ke) ? __ldcg(Bb + k) : mkc<R>(0, 0);
        }
      };
      V bc[8], bn[8];
      int tile = t >> 5;
      load(tile, 0, bc);
      for (; tile < ntiles; tile += nw) {
        const int m = (tile % mt) * 8 + gq;
        double acc[2][2][2] = {};  // [set][re|im][2]
#pragma unroll
        for (int s = 0; s < S; ++s) {
          if (s + 1 < S) load(tile, s + 1, bn);
          else load(tile + nw, 0, bn);
          const V* as = As + s * aelems;
#pragma unroll
          for (int u = 0; u < 8; ++u) {
            const int k = 4 * u + tq;
            if (4 * u >= K) break;
            V a = mkc<R>(0, 0);
            if (m < M && k < K) {
              a = OP == OP_N ? as[k * cpitch + m] : as[m * cpitch + k];
              if (OP == OP_H) a.y = -a.y;
            }
            const V b = bc[u];
            const int st = u & 1;
            dmma884(acc[st][0][0], acc[st][0][1], a.x, b.x);
            dmma884(acc[st][1][0], acc[st][1][1], a.x, b.y);
            dmma884(acc[st][0][0], acc[st][0][1], -a.y, b.y);
            dmma884(acc[st][1][0], acc[st][1][1], a.y, b.x);
          }
#pragma unroll
          for (int u = 0; u < 8; ++u) bc[u] = bn[u];
        }
        if (m < Me) {
#pragma unroll
          for (int v = 0; v < 2; ++v) {
            const int col = (tile / mt) * 8 + 2 * tq + v;
            if (col >= ncols) continue;
            V r = mkc<R>(acc[0][0][v] + acc[1][0][v], acc[0][1][v] + acc[1][1][v]);
            V* p = C + e.c + m + (int64_t)col * ldc;
            *p = accumulate ? cadd(*p, r) : r;
          }
        }
      }
      STAGE_TRACE(slot, 9);
      return;
    }
    for (int tile = t >> 5; tile < ntiles; tile += gthreads >> 5) {
      const int m = (tile % mt) * 8 + gq, n = (tile / mt) * 8 + gq;
      double acc[2][2][2] = {};  // [set][re|im][2]
#pragma unroll
      for (int s = 0; s < S; ++s) {
        const V* as = As + s * aelems;
        const V* Bb = B + (s == 0 ? e.b0 : e.b1) + (int64_t)n * ldb;
        for (int kc = 0; kc < K; kc += 32) {
          V bf[8];
#pragma unroll
          for (int u = 0; u < 8; ++u) {
            const int k = kc + 4 * u + tq;
            bf[u] = (n < ncols && k < Ke) ? __ldcg(Bb + k) : mkc<R>(0, 0);
          }
#pragma unroll
          for (int u = 0; u < 8; ++u) {
            const int k = kc + 4 * u + tq;
            if (kc + 4 * u >= K) break;
            V a = mkc<R>(0, 0);
            if (m < M && k < K) {
              a = OP == OP_N ? as[k * cpitch + m] : as[m * cpitch + k];
              if (OP == OP_H) a.y = -a.y;
            }
            const V b = bf[u];
            const int st = u & 1;
            dmma884(acc[st][0][0], acc[st][0][1], a.x, b.x);
            dmma884(acc[st][1][0], acc[st][1][1], a.x, b.y);
            dmma884(acc[st][0][0], acc[st][0][1], -a.y, b.y);
            dmma884(acc[st][1][0], acc[st][1][1], a.y, b.x);
          }
        }
      }
      if (m < Me) {
#pragma unroll
        for (int v = 0; v < 2; ++v) {
          const int col = (tile / mt) * 8 + 2 * tq + v;
          if (col >= ncols) continue;
          V r = mkc<R>(acc[0][0][v] + acc[1][0][v], acc[0][1][v] + acc[1][1][v]);
          V* p = C + e.c + m + (int64_t)col * ldc;
          *p = accumulate ? cadd(*p, r) : r;
        }
      }
    }
    STAGE_TRACE(slot, 9);
    return;
  }
  // Q lanes per output (power of two, Q * outputs <= threads of the group).
  // The K split is across the HIGH lane bits (part = lane / (32/Q)), so a
  // quarter-warp reads 8 consecutive outputs of one kk: distinct bank groups
  // for every image pitch (a low-bit split costs 2-way conflicts, measured
  // 1.5x on tools/microbench/gemv_lat.cu).
  const int nout = Me * ncols;
  int Q = 1;
  while (Q < 32 && 2 * Q * nout <= gthreads) Q *= 2;
  const int opw = 32 / Q;  // outputs per warp and pass
  const int lane = t & 31, part = lane / opw;
  // element (m, kk) of op(A_s): stride along kk
  const int ks = OP == OP_N ? M + 1 : 1;
  V* Cb = C + e.c;
  for (int o0 = 0; o0 < nout; o0 += gthreads / Q) {
    const int o = o0 + (t >> 5) * opw + lane % opw;
    // four independent partial sums: the FP64 dependent-issue latency, not
    // throughput, bounds this loop
    V acc = mkc<R>(0, 0), acc1 = acc, acc2 = acc, acc3 = acc;
    if (o < nout) {
      const int m = o % Me, cc = o / Me;
#pragma unroll
      for (int s = 0; s < S; ++s) {
        const V* as = As + s * aelems + (OP == OP_N ? m : m * cpitch);
        const V* bs = Bs + s * ncols * K + cc * K;
        int kk = part;
        for (; kk + 3 * Q < K; kk += 4 * Q) {
          const V a0 = as[kk * ks], a1 = as[(kk + Q) * ks], a2 = as[(kk + 2 * Q) * ks], a3 = as[(kk + 3 * Q) * ks];
          const V b0 = bs[kk], b1 = bs[kk + Q], b2 = bs[kk + 2 * Q], b3 = bs[kk + 3 * Q];
          if (OP == OP_H) {
            cfma_conj(acc, a0, b0);
            cfma_conj(acc1, a1, b1);
            cfma_conj(acc2, a2, b2);
            cfma_conj(acc3, a3, b3);
          } else {
            cfma(acc, a0, b0);
            cfma(acc1, a1, b1);
            cfma(acc2, a2, b2);
            cfma(acc3, a3, b3);
          }
        }
        for (; kk < K; kk += Q) {
          if (OP == OP_H) cfma_conj(acc, as[kk * ks], bs[kk]);
          else cfma(acc, as[kk * ks], bs[kk]);
        }
      }
      acc = cadd(cadd(acc, acc1), cadd(acc2, acc3));
    }
    for (int q = opw; q < 32; q *= 2) {
      acc.x += __shfl_xor_sync(0xffffffffu, acc.x, q);
      acc.y += __shfl_xor_sync(0xffffffffu, acc.y, q);
    }
    if (o0 == 0) {
      STAGE_TRACE(slot, 17);
      STAGE_TRACE(slot, 18);
    }
    if (o < nout && part == 0) {
      const int m = o % Me, cc = o / Me;
      V* p = Cb + m + (int64_t)cc * ldc;
      *p = accumulate ? cadd(*p, acc) : acc;
    }
  }
  STAGE_TRACE(slot, 9);
}


// Narrow entries (M <= 16 rows, <= 32 columns: the U/V chain projections of
// one probe, ~10^5 entries per launch): one WARP per entry, m8n8k4 DMMA
// fragments loaded straight from global memory (L1/L2 resident), no shared
// memory or block barriers.  Complex MAC = 4 real DMMAs.
template <int OP, int S>
__global__ void __launch_bounds__(256) bgemm_dmma_warp_kernel(const double2* __restrict__ A, int64_t lda,
                                                              const double2* __restrict__ B, int64_t ldb,
                                                              double2* __restrict__ C, int64_t ldc, int M, int K,
                                                              const GemmEnt* __restrict__ ents, int nent,
                                                              int accumulate, int ncols_all) {
  // programmatic dependent launch (apply stages): dependents may start at
  // once; B and C are touched only after the prerequisite grid has completed
  // (both are no-ops for ordinary launches)
  asm volatile("griddepcontrol.launch_dependents;");
  const int lane = threadIdx.x & 31;
  const int ei = blockIdx.x * 8 + (threadIdx.x >> 5);
  if (ei >= nent) return;
  const GemmEnt e = ents[ei];
  asm volatile("griddepcontrol.wait;" ::: "memory");
  const int ncols = ncols_all > 0 ? ncols_all : e.ncols;
  const int Me = min(M, e.mrows), Ke = min(K, e.krows);
  const int g = lane >> 2, t = lane & 3;
  double acc[2][4][2][2];  // [m tile][n tile][re|im][2]
#pragma unroll
  for (int a = 0; a < 2; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) acc[a][b][0][0] = acc[a][b][0][1] = acc[a][b][1][0] = acc[a][b][1][1] = 0.0;
#pragma unroll
  for (int s = 0; s < S; ++s) {
    const double2* Ab = A + (s == 0 ? e.a0 : e.a1);
    const double2* Bb = B + (s == 0 ? e.b0 : e.b1);
    for (int k0 = 0; k0 < K; k0 += 4) {
      const int k = k0 + t;
      double ar[2], ai[2], br[4], bi[4];
#pragma unroll
      for (int a = 0; a < 2; ++a) {
        const int m = a * 8 + g;
        double2 v = make_double2(0.0, 0.0);
        if (m < M && k < K) {
          if (OP == OP_N) v = Ab[m + (int64_t)k * lda];
          else {
            v = Ab[k + (int64_t)m * lda];
            if (OP == OP_H) v.y = -v.y;
          }
        }
        ar[a] = v.x;
        ai[a] = v.y;
      }
#pragma unroll
      for (int b = 0; b < 4; ++b) {
        const int n = b * 8 + g;
        double2 v = make_double2(0.0, 0.0);
        if (n < ncols && k < Ke) v = Bb[k + (int64_t)n * ldb];
        br[b] = v.x;
        bi[b] = v.y;
      }
#pragma unroll
      for (int a = 0; a < 2; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b) {
          dmma884(acc[a][b][0][0], acc[a][b][0][1], ar[a], br[b]);
          dmma884(acc[a][b][1][0], acc[a][b][1][1], ar[a], bi[b]);
        }
#pragma unroll
      for (int a = 0; a < 2; ++a) {
        const double nai = -ai[a];
#pragma unroll
        for (int b = 0; b < 4; ++b) {
          dmma884(acc[a][b][0][0], acc[a][b][0][1], nai, bi[b]);
          dmma884(acc[a][b][1][0], acc[a][b][1][1], ai[a], br[b]);
        }
      }
    }
  }
  double2* Cb = C + e.c;
#pragma unroll
  for (int a = 0; a < 2; ++a) {
    const int m = a * 8 + g;
    if (m >= Me) continue;
#pragma unroll
    for (int b = 0; b < 4; ++b)
#pragma unroll
      for (int v = 0; v < 2; ++v) {
        const int n = b * 8 + 2 * t + v;
        if (n >= ncols) continue;
        double2 r = make_double2(acc[a][b][0][v], acc[a][b][1][v]);
        double2* p = Cb + m + (int64_t)n * ldc;
        if (accumulate) {
          const double2 o = *p;
          r.x += o.x;
          r.y += o.y;
        }
        *p = r;
      }
  }
}

// Large-k complex128 path on DMMA (mma.sync m8n8k4 f64): one CTA = 4 x WN
// warps computes all M <= 32 MT rows of one output block for a column slab of
// BN = 8 NT WN columns (picked per launch to minimise padded columns: 66
// probe columns run as one 72-wide slab).  op(A_s) and B_s chunks of 16
// along K stream through a 2-stage cp.async ring as raw complex values
// (16-byte granules, zero-filled out of range), the next chunk in flight
// while the current one feeds the DMMAs.  Shared layouts keep fragment reads
// conflict-free: OP_N A [k][m] with pitch = 2 mod 8 granules, OP_T/H A [m][k]
// and B [col][k] with pitch = 4 mod 8.  Complex MAC = 4 real DMMAs.
template <int OP, int S, int MT, int WN, int NT>
__global__ void __launch_bounds__(128 * WN) bgemm_dmma_kernel(const double2* __restrict__ A, int64_t lda,
                                                              const double2* __restrict__ B, int64_t ldb,
                                                              double2* __restrict__ C, int64_t ldc, int M, int K,
                                                              const GemmEnt* __restrict__ ents, int accumulate,
                                                              int ncols_all) {
  constexpr int BM = 32 * MT, BN = 8 * NT * WN, BK = 16, NTHR = 128 * WN;
  constexpr int PA = OP == OP_N ? BM + 2 : BK + 4;  // A pitch (granules)
  constexpr int AEL = OP == OP_N ? BK * PA : BM * PA;
  constexpr int PB = BK + 4;
  constexpr int BEL = BN * PB;
  extern __shared__ __align__(16) double2 dsm_[];
  double2(*As)[AEL] = reinterpret_cast<double2(*)[AEL]>(dsm_);
  double2(*Bs)[BEL] = reinterpret_cast<double2(*)[BEL]>(dsm_ + 2 * AEL);
  asm volatile("griddepcontrol.launch_dependents;");  // see bgemm_dmma_warp_kernel
  const GemmEnt e = ents[blockIdx.x];
  asm volatile("griddepcontrol.wait;" ::: "memory");
  const int ncols = ncols_all > 0 ? ncols_all : e.ncols;
  const int Me = min(M, e.mrows), Ke = min(K, e.krows);
  const int n0 = blockIdx.y * BN;
  if (n0 >= ncols) return;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g = lane >> 2, t = lane & 3;
  const int wm = warp & 3, wn = warp >> 2;  // 4 x WN warps
  const int kch = (K + BK - 1) / BK, nch = S * kch;
  auto cp16 = [](double2* dst, const double2* src, bool ok) {
    const uint32_t d = (uint32_t)__cvta_generic_to_shared(dst);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(d), "l"(src), "r"(ok ? 16 : 0) : "memory");
  };
  auto load_chunk = [&](int c, int buf) {
    const int s = c / kch, k0 = (c % kch) * BK;
    const double2* Ab = A + (s == 0 ? e.a0 : e.a1);
    const double2* Bb = B + (s == 0 ? e.b0 : e.b1);
    for (int idx = tid; idx < BM * BK; idx += NTHR) {
      int m, kk;
      if (OP == OP_N) {
        m = idx % BM;
        kk = idx / BM;
      } else {
        kk = idx % BK;
        m = idx / BK;
      }
      const int gk = k0 + kk;
      const bool ok = m < M && gk < K;
      const double2* src = ok ? (OP == OP_N ? Ab + m + (int64_t)gk * lda : Ab + gk + (int64_t)m * lda) : Ab;
      cp16(&As[buf][OP == OP_N ? kk * PA + m : m * PA + kk], src, ok);
    }
    for (int idx = tid; idx < BK * BN; idx += NTHR) {
      const int kk = idx % BK, cc = idx / BK;
      const int gk = k0 + kk, gc = n0 + cc;
      const bool ok = gk < Ke && gc < ncols;
      cp16(&Bs[buf][cc * PB + kk], ok ? Bb + gk + (int64_t)gc * ldb : Bb, ok);
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  };
  double acc[MT][NT][2][2];
#pragma unroll
  for (int a = 0; a < MT; ++a)
#pragma unroll
    for (int b = 0; b < NT; ++b) acc[a][b][0][0] = acc[a][b][0][1] = acc[a][b][1][0] = acc[a][b][1][1] = 0.0;
  load_chunk(0, 0);
  for (int c = 0; c < nch; ++c) {
    const int buf = c & 1;
    if (c + 1 < nch) {
      load_chunk(c + 1, buf ^ 1);
      asm volatile("cp.async.wait_group 1;" ::: "memory");
    } else {
      asm volatile("cp.async.wait_group 0;" ::: "memory");
    }
    __syncthreads();
    const double2* as = As[buf];
    const double2* bs = Bs[buf];
#pragma unroll
    for (int ks = 0; ks < BK; ks += 4) {
      double ar[MT], ai[MT], br[NT], bi[NT];
#pragma unroll
      for (int a = 0; a < MT; ++a) {
        const int row = wm * 8 * MT + a * 8 + g;
        const double2 v = OP == OP_N ? as[(ks + t) * PA + row] : as[row * PA + ks + t];
        ar[a] = v.x;
        ai[a] = OP == OP_H ? -v.y : v.y;
      }
#pragma unroll
      for (int b = 0; b < NT; ++b) {
        const double2 v = bs[(wn * 8 * NT + b * 8 + g) * PB + ks + t];
        br[b] = v.x;
        bi[b] = v.y;
      }
#pragma unroll
      for (int a = 0; a < MT; ++a)
#pragma unroll
        for (int b = 0; b < NT; ++b) {
          dmma884(acc[a][b][0][0], acc[a][b][0][1], ar[a], br[b]);
          dmma884(acc[a][b][1][0], acc[a][b][1][1], ar[a], bi[b]);
        }
#pragma unroll
      for (int a = 0; a < MT; ++a) {
        const double nai = -ai[a];
#pragma unroll
        for (int b = 0; b < NT; ++b) {
          dmma884(acc[a][b][0][0], acc[a][b][0][1], nai, bi[b]);
          dmma884(acc[a][b][1][0], acc[a][b][1][1], ai[a], br[b]);
        }
      }
    }
    __syncthreads();  // the buffer is refilled by the next iteration's prefetch
  }
  double2* Cb = C + e.c;
#pragma unroll
  for (int a = 0; a < MT; ++a) {
    const int m = wm * 8 * MT + a * 8 + g;
    if (m >= Me) continue;
#pragma unroll
    for (int b = 0; b < NT; ++b)
#pragma unroll
      for (int v = 0; v < 2; ++v) {
        const int gc = n0 + wn * 8 * NT + b * 8 + 2 * t + v;
        if (gc >= ncols) continue;
        double2* p = Cb + m + (int64_t)gc * ldc;
        double2 r = make_double2(acc[a][b][0][v], acc[a][b][1][v]);
        if (accumulate) r = make_double2(p->x + r.x, p->y + r.y);
        *p = r;
      }
  }
}

// complex64 batched GEMM on the FP32 pipe (the recompression at complex64):
// CTA tile 16 TI x 16 TJ complex outputs (TI, TJ in {2, 4}, picked per launch
// for the least padding), 256 threads with TI x TJ outputs each
// (rows ty + 16 i, columns tx + 16 j: broadcast A reads, conflict-free B
// reads), K chunks of 16 through a 2-stage cp.async ring of raw complex
// values (8-byte granules, zero-filled out of range; op(A) conjugated in
// registers).  Complex MAC = 4 FFMA.
template <int OP, int S, int TI, int TJ>
__global__ void __launch_bounds__(256) bgemm_f32_kernel(const float2* __restrict__ A, int64_t lda,
                                                        const float2* __restrict__ B, int64_t ldb,
                                                        float2* __restrict__ C, int64_t ldc, int M, int K,
                                                        const GemmEnt* __restrict__ ents, int accumulate,
                                                        int ncols_all) {
  constexpr int BM = 16 * TI, BN = 16 * TJ, BK = 16;
  // +1 pitch: the transposed 8-byte fills (consecutive k in consecutive
  // threads) land in distinct banks
  __shared__ __align__(16) float2 As[2][BK][BM + 1], Bs[2][BK][BN + 1];
  const GemmEnt e = ents[blockIdx.x];
  const int ncols = ncols_all > 0 ? ncols_all : e.ncols;
  const int Me = min(M, e.mrows), Ke = min(K, e.krows);
  const int n0 = blockIdx.y * BN, m0 = blockIdx.z * BM;
  if (n0 >= ncols || m0 >= Me) return;
  const int tid = threadIdx.x, tx = tid & 15, ty = tid >> 4;
  const int kch = (K + BK - 1) / BK, nch = S * kch;
  auto cp8 = [](float2* dst, const float2* src, bool ok) {
    const uint32_t d = (uint32_t)__cvta_generic_to_shared(dst);
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"(d), "l"(src), "r"(ok ? 8 : 0) : "memory");
  };
  auto load_chunk = [&](int c, int buf) {
    const int s = c / kch, k0 = (c % kch) * BK;
    const float2* Ab = A + (s == 0 ? e.a0 : e.a1);
    const float2* Bb = B + (s == 0 ? e.b0 : e.b1);
#pragma unroll
    for (int q = 0; q < (BM * BK + 255) / 256; ++q) {
      const int idx = tid + q * 256;
      if (idx >= BM * BK) break;
      int m, kk;
      if (OP == OP_N) {
        m = idx % BM;
        kk = idx / BM;
      } else {
        kk = idx % BK;
        m = idx / BK;
      }
      const int gm = m0 + m, gk = k0 + kk;
      const bool ok = gm < M && gk < K;
      cp8(&As[buf][kk][m], ok ? (OP == OP_N ? Ab + gm + (int64_t)gk * lda : Ab + gk + (int64_t)gm * lda) : Ab, ok);
    }
#pragma unroll
    for (int q = 0; q < (BK * BN + 255) / 256; ++q) {
      const int idx = tid + q * 256;
      if (idx >= BK * BN) break;
      const int kk = idx % BK, cc = idx / BK;
      const int gk = k0 + kk, gc = n0 + cc;
      const bool ok = gk < Ke && gc < ncols;
      cp8(&Bs[buf][kk][cc], ok ? Bb + gk + (int64_t)gc * ldb : Bb, ok);
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  };
  float acc[TI][TJ][2];
#pragma unroll
  for (int i = 0; i < TI; ++i)
#pragma unroll
    for (int j = 0; j < TJ; ++j) acc[i][j][0] = acc[i][j][1] = 0.f;
  load_chunk(0, 0);
  for (int c = 0; c < nch; ++c) {
    const int buf = c & 1;
    if (c + 1 < nch) {
      load_chunk(c + 1, buf ^ 1);
      asm volatile("cp.async.wait_group 1;" ::: "memory");
    } else {
      asm volatile("cp.async.wait_group 0;" ::: "memory");
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < BK; ++kk) {
      // rows follow tx (consecutive lanes: consecutive rows -> coalesced C
      // stores, conflict-free A reads), columns follow ty (B reads broadcast)
      float2 a[TI], b[TJ];
#pragma unroll
      for (int i = 0; i < TI; ++i) {
        a[i] = As[buf][kk][tx + 16 * i];
        if (OP == OP_H) a[i].y = -a[i].y;
      }
#pragma unroll
      for (int j = 0; j < TJ; ++j) b[j] = Bs[buf][kk][ty + 16 * j];
#pragma unroll
      for (int i = 0; i < TI; ++i)
#pragma unroll
        for (int j = 0; j < TJ; ++j) {
          acc[i][j][0] = fmaf(a[i].x, b[j].x, acc[i][j][0]);
          acc[i][j][0] = fmaf(-a[i].y, b[j].y, acc[i][j][0]);
          acc[i][j][1] = fmaf(a[i].x, b[j].y, acc[i][j][1]);
          acc[i][j][1] = fmaf(a[i].y, b[j].x, acc[i][j][1]);
        }
    }
    __syncthreads();  // the buffer is refilled by the next iteration's prefetch
  }
  float2* Cb = C + e.c;
#pragma unroll
  for (int i = 0; i < TI; ++i) {
    const int m = m0 + tx + 16 * i;
    if (m >= Me) continue;
#pragma unroll
    for (int j = 0; j < TJ; ++j) {
      const int gc = n0 + ty + 16 * j;
      if (gc >= ncols) continue;
      float2* p = Cb + m + (int64_t)gc * ldc;
      float2 r = make_float2(acc[i][j][0], acc[i][j][1]);
      if (accumulate) r = make_float2(p->x + r.x, p->y + r.y);
      *p = r;
    }
  }
}

// dynamic shared memory of bgemm_dmma_kernel: 2-stage A and B rings
constexpr size_t dmma_smem_bytes(int op, int mt, int wn, int nt) {
  return 16 * 2 *
         ((size_t)(op == OP_N ? 16 * (32 * mt + 2) : 32 * mt * 20) + (size_t)8 * nt * wn * 20);
}

template <typename... KArgs, typename... Args>
void launch_pdl_smem(void (*kern)(KArgs...), dim3 grid, int block, int smem, cudaStream_t stream, bool pdl,
                     Args... args) {
  cudaLaunchConfig_t cfg = {};
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.gridDim = grid;
  cfg.blockDim = dim3(block);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cfg.attrs = pdl ? at : nullptr;
  cfg.numAttrs = pdl ? 1 : 0;
  BFLY_CUDA(cudaLaunchKernelEx(&cfg, kern, static_cast<KArgs>(args)...));
}

// kernel launch with the programmatic-stream-serialization attribute when pdl
template <typename... KArgs, typename... Args>
void launch_pdl(void (*kern)(KArgs...), dim3 grid, int block, cudaStream_t stream, bool pdl, Args... args) {
  cudaLaunchConfig_t cfg = {};
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.gridDim = grid;
  cfg.blockDim = dim3(block);
  cfg.dynamicSmemBytes = 0;
  cfg.stream = stream;
  cfg.attrs = pdl ? at : nullptr;
  cfg.numAttrs = pdl ? 1 : 0;
  BFLY_CUDA(cudaLaunchKernelEx(&cfg, kern, static_cast<KArgs>(args)...));
}
}  // namespace

template <typename R>
void launch_bgemm(Ctx* c, int op, int M, int K, int S, const cx<R>* A, int64_t lda, const cx<R>* B, int64_t ldb,
                  cx<R>* C, int64_t ldc, const GemmEnt* ents, int nent, int max_ncols, bool accumulate,
                  int ncols_all, bool pdl, L2Prefetch pf) {
  if (nent <= 0 || M <= 0 || max_ncols <= 0) return;
  const int kcols = ncols_all > 0 ? ncols_all : max_ncols;
  const size_t small_smem = sizeof(cx<R>) * (size_t)S * ((size_t)K * (M + 1) + (size_t)K * kcols);
  static const bool no_stage = std::getenv("BFLY_NO_STAGE_GEMM") != nullptr;
  static const int dmma_mink = std::getenv("BFLY_DMMA_MINK") ? std::atoi(std::getenv("BFLY_DMMA_MINK")) : 8;
  const bool dmma_cols = std::is_same<R, double>::value && kcols >= dmma_mink;
  // complex128 with 8..32 columns: the same staged kernel with DMMA tiles
  // (factor image only in shared memory)
  // (large blocks, M K >= 1024 -- the config-4 leaf-64 rank-32 butterfly: up to
  // 16 columns; wider applies run faster on the block DMMA GEMM, config-4
  // k = 32: 1.48 vs 1.81 ms.  Config 2's blocks are <= 512 entries)
  const bool big_blocks = (int64_t)M * K >= 1024;
  const bool stage_dm = dmma_cols && kcols <= (big_blocks ? 16 : 32);
  const size_t stage_smem = 16 + sizeof(cx<R>) * (size_t)stage_group_elems(op, M, K, S, stage_dm ? 0 : kcols);
  if (pdl && !no_stage && (dmma_cols ? stage_dm : kcols <= 16) && ncols_all > 0 && K > 0 &&
      stage_smem <= 96 * 1024) {
    KTimer timer(c, "bgemm_stage", 8.0 * M * K * S * (double)nent * kcols,
                 sizeof(cx<R>) * ((double)nent * S * (M * (double)K + K * kcols) + (double)nent * M * kcols));
    static const int wpe_env = std::getenv("BFLY_STAGE_WPE") ? std::atoi(std::getenv("BFLY_STAGE_WPE")) : 0;
    // DMMA groups: 2 warps up to 16 columns, 4 beyond (measured on the
    // config-2 apply: fewer threads per entry keep ~2 stage grids resident)
    // (large blocks: 4 warps, config-4 k = 8 / 16: 0.79 -> 0.74 / 1.25 -> 1.10 ms;
    // config 2's blocks keep 2)
    const int wpe = wpe_env > 0 ? std::min(wpe_env, 8)
                    : stage_dm ? (kcols <= 16 && !big_blocks ? 2 : 4)
                    : kcols <= 2 ? 1 : kcols <= 8 ? 2 : 4;
    const size_t grp_smem = stage_smem;
    static const int epb_env = std::getenv("BFLY_STAGE_EPB") ? std::atoi(std::getenv("BFLY_STAGE_EPB")) : 0;
    // entries per CTA for single-warp groups: measured on the config-2 apply
    // (k=1: 2 per CTA, k=2: 1 per CTA)
    int epb = wpe == 1 ? (epb_env > 0 ? std::min(epb_env, 8) : (kcols == 1 ? 2 : 1)) : 1;
    while (epb > 1 && epb * grp_smem > 100 * 1024) epb /= 2;
    cudaLaunchConfig_t cfg = {};
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.gridDim = dim3((unsigned)ceil_div((int64_t)nent, (int64_t)epb));
    cfg.blockDim = dim3(32 * wpe * epb);
    cfg.dynamicSmemBytes = epb * grp_smem;
    cfg.stream = c->stream;
    cfg.attrs = at;
    cfg.numAttrs = 1;
#define BST(OPV, SV)                                                                                        \
  do {                                                                                                      \
    auto kern = bgemm_stage_kernel<R, OPV, SV, false>;                                                      \
    if constexpr (std::is_same<R, double>::value)                                                           \
      if (stage_dm) kern = bgemm_stage_kernel<R, OPV, SV, true>;                                            \
    /* per device (a process may hold contexts on several GPUs); first use is eager, never in capture */  \
    static uint64_t attr_set[2] = {0, 0};                                                                   \
    if (!((attr_set[stage_dm] >> (c->device & 63)) & 1)) {                                                  \
      BFLY_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));        \
      attr_set[stage_dm] |= uint64_t(1) << (c->device & 63);                                                \
    }                                                                                                       \
    BFLY_CUDA(cudaLaunchKernelEx(&cfg, kern, A, lda, B, ldb, C, ldc, M, K, ents, nent, (int)accumulate, kcols, wpe, pf)); \
  } while (0)
    if (S == 1) {
      if (op == OP_N) BST(OP_N, 1);
      else if (op == OP_T) BST(OP_T, 1);
      else BST(OP_H, 1);
    } else {
      if (op == OP_N) BST(OP_N, 2);
      else if (op == OP_T) BST(OP_T, 2);
      else BST(OP_H, 2);
    }
#undef BST
    BFLY_LAUNCH_CHECK("bgemm_stage");
    return;
  }
  if (!dmma_cols && kcols <= 16 && K > 0 && small_smem <= 96 * 1024 && nent <= 0x7fffffff) {
    KTimer timer(c, "bgemm_small", 8.0 * M * K * S * (double)nent * kcols,
                 sizeof(cx<R>) * ((double)nent * S * (M * (double)K + K * kcols) + (double)nent * M * kcols));
#define BGS(OPV, SV)                                                                                           \
  do {                                                                                                         \
    auto kern = bgemm_small_kernel<R, OPV, SV>;                                                                \
    static uint64_t attr_96k = 0; /* per device: set once per kernel, never during graph capture */          \
    if (small_smem > 48 * 1024 && !((attr_96k >> (c->device & 63)) & 1)) {                                     \
      BFLY_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 96 * 1024));           \
      attr_96k |= uint64_t(1) << (c->device & 63);                                                             \
    }                                                                                                          \
    if (pdl) {                                                                                                 \
      cudaLaunchConfig_t cfg = {};                                                                             \
      cudaLaunchAttribute at[1];                                                                               \
      at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;                                          \
      at[0].val.programmaticStreamSerializationAllowed = 1;                                                    \
      cfg.gridDim = dim3(nent);                                                                                \
      cfg.blockDim = dim3(128);                                                                                \
      cfg.dynamicSmemBytes = small_smem;                                                                       \
      cfg.stream = c->stream;                                                                                  \
      cfg.attrs = at;                                                                                          \
      cfg.numAttrs = 1;                                                                                        \
      BFLY_CUDA(cudaLaunchKernelEx(&cfg, kern, A, lda, B, ldb, C, ldc, M, K, ents, (int)accumulate, ncols_all)); \
    } else {                                                                                                   \
      kern<<<nent, 128, small_smem, c->stream>>>(A, lda, B, ldb, C, ldc, M, K, ents, accumulate, ncols_all);   \
    }                                                                                                          \
  } while (0)
    if (S == 1) {
      if (op == OP_N) BGS(OP_N, 1);
      else if (op == OP_T) BGS(OP_T, 1);
      else BGS(OP_H, 1);
    } else {
      if (op == OP_N) BGS(OP_N, 2);
      else if (op == OP_T) BGS(OP_T, 2);
      else BGS(OP_H, 2);
    }
#undef BGS
    BFLY_LAUNCH_CHECK("bgemm_small");
    return;
  }
  if constexpr (std::is_same<R, double>::value) {
    static const bool no_dmma = std::getenv("BFLY_NO_DMMA_GEMM") != nullptr;
    static const bool no_warp = std::getenv("BFLY_NO_WARP_GEMM") != nullptr;
    if (!no_dmma && !no_warp && dmma_cols && max_ncols <= 32 && M <= 16 && K > 0) {
      static const char* wnames[3][2] = {{"bgemm_warp_N1", "bgemm_warp_N2"},
                                         {"bgemm_warp_T1", "bgemm_warp_T2"},
                                         {"bgemm_warp_H1", "bgemm_warp_H2"}};
      KTimer timer(c, wnames[op][S - 1], 8.0 * M * K * S * (double)nent * kcols,
                   sizeof(cx<R>) * ((double)nent * S * (M * (double)K + K * kcols) + (double)nent * M * kcols));
      const unsigned grid = (unsigned)ceil_div((int64_t)nent, (int64_t)8);
#define BW(OPV, SV)                                                                                          \
  launch_pdl(bgemm_dmma_warp_kernel<OPV, SV>, dim3(grid), 256, c->stream, pdl, A, lda, B, ldb, C, ldc, M, K, ents, nent, \
                                                               accumulate, ncols_all)
      if (S == 1) {
        if (op == OP_N) BW(OP_N, 1);
        else if (op == OP_T) BW(OP_T, 1);
        else BW(OP_H, 1);
      } else {
        if (op == OP_N) BW(OP_N, 2);
        else if (op == OP_T) BW(OP_T, 2);
        else BW(OP_H, 2);
      }
#undef BW
      BFLY_LAUNCH_CHECK("bgemm_warp");
      return;
    }
    if (!no_dmma && dmma_cols && M <= 64 && K > 0) {
      // column slab: the (WN, NT) shape with the fewest padded columns
      static const int shapes[4][2] = {{2, 4}, {3, 3}, {2, 3}, {3, 4}};
      int best = 0;
      int64_t best_cols = INT64_MAX;
      for (int i = 0; i < 4; ++i) {
        const int bn = 8 * shapes[i][0] * shapes[i][1];
        const int64_t cols = ceil_div((int64_t)max_ncols, (int64_t)bn) * bn;
        if (cols < best_cols || (cols == best_cols && bn > 8 * shapes[best][0] * shapes[best][1])) {
          best = i;
          best_cols = cols;
        }
      }
      const int WNv = shapes[best][0], NTv = shapes[best][1], BNv = 8 * WNv * NTv;
      const unsigned gy = (unsigned)ceil_div(max_ncols, BNv);
      if (gy > 65535) fail(PRECONDITION, "bgemm: grid too large");
      dim3 grid(nent, gy);
      static const char* names[3][2][2] = {{{"bgemm_dmma_N1_m32", "bgemm_dmma_N1_m64"}, {"bgemm_dmma_N2_m32", "bgemm_dmma_N2_m64"}},
                                           {{"bgemm_dmma_T1_m32", "bgemm_dmma_T1_m64"}, {"bgemm_dmma_T2_m32", "bgemm_dmma_T2_m64"}},
                                           {{"bgemm_dmma_H1_m32", "bgemm_dmma_H1_m64"}, {"bgemm_dmma_H2_m32", "bgemm_dmma_H2_m64"}}};
      KTimer timer(c, names[op][S - 1][M > 32], 8.0 * M * K * S * (double)nent * kcols,
                   sizeof(cx<R>) * ((double)nent * S * (M * (double)K + K * kcols) + (double)nent * M * kcols));
#define BDS(OPV, SV, MTV, WNV, NTV)                                                                             \
  do {                                                                                                          \
    auto kern = bgemm_dmma_kernel<OPV, SV, MTV, WNV, NTV>;                                                      \
    const int smem = (int)dmma_smem_bytes(OPV, MTV, WNV, NTV);                                                  \
    static uint64_t attr_set = 0; /* per device; first use is eager (never inside graph capture) */           \
    if (!((attr_set >> (c->device & 63)) & 1)) {                                                                \
      BFLY_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));                  \
      attr_set |= uint64_t(1) << (c->device & 63);                                                              \
    }                                                                                                           \
    launch_pdl_smem(kern, grid, 128 * WNV, smem, c->stream, pdl, A, lda, B, ldb, C, ldc, M, K, ents, accumulate, \
                    ncols_all);                                                                                 \
  } while (0)
#define BD(OPV, SV, MTV)                         \
  do {                                           \
    switch (best) {                              \
      case 0: BDS(OPV, SV, MTV, 2, 4); break;    \
      case 1: BDS(OPV, SV, MTV, 3, 3); break;    \
      case 2: BDS(OPV, SV, MTV, 2, 3); break;    \
      default: BDS(OPV, SV, MTV, 3, 4); break;   \
    }                                            \
  } while (0)
#define BD_OP(SV, MTV)                   \
  do {                                   \
    if (op == OP_N) BD(OP_N, SV, MTV);   \
    else if (op == OP_T) BD(OP_T, SV, MTV); \
    else BD(OP_H, SV, MTV);              \
  } while (0)
      if (M <= 32) {
        if (S == 1) BD_OP(1, 1);
        else BD_OP(2, 1);
      } else {
        if (S == 1) BD_OP(1, 2);
        else BD_OP(2, 2);
      }
#undef BD_OP
#undef BD
#undef BDS
      BFLY_LAUNCH_CHECK("bgemm_dmma");
      return;
    }
  }
  if constexpr (std::is_same<R, float>::value) {
    static const bool no_f32 = std::getenv("BFLY_NO_F32_GEMM") != nullptr;
    if (!no_f32 && K > 0) {
      // tile shape with the least padded output area (ties: the larger tile)
      static const int f32_env = std::getenv("BFLY_F32_TILE") ? std::atoi(std::getenv("BFLY_F32_TILE")) : -1;
      // shapes (TI, TJ): (2,2) (2,4) (4,2) (4,4) (2,8); BM = 16 TI, BN = 16 TJ
      static const int tshape[5][2] = {{2, 2}, {2, 4}, {4, 2}, {4, 4}, {2, 8}};
      int best = 0;
      int64_t best_area = INT64_MAX;
      for (int i = 0; i < 5; ++i) {
        const int bm = 16 * tshape[i][0], bn = 16 * tshape[i][1];
        const int64_t area = ceil_div((int64_t)M, (int64_t)bm) * bm * ceil_div((int64_t)max_ncols, (int64_t)bn) * bn;
        if (area < best_area || (area == best_area)) {
          best = i;
          best_area = area;
        }
      }
      if (f32_env >= 0 && f32_env < 5) best = f32_env;
      const int BMv = 16 * tshape[best][0], BNv = 16 * tshape[best][1];
      BFLY_HOST_TRACE("bgemm_f32 M %d K %d S %d ncols %lld nent %d tile %dx%d op %d", M, K, S, (long long)max_ncols, nent,
                      BMv, BNv, op);
      dim3 grid(nent, (unsigned)ceil_div(max_ncols, BNv), (unsigned)ceil_div(M, BMv));
      if (grid.y > 65535 || grid.z > 65535) fail(PRECONDITION, "bgemm: grid too large");
      const double nc = ncols_all > 0 ? ncols_all : max_ncols;
      KTimer timer(c, "bgemm_f32", 8.0 * M * K * S * (double)nent * nc,
                   sizeof(cx<R>) * ((double)nent * S * (M * (double)K + K * nc) + (double)nent * M * nc));
#define BFT(OPV, SV, TIV, TJV)                                                                          \
  bgemm_f32_kernel<OPV, SV, TIV, TJV><<<grid, 256, 0, c->stream>>>(A, lda, B, ldb, C, ldc, M, K, ents, \
                                                                   (int)accumulate, ncols_all)
#define BF(OPV, SV)                          \
  do {                                       \
    switch (best) {                          \
      case 0: BFT(OPV, SV, 2, 2); break;     \
      case 1: BFT(OPV, SV, 2, 4); break;     \
      case 2: BFT(OPV, SV, 4, 2); break;     \
      case 3: BFT(OPV, SV, 4, 4); break;     \
      default: BFT(OPV, SV, 2, 8); break;    \
    }                                        \
  } while (0)
      if (S == 1) {
        if (op == OP_N) BF(OP_N, 1);
        else if (op == OP_T) BF(OP_T, 1);
        else BF(OP_H, 1);
      } else {
        if (op == OP_N) BF(OP_N, 2);
        else if (op == OP_T) BF(OP_T, 2);
        else BF(OP_H, 2);
      }
#undef BF
#undef BFT
      BFLY_LAUNCH_CHECK("bgemm_f32");
      return;
    }
  }
  // K == 0: the product is an exact zero block
  dim3 grid(nent, (unsigned)ceil_div(max_ncols, TN), (unsigned)ceil_div(M, TM));
  if (grid.y > 65535 || grid.z > 65535) fail(PRECONDITION, "bgemm: grid too large");
  const double nc = ncols_all > 0 ? ncols_all : max_ncols;
  KTimer timer(c, "bgemm", 8.0 * M * K * S * (double)nent * nc,
               sizeof(cx<R>) * ((double)nent * S * (M * (double)K + K * nc) + (double)nent * M * nc));
#define BG(OPV, SV) bgemm_kernel<R, OPV, SV><<<grid, 256, 0, c->stream>>>(A, lda, B, ldb, C, ldc, M, K, ents, accumulate, ncols_all)
  if (S == 1) {
    if (op == OP_N) BG(OP_N, 1);
    else if (op == OP_T) BG(OP_T, 1);
    else BG(OP_H, 1);
  } else {
    if (op == OP_N) BG(OP_N, 2);
    else if (op == OP_T) BG(OP_T, 2);
    else BG(OP_H, 2);
  }
#undef BG
  BFLY_LAUNCH_CHECK("bgemm");
}

template void launch_bgemm<double>(Ctx*, int, int, int, int, const double2*, int64_t, const double2*, int64_t, double2*,
                                   int64_t, const GemmEnt*, int, int, bool, int, bool, L2Prefetch);
template void launch_bgemm<float>(Ctx*, int, int, int, int, const float2*, int64_t, const float2*, int64_t, float2*,
                                  int64_t, const GemmEnt*, int, int, bool, int, bool, L2Prefetch);

#ifdef BFLY_STAGE_TRACE
extern "C" __attribute__((visibility("default"))) int bfly_debug_stage_trace(unsigned long long* out, int reset) {
  if (reset) {
    unsigned long long init[64][10];
    for (auto& r : init) {
      r[0] = r[2] = r[6] = r[9] = ~0ull;
      r[1] = r[3] = r[4] = r[5] = r[7] = r[8] = 0;
    }
    return (int)cudaMemcpyToSymbol(g_stage_trace, init, sizeof(init));
  }
  return (int)cudaMemcpyFromSymbol(out, g_stage_trace, sizeof(g_stage_trace));
}
#endif
}  // namespace bfly
