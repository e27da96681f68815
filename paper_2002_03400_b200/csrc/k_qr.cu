// k_qr.cu -- K5 batched truncated column-pivoted QR and K6 batched core fit.
//
// K5 reproduces pivoted_qr_truncate (reference linalg.hpp:62-80) as computed
// by Eigen::ColPivHouseholderQR + householderQ(): max-updated-norm pivoting
// (first index on ties), Householder beta = -sign(Re c0)||x||,
// tau = conj((beta-c0)/beta), LAWN-176 norm downdating with direct
// recomputation at sqrt(eps), truncation |R_kk| > eps_t |R_00|.  The
// factorization stops at the first rejected pivot (later steps cannot change
// the kept columns), and Q(:,0:k) is formed in place (LAPACK ung2r order).
// One CTA (8 warps) per block; the block lives in shared memory.
//
// K6 is core_block + pinv_solve (reconstruct.hpp:125-138, linalg.hpp:128-139):
// B = (Q^H z) pinv(coeff), pinv through a one-sided Jacobi SVD of coeff^H
// (parallel round-robin pair ordering), singular values <= 1e-12 smax dropped.
#include <algorithm>
#include <cfloat>
#include <cstdlib>

#include "kernels.cuh"

namespace bfly {

namespace {

// threads per block by block size (measured): 128 up to ~32 x 34 (config 2
// leaves and transfer blocks), 256 for butterfly-sized blocks up to 128 x 128
// (config 4), 512 for saturated ones (more warps on the per-column work)
constexpr int QR_TINY = 128, QR_SMALL = 256, QR_BIG = 512;

// four warp sums at once, every lane receiving all four: the halves of the
// warp trade the values they do not keep (4 -> 2 -> 1 value per lane), three
// more butterfly steps, four broadcasts: 10 shuffles instead of 20
template <typename T> __device__ __forceinline__ void warp_sum4(T& a, T& b, T& c, T& d) {
  const int lane = threadIdx.x & 31;
  const bool hi = lane & 16;
  T k0 = hi ? c : a, k1 = hi ? d : b;
  k0 += __shfl_xor_sync(0xffffffffu, hi ? a : c, 16);
  k1 += __shfl_xor_sync(0xffffffffu, hi ? b : d, 16);
  const bool h8 = lane & 8;
  T k = h8 ? k1 : k0;
  k += __shfl_xor_sync(0xffffffffu, h8 ? k0 : k1, 8);
  k += __shfl_xor_sync(0xffffffffu, k, 4);
  k += __shfl_xor_sync(0xffffffffu, k, 2);
  k += __shfl_xor_sync(0xffffffffu, k, 1);
  a = __shfl_sync(0xffffffffu, k, 0);
  b = __shfl_sync(0xffffffffu, k, 8);
  c = __shfl_sync(0xffffffffu, k, 16);
  d = __shfl_sync(0xffffffffu, k, 24);
}

template <typename T> __device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

template <typename R> struct QrTraits;
template <> struct QrTraits<double> {
  static constexpr double tiny = DBL_MIN;
  static constexpr double sqrt_eps = 1.4901161193847656e-08;  // sqrt(DBL_EPSILON)
  static constexpr double jacobi_tol = 1e-15;
};
template <> struct QrTraits<float> {
  static constexpr float tiny = FLT_MIN;
  static constexpr float sqrt_eps = 3.4526698e-04f;  // sqrt(FLT_EPSILON)
  static constexpr float jacobi_tol = 1e-7f;
};

template <typename R, int QR_THREADS>
__global__ void __launch_bounds__(QR_THREADS) cpqr_kernel(const cx<R>* __restrict__ src, int64_t ld_src,
                                                          cx<R>* __restrict__ dst, int64_t ld_dst, int cap,
                                                          const QrEnt* __restrict__ ents, int32_t* ranks, double eps_t,
                                                          int zld, cx<R>* zglobal, int64_t zstride, double* margins) {
  using V = cx<R>;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const QrEnt e = ents[blockIdx.x];
  const int r = e.r1 + e.r2, w = e.cols;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  // the block lives in shared memory, or (oversized blocks) in a global
  // scratch slice with the same code path
  V* Z = zglobal ? zglobal + blockIdx.x * zstride : reinterpret_cast<V*>(smem_raw);  // zld x w
  R* nu = zglobal ? reinterpret_cast<R*>(smem_raw) : reinterpret_cast<R*>(Z + (size_t)zld * w);
  R* nd = nu + w;
  V* tau = reinterpret_cast<V*>(nd + w);
  __shared__ int s_big;
  __shared__ int s_k;
  __shared__ R s_total;

  V* out = dst + e.dst;
  if (r == 0 || w == 0) {
    for (int64_t i = threadIdx.x; i < ld_dst * cap; i += QR_THREADS) out[i] = mkc<R>(0, 0);
    if (threadIdx.x == 0) {
      ranks[e.rank_slot] = 0;
      if (margins) margins[e.rank_slot] = HUGE_VAL;
    }
    return;
  }
  // load the compact block
  for (int idx = threadIdx.x; idx < r * w; idx += QR_THREADS) {
    int i = idx % r, c = idx / r;
    const V* s = src + e.src + (int64_t)c * ld_src;
    Z[i + c * zld] = i < e.r1 ? s[i] : s[e.src_gap + (i - e.r1)];
  }
  __syncthreads();
  for (int c = warp; c < w; c += (QR_THREADS / 32)) {
    R s = 0;
    for (int i = lane; i < r; i += 32) s += cabs2(Z[i + c * zld]);
    s = warp_sum(s);
    if (lane == 0) nu[c] = nd[c] = sqrt(s);
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    R t = 0;
    for (int c = 0; c < w; ++c) t += nu[c] * nu[c];
    s_total = t;
  }
  __syncthreads();
  if (s_total == R(0)) {  // all-zero input: rank 0 (linalg.hpp:67-71)
    for (int64_t i = threadIdx.x; i < ld_dst * cap; i += QR_THREADS) out[i] = mkc<R>(0, 0);
    if (threadIdx.x == 0) {
      ranks[e.rank_slot] = 0;
      if (margins) margins[e.rank_slot] = HUGE_VAL;
    }
    return;
  }
  const int kmax = min(r, w);
  R head = 0, last_kept = 0, first_dropped = -1;
  int k = kmax;
  for (int j = 0; j < kmax; ++j) {
    // ---- pivot: first column with the largest updated norm
    if (warp == 0) {
      R best = -1;
      int bi = w;
      for (int c = j + lane; c < w; c += 32)
        if (nu[c] > best) { best = nu[c]; bi = c; }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        R ob = __shfl_xor_sync(0xffffffffu, best, o);
        int oi = __shfl_xor_sync(0xffffffffu, bi, o);
        if (ob > best || (ob == best && oi < bi)) { best = ob; bi = oi; }
      }
      if (lane == 0) s_big = bi;
    }
    __syncthreads();
    const int big = s_big;
    if (big != j) {
      for (int i = threadIdx.x; i < r; i += QR_THREADS) {
        V t = Z[i + j * zld];
        Z[i + j * zld] = Z[i + big * zld];
        Z[i + big * zld] = t;
      }
      if (threadIdx.x == 0) {
        R t = nu[j]; nu[j] = nu[big]; nu[big] = t;
        t = nd[j]; nd[j] = nd[big]; nd[big] = t;
      }
    }
    __syncthreads();
    // ---- Householder reflector of column j (makeHouseholderInPlace)
    if (warp == 0) {
      R tail = 0;
      for (int i = j + 1 + lane; i < r; i += 32) tail += cabs2(Z[i + j * zld]);
      tail = warp_sum(tail);
      V c0 = Z[j + j * zld];
      V t;
      R beta;
      bool trivial = tail <= QrTraits<R>::tiny && c0.y * c0.y <= QrTraits<R>::tiny;
      if (trivial) {
        t = mkc<R>(0, 0);
        beta = c0.x;
        for (int i = j + 1 + lane; i < r; i += 32) Z[i + j * zld] = mkc<R>(0, 0);
      } else {
        beta = sqrt(cabs2(c0) + tail);
        if (c0.x >= R(0)) beta = -beta;
        V d = mkc<R>(c0.x - beta, c0.y);
        // 1/d
        R dn = cabs2(d);
        V inv = mkc<R>(d.x / dn, -d.y / dn);
        for (int i = j + 1 + lane; i < r; i += 32) Z[i + j * zld] = cmul(Z[i + j * zld], inv);
        // tau = conj((beta - c0) / beta)
        t = mkc<R>((beta - c0.x) / beta, c0.y / beta);
      }
      if (lane == 0) {
        Z[j + j * zld] = mkc<R>(beta, 0);
        tau[j] = t;
      }
    }
    __syncthreads();
    const R absb = fabs(Z[j + j * zld].x);
    if (j == 0) head = absb;
    if (!(absb > R(eps_t) * head)) {
      k = j;
      first_dropped = absb;
      break;
    }
    last_kept = absb;
    // ---- apply H_j = I - tau v v^H to the trailing columns; downdate norms
    const V tj = tau[j];
    for (int c = j + 1 + warp; c < w; c += (QR_THREADS / 32)) {
      V dot = mkc<R>(0, 0);
      for (int i = j + 1 + lane; i < r; i += 32) cfma_conj(dot, Z[i + j * zld], Z[i + c * zld]);
      dot.x = warp_sum(dot.x);
      dot.y = warp_sum(dot.y);
      dot = cadd(dot, Z[j + c * zld]);
      V tt = cmul(tj, dot);
      for (int i = j + 1 + lane; i < r; i += 32) {
        V z = Z[i + c * zld];
        V v = Z[i + j * zld];
        Z[i + c * zld] = csub(z, cmul(v, tt));
      }
      V top = csub(Z[j + c * zld], tt);
      __syncwarp();
      if (lane == 0) Z[j + c * zld] = top;
      // LAWN-176 downdate (uniform across the warp)
      const R nuc = nu[c], ndc = nd[c];
      __syncwarp();
      if (nuc != R(0)) {
        R temp = sqrt(cabs2(top)) / nuc;
        temp = (R(1) + temp) * (R(1) - temp);
        if (temp < R(0)) temp = 0;
        R ratio = nuc / ndc;
        R temp2 = temp * ratio * ratio;
        if (temp2 <= QrTraits<R>::sqrt_eps) {
          R s = 0;
          for (int i = j + 1 + lane; i < r; i += 32) s += cabs2(Z[i + c * zld]);
          s = warp_sum(s);
          if (lane == 0) nu[c] = nd[c] = sqrt(s);
        } else if (lane == 0) {
          nu[c] = nuc * sqrt(temp);
        }
      }
      __syncwarp();
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    s_k = k;
    // rank margin at the cut (diagnostic): min(|R_{k-1}|/thr - 1, 1 - |R_k|/thr), thr = eps |R_00|
    if (margins) {
      const double thr = eps_t * (double)head;
      double m = (double)last_kept / thr - 1.0;
      if (first_dropped >= R(0)) m = fmin(m, 1.0 - (double)first_dropped / thr);
      margins[e.rank_slot] = m;
    }
  }
  __syncthreads();
  k = s_k;
  // ---- form Q(:, 0:k) in place: Q = H_0 ... H_{k-1} [I_k; 0], H_i = I - conj(tau_i) v v^H
  for (int i = k - 1; i >= 0; --i) {
    const V tq = cconj(tau[i]);
    for (int c = i + 1 + warp; c < k; c += (QR_THREADS / 32)) {
      V dot = Z[i + c * zld];  // v_i = 1
      V part = mkc<R>(0, 0);
      for (int q = i + 1 + lane; q < r; q += 32) cfma_conj(part, Z[q + i * zld], Z[q + c * zld]);
      part.x = warp_sum(part.x);
      part.y = warp_sum(part.y);
      dot = cadd(dot, part);
      V tt = cmul(tq, dot);
      for (int q = i + 1 + lane; q < r; q += 32) Z[q + c * zld] = csub(Z[q + c * zld], cmul(Z[q + i * zld], tt));
      __syncwarp();
      if (lane == 0) Z[i + c * zld] = csub(Z[i + c * zld], tt);
    }
    __syncthreads();
    for (int q = i + 1 + threadIdx.x; q < r; q += QR_THREADS) {
      V v = Z[q + i * zld];
      V nt = mkc<R>(-tq.x, -tq.y);
      Z[q + i * zld] = cmul(nt, v);
    }
    if (threadIdx.x == 0) Z[i + i * zld] = mkc<R>(R(1) - tq.x, -tq.y);
    for (int q = threadIdx.x; q < i; q += QR_THREADS) Z[q + i * zld] = mkc<R>(0, 0);
    __syncthreads();
  }
  // ---- write the padded-stacked Q block
  for (int64_t idx = threadIdx.x; idx < ld_dst * cap; idx += QR_THREADS) {
    int d = (int)(idx % ld_dst), c = (int)(idx / ld_dst);
    V v = mkc<R>(0, 0);
    if (c < k) {
      if (d < e.r1) v = Z[d + c * zld];
      else if (d >= e.dst_gap && d < e.dst_gap + e.r2) v = Z[e.r1 + (d - e.dst_gap) + c * zld];
    }
    out[idx] = v;
  }
  if (threadIdx.x == 0) ranks[e.rank_slot] = k;
}

// ------------------------------------------- K5, one or two warps per block
// The same factorization for blocks of at most 64 rows and 96 columns
// (config 2's leaves and transfer blocks, config 4's 64 x 66 blocks, config
// 1's transfer blocks) with NW = 1 or 2 warps per block and no wide barriers:
// the Householder vector of column j is built with thread = row (warp 0; the
// other warp waits at a 64-thread barrier); the trailing update, the norm
// downdates and the Q formation run with thread = column (each thread sums
// over the rows of its own column, so no shuffle reductions).  The block sits
// in shared memory with an odd column stride (33 or 65 complex = 1 mod 8
// 16-byte groups: a quarter-warp's column accesses hit 8 distinct bank
// groups).  (The 128 / 256-thread CTA version spent ~5 __syncthreads per
// pivot step: 260 us per config-2 launch, 3.7 ms per config-4 launch.)

// sum_{i in [i0, i1)} conj(a_i) b_i with four independent partial sums (the
// FP64 FMA latency chain of one running sum dominated the step)
template <typename V>
__device__ __forceinline__ V dot_conj(const V* __restrict__ a, const V* __restrict__ b, int i0, int i1) {
  V s0 = mkc<decltype(a->x)>(0, 0), s1 = s0, s2 = s0, s3 = s0;
  int i = i0;
  for (; i + 3 < i1; i += 4) {
    cfma_conj(s0, a[i], b[i]);
    cfma_conj(s1, a[i + 1], b[i + 1]);
    cfma_conj(s2, a[i + 2], b[i + 2]);
    cfma_conj(s3, a[i + 3], b[i + 3]);
  }
  for (; i < i1; ++i) cfma_conj(s0, a[i], b[i]);
  return cadd(cadd(s0, s1), cadd(s2, s3));
}

// NH = 2 (four warps, blocks of 33..64 rows): two lanes per trailing column,
// each summing / updating half of the rows (lane >> 4 picks the half, so a
// quarter-warp still walks 8 consecutive columns: conflict-free); the partial
// dots meet through one shuffle.  64 x 66 blocks (config 4): 46.3 -> 39.7 ms of
// CPQR per construction (profiles/r02_cpqr_nh2.txt).  A register-resident
// variant (a column in the registers of four lanes, reflector broadcast from
// shared memory, two barriers per step) measured 111 ms: 2.9x the
// instructions (row selects, per-quad redundant downdates) at one block per SM.
template <typename R, int NW, int NH>
__global__ void __launch_bounds__(32 * NW) cpqr_warp_kernel(const cx<R>* __restrict__ src, int64_t ld_src,
                                                            cx<R>* __restrict__ dst, int64_t ld_dst, int cap,
                                                            const QrEnt* __restrict__ ents, int32_t* ranks,
                                                            double eps_t, double* margins) {
  using V = cx<R>;
  constexpr int NT = 32 * NW;
  constexpr int LD = NW == 1 ? 33 : 65;  // column stride (complex), 1 mod 8
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const QrEnt e = ents[blockIdx.x];
  const int r = e.r1 + e.r2, w = e.cols;
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  V* Z = reinterpret_cast<V*>(smem_raw);  // LD x w
  R* nu = reinterpret_cast<R*>(Z + (size_t)LD * w);
  R* nd = nu + w;
  V* tau = reinterpret_cast<V*>(nd + w);
  __shared__ R s_red[NW];
  __shared__ int s_idx[NW];
  // trailing-column work split: CP columns per pass, lane half hh of NH
  constexpr int CP = NT / NH;
  const int ccol = NH == 1 ? t : warp * 16 + (lane & 15);
  const int hh = NH == 1 ? 0 : lane >> 4;
  __shared__ V s_beta_tau[2];  // (beta, 0), tau of the current step
  V* out = dst + e.dst;
  auto sync = [&]() {
    if (NW == 1)
      __syncwarp();
    else
      asm volatile("bar.sync 1, %0;" ::"n"(NT) : "memory");
  };
  auto zero_out = [&]() {
    for (int64_t i = t; i < ld_dst * cap; i += NT) out[i] = mkc<R>(0, 0);
    if (t == 0) {
      ranks[e.rank_slot] = 0;
      if (margins) margins[e.rank_slot] = HUGE_VAL;
    }
  };
  if (r == 0 || w == 0) {
    zero_out();
    return;
  }
  // load the compact block (threads sweep the elements column by column: every
  // thread busy and the loads independent -- with thread = row only r of the NT
  // threads loaded, one dependent-latency round per column) and the column norms
  // (thread = column)
  if (NW == 1) {
    for (int c = 0; c < w; ++c) {
      const V* sc = src + e.src + (int64_t)c * ld_src;
      for (int i = t; i < r; i += NT) Z[i + c * LD] = i < e.r1 ? sc[i] : sc[e.src_gap + (i - e.r1)];
    }
  } else {
    const int tot = r * w;
#pragma unroll 4
    for (int idx = t; idx < tot; idx += NT) {
      const int c = idx / r, i = idx - c * r;
      const V* sc = src + e.src + (int64_t)c * ld_src;
      Z[i + c * LD] = i < e.r1 ? sc[i] : sc[e.src_gap + (i - e.r1)];
    }
  }
  sync();
  for (int c = t; c < w; c += NT) {
    R s = 0;
    for (int i = 0; i < r; ++i) s += cabs2(Z[i + c * LD]);
    nu[c] = nd[c] = sqrt(s);
  }
  sync();
  R total = 0;
  for (int c = 0; c < w; ++c) total += nu[c] * nu[c];  // uniform
  if (total == R(0)) {  // all-zero input: rank 0 (linalg.hpp:67-71)
    zero_out();
    return;
  }
  const int kmax = min(r, w);
  R head = 0, last_kept = 0, first_dropped = -1;
  int k = kmax;
  for (int j = 0; j < kmax; ++j) {
    // ---- pivot: first column with the largest updated norm
    R best = -1;
    int bi = w;
    for (int c = j + t; c < w; c += NT)
      if (nu[c] > best) { best = nu[c]; bi = c; }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const R ob = __shfl_xor_sync(0xffffffffu, best, o);
      const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
      if (ob > best || (ob == best && oi < bi)) { best = ob; bi = oi; }
    }
    if (NW > 1) {
      if (lane == 0) {
        s_red[warp] = best;
        s_idx[warp] = bi;
      }
      sync();
      best = s_red[0];
      bi = s_idx[0];
#pragma unroll
      for (int q = 1; q < NW; ++q)
        if (s_red[q] > best || (s_red[q] == best && s_idx[q] < bi)) { best = s_red[q]; bi = s_idx[q]; }
    }
    if (bi != j) {
      for (int i = t; i < r; i += NT) {
        const V tmp = Z[i + j * LD];
        Z[i + j * LD] = Z[i + bi * LD];
        Z[i + bi * LD] = tmp;
      }
      if (t == 0) {
        R tmp = nu[j]; nu[j] = nu[bi]; nu[bi] = tmp;
        tmp = nd[j]; nd[j] = nd[bi]; nd[bi] = tmp;
      }
    }
    sync();
    // ---- Householder reflector of column j (makeHouseholderInPlace), warp 0, lane = row
    if (warp == 0) {
      R tail = 0;
      for (int i = j + 1 + lane; i < r; i += 32) tail += cabs2(Z[i + j * LD]);
      tail = warp_sum(tail);
      const V c0 = Z[j + j * LD];
      V tv;
      R beta;
      if (tail <= QrTraits<R>::tiny && c0.y * c0.y <= QrTraits<R>::tiny) {
        tv = mkc<R>(0, 0);
        beta = c0.x;
        for (int i = j + 1 + lane; i < r; i += 32) Z[i + j * LD] = mkc<R>(0, 0);
      } else {
        beta = sqrt(cabs2(c0) + tail);
        if (c0.x >= R(0)) beta = -beta;
        const V d = mkc<R>(c0.x - beta, c0.y);
        const R dn = cabs2(d);
        const V inv = mkc<R>(d.x / dn, -d.y / dn);
        for (int i = j + 1 + lane; i < r; i += 32) Z[i + j * LD] = cmul(Z[i + j * LD], inv);
        tv = mkc<R>((beta - c0.x) / beta, c0.y / beta);  // tau = conj((beta - c0) / beta)
      }
      __syncwarp();
      if (lane == 0) {
        Z[j + j * LD] = mkc<R>(beta, 0);
        tau[j] = tv;
        s_beta_tau[0] = mkc<R>(beta, 0);
        s_beta_tau[1] = tv;
      }
    }
    sync();
    const R absb = fabs(s_beta_tau[0].x);
    const V tj = s_beta_tau[1];
    if (j == 0) head = absb;
    if (!(absb > R(eps_t) * head)) {
      k = j;
      first_dropped = absb;
      break;
    }
    last_kept = absb;
    // ---- apply H_j = I - tau v v^H to the trailing columns (thread = column); downdate norms
    for (int cb = j + 1; cb < w; cb += CP) {
      const int c = cb + ccol;
      const bool act = c < w;
      V* zc = Z + (act ? c : j) * LD;
      const V* v = Z + j * LD;
      // this lane's rows [i0, i1) of (j, r)
      const int half = (r - j) / 2;  // rows of the first half (NH = 2)
      const int i0 = NH == 1 || hh == 0 ? j + 1 : j + 1 + half;
      const int i1 = NH == 1 || hh == 1 ? r : j + 1 + half;
      V part = mkc<R>(0, 0);
      if (act) part = dot_conj(v, zc, i0, i1);
      if (NH == 2) {
        part.x += __shfl_xor_sync(0xffffffffu, part.x, 16);
        part.y += __shfl_xor_sync(0xffffffffu, part.y, 16);
      }
      V tt = mkc<R>(0, 0);
      if (act) {
        tt = cmul(tj, cadd(zc[j], part));
        for (int i = i0; i < i1; ++i) zc[i] = csub(zc[i], cmul(v[i], tt));
      }
      if (NH == 2) __syncwarp();  // both halves updated before the norm is touched
      if (act && hh == 0) {
        const V top = csub(zc[j], tt);
        zc[j] = top;
        // LAWN-176 downdate
        const R nuc = nu[c], ndc = nd[c];
        if (nuc != R(0)) {
          R temp = sqrt(cabs2(top)) / nuc;
          temp = (R(1) + temp) * (R(1) - temp);
          if (temp < R(0)) temp = 0;
          const R ratio = nuc / ndc;
          const R temp2 = temp * ratio * ratio;
          if (temp2 <= QrTraits<R>::sqrt_eps) {
            R s2 = 0;
            for (int i = j + 1; i < r; ++i) s2 += cabs2(zc[i]);
            nu[c] = nd[c] = sqrt(s2);
          } else {
            nu[c] = nuc * sqrt(temp);
          }
        }
      }
    }
    sync();
  }
  if (t == 0 && margins) {
    // rank margin at the cut (diagnostic): min(|R_{k-1}|/thr - 1, 1 - |R_k|/thr), thr = eps |R_00|
    const double thr = eps_t * (double)head;
    double m = (double)last_kept / thr - 1.0;
    if (first_dropped >= R(0)) m = fmin(m, 1.0 - (double)first_dropped / thr);
    margins[e.rank_slot] = m;
  }
  sync();
  // ---- form Q(:, 0:k) in place: Q = H_0 ... H_{k-1} [I_k; 0], H_i = I - conj(tau_i) v v^H
  for (int i = k - 1; i >= 0; --i) {
    const V tq = cconj(tau[i]);
    const V* v = Z + i * LD;
    for (int cb = i + 1; cb < k; cb += CP) {
      const int c = cb + ccol;
      const bool act = c < k;
      V* zc = Z + (act ? c : i) * LD;
      const int half = (r - i) / 2;
      const int i0 = NH == 1 || hh == 0 ? i + 1 : i + 1 + half;
      const int i1 = NH == 1 || hh == 1 ? r : i + 1 + half;
      V part = mkc<R>(0, 0);
      if (act) part = dot_conj(v, zc, i0, i1);  // v_i = 1
      if (NH == 2) {
        part.x += __shfl_xor_sync(0xffffffffu, part.x, 16);
        part.y += __shfl_xor_sync(0xffffffffu, part.y, 16);
      }
      V tt = mkc<R>(0, 0);
      if (act) {
        tt = cmul(tq, cadd(zc[i], part));
        for (int q = i0; q < i1; ++q) zc[q] = csub(zc[q], cmul(v[q], tt));
      }
      if (NH == 2) __syncwarp();  // the other half has read zc[i]
      if (act && hh == 0) zc[i] = csub(zc[i], tt);
    }
    sync();
    for (int q = t; q < r; q += NT) {
      if (q > i) Z[q + i * LD] = cmul(mkc<R>(-tq.x, -tq.y), Z[q + i * LD]);
      else if (q == i) Z[i + i * LD] = mkc<R>(R(1) - tq.x, -tq.y);
      else Z[q + i * LD] = mkc<R>(0, 0);
    }
    sync();
  }
  // ---- write the padded-stacked Q block
  for (int c = 0; c < cap; ++c)
    for (int d = t; d < ld_dst; d += NT) {
      V v = mkc<R>(0, 0);
      if (c < k) {
        if (d < e.r1) v = Z[d + c * LD];
        else if (d >= e.dst_gap && d < e.dst_gap + e.r2) v = Z[e.r1 + (d - e.dst_gap) + c * LD];
      }
      out[d + (int64_t)c * ld_dst] = v;
    }
  if (t == 0) ranks[e.rank_slot] = k;
}

// --------------------------------------------------------------- core fit
template <typename R, int QR_THREADS>
__global__ void __launch_bounds__(QR_THREADS) core_fit_kernel(const cx<R>* __restrict__ Q, int64_t ldq,
                                                              const cx<R>* __restrict__ Zg, int64_t ldz,
                                                              const cx<R>* __restrict__ Cf, int64_t ldc,
                                                              cx<R>* __restrict__ B, int64_t ldb, int bcap,
                                                              const CoreEnt* __restrict__ ents, cx<R>* scratch,
                                                              int64_t scratch_stride, bool literal, int32_t* err_flag,
                                                              int use_smem) {
  using V = cx<R>;
  extern __shared__ __align__(16) unsigned char cf_smem[];
  const CoreEnt e = ents[blockIdx.x];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int ku = e.ku, kv = e.kv, w = e.w;
  V* out = B + e.b;
  // zero the whole block first (padding stays zero)
  for (int64_t i = threadIdx.x; i < ldb * bcap; i += QR_THREADS) out[i] = mkc<R>(0, 0);
  if (w < kv) {
    if (threadIdx.x == 0) atomicExch(err_flag, 1);
    return;
  }
  if (ku == 0 || kv == 0) return;
  V* proj = scratch + blockIdx.x * scratch_stride;  // ku x w
  const int kvp = kv + (kv & 1);
  // the Jacobi operands (coeff^H: w x kvp, and V: kvp x kvp) live in shared
  // memory when they fit (use_smem): every rotation is then a shared-memory
  // round trip instead of an L2 one; results are the same either way
  V* Ag = proj + (int64_t)ku * w;
  V* Vg = Ag + (int64_t)w * kvp;
  V* T = Vg + (int64_t)kvp * kvp;  // ku x kvp
  V* A = use_smem ? reinterpret_cast<V*>(cf_smem) : Ag;
  V* Vm = use_smem ? A + (int64_t)w * kvp : Vg;
  R* sv = reinterpret_cast<R*>(T + (int64_t)ku * kvp);
  __syncthreads();
  // proj = Q^H z
  for (int idx = threadIdx.x; idx < ku * w; idx += QR_THREADS) {
    int i = idx % ku, c = idx / ku;
    V s = mkc<R>(0, 0);
    const V* qc = Q + e.q + (int64_t)i * ldq;
    const V* zc = Zg + e.z + (int64_t)c * ldz;
    for (int q = 0; q < e.r1; ++q) cfma_conj(s, qc[q], zc[q]);
    for (int q = 0; q < e.r2; ++q) cfma_conj(s, qc[e.q_gap + q], zc[e.z_gap + q]);
    proj[idx] = s;
  }
  __syncthreads();
  if (literal) {
    for (int idx = threadIdx.x; idx < ku * kv; idx += QR_THREADS) {
      int i = idx % ku, j = idx / ku;
      V s = mkc<R>(0, 0);
      for (int c = 0; c < w; ++c) cfma(s, proj[i + c * ku], Cf[e.coeff + j + (int64_t)c * ldc]);
      out[i + (int64_t)j * ldb] = s;
    }
    return;
  }
  // A = coeff^H (w x kv), padded with a zero column to even count; V = I
  for (int idx = threadIdx.x; idx < w * kvp; idx += QR_THREADS) {
    int i = idx % w, j = idx / w;
    A[idx] = j < kv ? cconj(Cf[e.coeff + j + (int64_t)i * ldc]) : mkc<R>(0, 0);
  }
  for (int idx = threadIdx.x; idx < kvp * kvp; idx += QR_THREADS)
    Vm[idx] = (idx % kvp == idx / kvp) ? mkc<R>(1, 0) : mkc<R>(0, 0);
  __shared__ int s_rot;
  __syncthreads();
  const int npair = kvp / 2;
  for (int sweep = 0; sweep < 60; ++sweep) {
    if (threadIdx.x == 0) s_rot = 0;
    __syncthreads();
    for (int round = 0; round < kvp - 1; ++round) {
      for (int pi = warp; pi < npair; pi += (QR_THREADS / 32)) {
        // round-robin tournament: position 0 fixed, others rotate
        // (both arguments of the rotation lie in [0, 2 (kvp - 1)): a conditional
        // subtract instead of two integer divisions per pair)
        int ra = pi - 1 + round, rb = kvp - 2 - pi + round;
        if (ra >= kvp - 1) ra -= kvp - 1;
        if (rb >= kvp - 1) rb -= kvp - 1;
        int a = (pi == 0) ? 0 : 1 + ra;
        int b = 1 + rb;
        int p = min(a, b), q = max(a, b);
        V* ap = A + (int64_t)p * w;
        V* aq = A + (int64_t)q * w;
        R alpha = 0, beta = 0;
        V g = mkc<R>(0, 0);
        for (int i = lane; i < w; i += 32) {
          alpha += cabs2(ap[i]);
          beta += cabs2(aq[i]);
          cfma_conj(g, ap[i], aq[i]);
        }
        warp_sum4(alpha, beta, g.x, g.y);
        // every lane runs this scalar chain, so it is written with reciprocal
        // square roots: 2 rsqrt + 1 sqrt + 1 division (it was 3 sqrt + 5
        // divisions, and the FP64 pipe was the bound of config 4's 4096 fits)
        const R g2 = cabs2(g);
        if (g2 == R(0) || g2 <= QrTraits<R>::jacobi_tol * QrTraits<R>::jacobi_tol * (alpha * beta)) continue;
        if (lane == 0) s_rot = 1;
        const R ig = rsqrt(g2);                // 1 / |g|
        V ph = mkc<R>(g.x * ig, -g.y * ig);    // conj(e^{i phi})
        R zeta = (beta - alpha) * (R(0.5) * ig);
        R t = (zeta >= R(0) ? R(1) : R(-1)) / (fabs(zeta) + sqrt(R(1) + zeta * zeta));
        R cs = rsqrt(R(1) + t * t);
        R sn = cs * t;
        for (int i = lane; i < w; i += 32) {
          V x = ap[i], y = cmul(aq[i], ph);
          ap[i] = mkc<R>(cs * x.x - sn * y.x, cs * x.y - sn * y.y);
          aq[i] = mkc<R>(sn * x.x + cs * y.x, sn * x.y + cs * y.y);
        }
        V* vp = Vm + (int64_t)p * kvp;
        V* vq = Vm + (int64_t)q * kvp;
        for (int i = lane; i < kvp; i += 32) {
          V x = vp[i], y = cmul(vq[i], ph);
          vp[i] = mkc<R>(cs * x.x - sn * y.x, cs * x.y - sn * y.y);
          vq[i] = mkc<R>(sn * x.x + cs * y.x, sn * x.y + cs * y.y);
        }
      }
      __syncthreads();
    }
    if (!s_rot) break;
    __syncthreads();
  }
  // singular values and cutoff
  for (int j = warp; j < kvp; j += (QR_THREADS / 32)) {
    R s = 0;
    for (int i = lane; i < w; i += 32) s += cabs2(A[i + (int64_t)j * w]);
    s = warp_sum(s);
    if (lane == 0) sv[j] = sqrt(s);
  }
  __syncthreads();
  __shared__ R s_max;
  if (threadIdx.x == 0) {
    R m = 0;
    for (int j = 0; j < kvp; ++j) m = fmax(m, sv[j]);
    s_max = m;
  }
  __syncthreads();
  const R cutoff = R(1e-12) * s_max;
  // A columns <- A_j / s_j^2 (U_j / s_j) or 0
  for (int idx = threadIdx.x; idx < w * kvp; idx += QR_THREADS) {
    int j = idx / w;
    R s = sv[j];
    R f = (s > cutoff && s > R(0)) ? R(1) / (s * s) : R(0);
    A[idx] = mkc<R>(A[idx].x * f, A[idx].y * f);
  }
  __syncthreads();
  // T = proj * A  (ku x kvp)
  for (int idx = threadIdx.x; idx < ku * kvp; idx += QR_THREADS) {
    int i = idx % ku, j = idx / ku;
    V s = mkc<R>(0, 0);
    for (int c = 0; c < w; ++c) cfma(s, proj[i + c * ku], A[c + (int64_t)j * w]);
    T[idx] = s;
  }
  __syncthreads();
  // B = T * V^H  (ku x kv)
  for (int idx = threadIdx.x; idx < ku * kv; idx += QR_THREADS) {
    int i = idx % ku, j = idx / ku;
    V s = mkc<R>(0, 0);
    for (int q = 0; q < kvp; ++q) cfma_conj(s, Vm[j + (int64_t)q * kvp], T[i + (int64_t)q * ku]);
    // note: cfma_conj(s, a, b) = s + conj(a) b ; we need T(i,q) * conj(V(j,q))
    out[i + (int64_t)j * ldb] = s;
  }
}

}  // namespace

template <typename R>
void launch_cpqr(Ctx* c, const cx<R>* src, int64_t ld_src, cx<R>* dst, int64_t ld_dst, int cap, const QrEnt* ents,
                 int nent, int max_rows, int max_cols, int32_t* ranks, double eps, double* margins) {
  if (nent <= 0) return;
  if (max_rows <= 64 && max_cols <= 96 && !std::getenv("BFLY_CPQR_CTA")) {
    // one warp per block (<= 32 rows) or two (<= 64 rows); shared memory: the
    // block with an odd column stride, norms, tau
    // blocks of 33..64 rows: four warps with two lanes per trailing column
    // (BFLY_CPQR_NH=1: the two-warp, lane-per-column form)
    static const bool nh1 = std::getenv("BFLY_CPQR_NH") && std::atoi(std::getenv("BFLY_CPQR_NH")) == 1;
    const int nw = max_rows <= 32 ? 1 : nh1 ? 2 : 4;
    const int ld = nw == 1 ? 33 : 65;
    const size_t smem = sizeof(cx<R>) * ((size_t)ld * max_cols + max_cols) + 2 * sizeof(R) * max_cols;
    KTimer timer(c, "cpqr", 0.0, (double)sizeof(cx<R>) * nent * ((double)max_rows * max_cols + (double)ld_dst * cap));
    auto kern = nw == 1 ? cpqr_warp_kernel<R, 1, 1> : nw == 2 ? cpqr_warp_kernel<R, 2, 1> : cpqr_warp_kernel<R, 4, 2>;
    if (smem > 48 * 1024) BFLY_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    kern<<<nent, 32 * nw, smem, c->stream>>>(src, ld_src, dst, ld_dst, cap, ents, ranks, eps, margins);
    BFLY_LAUNCH_CHECK("cpqr_warp");
    return;
  }
  int zld = max_rows > 0 ? max_rows : 1;
  const size_t aux = 2 * sizeof(R) * max_cols + sizeof(cx<R>) * max_cols + 64;
  size_t smem = sizeof(cx<R>) * (size_t)zld * max_cols + aux;
  const int64_t area = (int64_t)max_rows * max_cols;
  const bool big = area >= 128 * 128, tiny = area <= 32 * 34;
  auto kern = big ? cpqr_kernel<R, QR_BIG> : tiny ? cpqr_kernel<R, QR_TINY> : cpqr_kernel<R, QR_SMALL>;
  const int nt = big ? QR_BIG : tiny ? QR_TINY : QR_SMALL;
  KTimer timer(c, "cpqr", 0.0, (double)sizeof(cx<R>) * nent * ((double)max_rows * max_cols + (double)ld_dst * cap));
  if (smem <= 200 * 1024) {
    BFLY_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    kern<<<nent, nt, smem, c->stream>>>(src, ld_src, dst, ld_dst, cap, ents, ranks, eps, zld, nullptr, 0, margins);
    BFLY_LAUNCH_CHECK("cpqr");
    return;
  }
  // oversized blocks (saturating ranks): blocks in global scratch, bounded chunks
  if (aux > 200 * 1024) fail(PRECONDITION, "cpqr: probe width " + std::to_string(max_cols) + " too large");
  BFLY_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)aux));
  const int64_t zstride = (int64_t)zld * max_cols;
  const int64_t chunk = std::max<int64_t>(1, std::min<int64_t>(nent, ((int64_t)1 << 31) / (zstride * sizeof(cx<R>))));
  DBuf<cx<R>> zbuf(c, (size_t)(chunk * zstride));
  for (int64_t e0 = 0; e0 < nent; e0 += chunk) {
    int n = (int)std::min<int64_t>(chunk, nent - e0);
    kern<<<n, nt, aux, c->stream>>>(src, ld_src, dst, ld_dst, cap, ents + e0, ranks, eps, zld, zbuf.p, zstride,
                                    margins);
    BFLY_LAUNCH_CHECK("cpqr");
  }
}

template <typename R>
void launch_core_fit(Ctx* c, const cx<R>* Q, int64_t ldq, const cx<R>* Z, int64_t ldz, const cx<R>* Cf, int64_t ldc,
                     cx<R>* B, int64_t ldb, int bcap, const CoreEnt* ents, int nent, int max_ku, int max_kv,
                     int max_w, bool literal, int32_t* err_flag) {
  if (nent <= 0) return;
  int kvp = max_kv + 1;
  int64_t stride = (int64_t)max_ku * max_w + (int64_t)max_w * kvp + (int64_t)kvp * kvp + (int64_t)max_ku * kvp + kvp + 8;
  DBuf<cx<R>> scratch(c, (size_t)stride * nent);
  KTimer timer(c, "core_fit", 0.0, 0.0);
  // Jacobi operands in shared memory when they fit (BFLY_COREFIT_SMEM=0: global scratch);
  // one warp per column pair of a round: 8 / 16 / 32 warps by the pair count
  static const bool smem_off = std::getenv("BFLY_COREFIT_SMEM") && std::atoi(std::getenv("BFLY_COREFIT_SMEM")) == 0;
  const size_t jbytes = sizeof(cx<R>) * ((size_t)max_w * kvp + (size_t)kvp * kvp);
  const int use_smem = !smem_off && !literal && jbytes <= 200 * 1024;
  const int npair = kvp / 2;
#define CF_LAUNCH(NTV)                                                                                              \
  do {                                                                                                              \
    auto kern = core_fit_kernel<R, NTV>;                                                                            \
    if (use_smem && jbytes > 48 * 1024)                                                                             \
      BFLY_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)jbytes));              \
    kern<<<nent, NTV, use_smem ? jbytes : 0, c->stream>>>(Q, ldq, Z, ldz, Cf, ldc, B, ldb, bcap, ents, scratch.p, stride, \
                                                          literal, err_flag, use_smem);                             \
  } while (0)
  if (use_smem && npair > 16) CF_LAUNCH(1024);
  else if (max_kv >= 64 || (use_smem && npair > 8)) CF_LAUNCH(QR_BIG);
  else CF_LAUNCH(QR_SMALL);
#undef CF_LAUNCH
  BFLY_LAUNCH_CHECK("core_fit");
}

template void launch_cpqr<double>(Ctx*, const double2*, int64_t, double2*, int64_t, int, const QrEnt*, int, int, int,
                                  int32_t*, double, double*);
template void launch_cpqr<float>(Ctx*, const float2*, int64_t, float2*, int64_t, int, const QrEnt*, int, int, int,
                                 int32_t*, double, double*);
template void launch_core_fit<double>(Ctx*, const double2*, int64_t, const double2*, int64_t, const double2*, int64_t,
                                      double2*, int64_t, int, const CoreEnt*, int, int, int, int, bool, int32_t*);
template void launch_core_fit<float>(Ctx*, const float2*, int64_t, const float2*, int64_t, const float2*, int64_t,
                                     float2*, int64_t, int, const CoreEnt*, int, int, int, int, bool, int32_t*);

}  // namespace bfly
