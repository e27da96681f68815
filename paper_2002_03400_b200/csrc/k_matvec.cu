// k_matvec.cu -- K2: kernel-evaluated black-box products on the FP64 pipe.
//
// Y(:, cols) = op(K)(:, seg rows) X_seg for the BASELINE operators
// (NUFFT exp(2 pi i x xi), 3D plates exp(ikr)/(4 pi r), 2D circle exp(ikr)/r),
// evaluated on the fly (the pattern of reference operators.hpp:430-439) and
// restricted to the nonzero rows of structured probes (reconstruct.hpp:72-85).
// Each CTA owns BM output points x BN columns: a BM x BK tile of kernel
// entries is evaluated once into shared memory and reused across all BN
// columns; the complex contraction is register tiled (TM x TN per thread).
// Long segments are split across gridDim.z into partial buffers that are
// reduced in a fixed order (no atomics -> bitwise reproducible results).
//
// Entry arithmetic is written so r, the phase and 1/r match the CPU oracle
// bit-for-bit (explicit __dmul_rn/fma, no contraction); sin/cos differ by ulps.
#include <algorithm>
#include <cstdlib>
#include <string>
#include <type_traits>
#include <vector>

#include "k_eval.cuh"
#include "kernels.cuh"

namespace bfly {

namespace {

using keval::kFourPi;
using keval::kTwoPi;
using keval::kernel_entry_fast;

struct MatvecItem {
  int64_t row0, rows;  // input point range of this work item
  int64_t x_off, ldx;  // X_seg(0, c0) offset
  int64_t ycol;        // first output column
  int64_t ybase;       // partial-buffer offset (split-K)
  int32_t ncols;
  int32_t pad_;
};

// K(i, j) with i a target (row) point and j a source (column) point.
template <int KIND>
__device__ __forceinline__ double2 kernel_entry(double tx, double ty, double tz, double sx, double sy, double sz,
                                                double kappa) {
  double sn, cs;
  if (KIND == KK_NUFFT) {
    double ph = __dmul_rn(tx, sx);
    double f = __dsub_rn(ph, rint(ph));
    sincos(__dmul_rn(kTwoPi, f), &sn, &cs);
    return make_double2(cs, sn);
  } else if (KIND == KK_PLATES) {
    double dx = __dsub_rn(tx, sx), dy = __dsub_rn(ty, sy), dz = __dsub_rn(tz, sz);
    double r = __dsqrt_rn(fma(dz, dz, fma(dy, dy, __dmul_rn(dx, dx))));
    double ph = __dmul_rn(kappa, r);
    double sc = __ddiv_rn(1.0, __dmul_rn(kFourPi, r));
    sincos(ph, &sn, &cs);
    return make_double2(__dmul_rn(cs, sc), __dmul_rn(sn, sc));
  } else {
    double dx = __dsub_rn(tx, sx), dy = __dsub_rn(ty, sy);
    double r = __dsqrt_rn(fma(dy, dy, __dmul_rn(dx, dx)));
    double ph = __dmul_rn(kappa, r);
    double sc = __ddiv_rn(1.0, r);
    sincos(ph, &sn, &cs);
    return make_double2(__dmul_rn(cs, sc), __dmul_rn(sn, sc));
  }
}

template <typename R, int KIND, int MODE, int BM, int BN, int TM, int TN, int BK>
__global__ void __launch_bounds__(256) matvec_kernel(Points outp, Points inp, double kappa, int64_t m_out,
                                                     const cx<R>* __restrict__ X, cx<R>* __restrict__ Y, int64_t ldy,
                                                     const MatvecItem* __restrict__ items, int64_t rows_per_split,
                                                     int64_t pstride) {
  using V = cx<R>;
  constexpr int CL = BN / TN, RL = BM / TM;
  static_assert(CL * RL == 256, "thread layout");
  static_assert(256 % BM == 0 || BM % 256 == 0, "eval layout");
  extern __shared__ __align__(16) unsigned char smem_raw[];
  V* Ks = reinterpret_cast<V*>(smem_raw);  // [BK][BM]
  V* Xs = Ks + BK * BM;                    // [BK][BN]

  const MatvecItem it = items[blockIdx.y];
  const int64_t i0 = (int64_t)blockIdx.x * BM;
  const int tid = threadIdx.x;
  const int cl = tid % CL, rl = tid / CL;

  // this split's input row range
  const int64_t kb = (int64_t)blockIdx.z * rows_per_split;
  const int64_t ke = min(it.rows, kb + rows_per_split);

  // eval mapping: each thread evaluates a fixed output row
  constexpr int EV_ROWS_PER_PASS = BM < 256 ? BM : 256;
  constexpr int EV_K_PER_PASS = 256 / EV_ROWS_PER_PASS;  // >= 1
  const int erow = tid % EV_ROWS_PER_PASS;
  const int ek0 = tid / EV_ROWS_PER_PASS;
  constexpr int EV_ROW_REPS = BM / EV_ROWS_PER_PASS;  // >= 1

  double ox[EV_ROW_REPS], oy[EV_ROW_REPS], oz[EV_ROW_REPS];
  bool ovalid[EV_ROW_REPS];
#pragma unroll
  for (int q = 0; q < EV_ROW_REPS; ++q) {
    int64_t gi = i0 + erow + q * EV_ROWS_PER_PASS;
    ovalid[q] = gi < m_out;
    int64_t gs = ovalid[q] ? gi : 0;
    ox[q] = outp.x[gs];
    oy[q] = KIND == KK_NUFFT ? 0.0 : outp.y[gs];
    oz[q] = KIND == KK_PLATES ? outp.z[gs] : 0.0;
  }

  V acc[TM][TN];
#pragma unroll
  for (int a = 0; a < TM; ++a)
#pragma unroll
    for (int b = 0; b < TN; ++b) acc[a][b] = mkc<R>(0, 0);

  for (int64_t k0 = kb; k0 < ke; k0 += BK) {
    // ---- evaluate the kernel tile into shared memory
#pragma unroll
    for (int q = 0; q < EV_ROW_REPS; ++q) {
#pragma unroll 4
      for (int kk = ek0; kk < BK; kk += EV_K_PER_PASS) {
        int64_t gj = k0 + kk;
        double2 v = make_double2(0.0, 0.0);
        if (ovalid[q] && gj < ke) {
          int64_t pj = it.row0 + gj;
          double ix = __ldg(inp.x + pj);
          double iy = KIND == KK_NUFFT ? 0.0 : __ldg(inp.y + pj);
          double iz = KIND == KK_PLATES ? __ldg(inp.z + pj) : 0.0;
          if (MODE == OP_N) v = kernel_entry<KIND>(ox[q], oy[q], oz[q], ix, iy, iz, kappa);
          else v = kernel_entry<KIND>(ix, iy, iz, ox[q], oy[q], oz[q], kappa);
          if (MODE == OP_H) v.y = -v.y;
        }
        Ks[kk * BM + erow + q * EV_ROWS_PER_PASS] = mkc<R>((R)v.x, (R)v.y);
      }
    }
    // ---- stage the probe tile
    for (int idx = tid; idx < BK * BN; idx += 256) {
      int kk = idx % BK, c = idx / BK;
      int64_t gj = k0 + kk;
      V v = mkc<R>(0, 0);
      if (gj < ke && c < it.ncols) v = X[it.x_off + gj + (int64_t)c * it.ldx];
      Xs[kk * BN + c] = v;
    }
    __syncthreads();
#pragma unroll 4
    for (int kk = 0; kk < BK; ++kk) {
      V a[TM], b[TN];
#pragma unroll
      for (int q = 0; q < TM; ++q) a[q] = Ks[kk * BM + rl + q * RL];
#pragma unroll
      for (int q = 0; q < TN; ++q) b[q] = Xs[kk * BN + cl + q * CL];
#pragma unroll
      for (int p = 0; p < TM; ++p)
#pragma unroll
        for (int q = 0; q < TN; ++q) cfma(acc[p][q], a[p], b[q]);
    }
    __syncthreads();
  }
  // ---- store (plain store; split-K partials go to their own slice)
  V* Yb = Y + it.ybase + (int64_t)blockIdx.z * pstride;
#pragma unroll
  for (int p = 0; p < TM; ++p) {
    int64_t gi = i0 + rl + p * RL;
    if (gi >= m_out) continue;
#pragma unroll
    for (int q = 0; q < TN; ++q) {
      int c = cl + q * CL;
      if (c < it.ncols) Yb[gi + (it.ycol + c) * ldy] = acc[p][q];
    }
  }
}

// ----------------------------------------------------------------------------
// complex128 path: contraction on the FP64 tensor path (mma.sync m8n8k4 f64).
// DMMA and DFMA share the FP64 pipe on B200 (profiles/r01_matvec_ncu.txt), so
// the win is issue slots: one DMMA does the work of 8 warp-wide DFMAs, which
// leaves the issue bandwidth to the kernel-entry evaluation.
// ----------------------------------------------------------------------------

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}
__device__ __forceinline__ double dneg(double a) {
  return __longlong_as_double(__double_as_longlong(a) ^ (long long)0x8000000000000000ULL);
}

// 8 warps stacked along the output rows; warp w owns rows [w*8*MT, (w+1)*8*MT)
// of the CTA tile and all 8*NT columns.  Shared memory (doubles):
//   Kre, Kim [BK][BM+8]   kernel tile, k-major: A fragments conflict free
//   Xre, Xim [BN][BK+4]   probe tile, column-major: B fragments conflict free
//   P[3][BK]              input points of the tile
template <int KIND, int MODE, int MT, int NT, int BK, int MINB, bool G3>
__global__ void __launch_bounds__(256, MINB) matvec_dmma_kernel(Points outp, Points inp, double kappa, int64_t m_out,
                                                             const double2* __restrict__ X, double2* __restrict__ Y,
                                                             int64_t ldy, const MatvecItem* __restrict__ items,
                                                             int64_t rows_per_split, int64_t pstride) {
  constexpr int BM = 64 * MT, BN = 8 * NT, SM = BM + 8, SX = BK + 4;
  constexpr int XPT = (BK * BN + 255) / 256;  // probe-tile elements per thread
  extern __shared__ __align__(16) double sm_d[];
  // G3: Gauss's 3-multiplication complex product (P1 = a c, P2 = b d,
  // P3 = (a+b)(c+d); re = P1 - P2, im = P3 - P1 - P2): a third "sum" plane
  constexpr int NPL = G3 ? 3 : 2;
  double* Kre = sm_d;
  double* Kim = Kre + BK * SM;
  double* Ksu = Kim + BK * SM;  // G3 only
  double* Xb = Kre + NPL * BK * SM;  // 2 buffers x NPL planes x BN x SX
  double* Pb = Xb + 2 * NPL * BN * SX;  // 2 buffers x [3][BK]

  const MatvecItem it = items[blockIdx.y];
  const int64_t i0 = (int64_t)blockIdx.x * BM;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g = lane >> 2, t = lane & 3;
  const int64_t kb = (int64_t)blockIdx.z * rows_per_split;
  const int64_t ke = min(it.rows, kb + rows_per_split);

  // evaluation mapping: thread -> fixed output row(s), strided k
  constexpr int EROWS = BM < 256 ? BM : 256;
  constexpr int EKSTEP = 256 / EROWS;
  constexpr int EREPS = BM / EROWS;
  const int erow = tid % EROWS, ek0 = tid / EROWS;
  double ox[EREPS], oy[EREPS], oz[EREPS];
  bool ovalid[EREPS];
#pragma unroll
  for (int q = 0; q < EREPS; ++q) {
    const int64_t gi = i0 + erow + q * EROWS;
    ovalid[q] = gi < m_out;
    const int64_t gs = ovalid[q] ? gi : 0;
    ox[q] = outp.x[gs];
    oy[q] = KIND == KK_NUFFT ? 0.0 : outp.y[gs];
    oz[q] = KIND == KK_PLATES ? outp.z[gs] : 0.0;
  }

  // register staging of the next probe tile / input points
  double2 xr[XPT];
  double pr[3];
  auto fetch = [&](int64_t k0) {
#pragma unroll
    for (int q = 0; q < XPT; ++q) {
      const int idx = tid + 256 * q;
      const int kk = idx % BK, cc = idx / BK;
      const int64_t gj = k0 + kk;
      xr[q] = (idx < BK * BN && gj < ke && cc < it.ncols) ? X[it.x_off + gj + (int64_t)cc * it.ldx]
                                                          : make_double2(0.0, 0.0);
    }
    if (tid < BK) {
      const int64_t gj = k0 + tid;
      const int64_t pj = it.row0 + (gj < ke ? gj : kb);
      pr[0] = inp.x[pj];
      pr[1] = KIND == KK_NUFFT ? 0.0 : inp.y[pj];
      pr[2] = KIND == KK_PLATES ? inp.z[pj] : 0.0;
    }
  };
  auto commit = [&](int buf) {
    double* xre = Xb + buf * NPL * BN * SX;
    double* xim = xre + BN * SX;
    double* xsu = xim + BN * SX;
#pragma unroll
    for (int q = 0; q < XPT; ++q) {
      const int idx = tid + 256 * q;
      if (idx < BK * BN) {
        const int kk = idx % BK, cc = idx / BK;
        xre[cc * SX + kk] = xr[q].x;
        xim[cc * SX + kk] = xr[q].y;
        if (G3) xsu[cc * SX + kk] = xr[q].x + xr[q].y;
      }
    }
    if (tid < BK) {
      double* p = Pb + buf * 3 * BK;
      p[tid] = pr[0];
      p[BK + tid] = pr[1];
      p[2 * BK + tid] = pr[2];
    }
  };

  double acc[MT][NT][NPL][2];  // [re|im] or [P1|P2|P3], 2 values
#pragma unroll
  for (int a = 0; a < MT; ++a)
#pragma unroll
    for (int b = 0; b < NT; ++b)
#pragma unroll
      for (int p = 0; p < NPL; ++p) acc[a][b][p][0] = acc[a][b][p][1] = 0.0;

  if (kb < ke) {
    fetch(kb);
    commit(0);
  }
  __syncthreads();
  int buf = 0;
  for (int64_t k0 = kb; k0 < ke; k0 += BK, buf ^= 1) {
    const double* P = Pb + buf * 3 * BK;
    // ---- evaluate the BM x BK kernel tile
#pragma unroll
    for (int q = 0; q < EREPS; ++q) {
#pragma unroll 4
      for (int kk = ek0; kk < BK; kk += EKSTEP) {
        double2 v = make_double2(0.0, 0.0);
        if (ovalid[q] && k0 + kk < ke) {
          const double ix = P[kk], iy = P[BK + kk], iz = P[2 * BK + kk];
          if (MODE == OP_N) v = kernel_entry_fast<KIND>(ox[q], oy[q], oz[q], ix, iy, iz, kappa);
          else v = kernel_entry_fast<KIND>(ix, iy, iz, ox[q], oy[q], oz[q], kappa);
          if (MODE == OP_H) v.y = -v.y;
        }
        Kre[kk * SM + erow + q * EROWS] = v.x;
        Kim[kk * SM + erow + q * EROWS] = v.y;
        if (G3) Ksu[kk * SM + erow + q * EROWS] = v.x + v.y;
      }
    }
    __syncthreads();
    const bool more = k0 + BK < ke;
    if (more) fetch(k0 + BK);  // global loads in flight during the MMAs
    // ---- complex contraction on DMMA: 4 real m8n8k4 per complex tile
    const double* xre = Xb + buf * NPL * BN * SX;
    const double* xim = xre + BN * SX;
    const double* xsu = xim + BN * SX;
#pragma unroll
    for (int ks = 0; ks < BK; ks += 4) {
      double ar[MT], ai[MT], br[NT], bi[NT], as_[MT], bs_[NT];
#pragma unroll
      for (int a = 0; a < MT; ++a) {
        const int row = warp * 8 * MT + a * 8 + g;
        ar[a] = Kre[(ks + t) * SM + row];
        ai[a] = Kim[(ks + t) * SM + row];
        if (G3) as_[a] = Ksu[(ks + t) * SM + row];
      }
#pragma unroll
      for (int b = 0; b < NT; ++b) {
        const int col = b * 8 + g;
        br[b] = xre[col * SX + ks + t];
        bi[b] = xim[col * SX + ks + t];
        if (G3) bs_[b] = xsu[col * SX + ks + t];
      }
      if constexpr (G3) {
#pragma unroll
        for (int a = 0; a < MT; ++a)
#pragma unroll
          for (int b = 0; b < NT; ++b) {
            dmma(acc[a][b][0][0], acc[a][b][0][1], ar[a], br[b]);
            dmma(acc[a][b][1][0], acc[a][b][1][1], ai[a], bi[b]);
            dmma(acc[a][b][2][0], acc[a][b][2][1], as_[a], bs_[b]);
          }
      } else {
        // two passes over the MT x NT tiles: a dependent MMA pair is 2*MT*NT
        // instructions apart (no fixed-latency waits between them)
#pragma unroll
        for (int a = 0; a < MT; ++a)
#pragma unroll
          for (int b = 0; b < NT; ++b) {
            dmma(acc[a][b][0][0], acc[a][b][0][1], ar[a], br[b]);
            dmma(acc[a][b][1][0], acc[a][b][1][1], ar[a], bi[b]);
          }
#pragma unroll
        for (int a = 0; a < MT; ++a) {
          const double nai = dneg(ai[a]);
#pragma unroll
          for (int b = 0; b < NT; ++b) {
            dmma(acc[a][b][0][0], acc[a][b][0][1], nai, bi[b]);
            dmma(acc[a][b][1][0], acc[a][b][1][1], ai[a], br[b]);
          }
        }
      }
    }
    if (more) commit(buf ^ 1);
    __syncthreads();
  }
  // ---- store: lane (g, t) holds C[g][2t], C[g][2t+1] of every 8x8 tile
  double2* Yb = Y + it.ybase + (int64_t)blockIdx.z * pstride;
#pragma unroll
  for (int a = 0; a < MT; ++a) {
    const int64_t gi = i0 + warp * 8 * MT + a * 8 + g;
    if (gi >= m_out) continue;
#pragma unroll
    for (int b = 0; b < NT; ++b)
#pragma unroll
      for (int v = 0; v < 2; ++v) {
        const int cc = b * 8 + 2 * t + v;
        if (cc >= it.ncols) continue;
        if constexpr (G3) {
          const double p1 = acc[a][b][0][v], p2 = acc[a][b][1][v], p3 = acc[a][b][NPL - 1][v];
          Yb[gi + (it.ycol + cc) * ldy] = make_double2(p1 - p2, p3 - p1 - p2);
        } else {
          Yb[gi + (it.ycol + cc) * ldy] = make_double2(acc[a][b][0][v], acc[a][b][1][v]);
        }
      }
  }
}

// Y(:, cols) = sum_z P_z(:, cols), fixed order
template <typename R>
__global__ void split_reduce_kernel(const cx<R>* __restrict__ P, int64_t pstride, int nsplit, cx<R>* Y, int64_t ldy,
                                    int64_t m, int64_t col0, int64_t ncols) {
  int64_t total = m * ncols;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
    int64_t i = t % m, c = t / m;
    int64_t off = i + (col0 + c) * ldy;
    cx<R> s = P[off];
    for (int z = 1; z < nsplit; ++z) s = cadd(s, P[z * pstride + off]);
    Y[off] = s;
  }
}

template <typename R, int KIND, int MODE, int BM, int BN, int TM, int TN, int DM = 0, int MT = 1, int NT = 1>
void run_cfg(Ctx* c, Points outp, Points inp, double kappa, int64_t m_out, const cx<R>* X, cx<R>* Y, int64_t ldy,
             const MatvecSeg* segs, int nseg) {
  constexpr int BK = 16;
  // work items: (segment, column tile)
  std::vector<MatvecItem> items;
  int64_t max_rows = 0, total_cols = 0, min_col = INT64_MAX, max_col = 0;
  for (int s = 0; s < nseg; ++s) {
    const MatvecSeg& g = segs[s];
    if (g.ncols <= 0) continue;
    if (g.rows <= 0) {  // empty probe: exact zero product
      BFLY_CUDA(cudaMemset2DAsync(Y + g.col0 * ldy, ldy * sizeof(cx<R>), 0, m_out * sizeof(cx<R>), g.ncols,
                                  c->stream));
      continue;
    }
    for (int tc = 0; tc < g.ncols; tc += BN) {
      MatvecItem it;
      it.row0 = g.row0;
      it.rows = g.rows;
      it.x_off = g.x_off + (int64_t)tc * g.ldx;
      it.ldx = g.ldx;
      it.ycol = g.col0 + tc;
      it.ybase = 0;
      it.ncols = std::min(BN, g.ncols - tc);
      it.pad_ = 0;
      items.push_back(it);
    }
    max_rows = std::max(max_rows, g.rows);
    total_cols += g.ncols;
    min_col = std::min(min_col, g.col0);
    max_col = std::max(max_col, g.col0 + (int64_t)g.ncols);
  }
  if (items.empty()) return;
  const int64_t gx = ceil_div(m_out, BM);
  const int64_t base_ctas = gx * (int64_t)items.size();
  // split long segments so the grid covers the GPU several times over
  const int64_t target = (int64_t)c->sm_count * 8;
  int nsplit = 1;
  if (base_ctas < target) nsplit = (int)std::min<int64_t>(ceil_div(target, base_ctas), ceil_div(max_rows, 4 * BK));
  nsplit = std::max(1, std::min(nsplit, 64));
  int64_t rows_per_split = ceil_div(ceil_div(max_rows, nsplit), BK) * BK;
  nsplit = (int)ceil_div(max_rows, rows_per_split);

  DBuf<MatvecItem> ditems(c, items.size());
  ditems.upload(items.data(), items.size());
  double kflops = 0, kbytes = 0;
  for (const auto& it : items) {
    kflops += 8.0 * (double)m_out * (double)it.rows * (double)it.ncols;
    kbytes += (double)sizeof(cx<R>) * ((double)it.rows + (double)m_out) * (double)it.ncols;
  }
  KTimer timer(c, "kernel_matvec", kflops, kbytes);
  using KernFn = void (*)(Points, Points, double, int64_t, const cx<R>*, cx<R>*, int64_t, const MatvecItem*, int64_t,
                          int64_t);
  size_t smem;
  KernFn kern;
  if constexpr (DM) {
    static_assert(BM == 64 * MT && BN == 8 * NT, "dmma tile");
    // Gauss 3M for the wide tiles (transfer levels: -5%); the narrow leaf-round
    // tiles keep 4M (3M adds register pressure there)
    static const bool g3_env = !std::getenv("BFLY_MV_4M");
    const bool g3 = g3_env && NT >= 4;
    const int npl = g3 ? 3 : 2;
    smem = sizeof(double) * (size_t)(npl * BK * (BM + 8) + 2 * npl * BN * (BK + 4) + 6 * BK);
    if (g3) kern = matvec_dmma_kernel<KIND, MODE, MT, NT, BK, (MT * NT <= 8 ? 2 : 1), true>;
    else kern = matvec_dmma_kernel<KIND, MODE, MT, NT, BK, (MT * NT <= 8 ? 2 : 1), false>;
  } else {
    smem = sizeof(cx<R>) * (size_t)BK * (BM + BN);
    kern = matvec_kernel<R, KIND, MODE, BM, BN, TM, TN, BK>;
  }
  BFLY_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  if (items.size() > 65535) fail(PRECONDITION, "matvec: too many work items");
  dim3 grid((unsigned)gx, (unsigned)items.size(), (unsigned)nsplit);
  if (nsplit == 1) {
    kern<<<grid, 256, smem, c->stream>>>(outp, inp, kappa, m_out, X, Y, ldy, ditems.p, rows_per_split, 0);
    BFLY_LAUNCH_CHECK("kernel_matvec");
    return;
  }
  // split z writes slice z (laid out exactly like Y); every CTA stores its full
  // tile (zeros for an empty row window), then a fixed-order reduction.
  const int64_t pstride = ldy * max_col;
  DBuf<cx<R>> part(c, (size_t)(pstride * nsplit));
  kern<<<grid, 256, smem, c->stream>>>(outp, inp, kappa, m_out, X, part.p, ldy, ditems.p, rows_per_split, pstride);
  BFLY_LAUNCH_CHECK("kernel_matvec");
  for (int s = 0; s < nseg; ++s) {
    const MatvecSeg& g = segs[s];
    if (g.ncols <= 0 || g.rows <= 0) continue;
    int64_t total = m_out * g.ncols;
    unsigned blocks = (unsigned)std::min<int64_t>(ceil_div(total, 256), (int64_t)c->sm_count * 16);
    split_reduce_kernel<R><<<blocks, 256, 0, c->stream>>>(part.p, pstride, nsplit, Y, ldy, m_out,
                                                          g.col0, g.ncols);
    BFLY_LAUNCH_CHECK("split_reduce");
  }
  (void)total_cols;
  (void)min_col;
}

template <typename R, int KIND, int MODE>
void dispatch_width(Ctx* c, Points outp, Points inp, double kappa, int64_t m_out, const cx<R>* X, cx<R>* Y,
                    int64_t ldy, const MatvecSeg* segs, int nseg) {
  int maxw = 0;
  for (int s = 0; s < nseg; ++s) maxw = std::max(maxw, segs[s].ncols);
  if constexpr (std::is_same<R, double>::value) {
    // complex128: DMMA tiles (BM = 64 MT rows, BN = 8 NT columns)
    if (maxw <= 8) run_cfg<R, KIND, MODE, 256, 8, 1, 1, 1, 4, 1>(c, outp, inp, kappa, m_out, X, Y, ldy, segs, nseg);
    else if (maxw <= 16) run_cfg<R, KIND, MODE, 256, 16, 1, 1, 1, 4, 2>(c, outp, inp, kappa, m_out, X, Y, ldy, segs, nseg);
    else if (maxw <= 24) run_cfg<R, KIND, MODE, 256, 24, 1, 1, 1, 4, 3>(c, outp, inp, kappa, m_out, X, Y, ldy, segs, nseg);
    else if (maxw <= 32) {
      // 2x4 warp tiles (122 regs, 2 CTAs/SM) beat 4x4 (232 regs, 1 CTA/SM) by 12% on config 2
      static const bool big = std::getenv("BFLY_MV_TILE") && std::string(std::getenv("BFLY_MV_TILE")) == "4x4";
      if (!big) run_cfg<R, KIND, MODE, 128, 32, 1, 1, 1, 2, 4>(c, outp, inp, kappa, m_out, X, Y, ldy, segs, nseg);
      else run_cfg<R, KIND, MODE, 256, 32, 1, 1, 1, 4, 4>(c, outp, inp, kappa, m_out, X, Y, ldy, segs, nseg);
    }
    else run_cfg<R, KIND, MODE, 128, 64, 1, 1, 1, 2, 8>(c, outp, inp, kappa, m_out, X, Y, ldy, segs, nseg);
    return;
  }
  if (maxw <= 8) run_cfg<R, KIND, MODE, 256, 8, 4, 2>(c, outp, inp, kappa, m_out, X, Y, ldy, segs, nseg);
  else if (maxw <= 16) run_cfg<R, KIND, MODE, 256, 16, 8, 2>(c, outp, inp, kappa, m_out, X, Y, ldy, segs, nseg);
  else if (maxw <= 32) run_cfg<R, KIND, MODE, 128, 32, 4, 4>(c, outp, inp, kappa, m_out, X, Y, ldy, segs, nseg);
  else run_cfg<R, KIND, MODE, 128, 64, 4, 8>(c, outp, inp, kappa, m_out, X, Y, ldy, segs, nseg);
}

template <typename R, int KIND>
void dispatch_mode(Ctx* c, int mode, Points outp, Points inp, double kappa, int64_t m_out, const cx<R>* X, cx<R>* Y,
                   int64_t ldy, const MatvecSeg* segs, int nseg) {
  if (mode == OP_N) dispatch_width<R, KIND, OP_N>(c, outp, inp, kappa, m_out, X, Y, ldy, segs, nseg);
  else if (mode == OP_T) dispatch_width<R, KIND, OP_T>(c, outp, inp, kappa, m_out, X, Y, ldy, segs, nseg);
  else dispatch_width<R, KIND, OP_H>(c, outp, inp, kappa, m_out, X, Y, ldy, segs, nseg);
}

}  // namespace

template <typename R>
void launch_kernel_matvec(Ctx* c, int kind, int mode, Points outp, Points inp, double kappa, int64_t m_out,
                          const cx<R>* X, cx<R>* Y, int64_t ldy, const MatvecSeg* segs, int nseg) {
  if (m_out <= 0 || nseg <= 0) return;
  if constexpr (std::is_same<R, double>::value) {
    if (!c->force_fp64 && matvec_oz_enabled() &&
        launch_kernel_matvec_oz(c, kind, mode, outp, inp, kappa, m_out, X, Y, ldy, segs, nseg))
      return;
  }
  if (kind == KK_NUFFT) dispatch_mode<R, KK_NUFFT>(c, mode, outp, inp, kappa, m_out, X, Y, ldy, segs, nseg);
  else if (kind == KK_PLATES) dispatch_mode<R, KK_PLATES>(c, mode, outp, inp, kappa, m_out, X, Y, ldy, segs, nseg);
  else if (kind == KK_CIRCLE) dispatch_mode<R, KK_CIRCLE>(c, mode, outp, inp, kappa, m_out, X, Y, ldy, segs, nseg);
  else fail(PRECONDITION, "kernel_matvec: unknown kernel kind");
}

template void launch_kernel_matvec<double>(Ctx*, int, int, Points, Points, double, int64_t, const double2*, double2*,
                                           int64_t, const MatvecSeg*, int);
template void launch_kernel_matvec<float>(Ctx*, int, int, Points, Points, double, int64_t, const float2*, float2*,
                                          int64_t, const MatvecSeg*, int);

}  // namespace bfly
