// k_corefit.cu -- K6 for saturated centre blocks: the core fit
// B = (R^H z) pinv(coeff) (core_block + pinv_solve, reference
// reconstruct.hpp:125-138, linalg.hpp:128-139) as batched DMMA GEMMs.
//
// For a kv x w probe-core coefficient block with w >= kv (the reference
// requires it, reconstruct.hpp:131-133) and full row rank,
//   pinv(coeff) = coeff^H G^-1,  G = coeff coeff^H  (kv x kv, Hermitian PD),
// and the pseudo-inverse is unique, so
//   B = P G^-1,  P = (R^H z) coeff^H.
// G^-1 comes from the Newton-Schulz iteration X <- X (2I - G X), X0 = I / ||G||_1,
// which converges quadratically for any nonsingular G (iterations ~ log2 cond(G));
// every step is two batched GEMMs (bgemm_dmma_kernel, 64-row bands).  A block
// whose residual ||I - G X||_F stays above 1e-12 sqrt(kv) -- cond(coeff) ~ 1e6 or
// more, where the reference's 1e-12 sigma_max cutoff could start to drop
// singular values -- is recomputed by the one-sided Jacobi pseudo-inverse of
// k_qr.cu, the reference's own semantics.  Saturated blocks (config 3: ~500 x
// 980, cond(coeff) ~ 6) converge in ~10 iterations.
//
// Round 1 ran every block through the one-sided Jacobi kernel: a 500 x 980
// block's columns stream through L2/HBM once per rotation round (config 3,
// n = 16384: 18.5 s of 24 s; n = 4096: 515 ms with 1.7 TB of DRAM traffic,
// profiles/r02_corefit_ncu.txt).
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "kernels.cuh"

namespace bfly {

namespace {

// dst (cols x rows, ld ldd) = src^H (src rows x cols, ld lds), per block
template <typename R>
__global__ void adjoint_blocks_kernel(const cx<R>* __restrict__ src, const int64_t* __restrict__ soff, int64_t lds,
                                      const int32_t* __restrict__ rows, const int32_t* __restrict__ cols,
                                      cx<R>* __restrict__ dst, int64_t dstride, int64_t ldd, int64_t dcols) {
  const int b = blockIdx.y;
  const int r = rows[b], c = cols[b];
  const cx<R>* s = src + soff[b];
  cx<R>* d = dst + (int64_t)b * dstride;
  // dst is ldd x dcols: element (j, i) = conj(src(i, j)); zero outside
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < ldd * dcols;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int j = (int)(idx % ldd), i = (int)(idx / ldd);  // dst row j (< c), col i (< r)
    cx<R> v = mkc<R>(0, 0);
    if (j < c && i < r) v = cconj(s[i + (int64_t)j * lds]);
    d[idx] = v;
  }
}

// per block: 1-norm of the Hermitian G (kv x kv, ld), X0 = I / ||G||_1
template <typename R>
__global__ void ns_init_kernel(const cx<R>* __restrict__ G, cx<R>* __restrict__ X, int64_t stride, int64_t ld,
                               const int32_t* __restrict__ kvs) {
  const int b = blockIdx.x, kv = kvs[b];
  const cx<R>* g = G + (int64_t)b * stride;
  cx<R>* x = X + (int64_t)b * stride;
  __shared__ R red[256];
  R m = 0;
  for (int j = threadIdx.x; j < kv; j += blockDim.x) {
    R s = 0;
    for (int i = 0; i < kv; ++i) s += sqrt(cabs2(g[i + (int64_t)j * ld]));
    m = fmax(m, s);
  }
  red[threadIdx.x] = m;
  __syncthreads();
  for (int s = blockDim.x / 2; s > 0; s >>= 1) {
    if (threadIdx.x < s) red[threadIdx.x] = fmax(red[threadIdx.x], red[threadIdx.x + s]);
    __syncthreads();
  }
  // X0 = I / ||G||_1: the eigenvalues of G X0 lie in [lambda_min / ||G||_1, 1]
  // (||G||_1 >= lambda_max), so ~log2(||G||_1 / lambda_min) + 6 steps converge
  const R n1 = red[0];
  const R a = n1 > R(0) ? R(1) / n1 : R(0);
  for (int64_t idx = threadIdx.x; idx < ld * ld; idx += blockDim.x) {
    const int i = (int)(idx % ld), j = (int)(idx / ld);
    x[idx] = mkc<R>((i == j && i < kv) ? a : R(0), R(0));
  }
}

// T <- 2I - T on the kv x kv part; optionally ||I - T_in||_F^2 -> res[b]
// (T_in = G X: the residual of the current iterate)
template <typename R>
__global__ void ns_step_kernel(cx<R>* __restrict__ T, int64_t stride, int64_t ld, const int32_t* __restrict__ kvs,
                               double* __restrict__ res) {
  const int b = blockIdx.y, kv = kvs[b];
  cx<R>* t = T + (int64_t)b * stride;
  double acc = 0;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < ld * ld;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int i = (int)(idx % ld), j = (int)(idx / ld);
    if (i >= kv || j >= kv) continue;
    cx<R> v = t[idx];
    const R d = i == j ? R(1) : R(0);
    acc += (double)((d - v.x) * (d - v.x) + v.y * v.y);
    t[idx] = mkc<R>(2 * d - v.x, -v.y);
  }
  if (res) {
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if ((threadIdx.x & 31) == 0) atomicAdd(&res[b], acc);
  }
}

// scatter the kv-column, ku-row result into the (zeroed) output B blocks
template <typename R>
__global__ void put_blocks_kernel(const cx<R>* __restrict__ src, int64_t sstride, int64_t lds,
                                  const int64_t* __restrict__ boff, const int32_t* __restrict__ kus,
                                  const int32_t* __restrict__ kvs, const int32_t* __restrict__ ok,
                                  cx<R>* __restrict__ B, int64_t ldb) {
  const int b = blockIdx.y;
  if (!ok[b]) return;
  const int ku = kus[b], kv = kvs[b];
  const cx<R>* s = src + (int64_t)b * sstride;
  cx<R>* d = B + boff[b];
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < (int64_t)ku * kv;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int i = (int)(idx % ku), j = (int)(idx / ku);
    d[i + (int64_t)j * ldb] = s[i + (int64_t)j * lds];
  }
}

int64_t up(int64_t x, int64_t m) { return (x + m - 1) / m * m; }

}  // namespace

template <typename R>
int64_t core_fit_big(Ctx* c, const cx<R>* Q, int64_t ldq, const cx<R>* Z, int64_t ldz, const cx<R>* Cf, int64_t ldc,
                     cx<R>* B, int64_t ldb, int bcap, const std::vector<CoreEnt>& ents,
                     std::vector<CoreEnt>& fallback) {
  using V = cx<R>;
  fallback.clear();
  if (ents.empty()) return 0;
  int maxku = 1, maxkv = 1, maxw = 1, maxr = 1;
  for (const auto& e : ents) {
    maxku = std::max(maxku, e.ku);
    maxkv = std::max(maxkv, e.kv);
    maxw = std::max(maxw, e.w);
    maxr = std::max(maxr, e.z_gap + e.r2);
  }
  const int64_t ldu = up(maxku, 8), ldv = up(maxkv, 8), ldw = up(maxw, 8);
  // per block: proj (ldu x ldw), A = coeff^H (ldw x ldv), G, X, T (ldv x ldv), P (ldu x ldv)
  const int64_t s_proj = ldu * ldw, s_a = ldw * ldv, s_sq = ldv * ldv, s_p = ldu * ldv;
  const int64_t per = s_proj + s_a + 3 * s_sq + s_p;
  // bounded chunks of blocks (~2 GB of scratch at a time)
  const int64_t chunk = std::max<int64_t>(1, std::min<int64_t>((int64_t)ents.size(),
                                                               ((int64_t)2 << 30) / (per * (int64_t)sizeof(V))));
  int64_t fitted = 0;
  for (size_t e0 = 0; e0 < ents.size(); e0 += (size_t)chunk) {
    const int nb = (int)std::min<int64_t>(chunk, (int64_t)ents.size() - (int64_t)e0);
    DBuf<V> proj(c, (size_t)(s_proj * nb)), A(c, (size_t)(s_a * nb)), G(c, (size_t)(s_sq * nb)),
        X(c, (size_t)(s_sq * nb)), T(c, (size_t)(s_sq * nb)), P(c, (size_t)(s_p * nb));
    // the GEMMs read the padding of their A operands (K up to the leading
    // dimension, only B's rows are masked): it must hold zeros, not NaNs
    proj.zero();
    G.zero();
    T.zero();
    P.zero();
    std::vector<int64_t> coff(nb), boff(nb);
    std::vector<int32_t> kus(nb), kvs(nb), ws(nb);
    for (int b = 0; b < nb; ++b) {
      const CoreEnt& e = ents[e0 + b];
      coff[b] = e.coeff;
      boff[b] = e.b;
      kus[b] = e.ku;
      kvs[b] = e.kv;
      ws[b] = e.w;
    }
    DBuf<int64_t> dcoff = to_device(c, coff), dboff = to_device(c, boff);
    DBuf<int32_t> dku = to_device(c, kus), dkv = to_device(c, kvs), dw = to_device(c, ws);
    // band entries: rows [m0, m0 + 64) of the block's M rows
    auto bands = [&](int64_t M_of(const CoreEnt&), auto&& fill) {
      std::vector<GemmEnt> v;
      for (int b = 0; b < nb; ++b) {
        const CoreEnt& e = ents[e0 + b];
        const int64_t M = M_of(e);
        for (int64_t m0 = 0; m0 < M; m0 += 64) {
          GemmEnt g{};
          fill(g, b, e, m0, std::min<int64_t>(64, M - m0));
          v.push_back(g);
        }
      }
      return v;
    };
    KTimer timer(c, "core_fit_big", 0.0, 0.0);
    // proj = Q^H z: both child slots of Q and z are contiguous rows [0, 2 gap)
    // (zero-padded), so one source of K = 2 gap
    {
      auto ge = bands([](const CoreEnt& e) -> int64_t { return e.ku; },
                      [&](GemmEnt& g, int b, const CoreEnt& e, int64_t m0, int64_t mr) {
                        g.a0 = e.q + m0 * ldq;
                        g.b0 = e.z;
                        g.c = (int64_t)b * s_proj + m0;
                        g.ncols = e.w;
                        g.mrows = (int32_t)mr;
                        g.krows = e.z_gap + e.r2;
                      });
      DBuf<GemmEnt> d = to_device(c, ge);
      launch_bgemm<R>(c, OP_H, 64, maxr, 1, Q, ldq, Z, ldz, proj.p, ldu, d.p, (int)ge.size(), maxw, false);
    }
    // A = coeff^H (w x kv)
    {
      dim3 grid((unsigned)std::min<int64_t>(64, (s_a + 255) / 256), (unsigned)nb);
      adjoint_blocks_kernel<R><<<grid, 256, 0, c->stream>>>(Cf, dcoff.p, ldc, dkv.p, dw.p, A.p, s_a, ldw, ldv);
      BFLY_LAUNCH_CHECK("adjoint_blocks");
    }
    // G = A^H A (kv x kv), P = proj A (ku x kv)
    {
      auto ge = bands([](const CoreEnt& e) -> int64_t { return e.kv; },
                      [&](GemmEnt& g, int b, const CoreEnt& e, int64_t m0, int64_t mr) {
                        g.a0 = (int64_t)b * s_a + m0 * ldw;
                        g.b0 = (int64_t)b * s_a;
                        g.c = (int64_t)b * s_sq + m0;
                        g.ncols = e.kv;
                        g.mrows = (int32_t)mr;
                        g.krows = e.w;
                      });
      DBuf<GemmEnt> d = to_device(c, ge);
      launch_bgemm<R>(c, OP_H, 64, maxw, 1, A.p, ldw, A.p, ldw, G.p, ldv, d.p, (int)ge.size(), maxkv, false);
      auto pe = bands([](const CoreEnt& e) -> int64_t { return e.ku; },
                      [&](GemmEnt& g, int b, const CoreEnt& e, int64_t m0, int64_t mr) {
                        g.a0 = (int64_t)b * s_proj + m0;
                        g.b0 = (int64_t)b * s_a;
                        g.c = (int64_t)b * s_p + m0;
                        g.ncols = e.kv;
                        g.mrows = (int32_t)mr;
                        g.krows = e.w;
                      });
      DBuf<GemmEnt> dp = to_device(c, pe);
      launch_bgemm<R>(c, OP_N, 64, maxw, 1, proj.p, ldu, A.p, ldw, P.p, ldu, dp.p, (int)pe.size(), maxkv, false);
    }
    proj.free();
    A.free();
    // Newton-Schulz: X <- X (2I - G X)
    ns_init_kernel<R><<<nb, 256, 0, c->stream>>>(G.p, X.p, s_sq, ldv, dkv.p);
    BFLY_LAUNCH_CHECK("ns_init");
    std::vector<GemmEnt> sqe = bands([](const CoreEnt& e) -> int64_t { return e.kv; },
                                     [&](GemmEnt& g, int b, const CoreEnt& e, int64_t m0, int64_t mr) {
                                       g.a0 = (int64_t)b * s_sq + m0;
                                       g.b0 = (int64_t)b * s_sq;
                                       g.c = (int64_t)b * s_sq + m0;
                                       g.ncols = e.kv;
                                       g.mrows = (int32_t)mr;
                                       g.krows = e.kv;
                                     });
    DBuf<GemmEnt> dsq = to_device(c, sqe);
    DBuf<double> res(c, (size_t)nb);
    std::vector<double> hres(nb, 1.0);
    const double tol2 = 1e-24;  // ||I - G X||_F^2 <= (1e-12)^2 kv
    std::vector<int32_t> ok(nb, 0);
    for (int it = 0; it < 60; ++it) {
      // T = G X
      launch_bgemm<R>(c, OP_N, 64, (int)ldv, 1, G.p, ldv, X.p, ldv, T.p, ldv, dsq.p, (int)sqe.size(), maxkv, false);
      const bool check = it >= 6 && (it % 2 == 0);
      if (check) res.zero();
      dim3 grid((unsigned)std::min<int64_t>(64, (s_sq + 255) / 256), (unsigned)nb);
      ns_step_kernel<R><<<grid, 256, 0, c->stream>>>(T.p, s_sq, ldv, dkv.p, check ? res.p : nullptr);
      BFLY_LAUNCH_CHECK("ns_step");
      if (check) {
        res.download(hres.data(), (size_t)nb);
        c->sync();
        bool all = true;
        for (int b = 0; b < nb; ++b) {
          ok[b] = hres[b] <= tol2 * (double)kvs[b];
          all = all && ok[b];
        }
        if (std::getenv("BFLY_DEBUG_CORE_FIT")) {
          std::fprintf(stderr, "[core_fit_big] it %d:", it);
          for (int b = 0; b < nb && b < 48; ++b)
            std::fprintf(stderr, " (ku %d kv %d w %d r %.2e)", kus[b], kvs[b], ws[b], std::sqrt(hres[b]));
          std::fprintf(stderr, "\n");
        }
        if (all) break;  // X is the converged inverse (the residual was of this X)
      }
      // X <- X T (out of place)
      DBuf<V> Xn(c, (size_t)(s_sq * nb));
      Xn.zero();
      launch_bgemm<R>(c, OP_N, 64, (int)ldv, 1, X.p, ldv, T.p, ldv, Xn.p, ldv, dsq.p, (int)sqe.size(), maxkv, false);
      X = std::move(Xn);
    }
    // B = P X (ku x kv) for the converged blocks; the others go to the Jacobi kernel
    {
      auto be = bands([](const CoreEnt& e) -> int64_t { return e.ku; },
                      [&](GemmEnt& g, int b, const CoreEnt& e, int64_t m0, int64_t mr) {
                        g.a0 = (int64_t)b * s_p + m0;
                        g.b0 = (int64_t)b * s_sq;
                        g.c = (int64_t)b * s_p + m0;
                        g.ncols = e.kv;
                        g.mrows = (int32_t)mr;
                        g.krows = e.kv;
                      });
      DBuf<V> Bt(c, (size_t)(s_p * nb));
      DBuf<GemmEnt> d = to_device(c, be);
      launch_bgemm<R>(c, OP_N, 64, (int)ldv, 1, P.p, ldu, X.p, ldv, Bt.p, ldu, d.p, (int)be.size(), maxkv, false);
      DBuf<int32_t> dok = to_device(c, ok);
      dim3 grid((unsigned)std::min<int64_t>(64, (s_p + 255) / 256), (unsigned)nb);
      put_blocks_kernel<R><<<grid, 256, 0, c->stream>>>(Bt.p, s_p, ldu, dboff.p, dku.p, dkv.p, dok.p, B, ldb);
      BFLY_LAUNCH_CHECK("put_blocks");
    }
    for (int b = 0; b < nb; ++b) {
      if (ok[b]) ++fitted;
      else fallback.push_back(ents[e0 + b]);
    }
  }
  (void)bcap;
  return fitted;
}

template int64_t core_fit_big<double>(Ctx*, const double2*, int64_t, const double2*, int64_t, const double2*, int64_t,
                                      double2*, int64_t, int, const std::vector<CoreEnt>&, std::vector<CoreEnt>&);
template int64_t core_fit_big<float>(Ctx*, const float2*, int64_t, const float2*, int64_t, const float2*, int64_t,
                                     float2*, int64_t, int, const std::vector<CoreEnt>&, std::vector<CoreEnt>&);

}  // namespace bfly
