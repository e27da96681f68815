// verify.cu -- level-wise residual sums of a butterfly against a dense copy
// of its operator, on the GPU: u_side_residual / v_side_residual /
// center_residual of the reference (reconstruct.hpp:443-503), used by the
// error-bound check of Theorems 5.1-5.3 (tools/bfly_cli.cpp:208-235, the
// `verify` subcommand).  Desk scale only: the operator is densified.
//
//   u-side, row level l in [l_m, L]:  sum_b || K_b - U U^H K_b ||_F^2
//   v-side, row level l in [0, l_m]:  sum_b || K_b - K_b V V^H ||_F^2
//   center (l = l_m):                 sum_b || K_b - U (U^H K_b V) V^H ||_F^2
// with K in tree order and b = (tau, nu) over the 2^L blocks of the level.
//
// The expanded nested bases U_{l,tau,nu} (rows T_tau) are built level by
// level from the leaves through the R (W) transfer blocks with batched GEMMs
// (padded-stacked children: rows [0, P_child) and [P_child, 2 P_child));
// every block product is a batched GEMM over the level, and the residual
// of a level is one deterministic sum of squared differences over the whole
// matrix (the blocks of a level tile it).
#include <cmath>
#include <vector>

#include "butterfly.h"
#include "kernels.cuh"
#include "operators.h"
#include "verify.h"

namespace bfly {

namespace {

constexpr int BIG = 1 << 30;

template <typename R>
__global__ void identity_cols_kernel(cx<R>* X, int64_t n, int64_t j0, int64_t cols, const int64_t* perm) {
  // X (n x cols) = columns perm[j0 + q] of the identity
  const int64_t total = n * cols;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = t % n, q = t / n;
    const int64_t src = perm ? perm[j0 + q] : j0 + q;
    X[t] = i == src ? cx<R>{1, 0} : cx<R>{0, 0};
  }
}

template <typename R>
__global__ void conj_transpose_kernel(const cx<R>* __restrict__ a, int64_t lda, int64_t rows, int64_t cols,
                                      cx<R>* __restrict__ b, int64_t ldb) {
  // b (cols x rows) = a^H
  const int64_t total = rows * cols;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = t % rows, j = t / rows;
    const cx<R> v = a[i + j * lda];
    b[j + i * ldb] = cx<R>{v.x, -v.y};
  }
}

// per-CTA partial sums of |a - b|^2 (b may be null): fixed grid, summed on the
// host in order -> deterministic
template <typename R>
__global__ void sumsq_diff_kernel(const cx<R>* __restrict__ a, const cx<R>* __restrict__ b, int64_t n,
                                  double* __restrict__ part) {
  double s = 0;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n; t += (int64_t)gridDim.x * blockDim.x) {
    double dx = (double)a[t].x, dy = (double)a[t].y;
    if (b) {
      dx -= (double)b[t].x;
      dy -= (double)b[t].y;
    }
    s += dx * dx + dy * dy;
  }
  __shared__ double red[256];
  red[threadIdx.x] = s;
  __syncthreads();
  for (int o = 128; o > 0; o >>= 1) {
    if (threadIdx.x < o) red[threadIdx.x] += red[threadIdx.x + o];
    __syncthreads();
  }
  if (threadIdx.x == 0) part[blockIdx.x] = red[0];
}

template <typename R>
double sumsq_diff(Ctx* c, const cx<R>* a, const cx<R>* b, int64_t n) {
  constexpr int G = 1024;
  DBuf<double> part(c, G);
  sumsq_diff_kernel<R><<<G, 256, 0, c->stream>>>(a, b, n, part.p);
  BFLY_LAUNCH_CHECK("sumsq_diff");
  std::vector<double> h(G);
  part.download(h.data(), G);
  c->sync();
  double s = 0;
  for (double v : h) s += v;
  return s;
}

GemmEnt gent(int64_t a0, int64_t b0, int64_t c, int ncols, int mrows = BIG, int krows = BIG) {
  GemmEnt e{};
  e.a0 = a0;
  e.b0 = b0;
  e.c = c;
  e.ncols = ncols;
  e.mrows = mrows;
  e.krows = krows;
  return e;
}

// Expanded bases of one side, one buffer per level: block i of level l at
// i * ld[l] * P[l] (ld = largest node of the level, zero rows below a node)
template <typename R>
struct Expanded {
  std::vector<DBuf<cx<R>>> buf;
  std::vector<int64_t> ld;
  std::vector<int> P;
};

// U side: levels L .. l_m, node tree = row tree
template <typename R>
Expanded<R> expand_u(Ctx* c, const DevButterfly<R>& bf) {
  const int L = bf.L, lm = bf.lm;
  const int64_t NB = bf.nb();
  Expanded<R> e;
  e.buf.resize(L + 1);
  e.ld.assign(L + 1, 0);
  e.P.assign(L + 1, 0);
  e.ld[L] = bf.uleaf.ld;
  e.P[L] = bf.PU(L);
  e.buf[L].reset(c, (size_t)(NB * e.ld[L] * std::max(1, e.P[L])));
  // leaves: copy the U leaf blocks (ld x cap, first P columns)
  {
    std::vector<GemmEnt> x;  // identity-free copy via copy2d per block would be NB launches: use a strided copy
    for (int64_t i = 0; i < NB; ++i)
      launch_copy2d<R>(c, e.buf[L].p + i * e.ld[L] * e.P[L], e.ld[L], bf.uleaf.block(i), bf.uleaf.ld, e.ld[L], e.P[L]);
  }
  for (int l = L - 1; l >= lm; --l) {
    const Level<R>& Rl = bf.r[l - lm];
    e.ld[l] = bf.rt.max_size(l);
    e.P[l] = Rl.P;
    e.buf[l].reset(c, (size_t)std::max<int64_t>(1, NB * e.ld[l] * std::max(1, e.P[l])));
    e.buf[l].zero();
    if (e.P[l] == 0 || e.P[l + 1] == 0) continue;
    std::vector<GemmEnt> ents;
    for (int64_t tau = 0; tau < (int64_t(1) << l); ++tau)
      for (int64_t nu = 0; nu < (int64_t(1) << (L - l)); ++nu) {
        const int64_t i = bidx(L, l, tau, nu);
        const int64_t base = i * e.ld[l] * e.P[l];
        for (int h = 0; h < 2; ++h) {
          const int64_t child = bidx(L, l + 1, 2 * tau + h, nu / 2);
          const int64_t rows = bf.rt.size(l + 1, 2 * tau + h);
          const int64_t roff = h == 0 ? 0 : bf.rt.size(l + 1, 2 * tau);
          ents.push_back(gent(child * e.ld[l + 1] * e.P[l + 1], i * Rl.stride() + h * Rl.gap, base + roff, e.P[l],
                              (int)rows));
        }
      }
    DBuf<GemmEnt> d = to_device(c, ents);
    launch_bgemm<R>(c, OP_N, (int)e.ld[l + 1], e.P[l + 1], 1, e.buf[l + 1].p, e.ld[l + 1], Rl.data.p, Rl.ld,
                    e.buf[l].p, e.ld[l], d.p, (int)ents.size(), e.P[l], false);
  }
  return e;
}

// V side: levels 0 .. l_m, node tree = column tree (node of level l sits at
// column-tree level L - l)
template <typename R>
Expanded<R> expand_v(Ctx* c, const DevButterfly<R>& bf) {
  const int L = bf.L, lm = bf.lm;
  const int64_t NB = bf.nb();
  Expanded<R> e;
  e.buf.resize(lm + 1);
  e.ld.assign(lm + 1, 0);
  e.P.assign(lm + 1, 0);
  e.ld[0] = bf.vleaf.ld;
  e.P[0] = bf.PV(0);
  e.buf[0].reset(c, (size_t)(NB * e.ld[0] * std::max(1, e.P[0])));
  for (int64_t i = 0; i < NB; ++i)
    launch_copy2d<R>(c, e.buf[0].p + i * e.ld[0] * e.P[0], e.ld[0], bf.vleaf.block(i), bf.vleaf.ld, e.ld[0], e.P[0]);
  for (int l = 1; l <= lm; ++l) {
    const Level<R>& Wl = bf.w[l - 1];
    e.ld[l] = bf.ct.max_size(L - l);
    e.P[l] = Wl.P;
    e.buf[l].reset(c, (size_t)std::max<int64_t>(1, NB * e.ld[l] * std::max(1, e.P[l])));
    e.buf[l].zero();
    if (e.P[l] == 0 || e.P[l - 1] == 0) continue;
    std::vector<GemmEnt> ents;
    for (int64_t tau = 0; tau < (int64_t(1) << l); ++tau)
      for (int64_t nu = 0; nu < (int64_t(1) << (L - l)); ++nu) {
        const int64_t i = bidx(L, l, tau, nu);
        const int64_t base = i * e.ld[l] * e.P[l];
        for (int h = 0; h < 2; ++h) {
          const int64_t child = bidx(L, l - 1, tau / 2, 2 * nu + h);
          const int64_t rows = bf.ct.size(L - l + 1, 2 * nu + h);
          const int64_t roff = h == 0 ? 0 : bf.ct.size(L - l + 1, 2 * nu);
          ents.push_back(gent(child * e.ld[l - 1] * e.P[l - 1], i * Wl.stride() + h * Wl.gap, base + roff, e.P[l],
                              (int)rows));
        }
      }
    DBuf<GemmEnt> d = to_device(c, ents);
    launch_bgemm<R>(c, OP_N, (int)e.ld[l - 1], e.P[l - 1], 1, e.buf[l - 1].p, e.ld[l - 1], Wl.data.p, Wl.ld,
                    e.buf[l].p, e.ld[l], d.p, (int)ents.size(), e.P[l], false);
  }
  return e;
}

// sum_b || K_b - B_b B_b^H K_b ||^2 over the 2^L blocks (row node level lr of
// `rows_tree`, column node level lc of `cols_tree`) of the m x n matrix K
// (ld m), basis block of (row node r, col node s) = bases(r, s)
template <typename R, typename BlockIndex>
double one_sided(Ctx* c, const cx<R>* K, int64_t m, int64_t n, const Tree& rows_tree, int lr, const Tree& cols_tree,
                 int lc, const cx<R>* E, int64_t ldE, int P, BlockIndex block_of) {
  if (P == 0) return sumsq_diff<R>(c, K, (const cx<R>*)nullptr, m * n);
  const int64_t nr = int64_t(1) << lr, ns = int64_t(1) << lc;
  // c1 (per block P x |S|) at block offset, columns packed per row node: for
  // row node r the c1 blocks of all s are contiguous (ld P, n columns)
  DBuf<cx<R>> c1(c, (size_t)(nr * (int64_t)P * n));
  DBuf<cx<R>> proj(c, (size_t)(m * n));
  std::vector<GemmEnt> e1, e2;
  int maxS = 1;
  for (int64_t r = 0; r < nr; ++r)
    for (int64_t s = 0; s < ns; ++s) {
      const int64_t rb = rows_tree.begin(lr, r), nrr = rows_tree.size(lr, r);
      const int64_t cb = cols_tree.begin(lc, s), ncs = cols_tree.size(lc, s);
      const int64_t blk = block_of(r, s);
      maxS = std::max<int>(maxS, (int)ncs);
      // c1 = E^H K_b  (P x |S|)
      e1.push_back(gent(blk * ldE * P, rb + cb * m, r * (int64_t)P * n + cb * P, (int)ncs, BIG, (int)nrr));
      // proj_b = E c1  (|T| x |S|)
      e2.push_back(gent(blk * ldE * P, r * (int64_t)P * n + cb * P, rb + cb * m, (int)ncs, (int)nrr, BIG));
    }
  DBuf<GemmEnt> d1 = to_device(c, e1), d2 = to_device(c, e2);
  launch_bgemm<R>(c, OP_H, P, (int)ldE, 1, E, ldE, K, m, c1.p, P, d1.p, (int)e1.size(), maxS, false);
  launch_bgemm<R>(c, OP_N, (int)ldE, P, 1, E, ldE, c1.p, P, proj.p, m, d2.p, (int)e2.size(), maxS, false);
  return sumsq_diff<R>(c, K, proj.p, m * n);
}

}  // namespace

template <typename R>
Residuals compute_residuals(Ctx* c, DevOp<R>* op, const DevButterfly<R>& bf) {
  const int64_t m = op->m, n = op->n;
  if (bf.m() != m || bf.n() != n) fail(DIMENSION, "residuals: butterfly and operator dimensions differ");
  const int L = bf.L, lm = bf.lm;
  // ---- dense K in tree order (rows and columns)
  DBuf<cx<R>> kt(c, (size_t)(m * n));
  {
    const int64_t cbatch = 256;
    DBuf<cx<R>> X(c, (size_t)(n * cbatch)), Y(c, (size_t)(m * cbatch));
    DBuf<int64_t> cperm, rperm;
    if (!bf.ct.identity) cperm = to_device(c, bf.ct.perm);
    if (!bf.rt.identity) rperm = to_device(c, bf.rt.perm);
    for (int64_t j0 = 0; j0 < n; j0 += cbatch) {
      const int64_t q = std::min(cbatch, n - j0);
      identity_cols_kernel<R><<<(unsigned)std::min<int64_t>(ceil_div(n * q, (int64_t)256), c->sm_count * 16), 256, 0,
                                c->stream>>>(X.p, n, j0, q, cperm.p);
      BFLY_LAUNCH_CHECK("identity_cols");
      if (bf.rt.identity) {
        op->apply_dense(OP_N, X.p, n, kt.p + j0 * m, m, q);
      } else {
        op->apply_dense(OP_N, X.p, n, Y.p, m, q);
        launch_permute_rows<R>(c, kt.p + j0 * m, m, Y.p, m, m, q, rperm.p, false);
      }
    }
  }
  Residuals out;
  out.knorm2 = sumsq_diff<R>(c, kt.p, (const cx<R>*)nullptr, m * n);
  // ---- U side, l = L .. l_m (blocks: row node tau at level l, column node nu at level L-l)
  Expanded<R> U = expand_u(c, bf);
  for (int l = L; l >= lm; --l)
    out.u.push_back(one_sided<R>(c, kt.p, m, n, bf.rt, l, bf.ct, L - l, U.buf[l].p, U.ld[l], U.P[l],
                                 [&](int64_t tau, int64_t nu) { return bidx(L, l, tau, nu); }));
  // ---- V side on K^H, l = 0 .. l_m (rows: column node nu at level L-l)
  Expanded<R> Vx = expand_v(c, bf);
  {
    DBuf<cx<R>> kh(c, (size_t)(m * n));
    conj_transpose_kernel<R><<<(unsigned)std::min<int64_t>(ceil_div(m * n, (int64_t)256), c->sm_count * 16), 256, 0,
                               c->stream>>>(kt.p, m, m, n, kh.p, n);
    BFLY_LAUNCH_CHECK("conj_transpose");
    for (int l = 0; l <= lm; ++l)
      out.v.push_back(one_sided<R>(c, kh.p, n, m, bf.ct, L - l, bf.rt, l, Vx.buf[l].p, Vx.ld[l], Vx.P[l],
                                   [&](int64_t nu, int64_t tau) { return bidx(L, l, tau, nu); }));
  }
  // ---- center: K_b - U (U^H K_b V) V^H
  {
    const int l = lm;
    const int Pu = U.P[l], Pv = Vx.P[l];
    const int64_t nt = int64_t(1) << l, nn = int64_t(1) << (L - l);
    const int64_t ldu = U.ld[l], ldv = Vx.ld[l];
    if (Pu == 0 || Pv == 0) {
      out.center = out.knorm2;
    } else {
      DBuf<cx<R>> c1(c, (size_t)(nt * (int64_t)Pu * n)), c2(c, (size_t)(bf.nb() * (int64_t)Pu * Pv));
      DBuf<cx<R>> vh(c, (size_t)(bf.nb() * (int64_t)Pv * ldv)), c3(c, (size_t)(nt * (int64_t)Pu * n));
      DBuf<cx<R>> proj(c, (size_t)(m * n));
      // V^H blocks (Pv x ld_v)
      for (int64_t i = 0; i < bf.nb(); ++i) {
        conj_transpose_kernel<R><<<(unsigned)ceil_div(ldv * Pv, (int64_t)256), 256, 0, c->stream>>>(
            Vx.buf[l].p + i * ldv * Pv, ldv, ldv, Pv, vh.p + i * Pv * ldv, Pv);
      }
      BFLY_LAUNCH_CHECK("conj_transpose");
      std::vector<GemmEnt> e1, e2, e3, e4;
      int maxS = 1;
      for (int64_t tau = 0; tau < nt; ++tau)
        for (int64_t nu = 0; nu < nn; ++nu) {
          const int64_t i = bidx(L, l, tau, nu);
          const int64_t rb = bf.rt.begin(l, tau), nrr = bf.rt.size(l, tau);
          const int64_t cb = bf.ct.begin(L - l, nu), ncs = bf.ct.size(L - l, nu);
          maxS = std::max<int>(maxS, (int)ncs);
          const int64_t c1off = tau * (int64_t)Pu * n + cb * Pu;
          e1.push_back(gent(i * ldu * Pu, rb + cb * m, c1off, (int)ncs, BIG, (int)nrr));          // c1 = U^H K_b
          e2.push_back(gent(c1off, i * ldv * Pv, i * (int64_t)Pu * Pv, Pv, BIG, (int)ncs));      // c2 = c1 V
          e3.push_back(gent(i * (int64_t)Pu * Pv, i * Pv * ldv, c1off, (int)ncs, BIG, BIG));     // c3 = c2 V^H
          e4.push_back(gent(i * ldu * Pu, c1off, rb + cb * m, (int)ncs, (int)nrr, BIG));          // proj = U c3
        }
      DBuf<GemmEnt> d1 = to_device(c, e1), d2 = to_device(c, e2), d3 = to_device(c, e3), d4 = to_device(c, e4);
      launch_bgemm<R>(c, OP_H, Pu, (int)ldu, 1, U.buf[l].p, ldu, kt.p, m, c1.p, Pu, d1.p, (int)e1.size(), maxS, false);
      launch_bgemm<R>(c, OP_N, Pu, (int)ldv, 1, c1.p, Pu, Vx.buf[l].p, ldv, c2.p, Pu, d2.p, (int)e2.size(), Pv, false);
      c3.zero();
      launch_bgemm<R>(c, OP_N, Pu, Pv, 1, c2.p, Pu, vh.p, Pv, c3.p, Pu, d3.p, (int)e3.size(), maxS, false);
      launch_bgemm<R>(c, OP_N, (int)ldu, Pu, 1, U.buf[l].p, ldu, c3.p, Pu, proj.p, m, d4.p, (int)e4.size(), maxS,
                      false);
      out.center = sumsq_diff<R>(c, kt.p, proj.p, m * n);
    }
  }
  return out;
}

template Residuals compute_residuals<double>(Ctx*, DevOp<double>*, const DevButterfly<double>&);
template Residuals compute_residuals<float>(Ctx*, DevOp<float>*, const DevButterfly<float>&);

}  // namespace bfly
