// operators.cu -- device black boxes: kernel-evaluated (NUFFT, plates,
// circle), dense, composition, butterfly and user callback.
#include <algorithm>

#include "operators.h"

namespace bfly {

template <typename R>
DBuf<cx<R>> DevOp<R>::pad_probes(int mode, const cx<R>* X, const std::vector<MatvecSeg>& segs, int64_t& c0,
                                 int64_t& w) {
  int64_t lo = INT64_MAX, hi = 0;
  for (const auto& s : segs) {
    lo = std::min<int64_t>(lo, s.col0);
    hi = std::max<int64_t>(hi, s.col0 + s.ncols);
  }
  c0 = segs.empty() ? 0 : lo;
  w = std::max<int64_t>(hi - c0, 0);
  const int64_t nin = in_dim(mode);
  DBuf<cx<R>> p(ctx, (size_t)(nin * std::max<int64_t>(w, 1)));
  p.zero();
  for (const auto& s : segs)
    if (s.rows > 0 && s.ncols > 0)
      launch_copy2d<R>(ctx, p.p + s.row0 + (s.col0 - c0) * nin, nin, X + s.x_off, s.ldx, s.rows, s.ncols);
  return p;
}

// A padded product writes every column of the span it is given, so a group of
// segments is cut into runs that tile a column range without gaps: the
// pieces of a probe split across ranks own interleaved column ranges of Y,
// and a run must not overwrite the columns of another group with zeros.
std::vector<std::vector<MatvecSeg>> column_runs(std::vector<MatvecSeg> segs) {
  std::sort(segs.begin(), segs.end(), [](const MatvecSeg& a, const MatvecSeg& b) { return a.col0 < b.col0; });
  std::vector<std::vector<MatvecSeg>> runs;
  int64_t end = -1;
  for (const auto& s : segs) {
    if (s.ncols <= 0) continue;
    if (runs.empty() || s.col0 != end) runs.emplace_back();
    runs.back().push_back(s);
    end = s.col0 + s.ncols;
  }
  return runs;
}

namespace {

// ------------------------------------------------ kernel-evaluated ops
template <typename R>
struct KernelOp : DevOp<R> {
  DBuf<double> tx, ty, tz, sx, sy, sz;
  double kappa = 0;
  bool restricts_rows() const override { return true; }
  void do_apply(int mode, const cx<R>* X, const std::vector<MatvecSeg>& segs, cx<R>* Y, int64_t ldy, int64_t o0,
                int64_t o1) override {
    Points tp{tx.p, ty.p, tz.p}, sp{sx.p, sy.p, sz.p};
    Points outp = mode == OP_N ? tp : sp, inp = mode == OP_N ? sp : tp;
    outp.x += o0;
    outp.y += o0;
    outp.z += o0;
    const int64_t mout = o1 - o0;
    for (const auto& s : segs) {
      this->evals += (double)mout * (double)s.rows;
      this->flops += 8.0 * (double)mout * (double)s.rows * (double)s.ncols;
    }
    launch_kernel_matvec<R>(this->ctx, this->kind, mode, outp, inp, kappa, mout, X, Y + o0, ldy, segs.data(),
                            (int)segs.size());
  }
};

// ---------------------------------------------------------- dense op
template <typename R>
struct DenseOp : DevOp<R> {
  DBuf<cx<R>> a;  // m x n column major
  bool restricts_rows() const override { return true; }
  void do_apply(int mode, const cx<R>* X, const std::vector<MatvecSeg>& segs, cx<R>* Y, int64_t ldy, int64_t o0,
                int64_t o1) override {
    Ctx* c = this->ctx;
    const int64_t m = this->m;
    for (const auto& s : segs) {
      const int64_t mout = o1 - o0;
      if (s.ncols <= 0) continue;
      if (s.rows <= 0) {
        BFLY_CUDA(cudaMemset2DAsync(Y + o0 + s.col0 * ldy, ldy * sizeof(cx<R>), 0, mout * sizeof(cx<R>), s.ncols,
                                    c->stream));
        continue;
      }
      GemmEnt e{};
      e.a0 = mode == OP_N ? s.row0 * m + o0 : s.row0 + o0 * m;
      e.b0 = 0;
      e.c = 0;
      e.ncols = s.ncols;
      e.mrows = 1 << 30;
      e.krows = 1 << 30;
      DBuf<GemmEnt> de = to_device(c, std::vector<GemmEnt>{e});
      launch_bgemm<R>(c, mode, (int)mout, (int)s.rows, 1, a.p, m, X + s.x_off, s.ldx, Y + o0 + s.col0 * ldy, ldy, de.p, 1,
                      s.ncols, false);
      this->flops += 8.0 * (double)mout * (double)s.rows * (double)s.ncols;
    }
  }
};

// ---------------------------------------------------- composition op
template <typename R>
struct ComposeOp : DevOp<R> {
  std::unique_ptr<DevOp<R>> f1, f2;  // A = f2 * f1
  void do_apply(int mode, const cx<R>* X, const std::vector<MatvecSeg>& segs, cx<R>* Y, int64_t ldy, int64_t o0,
                int64_t o1) override {
    DevOp<R>* first = mode == OP_N ? f1.get() : f2.get();
    DevOp<R>* second = mode == OP_N ? f2.get() : f1.get();
    const int64_t mid = first->out_dim(mode);
    int64_t wtot = 0;
    for (const auto& s : segs) wtot = std::max<int64_t>(wtot, s.col0 + s.ncols);
    DBuf<cx<R>> t(this->ctx, (size_t)(mid * std::max<int64_t>(wtot, 1)));
    double f0 = first->flops + second->flops, e0 = first->evals + second->evals;
    first->apply_segs(mode, X, segs, t.p, mid);
    std::vector<MatvecSeg> dense;
    for (const auto& s : segs) dense.push_back(MatvecSeg{0, mid, s.col0 * mid, mid, s.col0, s.ncols, 0});
    second->apply_segs(mode, t.p, dense, Y, ldy, o0, o1);
    this->flops += first->flops + second->flops - f0;
    this->evals += first->evals + second->evals - e0;
  }
};

// ------------------------------------------------------ butterfly op
template <typename R>
struct ButterflyOp : DevOp<R> {
  std::unique_ptr<DevButterfly<R>> bf;
  void do_apply(int mode, const cx<R>* X, const std::vector<MatvecSeg>& segs, cx<R>* Y, int64_t ldy, int64_t o0,
                int64_t o1) override {
    if (structured(mode, X, segs, Y, ldy, o0, o1)) {
      this->last_restricted = true;
      return;
    }
    // a basis projection was expected (BasisProj) and no product buffer came
    // along: nothing is computed, the caller multiplies again the plain way
    if (!Y) return;
    for (const auto& run : column_runs(segs)) {
      int64_t c0 = 0, w = 0;
      DBuf<cx<R>> xp = this->pad_probes(mode, X, run, c0, w);
      if (w <= 0) continue;
      bf->apply(mode, xp.p, this->in_dim(mode), Y + c0 * ldy, ldy, w);
      this->flops += bf->apply_flops(w);
    }
  }
  // G levels of the factorization in progress (BasisProj, operators.h), built
  // level by level as its transfer levels complete:
  //   V side: G(0) = Vn_leaf^H V_leaf;  G(j) = Wn_j^H blockdiag(G(j-1) children) W_j
  //   U side: G(L) = Un_leaf^H U_leaf;  G(j) = Rn_j^H blockdiag(G(j+1) children) R_j
  // (n = the new butterfly).  Two batched GEMMs per level.
  const DevButterfly<R>* g_owner = nullptr;
  uint64_t g_gen = 0;
  std::vector<std::unique_ptr<Level<R>>> gv, gu;  // gv[j] = level j; gu[k] = level L - k
  bool can_project(int mode, const BasisProj<R>& lp) override {
    static const bool off = std::getenv("BFLY_NO_STRUCT_APPLY") != nullptr;
    return !off && basis_product(mode, lp) != nullptr;
  }
  const Level<R>* basis_product(int mode, const BasisProj<R>& lp) {
    static const bool off = std::getenv("BFLY_NO_LEAF_FUSE") != nullptr;
    const DevButterfly<R>* nb = lp.nbf;
    if (off || !nb || !lp.C) return nullptr;
    const int L = bf->L, lm = bf->lm;
    if (nb->L != L || nb->lm != lm || !nb->rt.identity || !nb->ct.identity || !bf->rt.identity || !bf->ct.identity ||
        nb->rt.ranges != bf->rt.ranges || nb->ct.ranges != bf->ct.ranges)
      return nullptr;
    if (g_owner != nb || g_gen != lp.gen) {
      gv.clear();
      gu.clear();
      g_owner = nb;
      g_gen = lp.gen;
    }
    Ctx* c = this->ctx;
    const int64_t NB = bf->nb();
    const int BIG = 1 << 30;
    auto gent = [](int64_t a0, int64_t b0, int64_t cc, int krows) {
      GemmEnt e{};
      e.a0 = a0; e.b0 = b0; e.c = cc;
      e.mrows = 1 << 30; e.krows = krows;
      return e;
    };
    auto gemm = [&](int op, int M, int K, const cx<R>* A, int64_t lda, const cx<R>* B, int64_t ldb, cx<R>* C,
                    int64_t ldc, std::vector<GemmEnt>& e, int ncols) {
      if (e.empty() || M <= 0 || K <= 0 || ncols <= 0) return;
      for (auto& x : e) x.ncols = ncols;
      DBuf<GemmEnt> de = to_device(c, e);
      launch_bgemm<R>(c, op, M, K, 1, A, lda, B, ldb, C, ldc, de.p, (int)e.size(), ncols, false, ncols);
    };
    auto fresh = [&](int Pn, int Pi) {
      auto lv = std::make_unique<Level<R>>();
      lv->alloc(c, NB, std::max(Pn, 1), std::max(Pi, 1));
      lv->P = Pn;
      lv->data.zero();
      return lv;
    };
    if (mode == OP_H) {  // V side
      if (lp.level < 0 || lp.level >= lm) return nullptr;
      while ((int)gv.size() <= lp.level) {
        const int j = (int)gv.size();
        const int Pn = nb->PV(j), Pi = bf->PV(j);
        if (Pn <= 0 || Pi <= 0) return nullptr;
        auto g = fresh(Pn, Pi);
        std::vector<GemmEnt> e;
        if (j == 0) {
          if (nb->vleaf.ld < bf->ct.max_size(L)) return nullptr;
          for (int64_t nu = 0; nu < NB; ++nu)
            e.push_back(gent(nu * nb->vleaf.stride(), nu * bf->vleaf.stride(), nu * g->stride(), (int)bf->ct.size(L, nu)));
          gemm(OP_H, Pn, (int)nb->vleaf.ld, nb->vleaf.data.p, nb->vleaf.ld, bf->vleaf.data.p, bf->vleaf.ld, g->data.p,
               g->ld, e, Pi);
        } else {
          const Level<R>&wi = bf->w[j - 1], &wn = nb->w[j - 1], &gp = *gv[j - 1];
          const int Pnp = nb->PV(j - 1), Pip = bf->PV(j - 1);
          DBuf<cx<R>> T(c, (size_t)(NB * 2 * Pnp * std::max(Pi, 1)));
          T.zero();
          const int64_t tst = (int64_t)2 * Pnp * Pi;
          for (int64_t tau = 0; tau < (int64_t(1) << j); ++tau)
            for (int64_t nu = 0; nu < (int64_t(1) << (L - j)); ++nu) {
              const int64_t i = bidx(L, j, tau, nu);
              for (int h = 0; h < 2; ++h)
                e.push_back(gent(bidx(L, j - 1, tau / 2, 2 * nu + h) * gp.stride(), i * wi.stride() + h * wi.gap,
                                 i * tst + h * Pnp, BIG));
            }
          gemm(OP_N, Pnp, Pip, gp.data.p, gp.ld, wi.data.p, wi.ld, T.p, 2 * Pnp, e, Pi);
          std::vector<GemmEnt> e2;
          for (int64_t i = 0; i < NB; ++i) e2.push_back(gent(i * wn.stride(), i * tst, i * g->stride(), BIG));
          gemm(OP_H, Pn, 2 * Pnp, wn.data.p, wn.ld, T.p, 2 * Pnp, g->data.p, g->ld, e2, Pi);
        }
        for (int64_t tau = 0; tau < (int64_t(1) << j); ++tau)
          for (int64_t nu = 0; nu < (int64_t(1) << (L - j)); ++nu) {
            const int64_t i = bidx(L, j, tau, nu);
            g->ranks[i] = nb->v_rank(j, tau, nu);
            g->rows[i] = bf->v_rank(j, tau, nu);
          }
        gv.push_back(std::move(g));
      }
      return gv[lp.level].get();
    }
    if (mode != OP_N || lp.level <= lm || lp.level > L) return nullptr;
    while ((int)gu.size() <= L - lp.level) {  // U side
      const int j = L - (int)gu.size();
      const int Pn = nb->PU(j), Pi = bf->PU(j);
      if (Pn <= 0 || Pi <= 0) return nullptr;
      auto g = fresh(Pn, Pi);
      std::vector<GemmEnt> e;
      if (j == L) {
        if (nb->uleaf.ld < bf->rt.max_size(L)) return nullptr;
        for (int64_t tau = 0; tau < NB; ++tau)
          e.push_back(gent(tau * nb->uleaf.stride(), tau * bf->uleaf.stride(), tau * g->stride(), (int)bf->rt.size(L, tau)));
        gemm(OP_H, Pn, (int)nb->uleaf.ld, nb->uleaf.data.p, nb->uleaf.ld, bf->uleaf.data.p, bf->uleaf.ld, g->data.p,
             g->ld, e, Pi);
      } else {
        const Level<R>&ri = bf->r[j - lm], &rn = nb->r[j - lm], &gp = *gu[L - (j + 1)];
        const int Pnp = nb->PU(j + 1), Pip = bf->PU(j + 1);
        DBuf<cx<R>> T(c, (size_t)(NB * 2 * Pnp * std::max(Pi, 1)));
        T.zero();
        const int64_t tst = (int64_t)2 * Pnp * Pi;
        for (int64_t tau = 0; tau < (int64_t(1) << j); ++tau)
          for (int64_t nu = 0; nu < (int64_t(1) << (L - j)); ++nu) {
            const int64_t i = bidx(L, j, tau, nu);
            for (int h = 0; h < 2; ++h)
              e.push_back(gent(bidx(L, j + 1, 2 * tau + h, nu / 2) * gp.stride(), i * ri.stride() + h * ri.gap,
                               i * tst + h * Pnp, BIG));
          }
        gemm(OP_N, Pnp, Pip, gp.data.p, gp.ld, ri.data.p, ri.ld, T.p, 2 * Pnp, e, Pi);
        std::vector<GemmEnt> e2;
        for (int64_t i = 0; i < NB; ++i) e2.push_back(gent(i * rn.stride(), i * tst, i * g->stride(), BIG));
        gemm(OP_H, Pn, 2 * Pnp, rn.data.p, rn.ld, T.p, 2 * Pnp, g->data.p, g->ld, e2, Pi);
      }
      for (int64_t tau = 0; tau < (int64_t(1) << j); ++tau)
        for (int64_t nu = 0; nu < (int64_t(1) << (L - j)); ++nu) {
          const int64_t i = bidx(L, j, tau, nu);
          g->ranks[i] = nb->u_rank(j, tau, nu);
          g->rows[i] = bf->u_rank(j, tau, nu);
        }
      gu.push_back(std::move(g));
    }
    return gu[L - lp.level].get();
  }
  // Probes supported on the nodes of one level of this butterfly's own
  // input-side tree (a recompression over the same trees): blocks the zero
  // rows cannot reach are skipped (DevButterfly::apply_structured), and the
  // flops counted are the ones executed.  BFLY_NO_STRUCT_APPLY=1 keeps the
  // reference's padded products.
  bool structured(int mode, const cx<R>* X, const std::vector<MatvecSeg>& segs, cx<R>* Y, int64_t ldy, int64_t o0,
                  int64_t o1) {
    static const bool off = std::getenv("BFLY_NO_STRUCT_APPLY") != nullptr;
    if (off || segs.empty() || (mode != OP_N && mode != OP_H)) return false;
    const Tree& pt = mode == OP_N ? bf->ct : bf->rt;
    if (!pt.identity || segs[0].rows >= pt.n) return false;  // dense probes (leaf phases): the plain apply
    int p = -1;
    for (int l = 1; l <= bf->L && p < 0; ++l) {
      const auto& rg = pt.ranges[l];
      auto it = std::lower_bound(rg.begin(), rg.end(), segs[0].row0);
      if (it != rg.end() && *it == segs[0].row0 && it + 1 != rg.end() && *(it + 1) == segs[0].row0 + segs[0].rows)
        p = l;
    }
    if (p < 0) return false;
    std::vector<typename DevButterfly<R>::ProbeSeg> ps;
    const auto& rg = pt.ranges[p];
    bool uniform = true;
    int64_t maxrows = 0, cols = 0;
    for (const auto& s : segs) {
      auto it = std::lower_bound(rg.begin(), rg.end(), s.row0);
      if (it == rg.end() || *it != s.row0 || it + 1 == rg.end() || *(it + 1) != s.row0 + s.rows) return false;
      ps.push_back({(int64_t)(it - rg.begin()), s.x_off, s.col0, s.ncols});
      uniform = uniform && s.ldx == segs[0].ldx;
      maxrows = std::max(maxrows, s.rows);
      cols += std::max<int64_t>(s.ncols, 0);
    }
    // ragged nodes: the compact probes get one common leading dimension
    DBuf<cx<R>> tmp;
    const cx<R>* Xs = X;
    int64_t ld = segs[0].ldx;
    if (!uniform) {
      tmp.reset(this->ctx, (size_t)std::max<int64_t>(1, maxrows * cols));
      int64_t off = 0;
      for (size_t i = 0; i < segs.size(); ++i) {
        const auto& s = segs[i];
        if (s.rows > 0 && s.ncols > 0)
          launch_copy2d<R>(this->ctx, tmp.p + off, maxrows, X + s.x_off, s.ldx, s.rows, s.ncols);
        ps[i].x_off = off;
        off += maxrows * std::max<int64_t>(s.ncols, 0);
      }
      Xs = tmp.p;
      ld = maxrows;
    }
    std::sort(ps.begin(), ps.end(), [](const auto& a, const auto& b) { return a.node < b.node; });
    double fl = 0;
    BasisProj<R>* lp = this->cur_lp;
    // (BFLY_DEBUG_REJECT_PROJ: test hook -- decline every offered projection so the caller's retry runs)
    static const bool reject = std::getenv("BFLY_DEBUG_REJECT_PROJ") != nullptr;
    const Level<R>* G = lp && !reject ? basis_product(mode, *lp) : nullptr;
    if (!G && !Y) return false;  // neither a projection nor a product buffer: see do_apply
    if (!bf->apply_structured(mode, p, ps, Xs, ld, Y, ldy, o0, o1, &fl, G, lp ? lp->level : 0, G ? lp->C : nullptr,
                              G ? lp->ldc : 0))
      return false;
    if (lp) lp->done = G != nullptr;
    this->flops += fl;
    return true;
  }
};

// ------------------------------------------------------- callback op
template <typename R>
struct CallbackOp : DevOp<R> {
  bfly_apply_fn fn = nullptr;
  void* user = nullptr;
  void do_apply(int mode, const cx<R>* X, const std::vector<MatvecSeg>& segs, cx<R>* Y, int64_t ldy, int64_t o0,
                int64_t o1) override {
    Ctx* c = this->ctx;
    const int64_t nin = this->in_dim(mode), nout = this->out_dim(mode);
    for (const auto& run : column_runs(segs)) {
      int64_t c0 = 0, w = 0;
      DBuf<cx<R>> xp = this->pad_probes(mode, X, run, c0, w);
      if (w <= 0) continue;
      if (mode == OP_H) launch_conj<R>(c, xp.p, nin, w, nin);
      int rc = fn(user, mode == OP_N ? 0 : 1, xp.p, nin, Y + c0 * ldy, ldy, w, (void*)c->stream);
      if (rc != 0) fail(rc, "black-box callback failed with status " + std::to_string(rc));
      if (mode == OP_H) launch_conj<R>(c, Y + c0 * ldy, nout, w, ldy);
    }
  }
};

// structured-probe-aware callback: one call per probe with its nonzero rows
template <typename R>
struct CallbackRangeOp : DevOp<R> {
  bfly_apply_range_fn fn = nullptr;
  void* user = nullptr;
  void do_apply(int mode, const cx<R>* X, const std::vector<MatvecSeg>& segs, cx<R>* Y, int64_t ldy, int64_t o0,
                int64_t o1) override {
    Ctx* c = this->ctx;
    int64_t c0 = 0, w = 0;
    DBuf<cx<R>> xp = this->pad_probes(mode, X, segs, c0, w);
    if (w <= 0) return;
    const int64_t nin = this->in_dim(mode), nout = this->out_dim(mode);
    if (mode == OP_H) launch_conj<R>(c, xp.p, nin, w, nin);
    for (const auto& s : segs) {
      if (s.ncols <= 0) continue;
      const int64_t b = s.rows > 0 ? s.row0 : 0, e = s.rows > 0 ? s.row0 + s.rows : 0;
      int rc = fn(user, mode == OP_N ? 0 : 1, xp.p + (s.col0 - c0) * nin, nin, Y + s.col0 * ldy, ldy, s.ncols, b, e,
                  (void*)c->stream);
      if (rc != 0) fail(rc, "black-box callback failed with status " + std::to_string(rc));
      if (mode == OP_H) launch_conj<R>(c, Y + s.col0 * ldy, nout, s.ncols, ldy);
    }
  }
};

std::vector<double> column(const double* p, int64_t n, int axis) {
  std::vector<double> v(n);
  for (int64_t i = 0; i < n; ++i) v[i] = p[i * 3 + axis];
  return v;
}

}  // namespace

template <typename R>
std::unique_ptr<DevOp<R>> make_kernel_op(Ctx* c, int kind, int64_t m, int64_t n, const double* tgt, const double* src,
                                         double kappa) {
  if (kind != KK_NUFFT && kind != KK_PLATES && kind != KK_CIRCLE) fail(PRECONDITION, "unknown kernel operator kind");
  if (m < 1 || n < 1) fail(PRECONDITION, "kernel operator: empty point set");
  auto op = std::make_unique<KernelOp<R>>();
  op->kind = kind;
  op->m = m;
  op->n = n;
  op->ctx = c;
  op->kappa = kappa;
  op->tx = to_device(c, column(tgt, m, 0));
  op->ty = to_device(c, column(tgt, m, 1));
  op->tz = to_device(c, column(tgt, m, 2));
  op->sx = to_device(c, column(src, n, 0));
  op->sy = to_device(c, column(src, n, 1));
  op->sz = to_device(c, column(src, n, 2));
  c->sync();
  return op;
}

template <typename R>
std::unique_ptr<DevOp<R>> make_dense_op(Ctx* c, int64_t m, int64_t n, const std::vector<cx<R>>& a, bool is_real) {
  auto op = std::make_unique<DenseOp<R>>();
  op->kind = 0;
  op->m = m;
  op->n = n;
  op->ctx = c;
  op->is_real = is_real;
  op->a = to_device(c, a);
  c->sync();
  return op;
}

template <typename R>
std::unique_ptr<DevOp<R>> make_compose_op(Ctx* c, std::unique_ptr<DevOp<R>> f2, std::unique_ptr<DevOp<R>> f1) {
  if (f2->n != f1->m) fail(DIMENSION, "composition: inner dimensions differ");
  auto op = std::make_unique<ComposeOp<R>>();
  op->kind = 4;
  op->m = f2->m;
  op->n = f1->n;
  op->ctx = c;
  op->is_real = f1->is_real && f2->is_real;
  op->f1 = std::move(f1);
  op->f2 = std::move(f2);
  return op;
}

template <typename R>
std::unique_ptr<DevOp<R>> make_butterfly_op(Ctx* c, std::unique_ptr<DevButterfly<R>> bf) {
  auto op = std::make_unique<ButterflyOp<R>>();
  op->kind = 5;
  op->m = bf->m();
  op->n = bf->n();
  op->ctx = c;
  op->is_real = bf->is_real;
  op->bf = std::move(bf);
  return op;
}

template <typename R>
std::unique_ptr<DevOp<R>> make_callback_op(Ctx* c, int64_t m, int64_t n, bool is_real, bfly_apply_fn fn, void* user) {
  if (!fn) fail(PRECONDITION, "callback operator: null function");
  auto op = std::make_unique<CallbackOp<R>>();
  op->kind = 6;
  op->m = m;
  op->n = n;
  op->ctx = c;
  op->is_real = is_real;
  op->fn = fn;
  op->user = user;
  return op;
}

template <typename R>
std::unique_ptr<DevOp<R>> make_callback_range_op(Ctx* c, int64_t m, int64_t n, bool is_real, bfly_apply_range_fn fn,
                                                 void* user) {
  if (!fn) fail(PRECONDITION, "callback operator: null function");
  auto op = std::make_unique<CallbackRangeOp<R>>();
  op->kind = 6;
  op->m = m;
  op->n = n;
  op->ctx = c;
  op->is_real = is_real;
  op->fn = fn;
  op->user = user;
  return op;
}

template <typename R>
DevButterfly<R>* butterfly_of(DevOp<R>* op) {
  auto* b = dynamic_cast<ButterflyOp<R>*>(op);
  return b ? b->bf.get() : nullptr;
}

#define INST(R)                                                                                                  \
  template struct DevOp<R>;                                                                                      \
  template std::unique_ptr<DevOp<R>> make_kernel_op<R>(Ctx*, int, int64_t, int64_t, const double*, const double*, \
                                                       double);                                                  \
  template std::unique_ptr<DevOp<R>> make_dense_op<R>(Ctx*, int64_t, int64_t, const std::vector<cx<R>>&, bool);  \
  template std::unique_ptr<DevOp<R>> make_compose_op<R>(Ctx*, std::unique_ptr<DevOp<R>>, std::unique_ptr<DevOp<R>>); \
  template std::unique_ptr<DevOp<R>> make_butterfly_op<R>(Ctx*, std::unique_ptr<DevButterfly<R>>);                \
  template std::unique_ptr<DevOp<R>> make_callback_op<R>(Ctx*, int64_t, int64_t, bool, bfly_apply_fn, void*);      \
  template std::unique_ptr<DevOp<R>> make_callback_range_op<R>(Ctx*, int64_t, int64_t, bool, bfly_apply_range_fn,     \
                                                               void*);                                            \
  template DevButterfly<R>* butterfly_of<R>(DevOp<R>*);
INST(double)
INST(float)
#undef INST

}  // namespace bfly
