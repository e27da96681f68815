// ref_capi.cpp -- ORACLE (test infrastructure): the reference implementation
// itself (/root/reference/proj/include/bfly, compiled unmodified against the
// Eigen-API shim) driven through a small C API, used to pin the C oracle and
// as the "reference" CPU baseline.  The BASELINE operators are new
// BlackBoxOperator subclasses (operators.hpp:17-56 contract; entry formulas
// identical to oracle/bo_operators.c, no FP contraction); nothing in the
// reference tree is modified.
#include <omp.h>

#include <cmath>
#include <cstdint>
#include <cstring>
#include <memory>
#include <sstream>
#include <string>

#include "bfly/layout.hpp"
#include "bfly/reconstruct.hpp"
#include "bfly/serialize.hpp"

using namespace bfly;
using cplx = std::complex<double>;

namespace {

constexpr double kTwoPi = 6.283185307179586476925286766559;
constexpr double kFourPi = 12.566370614359172953850573533118;
thread_local std::string g_err;
int g_threads = 1;

// kernel-evaluated BASELINE operators (configs 0-2); kind: 1 nufft, 2 plates, 3 circle
class KernelOperator : public BlackBoxOperator<cplx> {
 public:
  KernelOperator(int kind, std::vector<double> tgt, std::vector<double> src, double kappa)
      : kind_(kind), t_(std::move(tgt)), s_(std::move(src)), kappa_(kappa) {}
  Index rows() const override { return (Index)t_.size() / 3; }
  Index cols() const override { return (Index)s_.size() / 3; }
  cplx entry(Index i, Index j) const {
    const double* t = &t_[3 * i];
    const double* s = &s_[3 * j];
    if (kind_ == 1) {
      double ph = t[0] * s[0];
      double f = ph - std::rint(ph);
      double ang = kTwoPi * f;
      return {std::cos(ang), std::sin(ang)};
    }
    double dx = t[0] - s[0], dy = t[1] - s[1], r;
    if (kind_ == 2) {
      double dz = t[2] - s[2];
      r = std::sqrt(std::fma(dz, dz, std::fma(dy, dy, dx * dx)));
      double ph = kappa_ * r, sc = 1.0 / (kFourPi * r);
      return {std::cos(ph) * sc, std::sin(ph) * sc};
    }
    r = std::sqrt(std::fma(dy, dy, dx * dx));
    double ph = kappa_ * r, sc = 1.0 / r;
    return {std::cos(ph) * sc, std::sin(ph) * sc};
  }

 protected:
  Mat do_apply(const Mat& x) const override { return product(x, false); }
  Mat do_apply_transpose(const Mat& y) const override { return product(y, true); }

 private:
  // skips all-zero input rows (structured probes are padded by probe_with)
  Mat product(const Mat& x, bool trans) const {
    const Index nin = x.rows(), nout = trans ? cols() : rows(), k = x.cols();
    std::vector<Index> nz;
    for (Index j = 0; j < nin; ++j)
      for (Index c = 0; c < k; ++c)
        if (x(j, c) != cplx(0)) {
          nz.push_back(j);
          break;
        }
    Mat y(nout, k);
#pragma omp parallel for schedule(dynamic, 16) num_threads(g_threads)
    for (Index i = 0; i < nout; ++i) {
      std::vector<cplx> acc(k, cplx(0));
      for (Index j : nz) {
        cplx e = trans ? entry(j, i) : entry(i, j);
        for (Index c = 0; c < k; ++c) acc[c] += e * x(j, c);
      }
      for (Index c = 0; c < k; ++c) y(i, c) = acc[c];
    }
    return y;
  }
  int kind_;
  std::vector<double> t_, s_;
  double kappa_;
};

// A = F2 F1, two sequential black-box products (config 3)
class CompositionOperator : public BlackBoxOperator<cplx> {
 public:
  CompositionOperator(std::unique_ptr<KernelOperator> f2, std::unique_ptr<KernelOperator> f1)
      : f2_(std::move(f2)), f1_(std::move(f1)) {}
  Index rows() const override { return f2_->rows(); }
  Index cols() const override { return f1_->cols(); }

 protected:
  Mat do_apply(const Mat& x) const override { return f2_->apply(f1_->apply(x)); }
  Mat do_apply_transpose(const Mat& y) const override { return f1_->apply_transpose(f2_->apply_transpose(y)); }

 private:
  std::unique_ptr<KernelOperator> f2_, f1_;
};

std::vector<double> pts(const double* p, int64_t n) { return std::vector<double>(p, p + 3 * n); }

PartitionTree tree_of(const double* p, int64_t n, int dim, int L) {
  PointSet ps;
  ps.dim = dim;
  ps.coords.resize(n);
  for (int64_t i = 0; i < n; ++i) ps.coords[i] = {p[3 * i], p[3 * i + 1], p[3 * i + 2]};
  return build_tree(ps, L);
}

// u ranks for levels center..L, then v ranks for levels 0..center (2^L each)
void rank_profile(const HybridButterfly<cplx>& bf, int32_t* out) {
  const int L = bf.levels, lm = bf.center;
  const int64_t nb = int64_t(1) << L;
  int64_t off = 0;
  for (int l = lm; l <= L; ++l, off += nb)
    for (Index t = 0; t < (Index(1) << l); ++t)
      for (Index u = 0; u < (Index(1) << (L - l)); ++u) out[off + bf.bidx(l, t, u)] = (int32_t)bf.u_rank(l, t, u);
  for (int l = 0; l <= lm; ++l, off += nb)
    for (Index t = 0; t < (Index(1) << l); ++t)
      for (Index u = 0; u < (Index(1) << (L - l)); ++u) out[off + bf.bidx(l, t, u)] = (int32_t)bf.v_rank(l, t, u);
}

struct Result {
  HybridButterfly<cplx> bf;
  FactorizationLog log;
};

template <class F>
int guard(F&& f) {
  try {
    f();
    return 0;
  } catch (const precondition_error& e) {
    g_err = e.what();
    return 1;
  } catch (const dimension_error& e) {
    g_err = e.what();
    return 2;
  } catch (const sequencing_error& e) {
    g_err = e.what();
    return 3;
  } catch (const format_error& e) {
    g_err = e.what();
    return 4;
  } catch (const conditioning_error& e) {
    g_err = e.what();
    return 5;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 9;
  }
}

}  // namespace

namespace {
template <typename BF>
void layout_of(const BF& bf, int kind, int64_t p, double* out, int32_t* owners) {
  LayoutSpec ls;
  ls.kind = (layout_kind)kind;
  ls.levels = bf.levels;
  ls.rank = 1;
  ls.processes = p;
  auto map = assign_ownership(bf, ls);
  Matrix<cplx> x = gaussian_matrix<cplx>(bf.cols(), 1, 2);
  auto res = simulated_parallel_apply(bf, x, ls);
  const auto& r = res.second;
  out[0] = r.exchange_volume;
  out[1] = (double)r.exchange_msgs;
  out[2] = r.alltoall_volume;
  out[3] = (double)r.alltoall_msgs;
  if (owners) {
    int32_t* o = owners;
    for (int v : map.u_leaf) *o++ = v;
    for (int v : map.v_leaf) *o++ = v;
    for (const auto& lv : map.r_owner)
      for (int v : lv) *o++ = v;
    for (const auto& lv : map.w_owner)
      for (int v : lv) *o++ = v;
    for (int v : map.b_owner) *o++ = v;
  }
}
}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }
void ref_set_threads(int t) { g_threads = t < 1 ? 1 : t; }

struct ref_op {
  std::unique_ptr<BlackBoxOperator<cplx>> op;
  PartitionTree rt, ct;
};
struct ref_bf {
  HybridButterfly<cplx> bf;
  FactorizationLog log;
};

// kind 1..3: tgt/src n x 3 row-major, points already in tree order; dims for the trees
int ref_op_kernel(int kind, int64_t m, int64_t n, const double* tgt, const double* src, double kappa, int dim, int L,
                  ref_op** out) {
  return guard([&] {
    auto h = std::make_unique<ref_op>();
    h->op = std::make_unique<KernelOperator>(kind, pts(tgt, m), pts(src, n), kappa);
    h->rt = tree_of(tgt, m, dim, L);
    h->ct = tree_of(src, n, dim, L);
    *out = h.release();
  });
}

// composition: f2 (x2 -> xi2), f1 (x1 -> xi1); A rows = x2, cols = xi1
int ref_op_compose(int64_t n, const double* x2, const double* xi2, const double* x1, const double* xi1, int L,
                   ref_op** out) {
  return guard([&] {
    auto h = std::make_unique<ref_op>();
    auto f2 = std::make_unique<KernelOperator>(1, pts(x2, n), pts(xi2, n), 0.0);
    auto f1 = std::make_unique<KernelOperator>(1, pts(x1, n), pts(xi1, n), 0.0);
    h->op = std::make_unique<CompositionOperator>(std::move(f2), std::move(f1));
    h->rt = tree_of(x2, n, 1, L);
    h->ct = tree_of(xi1, n, 1, L);
    *out = h.release();
  });
}

// a butterfly black box loaded from .bfh bytes (load_container path, serialize.hpp:148-177)
int ref_op_butterfly(const uint8_t* bytes, int64_t nbytes, ref_op** out) {
  return guard([&] {
    std::string s(reinterpret_cast<const char*>(bytes), (size_t)nbytes);
    std::istringstream is(s, std::ios::binary);
    HybridButterfly<cplx> bf = deserialize<cplx>(is);
    auto h = std::make_unique<ref_op>();
    h->rt = bf.row_tree;
    h->ct = bf.col_tree;
    h->op = std::make_unique<ButterflyOperator<cplx>>(std::move(bf));
    *out = h.release();
  });
}

// the reference's own synthetic butterfly (operators.hpp:131-178)
int ref_op_synth(int levels, int64_t rank, uint64_t seed, ref_op** out) {
  return guard([&] {
    SyntheticButterflySpec spec;
    spec.levels = levels;
    spec.rank = rank;
    spec.seed = seed;
    auto op = synth_butterfly_operator<cplx>(spec);
    auto h = std::make_unique<ref_op>();
    h->rt = op->butterfly().row_tree;
    h->ct = op->butterfly().col_tree;
    h->op = std::move(op);
    *out = h.release();
  });
}

void ref_op_free(ref_op* h) { delete h; }

int ref_factorize(ref_op* h, double tol, int64_t p, int64_t r0, int L, uint64_t seed, int threads, ref_bf** out) {
  return guard([&] {
    ReconstructionConfig cfg;
    cfg.tolerance = tol;
    cfg.oversampling = p;
    cfg.rank_guess = r0;
    cfg.levels = L;
    cfg.seed = seed;
    cfg.threads = threads;
    auto res = factorize<cplx>(*h->op, h->rt, h->ct, cfg);
    auto b = std::make_unique<ref_bf>();
    b->bf = std::move(res.first);
    b->log = std::move(res.second);
    *out = b.release();
  });
}

int64_t ref_rank_profile(const ref_bf* b, int32_t* out) {
  const int64_t len = (int64_t)(b->bf.levels + 2) << b->bf.levels;
  if (out) rank_profile(b->bf, out);
  return len;
}

// trans 0: bf x, 2: bf^H y ; interleaved complex, column-major
int ref_apply(const ref_bf* b, int trans, const double* x, int64_t k, double* y) {
  return guard([&] {
    const Index nin = trans ? b->bf.rows() : b->bf.cols(), nout = trans ? b->bf.cols() : b->bf.rows();
    Matrix<cplx> X(nin, k);
    std::memcpy(X.data(), x, sizeof(cplx) * nin * k);
    Matrix<cplx> Y = trans ? b->bf.apply_adjoint(X) : b->bf.apply(X);
    std::memcpy(y, Y.data(), sizeof(cplx) * nout * k);
  });
}

int ref_log(const ref_bf* b, int64_t* cols /* 2 per phase */, int32_t* rounds, int64_t* widths, double* total_s) {
  int i = 0;
  for (const auto& p : b->log.phases) {
    cols[2 * i] = p.forward_columns;
    cols[2 * i + 1] = p.transpose_columns;
    rounds[i] = p.rounds;
    widths[i] = p.probe_width;
    ++i;
  }
  *total_s = b->log.total_seconds;
  return i;
}

// PhaseStat::seconds / name (reconstruct.hpp:87-120) of every phase; returns the count
int ref_phase_seconds(const ref_bf* b, double* seconds, char* names /* 32 bytes per phase */) {
  int i = 0;
  for (const auto& p : b->log.phases) {
    if (seconds) seconds[i] = p.seconds;
    if (names) {
      std::memset(names + 32 * i, 0, 32);
      std::strncpy(names + 32 * i, p.name.c_str(), 31);
    }
    ++i;
  }
  return i;
}

double ref_estimate_error(ref_op* h, const ref_bf* b, int64_t k, uint64_t seed) {
  double e = -1;
  guard([&] { e = estimate_error<cplx>(*h->op, b->bf, k, seed); });
  return e;
}

int64_t ref_serialize(const ref_bf* b, uint8_t* buf) {
  std::string s = serialize_to_string(b->bf);
  if (buf) std::memcpy(buf, s.data(), s.size());
  return (int64_t)s.size();
}

void ref_bf_free(ref_bf* b) { delete b; }

// u_side_residual / v_side_residual / center_residual (reconstruct.hpp:443-503)
// against densify(op) (operators.hpp), as run_verify does (bfly_cli.cpp:208-235)
int ref_residuals(ref_op* h, const ref_bf* b, double* u, double* v, double* center, double* knorm2) {
  return guard([&] {
    Matrix<cplx> dense = densify(*h->op);
    *knorm2 = dense.squaredNorm();
    const int L = b->bf.levels, lm = b->bf.center;
    for (int l = L; l >= lm; --l) u[L - l] = u_side_residual(dense, b->bf, l);
    for (int l = 0; l <= lm; ++l) v[l] = v_side_residual(dense, b->bf, l);
    *center = center_residual(dense, b->bf);
  });
}

// ---- primitives for the golden vectors (tests/golden/make_golden.py)
// seed_mix(seed, words...) core.hpp:78-88 (up to 4 words)
uint64_t ref_seed_mix(uint64_t seed, int nw, const uint64_t* w) {
  switch (nw) {
    case 0: return seed_mix(seed);
    case 1: return seed_mix(seed, w[0]);
    case 2: return seed_mix(seed, w[0], w[1]);
    case 3: return seed_mix(seed, w[0], w[1], w[2]);
    default: return seed_mix(seed, w[0], w[1], w[2], w[3]);
  }
}

// gaussian_matrix<Scalar>(rows, cols, seed) linalg.hpp:16-25; complex: interleaved
int ref_gaussian(int is_complex, int64_t rows, int64_t cols, uint64_t seed, double* out) {
  return guard([&] {
    if (is_complex) {
      Matrix<cplx> g = gaussian_matrix<cplx>(rows, cols, seed);
      std::memcpy(out, g.data(), sizeof(cplx) * rows * cols);
    } else {
      Matrix<double> g = gaussian_matrix<double>(rows, cols, seed);
      std::memcpy(out, g.data(), sizeof(double) * rows * cols);
    }
  });
}

// pivoted_qr_truncate(w, eps) linalg.hpp:63-80 on a complex column-major
// matrix; q (rows x min(rows,cols)) receives the basis; returns the rank
// (-1 on error, -2 for zero input)
int64_t ref_cpqr(int64_t rows, int64_t cols, const double* w, double eps, double* q) {
  int64_t rank = -1;
  guard([&] {
    Matrix<cplx> W(rows, cols);
    std::memcpy(W.data(), w, sizeof(cplx) * rows * cols);
    OrthonormalBasis<cplx> b = pivoted_qr_truncate<cplx>(W, eps);
    rank = b.zero_input ? -2 : (int64_t)b.rank();
    if (b.rank() > 0) std::memcpy(q, b.q.data(), sizeof(cplx) * rows * b.rank());
  });
  return rank;
}

// Bounded CPU-baseline sample through the reference's own probe path:
// probe_with (padding + apply_adjoint = conj(apply_transpose(conj))) for
// `probes` row probes of tree level `level`, width `width`.  Returns seconds.
double ref_probe_sample(ref_op* h, int level, int probes, int64_t width, uint64_t seed) {
  double secs = -1;
  guard([&] {
    double t0 = omp_get_wtime();
    for (int tau = 0; tau < probes; ++tau) {
      auto probe = StructuredProbe<cplx>::row_probe(h->rt, level, tau, width, seed_mix(seed, 3, level, tau));
      auto y = probe_with(*h->op, h->rt, probe);
      (void)y;
    }
    secs = omp_get_wtime() - t0;
  });
  return secs;
}

// ---- process layouts (layout.hpp): closed-form model, ownership maps and
// the simulated sweep's tallies.  owners: (L+3) 2^L = u leaves, v leaves,
// R levels center..L-1, W levels 1..center, centre cores.
int ref_comm_cost(int kind, int levels, int64_t rank, int64_t p, double* out) {
  return guard([&] {
    LayoutSpec ls;
    ls.kind = (layout_kind)kind;
    ls.levels = levels;
    ls.rank = rank;
    ls.processes = p;
    auto r = comm_cost(ls);
    out[0] = r.exchange_volume;
    out[1] = (double)r.exchange_msgs;
    out[2] = r.alltoall_volume;
    out[3] = (double)r.alltoall_msgs;
  });
}


int ref_layout_synth(int levels, int64_t rank, uint64_t seed, int kind, int64_t p, double* out, int32_t* owners) {
  return guard([&] {
    SyntheticButterflySpec spec;
    spec.levels = levels;
    spec.rank = rank;
    spec.seed = seed;
    auto bf = synth_butterfly<cplx>(spec);
    layout_of(bf, kind, p, out, owners);
  });
}

int ref_layout_bf(const ref_bf* b, int kind, int64_t p, double* out, int32_t* owners) {
  return guard([&] { layout_of(b->bf, kind, p, out, owners); });
}

}  // extern "C"
