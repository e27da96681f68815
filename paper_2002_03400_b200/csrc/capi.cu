// capi.cu -- extern "C" boundary (include/bfly_b200.h).  No exception crosses
// it: every entry point returns a status and records the message.
#include <cstring>
#include <memory>
#include <string>

#include "../../include/bfly_b200.h"
#include "butterfly.h"
#include "layout.h"
#include "comm.h"
#include "factorizer.h"
#include "verify.h"
#include "operators.h"

using namespace bfly;

struct bfly_ctx {
  std::unique_ptr<Ctx> c;
};
struct bfly_tree {
  Tree t;
};
struct bfly_op {
  bfly_ctx* ctx = nullptr;
  int scalar = BFLY_Z;
  std::unique_ptr<DevOp<double>> z;
  std::unique_ptr<DevOp<float>> c;
  int64_t m() const { return z ? z->m : c->m; }
  int64_t n() const { return z ? z->n : c->n; }
  int kind() const { return z ? z->kind : c->kind; }
};
struct bfly_bf {
  bfly_ctx* ctx = nullptr;
  int scalar = BFLY_Z;
  std::unique_ptr<DevButterfly<double>> z;
  std::unique_ptr<DevButterfly<float>> c;
};
struct bfly_factorizer {
  bfly_ctx* ctx = nullptr;
  int scalar = BFLY_Z;
  std::unique_ptr<Factorizer<double>> z;
  std::unique_ptr<Factorizer<float>> c;
};

namespace {
thread_local std::string g_err;

template <class F>
int guard(Ctx* ctx, F&& f) {
  try {
    CtxScope scope(ctx);
    f();
    return BFLY_OK;
  } catch (const Error& e) {
    g_err = e.what();
    return e.code;
  } catch (const std::exception& e) {
    g_err = e.what();
    return BFLY_CUDA;
  }
}
Ctx* C_(bfly_ctx* c) { return c ? c->c.get() : nullptr; }

void check_scalar(int s) {
  if (s != BFLY_Z && s != BFLY_C && s != BFLY_D) fail(PRECONDITION, "unknown scalar type");
}

// host (user scalar layout) <-> device (internal storage) column-major copies
template <typename R>
void h2d(Ctx* c, int scalar, const void* h, int64_t ldh, cx<R>* d, int64_t rows, int64_t cols) {
  std::vector<cx<R>> tmp((size_t)(rows * cols));
  for (int64_t j = 0; j < cols; ++j)
    for (int64_t i = 0; i < rows; ++i) {
      if (scalar == BFLY_D) {
        double v = static_cast<const double*>(h)[i + j * ldh];
        tmp[i + j * rows] = mkc<R>((R)v, 0);
      } else if (scalar == BFLY_Z) {
        const double* p = static_cast<const double*>(h) + 2 * (i + j * ldh);
        tmp[i + j * rows] = mkc<R>((R)p[0], (R)p[1]);
      } else {
        const float* p = static_cast<const float*>(h) + 2 * (i + j * ldh);
        tmp[i + j * rows] = mkc<R>((R)p[0], (R)p[1]);
      }
    }
  BFLY_CUDA(cudaMemcpyAsync(d, tmp.data(), tmp.size() * sizeof(cx<R>), cudaMemcpyHostToDevice, c->stream));
  c->sync();
}
template <typename R>
void d2h(Ctx* c, int scalar, const cx<R>* d, int64_t rows, int64_t cols, void* h, int64_t ldh) {
  std::vector<cx<R>> tmp((size_t)(rows * cols));
  BFLY_CUDA(cudaMemcpyAsync(tmp.data(), d, tmp.size() * sizeof(cx<R>), cudaMemcpyDeviceToHost, c->stream));
  c->sync();
  for (int64_t j = 0; j < cols; ++j)
    for (int64_t i = 0; i < rows; ++i) {
      cx<R> v = tmp[i + j * rows];
      if (scalar == BFLY_D) static_cast<double*>(h)[i + j * ldh] = (double)v.x;
      else if (scalar == BFLY_Z) {
        double* p = static_cast<double*>(h) + 2 * (i + j * ldh);
        p[0] = (double)v.x;
        p[1] = (double)v.y;
      } else {
        float* p = static_cast<float*>(h) + 2 * (i + j * ldh);
        p[0] = (float)v.x;
        p[1] = (float)v.y;
      }
    }
}

// fast path for host buffers already in the internal layout (Z / C, ld == rows):
// one pinned-or-pageable cudaMemcpyAsync each way
template <typename R>
bool direct_layout(int scalar, int64_t ld, int64_t rows) {
  return scalar != BFLY_D && ld == rows;
}

template <typename R>
void op_apply_t(bfly_op* op, DevOp<R>* o, int trans, const void* x, int64_t ldx, void* y, int64_t ldy, int64_t k,
                int on_device) {
  Ctx* c = C_(op->ctx);
  const int64_t nin = o->in_dim(trans), nout = o->out_dim(trans);
  if (ldx < nin || ldy < nout) fail(DIMENSION, "apply: leading dimension smaller than the row count");
  if (k <= 0) return;
  if (on_device) {
    o->apply_dense(trans, static_cast<const cx<R>*>(x), ldx, static_cast<cx<R>*>(y), ldy, k);
    return;
  }
  DBuf<cx<R>> dx(c, (size_t)(nin * k)), dy(c, (size_t)(nout * k));
  if (direct_layout<R>(op->scalar, ldx, nin))
    BFLY_CUDA(cudaMemcpyAsync(dx.p, x, sizeof(cx<R>) * nin * k, cudaMemcpyHostToDevice, c->stream));
  else
    h2d<R>(c, op->scalar, x, ldx, dx.p, nin, k);
  o->apply_dense(trans, dx.p, nin, dy.p, nout, k);
  if (direct_layout<R>(op->scalar, ldy, nout)) {
    BFLY_CUDA(cudaMemcpyAsync(y, dy.p, sizeof(cx<R>) * nout * k, cudaMemcpyDeviceToHost, c->stream));
    c->sync();
  } else {
    d2h<R>(c, op->scalar, dy.p, nout, k, y, ldy);
  }
}

template <typename R>
void bf_apply_t(bfly_bf* bf, DevButterfly<R>* b, int trans, const void* x, int64_t ldx, void* y, int64_t ldy, int64_t k,
                int on_device) {
  Ctx* c = C_(bf->ctx);
  const int64_t nin = trans == BFLY_N ? b->n() : b->m(), nout = trans == BFLY_N ? b->m() : b->n();
  if (ldx < nin || ldy < nout) fail(DIMENSION, "HybridButterfly::apply: leading dimension smaller than the row count");
  if (k <= 0) return;
  if (on_device) {
    b->apply(trans, static_cast<const cx<R>*>(x), ldx, static_cast<cx<R>*>(y), ldy, k);
    return;
  }
  DBuf<cx<R>> dx(c, (size_t)(nin * k)), dy(c, (size_t)(nout * k));
  if (direct_layout<R>(bf->scalar, ldx, nin))
    BFLY_CUDA(cudaMemcpyAsync(dx.p, x, sizeof(cx<R>) * nin * k, cudaMemcpyHostToDevice, c->stream));
  else
    h2d<R>(c, bf->scalar, x, ldx, dx.p, nin, k);
  b->apply(trans, dx.p, nin, dy.p, nout, k);
  if (direct_layout<R>(bf->scalar, ldy, nout)) {
    BFLY_CUDA(cudaMemcpyAsync(y, dy.p, sizeof(cx<R>) * nout * k, cudaMemcpyDeviceToHost, c->stream));
    c->sync();
  } else {
    d2h<R>(c, bf->scalar, dy.p, nout, k, y, ldy);
  }
}

template <typename R>
void bf_apply_layout_t(bfly_bf* bf, DevButterfly<R>* b, int trans, int kind, int64_t p, const void* x, int64_t ldx,
                       void* y, int64_t ldy, int64_t k, int on_device, double* report) {
  Ctx* c = C_(bf->ctx);
  const int64_t nin = trans == BFLY_N ? b->n() : b->m(), nout = trans == BFLY_N ? b->m() : b->n();
  if (ldx < nin || ldy < nout) fail(DIMENSION, "apply_layout: leading dimension smaller than the row count");
  if (p < 1 || p > (int64_t(1) << 30)) fail(PRECONDITION, "apply_layout: bad process count");
  if (on_device) {
    b->apply_layout(trans, kind, (int)p, static_cast<const cx<R>*>(x), ldx, static_cast<cx<R>*>(y), ldy, k, report);
    c->sync();
    return;
  }
  DBuf<cx<R>> dx(c, (size_t)(nin * std::max<int64_t>(k, 1))), dy(c, (size_t)(nout * std::max<int64_t>(k, 1)));
  if (k > 0) h2d<R>(c, bf->scalar, x, ldx, dx.p, nin, k);
  b->apply_layout(trans, kind, (int)p, dx.p, nin, dy.p, nout, k, report);
  if (k > 0) d2h<R>(c, bf->scalar, dy.p, nout, k, y, ldy);
  c->sync();
}

template <typename R>
double estimate_error_t(Ctx* c, DevOp<R>* op, DevButterfly<R>* bf, int64_t k, uint64_t seed) {
  if (k < 1) fail(PRECONDITION, "estimate_error: k >= 1 required");
  const int64_t n = op->n, m = op->m;
  if (bf->m() != m || bf->n() != n) fail(DIMENSION, "estimate_error: butterfly and operator dimensions differ");
  DBuf<cx<R>> om(c, (size_t)(n * k)), ex(c, (size_t)(m * k)), ap(c, (size_t)(m * k));
  GaussEnt ge{0, n, n, k, seed_mix_host(seed_mix_host(seed, {5}), {0x6d617472ULL})};
  DBuf<GaussEnt> dge = to_device(c, std::vector<GaussEnt>{ge});
  launch_gauss<R>(c, om.p, dge.p, 1, n * k, op->is_real);
  op->apply_dense(OP_N, om.p, n, ex.p, m, k);
  bf->apply(OP_N, om.p, n, ap.p, m, k);
  DBuf<double> acc(c, 2);
  acc.zero();
  launch_diff_norms<R>(c, ex.p, ap.p, m * k, acc.p);
  double h[2];
  acc.download(h, 2);
  c->sync();
  if (h[1] == 0.0) fail(CONDITIONING, "estimate_error: ||A Omega||_F is zero, relative error undefined");
  return std::sqrt(h[0]) / std::sqrt(h[1]);
}

template <typename R>
std::unique_ptr<DevButterfly<R>> upload_host(Ctx* c, const HostButterfly& h, bool is_real) {
  auto d = DevButterfly<R>::from_host(c, h);
  d->is_real = is_real;
  return d;
}

}  // namespace

namespace {
template <typename R>
int64_t rank_profile_t(const DevButterfly<R>& b, int32_t* out) {
  int64_t nbk = b.nb(), off = 0;
  for (int l = b.lm; l <= b.L; ++l) {
    if (out)
      for (int64_t tau = 0; tau < (int64_t(1) << l); ++tau)
        for (int64_t nu = 0; nu < (int64_t(1) << (b.L - l)); ++nu) out[off + bidx(b.L, l, tau, nu)] = b.u_rank(l, tau, nu);
    off += nbk;
  }
  for (int l = 0; l <= b.lm; ++l) {
    if (out)
      for (int64_t tau = 0; tau < (int64_t(1) << l); ++tau)
        for (int64_t nu = 0; nu < (int64_t(1) << (b.L - l)); ++nu) out[off + bidx(b.L, l, tau, nu)] = b.v_rank(l, tau, nu);
    off += nbk;
  }
  return off;
}
}  // namespace

extern "C" {

const char* bfly_last_error(void) { return g_err.c_str(); }
const char* bfly_version(void) { return "bfly_b200 0.1 (sm_100a)"; }

int bfly_ctx_create(int device, bfly_ctx** out) {
  *out = nullptr;
  return guard(nullptr, [&] {
    auto h = std::make_unique<bfly_ctx>();
    h->c = std::make_unique<Ctx>(device);
    *out = h.release();
  });
}

int bfly_ctx_destroy(bfly_ctx* ctx) {
  if (!ctx) return BFLY_OK;
  int rc = guard(C_(ctx), [&] { comm_destroy(C_(ctx)); });
  delete ctx;
  return rc;
}

int64_t bfly_ctx_launches(const bfly_ctx* ctx) { return ctx ? ctx->c->launches : 0; }
int bfly_ctx_synchronize(bfly_ctx* ctx) {
  return guard(C_(ctx), [&] { C_(ctx)->sync(); });
}
void* bfly_ctx_stream(bfly_ctx* ctx) { return ctx ? (void*)ctx->c->stream : nullptr; }

int bfly_ctx_profile(bfly_ctx* ctx, int enable) {
  return guard(C_(ctx), [&] {
    Ctx* c = C_(ctx);
    c->resolve_records();
    if (enable < 0) c->stats.clear();
    c->profiling = enable > 0;
  });
}

int64_t bfly_ctx_profile_report(bfly_ctx* ctx, char* buf, int64_t len) {
  std::string js = "{";
  int rc = guard(C_(ctx), [&] {
    Ctx* c = C_(ctx);
    c->resolve_records();
    bool first = true;
    for (auto& kv : c->stats) {
      char tmp[256];
      std::snprintf(tmp, sizeof tmp, "%s\"%s\": {\"launches\": %lld, \"ms\": %.6f, \"flops\": %.6e, \"bytes\": %.6e}",
                    first ? "" : ", ", kv.first.c_str(), (long long)kv.second.launches, kv.second.ms, kv.second.flops,
                    kv.second.bytes);
      js += tmp;
      first = false;
    }
  });
  js += "}";
  if (rc != BFLY_OK) return -1;
  if (buf && len > 0) {
    std::strncpy(buf, js.c_str(), (size_t)len - 1);
    buf[len - 1] = 0;
  }
  return (int64_t)js.size() + 1;
}

int bfly_comm_unique_id(uint8_t* id_out) {
  return guard(nullptr, [&] { comm_unique_id(id_out); });
}
int bfly_ctx_set_comm(bfly_ctx* ctx, int rank, int world, const uint8_t* id) {
  return guard(C_(ctx), [&] { comm_init(C_(ctx), rank, world, id); });
}
int bfly_ctx_set_host_comm(bfly_ctx* ctx, int rank, int world, const bfly_host_comm* hc) {
  return guard(C_(ctx), [&] { comm_init_host(C_(ctx), rank, world, hc); });
}
int bfly_ctx_comm_info(const bfly_ctx* ctx, int* rank, int* world, int* transport) {
  if (!ctx) return BFLY_PRECONDITION;
  const Ctx* c = ctx->c.get();
  if (rank) *rank = c->rank;
  if (world) *world = c->world;
  if (transport) *transport = c->comm ? 1 : c->host ? 2 : 0;
  return BFLY_OK;
}

// ------------------------------------------------------------------ trees
int bfly_tree_build(int dim, int64_t n, const double* coords, int levels, bfly_tree** out) {
  *out = nullptr;
  return guard(nullptr, [&] {
    auto t = std::make_unique<bfly_tree>();
    t->t = Tree::build(dim, n, coords, levels);
    *out = t.release();
  });
}
int bfly_tree_from_table(int64_t n, int levels, const int64_t* perm, const int64_t* ranges, bfly_tree** out) {
  *out = nullptr;
  return guard(nullptr, [&] {
    auto t = std::make_unique<bfly_tree>();
    t->t = Tree::from_table(n, levels, perm, ranges);
    *out = t.release();
  });
}
int bfly_tree_info(const bfly_tree* t, int64_t* n, int* levels) {
  if (!t) return BFLY_PRECONDITION;
  if (n) *n = t->t.n;
  if (levels) *levels = t->t.levels;
  return BFLY_OK;
}
int bfly_tree_table(const bfly_tree* t, int64_t* perm, int64_t* ranges) {
  if (!t) return BFLY_PRECONDITION;
  t->t.table(perm, ranges);
  return BFLY_OK;
}
void bfly_tree_destroy(bfly_tree* t) { delete t; }
int bfly_depth_for(int64_t n, int64_t leaf) {
  int d = -1;
  guard(nullptr, [&] { d = depth_for(n, leaf); });
  return d;
}

// ------------------------------------------------------- point generators
void bfly_points_uniform(int64_t n, uint64_t seed, uint64_t tag, double lo, double hi, double* out) {
  uint64_t st = seed_mix_host(seed, {tag});
  for (int64_t i = 0; i < n; ++i) {
    st += kGamma;
    double u = (double)(mix64(st) >> 11) * 0x1p-53;
    out[i * 3 + 0] = lo + (hi - lo) * u;
    out[i * 3 + 1] = 0.0;
    out[i * 3 + 2] = 0.0;
  }
}
void bfly_points_plate(int64_t side, double z, double* out) {
  double h = 1.0 / (double)side;
  for (int64_t a = 0; a < side; ++a)
    for (int64_t b = 0; b < side; ++b) {
      int64_t i = a * side + b;
      out[i * 3 + 0] = ((double)b + 0.5) * h;
      out[i * 3 + 1] = ((double)a + 0.5) * h;
      out[i * 3 + 2] = z;
    }
}
void bfly_points_half_circle(int64_t n, int upper, double* out) {
  for (int64_t i = 0; i < n; ++i) {
    double th = ((double)i + 0.5) * M_PI / (double)n + (upper ? 0.0 : M_PI);
    out[i * 3 + 0] = std::cos(th);
    out[i * 3 + 1] = std::sin(th);
    out[i * 3 + 2] = 0.0;
  }
}

// -------------------------------------------------------------- operators
int bfly_op_kernel(bfly_ctx* ctx, int kind, int64_t m, int64_t n, const double* tgt, const double* src,
                   double wavenumber, int scalar, bfly_op** out) {
  *out = nullptr;
  return guard(C_(ctx), [&] {
    check_scalar(scalar);
    if (scalar == BFLY_D) fail(PRECONDITION, "kernel operators are complex-valued");
    auto h = std::make_unique<bfly_op>();
    h->ctx = ctx;
    h->scalar = scalar;
    if (scalar == BFLY_Z) h->z = make_kernel_op<double>(C_(ctx), kind, m, n, tgt, src, wavenumber);
    else h->c = make_kernel_op<float>(C_(ctx), kind, m, n, tgt, src, wavenumber);
    *out = h.release();
  });
}

int bfly_op_compose(bfly_ctx* ctx, bfly_op* f2, bfly_op* f1, bfly_op** out) {
  *out = nullptr;
  return guard(C_(ctx), [&] {
    if (!f1 || !f2 || f1->scalar != f2->scalar) fail(PRECONDITION, "compose: factors must share a scalar type");
    auto h = std::make_unique<bfly_op>();
    h->ctx = ctx;
    h->scalar = f1->scalar;
    if (f1->z) h->z = make_compose_op<double>(C_(ctx), std::move(f2->z), std::move(f1->z));
    else h->c = make_compose_op<float>(C_(ctx), std::move(f2->c), std::move(f1->c));
    delete f1;
    delete f2;
    *out = h.release();
  });
}

int bfly_op_dense(bfly_ctx* ctx, int64_t m, int64_t n, const double* a, int scalar, bfly_op** out) {
  *out = nullptr;
  return guard(C_(ctx), [&] {
    check_scalar(scalar);
    auto h = std::make_unique<bfly_op>();
    h->ctx = ctx;
    h->scalar = scalar;
    if (scalar == BFLY_C) {
      std::vector<float2> v((size_t)(m * n));
      const float* f = reinterpret_cast<const float*>(a);
      for (int64_t i = 0; i < m * n; ++i) v[i] = make_float2(f[2 * i], f[2 * i + 1]);
      h->c = make_dense_op<float>(C_(ctx), m, n, v, false);
    } else {
      std::vector<double2> v((size_t)(m * n));
      for (int64_t i = 0; i < m * n; ++i)
        v[i] = scalar == BFLY_D ? make_double2(a[i], 0.0) : make_double2(a[2 * i], a[2 * i + 1]);
      h->z = make_dense_op<double>(C_(ctx), m, n, v, scalar == BFLY_D);
    }
    *out = h.release();
  });
}

int bfly_op_butterfly(bfly_ctx* ctx, bfly_bf* bf, bfly_op** out) {
  *out = nullptr;
  return guard(C_(ctx), [&] {
    auto h = std::make_unique<bfly_op>();
    h->ctx = ctx;
    h->scalar = bf->scalar;
    if (bf->z) h->z = make_butterfly_op<double>(C_(ctx), std::move(bf->z));
    else h->c = make_butterfly_op<float>(C_(ctx), std::move(bf->c));
    delete bf;
    *out = h.release();
  });
}

int bfly_op_callback(bfly_ctx* ctx, int64_t m, int64_t n, int scalar, bfly_apply_fn fn, void* user, bfly_op** out) {
  *out = nullptr;
  return guard(C_(ctx), [&] {
    check_scalar(scalar);
    auto h = std::make_unique<bfly_op>();
    h->ctx = ctx;
    h->scalar = scalar;
    if (scalar == BFLY_C) h->c = make_callback_op<float>(C_(ctx), m, n, false, fn, user);
    else h->z = make_callback_op<double>(C_(ctx), m, n, scalar == BFLY_D, fn, user);
    *out = h.release();
  });
}

int bfly_op_callback_ranged(bfly_ctx* ctx, int64_t m, int64_t n, int scalar, bfly_apply_range_fn fn, void* user,
                            bfly_op** out) {
  *out = nullptr;
  return guard(C_(ctx), [&] {
    check_scalar(scalar);
    auto h = std::make_unique<bfly_op>();
    h->ctx = ctx;
    h->scalar = scalar;
    if (scalar == BFLY_C) h->c = make_callback_range_op<float>(C_(ctx), m, n, false, fn, user);
    else h->z = make_callback_range_op<double>(C_(ctx), m, n, scalar == BFLY_D, fn, user);
    *out = h.release();
  });
}

int bfly_op_info(const bfly_op* op, int64_t* m, int64_t* n, int* scalar, int* kind) {
  if (!op) return BFLY_PRECONDITION;
  if (m) *m = op->m();
  if (n) *n = op->n();
  if (scalar) *scalar = op->scalar;
  if (kind) *kind = op->kind();
  return BFLY_OK;
}

int bfly_op_apply(bfly_op* op, int trans, const void* x, int64_t ldx, void* y, int64_t ldy, int64_t k, int on_device) {
  return guard(C_(op->ctx), [&] {
    if (trans < 0 || trans > 2) fail(PRECONDITION, "apply: trans must be N, T or H");
    if (op->z) op_apply_t<double>(op, op->z.get(), trans, x, ldx, y, ldy, k, on_device);
    else op_apply_t<float>(op, op->c.get(), trans, x, ldx, y, ldy, k, on_device);
  });
}

int bfly_op_counters(const bfly_op* op, int64_t* fwd, int64_t* tr) {
  if (!op) return BFLY_PRECONDITION;
  *fwd = op->z ? op->z->fwd : op->c->fwd;
  *tr = op->z ? op->z->tr : op->c->tr;
  return BFLY_OK;
}
int bfly_op_reset_counters(bfly_op* op) {
  if (!op) return BFLY_PRECONDITION;
  if (op->z) op->z->fwd = op->z->tr = 0;
  else op->c->fwd = op->c->tr = 0;
  return BFLY_OK;
}
void bfly_op_destroy(bfly_op* op) {
  if (!op) return;
  guard(C_(op->ctx), [&] {
    op->z.reset();
    op->c.reset();
  });
  delete op;
}

// ---------------------------------------------------------- reconstruction
void bfly_cfg_default(bfly_recon_cfg* c) {
  c->tolerance = 1e-6;
  c->oversampling = 2;
  c->rank_guess = 4;
  c->levels = 4;
  c->center = -1;
  c->seed = 0;
  c->hard_cap = -1;
  c->threads = 1;
  c->literal_transpose_core = 0;
  c->max_batch_probes = 0;
  c->virtual_ranks = 0;
  c->reserved_ = 0;
}

int bfly_factorizer_create(bfly_ctx* ctx, bfly_op* op, const bfly_tree* rt, const bfly_tree* ct,
                           const bfly_recon_cfg* cfg, bfly_factorizer** out) {
  *out = nullptr;
  return guard(C_(ctx), [&] {
    auto h = std::make_unique<bfly_factorizer>();
    h->ctx = ctx;
    h->scalar = op->scalar;
    if (op->z) h->z = std::make_unique<Factorizer<double>>(C_(ctx), op->z.get(), rt->t, ct->t, *cfg);
    else h->c = std::make_unique<Factorizer<float>>(C_(ctx), op->c.get(), rt->t, ct->t, *cfg);
    *out = h.release();
  });
}

#define FZ_CALL(f, expr) \
  guard(C_((f)->ctx), [&] { if ((f)->z) (f)->z->expr; else (f)->c->expr; })

int bfly_factorizer_leaf_row_bases(bfly_factorizer* f) { return FZ_CALL(f, leaf_row_bases()); }
int bfly_factorizer_leaf_col_bases(bfly_factorizer* f) { return FZ_CALL(f, leaf_col_bases()); }
int bfly_factorizer_transfer_level_w(bfly_factorizer* f, int l) { return FZ_CALL(f, transfer_level_w(l)); }
int bfly_factorizer_transfer_level_r(bfly_factorizer* f, int l) { return FZ_CALL(f, transfer_level_r(l)); }
int bfly_factorizer_complete(const bfly_factorizer* f) { return f->z ? f->z->complete() : f->c->complete(); }

int bfly_factorizer_take(bfly_factorizer* f, bfly_bf** out, bfly_log* log) {
  *out = nullptr;
  return guard(C_(f->ctx), [&] {
    auto h = std::make_unique<bfly_bf>();
    h->ctx = f->ctx;
    h->scalar = f->scalar;
    if (f->z) {
      h->z = f->z->take(log);
      h->z->to_host().validate();
    } else {
      h->c = f->c->take(log);
      h->c->to_host().validate();
    }
    *out = h.release();
  });
}
void bfly_factorizer_destroy(bfly_factorizer* f) {
  if (!f) return;
  guard(C_(f->ctx), [&] {
    f->z.reset();
    f->c.reset();
  });
  delete f;
}

int bfly_factorize(bfly_ctx* ctx, bfly_op* op, const bfly_tree* rt, const bfly_tree* ct, const bfly_recon_cfg* cfg,
                   bfly_bf** out, bfly_log* log) {
  *out = nullptr;
  return guard(C_(ctx), [&] {
    auto h = std::make_unique<bfly_bf>();
    h->ctx = ctx;
    h->scalar = op->scalar;
    Ctx* c = C_(ctx);
    auto run_once = [&] {
      if (op->z) {
        Factorizer<double> f(c, op->z.get(), rt->t, ct->t, *cfg);
        f.run();
        h->z = f.take(log);
      } else {
        Factorizer<float> f(c, op->c.get(), rt->t, ct->t, *cfg);
        f.run();
        h->c = f.take(log);
      }
    };
    // K2 range checks are deferred to the end of the factorization (no host
    // sync per black-box product); on an out-of-range entry the whole
    // factorization is recomputed on the FP64 path, operator counters restored
    auto counters = [&](int64_t* v, double* w, bool save) {
      if (op->z) {
        if (save) { v[0] = op->z->fwd; v[1] = op->z->tr; w[0] = op->z->flops; w[1] = op->z->evals; }
        else { op->z->fwd = v[0]; op->z->tr = v[1]; op->z->flops = w[0]; op->z->evals = w[1]; }
      } else {
        if (save) { v[0] = op->c->fwd; v[1] = op->c->tr; w[0] = op->c->flops; w[1] = op->c->evals; }
        else { op->c->fwd = v[0]; op->c->tr = v[1]; op->c->flops = w[0]; op->c->evals = w[1]; }
      }
    };
    int64_t cv[2];
    double cw[2];
    counters(cv, cw, true);
    struct Reset {
      Ctx* c;
      ~Reset() {
        // an exception may leave a flag set by a launch of the failed run
        if (c->oz_deferred) c->clear_oz_flag();
        c->oz_deferred = c->force_fp64 = false;
      }
    } reset{c};
    c->clear_oz_flag();
    c->oz_deferred = true;
    run_once();
    c->oz_deferred = false;
    if (c->take_oz_overflow()) {
      counters(cv, cw, false);
      h->z.reset();
      h->c.reset();
      c->force_fp64 = true;
      run_once();
      if (log) log->products_recomputed = 1;
    }
    *out = h.release();
  });
}

int bfly_estimate_error(bfly_op* op, bfly_bf* bf, int64_t k, uint64_t seed, double* err) {
  return guard(C_(op->ctx), [&] {
    if (op->scalar != bf->scalar) fail(PRECONDITION, "estimate_error: scalar types differ");
    if (op->z) *err = estimate_error_t<double>(C_(op->ctx), op->z.get(), bf->z.get(), k, seed);
    else *err = estimate_error_t<float>(C_(op->ctx), op->c.get(), bf->c.get(), k, seed);
  });
}

int bfly_residuals(bfly_op* op, bfly_bf* bf, double* u_res, double* v_res, double* center, double* knorm2) {
  return guard(C_(op->ctx), [&] {
    if (op->scalar != bf->scalar) fail(PRECONDITION, "residuals: scalar types differ");
    Residuals r = op->z ? compute_residuals<double>(C_(op->ctx), op->z.get(), *bf->z)
                        : compute_residuals<float>(C_(op->ctx), op->c.get(), *bf->c);
    for (size_t i = 0; i < r.u.size(); ++i) u_res[i] = r.u[i];
    for (size_t i = 0; i < r.v.size(); ++i) v_res[i] = r.v[i];
    *center = r.center;
    *knorm2 = r.knorm2;
  });
}

// -------------------------------------------------------------- butterfly
int bfly_apply(bfly_bf* bf, int trans, const void* x, int64_t ldx, void* y, int64_t ldy, int64_t k, int on_device) {
  return guard(C_(bf->ctx), [&] {
    if (trans < 0 || trans > 2) fail(PRECONDITION, "apply: trans must be N, T or H");
    if (bf->z) bf_apply_t<double>(bf, bf->z.get(), trans, x, ldx, y, ldy, k, on_device);
    else bf_apply_t<float>(bf, bf->c.get(), trans, x, ldx, y, ldy, k, on_device);
  });
}

int bfly_apply_layout(bfly_bf* bf, int trans, int kind, int64_t processes, const void* x, int64_t ldx, void* y,
                      int64_t ldy, int64_t k, int on_device, double* report) {
  return guard(C_(bf->ctx), [&] {
    if (bf->z) bf_apply_layout_t<double>(bf, bf->z.get(), trans, kind, processes, x, ldx, y, ldy, k, on_device, report);
    else bf_apply_layout_t<float>(bf, bf->c.get(), trans, kind, processes, x, ldx, y, ldy, k, on_device, report);
  });
}

int bfly_comm_cost(int kind, int levels, int64_t rank, int64_t processes, double* out) {
  if (!layout_valid(kind, levels, rank, processes)) {
    g_err = "comm_cost: invalid LayoutSpec (kind, levels >= 1, rank >= 1, power-of-two p <= 2^L)";
    return BFLY_PRECONDITION;
  }
  const CommReport r = comm_cost(kind, levels, rank, processes);
  if (out) {
    out[0] = r.exchange_volume;
    out[1] = (double)r.exchange_msgs;
    out[2] = r.alltoall_volume;
    out[3] = (double)r.alltoall_msgs;
  }
  return BFLY_OK;
}

int64_t bfly_layout_owners(int kind, int levels, int center, int64_t processes, int32_t* out) {
  if (!layout_valid(kind, levels, 1, processes) || center < 0 || center > levels) {
    g_err = "layout_owners: invalid layout";
    return -BFLY_PRECONDITION;
  }
  const int L = levels, g = layout_log_p(processes);
  const int64_t nb = int64_t(1) << L;
  const int64_t len = (int64_t)(L + 3) * nb;
  if (!out) return len;
  int32_t* o = out;
  for (int64_t tau = 0; tau < nb; ++tau) *o++ = layout_owner(kind, L, g, 1, L, tau, 0);  // u leaves
  for (int64_t nu = 0; nu < nb; ++nu) *o++ = layout_owner(kind, L, g, 0, 0, 0, nu);      // v leaves
  for (int l = center; l < L; ++l)                                                       // R levels
    for (int64_t i = 0; i < nb; ++i) *o++ = layout_owner(kind, L, g, 1, l, i >> (L - l), i & ((int64_t(1) << (L - l)) - 1));
  for (int l = 1; l <= center; ++l)                                                      // W levels
    for (int64_t i = 0; i < nb; ++i) *o++ = layout_owner(kind, L, g, 0, l, i >> (L - l), i & ((int64_t(1) << (L - l)) - 1));
  for (int64_t i = 0; i < nb; ++i)                                                       // centre cores
    *o++ = layout_owner(kind, L, g, 0, center, i >> (L - center), i & ((int64_t(1) << (L - center)) - 1));
  return len;
}

int bfly_bf_info(const bfly_bf* bf, int* levels, int* center, int64_t* m, int64_t* n, int64_t* nnz, int64_t* max_rank,
                 int* scalar) {
  if (!bf) return BFLY_PRECONDITION;
  if (bf->z) {
    if (levels) *levels = bf->z->L;
    if (center) *center = bf->z->lm;
    if (m) *m = bf->z->m();
    if (n) *n = bf->z->n();
    if (nnz) *nnz = bf->z->nnz();
    if (max_rank) *max_rank = bf->z->max_rank();
  } else {
    if (levels) *levels = bf->c->L;
    if (center) *center = bf->c->lm;
    if (m) *m = bf->c->m();
    if (n) *n = bf->c->n();
    if (nnz) *nnz = bf->c->nnz();
    if (max_rank) *max_rank = bf->c->max_rank();
  }
  if (scalar) *scalar = bf->scalar;
  return BFLY_OK;
}


int64_t bfly_rank_profile(const bfly_bf* bf, int32_t* out) {
  if (!bf) return -1;
  return bf->z ? rank_profile_t(*bf->z, out) : rank_profile_t(*bf->c, out);
}

int64_t bfly_serialize(const bfly_bf* bf, uint8_t* buf) {
  int64_t n = -1;
  int rc = guard(C_(bf->ctx), [&] {
    const int tag = bf->scalar == BFLY_D ? 0 : 1;
    n = bf->z ? bf->z->serialize(tag, buf) : bf->c->serialize(tag, buf);
  });
  return rc == BFLY_OK ? n : -1;
}

int bfly_deserialize(bfly_ctx* ctx, const uint8_t* buf, int64_t nbytes, int scalar, bfly_bf** out) {
  *out = nullptr;
  return guard(C_(ctx), [&] {
    check_scalar(scalar);
    HostButterfly h = HostButterfly::deserialize(buf, nbytes);
    if ((scalar == BFLY_D) != h.is_real)
      fail(FORMAT, "container scalar type does not match the requested type");
    auto b = std::make_unique<bfly_bf>();
    b->ctx = ctx;
    b->scalar = scalar;
    if (scalar == BFLY_C) b->c = upload_host<float>(C_(ctx), h, false);
    else b->z = upload_host<double>(C_(ctx), h, h.is_real);
    *out = b.release();
  });
}

int bfly_synth_butterfly(bfly_ctx* ctx, int levels, int64_t leaf, int64_t rank, uint64_t seed, int scalar, double perturb,
                         bfly_bf** out) {
  *out = nullptr;
  return guard(C_(ctx), [&] {
    check_scalar(scalar);
    HostButterfly h = synth_host(levels, leaf, rank, seed, scalar == BFLY_D, perturb);
    auto b = std::make_unique<bfly_bf>();
    b->ctx = ctx;
    b->scalar = scalar;
    if (scalar == BFLY_C) b->c = upload_host<float>(C_(ctx), h, false);
    else b->z = upload_host<double>(C_(ctx), h, h.is_real);
    *out = b.release();
  });
}

int bfly_bf_convert(bfly_bf* bf, int scalar, bfly_bf** out) {
  *out = nullptr;
  return guard(C_(bf->ctx), [&] {
    check_scalar(scalar);
    HostButterfly h = bf->z ? bf->z->to_host() : bf->c->to_host();
    auto b = std::make_unique<bfly_bf>();
    b->ctx = bf->ctx;
    b->scalar = scalar;
    if (scalar == BFLY_C) b->c = upload_host<float>(C_(bf->ctx), h, false);
    else b->z = upload_host<double>(C_(bf->ctx), h, scalar == BFLY_D);
    *out = b.release();
  });
}

void bfly_bf_destroy(bfly_bf* bf) {
  if (!bf) return;
  guard(C_(bf->ctx), [&] {
    bf->z.reset();
    bf->c.reset();
  });
  delete bf;
}

// ------------------------------------------------------------ dense helpers
uint64_t bfly_seed_mix(uint64_t seed, int nwords, const uint64_t* words) { return seed_mix_host_n(seed, nwords, words); }

int bfly_gaussian(bfly_ctx* ctx, int64_t rows, int64_t cols, uint64_t seed, int scalar, void* out_host) {
  return guard(C_(ctx), [&] {
    check_scalar(scalar);
    if (rows < 1 || cols < 1) fail(PRECONDITION, "gaussian_matrix: dimensions must be positive");
    Ctx* c = C_(ctx);
    GaussEnt ge{0, rows, rows, cols, seed_mix_host(seed, {0x6d617472ULL})};
    DBuf<GaussEnt> dge = to_device(c, std::vector<GaussEnt>{ge});
    if (scalar == BFLY_C) {
      DBuf<float2> d(c, (size_t)(rows * cols));
      launch_gauss<float>(c, d.p, dge.p, 1, rows * cols, false);
      d2h<float>(c, scalar, d.p, rows, cols, out_host, rows);
    } else {
      DBuf<double2> d(c, (size_t)(rows * cols));
      launch_gauss<double>(c, d.p, dge.p, 1, rows * cols, scalar == BFLY_D);
      d2h<double>(c, scalar, d.p, rows, cols, out_host, rows);
    }
  });
}

int bfly_cpqr_truncate(bfly_ctx* ctx, int64_t rows, int64_t cols, const double* z_host, double eps, double* q_host,
                       int64_t* k_out) {
  return guard(C_(ctx), [&] {
    if (rows == 0 || cols == 0) fail(PRECONDITION, "pivoted_qr_truncate: empty input");
    Ctx* c = C_(ctx);
    DBuf<double2> z(c, (size_t)(rows * cols)), q(c, (size_t)(rows * std::min(rows, cols)));
    h2d<double>(c, BFLY_Z, z_host, rows, z.p, rows, cols);
    QrEnt e{};
    e.r1 = (int32_t)rows;
    e.cols = (int32_t)cols;
    DBuf<QrEnt> de = to_device(c, std::vector<QrEnt>{e});
    DBuf<int32_t> rk(c, 1);
    int cap = (int)std::min(rows, cols);
    launch_cpqr<double>(c, z.p, rows, q.p, rows, cap, de.p, 1, (int)rows, (int)cols, rk.p, eps);
    int32_t k = 0;
    rk.download(&k, 1);
    c->sync();
    *k_out = k;
    if (k > 0) d2h<double>(c, BFLY_Z, q.p, rows, k, q_host, rows);
  });
}

int bfly_pinv(bfly_ctx* ctx, int64_t rows, int64_t cols, const double* m_host, double tol, double* out_host) {
  return guard(C_(ctx), [&] {
    if (rows == 0 || cols == 0) fail(PRECONDITION, "pinv_solve: empty input");
    if (tol != 1e-12) fail(PRECONDITION, "pinv: the device path implements the reference cutoff 1e-12");
    Ctx* c = C_(ctx);
    // wide (rows <= cols): B = I * pinv(M) via the core-fit kernel; tall: pinv(M) = pinv(M^H)^H
    const bool wide = rows <= cols;
    const int64_t kr = wide ? rows : cols, w = wide ? cols : rows;
    std::vector<double2> mm((size_t)(kr * w));
    for (int64_t i = 0; i < rows; ++i)
      for (int64_t j = 0; j < cols; ++j) {
        double2 v = make_double2(m_host[2 * (i + j * rows)], m_host[2 * (i + j * rows) + 1]);
        if (wide) mm[i + j * kr] = v;
        else mm[j + i * kr] = make_double2(v.x, -v.y);
      }
    std::vector<double2> eye((size_t)(w * w), make_double2(0, 0));
    for (int64_t i = 0; i < w; ++i) eye[i + i * w] = make_double2(1, 0);
    DBuf<double2> dm = to_device(c, mm), di = to_device(c, eye), db(c, (size_t)(w * kr));
    CoreEnt e{};
    e.r1 = (int32_t)w;
    e.ku = (int32_t)w;
    e.kv = (int32_t)kr;
    e.w = (int32_t)w;
    DBuf<CoreEnt> de = to_device(c, std::vector<CoreEnt>{e});
    DBuf<int32_t> flag(c, 1);
    flag.zero();
    launch_core_fit<double>(c, di.p, w, di.p, w, dm.p, kr, db.p, w, (int)kr, de.p, 1, (int)w, (int)kr, (int)w, false,
                            flag.p);
    std::vector<double2> res((size_t)(w * kr));
    db.download(res.data(), res.size());
    c->sync();
    // wide: out (cols x rows) = res (w x kr); tall: out = res^H
    for (int64_t i = 0; i < cols; ++i)
      for (int64_t j = 0; j < rows; ++j) {
        double2 v = wide ? res[i + j * w] : res[j + i * w];
        if (!wide) v.y = -v.y;
        out_host[2 * (i + j * cols)] = v.x;
        out_host[2 * (i + j * cols) + 1] = v.y;
      }
  });
}

}  // extern "C"

// ------------------------------------------------------------- shard plan
#include "shard.h"
extern "C" {
int bfly_shard_chunk(int64_t n, int world, int rank, int64_t* begin, int64_t* end) {
  if (world < 1 || rank < 0 || rank >= world || n < 0) return BFLY_PRECONDITION;
  auto be = shard_chunk(n, world, rank);
  *begin = be.first;
  *end = be.second;
  return BFLY_OK;
}
int64_t bfly_shard_blocks(int levels, int level, int side, int world, int rank, int64_t* out) {
  if (world < 1 || rank < 0 || rank >= world || levels < 0 || level < 0 || level > levels || side < 0 || side > 2)
    return -1;
  std::vector<int64_t> v = shard_blocks(levels, level, side, world, rank);
  if (out) std::copy(v.begin(), v.end(), out);
  return (int64_t)v.size();
}
int64_t bfly_vrank_times(double* out, int64_t cap) {
  const std::vector<double>& t = vrank_table();
  if (out) std::copy(t.begin(), t.begin() + std::min<int64_t>(cap, (int64_t)t.size()), out);
  return (int64_t)t.size();
}
}
