// butterfly.cu -- device hybrid butterfly: apply (K3), accounting, host
// export/import and the .bfh container.
//
// apply follows butterfly.hpp:71-118 (V leaves -> W^H levels -> B -> R levels
// -> U leaves), apply_adjoint :122-184 and apply_transpose :187-193; every
// level is one batched block-GEMM launch over the padded level buffers.
#include <algorithm>
#include <atomic>
#include <cfloat>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <thread>

#include "butterfly.h"

namespace bfly {

// =================================================================== host
void HostButterfly::validate() const {
  int64_t nbk = int64_t(1) << L;
  if (lm < 0 || lm > L) fail(DIMENSION, "HybridButterfly: center level out of range");
  if ((int64_t)u.size() != nbk || (int64_t)v.size() != nbk || (int64_t)b.size() != nbk)
    fail(DIMENSION, "HybridButterfly: leaf/core block count mismatch");
  if ((int)r.size() != L - lm || (int)w.size() != lm) fail(DIMENSION, "HybridButterfly: factor level count mismatch");
  for (int64_t t = 0; t < nbk; ++t)
    if (u[t].rows != rt.size(L, t)) fail(DIMENSION, "HybridButterfly: U leaf height mismatch");
  for (int64_t t = 0; t < nbk; ++t)
    if (v[t].rows != ct.size(L, t)) fail(DIMENSION, "HybridButterfly: V leaf height mismatch");
  for (int l = lm; l < L; ++l)
    for (int64_t tau = 0; tau < (int64_t(1) << l); ++tau)
      for (int64_t nu = 0; nu < (int64_t(1) << (L - l)); ++nu)
        if (r[l - lm][bidx(L, l, tau, nu)].rows != u_rank(l + 1, 2 * tau, nu / 2) + u_rank(l + 1, 2 * tau + 1, nu / 2))
          fail(DIMENSION, "HybridButterfly: R block height mismatch");
  for (int l = 1; l <= lm; ++l)
    for (int64_t tau = 0; tau < (int64_t(1) << l); ++tau)
      for (int64_t nu = 0; nu < (int64_t(1) << (L - l)); ++nu)
        if (w[l - 1][bidx(L, l, tau, nu)].rows != v_rank(l - 1, tau / 2, 2 * nu) + v_rank(l - 1, tau / 2, 2 * nu + 1))
          fail(DIMENSION, "HybridButterfly: W block height mismatch");
  for (int64_t tau = 0; tau < (int64_t(1) << lm); ++tau)
    for (int64_t nu = 0; nu < (int64_t(1) << (L - lm)); ++nu) {
      const HostBlock& bb = b[bidx(L, lm, tau, nu)];
      if (bb.rows != u_rank(lm, tau, nu) || bb.cols != v_rank(lm, tau, nu))
        fail(DIMENSION, "HybridButterfly: B block shape mismatch");
    }
}

int64_t HostButterfly::nnz() const {
  int64_t s = 0;
  auto add = [&](const std::vector<HostBlock>& v_) {
    for (const auto& x : v_) s += x.rows * x.cols;
  };
  add(u); add(v); add(b);
  for (const auto& l : r) add(l);
  for (const auto& l : w) add(l);
  return s;
}

int64_t HostButterfly::max_rank() const {
  int64_t m = 0;
  auto upd = [&](const std::vector<HostBlock>& v_) {
    for (const auto& x : v_) m = std::max(m, x.cols);
  };
  upd(u); upd(v);
  for (const auto& l : r) upd(l);
  for (const auto& l : w) upd(l);
  return m;
}

namespace {
struct Writer {
  std::vector<uint8_t> buf;
  void put(const void* p, size_t n) {
    const uint8_t* c = static_cast<const uint8_t*>(p);
    buf.insert(buf.end(), c, c + n);
  }
  void u32(uint32_t v) { put(&v, 4); }
  void u64(uint64_t v) { put(&v, 8); }
};
struct Reader {
  const uint8_t* p;
  int64_t n, pos = 0;
  const char* section = "header";
  void get(void* d, int64_t k) {
    if (pos + k > n)
      fail(FORMAT, std::string("container truncated in section ") + section + " at offset " + std::to_string(pos));
    std::memcpy(d, p + pos, (size_t)k);
    pos += k;
  }
  uint32_t u32() { uint32_t v; get(&v, 4); return v; }
  uint64_t u64() { uint64_t v; get(&v, 8); return v; }
};
void put_tree(Writer& w, const Tree& t) {
  w.u64((uint64_t)t.n);
  w.u32((uint32_t)t.levels);
  for (int64_t i = 0; i < t.n; ++i) w.u64((uint64_t)t.perm[i]);
  for (const auto& lv : t.ranges)
    for (int64_t x : lv) w.u64((uint64_t)x);
}
Tree get_tree(Reader& r) {
  uint64_t n = r.u64();
  uint32_t levels = r.u32();
  if (levels > 40 || n > (uint64_t(1) << 40)) fail(FORMAT, "container: bad tree header");
  std::vector<int64_t> perm(n);
  for (auto& x : perm) x = (int64_t)r.u64();
  std::vector<int64_t> flat;
  for (uint32_t l = 0; l <= levels; ++l)
    for (uint64_t j = 0; j <= (uint64_t(1) << l); ++j) flat.push_back((int64_t)r.u64());
  return Tree::from_table((int64_t)n, (int)levels, perm.data(), flat.data());
}
void put_block(Writer& w, const HostBlock& b, bool real) {
  w.u64((uint64_t)b.rows);
  w.u64((uint64_t)b.cols);
  if (!real) {
    w.put(b.a.data(), sizeof(std::complex<double>) * b.a.size());
  } else {
    for (const auto& z : b.a) {
      double re = z.real();
      w.put(&re, 8);
    }
  }
}
HostBlock get_block(Reader& r, bool real) {
  HostBlock b;
  b.rows = (int64_t)r.u64();
  b.cols = (int64_t)r.u64();
  if (b.rows < 0 || b.cols < 0 || b.rows * b.cols * (real ? 8 : 16) > r.n - r.pos)
    fail(FORMAT, std::string("container truncated in section ") + r.section + " at offset " + std::to_string(r.pos));
  b.a.resize(b.rows * b.cols);
  if (!real) {
    r.get(b.a.data(), (int64_t)(16 * b.a.size()));
  } else {
    for (auto& z : b.a) {
      double re;
      r.get(&re, 8);
      z = re;
    }
  }
  return b;
}
}  // namespace

std::vector<uint8_t> HostButterfly::serialize(int scalar_tag) const {
  Writer wr;
  wr.u32(0x31484642u);  // "BFH1"
  wr.u32(1);
  uint8_t tag = (uint8_t)scalar_tag;
  wr.put(&tag, 1);
  wr.u32((uint32_t)L);
  wr.u32((uint32_t)lm);
  wr.u64((uint64_t)rt.n);
  wr.u64((uint64_t)ct.n);
  wr.u64((uint64_t)nnz());
  wr.u64((uint64_t)max_rank());
  put_tree(wr, rt);
  put_tree(wr, ct);
  bool real = tag == 0;
  for (const auto& x : u) put_block(wr, x, real);
  for (const auto& lv : r)
    for (const auto& x : lv) put_block(wr, x, real);
  for (const auto& x : b) put_block(wr, x, real);
  for (const auto& lv : w)
    for (const auto& x : lv) put_block(wr, x, real);
  for (const auto& x : v) put_block(wr, x, real);
  return wr.buf;
}

HostButterfly HostButterfly::deserialize(const uint8_t* buf, int64_t n) {
  Reader rd{buf, n};
  if (rd.u32() != 0x31484642u) fail(FORMAT, "bad container magic");
  uint32_t version = rd.u32();
  if (version != 1) fail(FORMAT, "unsupported container version " + std::to_string(version));
  uint8_t tag;
  rd.get(&tag, 1);
  HostButterfly h;
  h.is_real = tag == 0;
  h.L = (int)rd.u32();
  h.lm = (int)rd.u32();
  rd.u64(); rd.u64(); rd.u64(); rd.u64();
  if (h.L < 0 || h.L > 30 || h.lm < 0 || h.lm > h.L) fail(FORMAT, "container: bad level header");
  rd.section = "row_tree";
  h.rt = get_tree(rd);
  rd.section = "col_tree";
  h.ct = get_tree(rd);
  int64_t nbk = int64_t(1) << h.L;
  rd.section = "U";
  for (int64_t i = 0; i < nbk; ++i) h.u.push_back(get_block(rd, h.is_real));
  rd.section = "R";
  h.r.resize(h.L - h.lm);
  for (auto& lv : h.r)
    for (int64_t i = 0; i < nbk; ++i) lv.push_back(get_block(rd, h.is_real));
  rd.section = "B";
  for (int64_t i = 0; i < nbk; ++i) h.b.push_back(get_block(rd, h.is_real));
  rd.section = "W";
  h.w.resize(h.lm);
  for (auto& lv : h.w)
    for (int64_t i = 0; i < nbk; ++i) lv.push_back(get_block(rd, h.is_real));
  rd.section = "V";
  for (int64_t i = 0; i < nbk; ++i) h.v.push_back(get_block(rd, h.is_real));
  h.validate();
  return h;
}

// ------------------------------------------------------ host generators
void host_gaussian(int64_t rows, int64_t cols, uint64_t seed, bool is_real, std::complex<double>* out) {
  uint64_t st = seed_mix_host(seed, {0x6d617472ULL});
  int64_t total = rows * cols;
  auto pair = [&](double& c, double& s) {
    st += kGamma;
    double u1 = ((double)(mix64(st) >> 11) + 1.0) * 0x1p-53;
    st += kGamma;
    double u2 = ((double)(mix64(st) >> 11) + 1.0) * 0x1p-53;
    double radius = std::sqrt(-2.0 * std::log(u1));
    double angle = 6.283185307179586476925286766559 * u2;
    s = radius * std::sin(angle);
    c = radius * std::cos(angle);
  };
  if (!is_real) {
    for (int64_t t = 0; t < total; ++t) {
      double c, s;
      pair(c, s);
      out[t] = {c, s};
    }
  } else {
    for (int64_t t = 0; t < total; t += 2) {
      double c, s;
      pair(c, s);
      out[t] = c;
      if (t + 1 < total) out[t + 1] = s;
    }
  }
}

namespace {
using cd = std::complex<double>;

// Householder QR + Q(:, 0:cols) (operators.hpp:124-129 random_orthonormal),
// same arithmetic as the oracle's restatement of Eigen's HouseholderQR.
void householder_q(int64_t rows, int64_t cols, std::vector<cd>& qr, std::vector<cd>& q) {
  std::vector<cd> hc(cols);
  auto apply_left = [&](cd* m, int64_t ld, int64_t n, int64_t ncols, const cd* ess, cd tau) {
    if (n == 1) {
      for (int64_t j = 0; j < ncols; ++j) m[j * ld] *= (1.0 - tau);
      return;
    }
    if (tau == 0.0) return;
    for (int64_t j = 0; j < ncols; ++j) {
      cd* col = m + j * ld;
      cd tmp = col[0];
      for (int64_t i = 1; i < n; ++i) tmp += std::conj(ess[i - 1]) * col[i];
      cd t = tau * tmp;
      col[0] -= t;
      for (int64_t i = 1; i < n; ++i) col[i] -= ess[i - 1] * t;
    }
  };
  for (int64_t k = 0; k < cols; ++k) {
    cd* x = qr.data() + k + k * rows;
    int64_t n = rows - k;
    double tail = 0;
    for (int64_t i = 1; i < n; ++i) tail += std::norm(x[i]);
    cd c0 = x[0];
    double beta;
    cd tau;
    if (tail <= DBL_MIN && c0.imag() * c0.imag() <= DBL_MIN) {
      beta = c0.real();
      tau = 0;
      for (int64_t i = 1; i < n; ++i) x[i] = 0;
    } else {
      beta = std::sqrt(std::norm(c0) + tail);
      if (c0.real() >= 0) beta = -beta;
      cd d = c0 - beta;
      for (int64_t i = 1; i < n; ++i) x[i] = x[i] / d;
      tau = std::conj((beta - c0) / beta);
    }
    x[0] = beta;
    hc[k] = tau;
    apply_left(qr.data() + k + (k + 1) * rows, rows, n, cols - k - 1, x + 1, tau);
  }
  q.assign(rows * cols, 0.0);
  for (int64_t i = 0; i < cols; ++i) q[i + i * rows] = 1.0;
  for (int64_t j = cols - 1; j >= 0; --j)
    apply_left(q.data() + j + j * rows, rows, rows - j, cols - j, qr.data() + j + 1 + j * rows, std::conj(hc[j]));
}

HostBlock random_orthonormal(int64_t rows, int64_t cols, uint64_t seed, bool real) {
  std::vector<cd> g(rows * cols), q;
  host_gaussian(rows, cols, seed, real, g.data());
  householder_q(rows, cols, g, q);
  HostBlock b;
  b.rows = rows;
  b.cols = cols;
  b.a = std::move(q);
  return b;
}

void perturb(HostBlock& x, uint64_t seed, uint64_t kind, uint64_t level, uint64_t idx, double rel, bool real) {
  if (x.a.empty() || rel == 0.0) return;
  std::vector<cd> e(x.a.size());
  host_gaussian(x.rows, x.cols, seed_mix_host(seed, {7, kind, level, idx}), real, e.data());
  double nx = 0, ne = 0;
  for (size_t i = 0; i < e.size(); ++i) {
    nx += std::norm(x.a[i]);
    ne += std::norm(e[i]);
  }
  double f = rel * std::sqrt(nx) / std::sqrt(ne);
  for (size_t i = 0; i < e.size(); ++i) x.a[i] += f * e[i];
}

template <typename F>
void par_for(int64_t n, F fn) {
  unsigned nt = std::max(1u, std::min(32u, std::thread::hardware_concurrency()));
  std::vector<std::thread> pool;
  std::atomic<int64_t> next{0};
  for (unsigned t = 0; t < nt; ++t)
    pool.emplace_back([&] {
      for (;;) {
        int64_t i = next.fetch_add(1);
        if (i >= n) return;
        fn(i);
      }
    });
  for (auto& t : pool) t.join();
}
}  // namespace

HostButterfly synth_host(int levels, int64_t leaf, int64_t rank, uint64_t seed, bool real, double rel) {
  if (rank < 1 || rank > leaf) fail(PRECONDITION, "synth_butterfly: rank must lie in [1, leaf]");
  if (levels < 2) fail(PRECONDITION, "synth_butterfly: at least 2 levels required");
  int64_t n = (int64_t(1) << levels) * leaf;
  HostButterfly h;
  h.L = levels;
  h.lm = levels / 2;
  h.is_real = real;
  std::vector<double> line(3 * n, 0.0);
  for (int64_t i = 0; i < n; ++i) line[3 * i] = (double)i;
  h.rt = Tree::build(1, n, line.data(), levels);
  h.ct = h.rt;
  int64_t nbk = int64_t(1) << levels;
  auto mix = [&](uint64_t kind, uint64_t level, uint64_t idx) { return seed_mix_host(seed, {6, kind, level, idx}); };
  h.u.resize(nbk);
  h.v.resize(nbk);
  h.b.resize(nbk);
  h.r.assign(levels - h.lm, std::vector<HostBlock>(nbk));
  h.w.assign(h.lm, std::vector<HostBlock>(nbk));
  par_for(nbk, [&](int64_t i) {
    h.u[i] = random_orthonormal(leaf, rank, mix(1, 0, i), real);
    h.v[i] = random_orthonormal(leaf, rank, mix(2, 0, i), real);
    perturb(h.u[i], seed, 1, 0, i, rel, real);
    perturb(h.v[i], seed, 2, 0, i, rel, real);
    HostBlock& bb = h.b[i];
    bb.rows = bb.cols = rank;
    bb.a.resize(rank * rank);
    host_gaussian(rank, rank, mix(5, 0, i), real, bb.a.data());
    perturb(bb, seed, 5, 0, i, rel, real);
  });
  for (int l = h.lm; l < levels; ++l)
    par_for(nbk, [&](int64_t i) {
      h.r[l - h.lm][i] = random_orthonormal(2 * rank, rank, mix(3, l, i), real);
      perturb(h.r[l - h.lm][i], seed, 3, l, i, rel, real);
    });
  for (int l = 1; l <= h.lm; ++l)
    par_for(nbk, [&](int64_t i) {
      h.w[l - 1][i] = random_orthonormal(2 * rank, rank, mix(4, l, i), real);
      perturb(h.w[l - 1][i], seed, 4, l, i, rel, real);
    });
  h.validate();
  return h;
}

// ================================================================= device
template <typename R>
void Level<R>::finish_ranks(Ctx* c) {
  dranks.download(ranks.data(), ranks.size());
  c->sync();
  P = 0;
  for (int32_t x : ranks) P = std::max(P, (int)x);
}

template <typename R>
void DevButterfly<R>::setup_trees(Ctx* c, const Tree& row, const Tree& col, int levels, int center) {
  ctx = c;
  L = levels;
  lm = center;
  rt = row;
  ct = col;
  if (!rt.identity) rperm = to_device(c, rt.perm);
  if (!ct.identity) cperm = to_device(c, ct.perm);
  leaves_uniform_r = rt.max_size(L) * nb() == rt.n;
  leaves_uniform_c = ct.max_size(L) * nb() == ct.n;
  r.clear();
  w.clear();
  r.resize(L - lm);
  w.resize(lm);
}

template <typename R>
int64_t DevButterfly<R>::nnz() const {
  int64_t s = 0;
  for (int64_t i = 0; i < nb(); ++i) {
    s += rt.size(L, i) * uleaf.ranks[i] + ct.size(L, i) * vleaf.ranks[i];
    s += (int64_t)b.rows[i] * b.ranks[i];
  }
  for (const auto& lv : r)
    for (int64_t i = 0; i < nb(); ++i) s += (int64_t)lv.rows[i] * lv.ranks[i];
  for (const auto& lv : w)
    for (int64_t i = 0; i < nb(); ++i) s += (int64_t)lv.rows[i] * lv.ranks[i];
  return s;
}

template <typename R>
int64_t DevButterfly<R>::max_rank() const {
  int64_t m = std::max(uleaf.P, vleaf.P);
  for (const auto& lv : r) m = std::max<int64_t>(m, lv.P);
  for (const auto& lv : w) m = std::max<int64_t>(m, lv.P);
  return m;
}

template <typename R>
double DevButterfly<R>::apply_flops(int64_t k) const {
  return 8.0 * (double)nnz() * (double)k;
}
template <typename R>
double DevButterfly<R>::apply_bytes(int64_t k) const {
  return (double)sizeof(cx<R>) * ((double)nnz() + (double)(m() + n()) * (double)k);
}

template <typename R>
int DevButterfly<R>::max_p() const {
  int maxP = 1;
  for (int l = 0; l <= lm; ++l) maxP = std::max(maxP, PV(l));
  for (int l = lm; l <= L; ++l) maxP = std::max(maxP, PU(l));
  return maxP;
}

template <typename R>
DevButterfly<R>::~DevButterfly() {
  for (auto& g : graphs_)
    if (g->exec) cudaGraphExecDestroy(g->exec);
}

template <typename R>
bool DevButterfly<R>::apply_graph(int trans, const cx<R>* x, int64_t ldx, cx<R>* y, int64_t ldy, int64_t k) {
  static const bool disabled = std::getenv("BFLY_NO_GRAPHS") != nullptr;
  if (disabled || ctx->profiling || trans == OP_T || !rt.identity || !ct.identity) return false;
  GraphEntry* g = nullptr;
  for (auto& e : graphs_)
    if (e->trans == trans && e->x == x && e->y == y && e->ldx == ldx && e->ldy == ldy && e->k == k) g = e.get();
  if (!g) {
    if (graphs_.size() >= 8) {
      if (graphs_.front()->exec) cudaGraphExecDestroy(graphs_.front()->exec);
      graphs_.erase(graphs_.begin());
    }
    graphs_.push_back(std::make_unique<GraphEntry>());
    g = graphs_.back().get();
    g->trans = trans;
    g->x = x;
    g->y = y;
    g->ldx = ldx;
    g->ldy = ldy;
    g->k = k;
  }
  if (++g->uses < 2) return false;  // first call runs eagerly (builds the stage plan)
  if (!g->exec) {
    const size_t nbuf = (size_t)(nb() * max_p() * k);
    g->b0.reset(ctx, nbuf);
    g->b1.reset(ctx, nbuf);
    ctx->sync();
    const int64_t l0 = ctx->launches;
    cudaGraph_t graph;
    BFLY_CUDA(cudaStreamBeginCapture(ctx->stream, cudaStreamCaptureModeThreadLocal));
    try {
      if (trans == OP_N) apply_n(x, ldx, y, ldy, k, g->b0.p, g->b1.p);
      else apply_h(x, ldx, y, ldy, k, g->b0.p, g->b1.p);
    } catch (...) {
      cudaStreamEndCapture(ctx->stream, &graph);
      throw;
    }
    BFLY_CUDA(cudaStreamEndCapture(ctx->stream, &graph));
    g->kernels = ctx->launches - l0;
    ctx->launches = l0;
    BFLY_CUDA(cudaGraphInstantiate(&g->exec, graph, 0));
    cudaGraphDestroy(graph);
  }
  BFLY_CUDA(cudaGraphLaunch(g->exec, ctx->stream));
  ctx->launches += g->kernels;
  return true;
}

template <typename R>
void DevButterfly<R>::apply(int trans, const cx<R>* x, int64_t ldx, cx<R>* y, int64_t ldy, int64_t k) {
  Ctx* c = ctx;
  if (k <= 0) return;
  if (apply_graph(trans, x, ldx, y, ldy, k)) return;
  const bool fwd = trans == OP_N;
  const Tree& tin = fwd ? ct : rt;
  const Tree& tout = fwd ? rt : ct;
  const int64_t nin = tin.n, nout = tout.n;
  const DBuf<int64_t>& pin = fwd ? cperm : rperm;
  const DBuf<int64_t>& pout = fwd ? rperm : cperm;
  DBuf<cx<R>> xin, yout;
  const cx<R>* xt = x;
  int64_t ldxt = ldx;
  if (!tin.identity || trans == OP_T) {
    xin.reset(c, (size_t)(nin * k));
    if (!tin.identity) launch_permute_rows<R>(c, xin.p, nin, x, ldx, nin, k, pin.p, false);
    else launch_copy2d<R>(c, xin.p, nin, x, ldx, nin, k);
    if (trans == OP_T) launch_conj<R>(c, xin.p, nin, k, nin);
    xt = xin.p;
    ldxt = nin;
  }
  cx<R>* yt = y;
  int64_t ldyt = ldy;
  if (!tout.identity) {
    yout.reset(c, (size_t)(nout * k));
    yt = yout.p;
    ldyt = nout;
  }
  if (fwd) apply_n(xt, ldxt, yt, ldyt, k);
  else apply_h(xt, ldxt, yt, ldyt, k);
  if (!tout.identity) launch_permute_rows<R>(c, y, ldy, yt, nout, nout, k, pout.p, true);
  if (trans == OP_T) launch_conj<R>(c, y, nout, k, ldy);
}

namespace {
GemmEnt ent(int64_t a0, int64_t a1, int64_t b0, int64_t b1, int64_t c, int mrows, int krows) {
  GemmEnt e;
  e.a0 = a0; e.a1 = a1; e.b0 = b0; e.b1 = b1; e.c = c;
  e.ncols = 0; e.mrows = mrows; e.krows = krows; e.pad_ = 0;
  return e;
}
// the used prefix (ld x cols) of every block of a factor level
template <typename R>
L2Prefetch l2pf(const Level<R>& lv, int cols) {
  L2Prefetch p;
  p.base = lv.data.p;
  p.stride = lv.stride() * (int64_t)sizeof(cx<R>);
  p.len = std::min<int64_t>(lv.stride(), lv.ld * (int64_t)std::max(cols, 1)) * (int64_t)sizeof(cx<R>);
  return p;
}
}  // namespace

// Stage plans (butterfly.hpp:71-193): K x = U_L R_{L-1} .. R_lm B W_lm .. W_1 V_0^H x.
// Entry e of a stage computes C[c_e] = sum_s op(A[a_s]) B[b_s]; pad_ carries
// the stage index (BFLY_STAGE_TRACE instrumentation only).
template <typename R>
void DevButterfly<R>::build_plan_n() {
  Plan& pl = plan_n_;
  pl = Plan();
  const int64_t NB = nb();
  const int BIG = 1 << 30;
  auto add = [&](int op, int M, int K, int S, const Level<R>& lv, int64_t ld_out, int pfcols, int side,
                 int level) -> StageDesc& {
    pl.st.emplace_back();
    StageDesc& d = pl.st.back();
    d.op = op; d.M = M; d.K = K; d.S = S; d.A = lv.data.p; d.lda = lv.ld; d.ld_out = ld_out;
    d.pf = l2pf(lv, pfcols);
    d.own_side = side;
    d.own_level = level;
    return d;
  };
  auto push = [](StageDesc& d, const GemmEnt& e, int64_t tau, int64_t nu) {
    d.h.push_back(e);
    d.own_tau.push_back(tau);
    d.own_nu.push_back(nu);
  };
  {
    StageDesc& d = add(OP_H, PV(0), (int)vleaf.ld, 1, vleaf, NB * PV(0), PV(0), 0, 0);
    for (int64_t nu = 0; nu < NB; ++nu)
      push(d, ent(nu * vleaf.stride(), 0, ct.begin(L, nu), 0, nu * PV(0), BIG, (int)ct.size(L, nu)), 0, nu);
  }
  for (int l = 1; l <= lm; ++l) {
    const Level<R>& wl = w[l - 1];
    StageDesc& d = add(OP_H, PV(l), 2 * PV(l - 1), 1, wl, NB * PV(l), PV(l), 0, l);
    for (int64_t tau = 0; tau < (int64_t(1) << l); ++tau)
      for (int64_t nu = 0; nu < (int64_t(1) << (L - l)); ++nu) {
        int64_t i = bidx(L, l, tau, nu);
        push(d, ent(i * wl.stride(), 0, bidx(L, l - 1, tau / 2, 2 * nu) * PV(l - 1), 0, i * PV(l), BIG, BIG), tau,
             nu);
      }
  }
  {
    StageDesc& d = add(OP_N, PU(lm), PV(lm), 1, b, NB * PU(lm), PV(lm), 0, lm);
    for (int64_t i = 0; i < NB; ++i)
      push(d, ent(i * b.stride(), 0, i * PV(lm), 0, i * PU(lm), BIG, BIG), i >> (L - lm),
           i & ((int64_t(1) << (L - lm)) - 1));
  }
  for (int l = lm; l < L; ++l) {
    const Level<R>& rl = r[l - lm];
    StageDesc& d = add(OP_N, PU(l + 1), PU(l), 2, rl, NB * PU(l + 1), PU(l), 1, l + 1);
    for (int64_t tp = 0; tp < (int64_t(1) << (l + 1)); ++tp)
      for (int64_t np = 0; np < (int64_t(1) << (L - l - 1)); ++np) {
        int64_t tau = tp >> 1, h = tp & 1;
        int64_t i0 = bidx(L, l, tau, 2 * np), i1 = bidx(L, l, tau, 2 * np + 1);
        push(d, ent(i0 * rl.stride() + h * rl.gap, i1 * rl.stride() + h * rl.gap, i0 * PU(l), i1 * PU(l),
                    bidx(L, l + 1, tp, np) * PU(l + 1), BIG, BIG), tp, np);
      }
  }
  {
    StageDesc& d = add(OP_N, (int)uleaf.ld, PU(L), 1, uleaf, 0, PU(L), 1, L);
    for (int64_t tau = 0; tau < NB; ++tau)
      push(d, ent(tau * uleaf.stride(), 0, tau * PU(L), 0, rt.begin(L, tau), (int)rt.size(L, tau), BIG), tau, 0);
  }
  upload_plan(pl);
}

template <typename R>
void DevButterfly<R>::build_plan_h() {
  Plan& pl = plan_h_;
  pl = Plan();
  const int64_t NB = nb();
  const int BIG = 1 << 30;
  auto add = [&](int op, int M, int K, int S, const Level<R>& lv, int64_t ld_out, int pfcols, int side,
                 int level) -> StageDesc& {
    pl.st.emplace_back();
    StageDesc& d = pl.st.back();
    d.op = op; d.M = M; d.K = K; d.S = S; d.A = lv.data.p; d.lda = lv.ld; d.ld_out = ld_out;
    d.pf = l2pf(lv, pfcols);
    d.own_side = side;
    d.own_level = level;
    return d;
  };
  auto push = [](StageDesc& d, const GemmEnt& e, int64_t tau, int64_t nu) {
    d.h.push_back(e);
    d.own_tau.push_back(tau);
    d.own_nu.push_back(nu);
  };
  {
    StageDesc& d = add(OP_H, PU(L), (int)uleaf.ld, 1, uleaf, NB * PU(L), PU(L), 1, L);
    for (int64_t tau = 0; tau < NB; ++tau)
      push(d, ent(tau * uleaf.stride(), 0, rt.begin(L, tau), 0, tau * PU(L), BIG, (int)rt.size(L, tau)), tau, 0);
  }
  for (int l = L - 1; l >= lm; --l) {
    const Level<R>& rl = r[l - lm];
    StageDesc& d = add(OP_H, PU(l), PU(l + 1), 2, rl, NB * PU(l), PU(l), 1, l);
    for (int64_t tau = 0; tau < (int64_t(1) << l); ++tau)
      for (int64_t nu = 0; nu < (int64_t(1) << (L - l)); ++nu) {
        int64_t i = bidx(L, l, tau, nu);
        push(d, ent(i * rl.stride(), i * rl.stride() + rl.gap, bidx(L, l + 1, 2 * tau, nu / 2) * PU(l + 1),
                    bidx(L, l + 1, 2 * tau + 1, nu / 2) * PU(l + 1), i * PU(l), BIG, BIG), tau, nu);
      }
  }
  {
    StageDesc& d = add(OP_H, PV(lm), PU(lm), 1, b, NB * PV(lm), PV(lm), 0, lm);
    for (int64_t i = 0; i < NB; ++i)
      push(d, ent(i * b.stride(), 0, i * PU(lm), 0, i * PV(lm), BIG, BIG), i >> (L - lm),
           i & ((int64_t(1) << (L - lm)) - 1));
  }
  for (int l = lm; l >= 1; --l) {
    const Level<R>& wl = w[l - 1];
    StageDesc& d = add(OP_N, PV(l - 1), PV(l), 2, wl, NB * PV(l - 1), PV(l), 0, l - 1);
    for (int64_t tp = 0; tp < (int64_t(1) << (l - 1)); ++tp)
      for (int64_t npp = 0; npp < (int64_t(1) << (L - l + 1)); ++npp) {
        int64_t nu = npp >> 1, h = npp & 1;
        int64_t i0 = bidx(L, l, 2 * tp, nu), i1 = bidx(L, l, 2 * tp + 1, nu);
        push(d, ent(i0 * wl.stride() + h * wl.gap, i1 * wl.stride() + h * wl.gap, i0 * PV(l), i1 * PV(l),
                    bidx(L, l - 1, tp, npp) * PV(l - 1), BIG, BIG), tp, npp);
      }
  }
  {
    StageDesc& d = add(OP_N, (int)vleaf.ld, PV(0), 1, vleaf, 0, PV(0), 0, 0);
    for (int64_t nu = 0; nu < NB; ++nu)
      push(d, ent(nu * vleaf.stride(), 0, nu * PV(0), 0, ct.begin(L, nu), (int)ct.size(L, nu), BIG), 0, nu);
  }
  upload_plan(pl);
}

template <typename R>
void DevButterfly<R>::upload_plan(Plan& pl) {
  for (size_t i = 0; i < pl.st.size(); ++i) {
    for (auto& e : pl.st[i].h) e.pad_ = (int32_t)i;
    pl.st[i].d = to_device(ctx, pl.st[i].h);
  }
}

// One launch per stage, ping-ponging the coefficient vector between buf0 and
// buf1; every stage is a programmatic dependent launch that prefetches the
// next stage's factor level into L2 (see bgemm_stage_kernel).
template <typename R>
void DevButterfly<R>::run_plan(Plan& pl, const cx<R>* x, int64_t ldx, cx<R>* y, int64_t ldy, int64_t k,
                               cx<R>* buf0, cx<R>* buf1) {
  Ctx* c = ctx;
  const int64_t NB = nb();
  DBuf<cx<R>> b0, b1;
  if (!buf0) {
    b0.reset(c, (size_t)(NB * max_p() * k));
    b1.reset(c, (size_t)(NB * max_p() * k));
    buf0 = b0.p;
    buf1 = b1.p;
  }
  cx<R>* bufs[2] = {buf0, buf1};
  const int n = (int)pl.st.size();
  const cx<R>* in = x;
  int64_t ldin = ldx;
  for (int i = 0; i < n; ++i) {
    const StageDesc& d = pl.st[i];
    const bool final = i == n - 1;
    cx<R>* out = final ? y : bufs[i % 2];
    const int64_t ldout = final ? ldy : d.ld_out;
    // L2 prefetch of the next stage's factor level: off by default -- the next
    // stage's CTAs become resident early (PDL) and stage their factor blocks
    // by TMA themselves; measured k=1 71.6 -> 68.7 us without the prefetch
    static const bool l2pf = std::getenv("BFLY_L2PF") && std::atoi(std::getenv("BFLY_L2PF")) != 0;
    launch_bgemm<R>(c, d.op, d.M, d.K, d.S, d.A, d.lda, in, ldin, out, ldout, d.d.p, (int)d.h.size(), (int)k, false,
                    (int)k, true, (final || !l2pf) ? L2Prefetch() : pl.st[i + 1].pf);
    in = out;
    ldin = ldout;
  }
}

template <typename R>
void DevButterfly<R>::apply_n(const cx<R>* xt, int64_t ldx, cx<R>* yt, int64_t ldy, int64_t k, cx<R>* buf0,
                               cx<R>* buf1) {
  if (!have_n_) {
    build_plan_n();
    have_n_ = true;
  }
  run_plan(plan_n_, xt, ldx, yt, ldy, k, buf0, buf1);
}

template <typename R>
void DevButterfly<R>::apply_h(const cx<R>* yt, int64_t ldy, cx<R>* xt, int64_t ldx, int64_t k, cx<R>* buf0,
                               cx<R>* buf1) {
  if (!have_h_) {
    build_plan_h();
    have_h_ = true;
  }
  run_plan(plan_h_, yt, ldy, xt, ldx, k, buf0, buf1);
}

// Structured apply (see butterfly.h).  The stages are the ones of
// build_plan_n / build_plan_h; every entry carries the column window of the
// probes whose support reaches its block.  pt = the input-side tree, q = a
// node's level in it; a node at q >= plevel sees the one probe above it, a
// node at q < plevel the probes below it.  While the two sources of an entry
// sit at q > plevel they share a window (one S = 2 entry); from q == plevel
// upwards their windows are disjoint column ranges of the same output block,
// so the entry splits into two S = 1 entries and nothing reads a column it
// did not produce (no zero-filled coefficient buffers).
template <typename R>
bool DevButterfly<R>::apply_structured(int trans, int plevel, const std::vector<ProbeSeg>& segs, const cx<R>* X,
                                       int64_t ldx, cx<R>* y, int64_t ldy, int64_t o0, int64_t o1,
                                       double* flops_done, const Level<R>* G, int glevel, cx<R>* proj_c,
                                       int64_t proj_ldc) {
  Ctx* c = ctx;
  if ((trans != OP_N && trans != OP_H) || !rt.identity || !ct.identity) return false;
  if (plevel < 0 || plevel > L || segs.empty()) return false;
  const bool fwd = trans == OP_N;
  const Tree& pt = fwd ? ct : rt;
  const Tree& ot = fwd ? rt : ct;
  const int p = plevel;
  const int64_t NP = int64_t(1) << p, NB = nb();
  // basis projection at level glevel (see butterfly.h): V side levels 0..lm-1
  // for OP_H products, U side levels lm+1..L for OP_N products
  const bool proj = G != nullptr && proj_c != nullptr && (fwd ? (glevel > lm && glevel <= L) : (glevel >= 0 && glevel < lm));
  if (G && !proj) return false;
  // cs[j]: first column of probe node j (absent probes have zero width)
  std::vector<int64_t> cs(NP + 1, -1), xo(NP, -1);
  {
    int64_t col = segs[0].col0, prev = -1;
    for (const auto& s : segs) {
      if (s.node <= prev || s.node >= NP || s.col0 != col || s.ncols < 0) return false;
      for (int64_t j = prev + 1; j <= s.node; ++j) cs[j] = col;
      xo[s.node] = s.x_off;
      col += s.ncols;
      prev = s.node;
    }
    for (int64_t j = prev + 1; j <= NP; ++j) cs[j] = col;
  }
  const int64_t wend = cs[NP];
  if (wend - cs[0] <= 0) return true;
  // output restriction: a block is needed when its output-side node holds
  // requested points (its sources sit at that node's parent, so every block a
  // kept entry reads was kept too)
  const bool restrict_out = o1 >= 0 && (o0 > 0 || o1 < ot.n);
  auto need = [&](int q, int64_t u) { return !restrict_out || (ot.begin(q, u) < o1 && ot.end(q, u) > o0); };
  auto win = [&](int q, int64_t t, int64_t& c0, int64_t& nc) {
    int64_t j0, j1;
    if (q >= p) {
      j0 = t >> (q - p);
      j1 = j0 + 1;
    } else {
      j0 = t << (p - q);
      j1 = (t + 1) << (p - q);
    }
    c0 = cs[j0];
    nc = cs[j1] - cs[j0];
  };
  struct Stage {
    int op = 0, M = 0, K = 0, S = 1;
    const cx<R>* A = nullptr;
    int64_t lda = 0, ld_out = 0;
    std::vector<GemmEnt> h;
    int maxc = 0;
  };
  // coefficient buffers span every column of the batch
  DBuf<cx<R>> b0(c, (size_t)(NB * max_p() * wend)), b1(c, (size_t)(NB * max_p() * wend));
  cx<R>* bufs[2] = {b0.p, b1.p};
  const cx<R>* in = X;
  int64_t ldin = ldx;
  int nlaunched = 0;
  Stage cur;
  bool have_cur = false;
  // a stage is launched as soon as the next one begins (or at the end, as the
  // final stage writing y): the host plans stage i + 1 while the GPU runs stage i
  auto flush = [&](bool final) {
    if (!have_cur) return;
    cx<R>* out = final ? (proj ? proj_c : y) : bufs[nlaunched % 2];
    const int64_t ldout = final ? (proj ? proj_ldc : ldy) : cur.ld_out;
    if (!cur.h.empty()) {
      DBuf<GemmEnt> de = to_device(c, cur.h);
      launch_bgemm<R>(c, cur.op, cur.M, cur.K, cur.S, cur.A, cur.lda, in, ldin, out, ldout, de.p, (int)cur.h.size(),
                      cur.maxc, false, 0, true);
    }
    in = out;
    ldin = ldout;
    ++nlaunched;
    have_cur = false;
  };
  double flops = 0;
  auto add = [&](int op, int M, int K, int S, const Level<R>& lv, int64_t ld_out) -> Stage& {
    flush(false);
    cur = Stage();
    cur.op = op; cur.M = M; cur.K = K; cur.S = S; cur.A = lv.data.p; cur.lda = lv.ld; cur.ld_out = ld_out;
    have_cur = true;
    return cur;
  };
  // a0/a1/b0/b1/c: element offsets without the window; the window's first
  // column is added to the coefficient operands (ld_in) and the output (ld_out)
  auto push = [&](Stage& d, int64_t a0, int64_t a1, int64_t b0, int64_t b1, int64_t cc, int mrows, int krows,
                  int64_t c0, int64_t nc, int64_t ld_in, int64_t ld_o, double nz) {
    if (nc <= 0) return;
    GemmEnt e = ent(a0, a1, b0 + c0 * ld_in, b1 + c0 * ld_in, cc + c0 * ld_o, mrows, krows);
    e.ncols = (int32_t)nc;
    d.h.push_back(e);
    d.maxc = std::max<int>(d.maxc, (int)nc);
    flops += 8.0 * nz * (double)nc;
  };
  const int BIG = 1 << 30;
  int64_t c0, nc;
  if (fwd) {
    {  // V leaves: coefficients of the probes' own rows
      Stage& d = add(OP_H, PV(0), (int)vleaf.ld, 1, vleaf, NB * PV(0));
      for (int64_t nu = 0; nu < NB; ++nu) {
        win(L, nu, c0, nc);
        if (nc <= 0) continue;
        const int64_t j = p >= L ? nu : nu >> (L - p);  // p <= L: the probe above the leaf
        GemmEnt e = ent(nu * vleaf.stride(), 0, xo[j] + (ct.begin(L, nu) - ct.begin(p, j)), 0,
                        nu * PV(0) + c0 * d.ld_out, BIG, (int)ct.size(L, nu));
        e.ncols = (int32_t)nc;
        d.h.push_back(e);
        d.maxc = std::max<int>(d.maxc, (int)nc);
        flops += 8.0 * (double)ct.size(L, nu) * vleaf.ranks[nu] * (double)nc;
      }
    }
    for (int l = 1; l <= lm; ++l) {
      const Level<R>& wl = w[l - 1];
      const int q = L - l;  // column level of the outputs
      const bool shared = q >= p;
      const int64_t ld_in = NB * PV(l - 1);
      Stage& d = add(OP_H, PV(l), shared ? 2 * PV(l - 1) : PV(l - 1), 1, wl, NB * PV(l));
      for (int64_t tau = 0; tau < (int64_t(1) << l); ++tau)
        for (int64_t nu = 0; nu < (int64_t(1) << q); ++nu) {
          const int64_t i = bidx(L, l, tau, nu), src = bidx(L, l - 1, tau / 2, 2 * nu);
          if (!need(l, tau)) continue;
          if (shared) {
            win(q, nu, c0, nc);
            push(d, i * wl.stride(), 0, src * PV(l - 1), 0, i * PV(l), BIG, BIG, c0, nc, ld_in, d.ld_out,
                 (double)wl.rows[i] * wl.ranks[i]);
          } else {
            for (int h = 0; h < 2; ++h) {
              win(q + 1, 2 * nu + h, c0, nc);
              push(d, i * wl.stride() + h * wl.gap, 0, (src + h) * PV(l - 1), 0, i * PV(l), BIG, BIG, c0, nc, ld_in,
                   d.ld_out, (double)v_rank(l - 1, tau / 2, 2 * nu + h) * wl.ranks[i]);
            }
          }
        }
    }
    {
      Stage& d = add(OP_N, PU(lm), PV(lm), 1, b, NB * PU(lm));
      const int64_t ld_in = NB * PV(lm);
      for (int64_t i = 0; i < NB; ++i) {
        if (!need(lm, i >> (L - lm))) continue;
        win(L - lm, i & ((int64_t(1) << (L - lm)) - 1), c0, nc);
        push(d, i * b.stride(), 0, i * PV(lm), 0, i * PU(lm), BIG, BIG, c0, nc, ld_in, d.ld_out,
             (double)b.rows[i] * b.ranks[i]);
      }
    }
    for (int l = lm; l < (proj ? glevel : L); ++l) {
      const Level<R>& rl = r[l - lm];
      const int q = L - l - 1;  // column level of the outputs
      const bool shared = q >= p;
      const int64_t ld_in = NB * PU(l);
      Stage& d = add(OP_N, PU(l + 1), PU(l), shared ? 2 : 1, rl, NB * PU(l + 1));
      for (int64_t tp = 0; tp < (int64_t(1) << (l + 1)); ++tp)
        for (int64_t np = 0; np < (int64_t(1) << q); ++np) {
          const int64_t tau = tp >> 1, h = tp & 1;
          const int64_t i0 = bidx(L, l, tau, 2 * np), i1 = i0 + 1, o = bidx(L, l + 1, tp, np);
          const double rows_h = (double)u_rank(l + 1, tp, np);
          if (!need(l + 1, tp)) continue;
          if (shared) {
            win(q, np, c0, nc);
            push(d, i0 * rl.stride() + h * rl.gap, i1 * rl.stride() + h * rl.gap, i0 * PU(l), i1 * PU(l), o * PU(l + 1),
                 BIG, BIG, c0, nc, ld_in, d.ld_out, rows_h * (rl.ranks[i0] + rl.ranks[i1]));
          } else {
            for (int s = 0; s < 2; ++s) {
              const int64_t is = i0 + s;
              win(q + 1, 2 * np + s, c0, nc);
              push(d, is * rl.stride() + h * rl.gap, 0, is * PU(l), 0, o * PU(l + 1), BIG, BIG, c0, nc, ld_in,
                   d.ld_out, rows_h * rl.ranks[is]);
            }
          }
        }
    }
    if (proj) {  // coefficients in the other butterfly's U basis of level glevel
      const int t = glevel, q = L - t;
      Stage& d = add(OP_N, G->P, PU(t), 1, *G, 0);
      const int64_t ld_in = NB * PU(t);
      for (int64_t tp = 0; tp < (int64_t(1) << t); ++tp)
        for (int64_t np = 0; np < (int64_t(1) << q); ++np) {
          if (!need(t, tp)) continue;
          const int64_t i = bidx(L, t, tp, np);
          win(q, np, c0, nc);
          push(d, i * G->stride(), 0, i * PU(t), 0, tp * G->P, BIG, BIG, c0, nc, ld_in, proj_ldc,
               (double)G->ranks[i] * G->rows[i]);
        }
    } else {  // U leaves: every probe reaches every row
      Stage& d = add(OP_N, (int)uleaf.ld, PU(L), 1, uleaf, 0);
      const int64_t ld_in = NB * PU(L);
      for (int64_t tau = 0; tau < NB; ++tau)
        if (need(L, tau))
          push(d, tau * uleaf.stride(), 0, tau * PU(L), 0, rt.begin(L, tau), (int)rt.size(L, tau), BIG, cs[0],
               wend - cs[0], ld_in, ldy, (double)rt.size(L, tau) * uleaf.ranks[tau]);
    }
  } else {
    {  // U leaves
      Stage& d = add(OP_H, PU(L), (int)uleaf.ld, 1, uleaf, NB * PU(L));
      for (int64_t tau = 0; tau < NB; ++tau) {
        win(L, tau, c0, nc);
        if (nc <= 0) continue;
        const int64_t j = tau >> (L - p);
        GemmEnt e = ent(tau * uleaf.stride(), 0, xo[j] + (rt.begin(L, tau) - rt.begin(p, j)), 0,
                        tau * PU(L) + c0 * d.ld_out, BIG, (int)rt.size(L, tau));
        e.ncols = (int32_t)nc;
        d.h.push_back(e);
        d.maxc = std::max<int>(d.maxc, (int)nc);
        flops += 8.0 * (double)rt.size(L, tau) * uleaf.ranks[tau] * (double)nc;
      }
    }
    for (int l = L - 1; l >= lm; --l) {
      const Level<R>& rl = r[l - lm];
      const bool shared = l >= p;  // the outputs' row level
      const int64_t ld_in = NB * PU(l + 1);
      Stage& d = add(OP_H, PU(l), PU(l + 1), shared ? 2 : 1, rl, NB * PU(l));
      for (int64_t tau = 0; tau < (int64_t(1) << l); ++tau)
        for (int64_t nu = 0; nu < (int64_t(1) << (L - l)); ++nu) {
          const int64_t i = bidx(L, l, tau, nu);
          const int64_t s0 = bidx(L, l + 1, 2 * tau, nu / 2), s1 = bidx(L, l + 1, 2 * tau + 1, nu / 2);
          if (!need(L - l, nu)) continue;
          if (shared) {
            win(l, tau, c0, nc);
            push(d, i * rl.stride(), i * rl.stride() + rl.gap, s0 * PU(l + 1), s1 * PU(l + 1), i * PU(l), BIG, BIG, c0,
                 nc, ld_in, d.ld_out, (double)rl.rows[i] * rl.ranks[i]);
          } else {
            for (int h = 0; h < 2; ++h) {
              win(l + 1, 2 * tau + h, c0, nc);
              push(d, i * rl.stride() + h * rl.gap, 0, (h ? s1 : s0) * PU(l + 1), 0, i * PU(l), BIG, BIG, c0, nc,
                   ld_in, d.ld_out, (double)u_rank(l + 1, 2 * tau + h, nu / 2) * rl.ranks[i]);
            }
          }
        }
    }
    {
      Stage& d = add(OP_H, PV(lm), PU(lm), 1, b, NB * PV(lm));
      const int64_t ld_in = NB * PU(lm);
      for (int64_t i = 0; i < NB; ++i) {
        if (!need(L - lm, i & ((int64_t(1) << (L - lm)) - 1))) continue;
        win(lm, i >> (L - lm), c0, nc);
        push(d, i * b.stride(), 0, i * PU(lm), 0, i * PV(lm), BIG, BIG, c0, nc, ld_in, d.ld_out,
             (double)b.rows[i] * b.ranks[i]);
      }
    }
    for (int l = lm; l >= (proj ? glevel + 1 : 1); --l) {
      const Level<R>& wl = w[l - 1];
      const bool shared = l - 1 >= p;  // the outputs' row level
      const int64_t ld_in = NB * PV(l);
      Stage& d = add(OP_N, PV(l - 1), PV(l), shared ? 2 : 1, wl, NB * PV(l - 1));
      for (int64_t tp = 0; tp < (int64_t(1) << (l - 1)); ++tp)
        for (int64_t npp = 0; npp < (int64_t(1) << (L - l + 1)); ++npp) {
          const int64_t nu = npp >> 1, h = npp & 1;
          const int64_t i0 = bidx(L, l, 2 * tp, nu), i1 = bidx(L, l, 2 * tp + 1, nu), o = bidx(L, l - 1, tp, npp);
          const double rows_h = (double)v_rank(l - 1, tp, npp);
          if (!need(L - l + 1, npp)) continue;
          if (shared) {
            win(l - 1, tp, c0, nc);
            push(d, i0 * wl.stride() + h * wl.gap, i1 * wl.stride() + h * wl.gap, i0 * PV(l), i1 * PV(l), o * PV(l - 1),
                 BIG, BIG, c0, nc, ld_in, d.ld_out, rows_h * (wl.ranks[i0] + wl.ranks[i1]));
          } else {
            for (int s = 0; s < 2; ++s) {
              const int64_t is = s ? i1 : i0;
              win(l, 2 * tp + s, c0, nc);
              push(d, is * wl.stride() + h * wl.gap, 0, is * PV(l), 0, o * PV(l - 1), BIG, BIG, c0, nc, ld_in,
                   d.ld_out, rows_h * wl.ranks[is]);
            }
          }
        }
    }
    if (proj) {  // coefficients in the other butterfly's V basis of level glevel
      const int t = glevel, q = L - t;
      Stage& d = add(OP_N, G->P, PV(t), 1, *G, 0);
      const int64_t ld_in = NB * PV(t);
      for (int64_t tt = 0; tt < (int64_t(1) << t); ++tt)
        for (int64_t nu = 0; nu < (int64_t(1) << q); ++nu) {
          if (!need(q, nu)) continue;
          const int64_t i = bidx(L, t, tt, nu);
          win(t, tt, c0, nc);
          push(d, i * G->stride(), 0, i * PV(t), 0, nu * G->P, BIG, BIG, c0, nc, ld_in, proj_ldc,
               (double)G->ranks[i] * G->rows[i]);
        }
    } else {  // V leaves: every probe reaches every column point
      Stage& d = add(OP_N, (int)vleaf.ld, PV(0), 1, vleaf, 0);
      const int64_t ld_in = NB * PV(0);
      for (int64_t nu = 0; nu < NB; ++nu)
        if (need(L, nu))
          push(d, nu * vleaf.stride(), 0, nu * PV(0), 0, ct.begin(L, nu), (int)ct.size(L, nu), BIG, cs[0],
               wend - cs[0], ld_in, ldy, (double)ct.size(L, nu) * vleaf.ranks[nu]);
    }
  }
  flush(true);
  if (flops_done) *flops_done = flops;
  return true;
}

// ------------------------------------------------------- host <-> device
namespace {
template <typename R>
std::vector<std::complex<double>> download_level(const Level<R>& lv, int64_t nbk) {
  std::vector<cx<R>> raw((size_t)(nbk * lv.stride()));
  lv.data.download(raw.data(), raw.size());
  BFLY_CUDA(cudaStreamSynchronize(lv.data.ctx->stream));
  std::vector<std::complex<double>> out(raw.size());
  for (size_t i = 0; i < raw.size(); ++i) out[i] = {(double)raw[i].x, (double)raw[i].y};
  return out;
}
// compact block: rows [0, r1) from stored [0, r1), rows [r1, r1+r2) from [gap, gap+r2)
HostBlock extract(const std::vector<std::complex<double>>& raw, int64_t base, int64_t ld, int64_t r1, int64_t r2,
                  int64_t gap, int64_t cols) {
  HostBlock b;
  b.rows = r1 + r2;
  b.cols = cols;
  b.a.resize(b.rows * cols);
  for (int64_t c = 0; c < cols; ++c) {
    for (int64_t i = 0; i < r1; ++i) b.a[i + c * b.rows] = raw[base + i + c * ld];
    for (int64_t i = 0; i < r2; ++i) b.a[r1 + i + c * b.rows] = raw[base + gap + i + c * ld];
  }
  return b;
}
template <typename R>
void upload_level(Ctx* c, Level<R>& lv, int64_t nbk, const std::vector<const HostBlock*>& blocks,
                  const std::vector<int64_t>& r1s, int64_t gap, int64_t ld) {
  int P = 0;
  for (auto* b : blocks) P = std::max<int>(P, (int)b->cols);
  lv.alloc(c, nbk, ld, std::max(P, 1));
  lv.P = P;
  lv.gap = (int)gap;
  std::vector<cx<R>> raw((size_t)(nbk * lv.stride()), mkc<R>(0, 0));
  for (int64_t i = 0; i < nbk; ++i) {
    const HostBlock* b = blocks[i];
    int64_t r1 = r1s[i], r2 = b->rows - r1;
    for (int64_t col = 0; col < b->cols; ++col) {
      for (int64_t q = 0; q < r1; ++q) {
        auto z = b->a[q + col * b->rows];
        raw[i * lv.stride() + q + col * lv.ld] = mkc<R>((R)z.real(), (R)z.imag());
      }
      for (int64_t q = 0; q < r2; ++q) {
        auto z = b->a[r1 + q + col * b->rows];
        raw[i * lv.stride() + gap + q + col * lv.ld] = mkc<R>((R)z.real(), (R)z.imag());
      }
    }
    lv.ranks[i] = (int32_t)b->cols;
    lv.rows[i] = (int32_t)b->rows;
  }
  lv.data.upload(raw.data(), raw.size());
  lv.dranks.upload(lv.ranks.data(), lv.ranks.size());
  c->sync();
}
}  // namespace

template <typename R>
HostButterfly DevButterfly<R>::to_host() const {
  HostButterfly h;
  h.L = L;
  h.lm = lm;
  h.is_real = is_real;
  h.rt = rt;
  h.ct = ct;
  const int64_t NB = nb();
  {
    auto raw = download_level(uleaf, NB);
    for (int64_t t = 0; t < NB; ++t) h.u.push_back(extract(raw, t * uleaf.stride(), uleaf.ld, rt.size(L, t), 0, 0, uleaf.ranks[t]));
  }
  {
    auto raw = download_level(vleaf, NB);
    for (int64_t t = 0; t < NB; ++t) h.v.push_back(extract(raw, t * vleaf.stride(), vleaf.ld, ct.size(L, t), 0, 0, vleaf.ranks[t]));
  }
  h.r.resize(L - lm);
  for (int l = lm; l < L; ++l) {
    const Level<R>& lv = r[l - lm];
    auto raw = download_level(lv, NB);
    for (int64_t tau = 0; tau < (int64_t(1) << l); ++tau)
      for (int64_t nu = 0; nu < (int64_t(1) << (L - l)); ++nu) {
        int64_t i = bidx(L, l, tau, nu);
        h.r[l - lm].resize(NB);
        h.r[l - lm][i] = extract(raw, i * lv.stride(), lv.ld, u_rank(l + 1, 2 * tau, nu / 2),
                                 u_rank(l + 1, 2 * tau + 1, nu / 2), lv.gap, lv.ranks[i]);
      }
  }
  h.w.resize(lm);
  for (int l = 1; l <= lm; ++l) {
    const Level<R>& lv = w[l - 1];
    auto raw = download_level(lv, NB);
    h.w[l - 1].resize(NB);
    for (int64_t tau = 0; tau < (int64_t(1) << l); ++tau)
      for (int64_t nu = 0; nu < (int64_t(1) << (L - l)); ++nu) {
        int64_t i = bidx(L, l, tau, nu);
        h.w[l - 1][i] = extract(raw, i * lv.stride(), lv.ld, v_rank(l - 1, tau / 2, 2 * nu),
                                v_rank(l - 1, tau / 2, 2 * nu + 1), lv.gap, lv.ranks[i]);
      }
  }
  {
    auto raw = download_level(b, NB);
    h.b.resize(NB);
    for (int64_t tau = 0; tau < (int64_t(1) << lm); ++tau)
      for (int64_t nu = 0; nu < (int64_t(1) << (L - lm)); ++nu) {
        int64_t i = bidx(L, lm, tau, nu);
        h.b[i] = extract(raw, i * b.stride(), b.ld, u_rank(lm, tau, nu), 0, 0, v_rank(lm, tau, nu));
      }
  }
  return h;
}

template <typename R>
std::unique_ptr<DevButterfly<R>> DevButterfly<R>::from_host(Ctx* c, const HostButterfly& h) {
  h.validate();
  auto d = std::make_unique<DevButterfly<R>>();
  d->setup_trees(c, h.rt, h.ct, h.L, h.lm);
  d->is_real = h.is_real;
  const int64_t NB = d->nb();
  const int L = h.L, lm = h.lm;
  std::vector<const HostBlock*> blocks(NB);
  std::vector<int64_t> r1(NB);
  for (int64_t i = 0; i < NB; ++i) { blocks[i] = &h.u[i]; r1[i] = h.u[i].rows; }
  upload_level(c, d->uleaf, NB, blocks, r1, 0, h.rt.max_size(L));
  for (int64_t i = 0; i < NB; ++i) { blocks[i] = &h.v[i]; r1[i] = h.v[i].rows; }
  upload_level(c, d->vleaf, NB, blocks, r1, 0, h.ct.max_size(L));
  for (int l = L - 1; l >= lm; --l) {
    int gap = d->PU(l + 1);
    for (int64_t tau = 0; tau < (int64_t(1) << l); ++tau)
      for (int64_t nu = 0; nu < (int64_t(1) << (L - l)); ++nu) {
        int64_t i = bidx(L, l, tau, nu);
        blocks[i] = &h.r[l - lm][i];
        r1[i] = h.u_rank(l + 1, 2 * tau, nu / 2);
      }
    upload_level(c, d->r[l - lm], NB, blocks, r1, gap, 2 * std::max(gap, 0) > 0 ? 2 * gap : 1);
  }
  for (int l = 1; l <= lm; ++l) {
    int gap = d->PV(l - 1);
    for (int64_t tau = 0; tau < (int64_t(1) << l); ++tau)
      for (int64_t nu = 0; nu < (int64_t(1) << (L - l)); ++nu) {
        int64_t i = bidx(L, l, tau, nu);
        blocks[i] = &h.w[l - 1][i];
        r1[i] = h.v_rank(l - 1, tau / 2, 2 * nu);
      }
    upload_level(c, d->w[l - 1], NB, blocks, r1, gap, gap > 0 ? 2 * gap : 1);
  }
  for (int64_t i = 0; i < NB; ++i) { blocks[i] = &h.b[i]; r1[i] = h.b[i].rows; }
  upload_level(c, d->b, NB, blocks, r1, 0, std::max(d->PU(lm), 1));
  // B's P is its column count; keep rows info for nnz
  return d;
}

namespace {
struct ByteSink {
  uint8_t* out;
  int64_t pos = 0;
  void put(const void* p, size_t n) {
    if (out) std::memcpy(out + pos, p, n);
    pos += (int64_t)n;
  }
  void u32(uint32_t v) { put(&v, 4); }
  void u64(uint64_t v) { put(&v, 8); }
};

// One level's blocks in .bfh layout (serialize.hpp:103-127): per block the
// u64 row and column counts, then the compact column-major payload (rows
// [0, r1) and [gap, gap + r2) of every column) as f64 (real) or c128.
// Byte-granular stores: the payload's file offset has no alignment.
struct PackBlk {
  int64_t off;      // byte offset of the block header in the output
  int32_t r1, r2, cols, pad_;
};
template <typename R>
__global__ void pack_level_kernel(const cx<R>* __restrict__ data, int64_t ld, int64_t stride, int64_t gap,
                                  const PackBlk* __restrict__ blks, int nb, int real, uint8_t* __restrict__ out) {
  for (int i = blockIdx.x; i < nb; i += gridDim.x) {
    const PackBlk b = blks[i];
    const int64_t rows = b.r1 + b.r2;
    uint8_t* dst = out + b.off;
    if (threadIdx.x < 16) {
      const uint64_t v = threadIdx.x < 8 ? (uint64_t)rows : (uint64_t)b.cols;
      dst[threadIdx.x] = (uint8_t)(v >> (8 * (threadIdx.x & 7)));
    }
    dst += 16;
    const cx<R>* blk = data + (int64_t)i * stride;
    const int64_t n = rows * b.cols;
    for (int64_t e = threadIdx.x; e < n; e += blockDim.x) {
      const int64_t c = e / rows, q = e - c * rows;
      const cx<R> v = blk[c * ld + (q < b.r1 ? q : gap + (q - b.r1))];
      if (real) {
        const double x = (double)v.x;
        const uint64_t u = (uint64_t)__double_as_longlong(x);
#pragma unroll
        for (int t = 0; t < 8; ++t) dst[8 * e + t] = (uint8_t)(u >> (8 * t));
      } else {
        const uint64_t u0 = (uint64_t)__double_as_longlong((double)v.x);
        const uint64_t u1 = (uint64_t)__double_as_longlong((double)v.y);
#pragma unroll
        for (int t = 0; t < 8; ++t) {
          dst[16 * e + t] = (uint8_t)(u0 >> (8 * t));
          dst[16 * e + 8 + t] = (uint8_t)(u1 >> (8 * t));
        }
      }
    }
  }
}
}  // namespace

template <typename R>
int64_t DevButterfly<R>::serialize(int tag, uint8_t* out) const {
  ByteSink bs{out};
  const bool real = tag == 0;
  const int64_t NB = nb();
  bs.u32(0x31484642u);
  bs.u32(1);
  uint8_t t8 = (uint8_t)tag;
  bs.put(&t8, 1);
  bs.u32((uint32_t)L);
  bs.u32((uint32_t)lm);
  bs.u64((uint64_t)rt.n);
  bs.u64((uint64_t)ct.n);
  bs.u64((uint64_t)nnz());
  bs.u64((uint64_t)max_rank());
  for (const Tree* t : {&rt, &ct}) {
    bs.u64((uint64_t)t->n);
    bs.u32((uint32_t)t->levels);
    bs.put(t->perm.data(), sizeof(int64_t) * t->perm.size());
    for (const auto& lv : t->ranges) bs.put(lv.data(), sizeof(int64_t) * lv.size());
  }
  // levels: block headers + payloads, packed on the device into one buffer
  // (exact file layout) and copied to the host once
  const int64_t body0 = bs.pos;
  const int64_t esz = real ? 8 : 16;
  struct LevelJob {
    const Level<R>* lv;
    std::vector<PackBlk> blks;
  };
  std::vector<LevelJob> jobs;
  int64_t pos = 0;  // relative to body0
  auto emit = [&](const Level<R>& lv, auto rows_of) {
    LevelJob j{&lv, std::vector<PackBlk>((size_t)NB)};
    for (int64_t i = 0; i < NB; ++i) {
      int64_t r1, r2;
      rows_of(i, r1, r2);
      PackBlk& b = j.blks[(size_t)i];
      b.off = pos;
      b.r1 = (int32_t)r1;
      b.r2 = (int32_t)r2;
      b.cols = lv.ranks[i];
      b.pad_ = 0;
      pos += 16 + (r1 + r2) * (int64_t)b.cols * esz;
    }
    jobs.push_back(std::move(j));
  };
  emit(uleaf, [&](int64_t i, int64_t& r1, int64_t& r2) { r1 = rt.size(L, i); r2 = 0; });
  for (int l = lm; l < L; ++l)
    emit(r[l - lm], [&](int64_t i, int64_t& r1, int64_t& r2) {
      int64_t tau = i >> (L - l), nu = i & ((int64_t(1) << (L - l)) - 1);
      r1 = u_rank(l + 1, 2 * tau, nu / 2);
      r2 = u_rank(l + 1, 2 * tau + 1, nu / 2);
    });
  emit(b, [&](int64_t i, int64_t& r1, int64_t& r2) { r1 = b.rows[i]; r2 = 0; });
  for (int l = 1; l <= lm; ++l)
    emit(w[l - 1], [&](int64_t i, int64_t& r1, int64_t& r2) {
      int64_t tau = i >> (L - l), nu = i & ((int64_t(1) << (L - l)) - 1);
      r1 = v_rank(l - 1, tau / 2, 2 * nu);
      r2 = v_rank(l - 1, tau / 2, 2 * nu + 1);
    });
  emit(vleaf, [&](int64_t i, int64_t& r1, int64_t& r2) { r1 = ct.size(L, i); r2 = 0; });
  if (out && pos > 0) {
    Ctx* c = ctx;
    DBuf<uint8_t> body(c, (size_t)pos);
    for (const LevelJob& j : jobs) {
      DBuf<PackBlk> db = to_device(c, j.blks);
      const unsigned grid = (unsigned)std::min<int64_t>(NB, (int64_t)c->sm_count * 16);
      pack_level_kernel<R><<<grid, 256, 0, c->stream>>>(j.lv->data.p, j.lv->ld, j.lv->stride(), j.lv->gap, db.p,
                                                        (int)NB, real ? 1 : 0, body.p);
      BFLY_LAUNCH_CHECK("pack_level");
    }
    BFLY_CUDA(cudaMemcpyAsync(out + body0, body.p, (size_t)pos, cudaMemcpyDeviceToHost, c->stream));
    BFLY_CUDA(cudaStreamSynchronize(c->stream));
  }
  return body0 + pos;
}

template struct Level<double>;
template struct Level<float>;
template struct DevButterfly<double>;
template struct DevButterfly<float>;

}  // namespace bfly
