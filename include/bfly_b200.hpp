// bfly_b200.hpp -- header-only C++ adapter between the reference library
// (bfly::BlackBoxOperator / HybridButterfly / ReconstructionConfig, the
// reference's include/bfly/*.hpp) and the B200 C ABI (bfly_b200.h).
//
// Include it AFTER the reference headers.  It gives reference users a
// drop-in GPU factorizer:
//
//   bfly_b200::Context gpu(0);
//   auto [bf, log] = bfly_b200::factorize(gpu, op, row_tree, col_tree, cfg);
//
// where `op` is ANY bfly::BlackBoxOperator<Scalar> (its apply /
// apply_transpose are called through the stream-ordered callback, exactly as
// the reference's Factorizer calls them, operators.hpp:27-38) and the result
// is a reference bfly::HybridButterfly<Scalar> (built from the .bfh bytes the
// GPU writes, serialize.hpp:148-177).  Built-in kernel operators
// (bfly_op_kernel) skip the callback and evaluate on the device.
#pragma once

#include <cuda_runtime.h>

#include <complex>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <sstream>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "bfly_b200.h"

namespace bfly_b200 {

inline void check(int rc) {
  if (rc == BFLY_OK) return;
  const std::string msg = bfly_last_error();
  switch (rc) {  // the reference error hierarchy (core.hpp:43-60)
    case BFLY_PRECONDITION: throw bfly::precondition_error(msg);
    case BFLY_DIMENSION: throw bfly::dimension_error(msg);
    case BFLY_SEQUENCING: throw bfly::sequencing_error(msg);
    case BFLY_FORMAT: throw bfly::format_error(msg);
    case BFLY_CONDITIONING: throw bfly::conditioning_error(msg);
    default: throw bfly::error("bfly_b200: " + msg);
  }
}

template <class S> struct scalar_id;
template <> struct scalar_id<std::complex<double>> { static constexpr int value = BFLY_Z; };
template <> struct scalar_id<double> { static constexpr int value = BFLY_D; };

class Context {
 public:
  explicit Context(int device = 0) { check(bfly_ctx_create(device, &h_)); }
  ~Context() { bfly_ctx_destroy(h_); }
  Context(const Context&) = delete;
  Context& operator=(const Context&) = delete;
  bfly_ctx* get() const { return h_; }

 private:
  bfly_ctx* h_ = nullptr;
};

namespace detail {

// device layout: complex128 for BFLY_Z and BFLY_D (real64 uses complex storage)
template <class S>
struct Bridge {
  const bfly::BlackBoxOperator<S>* op;
  static int call(void* user, int trans, const void* x_dev, int64_t ldx, void* y_dev, int64_t ldy, int64_t k,
                  void* stream) {
    auto* self = static_cast<Bridge*>(user);
    if (std::getenv("BFLY_ADAPTER_TRACE"))
      std::fprintf(stderr, "[bridge] trans %d ldx %lld ldy %lld k %lld\n", trans, (long long)ldx, (long long)ldy,
                   (long long)k);
    try {
      auto s = static_cast<cudaStream_t>(stream);
      const bfly::Index nin = trans ? self->op->rows() : self->op->cols();
      const bfly::Index nout = trans ? self->op->cols() : self->op->rows();
      std::vector<std::complex<double>> hx((size_t)(nin * k)), hy((size_t)(nout * k));
      cudaMemcpy2DAsync(hx.data(), sizeof(std::complex<double>) * nin, x_dev, sizeof(std::complex<double>) * ldx,
                        sizeof(std::complex<double>) * nin, k, cudaMemcpyDeviceToHost, s);
      cudaStreamSynchronize(s);
      bfly::Matrix<S> X(nin, k);
      for (bfly::Index j = 0; j < k; ++j)
        for (bfly::Index i = 0; i < nin; ++i) {
          if constexpr (std::is_same<S, double>::value) X(i, j) = hx[i + j * nin].real();
          else X(i, j) = hx[i + j * nin];
        }
      // plain products through the reference's own public wrappers (counted)
      bfly::Matrix<S> Y = trans ? self->op->apply_transpose(X) : self->op->apply(X);
      for (bfly::Index j = 0; j < k; ++j)
        for (bfly::Index i = 0; i < nout; ++i) hy[i + j * nout] = Y(i, j);
      cudaMemcpy2DAsync(y_dev, sizeof(std::complex<double>) * ldy, hy.data(), sizeof(std::complex<double>) * nout,
                        sizeof(std::complex<double>) * nout, k, cudaMemcpyHostToDevice, s);
      cudaStreamSynchronize(s);
      return 0;
    } catch (const bfly::dimension_error&) {
      return BFLY_DIMENSION;
    } catch (...) {
      return BFLY_PRECONDITION;
    }
  }
};

inline bfly_tree* make_tree(const bfly::PartitionTree& t) {
  std::vector<int64_t> perm(t.permutation().begin(), t.permutation().end()), flat;
  for (const auto& lv : t.range_table()) flat.insert(flat.end(), lv.begin(), lv.end());
  bfly_tree* h = nullptr;
  check(bfly_tree_from_table(t.size(), t.levels(), perm.data(), flat.data(), &h));
  return h;
}

inline bfly_recon_cfg make_cfg(const bfly::ReconstructionConfig& c) {
  bfly_recon_cfg g;
  bfly_cfg_default(&g);
  g.tolerance = c.tolerance;
  g.oversampling = c.oversampling;
  g.rank_guess = c.rank_guess;
  g.levels = c.levels;
  g.center = c.center;
  g.seed = c.seed;
  g.hard_cap = c.hard_cap;
  g.threads = c.threads;
  g.literal_transpose_core = c.literal_transpose_core ? 1 : 0;
  return g;
}

inline bfly::FactorizationLog to_log(const bfly_log& l) {
  bfly::FactorizationLog log;
  for (int i = 0; i < l.nphases; ++i) {
    bfly::PhaseStat p;
    p.name = l.phases[i].name;
    p.forward_columns = l.phases[i].forward_columns;
    p.transpose_columns = l.phases[i].transpose_columns;
    p.seconds = l.phases[i].seconds;
    p.rounds = l.phases[i].rounds;
    p.probe_width = l.phases[i].probe_width;
    log.phases.push_back(p);
  }
  log.peak_probe_bytes = l.peak_probe_bytes;
  log.peak_concurrent_probes = l.peak_concurrent_probes;
  log.rank_capped = l.rank_capped != 0;
  log.total_seconds = l.total_seconds;
  return log;
}

}  // namespace detail

// to_reference(bf): the GPU butterfly as a reference HybridButterfly (via .bfh)
template <class S>
bfly::HybridButterfly<S> to_reference(const bfly_bf* bf) {
  const int64_t n = bfly_serialize(bf, nullptr);
  if (n < 0) check(BFLY_CUDA);
  std::string bytes((size_t)n, '\0');
  bfly_serialize(bf, reinterpret_cast<uint8_t*>(&bytes[0]));
  std::istringstream is(bytes, std::ios::binary);
  return bfly::deserialize<S>(is);
}

// factorize() (reconstruct.hpp:412-419) on the GPU for any reference operator
template <class S>
std::pair<bfly::HybridButterfly<S>, bfly::FactorizationLog> factorize(Context& ctx,
                                                                      const bfly::BlackBoxOperator<S>& op,
                                                                      const bfly::PartitionTree& row_tree,
                                                                      const bfly::PartitionTree& col_tree,
                                                                      const bfly::ReconstructionConfig& cfg) {
  detail::Bridge<S> bridge{&op};
  bfly_op* dop = nullptr;
  check(bfly_op_callback(ctx.get(), op.rows(), op.cols(), scalar_id<S>::value, &detail::Bridge<S>::call, &bridge,
                         &dop));
  bfly_tree* rt = detail::make_tree(row_tree);
  bfly_tree* ct = detail::make_tree(col_tree);
  bfly_recon_cfg c = detail::make_cfg(cfg);
  bfly_bf* bf = nullptr;
  bfly_log log{};
  const int rc = bfly_factorize(ctx.get(), dop, rt, ct, &c, &bf, &log);
  bfly_tree_destroy(rt);
  bfly_tree_destroy(ct);
  bfly_op_destroy(dop);
  check(rc);
  auto out = std::make_pair(to_reference<S>(bf), detail::to_log(log));
  bfly_bf_destroy(bf);
  return out;
}

}  // namespace bfly_b200
