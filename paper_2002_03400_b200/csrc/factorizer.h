// factorizer.h -- Algorithm 2 driver on the GPU (reference Factorizer,
// reconstruct.hpp:145-410): same phase order, seeds, probe widths,
// truncation and stop rule; every level runs as a handful of batched launches.
#pragma once

#include <chrono>
#include <memory>
#include <string>
#include <vector>

#include "../../include/bfly_b200.h"
#include "butterfly.h"
#include "operators.h"

namespace bfly {

template <typename R>
class Factorizer {
 public:
  Factorizer(Ctx* c, DevOp<R>* op, const Tree& rt, const Tree& ct, const bfly_recon_cfg& cfg);
  void leaf_row_bases();
  void leaf_col_bases();
  void transfer_level_w(int l);
  void transfer_level_r(int l);
  bool complete() const { return core_done_; }
  void run();
  std::unique_ptr<DevButterfly<R>> take(bfly_log* log);
  const bfly_log& log() const { return log_; }

 private:
  using V = cx<R>;
  using clock = std::chrono::steady_clock;
  Ctx* c_;
  DevOp<R>* op_;
  bfly_recon_cfg cfg_;
  std::unique_ptr<DevButterfly<R>> bf_;
  bfly_log log_{};
  bool v_done_ = false, u_done_ = false, core_done_ = false;
  int next_w_ = 1, next_r_ = 0;
  double flops_ = 0;  // chain + QR + core-fit work (black box counted by the operator)

  bfly_phase& new_phase(const std::string& name);
  void end_phase(bfly_phase& st, clock::time_point t0, int64_t f0, int64_t tr0);
  void note_probe_bytes(double scalars, int64_t probes);
  void run_leaf_phase(const char* name, bool row_side);
  // black-box product of a batch of structured probes (cores in G) into Y
  // (out_dim x wtot, tree ordered on return)
  void probe_products(int mode, const Tree& probe_tree, int level, const std::vector<int64_t>& nodes,
                      const std::vector<int>& widths, const std::vector<int64_t>& col0, const std::vector<int64_t>& goff,
                      const V* G, int64_t wtot, DBuf<V>& Y);
  double qr_flops(double a, double w, double k) const;
};

}  // namespace bfly
