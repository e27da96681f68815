// adapter_demo.cpp -- drop-in check of include/bfly_b200.hpp: the reference's
// own operators (compiled unmodified against the Eigen-API shim) factorized
// by the B200 library through the C-ABI callback, compared with the
// reference's CPU factorize() in the same process.  Exit code 0 = parity.
#include <cstdio>

#include "bfly/reconstruct.hpp"
#include "bfly/serialize.hpp"
#include "../../include/bfly_b200.hpp"

using namespace bfly;
using cplx = std::complex<double>;

template <class S>
static int compare(const char* name, const BlackBoxOperator<S>& op, const PartitionTree& rt, const PartitionTree& ct,
                   const ReconstructionConfig& cfg, bfly_b200::Context& gpu) {
  std::fprintf(stderr, "[demo] %s: cpu factorize\n", name);
  auto cpu = factorize<S>(op, rt, ct, cfg);
  std::fprintf(stderr, "[demo] %s: gpu factorize\n", name);
  auto gpu_res = bfly_b200::factorize<S>(gpu, op, rt, ct, cfg);
  std::fprintf(stderr, "[demo] %s: compare\n", name);
  const HybridButterfly<S>& a = cpu.first;
  const HybridButterfly<S>& b = gpu_res.first;
  bool ranks = true;
  for (int l = a.center; l <= a.levels; ++l)
    for (Index t = 0; t < (Index(1) << l); ++t)
      for (Index u = 0; u < (Index(1) << (a.levels - l)); ++u) ranks &= a.u_rank(l, t, u) == b.u_rank(l, t, u);
  for (int l = 0; l <= a.center; ++l)
    for (Index t = 0; t < (Index(1) << l); ++t)
      for (Index u = 0; u < (Index(1) << (a.levels - l)); ++u) ranks &= a.v_rank(l, t, u) == b.v_rank(l, t, u);
  Matrix<S> x = gaussian_matrix<S>(op.cols(), 8, 77);
  double rel = (a.apply(x) - b.apply(x)).norm() / a.apply(x).norm();
  bool cols = cpu.second.phases.size() == gpu_res.second.phases.size();
  for (size_t i = 0; cols && i < cpu.second.phases.size(); ++i)
    cols = cpu.second.phases[i].forward_columns == gpu_res.second.phases[i].forward_columns &&
           cpu.second.phases[i].transpose_columns == gpu_res.second.phases[i].transpose_columns &&
           cpu.second.phases[i].rounds == gpu_res.second.phases[i].rounds;
  double err = estimate_error<S>(op, b, 16, 5);
  std::printf("%s: ranks %s, bookkeeping %s, apply rel diff %.3e, GPU factorization error %.3e\n", name,
              ranks ? "identical" : "DIFFER", cols ? "identical" : "DIFFER", rel, err);
  return (ranks && cols && rel < 1e-10) ? 0 : 1;
}

int main() {
  std::fprintf(stderr, "[demo] context\n");
  bfly_b200::Context gpu(0);
  int bad = 0;
  {
    SyntheticButterflySpec spec;
    spec.levels = 6;
    spec.rank = 4;
    spec.seed = 3;
    auto op = synth_butterfly_operator<cplx>(spec);
    ReconstructionConfig cfg;
    cfg.levels = 6;
    cfg.tolerance = 1e-10;
    cfg.seed = 1003;
    bad += compare<cplx>("synthetic complex L=6 r=4", *op, op->butterfly().row_tree, op->butterfly().col_tree, cfg, gpu);
  }
  {
    SyntheticButterflySpec spec;
    spec.levels = 5;
    spec.rank = 8;
    spec.seed = 7;
    auto op = synth_butterfly_operator<double>(spec);
    ReconstructionConfig cfg;
    cfg.levels = 5;
    cfg.tolerance = 1e-10;
    cfg.seed = 1007;
    bad += compare<double>("synthetic real L=5 r=8", *op, op->butterfly().row_tree, op->butterfly().col_tree, cfg, gpu);
  }
  {
    Helmholtz3DConfig hc;
    hc.n = 512;
    Helmholtz3DOperator op(hc);
    auto rt = build_tree(op.targets(), 4);
    auto ct = build_tree(op.sources(), 4);
    ReconstructionConfig cfg;
    cfg.levels = 4;
    cfg.tolerance = 1e-4;
    cfg.seed = 6;
    bad += compare<cplx>("reference Helmholtz3D hemispheres n=512", op, rt, ct, cfg, gpu);
  }
  std::printf(bad ? "ADAPTER PARITY FAILED\n" : "ADAPTER PARITY OK\n");
  return bad;
}
