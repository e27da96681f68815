// shard.h -- how a level's work units are split across ranks (host logic
// shared by the factorizer and the C ABI; tested multi-process on CPU).
#pragma once

#include <algorithm>
#include <cstdint>
#include <utility>
#include <vector>

namespace bfly {

// contiguous chunk r of n units: [r*c, (r+1)*c) clipped, c = ceil(n/world)
inline std::pair<int64_t, int64_t> shard_chunk(int64_t n, int world, int r) {
  const int64_t c = (n + world - 1) / world;
  return {std::min(n, r * c), std::min(n, (r + 1) * c)};
}

// Block indices (tau * 2^(L-l) + nu) rank r produces at a level.  Every
// level is split into equal contiguous chunks of its 2^L blocks, so levels
// with fewer probes than ranks still keep every rank busy (a probe's
// partner nodes -- its output rows -- are split across ranks):
//   side 0: leaves (2^L units = blocks)
//   side 1: W level l, tau-major block order: chunk [r*c, (r+1)*c) of the
//           block indices themselves (in place for ncclAllGather)
//   side 2: R level l, nu-major order u = nu * 2^l + tau (a column probe's
//           blocks are strided by 2^(L-l) in the tau-major layout)
inline std::vector<int64_t> shard_blocks(int L, int l, int side, int world, int r) {
  std::vector<int64_t> out;
  const int64_t nb = int64_t(1) << L;
  auto [b, e] = shard_chunk(nb, world, r);
  if (side == 0 || side == 1) {
    for (int64_t i = b; i < e; ++i) out.push_back(i);
  } else {
    const int64_t nnu = int64_t(1) << (L - l), ntau = int64_t(1) << l;
    for (int64_t u = b; u < e; ++u) out.push_back((u % ntau) * nnu + u / ntau);
  }
  return out;
}

// Probe pieces of a unit chunk [u0, u1) of a level whose units are ordered
// probe-major (npart partner nodes per probe): (probe, first, end partner).
struct ProbePiece {
  int64_t probe, p0, p1;
};
inline std::vector<ProbePiece> probe_pieces(int64_t u0, int64_t u1, int64_t npart) {
  std::vector<ProbePiece> out;
  for (int64_t u = u0; u < u1;) {
    const int64_t p = u / npart, a = u - p * npart, b = std::min(npart, a + (u1 - u));
    out.push_back(ProbePiece{p, a, b});
    u += b - a;
  }
  return out;
}

}  // namespace bfly
