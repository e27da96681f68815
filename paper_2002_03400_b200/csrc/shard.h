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

// Block indices (tau * 2^(L-l) + nu) rank r produces at a level.
//   side 0: leaves (2^L units = blocks)
//   side 1: W level l, units = row probes tau  -> blocks [tau*2^(L-l), ...) contiguous
//   side 2: R level l, units = column probes nu -> blocks strided by 2^(L-l)
inline std::vector<int64_t> shard_blocks(int L, int l, int side, int world, int r) {
  std::vector<int64_t> out;
  if (side == 0) {
    auto [b, e] = shard_chunk(int64_t(1) << L, world, r);
    for (int64_t i = b; i < e; ++i) out.push_back(i);
  } else if (side == 1) {
    const int64_t nnu = int64_t(1) << (L - l);
    auto [b, e] = shard_chunk(int64_t(1) << l, world, r);
    for (int64_t tau = b; tau < e; ++tau)
      for (int64_t nu = 0; nu < nnu; ++nu) out.push_back(tau * nnu + nu);
  } else {
    const int64_t nnu = int64_t(1) << (L - l), ntau = int64_t(1) << l;
    auto [b, e] = shard_chunk(nnu, world, r);
    for (int64_t nu = b; nu < e; ++nu)
      for (int64_t tau = 0; tau < ntau; ++tau) out.push_back(tau * nnu + nu);
  }
  return out;
}

}  // namespace bfly
