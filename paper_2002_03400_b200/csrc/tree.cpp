// tree.cpp -- host partition tree construction (reference tree.hpp:75-201).
#include "tree.h"

#include <algorithm>
#include <cmath>
#include <limits>
#include <numeric>

#include "common.cuh"

namespace bfly {

int64_t Tree::max_size(int l) const {
  int64_t m = 0;
  for (size_t j = 0; j + 1 < ranges[l].size(); ++j) m = std::max(m, ranges[l][j + 1] - ranges[l][j]);
  return m;
}

void Tree::finalize() {
  identity = true;
  for (int64_t i = 0; i < n && identity; ++i) identity = perm[i] == i;
}

Tree Tree::build(int dim, int64_t n, const double* coords, int levels) {
  if (dim < 1 || dim > 3) fail(PRECONDITION, "PointSet: dim must be 1..3");
  if (n < 1) fail(PRECONDITION, "PointSet: at least one point required");
  for (int64_t i = 0; i < n; ++i)
    for (int a = 0; a < dim; ++a)
      if (!std::isfinite(coords[i * 3 + a])) fail(PRECONDITION, "PointSet: non-finite coordinate");
  if (levels < 0 || levels > 62 || (int64_t(1) << levels) > n)
    fail(PRECONDITION, "PartitionTree: 2^L must not exceed the point count");
  Tree t;
  t.levels = levels;
  t.n = n;
  t.perm.resize(n);
  std::iota(t.perm.begin(), t.perm.end(), int64_t(0));
  t.ranges.resize(levels + 1);
  t.ranges[0] = {0, n};
  for (int l = 0; l < levels; ++l) {
    const auto& cur = t.ranges[l];
    std::vector<int64_t> next;
    next.reserve(cur.size() * 2 - 1);
    for (size_t j = 0; j + 1 < cur.size(); ++j) {
      int64_t b = cur[j], e = cur[j + 1];
      double lo[3] = {0, 0, 0}, hi[3] = {0, 0, 0};
      for (int a = 0; a < dim; ++a) {
        lo[a] = std::numeric_limits<double>::infinity();
        hi[a] = -std::numeric_limits<double>::infinity();
      }
      for (int64_t i = b; i < e; ++i)
        for (int a = 0; a < dim; ++a) {
          double c = coords[t.perm[i] * 3 + a];
          lo[a] = std::min(lo[a], c);
          hi[a] = std::max(hi[a], c);
        }
      int axis = 0;
      for (int a = 1; a < dim; ++a)
        if (hi[a] - lo[a] > hi[axis] - lo[axis]) axis = a;
      std::stable_sort(t.perm.begin() + b, t.perm.begin() + e,
                       [&](int64_t x, int64_t y) { return coords[x * 3 + axis] < coords[y * 3 + axis]; });
      next.push_back(b);
      next.push_back(b + (e - b + 1) / 2);
    }
    next.push_back(n);
    t.ranges[l + 1] = std::move(next);
  }
  t.finalize();
  return t;
}

Tree Tree::from_table(int64_t n, int levels, const int64_t* perm, const int64_t* flat) {
  if (levels < 0 || levels > 40 || n < 1) fail(PRECONDITION, "PartitionTree: bad table");
  Tree t;
  t.levels = levels;
  t.n = n;
  t.perm.assign(perm, perm + n);
  t.ranges.resize(levels + 1);
  int64_t off = 0;
  for (int l = 0; l <= levels; ++l) {
    int64_t cnt = (int64_t(1) << l) + 1;
    t.ranges[l].assign(flat + off, flat + off + cnt);
    off += cnt;
    if (t.ranges[l].front() != 0 || t.ranges[l].back() != n) fail(PRECONDITION, "PartitionTree: ranges must tile [0, n)");
  }
  t.finalize();
  return t;
}

void Tree::table(int64_t* perm_out, int64_t* ranges_out) const {
  if (perm_out) std::copy(perm.begin(), perm.end(), perm_out);
  if (ranges_out) {
    int64_t off = 0;
    for (const auto& r : ranges) {
      std::copy(r.begin(), r.end(), ranges_out + off);
      off += (int64_t)r.size();
    }
  }
}

int depth_for(int64_t n, int64_t leaf_cap) {
  if (leaf_cap < 1) fail(PRECONDITION, "depth_for: leaf_cap >= 1 required");
  int levels = 0;
  while ((n >> (levels + 1)) >= leaf_cap) ++levels;
  return levels;
}

}  // namespace bfly
