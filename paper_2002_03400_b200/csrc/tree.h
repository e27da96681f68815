// tree.h -- host partition tree (setup, not hot path).
// PartitionTree (reference tree.hpp:66-216): complete bisection tree, node
// (l, j) owns a contiguous range of the permuted ordering.
#pragma once

#include <cstdint>
#include <vector>

namespace bfly {

struct Tree {
  int levels = 0;
  int64_t n = 0;
  std::vector<int64_t> perm;                 // tree slot -> original index
  std::vector<std::vector<int64_t>> ranges;  // ranges[l] has 2^l + 1 entries
  bool identity = true;

  int64_t begin(int l, int64_t j) const { return ranges[l][j]; }
  int64_t end(int l, int64_t j) const { return ranges[l][j + 1]; }
  int64_t size(int l, int64_t j) const { return ranges[l][j + 1] - ranges[l][j]; }
  int64_t max_size(int l) const;
  void finalize();  // recompute `identity`

  // tree.hpp:75-101 (+ split :178-201)
  static Tree build(int dim, int64_t n, const double* coords, int levels);
  static Tree from_table(int64_t n, int levels, const int64_t* perm, const int64_t* flat_ranges);
  void table(int64_t* perm_out, int64_t* ranges_out) const;
};

int depth_for(int64_t n, int64_t leaf_cap);

}  // namespace bfly
