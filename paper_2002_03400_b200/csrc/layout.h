// layout.h -- process layouts of the butterfly apply (reference inc/layout.hpp).
//
// A layout assigns every factor block, and with it the coefficient block it
// produces, to one of p = 2^g processes.  Block labels are L-bit strings: the
// column-wise label of (level l, tau, nu) is tau's l bits followed by nu's
// L-l bits reversed, the row-wise label nu's L-l bits followed by tau's l
// bits reversed; the owner is the label's top g bits (layout.hpp:97-111).
// column: every factor column-labelled; row: every factor row-labelled;
// hybrid: U side (R levels, U leaves) column-labelled and V side (W levels,
// V leaves, centre cores) row-labelled (layout.hpp:139-188), so the V chain
// stays on the owner of the input leaves' top bits and the U chain on the
// owner of the output leaves' top bits while p^2 <= 2^L, and the only data
// movement is the handoff at the centre.
#pragma once

#include <cstdint>

namespace bfly {

enum LayoutKind { LAYOUT_COLUMN = 0, LAYOUT_ROW = 1, LAYOUT_HYBRID = 2 };

// g = floor(log2 p) (layout.hpp:35-39)
inline int layout_log_p(int64_t p) {
  int g = 0;
  while ((int64_t(1) << (g + 1)) <= p) ++g;
  return g;
}

// LayoutSpec::validate (layout.hpp:41-48): false on an invalid spec
inline bool layout_valid(int kind, int levels, int64_t rank, int64_t p) {
  return kind >= 0 && kind <= 2 && levels >= 1 && rank >= 1 && p >= 1 && (p & (p - 1)) == 0 &&
         p <= (int64_t(1) << levels);
}

inline int64_t layout_bit_reverse(int64_t v, int bits) {
  int64_t out = 0;
  for (int i = 0; i < bits; ++i) out |= ((v >> i) & 1) << (bits - 1 - i);
  return out;
}

// side 0: V side (V leaves, W levels, centre cores); side 1: U side (R levels,
// U leaves at level L)
inline int layout_owner(int kind, int L, int g, int side, int level, int64_t tau, int64_t nu) {
  const bool column = side == 1 ? kind != LAYOUT_ROW : kind == LAYOUT_COLUMN;
  const int64_t label = column ? (tau << (L - level)) | layout_bit_reverse(nu, L - level)
                               : (nu << level) | layout_bit_reverse(tau, level);
  return (int)(label >> (L - g));
}

// Per-process communication tallies of one apply, in scalars per input
// column (CommCostReport, layout.hpp:52-66).
struct CommReport {
  double exchange_volume = 0.0;
  int64_t exchange_msgs = 0;
  double alltoall_volume = 0.0;
  int64_t alltoall_msgs = 0;
};

// Closed-form model for constant rank r and n = r 2^L (layout.hpp:70-88):
// column/row exchange at each of the g owner bits, hybrid only at the
// max(0, 2g - L) bits neither half covers; one all-to-all of the per-process
// state.
inline CommReport comm_cost(int kind, int L, int64_t rank, int64_t p) {
  CommReport rep;
  const double per_proc = (double)rank * (double)(int64_t(1) << L) / (double)p;
  const int g = layout_log_p(p);
  const int64_t exch = kind == LAYOUT_HYBRID ? (2 * g - L > 0 ? 2 * g - L : 0) : g;
  rep.exchange_msgs = exch;
  rep.exchange_volume = per_proc * (double)exch;
  rep.alltoall_volume = per_proc;
  const int64_t a = (int64_t(1) << L) / p, b = p - 1;
  rep.alltoall_msgs = a < b ? a : b;
  return rep;
}

}  // namespace bfly
