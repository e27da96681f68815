// verify.h -- level-wise residual sums against a dense operator (verify.cu).
#pragma once

#include <vector>

#include "butterfly.h"
#include "operators.h"

namespace bfly {

struct Residuals {
  std::vector<double> u;  // l = L .. l_m   (u_side_residual, reconstruct.hpp:443-460)
  std::vector<double> v;  // l = 0 .. l_m   (v_side_residual, :462-480)
  double center = 0;      // center_residual (:482-502)
  double knorm2 = 0;      // ||K||_F^2
};

template <typename R>
Residuals compute_residuals(Ctx* c, DevOp<R>* op, const DevButterfly<R>& bf);

}  // namespace bfly
