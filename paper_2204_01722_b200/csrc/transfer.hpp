// p-level transfer operators (Prolongation, multigrid.hpp:25-74).
#pragma once

#include "operator.hpp"

namespace hxg {

class Transfer {
 public:
  Transfer(const int cells[3], int fine_order, int coarse_order);
  // Prolongation::apply (multigrid.hpp:30-50).
  void prolong(const double* xc, double* xf, cudaStream_t s);
  // Prolongation::apply_transpose (multigrid.hpp:52-73).
  void restrict_to(const double* xf, double* xc, cudaStream_t s);

 private:
  int pf_, pc_;
  BoxDev fine_, coarse_;
  DevBuf<double> ctof_;
  std::vector<double> ctof_h_;  // host copy (passed by value to the kernels)
  DevBuf<double> evf_, evc_;
};

}  // namespace hxg
