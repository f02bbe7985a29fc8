// Primal-dual interior-point LP solver (Mehrotra predictor-corrector) for
//   minimize c^T x   subject to   a_r^T x >= b_r  (r = 1..m),  x free.
// Newton systems A^T D A dx = rhs are solved with a skyline (envelope)
// Cholesky under a reverse Cuthill-McKee ordering of the sparse rows; rows
// flagged `dense` (the per-stage freeze budgets, which couple every backward
// node of a stage) enter through a Sherman-Morrison-Woodbury update, so the
// envelope stays narrow. Written for the freeze-ratio LP (lp.cpp); no
// counterpart in the reference, whose dense tableau simplex is
// proj/include/pipefreeze/simplex.hpp.
#pragma once

#include <vector>

namespace pipefreeze::ipm {

struct Row {
  std::vector<int> idx;
  std::vector<double> val;
  double rhs{0.0};
  bool dense{false};
};

struct Problem {
  int n{0};
  std::vector<double> c;
  std::vector<Row> rows;
};

struct Result {
  std::vector<double> x;
  std::vector<double> z;  // row duals
  long iterations{0};
  bool converged{false};
  double primal_residual{0.0};
  double dual_residual{0.0};
  double mu{0.0};
};

Result solve(const Problem& p, const std::vector<double>& x0, double tol = 1e-10, int max_iter = 300);

}  // namespace pipefreeze::ipm
