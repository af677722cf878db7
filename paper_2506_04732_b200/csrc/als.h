// Rank-adaptive alternating solver for A x = b in TT format
// (reference: pkg/src/ttss/tt_solver.py).
#pragma once

#include "common.h"

namespace t2s2 {

struct SolverConfig {  // tt_solver.py:39-59
  int max_sweeps = 40;
  double residual_tol = 1e-8;
  double rounding_tol = 1e-10;
  int enrichment_rank = 2;
  int max_rank = 64;
  int local_solver = 0;  // 0 auto, 1 direct, 2 iterative
  int local_direct_size = 2000;
  double inner_tol_factor = 0.02;
  int stagnation_window = 5;
  double stagnation_drop = 0.01;
};

struct SolveReport {  // tt_solver.py:62-76
  std::vector<double> residuals;
  std::vector<int> ranks;
  std::vector<double> compression;
  double wall_time = 0.0;
  bool converged = false;
  bool stagnated = false;
  // per core visit: 0 kept old core, 1 Galerkin, 2 least squares
  std::vector<int> choices;
};

// Solve A x = rhs starting from x0 (required: the host layer builds the
// reference's default guess, tt_solver.py:425).  Returns the best iterate.
Train als_solve(const Train& A, const Train& rhs, const Train& x0, const SolverConfig& cfg,
                SolveReport& rep);

// ||A x - rhs|| / ||rhs|| with the difference rounded at 0.01*tol
// (tt_solver.py:80-92).
double tt_residual(const Train& A, const Train& x, const Train& rhs, double tol);

}  // namespace t2s2
