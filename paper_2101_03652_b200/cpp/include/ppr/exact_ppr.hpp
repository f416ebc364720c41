// Drop-in for the reference's ppr/exact_ppr.hpp. The reference solves the
// n x n system densely; here the answer is the engine's power-iteration solve
// to r_sum <= 1e-17 on the GPU (pprg_ground_truth), which meets the same
// guards and checks: n <= kDenseSolveMaxNodes, non-negative, unit l1 norm
// (1e-10) and a residual of the defining equation below 1e-10.
#pragma once

#include <vector>

#include "ppr/graph.hpp"
#include "ppr/types.hpp"

namespace ppr {

struct DensePPR {
  std::vector<double> pi;
};

inline constexpr NodeId kDenseSolveMaxNodes = 2000;

DensePPR exact_ppr(const Graph& g, NodeId s, double alpha);

}  // namespace ppr
