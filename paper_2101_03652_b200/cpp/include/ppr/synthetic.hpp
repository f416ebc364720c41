// Drop-in for the reference's ppr/synthetic.hpp: the seeded random digraph of
// its tests (synthetic.cpp). Degrees then targets are drawn from one Rng
// stream on the host (bit-identical graph); the CSR goes to the GPU.
#pragma once

#include "ppr/graph.hpp"
#include "ppr/rng.hpp"
#include "ppr/types.hpp"

namespace ppr {

Graph random_graph(NodeId n, std::uint32_t min_out, std::uint32_t max_out, std::uint64_t seed);

}  // namespace ppr
