// Drop-in for /root/reference/proj/core/include/ppr/walk_index.hpp. The
// index is built on the GPU with Philox walks (rng-id 2).
#pragma once

#include <memory>
#include <span>
#include <string>
#include <vector>

#include "ppr/graph.hpp"
#include "ppr/rng.hpp"
#include "ppr/types.hpp"

struct pprg_index;

namespace ppr {

inline constexpr std::uint8_t kRngIdPhilox4x32_10 = 2;

// One alpha-random walk on the host from a caller's Rng stream
// (walk_index.hpp:16): stop with probability alpha, else move to a uniform
// effective out-neighbour (dead ends jump to source). The GPU engines draw
// their walks from Philox streams instead.
NodeId random_walk(const Graph& g, NodeId start, NodeId source, double alpha, Rng& rng);

class WalkIndex {
 public:
  double alpha() const { return alpha_; }
  std::uint64_t seed() const { return seed_; }
  std::uint8_t rng_id() const { return kRngIdPhilox4x32_10; }
  NodeId node_count() const { return static_cast<NodeId>(offsets_.size() - 1); }
  EdgeId endpoint_count() const { return endpoints_.size(); }
  std::span<const NodeId> endpoints_of(NodeId v) const {
    return {endpoints_.data() + offsets_[v], static_cast<std::size_t>(offsets_[v + 1] - offsets_[v])};
  }
  void check_compatible(const Graph& g) const;
  // Device copy bound to g (uploaded on first use with a graph when the index
  // came from a file without one).
  pprg_index* device_handle(const Graph& g) const;
  pprg_index* device_handle() const { return dev_.get(); }

 private:
  friend WalkIndex build_index(const Graph&, double, std::uint64_t);
  friend WalkIndex load_index(const std::string&, const Graph&);
  friend WalkIndex load_index(const std::string&);
  friend void save_index(const WalkIndex&, const std::string&);
  double alpha_ = 0;
  std::uint64_t seed_ = 0;
  std::vector<std::uint64_t> offsets_;
  std::vector<NodeId> endpoints_;
  mutable std::shared_ptr<pprg_index> dev_;
  mutable const void* dev_graph_ = nullptr;
};

WalkIndex build_index(const Graph& g, double alpha, std::uint64_t seed);
void save_index(const WalkIndex& index, const std::string& path);
// load_index(path) (walk_index.cpp:83-104) keeps the index on the host until
// it first serves a graph; the two-argument form binds it immediately.
WalkIndex load_index(const std::string& path);
WalkIndex load_index(const std::string& path, const Graph& g);

}  // namespace ppr
