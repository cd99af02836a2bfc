// Drop-in: the degree split used by the degree-aware / block-search bottom-up
// kernels (reference: proj/include/etbfs/preprocess.hpp:12-69). Same layout;
// split_degree_aware runs on the GPU (a stable key sort of every row by
// descending neighbour degree). The ET-BFS kernels on the device do not read it
// (relaid rows already list neighbours by descending degree); callers still
// build it to select those kernels, exactly as with the reference.
#pragma once

#include <cstdint>
#include <span>
#include <vector>

#include "etbfs/types.hpp"

namespace etbfs {

struct DegreeSplitAdjacency {
  std::vector<vertex_t> in_plus;             // kNoVertex where no neighbour qualifies
  std::vector<std::uint64_t> minus_offsets;  // vertex_count + 1 entries
  std::vector<vertex_t> minus_cols;
  vertex_t neighbor_limit = kNoVertex;

  std::span<const vertex_t> in_minus(vertex_t v) const {
    return {minus_cols.data() + minus_offsets[v], minus_cols.data() + minus_offsets[v + 1]};
  }
};

// Neighbours >= neighbor_limit are dropped from both parts (kNoVertex keeps all).
DegreeSplitAdjacency split_degree_aware(const CsrGraph& graph, vertex_t neighbor_limit = kNoVertex);

}  // namespace etbfs
