// Drop-in: traversal policy, stats and whole-graph kernels (reference:
// proj/include/etbfs/bfs.hpp:19-123). The whole-graph kernels run the same
// persistent sm_100a kernel as et_bfs over an all-core layout.
#pragma once

#include <cstdint>
#include <string>

#include "etbfs/preprocess.hpp"
#include "etbfs/types.hpp"

namespace etbfs {

struct HybridPolicy {
  double alpha = 14.0;
  double beta = 24.0;
};

struct KernelStats {
  std::uint64_t levels = 0;
  std::uint64_t bottom_up_levels = 0;
  std::uint64_t probes = 0;          // not counted on the GPU (always 0)
  std::uint64_t skipped_blocks = 0;  // not counted on the GPU (always 0)
  std::string direction_trace;
};

BfsTree bfs_top_down(const CsrGraph& graph, vertex_t root, KernelStats* stats = nullptr);

BfsTree bfs_hybrid(const CsrGraph& graph, vertex_t root, const HybridPolicy& policy = {},
                   KernelStats* stats = nullptr);

// Hybrid driver with the degree-aware bottom-up phase / the standalone
// block-search sweep (bfs.hpp:57-65). The split must cover the whole graph.
BfsTree bfs_degree_aware(const CsrGraph& graph, const DegreeSplitAdjacency& split, vertex_t root,
                         const HybridPolicy& policy = {}, KernelStats* stats = nullptr);
BfsTree bfs_block_search(const CsrGraph& graph, const DegreeSplitAdjacency& split, vertex_t root,
                         KernelStats* stats = nullptr);

std::uint64_t restricted_edge_count(const CsrGraph& graph, vertex_t limit);

}  // namespace etbfs
