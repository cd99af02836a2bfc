// Drop-in: traversal policy, stats and whole-graph kernels (reference:
// proj/include/etbfs/bfs.hpp:19-123). The whole-graph kernels run the same
// persistent sm_100a kernel as et_bfs over an all-core layout.
#pragma once

#include <cstdint>
#include <string>
#include <utility>
#include <vector>

#include "etbfs/bitmap.hpp"
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
  std::uint64_t probes = 0;          // step layer: bottom-up probes (whole-graph kernels: 0)
  std::uint64_t skipped_blocks = 0;  // step layer: fully visited blocks skipped
  std::string direction_trace;
};

BfsTree bfs_top_down(const CsrGraph& graph, vertex_t root, KernelStats* stats = nullptr);

BfsTree bfs_hybrid(const CsrGraph& graph, vertex_t root, const HybridPolicy& policy = {},
                   KernelStats* stats = nullptr);

enum class BottomUpKind {
  kClassic,      // per-vertex neighbour scan probing the current frontier
  kDegreeAware,  // highest-degree probe pass, then the descending remainder
  kBlockSearch,  // 64-vertex block sweep with the merged degree-aware probe
};

// Lowest set bit of a non-zero not-yet-visited mask: its position and the mask
// without it (bfs.hpp:44).
std::pair<std::uint32_t, std::uint64_t> block_search_unvisited(std::uint64_t not_visited);

// Step and driver layer (bfs.hpp:66-120), run on the GPU over the caller's
// state: frontier members below `limit`, neighbours at or above it skipped;
// steps update visited / next and parents and never touch current.
struct StepResult {
  std::uint64_t claimed = 0;  // vertices newly visited this step
  std::uint64_t scout = 0;    // degree sum of the claimed vertices (top-down only)
};

StepResult top_down_step(const CsrGraph& graph, FrontierState& state,
                         std::vector<vertex_t>& parent, vertex_t limit,
                         KernelStats* stats = nullptr);
StepResult bottom_up_step(const CsrGraph& graph, FrontierState& state,
                          std::vector<vertex_t>& parent, vertex_t limit,
                          KernelStats* stats = nullptr);
StepResult degree_aware_step(const CsrGraph& graph, const DegreeSplitAdjacency& split,
                             FrontierState& state, std::vector<vertex_t>& parent, vertex_t limit,
                             KernelStats* stats = nullptr);
StepResult block_search_step(const CsrGraph& graph, const DegreeSplitAdjacency& split,
                             FrontierState& state, std::vector<vertex_t>& parent, vertex_t limit,
                             KernelStats* stats = nullptr);
void run_top_down(const CsrGraph& graph, FrontierState& state, std::vector<vertex_t>& parent,
                  vertex_t limit, KernelStats* stats = nullptr);
void run_hybrid(const CsrGraph& graph, const DegreeSplitAdjacency* split, BottomUpKind kind,
                FrontierState& state, std::vector<vertex_t>& parent, vertex_t limit,
                const HybridPolicy& policy, KernelStats* stats = nullptr);
void run_block_search(const CsrGraph& graph, const DegreeSplitAdjacency& split,
                      FrontierState& state, std::vector<vertex_t>& parent, vertex_t limit,
                      KernelStats* stats = nullptr);

// Hybrid driver with the degree-aware bottom-up phase / the standalone
// block-search sweep (bfs.hpp:57-65). The split must cover the whole graph.
BfsTree bfs_degree_aware(const CsrGraph& graph, const DegreeSplitAdjacency& split, vertex_t root,
                         const HybridPolicy& policy = {}, KernelStats* stats = nullptr);
BfsTree bfs_block_search(const CsrGraph& graph, const DegreeSplitAdjacency& split, vertex_t root,
                         KernelStats* stats = nullptr);

std::uint64_t restricted_edge_count(const CsrGraph& graph, vertex_t limit);

}  // namespace etbfs
