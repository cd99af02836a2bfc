// Drop-in: the composite edge-tree BFS (reference: proj/include/etbfs/et_bfs.hpp:10-56).
#pragma once

#include "etbfs/bfs.hpp"
#include "etbfs/bitmap.hpp"
#include "etbfs/preprocess.hpp"
#include "etbfs/types.hpp"

namespace etbfs {

enum class CoreKernel {
  kTopDown,
  kHybrid,
  kDegreeAware,        // hybrid; device rows are already degree-ordered
  kBlockSearch,        // bottom-up sweeps to the fixpoint, no top-down level
  kHybridBlockSearch,  // hybrid with the bottom-up sweep
};

enum class TreeReplay {
  kTeet,
  kTeolv,
};

// Tree replay over caller-held state (et_bfs.hpp:30-37), on the GPU: for every
// entry whose guard is visited (teet: the tree's core edge vertex; teolv: the
// entry's src, height-0 layouts) parent[dst] = src unless already set.
void teet(const EdgeTreeList& etl, const Bitmap& visited, std::vector<vertex_t>& parent);
void teolv(const EdgeTreeList& etl, const Bitmap& visited, std::vector<vertex_t>& parent);

// The start-side walk (et_bfs.hpp:39-43): BFS inside the edge tree containing
// start, parents oriented away from it; returns the tree's core edge vertex
// (its parent set to the adjacent tree vertex) or kNoVertex for a pure tree.
// O(tree size) host work here as in the product path's start patch.
vertex_t traverse_return_core_edge(const ClassifiedGraph& cg, vertex_t start, BfsTree& tree);

// The split-based kernels require a split matching the core block (as the
// reference checks, et_bfs.cpp:69-78) but the device does not read it: its
// relaid rows already list neighbours by descending degree.

// et_bfs over a relaid graph. The first call on a given (cg, etl) pair uploads
// it and builds the device layout; later calls on the same objects reuse it
// (keyed by address and size). For repeated traversals prefer the device
// session calls of include/etbfs_cuda.h (etb_layout_build + etb_bfs_device).
BfsTree et_bfs(const ClassifiedGraph& cg, const EdgeTreeList& etl, vertex_t start,
               CoreKernel kernel = CoreKernel::kHybrid, TreeReplay replay = TreeReplay::kTeet,
               const DegreeSplitAdjacency* split = nullptr, const HybridPolicy& policy = {},
               KernelStats* stats = nullptr);

}  // namespace etbfs
