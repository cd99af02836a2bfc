// Drop-in: the composite edge-tree BFS (reference: proj/include/etbfs/et_bfs.hpp:10-56).
#pragma once

#include "etbfs/bfs.hpp"
#include "etbfs/types.hpp"

namespace etbfs {

enum class CoreKernel {
  kTopDown,
  kHybrid,
  kDegreeAware,        // needs a degree split: not built on the GPU yet
  kBlockSearch,        // idem
  kHybridBlockSearch,  // idem
};

enum class TreeReplay {
  kTeet,
  kTeolv,
};

struct DegreeSplitAdjacency;  // reference preprocess.hpp:26; accepted, must be null

// et_bfs over a relaid graph. The first call on a given (cg, etl) pair uploads
// it and builds the device layout; later calls on the same objects reuse it
// (keyed by address and size). For repeated traversals prefer the device
// session API in etbfs/gpu.hpp.
BfsTree et_bfs(const ClassifiedGraph& cg, const EdgeTreeList& etl, vertex_t start,
               CoreKernel kernel = CoreKernel::kHybrid, TreeReplay replay = TreeReplay::kTeet,
               const DegreeSplitAdjacency* split = nullptr, const HybridPolicy& policy = {},
               KernelStats* stats = nullptr);

}  // namespace etbfs
