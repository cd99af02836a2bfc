// Drop-in: relayout + edge-tree extraction (reference:
// proj/include/etbfs/relayout.hpp:40-52). Both run on the GPU (etb_layout_*);
// the placement order is bit-identical to the reference's queue walk.
#pragma once

#include <cstdint>

#include "etbfs/types.hpp"

namespace etbfs {

// Throws std::invalid_argument if types.size() != graph.vertex_count.
ClassifiedGraph relayout_csr(const CsrGraph& graph, const std::vector<VertexType>& types,
                             std::int64_t mh = -1);

// Throws std::runtime_error with the reference's messages when the typed trees
// are not trees hanging from at most one core vertex.
EdgeTreeList extract_edge_tree_list(const ClassifiedGraph& cg);

}  // namespace etbfs
