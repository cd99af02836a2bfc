// Drop-in: CSR construction (reference: proj/include/etbfs/build.hpp:11-19).
// build_csr runs on the GPU (etb_graph_from_edges): one 64-bit key radix sort
// plus unique instead of per-row sorts; identical, canonical output.
#pragma once

#include <cstdint>
#include <vector>

#include "etbfs/types.hpp"

namespace etbfs {

struct BuildStats {
  std::uint64_t dropped_self_loops = 0;
  std::uint64_t dropped_duplicates = 0;
};

CsrGraph build_csr(const EdgeList& edges, BuildStats* stats = nullptr);

// Inverse of a new2old permutation (reference build.hpp:36); throws
// std::invalid_argument when the input is not a permutation.
std::vector<vertex_t> invert_permutation(const std::vector<vertex_t>& new2old);

}  // namespace etbfs
