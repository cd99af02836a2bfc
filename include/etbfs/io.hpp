// Drop-in: graph and parent-tree files (reference: proj/include/etbfs/io.hpp:9-45,
// proj/src/io.cpp:47-181). Same formats, byte for byte, and the same error
// types and messages, so files move freely between the CPU reference tools and
// GPU runs.
//
//   ETG1 (binary graph): "ETG1", u64 vertex_count, u64 edge_count, then
//   edge_count (u64 src, u64 dst) pairs, all little endian.
//   Text graph: "src dst" per line, '#' comments; writing emits "# vertices N".
//   ETT1 (parent tree): "ETT1", u64 vertex_count, u64 root, vertex_count u64
//   parent slots (all ones = unreached).
//
// Read errors throw std::runtime_error naming the path and the byte offset or
// line; an unknown format name throws std::invalid_argument.
#pragma once

#include <string>

#include "etbfs/types.hpp"

namespace etbfs {

enum class GraphFormat { kBinary, kText };

void write_graph(const std::string& path, const EdgeList& edges, GraphFormat format);
EdgeList read_graph(const std::string& path, GraphFormat format);

void write_tree(const std::string& path, const BfsTree& tree);
BfsTree read_tree(const std::string& path);

GraphFormat parse_graph_format(const std::string& name);

}  // namespace etbfs
