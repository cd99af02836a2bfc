// C++ drop-in, checker side and helpers (include/etbfs/{preprocess,validate,
// bench}.hpp): split_degree_aware, oracle_bfs and validate_bfs_tree run on the
// GPU through the C-ABI (csrc/graph_tools.cu); translate_tree, tree_levels,
// select_roots and compute_gteps are the host bookkeeping around them, with the
// reference's semantics and messages (proj/src/validate.cpp:77-175,
// proj/src/bench.cpp:211-242, proj/src/preprocess.cpp:16-60).
#include <cstring>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "etbfs/bench.hpp"
#include "etbfs/preprocess.hpp"
#include "etbfs/validate.hpp"
#include "etbfs_cuda.h"

namespace etbfs {
namespace {

void check(int rc) {
  if (rc == ETB_OK) return;
  const std::string msg = etb_last_error();
  if (rc == ETB_EINVAL) throw std::invalid_argument(msg);
  throw std::runtime_error(msg);
}

struct GraphDel {
  void operator()(etb_graph* g) const { etb_graph_free(g); }
};
using GraphPtr = std::unique_ptr<etb_graph, GraphDel>;

GraphPtr upload(const CsrGraph& g) {
  if (g.row_offsets.size() != g.vertex_count + 1)
    throw std::invalid_argument("etbfs: CsrGraph row_offsets size mismatch");
  etb_graph* h = nullptr;
  check(etb_graph_from_csr(g.vertex_count, g.row_offsets.data(), g.col_indices.data(), &h));
  return GraphPtr(h);
}

uint64_t splitmix(uint64_t& state) {
  uint64_t z = (state += 0x9e3779b97f4a7c15ull);
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}

}  // namespace

DegreeSplitAdjacency split_degree_aware(const CsrGraph& graph, vertex_t neighbor_limit) {
  DegreeSplitAdjacency split;
  split.neighbor_limit = neighbor_limit;
  const uint64_t n = graph.vertex_count;
  split.in_plus.assign(n, kNoVertex);
  split.minus_offsets.assign(n + 1, 0);
  if (n == 0) return split;
  GraphPtr g = upload(graph);
  check(etb_graph_degree_split(g.get(), neighbor_limit, nullptr, split.minus_offsets.data(),
                               nullptr));
  split.minus_cols.resize(split.minus_offsets[n]);
  check(etb_graph_degree_split(g.get(), neighbor_limit, split.in_plus.data(),
                               split.minus_offsets.data(), split.minus_cols.data()));
  return split;
}

std::vector<std::uint64_t> oracle_bfs(const CsrGraph& graph, vertex_t root) {
  if (root >= graph.vertex_count) throw std::invalid_argument("oracle_bfs: root out of range");
  GraphPtr g = upload(graph);
  std::vector<std::uint64_t> level(graph.vertex_count);
  check(etb_graph_levels(g.get(), root, level.data()));
  return level;
}

// Levels read off the tree as it is (validate.cpp:18-67): memoised chain walks;
// vertices on cyclic or dead-ended chains keep kUnreached.
std::vector<std::uint64_t> tree_levels(const BfsTree& tree) {
  const uint64_t n = tree.parent.size();
  std::vector<std::uint64_t> level(n, kUnreached);
  std::vector<uint8_t> state(n, 0);  // 0 open, 1 resolved, 2 bad, 3 on the current path
  if (tree.root < n && tree.parent[tree.root] == tree.root) {
    level[tree.root] = 0;
    state[tree.root] = 1;
  }
  std::vector<vertex_t> path;
  for (vertex_t v = 0; v < n; ++v) {
    if (tree.parent[v] == kNoVertex || state[v] != 0) continue;
    path.clear();
    vertex_t x = v;
    bool good = false;
    uint64_t base = 0;
    for (;;) {
      if (state[x] == 1) {
        good = true;
        base = level[x];
        break;
      }
      if (state[x] == 2 || state[x] == 3) break;
      const vertex_t p = tree.parent[x];
      if (p == kNoVertex || p >= n) break;
      state[x] = 3;
      path.push_back(x);
      x = p;
    }
    for (size_t i = path.size(); i-- > 0;) {
      if (good) {
        level[path[i]] = base + (path.size() - i);
        state[path[i]] = 1;
      } else {
        state[path[i]] = 2;
      }
    }
  }
  return level;
}

ValidationReport validate_bfs_tree(const CsrGraph& graph, const BfsTree& tree) {
  const uint64_t n = graph.vertex_count;
  if (tree.parent.size() != n)
    throw std::invalid_argument("validate_bfs_tree: tree does not match graph vertex count");
  if (tree.root >= n) throw std::invalid_argument("validate_bfs_tree: root out of range");
  GraphPtr g = upload(graph);
  uint64_t counts[8] = {}, where[5 * 25] = {};
  uint32_t first[5] = {};
  check(etb_graph_validate_tree(g.get(), tree.root, tree.parent.data(), counts, where, first));
  ValidationReport rep;
  rep.passed = counts[0] != 0;
  rep.reached_count = counts[6];
  rep.traversed_edge_count = counts[7];
  for (int r = 1; r <= 5; ++r)
    for (uint32_t i = 0; i < first[r - 1]; ++i) {
      uint64_t w = where[(r - 1) * 25 + i];
      std::string msg;
      switch (r) {
        case kRuleRootParent: msg = "root is not its own parent"; break;
        case kRuleChains:
          msg = (w >> 62) & 1 ? "parent chain dead-ends before the root"
                              : "parent chain contains a cycle";
          w &= ~(uint64_t{1} << 62);
          break;
        case kRuleParentEdge:
          msg = tree.parent[w] >= n ? "parent is not a vertex" : "parent is not a neighbor";
          break;
        case kRuleLevelSpan: msg = "edge spans more than one level"; break;
        default:
          msg = tree.parent[w] != kNoVertex ? "vertex outside the root's component has a parent"
                                            : "component vertex missing from the tree";
      }
      rep.failures.push_back({r, w, std::move(msg)});
    }
  return rep;
}

BfsTree translate_tree(const BfsTree& tree, const std::vector<vertex_t>& new2old) {
  const uint64_t n = new2old.size();
  if (tree.parent.size() != n)
    throw std::invalid_argument("translate_tree: permutation does not match tree");
  BfsTree out;
  out.parent.assign(n, kNoVertex);
  for (vertex_t v = 0; v < n; ++v) {
    const vertex_t p = tree.parent[v];
    if (p == kNoVertex) continue;
    if (p >= n) throw std::invalid_argument("translate_tree: parent index out of range");
    out.parent[new2old[v]] = new2old[p];
  }
  if (tree.root >= n) throw std::invalid_argument("translate_tree: root out of range");
  out.root = new2old[tree.root];
  return out;
}

double compute_gteps(std::uint64_t traversed_edges, double elapsed_seconds) {
  if (!(elapsed_seconds > 0.0))
    throw std::invalid_argument("compute_gteps: elapsed time must be positive");
  return static_cast<double>(traversed_edges) / elapsed_seconds / 1e9;
}

std::vector<vertex_t> select_roots(const CsrGraph& graph, std::uint64_t count, std::uint64_t seed) {
  if (count == 0) throw std::invalid_argument("select_roots: count must be >= 1");
  uint64_t eligible = 0;
  for (uint64_t d : graph.degrees) eligible += d > 0;
  if (eligible == 0)
    throw std::runtime_error("select_roots: graph has no vertex with degree >= 1");
  std::vector<vertex_t> roots;
  roots.reserve(count);
  std::vector<uint8_t> taken(graph.vertex_count, 0);
  uint64_t distinct = 0, state = seed;
  while (roots.size() < count) {
    const vertex_t v = splitmix(state) % graph.vertex_count;
    if (graph.degrees[v] == 0) continue;
    if (taken[v] && distinct < eligible) continue;  // repeats only once all are taken
    if (!taken[v]) {
      taken[v] = 1;
      ++distinct;
    }
    roots.push_back(v);
  }
  return roots;
}

}  // namespace etbfs
