// C++ drop-in: the step and driver layer (include/etbfs/bfs.hpp, reference
// proj/include/etbfs/bfs.hpp:66-120) over etb_steps_run (csrc/steps.cu). The
// caller's FrontierState words and parent vector go to the device and back
// around each call; a driver keeps them resident for all of its levels. The
// device graph is cached for the last CsrGraph seen, keyed by its content
// (rows and columns), so a graph rebuilt at the same addresses or edited in
// place is uploaded again.
#include <bit>
#include <memory>
#include <mutex>
#include <stdexcept>
#include <string>
#include <vector>

#include "etbfs/bfs.hpp"
#include "etbfs_cuda.h"
#include "etbfs_hash.hpp"

namespace etbfs {
namespace {

void check(int rc) {
  if (rc == ETB_OK) return;
  const std::string msg = etb_last_error();
  if (rc == ETB_EINVAL) throw std::invalid_argument(msg);
  throw std::runtime_error(msg);
}

struct Cached {
  uint64_t key = 0;
  uint64_t n = 0, nnz = 0;
  etb_graph* g = nullptr;
  ~Cached() {
    if (g) etb_graph_free(g);
  }
};
std::mutex g_mu;
Cached g_cache;

etb_graph* device_graph(const CsrGraph& graph) {
  if (graph.row_offsets.size() != graph.vertex_count + 1)
    throw std::invalid_argument("etbfs: CsrGraph row_offsets size mismatch");
  const uint64_t key = detail::hash_vec(graph.col_indices,
                                       detail::hash_vec(graph.row_offsets, graph.vertex_count));
  if (g_cache.g && g_cache.key == key && g_cache.n == graph.vertex_count &&
      g_cache.nnz == graph.col_indices.size())
    return g_cache.g;
  etb_graph* h = nullptr;
  check(etb_graph_from_csr(graph.vertex_count, graph.row_offsets.data(),
                           graph.col_indices.data(), &h));
  if (g_cache.g) etb_graph_free(g_cache.g);
  g_cache = {};
  g_cache.key = key;
  g_cache.n = graph.vertex_count;
  g_cache.nnz = graph.col_indices.size();
  g_cache.g = h;
  return h;
}

StepResult run_op(const CsrGraph& graph, int op, const DegreeSplitAdjacency* split,
                  FrontierState& state, std::vector<vertex_t>& parent, vertex_t limit,
                  const HybridPolicy& policy, KernelStats* stats) {
  const uint64_t n = graph.vertex_count;
  if (parent.size() != n) throw std::invalid_argument("bfs: parent size does not match graph");
  if (state.visited.bit_count() != n || state.current.bit_count() != n ||
      state.next.bit_count() != n)
    throw std::invalid_argument("bfs: frontier state does not match graph");
  std::lock_guard<std::mutex> lk(g_mu);
  etb_graph* g = device_graph(graph);
  uint64_t out[6] = {};
  std::string trace(4096, '\0');
  check(etb_steps_run(g, op, limit, state.visited.data(), state.current.data(),
                      state.next.data(), parent.data(), split ? split->in_plus.data() : nullptr,
                      split ? split->minus_offsets.data() : nullptr,
                      split ? split->minus_cols.data() : nullptr, policy.alpha, policy.beta,
                      out, op >= 4 ? trace.data() : nullptr, op >= 4 ? trace.size() : 0));
  if (stats) {
    stats->probes += out[2];
    stats->skipped_blocks += out[3];
    stats->levels += out[4];
    stats->bottom_up_levels += out[5];
    if (op >= 4) stats->direction_trace += trace.c_str();
  }
  return {out[0], out[1]};
}

void check_split(const CsrGraph& graph, const DegreeSplitAdjacency& split) {
  if (split.in_plus.size() != graph.vertex_count ||
      split.minus_offsets.size() != graph.vertex_count + 1)
    throw std::invalid_argument("bfs: split size does not match graph");
}

}  // namespace

std::pair<std::uint32_t, std::uint64_t> block_search_unvisited(std::uint64_t not_visited) {
  const std::uint64_t low = not_visited & (~not_visited + 1);
  return {static_cast<std::uint32_t>(std::countr_zero(low)), not_visited & ~low};
}

StepResult top_down_step(const CsrGraph& graph, FrontierState& state,
                         std::vector<vertex_t>& parent, vertex_t limit, KernelStats* stats) {
  return run_op(graph, 0, nullptr, state, parent, limit, {}, stats);
}

StepResult bottom_up_step(const CsrGraph& graph, FrontierState& state,
                          std::vector<vertex_t>& parent, vertex_t limit, KernelStats* stats) {
  return run_op(graph, 1, nullptr, state, parent, limit, {}, stats);
}

StepResult degree_aware_step(const CsrGraph& graph, const DegreeSplitAdjacency& split,
                             FrontierState& state, std::vector<vertex_t>& parent, vertex_t limit,
                             KernelStats* stats) {
  check_split(graph, split);
  return run_op(graph, 2, &split, state, parent, limit, {}, stats);
}

StepResult block_search_step(const CsrGraph& graph, const DegreeSplitAdjacency& split,
                             FrontierState& state, std::vector<vertex_t>& parent, vertex_t limit,
                             KernelStats* stats) {
  check_split(graph, split);
  return run_op(graph, 3, &split, state, parent, limit, {}, stats);
}

void run_top_down(const CsrGraph& graph, FrontierState& state, std::vector<vertex_t>& parent,
                  vertex_t limit, KernelStats* stats) {
  run_op(graph, 4, nullptr, state, parent, limit, {}, stats);
}

void run_hybrid(const CsrGraph& graph, const DegreeSplitAdjacency* split, BottomUpKind kind,
                FrontierState& state, std::vector<vertex_t>& parent, vertex_t limit,
                const HybridPolicy& policy, KernelStats* stats) {
  if (kind != BottomUpKind::kClassic && split == nullptr)
    throw std::invalid_argument("run_hybrid: bottom-up kind needs a degree split");
  if (!(policy.alpha > 0.0) || !(policy.beta > 0.0))
    throw std::invalid_argument("run_hybrid: alpha and beta must be positive");
  if (split) check_split(graph, *split);
  const int op = kind == BottomUpKind::kClassic ? 5 : (kind == BottomUpKind::kDegreeAware ? 6 : 7);
  run_op(graph, op, kind == BottomUpKind::kClassic ? nullptr : split, state, parent, limit,
         policy, stats);
}

void run_block_search(const CsrGraph& graph, const DegreeSplitAdjacency& split,
                      FrontierState& state, std::vector<vertex_t>& parent, vertex_t limit,
                      KernelStats* stats) {
  check_split(graph, split);
  run_op(graph, 8, &split, state, parent, limit, {}, stats);
}

}  // namespace etbfs

// ---- tree replay and the start-side walk (et_bfs.hpp:30-43) -------------------
#include "etbfs/et_bfs.hpp"

namespace etbfs {
namespace {

void replay(int leaves_only, const EdgeTreeList& etl, const Bitmap& visited,
            std::vector<vertex_t>& parent) {
  const size_t m = etl.entries.size();
  std::vector<uint64_t> src(m), dst(m), ce(m);
  for (size_t i = 0; i < m; ++i) {
    src[i] = etl.entries[i].src;
    dst[i] = etl.entries[i].dst;
    ce[i] = etl.entries[i].core_edge;
  }
  std::vector<uint64_t> words(visited.word_count());
  for (uint64_t w = 0; w < words.size(); ++w) words[w] = visited.word(w);
  check(etb_tree_replay(leaves_only, src.data(), dst.data(), ce.data(), m, words.data(),
                        words.size(), parent.data(), parent.size()));
}

}  // namespace

void teet(const EdgeTreeList& etl, const Bitmap& visited, std::vector<vertex_t>& parent) {
  replay(0, etl, visited, parent);
}

void teolv(const EdgeTreeList& etl, const Bitmap& visited, std::vector<vertex_t>& parent) {
  replay(1, etl, visited, parent);
}

vertex_t traverse_return_core_edge(const ClassifiedGraph& cg, vertex_t start, BfsTree& tree) {
  if (start >= cg.graph.vertex_count ||
      (cg.vertex_type[start] != VertexType::kTreeInternal &&
       cg.vertex_type[start] != VertexType::kTreeLeaf))
    throw std::invalid_argument("traverse_return_core_edge: start is not a tree vertex");
  const uint64_t core = cg.core_vertex_count;
  tree.parent[start] = start;
  vertex_t core_edge = kNoVertex;
  std::vector<vertex_t> frontier{start};
  for (size_t head = 0; head < frontier.size(); ++head) {
    const vertex_t u = frontier[head];
    for (vertex_t w : cg.graph.neighbors(u)) {
      if (w < core) {  // the tree's single attachment to the core
        core_edge = w;
        tree.parent[w] = u;
      } else if (tree.parent[w] == kNoVertex) {
        tree.parent[w] = u;
        frontier.push_back(w);
      }
    }
  }
  return core_edge;
}

}  // namespace etbfs
