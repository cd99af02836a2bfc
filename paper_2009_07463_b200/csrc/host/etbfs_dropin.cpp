// The C++ drop-in: the reference's public entry points
// (/root/reference/proj/include/etbfs/*.hpp) implemented over the C-ABI of
// include/etbfs_cuda.h. Host work here is marshalling only (vector <-> device
// buffers, status -> exception); every compute step runs on the GPU.
#include <algorithm>
#include <cmath>
#include <cstring>
#include <memory>
#include <mutex>
#include <stdexcept>
#include <string>

#include "etbfs/bfs.hpp"
#include "etbfs/build.hpp"
#include "etbfs/classify.hpp"
#include "etbfs/et_bfs.hpp"
#include "etbfs/kronecker.hpp"
#include "etbfs/preprocess.hpp"
#include "etbfs/relayout.hpp"
#include "etbfs/types.hpp"
#include "etbfs_cuda.h"
#include "etbfs_hash.hpp"

namespace etbfs {
namespace {

using detail::hash_bytes;
using detail::hash_vec;

void check(int rc) {
  if (rc == ETB_OK) return;
  const std::string msg = etb_last_error();
  if (rc == ETB_EINVAL) throw std::invalid_argument(msg);
  throw std::runtime_error(msg);
}

struct GraphDel {
  void operator()(etb_graph* g) const { etb_graph_free(g); }
};
struct LayoutDel {
  void operator()(etb_layout* l) const { etb_layout_free(l); }
};
using GraphPtr = std::unique_ptr<etb_graph, GraphDel>;
using LayoutPtr = std::unique_ptr<etb_layout, LayoutDel>;

GraphPtr upload(const CsrGraph& g) {
  if (g.row_offsets.size() != g.vertex_count + 1)
    throw std::invalid_argument("etbfs: CsrGraph row_offsets size mismatch");
  etb_graph* h = nullptr;
  check(etb_graph_from_csr(g.vertex_count, g.row_offsets.data(), g.col_indices.data(), &h));
  return GraphPtr(h);
}

CsrGraph download_graph(etb_graph* h) {
  CsrGraph g;
  uint64_t n = 0, m = 0;
  check(etb_graph_info(h, &n, &m));
  g.vertex_count = n;
  g.row_offsets.resize(n + 1);
  g.col_indices.resize(m);
  g.degrees.resize(n);
  check(etb_graph_download(h, g.row_offsets.data(), g.col_indices.data(), g.degrees.data()));
  return g;
}

std::vector<uint8_t> type_bytes(const std::vector<VertexType>& t) {
  std::vector<uint8_t> b(t.size());
  for (size_t i = 0; i < t.size(); ++i) b[i] = static_cast<uint8_t>(t[i]);
  return b;
}

LayoutPtr layout_from_types(etb_graph* g, const std::vector<uint8_t>& types, std::int64_t mh) {
  etb_layout* l = nullptr;
  check(etb_layout_build_types(g, types.data(), mh, &l));
  return LayoutPtr(l);
}

uint64_t hash_etl(const EdgeTreeList& etl) {
  return hash_bytes(etl.entries.data(), etl.entries.size() * sizeof(EdgeTreeEntry),
                    0xE71ull ^ etl.entries.size());
}

uint64_t hash_split(const DegreeSplitAdjacency& sp) {
  uint64_t h = hash_vec(sp.in_plus, 1);
  h = hash_vec(sp.minus_offsets, h);
  h = hash_vec(sp.minus_cols, h);
  return h;  // (neighbor_limit is checked against the core separately)
}

// A device layout built for a host ClassifiedGraph (relaid space). Relayout of
// an already relaid graph is the identity for the reference's own layouts;
// the maps below translate for any other valid input (e.g. a shuffled core).
// The cache key is the classified graph's CONTENT (rows, columns, types,
// new2old, core size, mh), so a new graph at freed addresses or an edit in
// place never reuses a stale layout.
struct DeviceCg {
  uint64_t key = 0;
  GraphPtr g;
  LayoutPtr l;
  std::vector<uint64_t> dev2cg, cg2dev;
  bool identity = true;
  EdgeTreeList etl;        // the canonical extract_edge_tree_list(cg)
  uint64_t etl_hash = 0;
  bool have_split = false;  // the canonical split_degree_aware(cg.graph, core), lazily
  uint64_t split_hash = 0;
};

std::mutex g_cache_mu;
std::unique_ptr<DeviceCg> g_cache;

uint64_t cg_key(const ClassifiedGraph& cg) {
  const CsrGraph& G = cg.graph;
  uint64_t h = hash_vec(G.row_offsets, G.vertex_count);
  h = hash_vec(G.col_indices, h);
  h = hash_bytes(cg.vertex_type.data(), cg.vertex_type.size() * sizeof(VertexType), h);
  h = hash_vec(cg.new2old, h);
  return h ^ (cg.core_vertex_count * 0x9E3779B97F4A7C15ull) ^ static_cast<uint64_t>(cg.mh + 2);
}

DeviceCg& device_cg(const ClassifiedGraph& cg) {
  const CsrGraph& G = cg.graph;
  if (cg.vertex_type.size() != G.vertex_count)
    throw std::invalid_argument("extract_edge_tree_list: types length does not match vertex count");
  const uint64_t key = cg_key(cg);
  if (g_cache && g_cache->key == key) return *g_cache;
  auto d = std::make_unique<DeviceCg>();
  d->key = key;
  d->g = upload(G);
  d->l = layout_from_types(d->g.get(), type_bytes(cg.vertex_type), cg.mh);
  d->dev2cg.resize(G.vertex_count);
  d->cg2dev.resize(G.vertex_count);
  check(etb_layout_download_maps(d->l.get(), d->dev2cg.data(), d->cg2dev.data(), nullptr));
  for (uint64_t i = 0; i < G.vertex_count && d->identity; ++i) d->identity = d->dev2cg[i] == i;
  etb_layout_info info;
  check(etb_layout_info_get(d->l.get(), &info));
  const uint64_t m = info.tree_vertex_count;
  std::vector<uint64_t> s(m), t(m), c(m);
  check(etb_layout_download_etl(d->l.get(), s.data(), t.data(), c.data()));
  d->etl.entries.resize(m);
  for (uint64_t i = 0; i < m; ++i) {
    d->etl.entries[i].src = d->dev2cg[s[i]];
    d->etl.entries[i].dst = d->dev2cg[t[i]];
    d->etl.entries[i].core_edge = c[i] == ETB_NO_VERTEX ? kNoVertex : d->dev2cg[c[i]];
  }
  if (!d->identity)
    std::sort(d->etl.entries.begin(), d->etl.entries.end(),
              [](const EdgeTreeEntry& a, const EdgeTreeEntry& b) { return a.dst < b.dst; });
  d->etl_hash = hash_etl(d->etl);
  g_cache = std::move(d);
  return *g_cache;
}

etb_bfs_options options(CoreKernel kernel, TreeReplay replay, const HybridPolicy& policy) {
  etb_bfs_options o{};
  switch (kernel) {
    case CoreKernel::kTopDown: o.kernel = ETB_KERNEL_TOP_DOWN; break;
    case CoreKernel::kHybrid: o.kernel = ETB_KERNEL_HYBRID; break;
    case CoreKernel::kDegreeAware: o.kernel = ETB_KERNEL_DEGREE_AWARE; break;
    case CoreKernel::kBlockSearch: o.kernel = ETB_KERNEL_BLOCK_SEARCH; break;
    case CoreKernel::kHybridBlockSearch: o.kernel = ETB_KERNEL_HYBRID_BLOCK_SEARCH; break;
  }
  o.replay = replay == TreeReplay::kTeolv ? ETB_REPLAY_TEOLV : ETB_REPLAY_TEET;
  o.alpha = policy.alpha;
  o.beta = policy.beta;
  return o;
}

void fill_stats(const etb_bfs_stats& s, KernelStats* stats) {
  if (!stats) return;
  stats->levels += s.levels;
  stats->bottom_up_levels += s.bottom_up_levels;
  stats->direction_trace += s.direction_trace;
}

BfsTree run(etb_layout* l, uint64_t n, uint64_t start_dev, const etb_bfs_options& o,
            KernelStats* stats, const std::vector<uint64_t>* dev2cg) {
  std::vector<uint64_t> parent(n);
  etb_bfs_stats st;
  check(etb_bfs(l, start_dev, &o, nullptr, parent.data(), stats ? &st : nullptr));
  if (stats) fill_stats(st, stats);
  BfsTree t;
  if (!dev2cg) {
    t.parent = std::move(parent);
    t.root = start_dev;
    return t;
  }
  t.parent.assign(n, kNoVertex);
  for (uint64_t i = 0; i < n; ++i)
    if (parent[i] != kNoVertex) t.parent[(*dev2cg)[i]] = (*dev2cg)[parent[i]];
  t.root = (*dev2cg)[start_dev];
  return t;
}

// Whole-graph traversal (bfs.hpp:50-53): every vertex typed core, so the core
// block is the whole graph and the α/β limit is vertex_count as in bfs.cpp.
BfsTree whole_graph(const CsrGraph& graph, vertex_t root, const etb_bfs_options& o,
                    KernelStats* stats) {
  if (root >= graph.vertex_count) throw std::invalid_argument("bfs: root out of range");
  if ((o.kernel == ETB_KERNEL_HYBRID || o.kernel == ETB_KERNEL_DEGREE_AWARE) &&
      (!(o.alpha > 0.0) || !(o.beta > 0.0)))
    throw std::invalid_argument("run_hybrid: alpha and beta must be positive");
  GraphPtr g = upload(graph);
  std::vector<uint8_t> types(graph.vertex_count, ETB_CI);
  LayoutPtr l = layout_from_types(g.get(), types, -1);
  std::vector<uint64_t> n2o(graph.vertex_count), o2n(graph.vertex_count);
  check(etb_layout_download_maps(l.get(), n2o.data(), o2n.data(), nullptr));
  return run(l.get(), graph.vertex_count, o2n[root], o, stats, &n2o);
}

}  // namespace

const char* to_string(VertexType t) {
  switch (t) {
    case VertexType::kCoreInternal: return "CI";
    case VertexType::kCoreEdge: return "CE";
    case VertexType::kTreeInternal: return "TI";
    case VertexType::kTreeLeaf: return "TL";
    case VertexType::kVertexZero: return "VZ";
  }
  return "?";
}

EdgeList generate_kronecker(const KroneckerParams& p) {
  // Argument checks before allocating, as kronecker.cpp:24-34 (same messages);
  // the C-ABI repeats them.
  if (p.scale > 48) throw std::invalid_argument("generate_kronecker: scale > 48");
  if (p.edgefactor < 1) throw std::invalid_argument("generate_kronecker: edgefactor < 1");
  if (std::fabs(p.a + p.b + p.c + p.d - 1.0) > 1e-12)
    throw std::invalid_argument("generate_kronecker: probabilities must sum to 1");
  const uint64_t n = uint64_t{1} << p.scale;
  if ((n * p.edgefactor) / p.edgefactor != n)
    throw std::runtime_error("generate_kronecker: tuple count overflows");
  etb_kron_params kp{p.scale, p.edgefactor, p.a, p.b, p.c, p.d, p.seed};
  EdgeList out;
  out.vertex_count = n;
  out.edges.resize(n * p.edgefactor);
  check(etb_generate_kronecker(&kp, reinterpret_cast<uint64_t*>(out.edges.data())));
  return out;
}

CsrGraph build_csr(const EdgeList& edges, BuildStats* stats) {
  static_assert(sizeof(Edge) == 16, "Edge must be two packed u64");
  etb_graph* h = nullptr;
  uint64_t loops = 0, dups = 0;
  check(etb_graph_from_edges(edges.vertex_count,
                             reinterpret_cast<const uint64_t*>(edges.edges.data()),
                             edges.edges.size(), &h, &loops, &dups));
  GraphPtr g(h);
  if (stats) {
    stats->dropped_self_loops = loops;
    stats->dropped_duplicates = dups;
  }
  return download_graph(g.get());
}

std::vector<vertex_t> invert_permutation(const std::vector<vertex_t>& new2old) {
  std::vector<vertex_t> old2new(new2old.size(), kNoVertex);
  for (size_t i = 0; i < new2old.size(); ++i) {
    const vertex_t o = new2old[i];
    if (o >= new2old.size() || old2new[o] != kNoVertex)
      throw std::invalid_argument("invert_permutation: input is not a permutation");
    old2new[o] = i;
  }
  return old2new;
}

std::vector<VertexType> classify_vertices(const CsrGraph& graph, std::int64_t mh) {
  if (mh < -1) throw std::invalid_argument("classify_vertices: mh must be -1 or >= 0");
  GraphPtr g = upload(graph);
  std::vector<uint8_t> t(graph.vertex_count);
  check(etb_classify(g.get(), mh, t.data(), nullptr));
  std::vector<VertexType> out(t.size());
  for (size_t i = 0; i < t.size(); ++i) out[i] = static_cast<VertexType>(t[i]);
  return out;
}

std::uint64_t compute_peak_height(const CsrGraph& graph) {
  GraphPtr g = upload(graph);
  uint64_t ph = 0;
  check(etb_peak_height(g.get(), &ph));
  return ph;
}

TypeCounts count_types(const std::vector<VertexType>& types) {
  TypeCounts c;
  for (VertexType t : types) {
    switch (t) {
      case VertexType::kCoreInternal: ++c.core_internal; break;
      case VertexType::kCoreEdge: ++c.core_edge; break;
      case VertexType::kTreeInternal: ++c.tree_internal; break;
      case VertexType::kTreeLeaf: ++c.tree_leaf; break;
      case VertexType::kVertexZero: ++c.vertex_zero; break;
    }
  }
  return c;
}

ClassifiedGraph relayout_csr(const CsrGraph& graph, const std::vector<VertexType>& types,
                             std::int64_t mh) {
  if (types.size() != graph.vertex_count)
    throw std::invalid_argument("relayout_csr: types length does not match vertex count");
  GraphPtr g = upload(graph);
  LayoutPtr l = layout_from_types(g.get(), type_bytes(types), mh);
  etb_layout_info info;
  check(etb_layout_info_get(l.get(), &info));
  const uint64_t n = graph.vertex_count;
  ClassifiedGraph cg;
  cg.new2old.resize(n);
  cg.old2new.resize(n);
  std::vector<uint8_t> t(n);
  check(etb_layout_download_maps(l.get(), cg.new2old.data(), cg.old2new.data(), t.data()));
  cg.vertex_type.resize(n);
  for (uint64_t i = 0; i < n; ++i) cg.vertex_type[i] = static_cast<VertexType>(t[i]);
  cg.graph.vertex_count = n;
  cg.graph.row_offsets.resize(n + 1);
  cg.graph.col_indices.resize(info.directed_edges);
  check(etb_layout_download_graph(l.get(), cg.graph.row_offsets.data(),
                                  cg.graph.col_indices.data()));
  cg.graph.degrees.resize(n);
  for (uint64_t v = 0; v < n; ++v)
    cg.graph.degrees[v] = cg.graph.row_offsets[v + 1] - cg.graph.row_offsets[v];
  cg.core_vertex_count = info.core_vertex_count;
  cg.mh = mh;
  return cg;
}

EdgeTreeList extract_edge_tree_list(const ClassifiedGraph& cg) {
  std::lock_guard<std::mutex> lk(g_cache_mu);
  return device_cg(cg).etl;
}

BfsTree et_bfs(const ClassifiedGraph& cg, const EdgeTreeList& etl, vertex_t start,
               CoreKernel kernel, TreeReplay replay, const DegreeSplitAdjacency* split,
               const HybridPolicy& policy, KernelStats* stats) {
  const uint64_t n = cg.graph.vertex_count;
  if (start >= n) throw std::invalid_argument("et_bfs: start out of range");
  if (replay == TreeReplay::kTeolv && cg.mh != 0)
    throw std::invalid_argument("et_bfs: leaves-only replay needs a height-0 classification");
  // et_bfs.cpp:69-70: the split-based kernels require a split; the device's
  // degree-sorted rows make its content unnecessary, so it is only checked.
  const bool needs_split = kernel == CoreKernel::kDegreeAware ||
                           kernel == CoreKernel::kBlockSearch ||
                           kernel == CoreKernel::kHybridBlockSearch;
  if (needs_split) {
    if (split == nullptr) throw std::invalid_argument("et_bfs: kernel needs a degree split");
    const uint64_t core = cg.core_vertex_count;
    const bool covers_core =
        split->neighbor_limit == core || (split->neighbor_limit == kNoVertex && core == n);
    if (split->in_plus.size() != n || !covers_core)
      throw std::invalid_argument("et_bfs: split does not match the core block");
  }
  const etb_bfs_options o = options(kernel, replay, policy);
  std::lock_guard<std::mutex> lk(g_cache_mu);
  DeviceCg& d = device_cg(cg);
  // The device replays the layout's own tree arrays, i.e. the canonical
  // extract_edge_tree_list(cg); a caller list that differs from it (edited, or
  // from another graph) is refused rather than silently ignored.
  if (etl.entries.size() != d.etl.entries.size() || hash_etl(etl) != d.etl_hash)
    throw std::invalid_argument(
        "et_bfs: edge tree list does not match extract_edge_tree_list(cg)");
  // Likewise the split: the device rows are already in the split's probe order,
  // which holds for the canonical split_degree_aware(cg.graph, core) only.
  if (needs_split) {
    if (!d.have_split) {
      d.split_hash = hash_split(split_degree_aware(cg.graph, cg.core_vertex_count));
      d.have_split = true;
    }
    if (hash_split(*split) != d.split_hash)
      throw std::invalid_argument(
          "et_bfs: split does not match split_degree_aware(cg.graph, core)");
  }
  return run(d.l.get(), n, d.cg2dev[start], o, stats, d.identity ? nullptr : &d.dev2cg);
}

BfsTree bfs_top_down(const CsrGraph& graph, vertex_t root, KernelStats* stats) {
  return whole_graph(graph, root, options(CoreKernel::kTopDown, TreeReplay::kTeet, {}), stats);
}

BfsTree bfs_hybrid(const CsrGraph& graph, vertex_t root, const HybridPolicy& policy,
                   KernelStats* stats) {
  return whole_graph(graph, root, options(CoreKernel::kHybrid, TreeReplay::kTeet, policy), stats);
}

namespace {
// bfs.cpp:25-30: the whole-graph split kernels need a split of the whole graph.
void check_full_split(const CsrGraph& graph, const DegreeSplitAdjacency& split) {
  if (split.in_plus.size() != graph.vertex_count)
    throw std::invalid_argument("bfs: split size does not match graph");
  if (split.neighbor_limit != kNoVertex && split.neighbor_limit < graph.vertex_count)
    throw std::invalid_argument("bfs: split excludes neighbors the traversal needs");
}
}  // namespace

BfsTree bfs_degree_aware(const CsrGraph& graph, const DegreeSplitAdjacency& split, vertex_t root,
                         const HybridPolicy& policy, KernelStats* stats) {
  if (root >= graph.vertex_count) throw std::invalid_argument("bfs: root out of range");
  check_full_split(graph, split);
  return whole_graph(graph, root, options(CoreKernel::kDegreeAware, TreeReplay::kTeet, policy),
                     stats);
}

BfsTree bfs_block_search(const CsrGraph& graph, const DegreeSplitAdjacency& split, vertex_t root,
                         KernelStats* stats) {
  if (root >= graph.vertex_count) throw std::invalid_argument("bfs: root out of range");
  check_full_split(graph, split);
  return whole_graph(graph, root, options(CoreKernel::kBlockSearch, TreeReplay::kTeet, {}), stats);
}

std::uint64_t restricted_edge_count(const CsrGraph& graph, vertex_t limit) {
  // bfs.cpp:50-59 on caller-held host rows (a query, not traversal work; the
  // device layouts carry their own count, etb_layout_restricted_edges).
  if (limit >= graph.vertex_count) return graph.directed_edge_count();
  uint64_t total = 0;
  for (vertex_t v = 0; v < limit; ++v) {
    const auto nb = graph.neighbors(v);
    total += static_cast<uint64_t>(std::lower_bound(nb.begin(), nb.end(), limit) - nb.begin());
  }
  return total;
}

}  // namespace etbfs
