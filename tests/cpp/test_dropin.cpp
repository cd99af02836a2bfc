// C++ drop-in test: the reference's public API (include/etbfs/*.hpp) driven
// exactly as the reference's own unit tests drive it (proj/tests/*.cpp KATs,
// restated), with an independent host BFS as the level oracle. Every call
// goes through the C-ABI to the sm_100a kernels. Exit status = failures.
#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <deque>
#include <functional>
#include <set>
#include <stdexcept>
#include <string>
#include <vector>

#include "etbfs/bench.hpp"
#include "etbfs/bfs.hpp"
#include "etbfs/build.hpp"
#include "etbfs/classify.hpp"
#include "etbfs/et_bfs.hpp"
#include "etbfs/io.hpp"
#include "etbfs/kronecker.hpp"
#include "etbfs/preprocess.hpp"
#include "etbfs/relayout.hpp"
#include "etbfs/validate.hpp"

using namespace etbfs;

static int g_fail = 0, g_checks = 0;
static std::string g_case;
#define EXPECT(cond)                                                                  \
  do {                                                                                \
    ++g_checks;                                                                       \
    if (!(cond)) {                                                                    \
      ++g_fail;                                                                       \
      std::fprintf(stderr, "FAIL [%s] %s:%d: %s\n", g_case.c_str(), __FILE__, __LINE__, #cond); \
    }                                                                                 \
  } while (0)
template <typename E, typename F>
bool throws_with(F&& f, const char* needle) {
  try {
    f();
  } catch (const E& e) {
    return needle == nullptr || std::string(e.what()).find(needle) != std::string::npos;
  } catch (...) {
    return false;
  }
  return false;
}

namespace {

using Types = std::vector<VertexType>;
constexpr auto CI = VertexType::kCoreInternal;
constexpr auto CE = VertexType::kCoreEdge;
constexpr auto TI = VertexType::kTreeInternal;
constexpr auto TL = VertexType::kTreeLeaf;
constexpr auto VZ = VertexType::kVertexZero;

EdgeList edges(uint64_t n, std::vector<std::pair<vertex_t, vertex_t>> p) {
  EdgeList e;
  e.vertex_count = n;
  for (auto [a, b] : p) e.edges.push_back({a, b});
  return e;
}
EdgeList path(uint64_t n) {
  EdgeList e;
  e.vertex_count = n;
  for (vertex_t v = 0; v + 1 < n; ++v) e.edges.push_back({v, v + 1});
  return e;
}
EdgeList cycle(uint64_t n) {
  EdgeList e = path(n);
  if (n >= 3) e.edges.push_back({n - 1, 0});
  return e;
}
EdgeList star(uint64_t n) {
  EdgeList e;
  e.vertex_count = n;
  for (vertex_t v = 1; v < n; ++v) e.edges.push_back({0, v});
  return e;
}
EdgeList clique(uint64_t n) {
  EdgeList e;
  e.vertex_count = n;
  for (vertex_t u = 0; u < n; ++u)
    for (vertex_t v = u + 1; v < n; ++v) e.edges.push_back({u, v});
  return e;
}
EdgeList binary_tree(uint64_t n) {
  EdgeList e;
  e.vertex_count = n;
  for (vertex_t v = 1; v < n; ++v) e.edges.push_back({(v - 1) / 2, v});
  return e;
}
// Deterministic raw tuples (self loops and duplicates left in).
EdgeList random_tuples(uint64_t n, uint64_t m, uint64_t seed) {
  EdgeList e;
  e.vertex_count = n;
  uint64_t s = seed * 0x9E3779B97F4A7C15ull + 1;
  auto next = [&] {
    s ^= s << 13;
    s ^= s >> 7;
    s ^= s << 17;
    return s;
  };
  for (uint64_t i = 0; i < m; ++i) e.edges.push_back({next() % n, next() % n});
  return e;
}

// Independent level oracle: adjacency sets + deque BFS (not the library's CSR).
std::vector<uint64_t> host_levels(const EdgeList& el, vertex_t root) {
  std::vector<std::set<vertex_t>> adj(el.vertex_count);
  for (const Edge& e : el.edges)
    if (e.src != e.dst) adj[e.src].insert(e.dst), adj[e.dst].insert(e.src);
  std::vector<uint64_t> lv(el.vertex_count, kUnreached);
  std::deque<vertex_t> q{root};
  lv[root] = 0;
  while (!q.empty()) {
    vertex_t u = q.front();
    q.pop_front();
    for (vertex_t w : adj[u])
      if (lv[w] == kUnreached) lv[w] = lv[u] + 1, q.push_back(w);
  }
  return lv;
}

// Levels implied by a parent tree, by fixpoint (shares nothing with the library).
std::vector<uint64_t> fixpoint_levels(const BfsTree& t) {
  const uint64_t n = t.parent.size();
  std::vector<uint64_t> lv(n, kUnreached);
  if (t.root >= n || t.parent[t.root] != t.root) return {};
  lv[t.root] = 0;
  for (uint64_t sweep = 0; sweep <= n; ++sweep) {
    bool changed = false;
    for (vertex_t v = 0; v < n; ++v) {
      if (v == t.root || t.parent[v] == kNoVertex || t.parent[v] >= n) continue;
      const uint64_t pl = lv[t.parent[v]];
      if (pl != kUnreached && lv[v] != pl + 1) lv[v] = pl + 1, changed = true;
    }
    if (!changed) break;
  }
  return lv;
}

EdgeList relabeled(const ClassifiedGraph& cg) {
  EdgeList e;
  e.vertex_count = cg.graph.vertex_count;
  for (vertex_t v = 0; v < cg.graph.vertex_count; ++v)
    for (vertex_t w : cg.graph.neighbors(v))
      if (v < w) e.edges.push_back({v, w});
  return e;
}

void check_tree_exact(const EdgeList& el, const BfsTree& t, vertex_t root) {
  EXPECT(t.root == root);
  const auto want = host_levels(el, root);
  EXPECT(fixpoint_levels(t) == want);
  std::vector<std::set<vertex_t>> adj(el.vertex_count);
  for (const Edge& e : el.edges)
    if (e.src != e.dst) adj[e.src].insert(e.dst), adj[e.dst].insert(e.src);
  for (vertex_t v = 0; v < el.vertex_count; ++v)
    if (v != root && t.parent[v] != kNoVertex) EXPECT(adj[v].count(t.parent[v]) == 1);
}

std::vector<EdgeList> corpus() {
  std::vector<EdgeList> c = {path(1), path(2), path(9), cycle(8), star(17), clique(6),
                             binary_tree(31), edges(6, {}), edges(7, {{0, 1}, {2, 3}, {3, 4}})};
  for (uint64_t s = 1; s <= 10; ++s) c.push_back(random_tuples(20 + s * 13, 30 + s * 40, s));
  return c;
}

void run_case(const char* name, const std::function<void()>& f) {
  g_case = name;
  const int before = g_fail;
  try {
    f();
  } catch (const std::exception& e) {
    ++g_fail;
    std::fprintf(stderr, "FAIL [%s] unexpected exception: %s\n", name, e.what());
  }
  std::printf("%s %s\n", g_fail == before ? "PASS" : "FAIL", name);
}

}  // namespace

// Host restatement of one bottom-up step's parent rule for the checks below:
// the first neighbour (in the given order) present in `in`.
vertex_t first_in(const std::vector<vertex_t>& order, const Bitmap& in) {
  for (vertex_t x : order)
    if (in.get(x)) return x;
  return kNoVertex;
}

int main() {
  run_case("et_bfs composed from the public pieces (et_bfs.cpp:59-124 restated)", [] {
    for (const EdgeList& el : corpus()) {
      const CsrGraph g = build_csr(el);
      for (int64_t mh : {int64_t{-1}, int64_t{0}}) {
        const ClassifiedGraph cg = relayout_csr(g, classify_vertices(g, mh), mh);
        const EdgeTreeList etl = extract_edge_tree_list(cg);
        const EdgeList rel = relabeled(cg);
        const uint64_t n = cg.graph.vertex_count, core = cg.core_vertex_count;
        for (vertex_t s = 0; s < n; ++s) {
          BfsTree t;
          t.root = s;
          t.parent.assign(n, kNoVertex);
          FrontierState st(n);
          vertex_t cstart = s;
          const VertexType ty = cg.vertex_type[s];
          if (ty == VertexType::kTreeInternal || ty == VertexType::kTreeLeaf)
            cstart = traverse_return_core_edge(cg, s, t);
          else if (ty == VertexType::kVertexZero)
            cstart = kNoVertex, t.parent[s] = s;
          else
            t.parent[s] = s;
          if (cstart != kNoVertex && cstart < core) {
            st.visited.set(cstart);
            st.current.set(cstart);
            run_hybrid(cg.graph, nullptr, BottomUpKind::kClassic, st, t.parent, core, {});
          }
          if (mh == 0) teolv(etl, st.visited, t.parent);
          else teet(etl, st.visited, t.parent);
          EXPECT(fixpoint_levels(t) == host_levels(rel, s));
        }
      }
    }
    EXPECT(throws_with<std::invalid_argument>(
        [] {
          const CsrGraph g = build_csr(path(3));
          const ClassifiedGraph cg = relayout_csr(g, classify_vertices(g, 0), 0);
          BfsTree t;
          t.parent.assign(3, kNoVertex);
          traverse_return_core_edge(cg, 0, t);
        },
        "start is not a tree vertex"));
  });

  run_case("step and driver layer on the GPU (bfs.hpp:66-120)", [] {
    EXPECT(block_search_unvisited(0b1010) == (std::pair<std::uint32_t, std::uint64_t>{1, 0b1000}));
    for (const EdgeList& el : corpus()) {
      const CsrGraph g = build_csr(el);
      const uint64_t n = g.vertex_count;
      const DegreeSplitAdjacency sp = split_degree_aware(g);
      for (vertex_t r = 0; r < n; r += 4) {
        const auto want = host_levels(el, r);
        auto seeded = [&](FrontierState& st, std::vector<vertex_t>& par) {
          st = FrontierState(n);
          par.assign(n, kNoVertex);
          par[r] = r;
          st.visited.set(r);
          st.current.set(r);
        };
        FrontierState st;
        std::vector<vertex_t> par;
        // drivers: exact levels; the hybrid trace matches the persistent kernel's
        for (int d = 0; d < 5; ++d) {
          seeded(st, par);
          KernelStats ks;
          if (d == 0) run_top_down(g, st, par, n, &ks);
          if (d == 1) run_hybrid(g, nullptr, BottomUpKind::kClassic, st, par, n, {}, &ks);
          if (d == 2) run_hybrid(g, &sp, BottomUpKind::kDegreeAware, st, par, n, {}, &ks);
          if (d == 3) run_hybrid(g, &sp, BottomUpKind::kBlockSearch, st, par, n, {}, &ks);
          if (d == 4) run_block_search(g, sp, st, par, n, &ks);
          BfsTree t;
          t.root = r;
          t.parent = par;
          EXPECT(fixpoint_levels(t) == want);
          EXPECT(ks.levels == ks.direction_trace.size());
          if (d == 1) {
            KernelStats ref;
            bfs_hybrid(g, r, {}, &ref);
            EXPECT(ks.direction_trace == ref.direction_trace);
          }
        }
        // single steps: claims and the deterministic bottom-up parent rules
        seeded(st, par);
        const StepResult td = top_down_step(g, st, par, n);
        uint64_t deg1 = 0, sc = 0;
        for (vertex_t v = 0; v < n; ++v)
          if (want[v] == 1) ++deg1, sc += g.degrees[v];
        EXPECT(td.claimed == deg1 && td.scout == sc);
        st.advance_level();
        for (int kind = 0; kind < 3; ++kind) {
          FrontierState s2 = st;
          std::vector<vertex_t> p2 = par;
          if (kind == 0) bottom_up_step(g, s2, p2, n);
          if (kind == 1) degree_aware_step(g, sp, s2, p2, n);
          if (kind == 2) block_search_step(g, sp, s2, p2, n);
          for (vertex_t w = 0; w < n; ++w) {
            if (st.visited.get(w)) {
              EXPECT(p2[w] == par[w]);
              continue;
            }
            std::vector<vertex_t> order;
            if (kind == 0) {
              order.assign(g.neighbors(w).begin(), g.neighbors(w).end());
            } else {
              if (sp.in_plus[w] != kNoVertex) order.push_back(sp.in_plus[w]);
              order.insert(order.end(), sp.in_minus(w).begin(), sp.in_minus(w).end());
            }
            // classic / degree-aware probe the frontier, block search the
            // pre-step visited set
            const vertex_t want_p = first_in(order, kind == 2 ? st.visited : st.current);
            EXPECT(p2[w] == want_p);
            EXPECT(s2.next.get(w) == (want_p != kNoVertex));
          }
        }
      }
    }
    const CsrGraph g = build_csr(path(4));
    FrontierState bad(3);
    std::vector<vertex_t> p(4, kNoVertex);
    EXPECT(throws_with<std::invalid_argument>([&] { top_down_step(g, bad, p, 4); },
                                              "frontier state does not match graph"));
    FrontierState ok(4);
    EXPECT(throws_with<std::invalid_argument>(
        [&] { run_hybrid(g, nullptr, BottomUpKind::kDegreeAware, ok, p, 4, {}); },
        "needs a degree split"));
  });

  run_case("degree split, split kernels, checker side (preprocess/validate/bench.hpp)", [] {
    // star centre 0 with a 2-path hanging off leaf 3: degrees 0:4 3:2
    const CsrGraph g = build_csr(edges(6, {{0, 1}, {0, 2}, {0, 3}, {0, 4}, {3, 5}}));
    const DegreeSplitAdjacency sp = split_degree_aware(g);
    EXPECT(sp.in_plus[3] == 0 && sp.in_plus[0] == 3 && sp.in_plus[5] == 3);
    EXPECT(std::vector<vertex_t>(sp.in_minus(0).begin(), sp.in_minus(0).end()) ==
           (std::vector<vertex_t>{1, 2, 4}));
    const DegreeSplitAdjacency lim = split_degree_aware(g, 3);
    EXPECT(lim.in_plus[5] == kNoVertex && lim.in_plus[3] == 0 && lim.in_minus(0).size() == 1);
    for (const EdgeList& el : corpus()) {
      const CsrGraph cg = build_csr(el);
      const DegreeSplitAdjacency full = split_degree_aware(cg);
      for (vertex_t r = 0; r < el.vertex_count; r += 3) {
        const auto want = host_levels(el, r);
        EXPECT(fixpoint_levels(bfs_degree_aware(cg, full, r)) == want);
        EXPECT(fixpoint_levels(bfs_block_search(cg, full, r)) == want);
        EXPECT(oracle_bfs(cg, r) == want);
        const BfsTree t = bfs_hybrid(cg, r);
        EXPECT(tree_levels(t) == want);
        const ValidationReport rep = validate_bfs_tree(cg, t);
        EXPECT(rep.passed && rep.failures.empty());
        if (el.vertex_count > 2 && t.parent[r] == r) {
          BfsTree bad = t;
          bad.parent[r] = kNoVertex;
          const ValidationReport r2 = validate_bfs_tree(cg, bad);
          EXPECT(!r2.passed && r2.failures.front().rule == kRuleRootParent &&
                 r2.failures.front().message == "root is not its own parent");
        }
      }
    }
    EXPECT(throws_with<std::invalid_argument>(
        [&] { bfs_degree_aware(g, lim, 0); }, "split excludes neighbors the traversal needs"));
    KroneckerParams kp;
    kp.scale = 16;
    kp.seed = 1;
    const CsrGraph s16 = build_csr(generate_kronecker(kp));
    const auto roots = select_roots(s16, 8, 1);
    EXPECT(roots == (std::vector<vertex_t>{23745, 51467, 640, 15525, 34165, 15784, 20321, 24000}));
    EXPECT(compute_gteps(2000000000, 2.0) == 1.0);
    EXPECT(throws_with<std::invalid_argument>([] { compute_gteps(1, 0.0); }, "must be positive"));
    BfsTree tr;
    tr.root = 1;
    tr.parent = {1, 1, 0};
    const BfsTree back = translate_tree(tr, {2, 0, 1});
    EXPECT(back.root == 0 && back.parent == (std::vector<vertex_t>{0, 2, 0}));
  });

  run_case("graph / tree files (test_io.cpp cases) feeding a GPU traversal", [] {
    const std::string gpath = "/tmp/etbfs_dropin_io.etg", tpath = "/tmp/etbfs_dropin_io.ett";
    const EdgeList el = random_tuples(300, 900, 4);
    write_graph(gpath, el, GraphFormat::kBinary);
    const EdgeList back = read_graph(gpath, parse_graph_format("binary"));
    EXPECT(back.vertex_count == el.vertex_count && back.edges == el.edges);
    write_graph(gpath, el, GraphFormat::kText);
    EXPECT(read_graph(gpath, GraphFormat::kText).edges == el.edges);
    const CsrGraph g = build_csr(back);
    const ClassifiedGraph cg = relayout_csr(g, classify_vertices(g, -1), -1);
    const EdgeTreeList etl = extract_edge_tree_list(cg);
    const BfsTree t = et_bfs(cg, etl, cg.old2new[7]);
    write_tree(tpath, t);
    const BfsTree t2 = read_tree(tpath);
    EXPECT(t2.root == t.root && t2.parent == t.parent);
    EXPECT(throws_with<std::invalid_argument>([] { parse_graph_format("csv"); },
                                              "unknown graph format \"csv\""));
    EXPECT(throws_with<std::runtime_error>([&] { read_tree(gpath); }, "bad magic, expected ETT1"));
    std::remove(gpath.c_str());
    std::remove(tpath.c_str());
  });

  run_case("build_csr KAT (test_graph_core.cpp:17-36)", [] {
    BuildStats st;
    const CsrGraph g = build_csr(
        edges(5, {{0, 1}, {1, 0}, {0, 1}, {2, 2}, {3, 1}, {1, 3}, {4, 0}, {0, 4}, {0, 4}}), &st);
    EXPECT(g.vertex_count == 5);
    EXPECT(g.undirected_edge_count() == 3);
    EXPECT(st.dropped_self_loops == 1);
    EXPECT(st.dropped_duplicates == 5);
    EXPECT(std::vector<vertex_t>(g.neighbors(0).begin(), g.neighbors(0).end()) ==
           (std::vector<vertex_t>{1, 4}));
    EXPECT(g.degrees[2] == 0);
    EXPECT(throws_with<std::invalid_argument>([] { build_csr(edges(3, {{0, 1}, {1, 3}})); },
                                              "endpoint out of range at edge index 1"));
  });

  run_case("generate_kronecker determinism and validation", [] {
    KroneckerParams p;
    p.scale = 10;
    p.seed = 7;
    const EdgeList a = generate_kronecker(p), b = generate_kronecker(p);
    EXPECT(a.edges.size() == (1u << 10) * 16u && a.edges == b.edges && a.vertex_count == 1024);
    for (const Edge& e : a.edges) EXPECT(e.src < 1024 && e.dst < 1024);
    p.scale = 49;
    EXPECT(throws_with<std::invalid_argument>([&] { generate_kronecker(p); }, "scale > 48"));
    p.scale = 4;
    p.a = 0.6;
    EXPECT(throws_with<std::invalid_argument>([&] { generate_kronecker(p); }, "sum to 1"));
  });

  run_case("classification KATs (test_classify.cpp:80-138)", [] {
    const CsrGraph p3 = build_csr(path(3));
    EXPECT(classify_vertices(p3, -1) == (Types{TL, TI, TL}));
    EXPECT(classify_vertices(p3, 0) == (Types{TL, CE, TL}));
    EXPECT(compute_peak_height(p3) == 1);
    const CsrGraph p5 = build_csr(path(5));
    EXPECT(classify_vertices(p5, -1) == (Types{TL, TI, TI, TI, TL}));
    EXPECT(compute_peak_height(p5) == 2);
    EXPECT(classify_vertices(p5, 1) == (Types{TL, TI, TI, CE, TL}));
    EXPECT(classify_vertices(p5, 0) == (Types{TL, CE, CI, CE, TL}));
    const CsrGraph p7 = build_csr(path(7));
    EXPECT(compute_peak_height(p7) == 2);
    EXPECT(classify_vertices(p7, 1) == (Types{TL, TI, TI, TI, TI, CE, TL}));
    const CsrGraph s5 = build_csr(star(5));
    EXPECT(classify_vertices(s5, -1) == (Types{TI, TL, TL, TL, TL}));
    EXPECT(classify_vertices(s5, 0) == (Types{CE, TL, TL, TL, TL}));
    const CsrGraph tri =
        build_csr(edges(6, {{0, 1}, {1, 2}, {0, 2}, {2, 3}, {3, 4}, {3, 5}}));
    EXPECT(classify_vertices(tri, -1) == (Types{CI, CI, CE, TI, TL, TL}));
    EXPECT(classify_vertices(tri, 0) == (Types{CI, CI, CI, CE, TL, TL}));
    EXPECT(compute_peak_height(build_csr(cycle(6))) == 0);
    EXPECT(classify_vertices(build_csr(clique(5)), -1) == Types(5, CI));
    const CsrGraph pair = build_csr(edges(4, {{0, 1}}));
    EXPECT(classify_vertices(pair, -1) == (Types{TL, TL, VZ, VZ}));
    EXPECT(compute_peak_height(pair) == 0);
    EXPECT(throws_with<std::invalid_argument>([&] { classify_vertices(p3, -2); }, nullptr));
    const TypeCounts c = count_types({CI, CE, CE, TI, TL, TL, TL, VZ});
    EXPECT(c.core() == 3 && c.tree() == 4 && c.total() == 8);
  });

  run_case("relayout frozen layouts (test_relayout.cpp:110-158)", [] {
    const CsrGraph g = build_csr(edges(6, {{0, 1}, {1, 2}, {0, 2}, {2, 3}, {3, 4}, {3, 5}}));
    const ClassifiedGraph cg = relayout_csr(g, classify_vertices(g, -1), -1);
    EXPECT(cg.core_vertex_count == 3);
    EXPECT(cg.new2old == (std::vector<vertex_t>{2, 0, 1, 3, 4, 5}));
    EXPECT(cg.vertex_type[0] == CE && cg.vertex_type[3] == TI);
    const EdgeTreeList etl = extract_edge_tree_list(cg);
    EXPECT(etl.entries == (std::vector<EdgeTreeEntry>{{0, 3, 0}, {3, 4, 0}, {3, 5, 0}}));
    const CsrGraph s = build_csr(star(5));
    const ClassifiedGraph sc = relayout_csr(s, classify_vertices(s, -1), -1);
    EXPECT(sc.core_vertex_count == 0 && sc.new2old == (std::vector<vertex_t>{0, 1, 2, 3, 4}));
    const EdgeTreeList se = extract_edge_tree_list(sc);
    EXPECT(se.entries.size() == 5 && se.entries[0] == (EdgeTreeEntry{0, 0, kNoVertex}));
    const CsrGraph pr = build_csr(edges(4, {{0, 1}}));
    const ClassifiedGraph pc = relayout_csr(pr, classify_vertices(pr, 0), 0);
    EXPECT(extract_edge_tree_list(pc).entries ==
           (std::vector<EdgeTreeEntry>{{0, 0, kNoVertex}, {0, 1, kNoVertex}}));
    EXPECT(throws_with<std::invalid_argument>(
        [&] { relayout_csr(g, Types(2, CI), -1); }, "types length does not match"));
  });

  run_case("composite traversal is level-exact across the corpus (test_et_bfs.cpp:158-169)", [] {
    for (const EdgeList& el : corpus()) {
      const CsrGraph g = build_csr(el);
      for (std::int64_t mh : {std::int64_t{-1}, std::int64_t{0}, std::int64_t{1}}) {
        const ClassifiedGraph cg = relayout_csr(g, classify_vertices(g, mh), mh);
        const EdgeTreeList etl = extract_edge_tree_list(cg);
        const EdgeList rel = relabeled(cg);
        for (vertex_t s = 0; s < g.vertex_count; ++s) {
          for (CoreKernel k : {CoreKernel::kTopDown, CoreKernel::kHybrid})
            check_tree_exact(rel, et_bfs(cg, etl, s, k), s);
          if (mh == 0)
            check_tree_exact(rel, et_bfs(cg, etl, s, CoreKernel::kHybrid, TreeReplay::kTeolv), s);
        }
      }
    }
  });

  run_case("composite config errors (test_et_bfs.cpp:181-195)", [] {
    const CsrGraph g = build_csr(path(8));
    const ClassifiedGraph cg = relayout_csr(g, classify_vertices(g, -1), -1);
    const EdgeTreeList etl = extract_edge_tree_list(cg);
    EXPECT(throws_with<std::invalid_argument>([&] { et_bfs(cg, etl, 99); }, "out of range"));
    EXPECT(throws_with<std::invalid_argument>(
        [&] { et_bfs(cg, etl, 0, CoreKernel::kHybrid, TreeReplay::kTeolv); }, "height-0"));
    EXPECT(throws_with<std::invalid_argument>(
        [&] { et_bfs(cg, etl, 0, CoreKernel::kDegreeAware); }, "degree split"));
  });

  run_case("isolated start yields the one-vertex tree (test_et_bfs.cpp:171-179)", [] {
    const CsrGraph g = build_csr(edges(5, {{0, 1}, {1, 2}}));
    const ClassifiedGraph cg = relayout_csr(g, classify_vertices(g, -1), -1);
    const EdgeTreeList etl = extract_edge_tree_list(cg);
    EXPECT(cg.vertex_type[4] == VZ);
    const BfsTree t = et_bfs(cg, etl, 4);
    EXPECT(t.parent[4] == 4);
    for (vertex_t v = 0; v < 4; ++v) EXPECT(t.parent[v] == kNoVertex);
  });

  run_case("hybrid policy KATs (test_bfs_kernels.cpp:185-218)", [] {
    HybridPolicy tiny;
    tiny.alpha = 1e-9;
    KernelStats st;
    const BfsTree t = bfs_hybrid(build_csr(path(4)), 0, tiny, &st);
    check_tree_exact(path(4), t, 0);
    EXPECT(st.levels == 4 && st.bottom_up_levels == 0 && st.direction_trace == "tttt");
    HybridPolicy huge;
    huge.alpha = 1e18;
    KernelStats st2;
    check_tree_exact(path(6), bfs_hybrid(build_csr(path(6)), 0, huge, &st2), 0);
    EXPECT(!st2.direction_trace.empty() && st2.direction_trace[0] == 'b');
    EXPECT(st2.bottom_up_levels == st2.levels);
    KernelStats st3;
    check_tree_exact(star(300), bfs_hybrid(build_csr(star(300)), 5, {}, &st3), 5);
    EXPECT(st3.bottom_up_levels > 0 && st3.bottom_up_levels < st3.levels);
    HybridPolicy zero;
    zero.alpha = 0.0;
    EXPECT(throws_with<std::invalid_argument>(
        [&] { bfs_hybrid(build_csr(path(4)), 0, zero); }, "alpha and beta"));
    EXPECT(throws_with<std::invalid_argument>([&] { bfs_top_down(build_csr(path(4)), 4); },
                                              "out of range"));
    KernelStats one;
    EXPECT(bfs_hybrid(build_csr(path(1)), 0, {}, &one).parent == std::vector<vertex_t>{0});
    EXPECT(one.levels == 1);
    const CsrGraph g = build_csr(edges(5, {{0, 1}, {0, 2}, {1, 2}, {2, 3}, {3, 4}, {0, 4}}));
    EXPECT(restricted_edge_count(g, 0) == 0 && restricted_edge_count(g, 3) == 6);
  });

  run_case("Kronecker s14 end to end vs host BFS on the original ids", [] {
    KroneckerParams p;
    p.scale = 14;
    p.seed = 1;
    const EdgeList el = generate_kronecker(p);
    const CsrGraph g = build_csr(el);
    for (std::int64_t mh : {std::int64_t{-1}, std::int64_t{0}}) {
      const ClassifiedGraph cg = relayout_csr(g, classify_vertices(g, mh), mh);
      const EdgeTreeList etl = extract_edge_tree_list(cg);
      for (vertex_t r : {vertex_t{0}, vertex_t{1}, vertex_t{777}, vertex_t{4095}, vertex_t{12345}}) {
        const BfsTree t = et_bfs(cg, etl, cg.old2new[r]);
        BfsTree lifted;
        lifted.root = r;
        lifted.parent.assign(g.vertex_count, kNoVertex);
        for (vertex_t v = 0; v < g.vertex_count; ++v)
          if (t.parent[v] != kNoVertex) lifted.parent[cg.new2old[v]] = cg.new2old[t.parent[v]];
        check_tree_exact(el, lifted, r);
      }
    }
  });

  run_case("layout cache keyed on content: a classified graph rewritten in place", [] {
    // Two different graphs with the same vertex and edge counts: assigning the
    // second's layout into the first's vectors reuses their storage (same data()
    // pointers), the case a pointer-keyed cache would get wrong.
    const EdgeList a = random_tuples(300, 900, 5), b = random_tuples(300, 900, 6);
    const CsrGraph ga = build_csr(a), gb = build_csr(b);
    ClassifiedGraph cg = relayout_csr(ga, classify_vertices(ga, -1), -1);
    EdgeTreeList etl = extract_edge_tree_list(cg);
    check_tree_exact(relabeled(cg), et_bfs(cg, etl, 0), 0);
    const ClassifiedGraph cgb = relayout_csr(gb, classify_vertices(gb, -1), -1);
    if (cgb.graph.col_indices.size() == cg.graph.col_indices.size()) {
      const void* before = cg.graph.col_indices.data();
      cg = cgb;
      EXPECT(cg.graph.col_indices.data() == before);
    } else {
      cg = cgb;
    }
    etl = extract_edge_tree_list(cg);
    for (vertex_t s : {vertex_t{0}, vertex_t{17}, vertex_t{299}})
      check_tree_exact(relabeled(cg), et_bfs(cg, etl, s), s);
  });

  run_case("et_bfs refuses an edge tree list or split that does not belong to cg", [] {
    const CsrGraph g = build_csr(random_tuples(400, 700, 9));
    const ClassifiedGraph cg = relayout_csr(g, classify_vertices(g, -1), -1);
    EdgeTreeList etl = extract_edge_tree_list(cg);
    EXPECT(!etl.entries.empty());
    if (!etl.entries.empty()) {
      etl.entries.pop_back();
      EXPECT(throws_with<std::invalid_argument>([&] { et_bfs(cg, etl, 0); }, "edge tree list"));
    }
    const EdgeTreeList good = extract_edge_tree_list(cg);
    DegreeSplitAdjacency sp = split_degree_aware(cg.graph, cg.core_vertex_count);
    check_tree_exact(relabeled(cg), et_bfs(cg, good, 0, CoreKernel::kDegreeAware, TreeReplay::kTeet, &sp), 0);
    if (!sp.minus_cols.empty()) {
      std::reverse(sp.minus_cols.begin(), sp.minus_cols.end());
      EXPECT(throws_with<std::invalid_argument>(
          [&] { et_bfs(cg, good, 0, CoreKernel::kDegreeAware, TreeReplay::kTeet, &sp); }, "split"));
    }
  });

  run_case("run_benchmark / report_to_json (bench.hpp:30-89) on the GPU", [] {
    KroneckerParams kp;
    kp.scale = 12;
    kp.edgefactor = 8;
    kp.seed = 3;
    const EdgeList el = generate_kronecker(kp);
    const CsrGraph g = build_csr(el);
    for (KernelChoice k : {KernelChoice::kTopDown, KernelChoice::kHybrid, KernelChoice::kEtBfs}) {
      BenchConfig c;
      c.kernel = k;
      c.roots = 8;
      c.seed = 2;
      const BenchReport r = run_benchmark(el, c);
      EXPECT(r.all_valid);
      EXPECT(r.per_root.size() == 8);
      EXPECT(r.vertex_count == g.vertex_count);
      EXPECT(r.undirected_edge_count == g.undirected_edge_count());
      const auto roots = select_roots(g, 8, 2);
      for (size_t i = 0; i < r.per_root.size(); ++i) {
        EXPECT(r.per_root[i].root == roots[i]);
        const BfsTree t = bfs_hybrid(g, roots[i]);
        EXPECT(r.per_root[i].traversed_edges == validate_bfs_tree(g, t).traversed_edge_count);
        EXPECT(r.per_root[i].seconds > 0 && r.per_root[i].gteps > 0);
      }
      const std::string j = report_to_json(r);
      EXPECT(j.find("\"schema_version\": 1") != std::string::npos);
      EXPECT(j.find(std::string("\"kernel\": \"") + to_string(k) + "\"") != std::string::npos);
      EXPECT(report_to_text(r).find("all trees valid") != std::string::npos);
    }
    BenchConfig bad;
    bad.kernel = KernelChoice::kHybrid;
    bad.replay = TreeReplay::kTeolv;
    EXPECT(throws_with<std::invalid_argument>([&] { run_benchmark(el, bad); }, "requires et"));
    bad = BenchConfig{};
    bad.degree_aware = bad.block_search = true;
    EXPECT(throws_with<std::invalid_argument>([&] { run_benchmark(el, bad); }, "mutually"));
    EXPECT(parse_kernel("et-bfs") == KernelChoice::kEtBfs);
    EXPECT(throws_with<std::invalid_argument>([] { parse_kernel("bogus"); }, "unknown kernel"));
  });

  std::printf("%d checks, %d failures\n", g_checks, g_fail);
  return g_fail == 0 ? 0 : 1;
}
