// The benchmark harness of the drop-in (include/etbfs/bench.hpp; reference:
// proj/src/bench.cpp:46-368) over the C-ABI: the pipeline the configuration
// implies is built on the device once (untimed, as bench.cpp:253-256), each
// root's traversal is timed from "root given" to "BfsTree in host memory"
// (bench.cpp:269-271), and every tree is validated on the device
// (validate_bfs_tree's rules 1-5 over the whole graph, plus the traversed-edge
// count of validate.cpp:151-156). Host work is marshalling and aggregation.
#include <algorithm>
#include <charconv>
#include <chrono>
#include <cstring>
#include <iomanip>
#include <map>
#include <memory>
#include <sstream>
#include <stdexcept>

#include "etbfs/bench.hpp"
#include "etbfs/io.hpp"
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
struct LayoutDel {
  void operator()(etb_layout* l) const { etb_layout_free(l); }
};

// bench.cpp:46-60 (same rules and messages), plus the two CPU-only relabels.
void check_config(const BenchConfig& c) {
  if (c.roots == 0) throw std::invalid_argument("bench: roots must be >= 1");
  if (c.threads == 0) throw std::invalid_argument("bench: threads must be >= 1");
  if (c.degree_aware && c.block_search)
    throw std::invalid_argument("bench: degree-aware and block-search are mutually exclusive");
  if (c.kernel == KernelChoice::kTopDown && (c.degree_aware || c.block_search))
    throw std::invalid_argument("bench: top-down has no bottom-up phase to adjust");
  const bool et_mode = c.et || c.kernel == KernelChoice::kEtBfs;
  if (c.replay == TreeReplay::kTeolv) {
    if (!et_mode) throw std::invalid_argument("bench: leaves-only replay requires et");
    if (c.mh != 0) throw std::invalid_argument("bench: leaves-only replay requires mh = 0");
  }
  if (c.mh < -1) throw std::invalid_argument("bench: mh must be -1 or >= 0");
  if (c.rm_zero || c.round_robin)
    throw std::invalid_argument(
        "bench: rm_zero / round_robin are CPU thread-balancing relabels, not part of the B200 "
        "path");
}

// The device core kernel for a configuration (bench.cpp:62-83's mapping).
int core_kernel(const BenchConfig& c) {
  switch (c.kernel) {
    case KernelChoice::kTopDown: return ETB_KERNEL_TOP_DOWN;
    case KernelChoice::kDegreeAware: return ETB_KERNEL_DEGREE_AWARE;
    case KernelChoice::kBlockSearch: return ETB_KERNEL_BLOCK_SEARCH;
    case KernelChoice::kHybrid:
    case KernelChoice::kEtBfs: break;
  }
  if (c.degree_aware) return ETB_KERNEL_DEGREE_AWARE;
  if (c.block_search) return ETB_KERNEL_HYBRID_BLOCK_SEARCH;
  return ETB_KERNEL_HYBRID;
}

// Shortest round-trip decimal for a double (JSON numbers).
std::string num(double x) {
  char buf[64];
  auto r = std::to_chars(buf, buf + sizeof buf, x);
  std::string s(buf, r.ptr);
  if (s.find_first_of(".eEn") == std::string::npos) s += ".0";
  return s;
}

std::string quoted(const std::string& s) {
  std::string o = "\"";
  for (char ch : s) {
    if (ch == '"' || ch == '\\') o += '\\';
    o += ch;
  }
  return o + "\"";
}

// A tiny JSON value: objects keep their keys sorted (as nlohmann's default
// std::map object), rendering with a two-space indent.
struct J {
  enum Kind { kRaw, kObject, kArray } kind = kRaw;
  std::string raw;
  std::map<std::string, J> obj;
  std::vector<J> arr;
  static J r(std::string v) {
    J j;
    j.raw = std::move(v);
    return j;
  }
  void dump(std::ostringstream& o, int ind) const {
    const std::string pad(ind + 2, ' '), end(ind, ' ');
    if (kind == kRaw) {
      o << raw;
    } else if (kind == kObject) {
      if (obj.empty()) {
        o << "{}";
        return;
      }
      o << "{\n";
      size_t i = 0;
      for (const auto& [k, v] : obj) {
        o << pad << quoted(k) << ": ";
        v.dump(o, ind + 2);
        o << (++i < obj.size() ? ",\n" : "\n");
      }
      o << end << "}";
    } else {
      if (arr.empty()) {
        o << "[]";
        return;
      }
      o << "[\n";
      for (size_t i = 0; i < arr.size(); ++i) {
        o << pad;
        arr[i].dump(o, ind + 2);
        o << (i + 1 < arr.size() ? ",\n" : "\n");
      }
      o << end << "]";
    }
  }
};

J obj() {
  J j;
  j.kind = J::kObject;
  return j;
}
J b(bool v) { return J::r(v ? "true" : "false"); }
J u(uint64_t v) { return J::r(std::to_string(v)); }
J i(int64_t v) { return J::r(std::to_string(v)); }
J d(double v) { return J::r(num(v)); }
J s(const std::string& v) { return J::r(quoted(v)); }

}  // namespace

const char* to_string(KernelChoice kernel) {
  switch (kernel) {
    case KernelChoice::kTopDown: return "top-down";
    case KernelChoice::kHybrid: return "hybrid";
    case KernelChoice::kDegreeAware: return "degree-aware";
    case KernelChoice::kBlockSearch: return "block-search";
    case KernelChoice::kEtBfs: return "et-bfs";
  }
  return "?";
}

KernelChoice parse_kernel(const std::string& name) {
  static const std::pair<const char*, KernelChoice> names[] = {
      {"top-down", KernelChoice::kTopDown}, {"hybrid", KernelChoice::kHybrid},
      {"degree-aware", KernelChoice::kDegreeAware}, {"block-search", KernelChoice::kBlockSearch},
      {"et-bfs", KernelChoice::kEtBfs}};
  for (const auto& [n, k] : names)
    if (name == n) return k;
  throw std::invalid_argument("unknown kernel \"" + name +
                              "\" (top-down, hybrid, degree-aware, block-search, et-bfs)");
}

BenchReport run_benchmark(const EdgeList& edges, const BenchConfig& config) {
  check_config(config);
  using Clock = std::chrono::steady_clock;
  BenchReport rep;
  rep.config = config;
  const bool et_mode = config.et || config.kernel == KernelChoice::kEtBfs;
  const uint64_t n = edges.vertex_count;

  // ---- untimed preprocessing (bench.cpp:253-256): device CSR + layout ---------
  const auto t0 = Clock::now();
  etb_graph* gh = nullptr;
  check(etb_graph_from_edges(n, reinterpret_cast<const uint64_t*>(edges.edges.data()),
                             edges.edges.size(), &gh, nullptr, nullptr));
  std::unique_ptr<etb_graph, GraphDel> g(gh);
  etb_layout* lh = nullptr;
  if (et_mode) {
    check(etb_layout_build(g.get(), config.mh, &lh));
  } else {
    // whole-graph kernels: every vertex in the traversed block (bfs.hpp:50-64)
    const std::vector<uint8_t> types(n, ETB_CI);
    check(etb_layout_build_types(g.get(), types.data(), -1, &lh));
  }
  std::unique_ptr<etb_layout, LayoutDel> lay(lh);
  std::vector<uint64_t> new2old(n), old2new(n);
  check(etb_layout_download_maps(lay.get(), new2old.data(), old2new.data(), nullptr));
  CsrGraph degs;  // degrees only, for select_roots
  degs.vertex_count = n;
  degs.degrees.resize(n);
  uint64_t dn = 0, dm = 0;
  check(etb_graph_info(g.get(), &dn, &dm));
  check(etb_graph_download(g.get(), nullptr, nullptr, degs.degrees.data()));
  rep.preprocessing_seconds = std::chrono::duration<double>(Clock::now() - t0).count();
  rep.vertex_count = n;
  rep.undirected_edge_count = dm / 2;

  const std::vector<vertex_t> roots = select_roots(degs, config.roots, config.seed);
  etb_bfs_options o{};
  o.kernel = core_kernel(config);
  o.replay = config.replay == TreeReplay::kTeolv ? ETB_REPLAY_TEOLV : ETB_REPLAY_TEET;
  o.alpha = config.policy.alpha;
  o.beta = config.policy.beta;

  // The BfsTree's host buffer (relaid ids), page-locked once so the copy runs at
  // link speed; the reference allocates its parent vector inside the timed call.
  std::vector<uint64_t> parent(std::max<uint64_t>(n, 1));
  const bool pinned = etb_host_register(parent.data(), parent.size() * 8) == ETB_OK;
  rep.all_valid = true;
  double gsum = 0.0, inv = 0.0;
  try {
    for (const vertex_t root : roots) {
      const uint64_t start = old2new[root];
      const auto a = Clock::now();
      check(etb_bfs(lay.get(), start, &o, nullptr, parent.data(), nullptr));
      const double sec = std::chrono::duration<double>(Clock::now() - a).count();
      uint64_t counts[6] = {};
      check(etb_result_validate(lay.get(), start, counts));
      uint64_t te = 0;
      check(etb_result_traversed_edges(lay.get(), &te));
      if (!config.tree_out.empty() && rep.per_root.empty()) {
        BfsTree t;  // lift_tree (bench.cpp:175-186)
        t.root = root;
        t.parent.assign(n, kNoVertex);
        for (uint64_t v = 0; v < n; ++v)
          if (parent[v] != ETB_NO_VERTEX) t.parent[new2old[v]] = new2old[parent[v]];
        write_tree(config.tree_out, t);
      }
      RootResult r;
      r.root = root;
      r.seconds = sec;
      r.traversed_edges = te;
      r.gteps = compute_gteps(te, sec);
      r.valid = counts[0] == 0 && counts[1] == 0 && counts[2] == 0 && counts[3] == 0 &&
                counts[4] == 0;
      rep.all_valid = rep.all_valid && r.valid;
      gsum += r.gteps;
      inv += 1.0 / sec;
      rep.per_root.push_back(r);
    }
  } catch (...) {
    if (pinned) etb_host_unregister(parent.data());
    throw;
  }
  if (pinned) etb_host_unregister(parent.data());
  const double k = static_cast<double>(rep.per_root.size());
  rep.mean_gteps = gsum / k;
  const auto [lo, hi] = std::minmax_element(
      rep.per_root.begin(), rep.per_root.end(),
      [](const RootResult& x, const RootResult& y) { return x.gteps < y.gteps; });
  rep.min_gteps = lo->gteps;
  rep.max_gteps = hi->gteps;
  rep.harmonic_mean_seconds = k / inv;
  return rep;
}

std::string report_to_json(const BenchReport& r) {
  const BenchConfig& c = r.config;
  J root = obj();
  root.obj["schema_version"] = i(1);
  J cfg = obj();
  cfg.obj["kernel"] = s(to_string(c.kernel));
  cfg.obj["mh"] = i(c.mh);
  cfg.obj["roots"] = u(c.roots);
  cfg.obj["seed"] = u(c.seed);
  cfg.obj["threads"] = u(c.threads);
  cfg.obj["alpha"] = d(c.policy.alpha);
  cfg.obj["beta"] = d(c.policy.beta);
  cfg.obj["replay"] = s(c.replay == TreeReplay::kTeolv ? "teolv" : "teet");
  cfg.obj["rm_zero"] = b(c.rm_zero);
  cfg.obj["round_robin"] = b(c.round_robin);
  cfg.obj["degree_aware"] = b(c.degree_aware);
  cfg.obj["block_search"] = b(c.block_search);
  cfg.obj["et"] = b(c.et);
  cfg.obj["segments"] = u(c.segments);
  root.obj["config"] = cfg;
  J gr = obj();
  gr.obj["vertex_count"] = u(r.vertex_count);
  gr.obj["undirected_edge_count"] = u(r.undirected_edge_count);
  root.obj["graph"] = gr;
  J ag = obj();
  ag.obj["mean_gteps"] = d(r.mean_gteps);
  ag.obj["min_gteps"] = d(r.min_gteps);
  ag.obj["max_gteps"] = d(r.max_gteps);
  ag.obj["harmonic_mean_seconds"] = d(r.harmonic_mean_seconds);
  ag.obj["preprocessing_seconds"] = d(r.preprocessing_seconds);
  ag.obj["all_valid"] = b(r.all_valid);
  root.obj["aggregate"] = ag;
  J pr;
  pr.kind = J::kArray;
  for (const RootResult& x : r.per_root) {
    J e = obj();
    e.obj["root"] = u(x.root);
    e.obj["seconds"] = d(x.seconds);
    e.obj["traversed_edges"] = u(x.traversed_edges);
    e.obj["gteps"] = d(x.gteps);
    e.obj["valid"] = b(x.valid);
    pr.arr.push_back(e);
  }
  root.obj["per_root"] = pr;
  std::ostringstream o;
  root.dump(o, 0);
  return o.str();
}

std::string report_to_text(const BenchReport& r) {
  const BenchConfig& c = r.config;
  std::ostringstream o;
  o << "kernel " << to_string(c.kernel) << (c.et && c.kernel != KernelChoice::kEtBfs ? "+et" : "")
    << (c.degree_aware ? "+degree-aware" : "") << (c.block_search ? "+block-search" : "")
    << "  threads " << c.threads << "  mh " << c.mh << "  (B200)\n";
  o << "graph: " << r.vertex_count << " vertices, " << r.undirected_edge_count
    << " undirected edges\n";
  o << "preprocessing: " << r.preprocessing_seconds << " s\n";
  o << std::setw(12) << "root" << std::setw(14) << "seconds" << std::setw(14) << "edges"
    << std::setw(12) << "GTEPS" << std::setw(7) << "valid" << "\n";
  for (const RootResult& x : r.per_root)
    o << std::setw(12) << x.root << std::setw(14) << std::setprecision(5) << x.seconds
      << std::setw(14) << x.traversed_edges << std::setw(12) << std::setprecision(5) << x.gteps
      << std::setw(7) << (x.valid ? "yes" : "NO") << "\n";
  o << "mean " << r.mean_gteps << " GTEPS  (min " << r.min_gteps << ", max " << r.max_gteps
    << ")  harmonic-mean time " << r.harmonic_mean_seconds << " s\n";
  o << (r.all_valid ? "all trees valid" : "VALIDATION FAILURES PRESENT") << "\n";
  return o.str();
}

}  // namespace etbfs
