// TEST INFRASTRUCTURE ONLY — never linked into the product.
//
// extern "C" shim over the *unmodified* reference library compiled from
// /root/reference/proj/src with -Detbfs=etbfs_ref (see oracle/Makefile).
// It lets pytest (ctypes), the golden-vector generator and bench.py's
// reference / cpu_baseline arm call the reference's own public API:
//   generate_kronecker   proj/include/etbfs/kronecker.hpp:34
//   build_csr            proj/include/etbfs/build.hpp:19
//   classify_vertices    proj/include/etbfs/classify.hpp:33, compute_peak_height :38
//   relayout_csr         proj/include/etbfs/relayout.hpp:40
//   extract_edge_tree_list proj/include/etbfs/relayout.hpp:52
//   et_bfs               proj/include/etbfs/et_bfs.hpp:53
//   oracle_bfs / validate_bfs_tree  proj/include/etbfs/validate.hpp:37-46
//   select_roots / run_benchmark    proj/include/etbfs/bench.hpp:78-84
//   write_graph / read_graph / write_tree / read_tree  proj/include/etbfs/io.hpp:23-31
// Nothing here re-implements reference logic; it only marshals vectors.
#include <chrono>
#include <cstdint>
#include <cstring>
#include <exception>
#include <string>
#include <vector>

#ifdef _OPENMP
#include <omp.h>
#endif

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

using namespace etbfs_ref;

namespace {
thread_local std::string g_err;
int fail(const std::exception& e) {
  g_err = e.what();
  return -1;
}
struct Prepared {
  ClassifiedGraph cg;
  EdgeTreeList etl;
};
EdgeList make_list(uint64_t n, const uint64_t* pairs, uint64_t count) {
  EdgeList el;
  el.vertex_count = n;
  el.edges.resize(count);
  for (uint64_t i = 0; i < count; ++i) el.edges[i] = {pairs[2 * i], pairs[2 * i + 1]};
  return el;
}
}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

// ---- degree split (preprocess.hpp:69) --------------------------------------------
// minus_cols == nullptr: sizes only (minus_offsets, n + 1, always written).
int ref_split_degree_aware(void* h, uint64_t limit, uint64_t* in_plus, uint64_t* minus_offsets,
                           uint64_t* minus_cols) {
  try {
    const CsrGraph& g = *static_cast<CsrGraph*>(h);
    const DegreeSplitAdjacency sp = split_degree_aware(g, limit);
    std::memcpy(minus_offsets, sp.minus_offsets.data(), sp.minus_offsets.size() * 8);
    if (in_plus) std::memcpy(in_plus, sp.in_plus.data(), sp.in_plus.size() * 8);
    if (minus_cols && !sp.minus_cols.empty())
      std::memcpy(minus_cols, sp.minus_cols.data(), sp.minus_cols.size() * 8);
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

// validate_bfs_tree with the report's per-rule failure counts (capped lists).
int ref_validate_report(void* h, uint64_t root, const uint64_t* parent, uint64_t* out8,
                        uint64_t* where125) {
  try {
    const CsrGraph& g = *static_cast<CsrGraph*>(h);
    BfsTree t;
    t.root = root;
    t.parent.assign(parent, parent + g.vertex_count);
    const ValidationReport rep = validate_bfs_tree(g, t);
    std::memset(out8, 0, 64);
    out8[0] = rep.passed;
    uint64_t idx[6] = {};
    for (const auto& f : rep.failures) {
      ++out8[f.rule];
      if (where125 && idx[f.rule] < 25) where125[(f.rule - 1) * 25 + idx[f.rule]++] = f.where;
    }
    out8[6] = rep.reached_count;
    out8[7] = rep.traversed_edge_count;
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

// ---- graph / tree files (io.hpp) ------------------------------------------------
int ref_write_graph(const char* path, int text, uint64_t n, const uint64_t* pairs, uint64_t count) {
  try {
    write_graph(path, make_list(n, pairs, count), text ? GraphFormat::kText : GraphFormat::kBinary);
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}
// pairs == nullptr: sizes only (the file is read twice).
int ref_read_graph(const char* path, int text, uint64_t* n, uint64_t* count, uint64_t* pairs) {
  try {
    const EdgeList el = read_graph(path, text ? GraphFormat::kText : GraphFormat::kBinary);
    *n = el.vertex_count;
    *count = el.edges.size();
    if (pairs)
      for (uint64_t i = 0; i < el.edges.size(); ++i) {
        pairs[2 * i] = el.edges[i].src;
        pairs[2 * i + 1] = el.edges[i].dst;
      }
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}
int ref_write_tree(const char* path, uint64_t n, uint64_t root, const uint64_t* parent) {
  try {
    BfsTree t;
    t.root = root;
    t.parent.assign(parent, parent + n);
    write_tree(path, t);
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}
int ref_read_tree(const char* path, uint64_t* n, uint64_t* root, uint64_t* parent) {
  try {
    const BfsTree t = read_tree(path);
    *n = t.parent.size();
    *root = t.root;
    if (parent) std::memcpy(parent, t.parent.data(), t.parent.size() * 8);
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

void ref_set_threads(int t) {
#ifdef _OPENMP
  omp_set_num_threads(t);
#else
  (void)t;
#endif
}

int ref_generate_kronecker(uint32_t scale, uint64_t ef, double a, double b, double c, double d,
                           uint64_t seed, uint64_t* out_pairs) {
  try {
    KroneckerParams p;
    p.scale = scale;
    p.edgefactor = ef;
    p.a = a;
    p.b = b;
    p.c = c;
    p.d = d;
    p.seed = seed;
    EdgeList el = generate_kronecker(p);
    std::memcpy(out_pairs, el.edges.data(), el.edges.size() * sizeof(Edge));
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

// CSR handle -------------------------------------------------------------
void* ref_build_csr(uint64_t n, const uint64_t* pairs, uint64_t count, uint64_t* self_loops,
                    uint64_t* dups) {
  try {
    BuildStats st;
    auto* g = new CsrGraph(build_csr(make_list(n, pairs, count), &st));
    if (self_loops) *self_loops = st.dropped_self_loops;
    if (dups) *dups = st.dropped_duplicates;
    return g;
  } catch (const std::exception& e) {
    fail(e);
    return nullptr;
  }
}
// An empty reference CsrGraph of n vertices and nnz directed edges whose arrays
// the caller fills in place (e.g. a device CSR downloaded straight into them:
// no second host copy of a scale-28 column array).
void* ref_csr_alloc(uint64_t n, uint64_t nnz, uint64_t** row_offsets, uint64_t** cols,
                    uint64_t** degrees) {
  try {
    auto* g = new CsrGraph;
    g->vertex_count = n;
    g->row_offsets.resize(n + 1);
    g->col_indices.resize(nnz);
    g->degrees.resize(n);
    *row_offsets = g->row_offsets.data();
    *cols = g->col_indices.data();
    *degrees = g->degrees.data();
    return g;
  } catch (const std::exception& e) {
    fail(e);
    return nullptr;
  }
}
uint64_t ref_csr_nnz(void* h) { return static_cast<CsrGraph*>(h)->col_indices.size(); }
uint64_t ref_csr_n(void* h) { return static_cast<CsrGraph*>(h)->vertex_count; }
void ref_csr_copy(void* h, uint64_t* row_offsets, uint64_t* cols) {
  auto* g = static_cast<CsrGraph*>(h);
  if (row_offsets) std::memcpy(row_offsets, g->row_offsets.data(), g->row_offsets.size() * 8);
  if (cols) std::memcpy(cols, g->col_indices.data(), g->col_indices.size() * 8);
}
void ref_csr_free(void* h) { delete static_cast<CsrGraph*>(h); }

int ref_classify(void* h, int64_t mh, uint8_t* types_out) {
  try {
    auto t = classify_vertices(*static_cast<CsrGraph*>(h), mh);
    for (size_t i = 0; i < t.size(); ++i) types_out[i] = static_cast<uint8_t>(t[i]);
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}
int64_t ref_peak_height(void* h) {
  try {
    return static_cast<int64_t>(compute_peak_height(*static_cast<CsrGraph*>(h)));
  } catch (const std::exception& e) {
    return fail(e);
  }
}

// Relayout + ETL handle ---------------------------------------------------
void* ref_prepare(void* h, int64_t mh) {
  try {
    const CsrGraph& g = *static_cast<CsrGraph*>(h);
    auto* p = new Prepared;
    p->cg = relayout_csr(g, classify_vertices(g, mh), mh);
    p->etl = extract_edge_tree_list(p->cg);
    return p;
  } catch (const std::exception& e) {
    fail(e);
    return nullptr;
  }
}
uint64_t ref_prep_core(void* p) { return static_cast<Prepared*>(p)->cg.core_vertex_count; }
uint64_t ref_prep_etl_size(void* p) { return static_cast<Prepared*>(p)->etl.entries.size(); }
uint64_t ref_prep_nnz(void* p) { return static_cast<Prepared*>(p)->cg.graph.col_indices.size(); }
uint64_t ref_prep_restricted_edges(void* p) {
  auto* pp = static_cast<Prepared*>(p);
  return restricted_edge_count(pp->cg.graph, pp->cg.core_vertex_count);
}
void ref_prep_copy(void* p, uint64_t* new2old, uint8_t* types, uint64_t* row_offsets,
                   uint64_t* cols, uint64_t* etl_src, uint64_t* etl_dst, uint64_t* etl_ce) {
  auto* pp = static_cast<Prepared*>(p);
  const auto& cg = pp->cg;
  const uint64_t n = cg.graph.vertex_count;
  if (new2old) std::memcpy(new2old, cg.new2old.data(), n * 8);
  if (types)
    for (uint64_t i = 0; i < n; ++i) types[i] = static_cast<uint8_t>(cg.vertex_type[i]);
  if (row_offsets) std::memcpy(row_offsets, cg.graph.row_offsets.data(), (n + 1) * 8);
  if (cols) std::memcpy(cols, cg.graph.col_indices.data(), cg.graph.col_indices.size() * 8);
  for (size_t i = 0; i < pp->etl.entries.size(); ++i) {
    if (etl_src) etl_src[i] = pp->etl.entries[i].src;
    if (etl_dst) etl_dst[i] = pp->etl.entries[i].dst;
    if (etl_ce) etl_ce[i] = pp->etl.entries[i].core_edge;
  }
}
void ref_prep_free(void* p) { delete static_cast<Prepared*>(p); }

// ---- lean entry points for scale 26 (host RAM) -----------------------------------
// FNV-1a-64 over bytes (SURVEY.md Appendix A convention); a hash, not reference logic.
static uint64_t fnv_bytes(const void* data, uint64_t len, uint64_t h = 0xcbf29ce484222325ull) {
  const unsigned char* p = static_cast<const unsigned char*>(data);
  for (uint64_t i = 0; i < len; ++i) {
    h ^= p[i];
    h *= 0x100000001b3ull;
  }
  return h;
}
uint64_t ref_fnv1a64(const void* data, uint64_t len) { return fnv_bytes(data, len); }

// generate_kronecker -> build_csr with the tuples freed before returning: the
// reference's own functions, without a second copy of the tuple list in Python
// (scale 26: 17 GB of tuples + the build's 34 GB fit a 62 GB host only this way).
void* ref_kron_csr(uint32_t scale, uint64_t ef, uint64_t seed, uint64_t* tuples_fnv,
                   uint64_t* self_loops, uint64_t* dups) {
  try {
    KroneckerParams p;
    p.scale = scale;
    p.edgefactor = ef;
    p.seed = seed;
    BuildStats st;
    CsrGraph* g;
    {
      EdgeList el = generate_kronecker(p);
      if (tuples_fnv) *tuples_fnv = fnv_bytes(el.edges.data(), el.edges.size() * sizeof(Edge));
      g = new CsrGraph(build_csr(el, &st));
    }
    if (self_loops) *self_loops = st.dropped_self_loops;
    if (dups) *dups = st.dropped_duplicates;
    return g;
  } catch (const std::exception& e) {
    fail(e);
    return nullptr;
  }
}
// FNV of the CSR arrays: out[0] row_offsets, out[1] col_indices.
void ref_csr_fnv(void* h, uint64_t* out) {
  const CsrGraph& g = *static_cast<CsrGraph*>(h);
  out[0] = fnv_bytes(g.row_offsets.data(), g.row_offsets.size() * 8);
  out[1] = fnv_bytes(g.col_indices.data(), g.col_indices.size() * 8);
}
// FNV of a prepared layout without copying it out: out[0] new2old, out[1] relaid
// row_offsets, out[2] relaid col_indices, out[3] ETL as (src,dst,core_edge) u64 rows.
void ref_prep_fnv(void* p, uint64_t* out) {
  const auto* pp = static_cast<Prepared*>(p);
  const auto& cg = pp->cg;
  out[0] = fnv_bytes(cg.new2old.data(), cg.new2old.size() * 8);
  out[1] = fnv_bytes(cg.graph.row_offsets.data(), cg.graph.row_offsets.size() * 8);
  out[2] = fnv_bytes(cg.graph.col_indices.data(), cg.graph.col_indices.size() * 8);
  uint64_t h = 0xcbf29ce484222325ull;
  for (const auto& e : pp->etl.entries) {
    const uint64_t row[3] = {e.src, e.dst, e.core_edge};
    h = fnv_bytes(row, 24, h);
  }
  out[3] = h;
}
// A layout produced elsewhere (byte-identical to relayout_csr + extract, as the
// parity tests pin) wrapped as the reference's ClassifiedGraph / EdgeTreeList, so
// the reference's et_bfs can be timed without re-running its single-threaded
// preprocessing. Arrays are in relaid space; types are VertexType codes.
void* ref_prep_from_arrays(uint64_t n, uint64_t core, int64_t mh, const uint64_t* new2old,
                           const uint8_t* types, const uint64_t* row, const uint64_t* col,
                           uint64_t etl_count, const uint64_t* etl_src, const uint64_t* etl_dst,
                           const uint64_t* etl_ce) {
  try {
    auto* p = new Prepared;
    ClassifiedGraph& cg = p->cg;
    cg.graph.vertex_count = n;
    cg.graph.row_offsets.assign(row, row + n + 1);
    cg.graph.col_indices.assign(col, col + row[n]);
    cg.graph.degrees.resize(n);
    for (uint64_t v = 0; v < n; ++v) cg.graph.degrees[v] = row[v + 1] - row[v];
    cg.vertex_type.resize(n);
    for (uint64_t v = 0; v < n; ++v) cg.vertex_type[v] = static_cast<VertexType>(types[v]);
    cg.new2old.assign(new2old, new2old + n);
    cg.old2new = invert_permutation(cg.new2old);
    cg.core_vertex_count = core;
    cg.mh = mh;
    p->etl.entries.resize(etl_count);
    for (uint64_t i = 0; i < etl_count; ++i)
      p->etl.entries[i] = EdgeTreeEntry{etl_src[i], etl_dst[i], etl_ce[i]};
    return p;
  } catch (const std::exception& e) {
    fail(e);
    return nullptr;
  }
}

// kernel: 0 top-down, 1 hybrid (et_bfs.hpp CoreKernel order); replay 0 teet, 1 teolv.
// Writes the relaid-space parent array and the direction trace; returns seconds.
double ref_et_bfs(void* p, uint64_t start, int kernel, int replay, double alpha, double beta,
                  uint64_t* parent_out, char* trace_out, uint64_t trace_cap) {
  try {
    auto* pp = static_cast<Prepared*>(p);
    HybridPolicy pol;
    pol.alpha = alpha;
    pol.beta = beta;
    KernelStats st;
    const auto t0 = std::chrono::steady_clock::now();
    BfsTree t = et_bfs(pp->cg, pp->etl, start, static_cast<CoreKernel>(kernel),
                       static_cast<TreeReplay>(replay), nullptr, pol, trace_out ? &st : nullptr);
    const double s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    if (parent_out) std::memcpy(parent_out, t.parent.data(), t.parent.size() * 8);
    if (trace_out && trace_cap > 0) {
      const size_t k = std::min<size_t>(st.direction_trace.size(), trace_cap - 1);
      std::memcpy(trace_out, st.direction_trace.data(), k);
      trace_out[k] = 0;
    }
    return s;
  } catch (const std::exception& e) {
    fail(e);
    return -1.0;
  }
}

// Whole-graph hybrid on a plain CSR (bfs.hpp:53) with its direction trace.
int ref_bfs_hybrid(void* h, uint64_t root, double alpha, double beta, uint64_t* parent_out,
                   char* trace_out, uint64_t trace_cap) {
  try {
    HybridPolicy pol;
    pol.alpha = alpha;
    pol.beta = beta;
    KernelStats st;
    BfsTree t = bfs_hybrid(*static_cast<CsrGraph*>(h), root, pol, &st);
    if (parent_out) std::memcpy(parent_out, t.parent.data(), t.parent.size() * 8);
    if (trace_out && trace_cap > 0) {
      const size_t k = std::min<size_t>(st.direction_trace.size(), trace_cap - 1);
      std::memcpy(trace_out, st.direction_trace.data(), k);
      trace_out[k] = 0;
    }
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

int ref_oracle_bfs(void* h, uint64_t root, uint64_t* levels_out) {
  try {
    auto lv = oracle_bfs(*static_cast<CsrGraph*>(h), root);
    std::memcpy(levels_out, lv.data(), lv.size() * 8);
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

// Validates a parent tree in the CSR's own index space. Returns 1 pass / 0 fail,
// -1 on error; writes the traversed-edge count (the GTEPS numerator) and the
// first failing rule id (0 if none).
int ref_validate(void* h, uint64_t root, const uint64_t* parent, uint64_t* te, int* first_rule) {
  try {
    const CsrGraph& g = *static_cast<CsrGraph*>(h);
    BfsTree t;
    t.root = root;
    t.parent.assign(parent, parent + g.vertex_count);
    ValidationReport r = validate_bfs_tree(g, t);
    if (te) *te = r.traversed_edge_count;
    if (first_rule) *first_rule = r.failures.empty() ? 0 : r.failures.front().rule;
    return r.passed ? 1 : 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

int ref_select_roots(void* h, uint64_t count, uint64_t seed, uint64_t* out) {
  try {
    auto r = select_roots(*static_cast<CsrGraph*>(h), count, seed);
    std::memcpy(out, r.data(), r.size() * 8);
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

// The reference's own harness (bench.cpp:244-299), unmodified: generate ->
// run_benchmark. kernel: 0 top-down, 1 hybrid, 4 et-bfs (KernelChoice order).
// Per-root seconds / traversed edges / valid flags land in the out arrays.
int ref_run_benchmark(uint32_t scale, uint64_t ef, uint64_t gen_seed, int kernel, int64_t mh,
                      int replay, uint64_t roots, uint64_t root_seed, uint64_t threads,
                      uint64_t* root_out, double* seconds_out, uint64_t* te_out, int* valid_out,
                      double* preprocessing_seconds, double* generate_seconds) {
  try {
    KroneckerParams p;
    p.scale = scale;
    p.edgefactor = ef;
    p.seed = gen_seed;
#ifdef _OPENMP
    omp_set_num_threads(static_cast<int>(threads));
#endif
    const auto t0 = std::chrono::steady_clock::now();
    EdgeList el = generate_kronecker(p);
    if (generate_seconds)
      *generate_seconds =
          std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    BenchConfig cfg;
    cfg.kernel = static_cast<KernelChoice>(kernel);
    cfg.mh = mh;
    cfg.roots = roots;
    cfg.seed = root_seed;
    cfg.threads = threads;
    cfg.replay = static_cast<TreeReplay>(replay);
    BenchReport rep = run_benchmark(el, cfg);
    for (size_t i = 0; i < rep.per_root.size(); ++i) {
      root_out[i] = rep.per_root[i].root;
      seconds_out[i] = rep.per_root[i].seconds;
      te_out[i] = rep.per_root[i].traversed_edges;
      valid_out[i] = rep.per_root[i].valid ? 1 : 0;
    }
    if (preprocessing_seconds) *preprocessing_seconds = rep.preprocessing_seconds;
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

}  // extern "C"
