/* TEST INFRASTRUCTURE ONLY — see etbfs_oracle.h. Plain-C restatement of the
 * reference's hot path; every function cites the reference file:line it
 * follows (paths relative to /root/reference/proj). */
#include "etbfs_oracle.h"

#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

static char g_err[256];
const char* orc_last_error(void) { return g_err; }
static void set_err(const char* m) {
  strncpy(g_err, m, sizeof(g_err) - 1);
  g_err[sizeof(g_err) - 1] = 0;
}

/* ---------------------------------------------------------------- rng ---- */
/* include/etbfs/rng.hpp:10-15 */
uint64_t orc_splitmix64(uint64_t* state) {
  uint64_t z = (*state += 0x9e3779b97f4a7c15ull);
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}
/* include/etbfs/rng.hpp:18-20 */
double orc_uniform01(uint64_t* state) {
  return (double)(orc_splitmix64(state) >> 11) * 0x1.0p-53;
}

/* ------------------------------------------------------------ generator -- */
/* src/kronecker.cpp:23-69: counter-based R-MAT, no label permutation. */
int orc_generate_kronecker(uint32_t scale, uint64_t ef, double a, double b, double c, double d,
                           uint64_t seed, uint64_t* out) {
  if (scale > 48) { set_err("generate_kronecker: scale > 48"); return -1; }
  if (ef < 1) { set_err("generate_kronecker: edgefactor < 1"); return -1; }
  if (fabs(a + b + c + d - 1.0) > 1e-12) {
    set_err("generate_kronecker: probabilities must sum to 1");
    return -1;
  }
  const uint64_t n = (uint64_t)1 << scale;
  const uint64_t t = n * ef;
  const double ab = a + b, abc = ab + c; /* kronecker.cpp:40-41 */
  for (uint64_t i = 0; i < t; ++i) {
    uint64_t state = seed ^ (i * 0x2545f4914f6cdd1dull); /* :48 */
    uint64_t s = 0, dd = 0;
    for (uint32_t l = 0; l < scale; ++l) { /* :51-65 */
      const double u = orc_uniform01(&state);
      s <<= 1;
      dd <<= 1;
      if (u < a) {
      } else if (u < ab) {
        dd |= 1;
      } else if (u < abc) {
        s |= 1;
      } else {
        s |= 1;
        dd |= 1;
      }
    }
    out[2 * i] = s;
    out[2 * i + 1] = dd;
  }
  return 0;
}

/* ------------------------------------------------------------------ CSR -- */
static int cmp_u64(const void* x, const void* y) {
  const uint64_t a = *(const uint64_t*)x, b = *(const uint64_t*)y;
  return a < b ? -1 : (a > b);
}

/* src/build.cpp:21-87: count, scatter both directions, per-row sort+unique,
 * compact; duplicates counted per direction then halved (:80). */
orc_csr* orc_build_csr(uint64_t n, const uint64_t* pairs, uint64_t count, uint64_t* self_loops,
                       uint64_t* dups) {
  for (uint64_t i = 0; i < count; ++i)
    if (pairs[2 * i] >= n || pairs[2 * i + 1] >= n) {
      snprintf(g_err, sizeof g_err, "build_csr: endpoint out of range at edge index %llu",
               (unsigned long long)i);
      return NULL;
    }
  uint64_t* off = calloc(n + 1, 8);
  uint64_t loops = 0;
  for (uint64_t i = 0; i < count; ++i) {
    const uint64_t s = pairs[2 * i], d = pairs[2 * i + 1];
    if (s == d) { ++loops; continue; }
    ++off[s + 1];
    ++off[d + 1];
  }
  for (uint64_t v = 0; v < n; ++v) off[v + 1] += off[v];
  uint64_t* col = malloc((off[n] ? off[n] : 1) * 8);
  uint64_t* cur = malloc((n ? n : 1) * 8);
  memcpy(cur, off, n * 8);
  for (uint64_t i = 0; i < count; ++i) {
    const uint64_t s = pairs[2 * i], d = pairs[2 * i + 1];
    if (s == d) continue;
    col[cur[s]++] = d;
    col[cur[d]++] = s;
  }
  free(cur);
  uint64_t* noff = calloc(n + 1, 8);
  uint64_t dropped = 0, w = 0;
  for (uint64_t v = 0; v < n; ++v) {
    uint64_t b = off[v], e = off[v + 1];
    qsort(col + b, e - b, 8, cmp_u64);
    uint64_t kept = 0;
    for (uint64_t k = b; k < e; ++k)
      if (kept == 0 || col[k] != col[w - 1]) { col[w++] = col[k]; ++kept; }
    dropped += (e - b) - kept;
    noff[v + 1] = noff[v] + kept;
  }
  free(off);
  orc_csr* g = malloc(sizeof *g);
  g->n = n;
  g->nnz = noff[n];
  g->row = noff;
  g->col = realloc(col, (w ? w : 1) * 8);
  if (self_loops) *self_loops = loops;
  if (dups) *dups = dropped / 2;
  return g;
}
void orc_csr_free(orc_csr* g) {
  if (!g) return;
  free(g->row);
  free(g->col);
  free(g);
}
uint64_t orc_csr_n(const orc_csr* g) { return g->n; }
uint64_t orc_csr_nnz(const orc_csr* g) { return g->nnz; }
void orc_csr_copy(const orc_csr* g, uint64_t* row, uint64_t* col) {
  if (row) memcpy(row, g->row, (g->n + 1) * 8);
  if (col) memcpy(col, g->col, g->nnz * 8);
}
static inline uint64_t deg(const orc_csr* g, uint64_t v) { return g->row[v + 1] - g->row[v]; }

/* ------------------------------------------------------------- classify -- */
/* src/classify.cpp:10-52: leaf pass, then Gauss-Seidel rounds reading the
 * live counter num_new mid-round (:35-37), finally CE = untouched vertex that
 * lost a neighbour (:47-50). Returns the productive round count. */
int64_t orc_classify(const orc_csr* g, int64_t mh, uint8_t* type) {
  if (mh < -1) { set_err("classify_vertices: mh must be -1 or >= 0"); return -1; }
  const uint64_t n = g->n;
  uint64_t* num_pre = malloc((n ? n : 1) * 8);
  uint64_t* num_new = malloc((n ? n : 1) * 8);
  for (uint64_t v = 0; v < n; ++v) {
    type[v] = ORC_CI;
    num_pre[v] = num_new[v] = deg(g, v);
  }
  int found = 0;
  for (uint64_t v = 0; v < n; ++v) {
    if (num_pre[v] == 0) {
      type[v] = ORC_VZ;
    } else if (num_pre[v] == 1) {
      type[v] = ORC_TL;
      for (uint64_t k = g->row[v]; k < g->row[v + 1]; ++k) --num_new[g->col[k]];
      found = 1;
    }
  }
  int64_t productive = 0, h = 1;
  while (found && (mh == -1 || h <= mh)) {
    found = 0;
    memcpy(num_pre, num_new, n * 8);
    for (uint64_t v = 0; v < n; ++v) {
      if (type[v] != ORC_CI) continue;
      if (num_pre[v] == 0 || num_new[v] == 1) {
        type[v] = ORC_TI;
        for (uint64_t k = g->row[v]; k < g->row[v + 1]; ++k) --num_new[g->col[k]];
        found = 1;
      }
    }
    if (found) ++productive;
    ++h;
  }
  for (uint64_t v = 0; v < n; ++v)
    if (type[v] == ORC_CI && num_new[v] != deg(g, v)) type[v] = ORC_CE;
  free(num_pre);
  free(num_new);
  return productive;
}

/* ------------------------------------------------------------- relayout -- */
static int is_core(uint8_t t) { return t == ORC_CI || t == ORC_CE; }
static int is_tree(uint8_t t) { return t == ORC_TI || t == ORC_TL; }

static const orc_csr* g_sort_graph; /* qsort context for the core order */
static int cmp_core(const void* x, const void* y) {
  const uint64_t a = *(const uint64_t*)x, b = *(const uint64_t*)y;
  const uint64_t da = deg(g_sort_graph, a), db = deg(g_sort_graph, b);
  if (da != db) return da > db ? -1 : 1; /* degree descending */
  return a < b ? -1 : (a > b);           /* id ascending */
}

/* build.cpp:144-166: relabel through new2old, re-sort rows ascending. */
static void relabel(const orc_csr* g, const uint64_t* new2old, const uint64_t* old2new,
                    orc_csr* out) {
  const uint64_t n = g->n;
  out->n = n;
  out->nnz = g->nnz;
  out->row = calloc(n + 1, 8);
  out->col = malloc((g->nnz ? g->nnz : 1) * 8);
  for (uint64_t v = 0; v < n; ++v) out->row[v + 1] = out->row[v] + deg(g, new2old[v]);
  for (uint64_t v = 0; v < n; ++v) {
    const uint64_t o = new2old[v];
    uint64_t* dst = out->col + out->row[v];
    for (uint64_t k = g->row[o]; k < g->row[o + 1]; ++k) *dst++ = old2new[g->col[k]];
    qsort(out->col + out->row[v], deg(g, o), 8, cmp_u64);
  }
}

/* relayout.cpp:25-87: core block (degree desc, id asc), then per-CE trees in
 * core order each placed BFS-from-root (:44-69), whole-component trees rooted
 * at the smallest unplaced id (:72-73), then VZ (:75-76). */
orc_cg* orc_relayout(const orc_csr* g, const uint8_t* types, int64_t mh) {
  const uint64_t n = g->n;
  uint64_t* new2old = malloc((n ? n : 1) * 8);
  uint64_t cnt = 0;
  for (uint64_t v = 0; v < n; ++v)
    if (is_core(types[v])) new2old[cnt++] = v;
  const uint64_t core = cnt;
  g_sort_graph = g;
  qsort(new2old, core, 8, cmp_core);
  char* placed = calloc(n ? n : 1, 1);
  uint64_t* queue = malloc((n ? n : 1) * 8);
#define PLACE_TREE(root_)                                                   \
  do {                                                                      \
    const uint64_t proot = (root_);                                         \
    uint64_t qh = 0, qt = 0;                                                \
    placed[proot] = 1;                                                      \
    queue[qt++] = proot;                                                    \
    while (qh < qt) {                                                       \
      const uint64_t u = queue[qh++];                                       \
      new2old[cnt++] = u;                                                   \
      for (uint64_t k = g->row[u]; k < g->row[u + 1]; ++k) {                \
        const uint64_t w = g->col[k];                                       \
        if (is_tree(types[w]) && !placed[w]) { placed[w] = 1; queue[qt++] = w; } \
      }                                                                     \
    }                                                                       \
  } while (0)
  for (uint64_t i = 0; i < core; ++i) {
    const uint64_t c = new2old[i];
    if (types[c] != ORC_CE) continue;
    for (uint64_t k = g->row[c]; k < g->row[c + 1]; ++k) {
      const uint64_t w = g->col[k];
      if (is_tree(types[w]) && !placed[w]) PLACE_TREE(w);
    }
  }
  for (uint64_t v = 0; v < n; ++v)
    if (is_tree(types[v]) && !placed[v]) PLACE_TREE(v);
  for (uint64_t v = 0; v < n; ++v)
    if (types[v] == ORC_VZ) new2old[cnt++] = v;
#undef PLACE_TREE
  free(placed);
  free(queue);
  orc_cg* cg = calloc(1, sizeof *cg);
  cg->new2old = new2old;
  cg->old2new = malloc((n ? n : 1) * 8);
  for (uint64_t i = 0; i < n; ++i) cg->old2new[new2old[i]] = i;
  relabel(g, new2old, cg->old2new, &cg->g);
  cg->types = malloc(n ? n : 1);
  for (uint64_t i = 0; i < n; ++i) cg->types[i] = types[new2old[i]];
  cg->core = core;
  cg->mh = mh;
  return cg;
}
void orc_cg_free(orc_cg* cg) {
  if (!cg) return;
  free(cg->g.row);
  free(cg->g.col);
  free(cg->new2old);
  free(cg->old2new);
  free(cg->types);
  free(cg);
}
uint64_t orc_cg_core(const orc_cg* cg) { return cg->core; }
uint64_t orc_cg_nnz(const orc_cg* cg) { return cg->g.nnz; }
const orc_csr* orc_cg_graph(const orc_cg* cg) { return &cg->g; }
void orc_cg_copy(const orc_cg* cg, uint64_t* new2old, uint8_t* types, uint64_t* row, uint64_t* col) {
  const uint64_t n = cg->g.n;
  if (new2old) memcpy(new2old, cg->new2old, n * 8);
  if (types) memcpy(types, cg->types, n);
  orc_csr_copy(&cg->g, row, col);
}

/* relayout.cpp:89-169: one entry per tree vertex, (src, dst, core_edge),
 * sorted by dst; throws (here: returns -1) on non-tree shapes. */
typedef struct { uint64_t s, d, c; } ent3;
static int cmp_ent(const void* x, const void* y) {
  const uint64_t a = ((const ent3*)x)->d, b = ((const ent3*)y)->d;
  return a < b ? -1 : (a > b);
}
int64_t orc_extract_etl(const orc_cg* cg, uint64_t* src, uint64_t* dst, uint64_t* core_edge) {
  const orc_csr* g = &cg->g;
  const uint64_t n = g->n, core = cg->core;
  char* placed = calloc(n ? n : 1, 1);
  uint64_t* parent = malloc((n ? n : 1) * 8);
  uint64_t* queue = malloc((n ? n : 1) * 8);
  ent3* e = malloc((n ? n : 1) * sizeof(ent3));
  uint64_t ne = 0;
  int64_t rc = 0;
  for (uint64_t v = 0; v < n; ++v) parent[v] = ORC_NO_VERTEX;
  /* walk_tree, relayout.cpp:104-132 */
#define WALK(root_, ce_)                                                                 \
  do {                                                                                   \
    const uint64_t wroot = (root_), wce = (ce_);                                         \
    uint64_t qh = 0, qt = 0;                                                             \
    queue[qt++] = wroot;                                                                 \
    while (qh < qt && rc == 0) {                                                         \
      const uint64_t u = queue[qh++];                                                    \
      for (uint64_t k = g->row[u]; k < g->row[u + 1]; ++k) {                             \
        const uint64_t w = g->col[k];                                                    \
        if (w < core) {                                                                  \
          if (u != wroot || w != wce) {                                                \
            set_err("extract_edge_tree_list: edge tree touches the core more than once"); \
            rc = -1; break;                                                              \
          }                                                                              \
          continue;                                                                      \
        }                                                                                \
        if (!is_tree(cg->types[w])) {                                                    \
          set_err("extract_edge_tree_list: isolated-typed vertex has incident edges");   \
          rc = -1; break;                                                                \
        }                                                                                \
        if (placed[w]) {                                                                 \
          if (w != parent[u]) {                                                          \
            set_err("extract_edge_tree_list: cycle through tree vertices");              \
            rc = -1; break;                                                              \
          }                                                                              \
          continue;                                                                      \
        }                                                                                \
        placed[w] = 1; parent[w] = u;                                                    \
        e[ne].s = u; e[ne].d = w; e[ne].c = wce; ++ne;                                  \
        queue[qt++] = w;                                                                 \
      }                                                                                  \
    }                                                                                    \
  } while (0)
  for (uint64_t c = 0; c < core && rc == 0; ++c) { /* :136-151 */
    if (cg->types[c] != ORC_CE) continue;
    for (uint64_t k = g->row[c]; k < g->row[c + 1] && rc == 0; ++k) {
      const uint64_t w = g->col[k];
      if (w < core) continue;
      if (!is_tree(cg->types[w])) {
        set_err("extract_edge_tree_list: isolated-typed vertex has incident edges");
        rc = -1; break;
      }
      if (placed[w]) {
        set_err("extract_edge_tree_list: edge tree touches the core more than once");
        rc = -1; break;
      }
      placed[w] = 1; parent[w] = c;
      e[ne].s = c; e[ne].d = w; e[ne].c = c; ++ne;
      WALK(w, c);
    }
  }
  for (uint64_t v = core; v < n && rc == 0; ++v) { /* :153-159 */
    if (!is_tree(cg->types[v]) || placed[v]) continue;
    placed[v] = 1; parent[v] = v;
    e[ne].s = v; e[ne].d = v; e[ne].c = ORC_NO_VERTEX; ++ne;
    WALK(v, ORC_NO_VERTEX);
  }
#undef WALK
  if (rc == 0) { /* :161-164 */
    uint64_t tree_typed = 0;
    for (uint64_t v = 0; v < n; ++v) tree_typed += is_tree(cg->types[v]);
    if (ne != tree_typed) {
      set_err("extract_edge_tree_list: classification does not match layout");
      rc = -1;
    }
  }
  if (rc == 0) {
    qsort(e, ne, sizeof(ent3), cmp_ent); /* :166-167 */
    for (uint64_t i = 0; i < ne; ++i) {
      if (src) src[i] = e[i].s;
      if (dst) dst[i] = e[i].d;
      if (core_edge) core_edge[i] = e[i].c;
    }
    rc = (int64_t)ne;
  }
  free(placed);
  free(parent);
  free(queue);
  free(e);
  return rc;
}

/* ------------------------------------------------------------------ BFS -- */
/* bfs.cpp:50-59 */
uint64_t orc_restricted_edge_count(const orc_csr* g, uint64_t limit) {
  if (limit >= g->n) return g->nnz;
  uint64_t total = 0;
  for (uint64_t v = 0; v < limit; ++v)
    for (uint64_t k = g->row[v]; k < g->row[v + 1] && g->col[k] < limit; ++k) ++total;
  return total;
}

/* validate.cpp:77-91: textbook queue BFS. */
int orc_bfs_levels(const orc_csr* g, uint64_t root, uint64_t* level) {
  if (root >= g->n) { set_err("oracle_bfs: root out of range"); return -1; }
  uint64_t* q = malloc(g->n * 8);
  for (uint64_t v = 0; v < g->n; ++v) level[v] = ORC_UNREACHED;
  uint64_t qh = 0, qt = 0;
  q[qt++] = root;
  level[root] = 0;
  while (qh < qt) {
    const uint64_t u = q[qh++];
    for (uint64_t k = g->row[u]; k < g->row[u + 1]; ++k) {
      const uint64_t w = g->col[k];
      if (level[w] != ORC_UNREACHED) continue;
      level[w] = level[u] + 1;
      q[qt++] = w;
    }
  }
  free(q);
  return 0;
}

/* bench.cpp:217-242: splitmix64 draws modulo n, redraw degree-0 and repeats
 * while distinct eligible vertices remain. */
int orc_select_roots(const orc_csr* g, uint64_t count, uint64_t seed, uint64_t* out) {
  if (count == 0) { set_err("select_roots: count must be >= 1"); return -1; }
  uint64_t eligible = 0;
  for (uint64_t v = 0; v < g->n; ++v) eligible += deg(g, v) > 0;
  if (eligible == 0) { set_err("select_roots: graph has no vertex with degree >= 1"); return -1; }
  char* taken = calloc(g->n, 1);
  uint64_t distinct = 0, got = 0, state = seed;
  while (got < count) {
    const uint64_t v = orc_splitmix64(&state) % g->n;
    if (deg(g, v) == 0) continue;
    if (taken[v] && distinct < eligible) continue;
    if (!taken[v]) { taken[v] = 1; ++distinct; }
    out[got++] = v;
  }
  free(taken);
  return 0;
}

/* validate.cpp:151-156 */
uint64_t orc_traversed_edges(const orc_csr* g, const uint64_t* level) {
  uint64_t s = 0;
  for (uint64_t v = 0; v < g->n; ++v)
    if (level[v] != ORC_UNREACHED) s += deg(g, v);
  return s / 2;
}

static int has_edge(const orc_csr* g, uint64_t a, uint64_t b) {
  uint64_t lo = g->row[a], hi = g->row[a + 1];
  while (lo < hi) {
    const uint64_t mid = lo + (hi - lo) / 2;
    if (g->col[mid] < b) lo = mid + 1; else hi = mid;
  }
  return lo < g->row[a + 1] && g->col[lo] == b;
}

/* validate.cpp:95-158 restated against exact oracle levels. */
uint64_t orc_check_tree(const orc_csr* g, uint64_t root, const uint64_t* parent,
                        const uint64_t* level) {
  if (parent[root] != root) return root + 1;
  for (uint64_t v = 0; v < g->n; ++v) {
    const uint64_t p = parent[v];
    if ((p == ORC_NO_VERTEX) != (level[v] == ORC_UNREACHED)) return v + 1; /* rule 5 */
    if (p == ORC_NO_VERTEX || v == root) continue;
    if (p >= g->n || !has_edge(g, v, p)) return v + 1;                     /* rule 3 */
    if (level[p] + 1 != level[v]) return v + 1;                            /* rules 2, 4 */
  }
  return 0;
}

/* bfs.cpp:232-293 replayed from exact per-level counts: claimed(level) is the
 * number of core vertices at that distance and scout the sum of their full
 * degrees — both thread-count invariant — so the α/β trace is determined. */
int64_t orc_hybrid_trace(const orc_csr* g, uint64_t limit, uint64_t start, double alpha,
                         double beta, char* trace, uint64_t cap) {
  if (limit > g->n) limit = g->n;
  if (start >= limit) { set_err("hybrid_trace: start outside the core"); return -1; }
  uint64_t* level = malloc(limit * 8);
  uint64_t* q = malloc(limit * 8);
  for (uint64_t v = 0; v < limit; ++v) level[v] = ORC_UNREACHED;
  uint64_t qh = 0, qt = 0, maxl = 0;
  q[qt++] = start;
  level[start] = 0;
  while (qh < qt) {
    const uint64_t u = q[qh++];
    for (uint64_t k = g->row[u]; k < g->row[u + 1]; ++k) {
      const uint64_t w = g->col[k];
      if (w >= limit) break;
      if (level[w] != ORC_UNREACHED) continue;
      level[w] = level[u] + 1;
      if (level[w] > maxl) maxl = level[w];
      q[qt++] = w;
    }
  }
  uint64_t* cl = calloc(maxl + 2, 8);
  uint64_t* sc = calloc(maxl + 2, 8);
  for (uint64_t v = 0; v < limit; ++v)
    if (level[v] != ORC_UNREACHED) { ++cl[level[v]]; sc[level[v]] += deg(g, v); }
  uint64_t frontier = 1, scout = deg(g, start), L = 0, len = 0;
  double etc = (double)orc_restricted_edge_count(g, limit);
#define PUSH(ch) do { if (len + 1 < cap) trace[len] = (ch); ++len; } while (0)
  while (frontier > 0) {
    if ((double)scout > etc / alpha) {
      uint64_t awake = frontier, prev;
      do {
        prev = awake;
        PUSH('b');
        ++L;
        awake = cl[L];
      } while (awake > 0 && (awake >= prev || (double)awake > (double)limit / beta));
      frontier = awake;
      scout = 1;
    } else {
      etc -= (double)scout;
      PUSH('t');
      ++L;
      frontier = cl[L];
      scout = sc[L];
    }
  }
#undef PUSH
  if (cap > 0) trace[len < cap ? len : cap - 1] = 0;
  free(level); free(q); free(cl); free(sc);
  return (int64_t)len;
}

/* FNV-1a-64 over raw bytes (SURVEY.md Appendix A anchor hash). */
uint64_t orc_fnv1a64(const void* data, uint64_t len) {
  const unsigned char* p = (const unsigned char*)data;
  uint64_t h = 0xcbf29ce484222325ull;
  for (uint64_t i = 0; i < len; ++i) h = (h ^ p[i]) * 0x100000001b3ull;
  return h;
}
