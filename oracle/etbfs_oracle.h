/* TEST INFRASTRUCTURE ONLY — the CPU checker, never the thing measured or shipped.
 *
 * Plain-C restatement of the reference's hot path (arXiv 2009.07463, `etbfs`
 * library under /root/reference/proj). Each function cites the reference
 * file:line it restates. Parity of this restatement is pinned against the
 * compiled reference (oracle/_ref, tests/golden/ fixtures made by
 * tests/golden/make_golden.py); see tests/test_oracle.py.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may
 * load this library.
 */
#ifndef ETBFS_ORACLE_H
#define ETBFS_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define ORC_NO_VERTEX (~(uint64_t)0)
#define ORC_UNREACHED (~(uint64_t)0)

/* VertexType numbering (types.hpp:55-61). */
enum { ORC_CI = 0, ORC_CE = 1, ORC_TI = 2, ORC_TL = 3, ORC_VZ = 4 };

typedef struct {
  uint64_t n;
  uint64_t nnz;       /* directed edge slots */
  uint64_t* row;      /* n + 1 */
  uint64_t* col;      /* nnz, ascending per row */
} orc_csr;

typedef struct {
  orc_csr g;          /* relabelled graph */
  uint64_t* new2old;
  uint64_t* old2new;
  uint8_t* types;     /* by new id */
  uint64_t core;
  int64_t mh;
} orc_cg;

const char* orc_last_error(void);

/* rng.hpp:10-20 */
uint64_t orc_splitmix64(uint64_t* state);
double orc_uniform01(uint64_t* state);

/* kronecker.cpp:23-69. out_pairs holds 2 * 2^scale * ef u64 (src, dst). */
int orc_generate_kronecker(uint32_t scale, uint64_t ef, double a, double b, double c, double d,
                           uint64_t seed, uint64_t* out_pairs);

/* build.cpp:21-87 */
orc_csr* orc_build_csr(uint64_t n, const uint64_t* pairs, uint64_t count, uint64_t* self_loops,
                       uint64_t* dups);
void orc_csr_free(orc_csr* g);
uint64_t orc_csr_n(const orc_csr* g);
uint64_t orc_csr_nnz(const orc_csr* g);
void orc_csr_copy(const orc_csr* g, uint64_t* row, uint64_t* col);

/* classify.cpp:10-61 (exact Gauss-Seidel sweep). Returns productive rounds
 * (compute_peak_height when mh == -1), or -1 on error. */
int64_t orc_classify(const orc_csr* g, int64_t mh, uint8_t* types);

/* relayout.cpp:25-87 + build.cpp:133-166 */
orc_cg* orc_relayout(const orc_csr* g, const uint8_t* types, int64_t mh);
void orc_cg_free(orc_cg* cg);
uint64_t orc_cg_core(const orc_cg* cg);
uint64_t orc_cg_nnz(const orc_cg* cg);
void orc_cg_copy(const orc_cg* cg, uint64_t* new2old, uint8_t* types, uint64_t* row, uint64_t* col);
const orc_csr* orc_cg_graph(const orc_cg* cg);

/* relayout.cpp:89-169. Returns the entry count (sorted by dst) or -1 with
 * orc_last_error() set to the reference's error message. Arrays may be NULL
 * to query the count. */
int64_t orc_extract_etl(const orc_cg* cg, uint64_t* src, uint64_t* dst, uint64_t* core_edge);

/* bfs.cpp:50-59 */
uint64_t orc_restricted_edge_count(const orc_csr* g, uint64_t limit);

/* validate.cpp:77-91 */
int orc_bfs_levels(const orc_csr* g, uint64_t root, uint64_t* levels);

/* bench.cpp:217-242 */
int orc_select_roots(const orc_csr* g, uint64_t count, uint64_t seed, uint64_t* out);

/* validate.cpp:151-156: half the degree sum of reached vertices. */
uint64_t orc_traversed_edges(const orc_csr* g, const uint64_t* levels);

/* Parent-tree check against oracle levels (validate.cpp:95-158 rules 1, 3, 5 plus
 * level[parent] == level - 1, which implies rules 2 and 4 given exact levels).
 * parent uses ORC_NO_VERTEX for unreached. Returns 0 when valid, else the first
 * offending vertex + 1. */
uint64_t orc_check_tree(const orc_csr* g, uint64_t root, const uint64_t* parent,
                        const uint64_t* levels);

/* The α/β direction trace run_hybrid (bfs.cpp:232-293) takes over the core
 * [0, limit) of a relaid graph, given per-level claimed counts and scouts.
 * Computed from an oracle BFS restricted to [0, limit) seeded at `start`.
 * Writes a NUL-terminated string of 't'/'b'; returns its length. */
int64_t orc_hybrid_trace(const orc_csr* g, uint64_t limit, uint64_t start, double alpha,
                         double beta, char* trace, uint64_t cap);

/* FNV-1a-64 over raw bytes (Appendix A anchors). */
uint64_t orc_fnv1a64(const void* data, uint64_t len);

#ifdef __cplusplus
}
#endif
#endif
