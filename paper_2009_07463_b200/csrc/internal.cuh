// Internal device data structures shared by the kernels and the C-ABI.
#pragma once

#include <memory>
#include <string>
#include <vector>

#include "../../include/etbfs_cuda.h"
#include "common.cuh"

namespace etb {

// CsrGraph (types.hpp:38-50) in HBM with 32-bit column ids: n <= 2^32 - 2.
struct DevGraph {
  uint64_t n = 0;
  uint64_t nnz = 0;       // directed slots
  DevBuf<uint64_t> row;   // n + 1
  DevBuf<uint32_t> col;   // nnz, ascending per row
  DevBuf<uint32_t> deg;   // n
};

// Generated / uploaded tuples -> CSR (build.cpp:21-87). Input tuples are given
// either as device u32 (src,dst) arrays or produced by the generator directly
// into the sort keys.
void build_csr_from_device_tuples(uint64_t n, const uint32_t* src, const uint32_t* dst,
                                  uint64_t count, DevGraph& out, uint64_t* self_loops,
                                  uint64_t* dups, cudaStream_t s);
void build_csr_from_generator(const etb_kron_params& p, DevGraph& out, uint64_t* self_loops,
                              uint64_t* dups, cudaStream_t s);
// Host u64 pairs (validated by the caller) -> device CSR, chunked upload.
void build_csr_from_host_pairs(uint64_t n, const uint64_t* pairs, uint64_t count, DevGraph& out,
                               uint64_t* self_loops, uint64_t* dups, cudaStream_t s);
// Generator into device u32 tuple arrays (count = 2^scale * ef).
void kron_generate_tuples(const etb_kron_params& p, uint64_t first, uint64_t count, uint32_t* src,
                          uint32_t* dst, cudaStream_t s);
void kron_generate_pairs64(const etb_kron_params& p, uint64_t first, uint64_t count,
                           uint64_t* pairs, cudaStream_t s);
void kron_validate(const etb_kron_params& p);

// classify_vertices (classify.cpp:10-61): device u8 types in original ids.
void classify_device(const DevGraph& g, int64_t mh, DevBuf<uint8_t>& type, uint64_t counts[5],
                     uint64_t* productive_rounds, cudaStream_t s);

// The BFS-ready layout (relayout_csr + extract_edge_tree_list), relaid ids.
struct DevLayout {
  uint64_t n = 0, nc = 0, nt = 0, nz = 0;
  int64_t mh = -1;
  uint64_t ecore = 0;            // restricted_edge_count(graph, core)
  uint64_t nnz_full = 0;         // directed edges of the whole graph
  uint64_t tree_count = 0, max_tree = 0;
  DevBuf<uint32_t> new2old, old2new;  // n
  DevBuf<uint8_t> type;               // n, relaid
  DevBuf<uint32_t> degn;              // n, full degree by relaid id
  // core-only CSR (the core prefix of every core row of the relabelled graph)
  DevBuf<uint64_t> crow;   // nc + 1
  DevBuf<uint32_t> ccol;   // ecore
  DevBuf<uint32_t> cfirst; // nc: first (highest-degree) core neighbour or kNone32
  DevBuf<uint32_t> csecond; // nc: second core neighbour | bit 31 if it ends the row, or kNone32
  DevBuf<uint2> cthird;     // nc: {third, fourth} core neighbours, same flags
  DevBuf<uint2> cmeta;     // nc: {core degree, full degree} — one load per claim
  // connected components of the core graph: per core vertex, the size of its
  // component (host copy; a traversal ends once the start's component is
  // exhausted, as once the whole core is)
  std::vector<uint32_t> h_comp_size;
  // edge-tree arrays, index t - nc for t in [nc, nc + nt)
  DevBuf<uint32_t> tsrc;    // tree parent (CE for attached roots, self for component roots)
  DevBuf<uint32_t> tanchor; // CE, or kNone32 for whole-component trees
  DevBuf<uint32_t> tdepth;  // distance to the CE (attached) or to the root (component)
  // host copies for the start-in-tree walk (et_bfs.cpp:34-57)
  std::vector<uint32_t> h_tsrc, h_tdepth, h_tanchor, h_tree_start;
  // The source graph (the on-demand full relabelled CSR, the validator): shared
  // ownership, so freeing the graph handle first keeps it alive for the layout.
  std::shared_ptr<const DevGraph> src_graph;
};

void build_layout(const DevGraph& g, const uint8_t* type_dev, int64_t mh, DevLayout& L,
                  cudaStream_t s);
// Whole relabelled CSR (relabel_graph, build.cpp:144-166) into device buffers.
void build_full_relabelled(const DevLayout& L, DevBuf<uint64_t>& row, DevBuf<uint32_t>& col,
                           cudaStream_t s);

// validate_bfs_tree rules 1-5 on the device for a relaid {depth, parent} result:
// out[0..4] = violations of rules 1..5, out[5] = reached vertices.
void validate_result(const DevLayout& L, const uint2* dp, uint64_t root, uint64_t out[6],
                     cudaStream_t s);

// CUB wrappers (cub_ops.cu) — library sorts/scans used only in preprocessing.
void sort_keys_u64(DevBuf<uint64_t>& keys, DevBuf<uint64_t>& alt, uint64_t count, int end_bit,
                   cudaStream_t s);  // result left in `keys`
void sort_pairs_u64_u32(DevBuf<uint64_t>& keys, DevBuf<uint64_t>& kalt, DevBuf<uint32_t>& vals,
                        DevBuf<uint32_t>& valt, uint64_t count, int end_bit, cudaStream_t s);
uint64_t unique_u64(const uint64_t* in, uint64_t* out, uint64_t count, cudaStream_t s);
void exclusive_scan_u64(const uint64_t* in, uint64_t* out, uint64_t count, cudaStream_t s);
void exclusive_scan_u32_to_u64(const uint32_t* in, uint64_t* out, uint64_t count, cudaStream_t s);
uint64_t select_flagged_u32(const uint32_t* in, const uint8_t* flags, uint32_t* out, uint64_t count,
                            cudaStream_t s);
uint64_t reduce_sum_u64(const uint64_t* in, uint64_t count, cudaStream_t s);
void inclusive_max_scan_u32(const uint32_t* in, uint32_t* out, uint64_t count, cudaStream_t s);

// Scratch device counter helpers.
uint64_t read_u64(const uint64_t* dev, cudaStream_t s);

// graph_tools.cu: split_degree_aware / oracle_bfs / validate_bfs_tree on an
// uploaded graph (host outputs; h_minus may be null to size it from h_moff[n]).
void graph_degree_split(const DevGraph& g, uint64_t limit, uint64_t* h_in_plus, uint64_t* h_moff,
                        uint64_t* h_minus, cudaStream_t s);
void graph_levels(const DevGraph& g, uint64_t root, DevBuf<uint32_t>& lvl, cudaStream_t s);
// out[r] = failures of rule r (1..5; rule 2: bad chain representatives),
// out[6] reached, out[7] traversed edges; first[r] = sorted failure keys.
void graph_validate_tree(const DevGraph& g, uint64_t root, const uint64_t* h_parent,
                         uint64_t out[8], std::vector<uint64_t> first[6], cudaStream_t s);

// steps.cu: the reference's step / driver layer on caller state (host words and
// parents in, out). ops 0-3 steps (td, bu, degree-aware, block-search), 4
// run_top_down, 5-7 run_hybrid (classic, degree-aware, block-search), 8
// run_block_search; out = claimed, scout, probes, skipped blocks, levels,
// bottom-up levels.
void step_run(const DevGraph& g, int op, uint64_t limit, uint64_t* h_vis, uint64_t* h_cur,
              uint64_t* h_nxt, uint64_t* h_parent, const uint64_t* h_in_plus,
              const uint64_t* h_moff, const uint64_t* h_minus, double alpha, double beta,
              uint64_t out[6], std::string* trace, cudaStream_t s);

// steps.cu: teet / teolv (leaves_only) over a host edge tree list, visited
// words and parents.
void tree_replay_run(int leaves_only, const uint64_t* h_src, const uint64_t* h_dst,
                     const uint64_t* h_ce, uint64_t count, const uint64_t* h_vis, uint64_t words,
                     uint64_t* h_parent, uint64_t n, cudaStream_t s);

}  // namespace etb
