/* etbfs_cuda.h — the C-ABI drop-in boundary of the B200 edge-tree BFS.
 *
 * Plain C: pointers, sizes and int status codes; no torch or C++ types.
 * Every entry point returns ETB_OK (0) or a negative status and never lets
 * a C++ exception cross the ABI; etb_last_error() holds the message, which
 * for caller errors is the reference's own message text.
 *
 * Each function names the reference interface it replaces
 * (paths relative to /root/reference/proj):
 *
 *   etb_generate_kronecker      include/etbfs/kronecker.hpp:34  generate_kronecker
 *   etb_graph_from_edges        include/etbfs/build.hpp:19      build_csr
 *   etb_graph_generate          kronecker.hpp:34 + build.hpp:19 (fused, tuples never leave HBM)
 *   etb_graph_download          include/etbfs/types.hpp:38-50   CsrGraph fields
 *   etb_classify                include/etbfs/classify.hpp:33   classify_vertices
 *   etb_peak_height             include/etbfs/classify.hpp:38   compute_peak_height
 *   etb_layout_build(_types)    include/etbfs/relayout.hpp:40   relayout_csr
 *   etb_layout_download_etl     include/etbfs/relayout.hpp:52   extract_edge_tree_list
 *   etb_bfs / etb_bfs_device    include/etbfs/et_bfs.hpp:53     et_bfs (CoreKernel::kHybrid)
 *   etb_layout_restricted_edges include/etbfs/bfs.hpp:123       restricted_edge_count
 *   etb_graph_file_read/_write  include/etbfs/io.hpp:23-24      read_graph / write_graph
 *   etb_tree_file_read/_write   include/etbfs/io.hpp:30-31      read_tree / write_tree
 *   etb_graph_degree_split      include/etbfs/preprocess.hpp:69 split_degree_aware
 *   etb_graph_levels            include/etbfs/validate.hpp:37   oracle_bfs
 *   etb_graph_validate_tree     include/etbfs/validate.hpp:46   validate_bfs_tree
 *
 * Index spaces: "original" ids are the input graph's; "relaid" ids are the
 * relayout_csr space (core block [0, core), then edge trees, then isolated
 * vertices), exactly as the reference's ClassifiedGraph.
 */
#ifndef ETBFS_CUDA_H
#define ETBFS_CUDA_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define ETB_OK 0
#define ETB_EINVAL -1   /* std::invalid_argument in the reference */
#define ETB_ERUNTIME -2 /* std::runtime_error in the reference */
#define ETB_ECUDA -3    /* CUDA / NCCL failure (no reference analogue) */
#define ETB_ENOTSUP -4  /* not available in this build */

#define ETB_NO_VERTEX UINT64_MAX /* types.hpp:13 kNoVertex */
#define ETB_UNREACHED_DEPTH (-1)

/* VertexType numbering, types.hpp:55-61 */
enum { ETB_CI = 0, ETB_CE = 1, ETB_TI = 2, ETB_TL = 3, ETB_VZ = 4 };

/* CoreKernel (et_bfs.hpp:10-16). Relaid core rows list neighbours by descending
 * degree, so every bottom-up probe is already the reference's degree-aware order
 * (in_plus first, then the descending remainder): kDegreeAware and
 * kHybridBlockSearch run the hybrid driver, kBlockSearch runs bottom-up sweeps to
 * the fixpoint with no top-down level (run_block_search, bfs.cpp:295-305). No
 * separate degree split is needed on the device. */
enum {
  ETB_KERNEL_TOP_DOWN = 0,
  ETB_KERNEL_HYBRID = 1,
  ETB_KERNEL_DEGREE_AWARE = 2,
  ETB_KERNEL_BLOCK_SEARCH = 3,
  ETB_KERNEL_HYBRID_BLOCK_SEARCH = 4
};
/* TreeReplay (et_bfs.hpp:19-22). */
enum { ETB_REPLAY_TEET = 0, ETB_REPLAY_TEOLV = 1 };

typedef struct etb_graph etb_graph;   /* device CSR, original ids */
typedef struct etb_layout etb_layout; /* device ET layout, relaid ids, BFS-ready */

typedef struct {
  uint32_t scale;      /* kronecker.hpp:12-20 KroneckerParams */
  uint64_t edgefactor;
  double a, b, c, d;
  uint64_t seed;
} etb_kron_params;

typedef struct {
  uint64_t vertex_count;
  uint64_t core_vertex_count;   /* ClassifiedGraph::core_vertex_count */
  uint64_t tree_vertex_count;   /* EdgeTreeList size */
  uint64_t isolated_count;
  uint64_t core_directed_edges; /* restricted_edge_count(graph, core) */
  uint64_t directed_edges;      /* whole relabelled graph */
  uint64_t tree_count;
  uint64_t max_tree_size;
  int64_t mh;
} etb_layout_info;

typedef struct {
  int kernel;        /* ETB_KERNEL_* */
  int replay;        /* ETB_REPLAY_* */
  double alpha;      /* HybridPolicy, bfs.hpp:19-22 */
  double beta;
} etb_bfs_options;

typedef struct {
  uint32_t levels;           /* KernelStats::levels */
  uint32_t bottom_up_levels; /* KernelStats::bottom_up_levels */
  char direction_trace[256]; /* KernelStats::direction_trace, NUL-terminated */
  uint64_t level_claims[256];
  /* device time (ns) from kernel entry to: [0] end of init, [1 + L] end of level L;
   * total_ns to the end of the tree replay (block 0's view). */
  uint64_t level_ns[256];
  uint64_t total_ns;
} etb_bfs_stats;

/* ---- library ------------------------------------------------------------ */
const char* etb_last_error(void);
int etb_version(void);
int etb_device_count(int* count);
int etb_set_device(int device);

/* ---- (1) graph construction --------------------------------------------- */
/* Writes 2 * 2^scale * edgefactor u64 (src, dst) into host out_pairs. */
int etb_generate_kronecker(const etb_kron_params* p, uint64_t* out_pairs);
int etb_graph_from_edges(uint64_t vertex_count, const uint64_t* pairs, uint64_t count,
                         etb_graph** out, uint64_t* dropped_self_loops,
                         uint64_t* dropped_duplicates);
int etb_graph_generate(const etb_kron_params* p, etb_graph** out, uint64_t* dropped_self_loops,
                       uint64_t* dropped_duplicates);
/* Upload an existing CsrGraph (row_offsets n+1 u64, cols u64; rows must be sorted,
 * symmetric and duplicate free, as every CsrGraph the reference produces). */
int etb_graph_from_csr(uint64_t vertex_count, const uint64_t* row_offsets, const uint64_t* cols,
                       etb_graph** out);
int etb_graph_info(const etb_graph* g, uint64_t* vertex_count, uint64_t* directed_edges);
/* Any output may be NULL. row_offsets: n+1 u64, cols: directed_edges u64, degrees: n u64. */
int etb_graph_download(const etb_graph* g, uint64_t* row_offsets, uint64_t* cols,
                       uint64_t* degrees);
void etb_graph_free(etb_graph* g);

/* ---- checker-side and preprocessing helpers on a device graph ------------- */
/* split_degree_aware (preprocess.hpp:69): per vertex the highest-degree
 * neighbour below `limit` (in_plus, ETB_NO_VERTEX if none; ties: smallest id)
 * and the rest by descending degree, ascending id (minus). minus_offsets (n+1)
 * is always written; in_plus (n) and minus_cols (minus_offsets[n]) may be NULL
 * (sizing call). limit = ETB_NO_VERTEX keeps every neighbour. */
int etb_graph_degree_split(const etb_graph* g, uint64_t limit, uint64_t* in_plus,
                           uint64_t* minus_offsets, uint64_t* minus_cols);
/* oracle_bfs (validate.hpp:37): BFS levels from root (ETB_NO_VERTEX = unreached),
 * a plain level-synchronous device BFS independent of the ET-BFS kernels. */
int etb_graph_levels(const etb_graph* g, uint64_t root, uint64_t* levels);
/* validate_bfs_tree (validate.hpp:46) of a host parent array (n u64, original
 * ids of g) rooted at root: counts[0] = 1 if every rule holds, counts[r] =
 * failures of rule r (1..5; rule 2: bad parent chains), counts[6] reached
 * vertices, counts[7] traversed edges (half the reached degree sum). For each
 * rule the first (up to 25) failures in the reference's order go to
 * where[(r-1)*25 + i] (rule 4: the edge's smaller endpoint; rule 2: bit 62 set
 * for a dead end, clear for a cycle) with first_count[r-1] of them; both may
 * be NULL. */
int etb_graph_validate_tree(const etb_graph* g, uint64_t root, const uint64_t* parent,
                            uint64_t* counts, uint64_t* where, uint32_t* first_count);

/* ---- (2) edge-tree preprocessing ----------------------------------------- */
/* types_out (n u8, may be NULL); counts_out (5 u64 CI/CE/TI/TL/VZ, may be NULL). */
int etb_classify(const etb_graph* g, int64_t mh, uint8_t* types_out, uint64_t* counts_out);
int etb_peak_height(const etb_graph* g, uint64_t* peak_height);
/* classify_vertices(g, mh) + relayout_csr + extract_edge_tree_list, on device. */
int etb_layout_build(const etb_graph* g, int64_t mh, etb_layout** out);
/* relayout_csr(g, types, mh) with caller-supplied types (host, n u8). */
int etb_layout_build_types(const etb_graph* g, const uint8_t* types, int64_t mh,
                           etb_layout** out);
int etb_layout_info_get(const etb_layout* L, etb_layout_info* info);
/* new2old / old2new (n u64), types (n u8); any may be NULL. */
int etb_layout_download_maps(const etb_layout* L, uint64_t* new2old, uint64_t* old2new,
                             uint8_t* types);
/* The whole relabelled CSR (relabel_graph, build.cpp:144-166): row_offsets n+1,
 * cols info.directed_edges, both u64. */
int etb_layout_download_graph(const etb_layout* L, uint64_t* row_offsets, uint64_t* cols);
/* EdgeTreeList (relayout.hpp:52): tree_vertex_count entries sorted by dst;
 * core_edge uses ETB_NO_VERTEX for whole-component trees. */
int etb_layout_download_etl(const etb_layout* L, uint64_t* src, uint64_t* dst,
                            uint64_t* core_edge);
int etb_layout_restricted_edges(const etb_layout* L, uint64_t* count);
void etb_layout_free(etb_layout* L);

/* ---- (3)+(4) traversal ----------------------------------------------------- */
/* et_bfs from relaid `start`, results stay in HBM (the timed hot path). opts may be NULL
 * (kHybrid, kTeet, α=14, β=24). stats may be NULL (then no device->host copy). */
int etb_bfs_device(etb_layout* L, uint64_t start, const etb_bfs_options* opts,
                   etb_bfs_stats* stats);
/* et_bfs with host outputs (the reference-facing call): depth (n i32, -1 unreached)
 * and/or parent (n u64, ETB_NO_VERTEX unreached), relaid ids. Every host-output
 * call copies only the live prefix [0, core + tree) of the relaid id space over
 * PCIe; the isolated vertices that close it are unreached in every result (but
 * for an isolated start), so their range of the host arrays is filled by host
 * threads while the DMA runs. The arrays come back complete either way. */
int etb_bfs(etb_layout* L, uint64_t start, const etb_bfs_options* opts, int32_t* depth_out,
            uint64_t* parent_out, etb_bfs_stats* stats);
/* et_bfs with compact host outputs: parent (n u32, UINT32_MAX unreached) and/or
 * depth (n i32). The BfsTree content at half the bytes of etb_bfs. */
int etb_bfs_compact(etb_layout* L, uint64_t start, const etb_bfs_options* opts,
                    int32_t* depth_out, uint32_t* parent_out);
/* Device pointer to the last result: n interleaved {depth (i32, -1 unreached),
 * parent (u32, UINT32_MAX unreached)} pairs, relaid ids. */
int etb_result_device_ptr(etb_layout* L, uint32_t** dp);
/* The last result in ORIGINAL ids, as the reference's translate_tree +
 * tree_levels give it (validate.hpp:48-50): levels (n u64, ETB_NO_VERTEX =
 * kUnreached) and/or parent (n u64, ETB_NO_VERTEX unreached); either may be NULL. */
int etb_result_download_original(etb_layout* L, uint64_t* levels, uint64_t* parent);
/* Multi-GPU: after the caller wrote every rank's owned result slices (the ranges
 * of etb_layout_partition_bounds) into this rank's result buffer
 * (etb_result_device_ptr), the result is whole: etb_result_validate and
 * etb_result_traversed_edges then treat it as a single-device result. The next
 * traversal clears the mark. */
int etb_result_mark_assembled(etb_layout* L);
/* Copy the last result to host as compact i32 depth / u32 parent (UINT32_MAX unreached). */
int etb_result_download(etb_layout* L, int32_t* depth, uint32_t* parent);
/* ½ Σ full degree over reached vertices of the last result (validate.cpp:151-156). */
int etb_result_traversed_edges(etb_layout* L, uint64_t* te);
/* ---- (5) 1D core partition ------------------------------------------------ */
/* Split the core into `parts` partitions run by one kernel on this device (the
 * multi-GPU algorithm with the peer exchange in local memory); parts <= 1
 * restores the single-partition kernel. */
int etb_layout_partition(etb_layout* L, uint32_t parts);
/* The scope of the partitioned kernel's exchange (fences, counter atomics and
 * barrier polls): 1 = system scope, as between GPUs (set by etb_mp_export);
 * 0 = device scope, as between partitions sharing one GPU (the default of
 * etb_layout_partition). Lets the one-GPU emulation run the multi-GPU code path. */
int etb_layout_partition_scope(etb_layout* L, int system_scope);
/* The partition owning every relaid vertex among `parts` (owner: n u32): core
 * vertex v belongs to partition (v >> 8) mod parts (256-vertex blocks dealt
 * round robin over the degree-sorted core, as the paper's SRRS), a tree vertex
 * to its anchor's partition, component trees and isolated vertices to the
 * last one. */
int etb_layout_partition_owner(const etb_layout* L, uint32_t parts, uint32_t* owner);
/* One GPU per process: rank `rank` of `world` builds its partition and exports
 * an opaque blob (etb_mp_blob_size() bytes); after all blobs are exchanged
 * (ordered by rank) etb_mp_connect opens the peers' exchange blocks over CUDA
 * IPC. Every rank then calls etb_bfs_device with the same start; the kernels
 * synchronise through peer memory. etb_result_traversed_edges then returns this
 * rank's partial count. */
int etb_mp_blob_size(void);
int etb_mp_export(etb_layout* L, uint32_t world, uint32_t rank, void* blob_out);
int etb_mp_connect(etb_layout* L, const void* blobs);

/* Page-lock a caller buffer so result downloads run at full link speed. */
int etb_host_register(void* ptr, uint64_t bytes);
int etb_host_unregister(void* ptr);

/* validate_bfs_tree (validate.hpp:13-46) on the device over the whole graph for the
 * last result from relaid `start`: counts[0..4] = violations of rules 1..5 (root
 * parent, chains, parent edge, level span, reached set), counts[5] = reached
 * vertices. Rules 1-5 together imply every depth is the exact BFS distance. A
 * layout shares ownership of the graph it was built from, so etb_graph_free may
 * come first. */
int etb_result_validate(etb_layout* L, uint64_t start, uint64_t* counts);

/* Diagnostics: one traversal from `start` recording, per level and CTA, the
 * device time (ns since kernel entry) at which the CTA finished its step:
 * out[level * grid + cta] (cap entries). */
int etb_debug_block_stamps(etb_layout* L, uint64_t start, uint64_t* out, uint64_t cap,
                           uint32_t* grid, uint32_t* levels);
/* Diagnostics (libraries built with -DETB_WARP_STAMPS; zeros otherwise): for
 * the top-down level that claims depth `depth`, per warp (8 entries, physical
 * warp order): [0] ns since kernel entry at the warp's first chunk, clock64
 * cycles from then to [1] its list position known, [2] columns loaded, [3]
 * visited words loaded, [4] claim atomics returned, [5] chunk done; [6] chunk
 * index, [7] 1 if the chunk lies in one row. */
int etb_debug_warp_stamps(etb_layout* L, uint64_t start, int32_t depth, uint64_t* out,
                          uint64_t cap, uint32_t* nwarps);
/* Diagnostics: the raw globaltimer stamps of the last stats run ([0] entry, [1]
 * init end, [2 + L] level L end, [128 + L] conversion before level L end,
 * [255] replay end) and, at [192 + L], top-down level L's frontier edge count. */
int etb_debug_phase_stamps(etb_layout* L, uint64_t* out256);
/* Diagnostics of a -DETB_MISS_CYCLES build (zeros otherwise), 320 counters per
 * depth d: [d % 64] warp cycles in bottom-up steps, [64 + d % 64] in their
 * deferred-miss resolution, [128 + d % 32] deferred vertices, [160 + d % 32]
 * rows scanned past the second neighbour, [192 + d % 32] rows scanned by the
 * whole warp, [224 + d % 32] its 32-edge rounds, [256 + d % 64] the slowest
 * warp's miss-resolution cycles; reset != 0 clears them. */
int etb_debug_diag(etb_layout* L, uint64_t* out320, int reset);
/* Diagnostics (libraries built with -DETB_DEBUG_CHECKS; 0 otherwise): the
 * source line of the first failed device bounds check since the last call. */
int etb_debug_check_line(uint32_t* line);
/* Diagnostics: median event-timed duration (us) of an empty kernel launched
 * like the traversal (same grid, block, shared memory, cooperative). */
int etb_debug_launch_floor(etb_layout* L, int iters, double* empty_us);

/* ---- measurement ---------------------------------------------------------- */
/* Times etb_bfs_device per start with CUDA events on the layout's stream, after
 * `warmup` untimed runs; flush_l2 != 0 writes a >L2 buffer between roots (outside
 * the timed events). ms_out[i] per start. kernel_ms_out (may be NULL) receives the
 * BFS kernel's own event-timed duration per start. */
int etb_time_roots(etb_layout* L, const uint64_t* starts, uint64_t count, int warmup,
                   int flush_l2, const etb_bfs_options* opts, double* ms_out,
                   double* kernel_ms_out);

/* Wall-clock time (ms) of each etb_bfs_device call from `starts` up to its
 * completion (host timer around launch + stream synchronise): the call's launch
 * latency and start-side walk included, no L2 flush, no host copy. */
int etb_time_roots_wall(etb_layout* L, const uint64_t* starts, uint64_t count, int warmup,
                        const etb_bfs_options* opts, double* ms_out);

/* Algorithmic work of the traversal from relaid `start` (re-run with stats):
 * the bytes a direction-optimizing BFS with this root's level sequence must
 * move (work.cu: top-down levels read the frontier rows, bottom-up levels the
 * first-neighbour entry of every unvisited core vertex plus the probes up to
 * its first frontier neighbour, results written once, core-sized bitmaps once
 * per level, the tree replay, the unreached fill and the state reset).
 * levels (4 x 64 u64, may be NULL): per level frontier-or-unvisited vertices,
 * core columns read, claims, bottom-up first-probe misses; bytes (65 u64, may
 * be NULL): per level, then the replay/fill/reset tail; nlevels: levels run;
 * trace (65 chars, may be NULL): their directions; total_bytes: the sum. */
int etb_result_work(etb_layout* L, uint64_t start, const etb_bfs_options* opts,
                    uint64_t* levels, uint64_t* bytes, uint32_t* nlevels, char* trace,
                    uint64_t* total_bytes);

/* ---- step / driver layer (bfs.hpp:66-120) on caller-held state ------------ */
/* op: 0 top_down_step, 1 bottom_up_step, 2 degree_aware_step, 3 block_search_step,
 * 4 run_top_down, 5 run_hybrid (classic), 6 run_hybrid (degree-aware), 7 run_hybrid
 * (block-search), 8 run_block_search. visited/current/next: ceil(n/64) u64 bitmap
 * words, parent: n u64, all host, updated in place. in_plus / minus_offsets /
 * minus_cols: the degree split (ops 2, 3, 6, 7, 8; else NULL). stats (6 u64,
 * added to): claimed, scout, probes, skipped blocks, levels, bottom-up levels;
 * trace (drivers, may be NULL): one 't'/'b' per level, NUL-terminated within
 * trace_cap. */
int etb_steps_run(const etb_graph* g, int op, uint64_t limit, uint64_t* visited,
                  uint64_t* current, uint64_t* next, uint64_t* parent, const uint64_t* in_plus,
                  const uint64_t* minus_offsets, const uint64_t* minus_cols, double alpha,
                  double beta, uint64_t* stats, char* trace, uint64_t trace_cap);

/* teet / teolv (et_bfs.hpp:30-37) on the current device: entry i sets
 * parent[dst[i]] = src[i] if its guard (core_edge[i], or src[i] when leaves_only)
 * is set in the visited words and parent[dst[i]] is ETB_NO_VERTEX. */
int etb_tree_replay(int leaves_only, const uint64_t* src, const uint64_t* dst,
                    const uint64_t* core_edge, uint64_t count, const uint64_t* visited_words,
                    uint64_t words, uint64_t* parent, uint64_t n);

/* ---- graph and parent-tree files (io.hpp:9-45, io.cpp:47-181) ------------- */
/* Byte-identical to the reference's ETG1 / text graph and ETT1 tree files, with
 * its validation order and messages (runtime errors name the path and the byte
 * offset or line). Host-only: no GPU needed. */
#define ETB_FORMAT_BINARY 0 /* GraphFormat::kBinary (ETG1) */
#define ETB_FORMAT_TEXT 1   /* GraphFormat::kText */
typedef struct etb_edgefile etb_edgefile; /* a loaded edge list (host memory) */

int etb_graph_file_read(const char* path, int format, etb_edgefile** out);
/* Any output may be NULL; *pairs stays valid until etb_graph_file_free. */
int etb_graph_file_info(const etb_edgefile* f, uint64_t* vertex_count, uint64_t* edge_count,
                        const uint64_t** pairs);
void etb_graph_file_free(etb_edgefile* f);
int etb_graph_file_write(const char* path, int format, uint64_t vertex_count,
                         const uint64_t* pairs, uint64_t edge_count);
/* A graph file straight to a device CSR (read + etb_graph_from_edges). */
int etb_graph_from_file(const char* path, int format, etb_graph** out);
int etb_tree_file_write(const char* path, uint64_t vertex_count, uint64_t root,
                        const uint64_t* parent);
/* parent == NULL: only *vertex_count / *root (either may be NULL); else cap >= n. */
int etb_tree_file_read(const char* path, uint64_t* vertex_count, uint64_t* root,
                       uint64_t* parent, uint64_t cap);

#ifdef __cplusplus
}
#endif
#endif /* ETBFS_CUDA_H */
