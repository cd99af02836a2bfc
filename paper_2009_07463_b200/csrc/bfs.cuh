// Persistent ET-BFS kernel interface (bfs.cu).
#pragma once

#include "internal.cuh"

namespace etb {

// Chunk of a core row one warp expands in a top-down step.
constexpr uint32_t kTdChunk = 128;
// Start-tree patch entries carried inline in the kernel parameters.
constexpr int kInlinePatch = 4;

struct BfsParams {
  // core graph (relaid ids)
  const uint64_t* crow;
  const uint32_t* ccol;
  const uint32_t* cfirst;
  const uint32_t* csecond;  // second core neighbour, bit 31: last of its row (kNone32: none)
  const uint2* cthird;      // {third, fourth} core neighbours, same flags
  const uint32_t* degn;  // full degree (scout, bfs.cpp:80)
  const uint2* cmeta;    // per core vertex {core degree, full degree}
  uint64_t reachable;  // core vertices in the start's core component (set per root)
  uint32_t nc;
  uint32_t nwords;       // ceil(nc / 32)
  // edge trees
  const uint32_t* tsrc;
  const uint32_t* tanchor;
  const uint32_t* tdepth;
  uint32_t nt;
  // traversal state
  uint32_t* visited;
  uint32_t* fb0;
  uint32_t* fb1;
  uint32_t* fb2;
  uint32_t* qv0;  // frontier lists (vertex ids) ...
  uint32_t* qv1;
  uint64_t* qp0;  // ... and the exclusive prefix of their row-chunk counts
  uint64_t* qp1;
  unsigned long long* ctr;  // 4 level slots x 4 + conversion counters
  unsigned long long* bar;  // grid barrier counter (monotonic)
  // The other half of the double-buffered visited / fb0 / fb1 / ctr: this
  // traversal cleans it for the next one, so a traversal starts on clean state
  // without an init pass and its grid barrier.
  uint32_t* visited_next;
  uint32_t* fb0_next;
  uint32_t* fb1_next;
  uint32_t* fb2_next;
  unsigned long long* ctr_next;
  // outputs (relaid ids, all n vertices)
  uint2* dp;  // {depth (i32 bits, -1 unreached), parent (kNone32 unreached)} per vertex
  // per call
  uint32_t start;         // core vertex the core BFS starts at, kNone32 for none
  int32_t base_depth;     // depth of `start`
  uint32_t start_parent;  // parent of `start`
  uint32_t skip_lo, skip_hi;  // tree range filled by the start-side walk
  const uint32_t* patch;  // (vertex, depth, parent) triples
  uint32_t npatch;
  // Small patches travel in the launch parameters (no host-to-device copy in
  // the per-root sequence); ipatch[3 k .. 3 k + 2] for k < nipatch.
  uint32_t nipatch;
  uint32_t ipatch[3 * kInlinePatch];
  double alpha, beta, edges_to_check;
  double emit_limit;  // top-down levels with scout >= this skip work-item emission
  // A level the α/β rule runs top-down is executed as a frontier-restricted
  // bottom-up sweep when its frontier edges exceed td_as_bu x the unvisited core
  // vertices (0 = never; hybrid drivers only, CoreKernel::kTopDown stays
  // top-down): the claimed set — the unvisited core vertices with a frontier
  // neighbour — is the same, so depths, claims, scout and the α/β sequence are
  // the reference's; only the GPU cost differs.
  double td_as_bu;
  // Large-core kernel: a list-less top-down level whose frontier edges reach
  // split_ratio x the unvisited core vertices (0 = never) is executed split:
  // the frontier's hubs (relaid ids < split_bound) bottom-up, every row scan
  // ending at the first neighbour >= split_bound, the other frontier vertices
  // top-down from a filtered list. Same claimed set, depths and α/β sequence.
  double split_ratio;
  uint32_t split_bound;
  // The split level's halves: 0 = bottom-up, grid barrier, top-down; 1..32 = that
  // many warps per CTA run the top-down half first, beside the others' bottom-up
  // runs, then join them; 33.. = every warp goes from the bottom-up runs straight
  // to the top-down chunks; 0xFFFF = 16 or the latter by the tail's edge count
  uint32_t split_tdw;
  // small-core kernel: list-less top-down levels with at least this many
  // frontier edges claim atomic-free and count afterwards (as the large-core
  // kernel's); smaller ones claim with returning atomics
  double small_mode3_edges;
  int top_down_only;   // CoreKernel::kTopDown
  int bottom_up_only;  // CoreKernel::kBlockSearch: bottom-up levels to fixpoint
  // stats (may be null)
  char* trace;
  unsigned long long* level_claims;
  unsigned long long* bstamp;  // diagnostics: [level][block] step-end globaltimer, or null
  unsigned long long* wstamp;  // diagnostics (ETB_WARP_STAMPS builds): per-warp chunk phases
  int32_t wdepth;              //   of the top-down level claiming this depth
  uint32_t* nlevels;
};

struct BfsState {
  uint64_t n = 0;
  // visited / fb0 / fb1 / fb2, two halves each, in one allocation (one L2
  // access-policy window can cover the whole per-root bitmap state)
  DevBuf<uint32_t> bits;
  uint32_t* visited() const { return bits.get(); }
  uint32_t* fb0() const { return bits.get() + 2 * words; }
  uint32_t* fb1() const { return bits.get() + 4 * words; }
  uint32_t* fb2() const { return bits.get() + 6 * words; }
  DevBuf<uint32_t> qv0, qv1;
  DevBuf<uint64_t> qp0, qp1;
  DevBuf<unsigned long long> ctr, bar;
  DevBuf<uint2> dp;          // interleaved result: one 8-byte store per claim
  DevBuf<int32_t> tmp_depth;  // de-interleaved staging for host downloads
  DevBuf<uint32_t> tmp_parent;
  DevBuf<uint64_t> tmp_parent64;
  DevBuf<char> trace;
  DevBuf<unsigned long long> level_claims;
  DevBuf<uint32_t> nlevels;
  DevBuf<uint32_t> patch;
  HostBuf<uint32_t> h_patch;
  cudaEvent_t patch_done = nullptr;  // the pinned patch may be rewritten after this
  ~BfsState() {
    if (patch_done) cudaEventDestroy(patch_done);
  }
  uint32_t last_isolated = kNone32;  // isolated start to reset on the next call
  int grid = 0, block = 0;
  uint32_t parity = 0;  // which half of visited / fb0 / fb1 / ctr the next launch uses
  uint64_t words = 0;   // per half
  bool l2_window = false;  // the bitmap state has a persisting L2 access-policy window
  bool has_result = false;
  bool assembled = false;  // multi-GPU: the caller merged every rank's owned slices into dp
  uint64_t last_start = ~uint64_t{0};
};

void bfs_state_init(const DevLayout& L, BfsState& S, cudaStream_t s);
// persisting L2 window over one allocation on a stream (false: off / too large)
bool set_l2_window(cudaStream_t s, void* base, size_t bytes);
void empty_launch(const BfsState& S, cudaStream_t s);  // launch-cost floor (diagnostics)
void bfs_launch(const BfsParams& p, BfsState& S, cudaStream_t s);
// -DETB_MISS_CYCLES diagnostics: bottom-up step / miss-resolution warp cycles per depth
void debug_diag(uint64_t* out320, bool reset, cudaStream_t s);
// Fills depth/parent of the start's tree on the host (traverse_return_core_edge,
// et_bfs.cpp:34-57) and returns the core vertex to start from (kNone32 if the
// start's component is a pure tree or the start is isolated).
void bfs_prepare_start(const DevLayout& L, BfsState& S, uint64_t start, BfsParams& p,
                       cudaStream_t s);
void bfs_fill_params(const DevLayout& L, BfsState& S, BfsParams& p);
unsigned debug_check_line();  // checked builds: first failed device check's line

// work.cu: the algorithmic work of the traversal whose result is dp, from its
// depths and the direction trace of its nl levels (see work.cu): levels[4 L + k]
// counters, bytes[L] per level, bytes[nl] the replay / fill / reset tail;
// returns the total bytes.
uint64_t result_work(const DevLayout& L, const uint2* dp, const char* trace, int nl,
                     uint64_t* levels, uint64_t* bytes, cudaStream_t s);

}  // namespace etb
