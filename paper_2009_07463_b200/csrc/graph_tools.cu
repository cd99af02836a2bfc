// Device versions of the reference's checker-side and preprocessing helpers that
// callers reach through the public API (not the timed path):
//   degree split      split_degree_aware   proj/src/preprocess.cpp:16-60
//   reference levels  oracle_bfs           proj/src/validate.cpp:77-91
//   tree validation   validate_bfs_tree    proj/src/validate.cpp:95-158
// on an uploaded CsrGraph (etb_graph). Each is a few plain kernels plus CUB
// sorts; the validator derives levels from the parent chains by pointer
// jumping instead of a sequential walk.
#include <algorithm>
#include <vector>

#include "internal.cuh"

namespace etb {
namespace {

constexpr uint64_t kNone64 = ~uint64_t{0};

#define GRID_LOOP(i, n)                                                        \
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < (n); \
       i += (uint64_t)gridDim.x * blockDim.x)

// ---- degree split -----------------------------------------------------------
// cnt[v] = neighbours of v below `limit` (rows ascend: a prefix).
__global__ void eligible_kernel(const uint64_t* row, const uint32_t* col, uint64_t n,
                                uint64_t limit, uint64_t* cnt) {
  GRID_LOOP(v, n) {
    uint64_t lo = row[v], hi = row[v + 1];
    while (lo < hi) {
      const uint64_t m = (lo + hi) >> 1;
      if (col[m] < limit) lo = m + 1; else hi = m;
    }
    cnt[v] = lo - row[v];
  }
}

// Keys (v << 32 | ~deg(w)), values w for every eligible edge; a stable key sort
// then orders each row by descending degree with ascending ids on ties.
__global__ void split_keys_kernel(const uint64_t* row, const uint32_t* col, const uint32_t* deg,
                                  uint64_t n, const uint64_t* cnt, const uint64_t* pos,
                                  uint64_t* keys, uint32_t* vals) {
  const unsigned lane = threadIdx.x & 31;
  const uint64_t warp = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
  const uint64_t nwarps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  for (uint64_t v = warp; v < n; v += nwarps)
    for (uint64_t k = lane; k < cnt[v]; k += 32) {
      const uint32_t w = col[row[v] + k];
      keys[pos[v] + k] = (v << 32) | static_cast<uint32_t>(~deg[w]);
      vals[pos[v] + k] = w;
    }
}

__global__ void split_out_kernel(uint64_t n, const uint64_t* cnt, const uint64_t* pos,
                                 const uint32_t* sorted, uint64_t* in_plus) {
  GRID_LOOP(v, n) in_plus[v] = cnt[v] ? sorted[pos[v]] : kNone64;
}

__global__ void minus_kernel(uint64_t n, const uint64_t* cnt, const uint64_t* pos,
                             const uint64_t* moff, const uint32_t* sorted, uint64_t* minus) {
  const unsigned lane = threadIdx.x & 31;
  const uint64_t warp = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
  const uint64_t nwarps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  for (uint64_t v = warp; v < n; v += nwarps)
    for (uint64_t k = 1 + lane; k < cnt[v]; k += 32) minus[moff[v] + k - 1] = sorted[pos[v] + k];
}

__global__ void minus_count_kernel(uint64_t n, const uint64_t* cnt, uint64_t* out) {
  GRID_LOOP(v, n) out[v] = cnt[v] ? cnt[v] - 1 : 0;
}

// ---- reference levels: level-synchronous BFS ---------------------------------
__global__ void level_step_kernel(const uint64_t* row, const uint32_t* col, uint64_t n,
                                  uint32_t* lvl, uint32_t cur, unsigned long long* grew) {
  const unsigned lane = threadIdx.x & 31;
  const uint64_t warp = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
  const uint64_t nwarps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  unsigned long long g = 0;
  for (uint64_t v = warp; v < n; v += nwarps) {
    if (lvl[v] != cur) continue;
    for (uint64_t k = row[v] + lane; k < row[v + 1]; k += 32) {
      const uint32_t w = col[k];
      if (lvl[w] == kNone32 && atomicCAS(&lvl[w], kNone32, cur + 1) == kNone32) ++g;
    }
  }
  if (g) atomicAdd(grew, g);
}

// ---- tree validation -----------------------------------------------------------
// term: 0 chain continues, 1 the root (parent[root] == root), 2 unset parent,
// 3 parent outside [0, n).
__global__ void chain_init_kernel(const uint64_t* parent, uint64_t n, uint64_t root,
                                  uint8_t* term, uint64_t* anc, uint32_t* dist) {
  GRID_LOOP(v, n) {
    const uint64_t p = parent[v];
    uint8_t t = 0;
    if (v == root && p == root) t = 1;
    else if (p == kNone64) t = 2;
    else if (p >= n) t = 3;
    term[v] = t;
    anc[v] = t ? v : p;
    dist[v] = t == 0 ? 1u : 0u;
  }
}

// One pointer-jumping round (double buffered): a vertex whose ancestor is a
// terminal stops there.
__global__ void chain_jump_kernel(uint64_t n, const uint8_t* term, const uint64_t* anc,
                                  const uint32_t* dist, uint64_t* anc2, uint32_t* dist2,
                                  unsigned long long* moved) {
  unsigned long long mv = 0;
  GRID_LOOP(v, n) {
    const uint64_t a = anc[v];
    if (term[v] || term[a]) {
      anc2[v] = a;
      dist2[v] = dist[v];
    } else {
      anc2[v] = anc[a];
      dist2[v] = dist[v] + dist[a];
      ++mv;
    }
  }
  if (mv) atomicAdd(moved, mv);
}

struct Fails {
  uint64_t* keys[6];  // per rule 1..5 (index 0 unused): ordering keys of failures
  unsigned long long* cnt;  // [6] failures per rule
  uint64_t cap;
};

__device__ __forceinline__ void add_fail(const Fails& f, int rule, uint64_t key) {
  const unsigned long long i = atomicAdd(&f.cnt[rule], 1ull);
  if (i < f.cap) f.keys[rule][i] = key;
}

// Rules 1, 3 and 5, the levels, reached count and traversed edges. Rule 2's
// failures (chains that never reach the root) are the terminals / cycle
// vertices those chains end on; their key is the representative vertex.
__global__ void tree_rules_kernel(const uint64_t* row, const uint32_t* col, const uint32_t* deg,
                                  uint64_t n, uint64_t root, const uint64_t* parent,
                                  const uint8_t* term, const uint64_t* anc, const uint32_t* dist,
                                  const uint32_t* olvl, uint32_t* lvl, Fails f,
                                  unsigned long long* acc /* [2] reached, degree sum */) {
  unsigned long long reached = 0, degs = 0;
  GRID_LOOP(v, n) {
    const uint64_t p = parent[v];
    const uint64_t a = anc[v];
    const bool to_root = term[a] == 1 && (term[v] == 0 || v == a);
    lvl[v] = to_root ? dist[v] : kNone32;
    if (v == root && p != root) add_fail(f, 1, v);
    if (p != kNone64) {
      ++reached;
      degs += deg[v];
      if (!to_root) {  // a chain that dead-ends or cycles
        if (term[a] == 2 || term[a] == 3) add_fail(f, 2, (uint64_t{1} << 62) | a);  // broken
        else if (term[a] == 0) add_fail(f, 2, a);  // cycle (a lies on it)
      }
      if (!(v == root && p == v)) {
        if (p >= n) {
          add_fail(f, 3, v);
        } else {
          uint64_t lo = row[v], hi = row[v + 1];
          while (lo < hi) {
            const uint64_t m = (lo + hi) >> 1;
            if (col[m] < p) lo = m + 1; else hi = m;
          }
          if (lo == row[v + 1] || col[lo] != p) add_fail(f, 3, v);
        }
      }
    }
    const bool in_comp = olvl[v] != kNone32;
    if ((p != kNone64) != in_comp) add_fail(f, 5, v);
  }
  for (int o = 16; o; o >>= 1) {
    reached += __shfl_xor_sync(0xffffffffu, reached, o);
    degs += __shfl_xor_sync(0xffffffffu, degs, o);
  }
  if ((threadIdx.x & 31) == 0) {
    if (reached) atomicAdd(&acc[0], reached);
    if (degs) atomicAdd(&acc[1], degs);
  }
}

// Rule 4 over each undirected edge once (from its smaller endpoint), in the
// reference's order: key = (v, position in v's row).
__global__ void span_kernel(const uint64_t* row, const uint32_t* col, uint64_t n,
                            const uint32_t* lvl, Fails f) {
  const unsigned lane = threadIdx.x & 31;
  const uint64_t warp = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
  const uint64_t nwarps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  for (uint64_t v = warp; v < n; v += nwarps) {
    const uint32_t lv = lvl[v];
    if (lv == kNone32) continue;
    for (uint64_t k = row[v] + lane; k < row[v + 1]; k += 32) {
      const uint32_t w = col[k];
      if (w <= v) continue;
      const uint32_t lw = lvl[w];
      if (lw == kNone32) continue;
      if ((lv > lw ? lv - lw : lw - lv) > 1) add_fail(f, 4, (v << 32) | (k - row[v]));
    }
  }
}

}  // namespace

void graph_degree_split(const DevGraph& g, uint64_t limit, uint64_t* h_in_plus,
                        uint64_t* h_moff, uint64_t* h_minus, cudaStream_t s) {
  const uint64_t n = g.n;
  if (!n) {
    if (h_moff) h_moff[0] = 0;
    return;
  }
  DevBuf<uint64_t> cnt(n), pos(n + 1), mc(n + 1), moff(n + 1);
  eligible_kernel<<<grid_for(n, 256), 256, 0, s>>>(g.row.get(), g.col.get(), n, limit, cnt.get());
  ETB_LAUNCH_CHECK();
  DevBuf<uint64_t> cnt1(n + 1);
  ETB_CUDA(cudaMemcpyAsync(cnt1.get(), cnt.get(), n * 8, cudaMemcpyDeviceToDevice, s));
  ETB_CUDA(cudaMemsetAsync(cnt1.get() + n, 0, 8, s));
  exclusive_scan_u64(cnt1.get(), pos.get(), n + 1, s);
  const uint64_t total = read_u64(pos.get() + n, s);
  minus_count_kernel<<<grid_for(n, 256), 256, 0, s>>>(n, cnt.get(), mc.get());
  ETB_CUDA(cudaMemsetAsync(mc.get() + n, 0, 8, s));
  exclusive_scan_u64(mc.get(), moff.get(), n + 1, s);
  if (h_moff)
    ETB_CUDA(cudaMemcpyAsync(h_moff, moff.get(), (n + 1) * 8, cudaMemcpyDeviceToHost, s));
  if (!h_in_plus && !h_minus) {
    ETB_CUDA(cudaStreamSynchronize(s));
    return;
  }
  DevBuf<uint64_t> keys(total ? total : 1), kalt;
  DevBuf<uint32_t> vals(total ? total : 1), valt;
  split_keys_kernel<<<grid_for(n * 32, 256), 256, 0, s>>>(g.row.get(), g.col.get(), g.deg.get(), n,
                                                          cnt.get(), pos.get(), keys.get(),
                                                          vals.get());
  ETB_LAUNCH_CHECK();
  sort_pairs_u64_u32(keys, kalt, vals, valt, total, 64, s);
  DevBuf<uint64_t> in_plus(n), minus(std::max<uint64_t>(total, 1));
  split_out_kernel<<<grid_for(n, 256), 256, 0, s>>>(n, cnt.get(), pos.get(), vals.get(),
                                                    in_plus.get());
  ETB_LAUNCH_CHECK();
  minus_kernel<<<grid_for(n * 32, 256), 256, 0, s>>>(n, cnt.get(), pos.get(), moff.get(),
                                                     vals.get(), minus.get());
  ETB_LAUNCH_CHECK();
  const uint64_t mtotal = read_u64(moff.get() + n, s);
  if (h_in_plus)
    ETB_CUDA(cudaMemcpyAsync(h_in_plus, in_plus.get(), n * 8, cudaMemcpyDeviceToHost, s));
  if (h_minus && mtotal)
    ETB_CUDA(cudaMemcpyAsync(h_minus, minus.get(), mtotal * 8, cudaMemcpyDeviceToHost, s));
  ETB_CUDA(cudaStreamSynchronize(s));
}

void graph_levels(const DevGraph& g, uint64_t root, DevBuf<uint32_t>& lvl, cudaStream_t s) {
  const uint64_t n = g.n;
  lvl.alloc(n ? n : 1);
  ETB_CUDA(cudaMemsetAsync(lvl.get(), 0xFF, n * 4, s));
  const uint32_t zero = 0;
  ETB_CUDA(cudaMemcpyAsync(lvl.get() + root, &zero, 4, cudaMemcpyHostToDevice, s));
  DevBuf<unsigned long long> grew(1);
  for (uint32_t cur = 0;; ++cur) {
    ETB_CUDA(cudaMemsetAsync(grew.get(), 0, 8, s));
    level_step_kernel<<<grid_for(n * 32, 256), 256, 0, s>>>(g.row.get(), g.col.get(), n,
                                                            lvl.get(), cur, grew.get());
    ETB_LAUNCH_CHECK();
    unsigned long long h = 0;
    ETB_CUDA(cudaMemcpyAsync(&h, grew.get(), 8, cudaMemcpyDeviceToHost, s));
    ETB_CUDA(cudaStreamSynchronize(s));
    if (!h) break;
  }
}

void graph_validate_tree(const DevGraph& g, uint64_t root, const uint64_t* h_parent,
                         uint64_t out[8], std::vector<uint64_t> first[6], cudaStream_t s) {
  const uint64_t n = g.n;
  DevBuf<uint64_t> parent(n), anc(n), anc2(n);
  DevBuf<uint32_t> dist(n), dist2(n), lvl(n), olvl;
  DevBuf<uint8_t> term(n);
  ETB_CUDA(cudaMemcpyAsync(parent.get(), h_parent, n * 8, cudaMemcpyHostToDevice, s));
  graph_levels(g, root, olvl, s);  // the component (rule 5), independent of the tree
  chain_init_kernel<<<grid_for(n, 256), 256, 0, s>>>(parent.get(), n, root, term.get(), anc.get(),
                                                     dist.get());
  ETB_LAUNCH_CHECK();
  DevBuf<unsigned long long> moved(1);
  int rounds = 2;
  for (uint64_t x = n; x; x >>= 1) ++rounds;  // log2 n + 2 rounds reach every root-bound end
  for (int r = 0; r < rounds; ++r) {
    ETB_CUDA(cudaMemsetAsync(moved.get(), 0, 8, s));
    chain_jump_kernel<<<grid_for(n, 256), 256, 0, s>>>(n, term.get(), anc.get(), dist.get(),
                                                       anc2.get(), dist2.get(), moved.get());
    ETB_LAUNCH_CHECK();
    std::swap(anc, anc2);
    std::swap(dist, dist2);
    unsigned long long h = 0;
    ETB_CUDA(cudaMemcpyAsync(&h, moved.get(), 8, cudaMemcpyDeviceToHost, s));
    ETB_CUDA(cudaStreamSynchronize(s));
    if (!h) break;
  }
  Fails f{};
  const uint64_t cap = std::max<uint64_t>(n, 1) + 64;
  DevBuf<uint64_t> kb[6];
  for (int r = 1; r <= 5; ++r) {
    kb[r].alloc(r == 4 ? std::min<uint64_t>(g.nnz / 2 + 64, uint64_t{1} << 26) : cap);
    f.keys[r] = kb[r].get();
  }
  f.cap = cap;
  DevBuf<unsigned long long> cnt(6), acc(2);
  ETB_CUDA(cudaMemsetAsync(cnt.get(), 0, 48, s));
  ETB_CUDA(cudaMemsetAsync(acc.get(), 0, 16, s));
  f.cnt = cnt.get();
  tree_rules_kernel<<<grid_for(n, 256), 256, 0, s>>>(g.row.get(), g.col.get(), g.deg.get(), n,
                                                     root, parent.get(), term.get(), anc.get(),
                                                     dist.get(), olvl.get(), lvl.get(), f,
                                                     acc.get());
  ETB_LAUNCH_CHECK();
  Fails f4 = f;
  f4.cap = kb[4].size();
  span_kernel<<<grid_for(n * 32, 256), 256, 0, s>>>(g.row.get(), g.col.get(), n, lvl.get(), f4);
  ETB_LAUNCH_CHECK();
  unsigned long long hc[6], ha[2];
  ETB_CUDA(cudaMemcpyAsync(hc, cnt.get(), 48, cudaMemcpyDeviceToHost, s));
  ETB_CUDA(cudaMemcpyAsync(ha, acc.get(), 16, cudaMemcpyDeviceToHost, s));
  ETB_CUDA(cudaStreamSynchronize(s));
  for (int r = 1; r <= 5; ++r) {
    const uint64_t m = std::min<uint64_t>(hc[r], r == 4 ? kb[4].size() : cap);
    std::vector<uint64_t> keys(m);
    if (m) ETB_CUDA(cudaMemcpyAsync(keys.data(), kb[r].get(), m * 8, cudaMemcpyDeviceToHost, s));
    ETB_CUDA(cudaStreamSynchronize(s));
    std::sort(keys.begin(), keys.end());
    if (r == 2) keys.erase(std::unique(keys.begin(), keys.end()), keys.end());
    first[r] = std::move(keys);
    out[r] = r == 2 ? first[r].size() : hc[r];
  }
  out[6] = ha[0];
  out[7] = ha[1] / 2;
}

}  // namespace etb
