// (2b) relayout_csr + extract_edge_tree_list on sm_100a (src/relayout.cpp:25-169).
//
// The reference places vertices with a sequential queue walk. The same order
// is produced here data-parallel:
//   * core block: sort (degree desc, id asc) -> one radix sort of
//     ((~deg) << 32 | id) keys;
//   * edge trees are oriented by a level-synchronous BFS over tree vertices
//     seeded at every tree vertex adjacent to a core-edge vertex; trees that
//     never touch the core are rooted at their smallest id (min-label
//     propagation) and walked the same way;
//   * trees are ordered by (CE position, root id), component trees after them
//     by root id; inside a tree the BFS queue order is (depth, parent's new
//     id, own id), assigned one depth level at a time with per-tree cursors;
//   * isolated vertices close the index space in ascending id.
// The edge-tree list falls out: src = tree parent, core_edge = the tree's CE.
// Finally the core-only CSR (the core prefix of every core row) is rebuilt in
// the new ids with one key sort; that is all the traversal reads.
#include <algorithm>
#include <cstdlib>

#include "internal.cuh"

namespace etb {
namespace {

constexpr uint8_t CI = ETB_CI, CE = ETB_CE, TI = ETB_TI, TL = ETB_TL, VZ = ETB_VZ;
__device__ __forceinline__ bool is_core(uint8_t t) { return t == CI || t == CE; }
__device__ __forceinline__ bool is_tree(uint8_t t) { return t == TI || t == TL; }

enum : int { kErrNone = 0, kErrTouch = 1, kErrIsolated = 2, kErrCycle = 3 };
const char* err_text(int e) {
  switch (e) {
    case kErrTouch: return "extract_edge_tree_list: edge tree touches the core more than once";
    case kErrIsolated: return "extract_edge_tree_list: isolated-typed vertex has incident edges";
    case kErrCycle: return "extract_edge_tree_list: cycle through tree vertices";
  }
  return "";
}

#define GRID_LOOP(i, n)                                                        \
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < (n); \
       i += (uint64_t)gridDim.x * blockDim.x)

__global__ void class_count_kernel(const uint8_t* type, uint64_t n, unsigned long long* c) {
  unsigned long long k = 0, t = 0, z = 0;
  GRID_LOOP(v, n) {
    const uint8_t ty = type[v];
    k += is_core(ty);
    t += is_tree(ty);
    z += ty == VZ;
  }
  for (int o = 16; o; o >>= 1) {
    k += __shfl_xor_sync(0xffffffffu, k, o);
    t += __shfl_xor_sync(0xffffffffu, t, o);
    z += __shfl_xor_sync(0xffffffffu, z, o);
  }
  if ((threadIdx.x & 31) == 0) {
    if (k) atomicAdd(&c[0], k);
    if (t) atomicAdd(&c[1], t);
    if (z) atomicAdd(&c[2], z);
  }
}

__global__ void core_keys_kernel(const uint8_t* type, const uint32_t* deg, uint64_t n,
                                 uint64_t* keys, unsigned long long* cnt) {
  GRID_LOOP(v, n) {
    if (!is_core(type[v])) continue;
    const unsigned long long p = atomicAdd(cnt, 1ull);
    keys[p] = (uint64_t(0xFFFFFFFFu - deg[v]) << 32) | v;
  }
}

__global__ void scatter_sorted_kernel(const uint64_t* keys, uint64_t count, uint64_t base,
                                      uint32_t* new2old, uint32_t* old2new) {
  GRID_LOOP(i, count) {
    const uint32_t v = static_cast<uint32_t>(keys[i] & 0xFFFFFFFFu);
    new2old[base + i] = v;
    old2new[v] = static_cast<uint32_t>(base + i);
  }
}

// Tree seeds: tree vertices adjacent to the core. Also detects the reference's
// extract errors that are visible locally.
__global__ void tree_init_kernel(const uint64_t* row, const uint32_t* col, const uint8_t* type,
                                 uint64_t n, uint32_t* tpar, uint32_t* tdep, uint32_t* troot,
                                 uint32_t* tce, uint32_t* q, unsigned long long* qn, int* err) {
  GRID_LOOP(v, n) {
    const uint8_t t = type[v];
    tpar[v] = kNone32;
    if (t == VZ || t == CI) {
      // An isolated-typed vertex next to a CE or a tree vertex breaks extract.
      if (t == VZ)
        for (uint64_t k = row[v]; k < row[v + 1]; ++k) {
          const uint8_t tw = type[col[k]];
          if (tw == CE || is_tree(tw)) atomicMax(err, (int)kErrIsolated);
        }
      continue;
    }
    if (t == CE) continue;
    uint32_t c = kNone32, ncore = 0;
    for (uint64_t k = row[v]; k < row[v + 1]; ++k) {
      const uint32_t w = col[k];
      const uint8_t tw = type[w];
      if (is_core(tw)) {
        ++ncore;
        c = w;
        if (tw == CI) atomicMax(err, (int)kErrTouch);
      }
    }
    if (ncore > 1) atomicMax(err, (int)kErrTouch);
    if (ncore == 1) {
      tpar[v] = c;
      tdep[v] = 1;
      troot[v] = static_cast<uint32_t>(v);
      tce[v] = c;
      q[atomicAdd(qn, 1ull)] = static_cast<uint32_t>(v);
    }
  }
}

// One BFS level over tree vertices (warp per frontier vertex).
__global__ void tree_bfs_kernel(const uint64_t* row, const uint32_t* col, const uint8_t* type,
                                const uint32_t* q, uint64_t qn, uint32_t* tpar, uint32_t* tdep,
                                uint32_t* troot, uint32_t* tce, uint32_t* nq,
                                unsigned long long* nqn) {
  const unsigned lane = threadIdx.x & 31;
  const uint64_t warp = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
  const uint64_t nwarps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  for (uint64_t i = warp; i < qn; i += nwarps) {
    const uint32_t u = q[i];
    const uint32_t du = tdep[u], ru = troot[u], cu = tce[u];
    for (uint64_t k = row[u] + lane; k < row[u + 1]; k += 32) {
      const uint32_t w = col[k];
      if (!is_tree(type[w])) continue;
      if (atomicCAS(&tpar[w], kNone32, u) == kNone32) {
        tdep[w] = du + 1;
        troot[w] = ru;
        tce[w] = cu;
        nq[atomicAdd(nqn, 1ull)] = w;
      }
    }
  }
}

// Component trees: smallest id per tree-only component (label propagation
// with pointer jumping), restricted to tree vertices the core BFS missed.
__global__ void label_init_kernel(const uint8_t* type, const uint32_t* tpar, uint64_t n,
                                  uint32_t* lab) {
  GRID_LOOP(v, n) lab[v] = (is_tree(type[v]) && tpar[v] == kNone32) ? (uint32_t)v : kNone32;
}

__global__ void label_step_kernel(const uint64_t* row, const uint32_t* col, uint64_t n,
                                  uint32_t* lab, int* changed) {
  GRID_LOOP(v, n) {
    uint32_t l = lab[v];
    if (l == kNone32) continue;
    uint32_t m = l;
    for (uint64_t k = row[v]; k < row[v + 1]; ++k) {
      const uint32_t lw = lab[col[k]];
      if (lw < m) m = lw;
    }
    const uint32_t j = lab[m];
    if (j < m) m = j;
    if (m < l) {
      atomicMin(&lab[v], m);
      *changed = 1;
    }
  }
}

__global__ void component_roots_kernel(const uint32_t* lab, uint64_t n, uint32_t* tpar,
                                       uint32_t* tdep, uint32_t* troot, uint32_t* tce,
                                       uint32_t* q, unsigned long long* qn) {
  GRID_LOOP(v, n) {
    if (lab[v] != (uint32_t)v) continue;
    tpar[v] = static_cast<uint32_t>(v);
    tdep[v] = 0;
    troot[v] = static_cast<uint32_t>(v);
    tce[v] = kNone32;
    q[atomicAdd(qn, 1ull)] = static_cast<uint32_t>(v);
  }
}

__global__ void child_count_kernel(const uint8_t* type, const uint32_t* tpar, uint64_t n,
                                   uint32_t* nchild) {
  GRID_LOOP(v, n) {
    if (!is_tree(type[v])) continue;
    const uint32_t p = tpar[v];
    if (p != kNone32 && p != (uint32_t)v && is_tree(type[p])) atomicAdd(&nchild[p], 1u);
  }
}

// Every tree edge must be a parent/child link; a non-tree edge inside one tree
// is a cycle, between two trees it means one tree touches the core twice.
__global__ void tree_check_kernel(const uint64_t* row, const uint32_t* col, const uint8_t* type,
                                  const uint32_t* tpar, const uint32_t* troot,
                                  const uint32_t* nchild, uint64_t n, int* err) {
  GRID_LOOP(v, n) {
    if (!is_tree(type[v])) continue;
    if (tpar[v] == kNone32) {
      atomicMax(err, (int)kErrTouch);
      continue;
    }
    uint32_t tn = 0;
    for (uint64_t k = row[v]; k < row[v + 1]; ++k) {
      const uint32_t w = col[k];
      if (!is_tree(type[w])) continue;
      ++tn;
      if (w != tpar[v] && tpar[w] != (uint32_t)v)
        atomicMax(err, troot[w] != troot[v] ? (int)kErrTouch : (int)kErrCycle);
    }
    const uint32_t p = tpar[v];
    const uint32_t expect = nchild[v] + ((p != (uint32_t)v && is_tree(type[p])) ? 1u : 0u);
    if (tn != expect) atomicMax(err, (int)kErrCycle);
  }
}

// ---- placement -------------------------------------------------------------
__global__ void root_keys_kernel(const uint8_t* type, const uint32_t* tpar, const uint32_t* tce,
                                 const uint32_t* old2new, uint64_t n, uint64_t* keys,
                                 unsigned long long* cnt) {
  GRID_LOOP(v, n) {
    if (!is_tree(type[v])) continue;
    const uint32_t p = tpar[v];
    const bool attached_root = p != (uint32_t)v && !is_tree(type[p]);
    const bool comp_root = p == (uint32_t)v;
    if (!attached_root && !comp_root) continue;
    const uint64_t hi = comp_root ? 0xFFFFFFFFull : old2new[tce[v]];
    keys[atomicAdd(cnt, 1ull)] = (hi << 32) | v;
  }
}

__global__ void root_rank_kernel(const uint64_t* keys, uint64_t count, uint32_t* rank_of) {
  GRID_LOOP(i, count) rank_of[keys[i] & 0xFFFFFFFFu] = static_cast<uint32_t>(i);
}

__global__ void tree_size_kernel(const uint8_t* type, const uint32_t* troot,
                                 const uint32_t* rank_of, uint64_t n, uint32_t* size) {
  GRID_LOOP(v, n) if (is_tree(type[v])) atomicAdd(&size[rank_of[troot[v]]], 1u);
}

// Level index inside the tree: attached roots (depth 1) and component roots
// (depth 0) are both level 0.
__global__ void level_keys_kernel(const uint8_t* type, const uint32_t* tdep, const uint32_t* tce,
                                  uint64_t n, uint64_t* keys, unsigned long long* cnt,
                                  unsigned* maxlev) {
  GRID_LOOP(v, n) {
    if (!is_tree(type[v])) continue;
    const uint32_t lev = tdep[v] - (tce[v] != kNone32 ? 1u : 0u);
    keys[atomicAdd(cnt, 1ull)] = (uint64_t(lev) << 32) | v;
    atomicMax(maxlev, lev);
  }
}

__global__ void level_bounds_kernel(const uint64_t* keys, uint64_t count, unsigned maxlev,
                                    uint64_t* bounds) {
  GRID_LOOP(l, (uint64_t)maxlev + 2) {
    const uint64_t target = l << 32;
    uint64_t lo = 0, hi = count;
    while (lo < hi) {
      const uint64_t mid = (lo + hi) >> 1;
      if (keys[mid] < target) lo = mid + 1; else hi = mid;
    }
    bounds[l] = lo;
  }
}

__global__ void place_roots_kernel(const uint64_t* lkeys, uint64_t count, const uint32_t* rank_of,
                                   const uint64_t* off, uint64_t nc, uint32_t* old2new,
                                   uint32_t* new2old, uint64_t* cursor) {
  GRID_LOOP(i, count) {
    const uint32_t v = static_cast<uint32_t>(lkeys[i] & 0xFFFFFFFFu);
    const uint32_t r = rank_of[v];
    const uint32_t id = static_cast<uint32_t>(nc + off[r]);
    old2new[v] = id;
    new2old[id] = v;
    cursor[r] = off[r] + 1;
  }
}

__global__ void level_child_keys_kernel(const uint64_t* lkeys, uint64_t count, const uint32_t* tpar,
                                        const uint32_t* old2new, uint64_t* keys) {
  GRID_LOOP(i, count) {
    const uint32_t v = static_cast<uint32_t>(lkeys[i] & 0xFFFFFFFFu);
    keys[i] = (uint64_t(old2new[tpar[v]]) << 32) | v;
  }
}

__global__ void level_heads_kernel(const uint64_t* keys, uint64_t count, const uint32_t* troot,
                                   const uint32_t* rank_of, uint32_t* tree_of, uint32_t* head) {
  GRID_LOOP(i, count) {
    const uint32_t t = rank_of[troot[keys[i] & 0xFFFFFFFFu]];
    tree_of[i] = t;
    bool h = i == 0;
    if (!h) h = rank_of[troot[keys[i - 1] & 0xFFFFFFFFu]] != t;
    head[i] = h ? static_cast<uint32_t>(i) : 0u;
  }
}

__global__ void level_place_kernel(const uint64_t* keys, uint64_t count, const uint32_t* tree_of,
                                   const uint32_t* segstart, const uint64_t* cursor, uint64_t nc,
                                   uint32_t* old2new, uint32_t* new2old) {
  GRID_LOOP(i, count) {
    const uint32_t v = static_cast<uint32_t>(keys[i] & 0xFFFFFFFFu);
    const uint32_t id = static_cast<uint32_t>(nc + cursor[tree_of[i]] + (i - segstart[i]));
    old2new[v] = id;
    new2old[id] = v;
  }
}

__global__ void level_advance_kernel(const uint32_t* tree_of, const uint32_t* segstart,
                                     uint64_t count, uint64_t* cursor) {
  GRID_LOOP(i, count) {
    if (i + 1 == count || tree_of[i + 1] != tree_of[i]) cursor[tree_of[i]] += i - segstart[i] + 1;
  }
}

__global__ void vz_flags_kernel(const uint8_t* type, uint64_t n, uint32_t* flag) {
  GRID_LOOP(v, n) flag[v] = type[v] == VZ;
}

__global__ void vz_place_kernel(const uint8_t* type, const uint64_t* rankv, uint64_t n,
                                uint64_t base, uint32_t* old2new, uint32_t* new2old) {
  GRID_LOOP(v, n) {
    if (type[v] != VZ) continue;
    const uint32_t id = static_cast<uint32_t>(base + rankv[v]);
    old2new[v] = id;
    new2old[id] = static_cast<uint32_t>(v);
  }
}

__global__ void relaid_arrays_kernel(const uint32_t* new2old, const uint32_t* old2new,
                                     const uint8_t* type, const uint32_t* deg, const uint32_t* tpar,
                                     const uint32_t* tdep, const uint32_t* tce, uint64_t n,
                                     uint64_t nc, uint64_t nt, uint8_t* rtype, uint32_t* degn,
                                     uint32_t* tsrc, uint32_t* tanchor, uint32_t* tdepth) {
  GRID_LOOP(i, n) {
    const uint32_t v = new2old[i];
    rtype[i] = type[v];
    degn[i] = deg[v];
    if (i >= nc && i < nc + nt) {
      const uint64_t t = i - nc;
      const uint32_t p = tpar[v];
      tsrc[t] = p == v ? static_cast<uint32_t>(i) : old2new[p];
      tanchor[t] = tce[v] == kNone32 ? kNone32 : old2new[tce[v]];
      tdepth[t] = tdep[v];
    }
  }
}

// Core-only relaid CSR: per-row counts, then (new_src << b | new_dst) keys.
__global__ void core_count_kernel(const uint64_t* row, const uint32_t* col, const uint8_t* type,
                                  const uint32_t* new2old, uint64_t nc, uint32_t* cnt) {
  const unsigned lane = threadIdx.x & 31;
  const uint64_t warp = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
  const uint64_t nwarps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  for (uint64_t i = warp; i < nc; i += nwarps) {
    const uint32_t o = new2old[i];
    uint32_t c = 0;
    for (uint64_t k = row[o] + lane; k < row[o + 1]; k += 32) c += is_core(type[col[k]]);
    for (int s = 16; s; s >>= 1) c += __shfl_xor_sync(0xffffffffu, c, s);
    if (lane == 0) cnt[i] = c;
  }
}

__global__ void core_edge_keys_kernel(const uint64_t* row, const uint32_t* col, const uint8_t* type,
                                      const uint32_t* new2old, const uint32_t* old2new,
                                      const uint64_t* crow, uint64_t lo, uint64_t hi, int b,
                                      uint64_t* keys) {
  const unsigned lane = threadIdx.x & 31;
  const uint64_t warp = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
  const uint64_t nwarps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  const uint64_t kbase = crow[lo];
  for (uint64_t i = lo + warp; i < hi; i += nwarps) {
    const uint32_t o = new2old[i];
    uint64_t pos = crow[i] - kbase;
    for (uint64_t k0 = row[o]; k0 < row[o + 1]; k0 += 32) {
      const uint64_t k = k0 + lane;
      bool keep = false;
      uint32_t w = 0;
      if (k < row[o + 1]) {
        w = col[k];
        keep = is_core(type[w]);
      }
      const unsigned m = __ballot_sync(0xffffffffu, keep);
      if (keep) keys[pos + __popc(m & ((1u << lane) - 1))] = (i << b) | old2new[w];
      pos += __popc(m);
    }
  }
}

// Whole relabelled graph keys (relabel_graph, build.cpp:144-166).
__global__ void full_edge_keys_kernel(const uint64_t* row, const uint32_t* col,
                                      const uint32_t* new2old, const uint32_t* old2new,
                                      const uint64_t* nrow, uint64_t n, int b, uint64_t* keys) {
  const unsigned lane = threadIdx.x & 31;
  const uint64_t warp = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
  const uint64_t nwarps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  for (uint64_t i = warp; i < n; i += nwarps) {
    const uint32_t o = new2old[i];
    const uint64_t base = nrow[i];
    for (uint64_t k = row[o] + lane; k < row[o + 1]; k += 32)
      keys[base + (k - row[o])] = (i << b) | old2new[col[k]];
  }
}

__global__ void key_cols_kernel(const uint64_t* keys, uint64_t count, uint64_t mask,
                                uint32_t* col) {
  GRID_LOOP(i, count) col[i] = static_cast<uint32_t>(keys[i] & mask);
}

__global__ void first_nbr_kernel(const uint64_t* crow, const uint32_t* ccol, const uint32_t* degn,
                                 uint64_t nc, uint32_t* first, uint32_t* second, uint2* third,
                                 uint2* meta) {
  GRID_LOOP(i, nc) {
    const uint64_t d = crow[i + 1] - crow[i];
    first[i] = d ? ccol[crow[i]] : kNone32;
    second[i] = d >= 2 ? ccol[crow[i] + 1] | (d == 2 ? 0x80000000u : 0u) : kNone32;
    // third and fourth neighbours, bit 31 on the row's last one (kNone32: none)
    third[i] = make_uint2(d >= 3 ? ccol[crow[i] + 2] | (d == 3 ? 0x80000000u : 0u) : kNone32,
                          d >= 4 ? ccol[crow[i] + 3] | (d == 4 ? 0x80000000u : 0u) : kNone32);
    meta[i] = make_uint2(static_cast<uint32_t>(crow[i + 1] - crow[i]), degn[i]);
  }
}

__global__ void gather_u32_kernel(const uint32_t* src, const uint32_t* idx, uint64_t n,
                                  uint32_t* dst) {
  GRID_LOOP(i, n) dst[i] = src[idx[i]];
}

unsigned wgrid(uint64_t items) { return grid_for(items * 32, 256); }

template <typename T>
std::vector<T> to_host(const T* d, uint64_t n, cudaStream_t s) {
  std::vector<T> h(n);
  if (n) ETB_CUDA(cudaMemcpyAsync(h.data(), d, n * sizeof(T), cudaMemcpyDeviceToHost, s));
  ETB_CUDA(cudaStreamSynchronize(s));
  return h;
}

}  // namespace

// ---- core connected components (untimed preprocessing) -------------------------
// Union-find with hooking of the larger root under the smaller by CAS and path
// halving; every core edge (u < w) is hooked once, then every vertex is
// pointed at its root and the roots count their component.
// Parents only ever point at smaller ids (hooking and halving both move a
// pointer down), so every walk terminates; loads bypass L1 (the pointers change
// under concurrent CAS in L2).
__device__ __forceinline__ uint32_t uf_find(uint32_t* par, uint32_t v) {
  for (;;) {
    const uint32_t p = __ldcg(&par[v]);
    if (p == v) return v;
    const uint32_t g = __ldcg(&par[p]);
    if (g == p) return p;
    atomicCAS(&par[v], p, g);  // path halving
    v = g;
  }
}

__global__ void uf_init_kernel(uint32_t* par, uint32_t* size, uint64_t nc) {
  GRID_LOOP(v, nc) {
    par[v] = static_cast<uint32_t>(v);
    size[v] = 0;
  }
}

__global__ void uf_hook_kernel(const uint64_t* crow, const uint32_t* ccol, uint32_t* par,
                               uint64_t nc) {
  // warp per core vertex, lanes over its row
  const uint64_t gw = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
  const uint64_t nw = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  const unsigned lane = threadIdx.x & 31;
  for (uint64_t u = gw; u < nc; u += nw) {
    for (uint64_t e = crow[u] + lane; e < crow[u + 1]; e += 32) {
      const uint32_t w = ccol[e];
      if (w <= u) continue;
      uint32_t a = static_cast<uint32_t>(u), b = w;
      for (;;) {
        a = uf_find(par, a);
        b = uf_find(par, b);
        if (a == b) break;
        if (a > b) {
          const uint32_t t = a;
          a = b;
          b = t;
        }
        // hook the larger root b under a
        if (atomicCAS(&par[b], b, a) == b) break;
      }
    }
  }
}

__global__ void uf_flatten_kernel(uint32_t* par, uint32_t* size, uint64_t nc) {
  GRID_LOOP(v, nc) {
    const uint32_t r = uf_find(par, static_cast<uint32_t>(v));
    par[v] = r;
    atomicAdd(&size[r], 1u);
  }
}

__global__ void uf_size_of_kernel(const uint32_t* par, const uint32_t* size, uint64_t nc,
                                  uint32_t* out) {
  GRID_LOOP(v, nc) out[v] = size[par[v]];
}

void core_components(DevLayout& L, cudaStream_t s) {
  const uint64_t nc = L.nc;
  L.h_comp_size.assign(nc, 0);
  if (!nc) return;
  DevBuf<uint32_t> par(nc), size(nc);
  uf_init_kernel<<<grid_for(nc, 256), 256, 0, s>>>(par.get(), size.get(), nc);
  ETB_LAUNCH_CHECK();
  uf_hook_kernel<<<grid_for(nc * 32, 256), 256, 0, s>>>(L.crow.get(), L.ccol.get(), par.get(), nc);
  ETB_LAUNCH_CHECK();
  uf_flatten_kernel<<<grid_for(nc, 256), 256, 0, s>>>(par.get(), size.get(), nc);
  ETB_LAUNCH_CHECK();
  uf_size_of_kernel<<<grid_for(nc, 256), 256, 0, s>>>(par.get(), size.get(), nc, par.get());
  ETB_LAUNCH_CHECK();
  ETB_CUDA(cudaMemcpyAsync(L.h_comp_size.data(), par.get(), nc * 4, cudaMemcpyDeviceToHost, s));
  ETB_CUDA(cudaStreamSynchronize(s));
}

void build_layout(const DevGraph& g, const uint8_t* type, int64_t mh, DevLayout& L,
                  cudaStream_t s) {
  const uint64_t n = g.n;
  const uint64_t n1 = n ? n : 1;
  const unsigned gb = grid_for(n, 256);
  L.n = n;
  L.mh = mh;
  L.nnz_full = g.nnz;

  DevBuf<unsigned long long> ctr(16);
  ETB_CUDA(cudaMemsetAsync(ctr.get(), 0, 128, s));
  class_count_kernel<<<gb, 256, 0, s>>>(type, n, ctr.get());
  ETB_LAUNCH_CHECK();
  {
    auto h = to_host(reinterpret_cast<const uint64_t*>(ctr.get()), 3, s);
    L.nc = h[0];
    L.nt = h[1];
    L.nz = h[2];
  }
  const uint64_t nc = L.nc, nt = L.nt;
  L.new2old.alloc(n1);
  L.old2new.alloc(n1);

  // -- core block ------------------------------------------------------------
  {
    DevBuf<uint64_t> keys(nc ? nc : 1), alt;
    ETB_CUDA(cudaMemsetAsync(ctr.get(), 0, 8, s));
    core_keys_kernel<<<gb, 256, 0, s>>>(type, g.deg.get(), n, keys.get(), ctr.get());
    ETB_LAUNCH_CHECK();
    sort_keys_u64(keys, alt, nc, 64, s);
    if (nc) {
      scatter_sorted_kernel<<<grid_for(nc, 256), 256, 0, s>>>(keys.get(), nc, 0, L.new2old.get(),
                                                               L.old2new.get());
      ETB_LAUNCH_CHECK();
    }
  }

  // -- tree orientation (original ids) ----------------------------------------
  DevBuf<uint32_t> tpar(n1), tdep(n1), troot(n1), tce(n1);
  DevBuf<int> err(2);
  ETB_CUDA(cudaMemsetAsync(err.get(), 0, 8, s));
  {
    DevBuf<uint32_t> qa(nt ? nt : 1), qb(nt ? nt : 1);
    ETB_CUDA(cudaMemsetAsync(ctr.get(), 0, 8, s));
    tree_init_kernel<<<gb, 256, 0, s>>>(g.row.get(), g.col.get(), type, n, tpar.get(), tdep.get(),
                                        troot.get(), tce.get(), qa.get(), ctr.get(), err.get());
    ETB_LAUNCH_CHECK();
    auto bfs = [&](uint64_t qn) {
      int cur = 0;
      while (qn > 0) {
        unsigned long long* nl = ctr.get() + 1 + cur;
        ETB_CUDA(cudaMemsetAsync(nl, 0, 8, s));
        tree_bfs_kernel<<<wgrid(qn), 256, 0, s>>>(g.row.get(), g.col.get(), type,
                                                  cur ? qb.get() : qa.get(), qn, tpar.get(),
                                                  tdep.get(), troot.get(), tce.get(),
                                                  cur ? qa.get() : qb.get(), nl);
        ETB_LAUNCH_CHECK();
        qn = read_u64(reinterpret_cast<uint64_t*>(nl), s);
        cur ^= 1;
      }
    };
    bfs(read_u64(reinterpret_cast<uint64_t*>(ctr.get()), s));
    // component trees
    DevBuf<uint32_t> lab(n1);
    label_init_kernel<<<gb, 256, 0, s>>>(type, tpar.get(), n, lab.get());
    ETB_LAUNCH_CHECK();
    for (;;) {
      ETB_CUDA(cudaMemsetAsync(err.get() + 1, 0, 4, s));
      label_step_kernel<<<gb, 256, 0, s>>>(g.row.get(), g.col.get(), n, lab.get(), err.get() + 1);
      ETB_LAUNCH_CHECK();
      int changed = 0;
      ETB_CUDA(cudaMemcpyAsync(&changed, err.get() + 1, 4, cudaMemcpyDeviceToHost, s));
      ETB_CUDA(cudaStreamSynchronize(s));
      if (!changed) break;
    }
    ETB_CUDA(cudaMemsetAsync(ctr.get(), 0, 8, s));
    component_roots_kernel<<<gb, 256, 0, s>>>(lab.get(), n, tpar.get(), tdep.get(), troot.get(),
                                              tce.get(), qa.get(), ctr.get());
    ETB_LAUNCH_CHECK();
    bfs(read_u64(reinterpret_cast<uint64_t*>(ctr.get()), s));
    DevBuf<uint32_t> nchild(n1);
    ETB_CUDA(cudaMemsetAsync(nchild.get(), 0, n1 * 4, s));
    child_count_kernel<<<gb, 256, 0, s>>>(type, tpar.get(), n, nchild.get());
    tree_check_kernel<<<gb, 256, 0, s>>>(g.row.get(), g.col.get(), type, tpar.get(), troot.get(),
                                         nchild.get(), n, err.get());
    ETB_LAUNCH_CHECK();
    int e = 0;
    ETB_CUDA(cudaMemcpyAsync(&e, err.get(), 4, cudaMemcpyDeviceToHost, s));
    ETB_CUDA(cudaStreamSynchronize(s));
    if (e != kErrNone) throw std::runtime_error(err_text(e));
  }

  // -- tree placement -----------------------------------------------------------
  DevBuf<uint32_t> rank_of(n1);
  std::vector<uint64_t> h_off;
  if (nt) {
    DevBuf<uint64_t> rkeys(nt), alt;
    ETB_CUDA(cudaMemsetAsync(ctr.get(), 0, 8, s));
    root_keys_kernel<<<gb, 256, 0, s>>>(type, tpar.get(), tce.get(), L.old2new.get(), n,
                                        rkeys.get(), ctr.get());
    ETB_LAUNCH_CHECK();
    const uint64_t ntrees = read_u64(reinterpret_cast<uint64_t*>(ctr.get()), s);
    L.tree_count = ntrees;
    sort_keys_u64(rkeys, alt, ntrees, 64, s);
    root_rank_kernel<<<grid_for(ntrees, 256), 256, 0, s>>>(rkeys.get(), ntrees, rank_of.get());
    DevBuf<uint32_t> size(ntrees + 1);
    ETB_CUDA(cudaMemsetAsync(size.get(), 0, (ntrees + 1) * 4, s));
    tree_size_kernel<<<gb, 256, 0, s>>>(type, troot.get(), rank_of.get(), n, size.get());
    ETB_LAUNCH_CHECK();
    DevBuf<uint64_t> off(ntrees + 1), cursor(ntrees + 1);
    exclusive_scan_u32_to_u64(size.get(), off.get(), ntrees + 1, s);
    {
      auto hs = to_host(size.get(), ntrees, s);
      L.max_tree = hs.empty() ? 0 : *std::max_element(hs.begin(), hs.end());
    }
    h_off = to_host(off.get(), ntrees, s);

    // tree vertices by level
    DevBuf<uint64_t> lkeys(nt), lalt;
    DevBuf<unsigned> maxlev(1);
    ETB_CUDA(cudaMemsetAsync(ctr.get(), 0, 8, s));
    ETB_CUDA(cudaMemsetAsync(maxlev.get(), 0, 4, s));
    level_keys_kernel<<<gb, 256, 0, s>>>(type, tdep.get(), tce.get(), n, lkeys.get(), ctr.get(),
                                         maxlev.get());
    ETB_LAUNCH_CHECK();
    unsigned hmax = 0;
    ETB_CUDA(cudaMemcpyAsync(&hmax, maxlev.get(), 4, cudaMemcpyDeviceToHost, s));
    sort_keys_u64(lkeys, lalt, nt, 64, s);
    DevBuf<uint64_t> bounds((uint64_t)hmax + 2);
    level_bounds_kernel<<<grid_for(hmax + 2, 256), 256, 0, s>>>(lkeys.get(), nt, hmax,
                                                                bounds.get());
    ETB_LAUNCH_CHECK();
    auto hb = to_host(bounds.get(), (uint64_t)hmax + 2, s);
    // level 0 = roots
    place_roots_kernel<<<grid_for(hb[1], 256), 256, 0, s>>>(lkeys.get(), hb[1], rank_of.get(),
                                                            off.get(), nc, L.old2new.get(),
                                                            L.new2old.get(), cursor.get());
    ETB_LAUNCH_CHECK();
    DevBuf<uint64_t> ckeys, calt;
    DevBuf<uint32_t> tree_of, head, segstart;
    for (unsigned l = 1; l <= hmax; ++l) {
      const uint64_t b0 = hb[l], cnt = hb[l + 1] - hb[l];
      if (!cnt) continue;
      if (ckeys.size() < cnt) {
        ckeys.alloc(cnt);
        tree_of.alloc(cnt);
        head.alloc(cnt);
        segstart.alloc(cnt);
      }
      const unsigned gl = grid_for(cnt, 256);
      level_child_keys_kernel<<<gl, 256, 0, s>>>(lkeys.get() + b0, cnt, tpar.get(),
                                                 L.old2new.get(), ckeys.get());
      ETB_LAUNCH_CHECK();
      sort_keys_u64(ckeys, calt, cnt, 64, s);
      level_heads_kernel<<<gl, 256, 0, s>>>(ckeys.get(), cnt, troot.get(), rank_of.get(),
                                            tree_of.get(), head.get());
      inclusive_max_scan_u32(head.get(), segstart.get(), cnt, s);
      level_place_kernel<<<gl, 256, 0, s>>>(ckeys.get(), cnt, tree_of.get(), segstart.get(),
                                            cursor.get(), nc, L.old2new.get(), L.new2old.get());
      level_advance_kernel<<<gl, 256, 0, s>>>(tree_of.get(), segstart.get(), cnt, cursor.get());
      ETB_LAUNCH_CHECK();
    }
  }
  // -- isolated vertices ---------------------------------------------------------
  if (L.nz) {
    DevBuf<uint32_t> flag(n1);
    DevBuf<uint64_t> rankv(n1);
    vz_flags_kernel<<<gb, 256, 0, s>>>(type, n, flag.get());
    exclusive_scan_u32_to_u64(flag.get(), rankv.get(), n, s);
    vz_place_kernel<<<gb, 256, 0, s>>>(type, rankv.get(), n, nc + nt, L.old2new.get(),
                                       L.new2old.get());
    ETB_LAUNCH_CHECK();
  }

  // -- relaid per-vertex arrays + edge-tree list ------------------------------------
  L.type.alloc(n1);
  L.degn.alloc(n1);
  L.tsrc.alloc(nt ? nt : 1);
  L.tanchor.alloc(nt ? nt : 1);
  L.tdepth.alloc(nt ? nt : 1);
  relaid_arrays_kernel<<<gb, 256, 0, s>>>(L.new2old.get(), L.old2new.get(), type, g.deg.get(),
                                          tpar.get(), tdep.get(), tce.get(), n, nc, nt,
                                          L.type.get(), L.degn.get(), L.tsrc.get(),
                                          L.tanchor.get(), L.tdepth.get());
  ETB_LAUNCH_CHECK();
  L.h_tsrc = to_host(L.tsrc.get(), nt, s);
  L.h_tdepth = to_host(L.tdepth.get(), nt, s);
  L.h_tanchor = to_host(L.tanchor.get(), nt, s);
  L.h_tree_start.resize(h_off.size());
  for (size_t i = 0; i < h_off.size(); ++i) L.h_tree_start[i] = static_cast<uint32_t>(nc + h_off[i]);

  // -- core-only CSR in new ids ------------------------------------------------------
  L.crow.alloc(nc + 1);
  {
    DevBuf<uint32_t> cnt(nc + 1);
    ETB_CUDA(cudaMemsetAsync(cnt.get(), 0, (nc + 1) * 4, s));
    if (nc) {
      core_count_kernel<<<wgrid(nc), 256, 0, s>>>(g.row.get(), g.col.get(), type,
                                                  L.new2old.get(), nc, cnt.get());
      ETB_LAUNCH_CHECK();
    }
    exclusive_scan_u32_to_u64(cnt.get(), L.crow.get(), nc + 1, s);
  }
  L.ecore = read_u64(L.crow.get() + nc, s);
  L.ccol.alloc(L.ecore ? L.ecore : 1);
  // padded to whole bitmap words (the bottom-up step copies whole words' runs
  // with the TMA engine); the padding reads as "no neighbour"
  L.cfirst.alloc((nc + 31) / 32 * 32 + 32);
  ETB_CUDA(cudaMemsetAsync(L.cfirst.get(), 0xFF, L.cfirst.bytes(), s));
  L.csecond.alloc(nc ? nc : 1);
  L.cthird.alloc(nc ? nc : 1);
  // (csecond keeps a flag in bit 31 of a core id)
  if (nc >= (uint64_t{1} << 31)) throw std::runtime_error("relayout_csr: core of 2^31 vertices or more");
  L.cmeta.alloc(nc ? nc : 1);
  if (L.ecore) {
    // Rows sorted by one key sort of (new src << b | new dst), in buckets of
    // consecutive rows when the whole key array (x2 for the sort) would not fit.
    const int b = bits_for(nc);
    size_t free_b = 0, total_b = 0;
    ETB_CUDA(cudaMemGetInfo(&free_b, &total_b));
    uint64_t cap = L.ecore;
    if (const char* e = std::getenv("ETB_CSR_BUCKET_KEYS")) cap = std::strtoull(e, nullptr, 10);
    else if (L.ecore * 16 > static_cast<uint64_t>(free_b * 0.7))
      cap = static_cast<uint64_t>(free_b * 0.7) / 16;
    auto crow_at = [&](uint64_t i) { return read_u64(L.crow.get() + i, s); };
    DevBuf<uint64_t> keys, alt;
    for (uint64_t lo = 0; lo < nc;) {
      // largest hi with crow[hi] - crow[lo] <= cap (at least one row)
      const uint64_t base = crow_at(lo);
      uint64_t a = lo + 1, e = nc;
      while (a < e) {
        const uint64_t m = (a + e + 1) / 2;
        if (crow_at(m) - base <= cap) a = m; else e = m - 1;
      }
      const uint64_t hi = a;
      const uint64_t nk = crow_at(hi) - base;
      if (nk) {
        if (keys.size() < nk) keys.alloc(nk);
        core_edge_keys_kernel<<<wgrid(hi - lo), 256, 0, s>>>(g.row.get(), g.col.get(), type,
                                                             L.new2old.get(), L.old2new.get(),
                                                             L.crow.get(), lo, hi, b, keys.get());
        ETB_LAUNCH_CHECK();
        sort_keys_u64(keys, alt, nk, 2 * b, s);
        key_cols_kernel<<<grid_for(nk, 256), 256, 0, s>>>(keys.get(), nk, (uint64_t{1} << b) - 1,
                                                          L.ccol.get() + base);
        ETB_LAUNCH_CHECK();
      }
      lo = hi;
    }
  }
  if (nc) {
    first_nbr_kernel<<<grid_for(nc, 256), 256, 0, s>>>(L.crow.get(), L.ccol.get(), L.degn.get(),
                                                       nc, L.cfirst.get(), L.csecond.get(),
                                                       L.cthird.get(), L.cmeta.get());
    ETB_LAUNCH_CHECK();
  }
  core_components(L, s);
  ETB_CUDA(cudaStreamSynchronize(s));
}

void build_full_relabelled(const DevLayout& L, DevBuf<uint64_t>& row, DevBuf<uint32_t>& col,
                           cudaStream_t s) {
  const DevGraph& g = *L.src_graph;
  const uint64_t n = L.n;
  row.alloc(n + 1);
  exclusive_scan_u32_to_u64(L.degn.get(), row.get(), n, s);
  ETB_CUDA(cudaMemcpyAsync(row.get() + n, &g.nnz, 8, cudaMemcpyHostToDevice, s));
  col.alloc(g.nnz ? g.nnz : 1);
  if (!g.nnz) return;
  const int b = bits_for(n);
  DevBuf<uint64_t> keys(g.nnz), alt;
  full_edge_keys_kernel<<<wgrid(n), 256, 0, s>>>(g.row.get(), g.col.get(), L.new2old.get(),
                                                 L.old2new.get(), row.get(), n, b, keys.get());
  ETB_LAUNCH_CHECK();
  sort_keys_u64(keys, alt, g.nnz, 2 * b, s);
  key_cols_kernel<<<grid_for(g.nnz, 256), 256, 0, s>>>(keys.get(), g.nnz, (uint64_t{1} << b) - 1,
                                                       col.get());
  ETB_LAUNCH_CHECK();
  ETB_CUDA(cudaStreamSynchronize(s));
}

}  // namespace etb
