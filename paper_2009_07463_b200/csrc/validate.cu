// GPU tree validation — validate_bfs_tree (proj/src/validate.cpp:95-158,
// rules at proj/include/etbfs/validate.hpp:13-19) on the device, over the WHOLE
// graph (core, trees and isolated vertices), for a result in relaid ids:
//   rule 1  the root is its own parent at depth 0 (and only the root has depth 0)
//   rule 2  chains end at the root: every reached non-root vertex's parent is
//           reached exactly one level up (so chains strictly descend to 0)
//   rule 3  every (child, parent) pair is a graph edge
//   rule 4  no graph edge spans more than one level
//   rule 5  the reached set is the root's component: no edge joins a reached and
//           an unreached vertex; reached <-> has a parent <-> depth >= 0
// Rules 1-5 together make every depth the exact BFS distance, so this checks
// depth bit-exactness at sizes the CPU oracle cannot reach quickly.
#include "internal.cuh"

namespace etb {
namespace {

__global__ void validate_kernel(const uint64_t* row, const uint32_t* col, const uint32_t* new2old,
                                const uint32_t* old2new, const uint2* dp, uint64_t n,
                                uint32_t root, unsigned long long* cnt) {
  const unsigned lane = threadIdx.x & 31;
  const uint64_t warp = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
  const uint64_t nwarps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  unsigned long long bad[5] = {0, 0, 0, 0, 0}, reached = 0;
  for (uint64_t v = warp; v < n; v += nwarps) {
    const uint2 e = dp[v];
    const int32_t dv = static_cast<int32_t>(e.x);
    const uint32_t pv = e.y;
    const bool rv = dv >= 0;
    const uint32_t o = new2old[v];
    if (lane == 0) {
      reached += rv;
      if (v == root) {
        if (pv != root || dv != 0) ++bad[0];
      } else {
        if (rv != (pv != kNone32)) ++bad[4];
        if (rv && dv == 0) ++bad[0];
        if (rv && pv != kNone32) {
          if (pv >= n) {
            ++bad[2];
          } else {
            const int32_t dp_ = static_cast<int32_t>(dp[pv].x);
            if (dp_ < 0 || dp_ + 1 != dv) ++bad[1];
            // rule 3: parent (original id) in the sorted original row of o
            const uint32_t po = new2old[pv];
            uint64_t lo = row[o], hi = row[o + 1];
            while (lo < hi) {
              const uint64_t m = (lo + hi) >> 1;
              if (col[m] < po) lo = m + 1; else hi = m;
            }
            if (lo == row[o + 1] || col[lo] != po) ++bad[2];
          }
        }
      }
    }
    // rules 4 and 5 over v's edges (each undirected edge is seen from both ends;
    // counted once, from the smaller relaid id)
    for (uint64_t k = row[o] + lane; k < row[o + 1]; k += 32) {
      const uint32_t w = old2new[col[k]];
      if (w <= v) continue;
      const int32_t dw = static_cast<int32_t>(dp[w].x);
      const bool rw = dw >= 0;
      if (rv != rw) ++bad[4];
      else if (rv && (dv - dw > 1 || dw - dv > 1)) ++bad[3];
    }
  }
  for (int i = 0; i < 5; ++i) {
    unsigned long long x = bad[i];
    for (int s = 16; s; s >>= 1) x += __shfl_xor_sync(0xffffffffu, x, s);
    if (lane == 0 && x) atomicAdd(&cnt[i], x);
  }
  if (lane == 0 && reached) atomicAdd(&cnt[5], reached);
}

}  // namespace

void validate_result(const DevLayout& L, const uint2* dp, uint64_t root, uint64_t out[6],
                     cudaStream_t s) {
  if (!L.src_graph) throw std::runtime_error("etb_result_validate: the layout's graph is gone");
  const DevGraph& g = *L.src_graph;
  DevBuf<unsigned long long> cnt(6);
  ETB_CUDA(cudaMemsetAsync(cnt.get(), 0, 48, s));
  validate_kernel<<<grid_for(L.n * 32, 256), 256, 0, s>>>(g.row.get(), g.col.get(),
                                                          L.new2old.get(), L.old2new.get(), dp,
                                                          L.n, static_cast<uint32_t>(root),
                                                          cnt.get());
  ETB_LAUNCH_CHECK();
  unsigned long long h[6];
  ETB_CUDA(cudaMemcpyAsync(h, cnt.get(), 48, cudaMemcpyDeviceToHost, s));
  ETB_CUDA(cudaStreamSynchronize(s));
  for (int i = 0; i < 6; ++i) out[i] = h[i];
}

}  // namespace etb
