// Algorithmic work of one direction-optimizing traversal, from its result.
//
// The roofline of the timed kernel needs the bytes a DO-BFS with the
// reference's α/β rule must move for THIS root (SURVEY §8(d)'s B_alg counts
// every core edge once; the α/β traversal touches ~2% of them). Given the
// result depths and the direction trace, each level's work follows from the
// reference's step semantics alone (proj/src/bfs.cpp):
//   top-down  (bfs.cpp:61-86)  every frontier vertex (depth == d) scans its core
//             row: one row-bound read + 4 B per core neighbour; each claim
//             writes its result once;
//   bottom-up (bfs.cpp:88-111) every unvisited core vertex (depth > d or
//             unreached) scans its core row in id order until the first
//             neighbour in the frontier (depth == d): the first probe is the
//             contiguous first-neighbour entry (4 B), later probes add the row
//             bounds once and 4 B each;
// plus per level one read of the visited bitmap and one write of the next
// frontier bitmap (bottom-up also reads the frontier bitmap), core-sized
// (nc / 8 bytes each); the tree replay (et_bfs.cpp:14-32: 12 B read per tree
// entry, 4 B anchor depth, 8 B result write), the unreached core fill (8 B per
// unreached core vertex) and the reset of the state bitmaps for the next
// traversal (4 x nc / 8). The level sizes come from the depths, so this is
// independent of how the kernel schedules the work; it runs outside any timed
// region.
#include "bfs.cuh"

namespace etb {
namespace {

constexpr int kMaxWorkLevels = 64;

// Per level L (depth d = base + L) counters: [0] frontier (top-down) or
// unvisited (bottom-up) vertices, [1] core columns read (top-down: whole rows;
// bottom-up: probes beyond the first), [2] claims, [3] bottom-up vertices whose
// first probe missed (row bounds read).
__global__ void work_kernel(const uint64_t* crow, const uint32_t* ccol, const uint2* dp,
                            uint64_t nc, int32_t base, const char* dir, int nl,
                            unsigned long long* out) {
  __shared__ unsigned long long acc[kMaxWorkLevels][4];
  for (int i = threadIdx.x; i < kMaxWorkLevels * 4; i += blockDim.x) (&acc[0][0])[i] = 0;
  __syncthreads();
  for (uint64_t v = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; v < nc;
       v += (uint64_t)gridDim.x * blockDim.x) {
    const int32_t dv = static_cast<int32_t>(dp[v].x);
    const uint64_t rb = crow[v], re = crow[v + 1];
    for (int L = 0; L < nl; ++L) {
      const int32_t d = base + L;
      if (dv == d + 1) atomicAdd(&acc[L][2], 1ull);
      if (dir[L] == 't') {
        if (dv == d) {
          atomicAdd(&acc[L][0], 1ull);
          atomicAdd(&acc[L][1], static_cast<unsigned long long>(re - rb));
        }
      } else if (dv < 0 || dv > d) {
        atomicAdd(&acc[L][0], 1ull);
        uint64_t probes = 0;
        for (uint64_t k = rb; k < re; ++k) {
          ++probes;
          if (static_cast<int32_t>(dp[ccol[k]].x) == d) break;
        }
        if (probes > 1) {
          atomicAdd(&acc[L][1], static_cast<unsigned long long>(probes - 1));
          atomicAdd(&acc[L][3], 1ull);
        }
      }
    }
  }
  __syncthreads();
  for (int i = threadIdx.x; i < kMaxWorkLevels * 4; i += blockDim.x)
    if ((&acc[0][0])[i]) atomicAdd(&out[i], (&acc[0][0])[i]);
}

__global__ void min_core_depth_kernel(const uint2* dp, uint64_t nc, int* out) {
  int m = 0x7FFFFFFF;
  for (uint64_t v = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; v < nc;
       v += (uint64_t)gridDim.x * blockDim.x) {
    const int32_t d = static_cast<int32_t>(dp[v].x);
    if (d >= 0 && d < m) m = d;
  }
  for (int o = 16; o; o >>= 1) m = min(m, __shfl_xor_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0) atomicMin(out, m);
}

}  // namespace

// levels[4 * L + k] as work_kernel's counters, bytes[L] the level's algorithmic
// bytes; returns the total including the replay / fill / reset terms (bytes[nl]).
uint64_t result_work(const DevLayout& L, const uint2* dp, const char* trace, int nl,
                     uint64_t* levels, uint64_t* bytes, cudaStream_t s) {
  if (nl > kMaxWorkLevels) throw std::invalid_argument("etb_result_work: too many levels");
  const uint64_t nc = L.nc;
  DevBuf<int> mn(1);
  const int big = 0x7FFFFFFF;
  ETB_CUDA(cudaMemcpyAsync(mn.get(), &big, 4, cudaMemcpyHostToDevice, s));
  if (nc) {
    min_core_depth_kernel<<<grid_for(nc, 256), 256, 0, s>>>(dp, nc, mn.get());
    ETB_LAUNCH_CHECK();
  }
  int base = big;
  ETB_CUDA(cudaMemcpyAsync(&base, mn.get(), 4, cudaMemcpyDeviceToHost, s));
  DevBuf<char> dir(kMaxWorkLevels);
  DevBuf<unsigned long long> out(kMaxWorkLevels * 4);
  ETB_CUDA(cudaMemsetAsync(out.get(), 0, out.bytes(), s));
  ETB_CUDA(cudaMemcpyAsync(dir.get(), trace, nl, cudaMemcpyHostToDevice, s));
  ETB_CUDA(cudaStreamSynchronize(s));
  std::vector<unsigned long long> h(kMaxWorkLevels * 4, 0);
  if (nc && base != big && nl > 0) {
    work_kernel<<<grid_for(nc, 256), 256, 0, s>>>(L.crow.get(), L.ccol.get(), dp, nc, base,
                                                 dir.get(), nl, out.get());
    ETB_LAUNCH_CHECK();
    ETB_CUDA(cudaMemcpyAsync(h.data(), out.get(), out.bytes(), cudaMemcpyDeviceToHost, s));
    ETB_CUDA(cudaStreamSynchronize(s));
  }
  const uint64_t bm = (nc + 7) / 8;  // one core-sized bitmap
  uint64_t total = 0;
  for (int l = 0; l < nl; ++l) {
    const unsigned long long* c = &h[4 * l];
    uint64_t b;
    if (trace[l] == 't')
      b = 8 * c[0] + 4 * c[1] + 8 * c[2] + 2 * bm;
    else
      b = 4 * c[0] + 8 * c[3] + 4 * c[1] + 8 * c[2] + 3 * bm;
    if (levels)
      for (int k = 0; k < 4; ++k) levels[4 * l + k] = c[k];
    if (bytes) bytes[l] = b;
    total += b;
  }
  // tree replay, unreached core fill, next-traversal state reset
  uint64_t reached = 0;
  for (int l = 0; l < nl; ++l) reached += h[4 * l + 2];
  reached += base != big ? 1 : 0;
  const uint64_t tail = 24 * L.nt + 8 * (nc > reached ? nc - reached : 0) + bm + 4 * bm;
  if (bytes) bytes[nl] = tail;
  return total + tail;
}

}  // namespace etb
