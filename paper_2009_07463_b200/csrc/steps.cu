// The reference's step and driver layer (proj/include/etbfs/bfs.hpp:66-120,
// proj/src/bfs.cpp:61-305) on the device, for callers that drive a traversal
// level by level with their own FrontierState: top_down_step, bottom_up_step,
// degree_aware_step, block_search_step and the run_top_down / run_hybrid /
// run_block_search drivers, with the same limit semantics (frontier members
// below it, neighbours at or above it skipped), claim rules and counters.
// State is the caller's (64-bit bitmap words, u64 parents): uploaded, stepped
// in HBM, downloaded; a driver keeps it resident for all its levels. These are
// plain per-step kernels — the product traversal is the persistent kernel of
// bfs.cu.
#include <algorithm>

#include "internal.cuh"

namespace etb {
namespace {

using u64 = unsigned long long;
constexpr uint64_t kNo = ~uint64_t{0};

__device__ __forceinline__ bool bit(const u64* bm, uint64_t v) { return (bm[v >> 6] >> (v & 63)) & 1ull; }

struct StepDev {
  const uint64_t* row;
  const uint32_t* col;
  const uint32_t* deg;
  uint64_t limit;
  u64* vis;
  u64* cur;
  u64* nxt;
  uint64_t* parent;
  const uint64_t* in_plus;
  const uint64_t* moff;
  const uint64_t* minus;
  u64* acc;  // [0] claimed [1] scout [2] probes [3] skipped blocks
};

// top_down_step (bfs.cpp:61-86): a warp per frontier vertex, its row (up to the
// first neighbour >= limit) across the lanes; check-then-claim on visited.
__global__ void td_kernel(StepDev s, uint64_t words) {
  const unsigned lane = threadIdx.x & 31;
  const uint64_t warp = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
  const uint64_t nwarps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  u64 claimed = 0, scout = 0;
  for (uint64_t wi = warp; wi < words; wi += nwarps) {
    for (u64 word = s.cur[wi]; word; word &= word - 1) {
      const uint64_t v = wi * 64 + __ffsll(static_cast<long long>(word)) - 1;
      for (uint64_t k = s.row[v] + lane; k < s.row[v + 1]; k += 32) {
        const uint64_t w = s.col[k];
        if (w >= s.limit) break;  // rows ascend: the rest is above the limit too
        const u64 m = 1ull << (w & 63);
        if (!(s.vis[w >> 6] & m) && !(atomicOr(&s.vis[w >> 6], m) & m)) {
          s.parent[w] = v;
          atomicOr(&s.nxt[w >> 6], m);
          ++claimed;
          scout += s.deg[w];
        }
      }
    }
  }
  if (claimed) atomicAdd(&s.acc[0], claimed);
  if (scout) atomicAdd(&s.acc[1], scout);
}

// bottom_up_step (bfs.cpp:88-111): each unvisited vertex below the limit scans
// its row in index order and adopts the first neighbour in the frontier.
__global__ void bu_kernel(StepDev s) {
  u64 claimed = 0, probes = 0;
  for (uint64_t w = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; w < s.limit;
       w += (uint64_t)gridDim.x * blockDim.x) {
    if (bit(s.vis, w)) continue;
    for (uint64_t k = s.row[w]; k < s.row[w + 1]; ++k) {
      const uint64_t x = s.col[k];
      if (x >= s.limit) break;
      ++probes;
      if (bit(s.cur, x)) {
        s.parent[w] = x;
        atomicOr(&s.vis[w >> 6], 1ull << (w & 63));
        atomicOr(&s.nxt[w >> 6], 1ull << (w & 63));
        ++claimed;
        break;
      }
    }
  }
  if (claimed) atomicAdd(&s.acc[0], claimed);
  if (probes) atomicAdd(&s.acc[2], probes);
}

// degree_aware_step (bfs.cpp:113-154): pass one probes in_plus, pass two the
// descending-degree remainder with early exit (two launches: pass two sees pass
// one's claims, as the reference's two loops).
__global__ void da_kernel(StepDev s, int pass) {
  u64 claimed = 0, probes = 0;
  for (uint64_t w = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; w < s.limit;
       w += (uint64_t)gridDim.x * blockDim.x) {
    if (bit(s.vis, w)) continue;
    uint64_t found = kNo;
    if (pass == 0) {
      const uint64_t x = s.in_plus[w];
      if (x == kNo) continue;
      ++probes;
      if (bit(s.cur, x)) found = x;
    } else {
      for (uint64_t k = s.moff[w]; k < s.moff[w + 1]; ++k) {
        ++probes;
        if (bit(s.cur, s.minus[k])) {
          found = s.minus[k];
          break;
        }
      }
    }
    if (found != kNo) {
      s.parent[w] = found;
      atomicOr(&s.vis[w >> 6], 1ull << (w & 63));
      atomicOr(&s.nxt[w >> 6], 1ull << (w & 63));
      ++claimed;
    }
  }
  if (claimed) atomicAdd(&s.acc[0], claimed);
  if (probes) atomicAdd(&s.acc[2], probes);
}

// block_search_step (bfs.cpp:156-220): a thread per 64-vertex block; probes test
// the pre-step visited set (frozen for the sweep), claims are written back as
// one next word per block and folded into visited by fold_kernel afterwards.
__global__ void bs_kernel(StepDev s, uint64_t blocks) {
  u64 claimed = 0, probes = 0, skips = 0;
  for (uint64_t bi = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; bi < blocks;
       bi += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t base = bi * 64;
    u64 vw = s.vis[bi];
    if (base + 64 > s.limit) vw |= ~0ull << (s.limit - base);  // tail reads as visited
    u64 todo = ~vw;
    if (!todo) {
      ++skips;
      continue;
    }
    u64 claims = 0;
    for (; todo; todo &= todo - 1) {
      const int pos = __ffsll(static_cast<long long>(todo)) - 1;
      const uint64_t w = base + pos;
      uint64_t found = kNo;
      const uint64_t plus = s.in_plus[w];
      if (plus != kNo) {
        ++probes;
        if (bit(s.vis, plus)) found = plus;
      }
      if (found == kNo)
        for (uint64_t k = s.moff[w]; k < s.moff[w + 1]; ++k) {
          ++probes;
          if (bit(s.vis, s.minus[k])) {
            found = s.minus[k];
            break;
          }
        }
      if (found != kNo) {
        s.parent[w] = found;
        claims |= 1ull << pos;
        ++claimed;
      }
    }
    if (claims) s.nxt[bi] |= claims;
  }
  if (claimed) atomicAdd(&s.acc[0], claimed);
  if (probes) atomicAdd(&s.acc[2], probes);
  if (skips) atomicAdd(&s.acc[3], skips);
}

__global__ void fold_kernel(u64* vis, const u64* nxt, uint64_t words) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < words;
       i += (uint64_t)gridDim.x * blockDim.x)
    if (nxt[i]) vis[i] |= nxt[i];
}

// Seed frontier of run_hybrid (bfs.cpp:240-251): count and degree sum of the
// current words below words_for(limit).
__global__ void seed_kernel(const u64* cur, const uint32_t* deg, uint64_t words, u64* acc) {
  u64 cnt = 0, sc = 0;
  for (uint64_t wi = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; wi < words;
       wi += (uint64_t)gridDim.x * blockDim.x)
    for (u64 word = cur[wi]; word; word &= word - 1) {
      ++cnt;
      sc += deg[wi * 64 + __ffsll(static_cast<long long>(word)) - 1];
    }
  if (cnt) atomicAdd(&acc[0], cnt);
  if (sc) atomicAdd(&acc[1], sc);
}

// restricted_edge_count (bfs.cpp:50-59): neighbours below the limit of the
// vertices below it.
__global__ void restricted_kernel(const uint64_t* row, const uint32_t* col, uint64_t limit,
                                  u64* acc) {
  u64 t = 0;
  for (uint64_t v = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; v < limit;
       v += (uint64_t)gridDim.x * blockDim.x) {
    uint64_t lo = row[v], hi = row[v + 1];
    const uint64_t b = lo;
    while (lo < hi) {
      const uint64_t m = (lo + hi) >> 1;
      if (col[m] < limit) lo = m + 1; else hi = m;
    }
    t += lo - b;
  }
  if (t) atomicAdd(acc, t);
}

}  // namespace

// ops: 0 top_down_step, 1 bottom_up_step, 2 degree_aware_step, 3 block_search_step,
// 4 run_top_down, 5/6/7 run_hybrid (classic / degree-aware / block-search),
// 8 run_block_search. stats[0..5] += claimed, scout, probes, skipped blocks,
// levels, bottom-up levels; trace gets one char per level (drivers).
void step_run(const DevGraph& g, int op, uint64_t limit, uint64_t* h_vis, uint64_t* h_cur,
              uint64_t* h_nxt, uint64_t* h_parent, const uint64_t* h_in_plus,
              const uint64_t* h_moff, const uint64_t* h_minus, double alpha, double beta,
              uint64_t out[6], std::string* trace, cudaStream_t s) {
  const uint64_t n = g.n;
  const uint64_t words = (n + 63) / 64;
  const uint64_t lwords = (std::min(limit, n) + 63) / 64;
  limit = std::min(limit, n);
  DevBuf<u64> vis(words ? words : 1), cur(words ? words : 1), nxt(words ? words : 1);
  DevBuf<uint64_t> parent(n ? n : 1), in_plus, moff, minus;
  DevBuf<u64> acc(4);
  const size_t wb = words * 8;
  if (words) {
    ETB_CUDA(cudaMemcpyAsync(vis.get(), h_vis, wb, cudaMemcpyHostToDevice, s));
    ETB_CUDA(cudaMemcpyAsync(cur.get(), h_cur, wb, cudaMemcpyHostToDevice, s));
    ETB_CUDA(cudaMemcpyAsync(nxt.get(), h_nxt, wb, cudaMemcpyHostToDevice, s));
  }
  if (n) ETB_CUDA(cudaMemcpyAsync(parent.get(), h_parent, n * 8, cudaMemcpyHostToDevice, s));
  const bool split = op == 2 || op == 3 || op == 6 || op == 7 || op == 8;
  if (split) {
    in_plus.alloc(n ? n : 1);
    moff.alloc(n + 1);
    if (n) ETB_CUDA(cudaMemcpyAsync(in_plus.get(), h_in_plus, n * 8, cudaMemcpyHostToDevice, s));
    ETB_CUDA(cudaMemcpyAsync(moff.get(), h_moff, (n + 1) * 8, cudaMemcpyHostToDevice, s));
    const uint64_t nm = h_moff[n];
    minus.alloc(nm ? nm : 1);
    if (nm) ETB_CUDA(cudaMemcpyAsync(minus.get(), h_minus, nm * 8, cudaMemcpyHostToDevice, s));
  }
  StepDev d{g.row.get(), g.col.get(), g.deg.get(), limit, vis.get(), cur.get(), nxt.get(),
            parent.get(), in_plus.get(), moff.get(), minus.get(), acc.get()};
  u64 totals[4] = {};
  auto read_acc = [&](u64 h[4]) {
    ETB_CUDA(cudaMemcpyAsync(h, acc.get(), 32, cudaMemcpyDeviceToHost, s));
    ETB_CUDA(cudaStreamSynchronize(s));
    for (int i = 0; i < 4; ++i) totals[i] += h[i];
  };
  const unsigned gw = grid_for(lwords * 32, 256), gv = grid_for(limit, 256),
                 gb = grid_for(lwords, 256);
  // one step of kind k (0 td, 1 bu, 2 da, 3 bs); returns {claimed, scout}
  auto step = [&](int k) {
    ETB_CUDA(cudaMemsetAsync(acc.get(), 0, 32, s));
    d.cur = cur.get();
    d.nxt = nxt.get();
    if (k == 0) {
      td_kernel<<<gw, 256, 0, s>>>(d, lwords);
    } else if (k == 1) {
      bu_kernel<<<gv, 256, 0, s>>>(d);
    } else if (k == 2) {
      da_kernel<<<gv, 256, 0, s>>>(d, 0);
      da_kernel<<<gv, 256, 0, s>>>(d, 1);
    } else {
      bs_kernel<<<gb, 256, 0, s>>>(d, lwords);
      fold_kernel<<<gb, 256, 0, s>>>(vis.get(), nxt.get(), lwords);
    }
    ETB_LAUNCH_CHECK();
    u64 h[4];
    read_acc(h);
    return std::make_pair(h[0], h[1]);
  };
  uint64_t levels = 0, bu_levels = 0;
  auto advance = [&](char dir) {  // record_level + FrontierState::advance_level
    ++levels;
    if (dir == 'b') ++bu_levels;
    if (trace) trace->push_back(dir);
    std::swap(cur, nxt);
    ETB_CUDA(cudaMemsetAsync(nxt.get(), 0, wb, s));
  };
  if (op <= 3) {
    step(op);
  } else if (op == 4 || op == 8) {
    for (;;) {
      const auto r = step(op == 4 ? 0 : 3);
      advance(op == 4 ? 't' : 'b');
      if (r.first == 0) break;
    }
  } else {
    const int bk = op == 5 ? 1 : (op == 6 ? 2 : 3);
    DevBuf<u64> a2(2);
    ETB_CUDA(cudaMemsetAsync(a2.get(), 0, 16, s));
    seed_kernel<<<gb, 256, 0, s>>>(cur.get(), g.deg.get(), lwords, a2.get());
    DevBuf<u64> re(1);
    ETB_CUDA(cudaMemsetAsync(re.get(), 0, 8, s));
    restricted_kernel<<<gv, 256, 0, s>>>(g.row.get(), g.col.get(), limit, re.get());
    ETB_LAUNCH_CHECK();
    u64 seed[2], redges = 0;
    ETB_CUDA(cudaMemcpyAsync(seed, a2.get(), 16, cudaMemcpyDeviceToHost, s));
    ETB_CUDA(cudaMemcpyAsync(&redges, re.get(), 8, cudaMemcpyDeviceToHost, s));
    ETB_CUDA(cudaStreamSynchronize(s));
    uint64_t frontier = seed[0], scout = seed[1];
    double etc = static_cast<double>(redges);
    while (frontier > 0) {  // run_hybrid, bfs.cpp:266-292
      if (static_cast<double>(scout) > etc / alpha) {
        uint64_t awake = frontier, prev;
        do {
          prev = awake;
          const auto r = step(bk);
          advance('b');
          awake = r.first;
        } while (awake > 0 && (awake >= prev || static_cast<double>(awake) >
                                                    static_cast<double>(limit) / beta));
        frontier = awake;
        scout = 1;
      } else {
        etc -= static_cast<double>(scout);
        const auto r = step(0);
        advance('t');
        frontier = r.first;
        scout = r.second;
      }
    }
  }
  if (words) {
    ETB_CUDA(cudaMemcpyAsync(h_vis, vis.get(), wb, cudaMemcpyDeviceToHost, s));
    ETB_CUDA(cudaMemcpyAsync(h_cur, cur.get(), wb, cudaMemcpyDeviceToHost, s));
    ETB_CUDA(cudaMemcpyAsync(h_nxt, nxt.get(), wb, cudaMemcpyDeviceToHost, s));
  }
  if (n) ETB_CUDA(cudaMemcpyAsync(h_parent, parent.get(), n * 8, cudaMemcpyDeviceToHost, s));
  ETB_CUDA(cudaStreamSynchronize(s));
  out[0] = totals[0];
  out[1] = totals[1];
  out[2] = totals[2];
  out[3] = totals[3];
  out[4] = levels;
  out[5] = bu_levels;
}

}  // namespace etb

namespace etb {
namespace {

// teet / teolv (et_bfs.cpp:14-32): entry i writes parent[dst] = src when its
// guard vertex (the tree's core edge vertex / the entry's src) is visited and
// dst has no parent yet.
__global__ void replay_kernel(int leaves_only, const uint64_t* src, const uint64_t* dst,
                              const uint64_t* core_edge, uint64_t count,
                              const unsigned long long* vis, uint64_t* parent) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < count;
       i += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t guard = leaves_only ? src[i] : core_edge[i];
    if (guard == ~uint64_t{0}) continue;  // whole-component tree (TEET)
    if (((vis[guard >> 6] >> (guard & 63)) & 1ull) && parent[dst[i]] == ~uint64_t{0})
      parent[dst[i]] = src[i];
  }
}

}  // namespace

void tree_replay_run(int leaves_only, const uint64_t* h_src, const uint64_t* h_dst,
                     const uint64_t* h_ce, uint64_t count, const uint64_t* h_vis, uint64_t words,
                     uint64_t* h_parent, uint64_t n, cudaStream_t s) {
  DevBuf<uint64_t> src(count ? count : 1), dst(count ? count : 1), ce(count ? count : 1),
      parent(n ? n : 1);
  DevBuf<unsigned long long> vis(words ? words : 1);
  if (count) {
    ETB_CUDA(cudaMemcpyAsync(src.get(), h_src, count * 8, cudaMemcpyHostToDevice, s));
    ETB_CUDA(cudaMemcpyAsync(dst.get(), h_dst, count * 8, cudaMemcpyHostToDevice, s));
    ETB_CUDA(cudaMemcpyAsync(ce.get(), h_ce, count * 8, cudaMemcpyHostToDevice, s));
  }
  if (words) ETB_CUDA(cudaMemcpyAsync(vis.get(), h_vis, words * 8, cudaMemcpyHostToDevice, s));
  if (n) ETB_CUDA(cudaMemcpyAsync(parent.get(), h_parent, n * 8, cudaMemcpyHostToDevice, s));
  if (count) {
    replay_kernel<<<grid_for(count, 256), 256, 0, s>>>(leaves_only, src.get(), dst.get(),
                                                       ce.get(), count, vis.get(), parent.get());
    ETB_LAUNCH_CHECK();
  }
  if (n) ETB_CUDA(cudaMemcpyAsync(h_parent, parent.get(), n * 8, cudaMemcpyDeviceToHost, s));
  ETB_CUDA(cudaStreamSynchronize(s));
}

}  // namespace etb
