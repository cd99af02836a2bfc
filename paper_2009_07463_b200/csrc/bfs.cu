// (3)+(4) The ET-BFS traversal on sm_100a: one persistent cooperative kernel
// per root runs the whole of et_bfs (src/et_bfs.cpp:59-124) —
//   start           visited/frontier bitmaps sized to the CORE (not n), double
//                   buffered: this launch runs on a half the previous one
//                   cleaned and cleans the other; only the start bits are set
//                   (et_bfs.cpp:96-98);
//   level loop      the reference's α/β direction-optimizing driver
//                   (src/bfs.cpp:232-293), decided redundantly by every thread
//                   from grid-reduced counters, with no host round trip;
//                     top-down  (bfs.cpp:61-86): merge path — the frontier's
//                               rows concatenated and cut into 128-edge chunks
//                               dealt CTA-minor then grabbed from a counter,
//                               4 edges per lane in flight, check-then-atomicOr
//                               claims staged in smem and appended to the next
//                               list in batches; on the large-core kernel
//                               list-less levels claim with reductions and count
//                               afterwards (td_step);
//                     bottom-up (bfs.cpp:88-111): 8 visited words per warp, lane
//                               = vertex, first probe on the contiguous first-
//                               neighbour array (the highest-degree neighbour,
//                               since relaid ids are degree sorted), deferred
//                               scans for misses (two rows per lane, then the
//                               warp for long rows), one word write-back per
//                               word (bu_step; bu_sweep on late large levels);
//                   and stops once every core vertex is visited (the level the
//                   reference would run next claims nothing);
//   tree replay     TEET/TEOLV (et_bfs.cpp:14-32) as one streaming pass giving
//                   every tree vertex parent = src and depth = depth(anchor) +
//                   tree depth; unreached core vertices get -1 in the same phase;
//   start tree      the start-side walk (et_bfs.cpp:34-57) is precomputed on the
//                   host and applied as a patch (in the launch parameters when
//                   small).
// Levels are separated by a grid barrier; the grid is one CTA per SM
// (cooperative launch). DESIGN.md §4 lists the measured choices.
#include <cstdlib>
#include <algorithm>

#include "bfs_dev.cuh"
#include "bfs_part.cuh"

namespace etb {
namespace {

using namespace dev;

// One CTA per SM, 640 or 1024 threads (et_bfs_kernel<B>): 640 leaves 96
// registers per thread (no spills) and is faster on latency-bound levels
// (small cores), 1024 keeps more probes in flight (large cores); see block_for().
constexpr int kSmallBlock = 640;
constexpr int kMaxWarps = 32;
constexpr int kItemShift = 36;
constexpr unsigned long long kItemMask = (1ull << kItemShift) - 1;

constexpr int kEpl = kTdChunk / 32;  // edges per lane per top-down chunk
constexpr int kCbuf = kTdChunk;      // staged claims of one chunk (u32 vertex ids)
// visited words per warp per bottom-up iteration: 8 on the large-core kernel,
// 7 on the small-core one (s22: 5/6/7 all -0.5..-1 us per root against 8, 7 best)
constexpr int kBuU = 8, kBuUSmall = 7;
constexpr uint64_t kGrab = 4;        // top-down chunks per warp per grab on long levels
// bu_step loads the first neighbours together with the visited words (1) or
// after them, for the unvisited lanes only (0)
#ifndef ETB_BU_EAGER
#define ETB_BU_EAGER 0
#endif
// BfsParams::small_mode3_edges default (env ETB_SMALL_MODE3 overrides)
#ifndef ETB_SMALL_MODE3_DEFAULT
#define ETB_SMALL_MODE3_DEFAULT 2e6  // s22: +0.9% (938.5 vs 930.4 GTEPS; 5e5: neutral)
#endif
constexpr double kSmallMode3Default = ETB_SMALL_MODE3_DEFAULT;
// BfsParams::td_as_bu default (env ETB_TD_AS_BU overrides; 0 = off): s26 +6%
// harmonic-mean GTEPS (slowest roots 0.80 -> 0.62-0.68 ms), s22 neutral
constexpr double kTdAsBuDefault = 4.0;  // measured best at s26 (3..5 equal, 6 and up: no level)
// BfsParams::split_ratio / split_bound = nc / div defaults (env ETB_SPLIT_RATIO,
// ETB_SPLIT_DIV override)
#ifndef ETB_SPLIT_RATIO_DEFAULT
#define ETB_SPLIT_RATIO_DEFAULT 2.0  // s26 +3.8%, s28 +7.7% (1 / 1.5 / 2.5 / 3: +2.2 / 2.8 / 2.9 / 2.4% at s26)
#endif
constexpr double kSplitRatioDefault = ETB_SPLIT_RATIO_DEFAULT;
constexpr uint32_t kSplitAuto = 0xFFFFu;  // split_tdw: chosen per level from the tail's edges
constexpr unsigned long long kSplitShortTail = 1ull << 25;
#ifndef ETB_SPLIT_TDW_DEFAULT
#define ETB_SPLIT_TDW_DEFAULT kSplitAuto
#endif
constexpr uint32_t kSplitTdwDefault = ETB_SPLIT_TDW_DEFAULT;
constexpr double kSplitDivDefault = 1024.0;  // (s26, ratio 2: 512 -0.6%, 2048 -1.1%; ratio 1.5: 256 -0.6%, 4096 -1.2%)

// The step functions below are templates on their parameter view P: BfsParams
// (one partition: the whole core, the whole grid) or PartView (one partition of
// the 1D core partition, et_bfs_part_body: its owned visited words, its CTA
// group, row segments restricted to its owned neighbours). These accessors fold
// to the single-partition expressions for BfsParams.
__device__ __forceinline__ uint64_t wlo_of(const BfsParams&) { return 0; }
__device__ __forceinline__ uint32_t whi_of(const BfsParams& p) { return p.nwords; }
__device__ __forceinline__ unsigned cta_of(const BfsParams&) { return blockIdx.x; }
__device__ __forceinline__ unsigned ncta_of(const BfsParams&) { return gridDim.x; }
__device__ __forceinline__ uint32_t seg_off(const BfsParams&, uint32_t) { return 0; }
// bitmap word of the i-th word a bottom-up step sweeps, and of the k-th word of
// an aligned run of 8 starting at index i0 (run_word: one mapping per run)
__device__ __forceinline__ uint64_t word_at(const BfsParams&, uint64_t i) { return i; }
template <class P> struct IsPart { static constexpr bool value = false; };

struct WarpSmem {
  uint32_t cbuf[kCbuf];     // staged claims (top-down); with win: deferred misses (bottom-up)
  int32_t win[kTdChunk];    // merge-path window: list prefix minus chunk start
};

struct Smem {
  WarpSmem w[kMaxWarps];
  unsigned long long red[2][kMaxWarps];
  unsigned long long tot[4];  // level totals read once per CTA after the barrier
  unsigned int bu_next;       // bottom-up: the CTA's next run (reset at every grid barrier)
  unsigned int bu_bound;      // bounded bottom-up steps: neighbours >= this end a row
  unsigned int pad[2];
};
__device__ __forceinline__ Smem& smem_view() {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  return *reinterpret_cast<Smem*>(smem_raw);
}
// Bottom-up steps of the single-partition kernel hand out their CTA's runs
// (the same runs as the static warp striding) from a shared-memory counter, so
// warps that drew cheap runs take more and the level barrier waits less on the
// warps whose deferred misses were long.
#ifndef ETB_BU_DYN
#define ETB_BU_DYN 1
#endif
// The partitioned kernel's bottom-up steps likewise (its CTA's runs of owned
// words); the CTA's warps then push the CTA's runs after a CTA barrier.
#ifndef ETB_PART_DYN
#define ETB_PART_DYN 1
#endif
static_assert(sizeof(Smem) % 16 == 0, "the bottom-up pipes follow Smem, 16-byte aligned");

// Bottom-up runs fetched by the TMA engine (single-partition kernel, built with
// -DETB_BU_TMA=1): per warp a two-stage ring, each stage one run's first
// neighbours (kU x 32 u32, the contiguous cfirst slice) and the 16-byte-aligned
// span of its visited words, completing on the stage's mbarrier; a run is
// requested two iterations ahead, so the warp's chain per iteration is the
// frontier probe alone. Measured against the plain loads (64 roots x 3 steps,
// every root validated): s26 -1% (2474 vs 2502 GTEPS), s22 -0.3% — the first
// neighbour stream is not what the bottom-up levels wait on, and the 69 KB of
// stages come out of L1, which holds the hub words the probes hit. Off by
// default; kept as the measured alternative.
#ifndef ETB_BU_TMA
#define ETB_BU_TMA 0
#endif
template <int kU>
struct BuStage {
  uint32_t cf[kU * 32];
  uint32_t vw[12];  // kU words + up to 3 words of alignment on each side
};
template <int kU>
struct BuPipe {
  BuStage<kU> st[2];
  uint64_t bar[2];
};
static_assert(sizeof(BuPipe<8>) % 16 == 0 && sizeof(BuPipe<7>) % 16 == 0, "16-byte stages");

// Phase timestamps for stats (block 0 / thread 0): [256] entry, [257] after
// init, [258 + L] after level L, [320 + L] end of a split level's bottom-up
// half, [384 + L] end of a bitmap -> list conversion, [511] end of the tree replay.
__device__ __forceinline__ void stamp(const BfsParams& p, uint32_t slot) {
  if (p.level_claims && blockIdx.x == 0 && threadIdx.x == 0 && slot < 512)
    p.level_claims[slot] = gtimer();
}

// Block-reduce a (and b), add the CTA totals to da (and db), then the grid
// barrier: one bar.sync pair per level instead of three. Thread 0 both adds and
// arrives, so its release add publishes the totals with the CTA's writes; after
// the barrier it alone reads the n level totals at rd (one L2 request per CTA
// instead of one per warp: same-address requests serialise in the L2 slice)
// and hands them to the CTA in sm.tot.
__device__ void grid_sync_add(unsigned long long* bar, Smem& sm, unsigned long long a,
                              unsigned long long* da, unsigned long long b,
                              unsigned long long* db, const unsigned long long* rd, int n) {
  const unsigned lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  if (da) a = warp_sum(a);
  if (db) b = warp_sum(b);
  if (lane == 0) {
    sm.red[0][wib] = a;
    sm.red[1][wib] = b;
  }
  __syncthreads();
  if (threadIdx.x < 32) {
    const unsigned nwb = blockDim.x >> 5;
    if (da) a = warp_sum(lane < nwb ? sm.red[0][lane] : 0ull);
    if (db) b = warp_sum(lane < nwb ? sm.red[1][lane] : 0ull);
    if (lane == 0) {
      if (da && a) atomicAdd(da, a);
      if (db && b) atomicAdd(db, b);
      grid_arrive_wait(bar);
      for (int k = 0; k < n; ++k) sm.tot[k] = ld_volatile(&rd[k]);
    }
    if (threadIdx.x == 0) sm.bu_next = 0;
  }
  __syncthreads();
}

// Frontier list: vertices qv[0..nq) with at least one core edge, and the
// exclusive prefix qp[] of their core degrees (ne = total edges). A top-down
// level cuts the concatenated rows into 128-edge chunks (merge path): hub rows
// span many chunks, tiny rows share one, and every chunk is the same work. Each
// warp takes one chunk, then pulls more from a per-level counter: one at a
// time on levels of at most 8 chunks per warp, kGrab at a time on longer ones.
// Claims append (vertex, edge prefix) with one packed atomic per staged batch:
// slot[0] = (list length << 36) | edges returns both positions at once.

// Append the staged claims to the next list (vertices without core edges skipped).
// kStaged: the claims' core degrees are staged in cdeg (else read from cmeta,
// all loads of the batch in flight at once).
template <bool kStaged, class P>
__device__ void flush_claims(const P& p, const uint32_t* cbuf, const int32_t* cdeg,
                             uint32_t ncl, uint32_t* qv_out, uint64_t* qp_out,
                             unsigned long long* slot) {
  const unsigned lane = threadIdx.x & 31;
  unsigned long long cnt = 0, edges = 0;
  uint32_t d[kCbuf / 32];
#pragma unroll
  for (int k = 0; k < kCbuf / 32; ++k) {
    const uint32_t i = lane + 32 * k;
    d[k] = i >= ncl ? 0u : (kStaged ? static_cast<uint32_t>(cdeg[i]) : p.cmeta[cbuf[i]].x);
  }
#pragma unroll
  for (int k = 0; k < kCbuf / 32; ++k) {
    cnt += d[k] != 0;
    edges += d[k];
  }
  cnt = warp_sum(cnt);
  edges = warp_sum(edges);
  if (cnt == 0) return;
  unsigned long long old = 0;
  if (lane == 0) old = atomicAdd(slot, (cnt << kItemShift) | edges);
  old = __shfl_sync(0xffffffffu, old, 0);
  uint64_t vpos = old >> kItemShift, epos = old & kItemMask;
#pragma unroll
  for (int k = 0; k < kCbuf / 32; ++k) {
    if (32u * k >= ncl) break;  // warp-uniform
    const uint32_t i = lane + 32 * k;
    const uint32_t v = i < ncl ? cbuf[i] : 0u;
    const uint32_t take = d[k] != 0;
    const uint32_t kin = warp_incl_scan(take), din = warp_incl_scan(d[k]);
    if (take) {
      ETB_DCHECK(vpos + kin - 1 <= p.nc && v < p.nc);
      qv_out[vpos + kin - 1] = v;
      qp_out[vpos + kin - 1] = epos + din - d[k];
    }
    vpos += __shfl_sync(0xffffffffu, kin, 31);
    epos += __shfl_sync(0xffffffffu, din, 31);
  }
}

// Largest k with win[k] <= rel (win[0] <= 0 <= rel; win is nondecreasing).
__device__ __forceinline__ uint32_t win_search(const int32_t* win, int32_t rel) {
  uint32_t lo = 0, hi = kTdChunk;
  while (hi - lo > 1) {
    const uint32_t m = (lo + hi) >> 1;
    if (win[m] <= rel) lo = m; else hi = m;
  }
  return lo;
}

// Top-down step (bfs.cpp:61-86). Each lane owns 4 edges of the warp's chunk;
// their column loads, visited probes and claim atomics are issued before any
// result is consumed.
// kMode: 0 no list, 3 no list and no claim atomics returning (claims and scout
// counted after the level by scout_pass), 1 list (flush reads the degrees), 2 list with every
// target's degrees fetched alongside its visited word (early levels, where most
// targets are unvisited; after bottom-up most are visited and mode 1 is used).
template <int kMode, bool kLarge, class P>
__device__ void td_step(const P& p, uint32_t* cbuf, int32_t* win, const uint32_t* qv,
                        const uint64_t* qp, uint64_t nq, uint64_t ne, uint32_t* qv_out,
                        uint64_t* qp_out, uint32_t* fnext, unsigned long long* slot,
                        int32_t dnext, unsigned long long& scout_acc,
                        unsigned long long& claims_acc, uint32_t root, unsigned tdw = 0) {
  const unsigned lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  // tdw != 0: only the CTA's first tdw warps take part (a split level's
  // top-down half; the others are already in its bottom-up half)
  if (tdw && wib >= tdw) return;
  const uint64_t gw = (uint64_t)wib * ncta_of(p) + cta_of(p);  // CTA-minor: spread over SMs
  const uint64_t nw = tdw ? (uint64_t)ncta_of(p) * tdw : (uint64_t)(ncta_of(p) * blockDim.x) >> 5;
  const unsigned lt = (1u << lane) - 1;
  const uint64_t nu = (ne + kTdChunk - 1) / kTdChunk;
  for (uint64_t g0 = gw, gn = 1; g0 < nu;) {
    const uint64_t g1 = min(nu, g0 + gn);
    // root != kNone32: the first level, whose list is the start alone (not stored)
#ifdef ETB_WARP_STAMPS
    const bool rec = p.wstamp && dnext == p.wdepth && g0 == gw;
    unsigned long long* ws = p.wstamp + 8 * ((uint64_t)blockIdx.x * (blockDim.x >> 5) + wib);
    const long long c0 = clock64();
    if (rec && lane == 0) ws[0] = gtimer();
#endif
    uint64_t i = root != kNone32 ? 0 : find_vertex(qp, nq, g0 * kTdChunk);
    for (uint64_t c = g0; c < g1; ++c) {
      const uint64_t e0 = c * kTdChunk, e1 = min(ne, e0 + kTdChunk);
      const uint64_t qi = root != kNone32 ? 0 : qp[i];
      const uint64_t iend = root != kNone32 ? ne : (i + 1 < nq ? qp[i + 1] : ne);
      const bool single = iend >= e1;
#ifdef ETB_WARP_STAMPS
      if (rec && c == g0 && lane == 0) {
        ws[1] = clock_after(static_cast<uint32_t>(qi ^ iend)) - c0;
        ws[6] = c;
        ws[7] = single;
      }
#endif
      uint64_t inext;
      if (!single) {
        for (uint32_t k = lane; k < kTdChunk; k += 32) {
          const uint64_t ii = i + k;
          int32_t wv = 0x7FFFFFFF;
          if (ii < nq) {
            const uint64_t q = qp[ii];
            wv = q <= e0 ? (k == 0 ? 0 : -1) : (q - e0 > kTdChunk ? 0x7FFFFFFF : (int32_t)(q - e0));
          }
          win[k] = wv;
        }
        __syncwarp();
        // the row holding the next chunk's first edge; a chunk of 128 one-edge
        // rows ends exactly where row i + 128 starts, one past the window
        const uint32_t kk = win_search(win, kTdChunk);
        inext = i + kk;
        if (kk == kTdChunk - 1 && win[kk] < static_cast<int32_t>(kTdChunk) && inext + 1 < nq &&
            qp[inext + 1] <= e1)
          inext += 1;
      } else {
        inext = iend == e1 ? i + 1 : i;
      }
      // vertex and column position of each of the lane's 8 edges
      uint32_t u[kEpl], w[kEpl], vw[kEpl];
      bool cl[kEpl];
      if (single) {  // one row: its vertex and row start once for the chunk
        const uint32_t uu = root != kNone32 ? root : qv[i];
        const uint64_t base = p.crow[uu] + seg_off(p, uu) + (e0 - qi);
        ETB_DCHECK(uu < p.nc && base + (e1 - e0) <= p.crow[uu + 1]);
#pragma unroll
        for (int j = 0; j < kEpl; ++j) {
          const uint32_t rel = lane + 32 * j;
          u[j] = rel < e1 - e0 ? uu : kNone32;
          w[j] = u[j] != kNone32 ? p.ccol[base + rel] : kNone32;
        }
      } else {
        uint32_t k = win_search(win, static_cast<int32_t>(lane));
#pragma unroll
        for (int j = 0; j < kEpl; ++j) {
          const uint32_t rel = lane + 32 * j;
          while (k + 1 < kTdChunk && win[k + 1] <= static_cast<int32_t>(rel)) ++k;
          u[j] = rel < e1 - e0 ? qv[i + k] : kNone32;
          w[j] = static_cast<uint32_t>(k);  // relative vertex index for now
        }
#pragma unroll
        for (int j = 0; j < kEpl; ++j) {
          const uint32_t rel = lane + 32 * j;
          uint32_t col = kNone32;
          if (u[j] != kNone32) {
            const uint64_t vs = w[j] == 0 ? qi : e0 + static_cast<uint64_t>(max(win[w[j]], 0));
          ETB_DCHECK(u[j] < p.nc && e0 + rel >= vs &&
                     p.crow[u[j]] + seg_off(p, u[j]) + (e0 + rel - vs) < p.crow[u[j] + 1]);
            col = p.ccol[p.crow[u[j]] + seg_off(p, u[j]) + (e0 + rel - vs)];
          }
          w[j] = col;
        }
      }
#pragma unroll
      for (int j = 0; j < kEpl; ++j) ETB_DCHECK(w[j] == kNone32 || w[j] < p.nc);
      // With a list to emit (small frontiers) every target's {core, full}
      // degree is fetched with its visited word, off the claim's critical path;
      // without one only the claimed targets' full degree is read.
#ifdef ETB_WARP_STAMPS
      if (rec && c == g0 && lane == 0) ws[2] = clock_after(w[0] ^ w[1] ^ w[2] ^ w[3]) - c0;
#endif
      constexpr bool kEmit = kMode == 1 || kMode == 2, kPre = kMode == 2;
      uint2 mt[kPre ? kEpl : 1];
#pragma unroll
      for (int j = 0; j < kEpl; ++j) {
        // (mode 3 has no atomic return to fall back on: its probe reads L2, the
        // point of coherence, so an earlier level's claim is never missed)
        vw[j] = w[j] == kNone32 ? ~0u
                                : (kMode == 3 ? __ldcg(&p.visited[w[j] >> 5]) : p.visited[w[j] >> 5]);
        if (kPre) mt[j] = w[j] != kNone32 ? p.cmeta[w[j]] : make_uint2(0u, 0u);
      }
      if (kMode == 3) {
        // Atomic-free claims: every edge to a target that is unvisited at its
        // probe sets the target's visited and next-frontier bits (reductions,
        // no return) and writes its depth and parent; racing writers of one
        // target store the same depth and each a valid frontier parent. The
        // claims and scout are counted from the new frontier bitmap afterwards.
#pragma unroll
        for (int j = 0; j < kEpl; ++j) {
          const uint32_t bit = 1u << (w[j] & 31);
          cl[j] = false;
          if (!(vw[j] & bit)) {
            atomicOr(&p.visited[w[j] >> 5], bit);
            atomicOr(&fnext[w[j] >> 5], bit);
            p.dp[w[j]] = make_uint2(static_cast<uint32_t>(dnext), u[j]);
          }
        }
      } else {
#pragma unroll
        for (int j = 0; j < kEpl; ++j) {
          const uint32_t bit = 1u << (w[j] & 31);
          cl[j] = false;
          if (!(vw[j] & bit)) cl[j] = !(atomicOr(&p.visited[w[j] >> 5], bit) & bit);
        }
      }
#ifdef ETB_WARP_STAMPS
      if (rec && c == g0 && lane == 0) {
        ws[3] = clock_after(vw[0] ^ vw[1] ^ vw[2] ^ vw[3]) - c0;
        ws[4] = clock_after(cl[0] | cl[1] | cl[2] | cl[3]) - c0;
      }
#endif
      uint32_t dg[kEpl];
#pragma unroll
      for (int j = 0; j < kEpl; ++j) {
        dg[j] = 0;
        if (cl[j]) {
          p.dp[w[j]] = make_uint2(static_cast<uint32_t>(dnext), u[j]);
          atomicOr(&fnext[w[j] >> 5], 1u << (w[j] & 31));
          dg[j] = kPre ? mt[j].y : p.degn[w[j]];
        }
      }
      uint32_t ncl = 0;
      if (kPre) __syncwarp();  // the window is free: it stages the claims' core degrees
#pragma unroll
      for (int j = 0; j < kEpl; ++j) {
        scout_acc += dg[j];
        claims_acc += cl[j];
        if (kEmit) {
          const unsigned m = __ballot_sync(0xffffffffu, cl[j]);
          if (cl[j]) {
            cbuf[ncl + __popc(m & lt)] = w[j];
            if (kPre) win[ncl + __popc(m & lt)] = static_cast<int32_t>(mt[kPre ? j : 0].x);
          }
          ncl += __popc(m);
        }
      }
      if (kEmit && ncl) {
        __syncwarp();
        flush_claims<kPre>(p, cbuf, win, ncl, qv_out, qp_out, slot);
      }
      __syncwarp();
#ifdef ETB_WARP_STAMPS
      if (rec && c == g0 && lane == 0) ws[5] = clock64() - c0;
#endif
      i = inext;
    }
    if (nu <= nw) break;
    unsigned long long next = 0;
    // single chunks when the level is only a few chunks per warp (balance),
    // batches when it is long (fewer atomics on the shared counter)
    // Large-core kernel: guided grabs, 4..16 chunks shrinking with the chunks
    // left (estimated from this warp's last grab). On the s26 levels with
    // ~10^6 chunks the per-level counter is one L2 address: grabs of 4 kept it
    // saturated (one atomic per ~1.7 ns), grabs of 2 cost +20%, static ranges
    // +15% (imbalance); guided 4..16 measured -10% per root (538 -> 485 us).
    const uint64_t rem = nu - min(nu, g1);
    const uint64_t want = nu <= 8 * nw ? 1
                          : kLarge ? max(kGrab, min(uint64_t{16}, rem / (4 * nw)))
                                   : kGrab;
    if (lane == 0) next = nw + atomicAdd(&slot[2], (unsigned long long)want);
    g0 = __shfl_sync(0xffffffffu, next, 0);
    gn = want;
  }
}

// Bottom-up step (bfs.cpp:88-111). A warp takes kBuU consecutive visited words
// per iteration, lane = one vertex of each; all first-neighbour probes of the
// kBuU words are in flight together and each word is written back once.
// Vertices whose first (highest-degree) neighbour is not in the frontier are
// deferred to a per-warp smem list and scanned afterwards: one lane per vertex
// over the next kLaneFirst neighbours (early exit usually comes within a few
// probes), then the whole warp per vertex for the rest of a row that has not
// hit yet (so one long miss no longer holds a lane for hundreds of round
// trips; measured against lane-only scans up to 1024 neighbours: -0.5 us per
// root at s22, -2 us at s26).
constexpr int kMissCap = 2 * kCbuf;  // u32 entries per warp (the claim buffer + the window)
// deferred misses are resolved once more than this many are pending (or the buffer is full)
#ifndef ETB_MISS_FLUSH
#define ETB_MISS_FLUSH 1024
#endif
constexpr int kMissFlush = ETB_MISS_FLUSH;
#ifndef ETB_LANE_FIRST
#define ETB_LANE_FIRST 64
#endif
constexpr uint32_t kLaneFirst = ETB_LANE_FIRST;
// csecond entries: the second core neighbour; bit 31 set when it ends the row
// (cthird: the third and fourth, likewise; ETB_MISS_THIRD = 0 skips that stage)
#ifndef ETB_MISS_THIRD
#define ETB_MISS_THIRD 1
#endif
constexpr uint32_t kSecondMask = 0x7FFFFFFFu;
// bu_sweep on the large-core kernel once fewer than nc / kSweepT vertices are
// unvisited (measured at s26: 2 best, -5 us per root; inlined — out of line its
// call cost the rest of the kernel 3%)
#ifndef ETB_SWEEP_T
#define ETB_SWEEP_T 2.0
#endif
constexpr double kSweepT = ETB_SWEEP_T;

// Bottom-up list emission (a level predicted to hand over to top-down): the
// warp appends its claims, up to K per lane, to the next frontier list with one
// packed atomic, so the level after it needs no bitmap -> list conversion.
template <int K>
__device__ __forceinline__ void bu_append(const uint32_t (&v)[K], const uint32_t (&d)[K],
                                          uint32_t* qv_out, uint64_t* qp_out,
                                          unsigned long long* lslot) {
  const unsigned lane = threadIdx.x & 31;
  uint32_t c = 0;
  unsigned long long e = 0;
#pragma unroll
  for (int k = 0; k < K; ++k) {
    c += d[k] != 0;
    e += d[k];
  }
  if (!__any_sync(0xffffffffu, c != 0)) return;
  const uint32_t cin = warp_incl_scan(c);
  const unsigned long long ein = warp_incl_scan64(e);
  unsigned long long old = 0;
  if (lane == 31) old = atomicAdd(lslot, ((unsigned long long)cin << kItemShift) | ein);
  old = __shfl_sync(0xffffffffu, old, 31);
  uint64_t vpos = (old >> kItemShift) + cin - c, epos = (old & kItemMask) + ein - e;
#pragma unroll
  for (int k = 0; k < K; ++k) {
    if (!d[k]) continue;
    qv_out[vpos] = v[k];
    qp_out[vpos] = epos;
    ++vpos;
    epos += d[k];
  }
}

// Two rows scanned together by one lane, two probes each per round trip (the
// same four loads in flight as one row scanned four at a time), each row with
// its own early exit: a lane resolves two deferred vertices per pass (half
// the passes: s22 -1.3 us, s26 -14 us per root; a generic K-row version and
// four rows spilled).
// kBound: neighbours >= bound end the row (ta / tb report it).
template <bool kBound = false, class P>
__device__ __forceinline__ void scan_rows2(const P& p, const uint32_t* fcur, uint64_t ea,
                                           uint64_t enda, uint64_t eb, uint64_t endb,
                                           uint32_t& pa, uint32_t& pb, bool& ha, bool& hb,
                                           uint32_t bound = kNone32, bool* ta = nullptr,
                                           bool* tb = nullptr) {
  ha = hb = false;
  while (ea < enda || eb < endb) {
    ETB_DCHECK(enda <= p.crow[p.nc] && endb <= p.crow[p.nc]);
    uint32_t x0 = ea < enda ? p.ccol[ea] : kNone32;
    uint32_t x1 = ea + 1 < enda ? p.ccol[ea + 1] : kNone32;
    uint32_t y0 = eb < endb ? p.ccol[eb] : kNone32;
    uint32_t y1 = eb + 1 < endb ? p.ccol[eb + 1] : kNone32;
    if (kBound) {  // rows ascend: the first neighbour past the bound ends the scan
      if (ea < enda && (x0 >= bound || x1 >= bound)) {
        if (x0 >= bound) x0 = kNone32;
        x1 = kNone32;
        *ta = true;
        enda = ea + 2;  // this pair is the row's last
      }
      if (eb < endb && (y0 >= bound || y1 >= bound)) {
        if (y0 >= bound) y0 = kNone32;
        y1 = kNone32;
        *tb = true;
        endb = eb + 2;
      }
    }
    const bool bx0 = x0 != kNone32 && test_bit(fcur, x0);
    const bool bx1 = x1 != kNone32 && test_bit(fcur, x1);
    const bool by0 = y0 != kNone32 && test_bit(fcur, y0);
    const bool by1 = y1 != kNone32 && test_bit(fcur, y1);
    if (bx0 || bx1) {
      pa = bx0 ? x0 : x1;
      ha = true;
      enda = ea;
    } else {
      ea += 2;
    }
    if (by0 || by1) {
      pb = by0 ? y0 : y1;
      hb = true;
      endb = eb;
    } else {
      eb += 2;
    }
  }
}

// Diagnostics (-DETB_MISS_CYCLES builds only): per depth d (mod 64), the warp
// cycles spent in bottom-up steps [d] and in their miss resolution [64 + d],
// read with etb_debug_diag.
// [128 + d % 32] deferred vertices, [160 + ..] rows scanned past the second
// neighbour, [192 + ..] rows scanned by the whole warp, [224 + ..] the warp's
// 32-edge rounds on them, [256 + d] the slowest warp's miss-resolution cycles.
constexpr int kDiag = 320;
__device__ unsigned long long g_diag[kDiag];
#ifdef ETB_MISS_CYCLES
#define ETB_DIAG_BEGIN() const long long diag_c0 = clock64()
#define ETB_DIAG_END(slot)                                                            \
  do {                                                                                \
    if ((threadIdx.x & 31) == 0) {                                                    \
      const unsigned long long dc = clock64() - diag_c0;                              \
      atomicAdd(&g_diag[(slot) & 127], dc);                                           \
      if ((slot) >= 64) atomicMax(&g_diag[256 + ((slot) & 63)], dc);                  \
    }                                                                                 \
  } while (0)
#define ETB_DIAG_COUNT(slot, n)                                                       \
  do {                                                                                \
    if ((threadIdx.x & 31) == 0) atomicAdd(&g_diag[slot], (unsigned long long)(n));   \
  } while (0)
#else
#define ETB_DIAG_BEGIN() (void)0
#define ETB_DIAG_END(slot) (void)0
#define ETB_DIAG_COUNT(slot, n) (void)0
#endif

// Row scans of deferred vertices whose first `skip` neighbours missed.
// (kBound: a row ends at its first neighbour >= the CTA's bu_bound.)
template <bool kBound = false, class P>
__device__ void resolve_rows(const P& p, const uint32_t* fcur, uint32_t* fnext,
                             uint32_t* mbuf, uint32_t nmiss, int32_t dnext,
                             unsigned long long& claims_acc, uint32_t* qv_out,
                             uint64_t* qp_out, unsigned long long* lslot, uint32_t skip,
                             unsigned long long* scout) {
  const unsigned lane = threadIdx.x & 31;
  unsigned long long sc = 0;  // Σ full degree of the claims (when scout is wanted)
  [[maybe_unused]] const uint32_t bound = kBound ? smem_view().bu_bound : kNone32;
  __syncwarp();
  ETB_DIAG_COUNT(160 + (dnext & 31), nmiss);
  uint32_t nlong = 0;
  for (uint32_t i0 = 0; i0 < nmiss; i0 += 64) {
    const uint32_t va = i0 + lane < nmiss ? mbuf[i0 + lane] : kNone32;
    const uint32_t vb = i0 + 32 + lane < nmiss ? mbuf[i0 + 32 + lane] : kNone32;
    // the row bounds give the degrees too: one round trip before the scans
    uint64_t rba = 0, rea = 0, rbb = 0, reb = 0;
    if (va != kNone32) rba = p.crow[va], rea = p.crow[va + 1];
    if (vb != kNone32) rbb = p.crow[vb], reb = p.crow[vb + 1];
    const uint64_t la = min(rea, rba + skip + kLaneFirst), lb = min(reb, rbb + skip + kLaneFirst);
    uint32_t pa = 0, pb = 0;
    bool ha, hb;
    bool ta = false, tb = false;
    scan_rows2<kBound>(p, fcur, rba + skip, va != kNone32 ? la : 0, rbb + skip,
                       vb != kNone32 ? lb : 0, pa, pb, ha, hb, bound, &ta, &tb);
    const bool lnga = va != kNone32 && !ha && !ta && la < rea;
    const bool lngb = vb != kNone32 && !hb && !tb && lb < reb;
    if (ha) {
      p.dp[va] = make_uint2(static_cast<uint32_t>(dnext), pa);
      atomicOr(&p.visited[va >> 5], 1u << (va & 31));
      atomicOr(&fnext[va >> 5], 1u << (va & 31));
      ++claims_acc;
      if (scout) sc += p.degn[va];
    }
    if (hb) {
      p.dp[vb] = make_uint2(static_cast<uint32_t>(dnext), pb);
      atomicOr(&p.visited[vb >> 5], 1u << (vb & 31));
      atomicOr(&fnext[vb >> 5], 1u << (vb & 31));
      ++claims_acc;
      if (scout) sc += p.degn[vb];
    }
    if (lslot) {
      const uint32_t av[2] = {va, vb};
      const uint32_t ad[2] = {ha ? static_cast<uint32_t>(rea - rba) : 0u,
                              hb ? static_cast<uint32_t>(reb - rbb) : 0u};
      bu_append<2>(av, ad, qv_out, qp_out, lslot);
    }
    // compact long rows (no hit in the lane-scanned prefix) to the front of the
    // buffer (slots < i0 + 64 are already read)
    __syncwarp();
    const unsigned lma = __ballot_sync(0xffffffffu, lnga);
    if (lnga) mbuf[nlong + __popc(lma & ((1u << lane) - 1))] = va;
    nlong += __popc(lma);
    const unsigned lmb = __ballot_sync(0xffffffffu, lngb);
    if (lngb) mbuf[nlong + __popc(lmb & ((1u << lane) - 1))] = vb;
    nlong += __popc(lmb);
    __syncwarp();
  }
  ETB_DIAG_COUNT(192 + (dnext & 31), nlong);
  for (uint32_t i = 0; i < nlong; ++i) {
    const uint32_t v = mbuf[i];
    const uint64_t rb = p.crow[v] + skip + kLaneFirst, re = p.crow[v + 1];
    uint32_t par = kNone32;
    for (uint64_t e0 = rb; e0 < re; e0 += 32) {
      ETB_DIAG_COUNT(224 + (dnext & 31), 1);
      const uint64_t e = e0 + lane;
      uint32_t x = e < re ? p.ccol[e] : kNone32;
      const unsigned over = kBound ? __ballot_sync(0xffffffffu, e < re && x >= bound) : 0u;
      if (kBound && x >= bound) x = kNone32;
      const unsigned m = __ballot_sync(0xffffffffu, x != kNone32 && test_bit(fcur, x));
      if (m) {
        par = __shfl_sync(0xffffffffu, x, __ffs(m) - 1);
        break;
      }
      if (over) break;
    }
    if (lane == 0 && par != kNone32) {
      p.dp[v] = make_uint2(static_cast<uint32_t>(dnext), par);
      atomicOr(&p.visited[v >> 5], 1u << (v & 31));
      atomicOr(&fnext[v >> 5], 1u << (v & 31));
      ++claims_acc;
      if (scout) sc += p.degn[v];
    }
    if (lslot) {
      const uint32_t av[1] = {v}, ad[1] = {lane == 0 && par != kNone32 ? p.cmeta[v].x : 0u};
      bu_append<1>(av, ad, qv_out, qp_out, lslot);
    }
  }
  __syncwarp();
  if (scout) *scout += sc;
}

// Deferred misses: vertices whose first (highest-degree) neighbour is not in
// the frontier. Stage 1 probes every one's SECOND neighbour, four vertices per
// lane, from the layout's csecond array (bit 31: it is the row's last) — one
// gather and one probe per 128 vertices, no row-offset round trip; most core
// rows missing their first neighbour have two entries (the ET relayout moved
// the tree-like vertices out of the core), so this settles most of them.
// Stage 2 (resolve_rows) scans the rest of the longer rows. (Measured against
// a load-balanced warp scan of the rows, 128 edges per round trip: 1.7x slower
// for all misses, 1.14x for the rows past the second neighbour — its window
// bookkeeping is ~50 shuffles per round and a round covers 32 rows, not 64.)
template <bool kBound = false, class P>
__device__ void resolve_misses(const P& p, const uint32_t* fcur, uint32_t* fnext,
                               uint32_t* mbuf, uint32_t nmiss, int32_t dnext,
                               unsigned long long& claims_acc, uint32_t* qv_out,
                               uint64_t* qp_out, unsigned long long* lslot,
                               unsigned long long* scout) {
  const unsigned lane = threadIdx.x & 31, lt = (1u << lane) - 1;
  unsigned long long sc2 = 0;
  [[maybe_unused]] const uint32_t bound = kBound ? smem_view().bu_bound : kNone32;
  __syncwarp();
  ETB_DIAG_BEGIN();
  ETB_DIAG_COUNT(128 + (dnext & 31), nmiss);
  uint32_t nlong = 0;
  for (uint32_t i0 = 0; i0 < nmiss; i0 += 128) {
    uint32_t v[4], sc[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const uint32_t i = i0 + lane + 32u * k;
      v[k] = i < nmiss ? mbuf[i] : kNone32;
    }
#pragma unroll
    for (int k = 0; k < 4; ++k) sc[k] = v[k] != kNone32 ? p.csecond[v[k]] : kNone32;
    if (kBound) {  // a second neighbour past the bound: the row has ended
#pragma unroll
      for (int k = 0; k < 4; ++k)
        if (sc[k] != kNone32 && (sc[k] & kSecondMask) >= bound) sc[k] = kNone32;
    }
    bool h[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) h[k] = sc[k] != kNone32 && test_bit(fcur, sc[k] & kSecondMask);
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      if (!h[k]) continue;
      p.dp[v[k]] = make_uint2(static_cast<uint32_t>(dnext), sc[k] & kSecondMask);
      atomicOr(&p.visited[v[k] >> 5], 1u << (v[k] & 31));
      atomicOr(&fnext[v[k] >> 5], 1u << (v[k] & 31));
      ++claims_acc;
      if (scout) sc2 += p.degn[v[k]];
    }
    if (lslot) {
      uint32_t ad[4];
#pragma unroll
      for (int k = 0; k < 4; ++k) ad[k] = h[k] ? ((sc[k] >> 31) ? 2u : p.cmeta[v[k]].x) : 0u;
      bu_append<4>(v, ad, qv_out, qp_out, lslot);
    }
    // rows with more than two entries and no hit yet go on to the row scans,
    // compacted to the front of the buffer (slots < i0 + 128 are already read)
    __syncwarp();
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const bool more = v[k] != kNone32 && !h[k] && sc[k] != kNone32 && !(sc[k] >> 31);
      const unsigned m = __ballot_sync(0xffffffffu, more);
      if (more) mbuf[nlong + __popc(m & lt)] = v[k];
      nlong += __popc(m);
    }
    __syncwarp();
  }
#if ETB_MISS_THIRD
  // Stage 2: the rows past their second neighbour probe the third and fourth
  // (cthird, one 8-byte gather), four rows per lane; rows of five or more
  // entries with no hit yet go on to the row scans.
  uint32_t nl2 = 0;
  for (uint32_t i0 = 0; i0 < nlong; i0 += 128) {
    uint32_t v[4];
    uint2 t3[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const uint32_t i = i0 + lane + 32u * k;
      v[k] = i < nlong ? mbuf[i] : kNone32;
    }
#pragma unroll
    for (int k = 0; k < 4; ++k) t3[k] = v[k] != kNone32 ? p.cthird[v[k]] : make_uint2(kNone32, kNone32);
    if (kBound) {
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        if (t3[k].x != kNone32 && (t3[k].x & kSecondMask) >= bound) t3[k] = make_uint2(kNone32, kNone32);
        else if (t3[k].y != kNone32 && (t3[k].y & kSecondMask) >= bound) t3[k].y = kNone32;
      }
    }
    bool h3[4], h4[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      h3[k] = t3[k].x != kNone32 && test_bit(fcur, t3[k].x & kSecondMask);
      h4[k] = t3[k].y != kNone32 && test_bit(fcur, t3[k].y & kSecondMask);
    }
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      if (!h3[k] && !h4[k]) continue;
      const uint32_t par = (h3[k] ? t3[k].x : t3[k].y) & kSecondMask;
      p.dp[v[k]] = make_uint2(static_cast<uint32_t>(dnext), par);
      atomicOr(&p.visited[v[k] >> 5], 1u << (v[k] & 31));
      atomicOr(&fnext[v[k] >> 5], 1u << (v[k] & 31));
      ++claims_acc;
      if (scout) sc2 += p.degn[v[k]];
    }
    if (lslot) {
      uint32_t ad[4];
#pragma unroll
      for (int k = 0; k < 4; ++k) ad[k] = (h3[k] || h4[k]) ? p.cmeta[v[k]].x : 0u;
      bu_append<4>(v, ad, qv_out, qp_out, lslot);
    }
    __syncwarp();
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      // five or more entries: the fourth exists and is not flagged as the last
      const bool more = v[k] != kNone32 && !h3[k] && !h4[k] && t3[k].y != kNone32 &&
                        !(t3[k].y >> 31);
      const unsigned mk = __ballot_sync(0xffffffffu, more);
      if (more) mbuf[nl2 + __popc(mk & lt)] = v[k];
      nl2 += __popc(mk);
    }
    __syncwarp();
  }
  if (nl2)
    resolve_rows<kBound>(p, fcur, fnext, mbuf, nl2, dnext, claims_acc, qv_out, qp_out, lslot, 4,
                         scout);
#else
  if (nlong)
    resolve_rows<kBound>(p, fcur, fnext, mbuf, nlong, dnext, claims_acc, qv_out, qp_out, lslot, 2,
                         scout);
#endif
  if (scout) *scout += sc2;
  ETB_DIAG_END(64 + (dnext & 63));
}

// Request run r0 (kU visited words and their first neighbours) into pipe
// stage sg (lane 0; nothing past the sweep's end). The visited span is widened
// to 16-byte boundaries (the bitmap allocation covers the overhang); cfirst is
// padded to whole words at layout time.
template <int kU>
__device__ __forceinline__ void bu_issue(const BfsParams& p, BuPipe<kU>* pipe, int sg, uint64_t r0) {
  if (r0 >= p.nwords) return;
  const uint32_t nwd = static_cast<uint32_t>(min(static_cast<uint64_t>(kU), p.nwords - r0));
  const uint32_t cf_bytes = nwd * 128u;
  const uint64_t vlo = (r0 * 4) & ~uint64_t{15}, vhi = ((r0 + nwd) * 4 + 15) & ~uint64_t{15};
  const uint32_t vw_bytes = static_cast<uint32_t>(vhi - vlo);
  mbar_expect_tx(&pipe->bar[sg], cf_bytes + vw_bytes);
  bulk_g2s(pipe->st[sg].cf, p.cfirst + r0 * 32, cf_bytes, &pipe->bar[sg]);
  bulk_g2s(pipe->st[sg].vw, reinterpret_cast<const unsigned char*>(p.visited) + vlo, vw_bytes,
           &pipe->bar[sg]);
}
template <int kU, bool kBound = false, class P>
__device__ void bu_step(const P& p, uint32_t* mbuf, const uint32_t* fcur,
                        uint32_t* fnext, int32_t dnext, unsigned long long& claims_acc,
                        uint32_t* qv_out, uint64_t* qp_out, unsigned long long* lslot,
                        unsigned long long* scout = nullptr) {
  static_assert(32 * kU <= kMissCap, "one iteration's misses must fit the miss buffer");
  const unsigned lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const uint64_t gw = (uint64_t)cta_of(p) * (blockDim.x >> 5) + wib;
  const uint64_t nw = (uint64_t)(ncta_of(p) * blockDim.x) >> 5;
  const unsigned lt = (1u << lane) - 1;
  uint32_t nmiss = 0;
  unsigned long long scm = 0;  // main-pass claims' full degrees (scout wanted)
  ETB_DIAG_BEGIN();
  constexpr bool kTma = ETB_BU_TMA && !IsPart<P>::value;
  [[maybe_unused]] BuPipe<kU>* pipe = nullptr;
  [[maybe_unused]] const uint64_t rstep = nw * kU;
  if constexpr (kTma) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    pipe = reinterpret_cast<BuPipe<kU>*>(smem_raw + sizeof(Smem)) + wib;
    if (lane == 0) {
      mbar_init(&pipe->bar[0], 1);
      mbar_init(&pipe->bar[1], 1);
      fence_mbar_init();
      fence_proxy_async_global();
      bu_issue<kU>(p, pipe, 0, gw * kU);
      bu_issue<kU>(p, pipe, 1, gw * kU + rstep);
    }
    __syncwarp();
  }
  // (large-core kernel only, kU == kBuU: s26 +2.4%, s28 +1.6%; the small-core
  // kernel's short levels lose more to the counter than they gain: s22 -1.1%)
  // (partitioned kernel: p.dyn, set on the large-core instantiation only)
  bool kDyn = ETB_BU_DYN && !kTma && kU == kBuU;
  if constexpr (IsPart<P>::value) kDyn = kDyn && p.dyn;
  [[maybe_unused]] const uint64_t wpc = blockDim.x >> 5;
  auto grab = [&]() -> uint64_t {  // the CTA's next run: cta*wpc + (k / wpc)*nw + k % wpc
    unsigned k = 0;
    if (lane == 0) k = atomicAdd(&smem_view().bu_next, 1u);
    k = __shfl_sync(0xffffffffu, k, 0);
    return ((uint64_t)cta_of(p) * wpc + (uint64_t)(k / wpc) * nw + k % wpc) * kU;
  };
  int it = 0;
  for (uint64_t w0 = kDyn ? grab() : wlo_of(p) + gw * kU; w0 < whi_of(p);
       w0 = kDyn ? grab() : w0 + nw * kU, ++it) {
    // the run's words: w0 + k (one partition), or one owned-word mapping per
    // run (partitioned: aligned runs of 8 are 8 hub words G apart or one block)
    uint64_t wb = 0, ws = 0;
    if constexpr (IsPart<P>::value) {
      static_assert(kU == 8, "partition runs are aligned 8-word runs");
      wb = word_at(p, w0);
      ws = run_stride(p, w0);
    }
    auto wrd = [&](int k) -> uint64_t {
      if constexpr (IsPart<P>::value) return wb + k * ws;
      else return w0 + k;
    };
    uint32_t vis[kU];
    bool any = false;
    uint32_t f[kU];
    if constexpr (kTma) {
      const int sg = it & 1;
      mbar_wait(&pipe->bar[sg], (it >> 1) & 1);
      const BuStage<kU>& st = pipe->st[sg];
      const uint32_t off = static_cast<uint32_t>(w0 & 3);  // words before w0 in the aligned span
#pragma unroll
      for (int k = 0; k < kU; ++k) {
        vis[k] = w0 + k < whi_of(p) ? st.vw[off + k] : ~0u;
        any |= vis[k] != ~0u;
      }
#pragma unroll
      for (int k = 0; k < kU; ++k) f[k] = ((vis[k] >> lane) & 1u) ? kNone32 : st.cf[k * 32 + lane];
#ifdef ETB_DEBUG_CHECKS
#pragma unroll
      for (int k = 0; k < kU; ++k) {
        ETB_DCHECK(w0 + k >= whi_of(p) || vis[k] == __ldcg(&p.visited[w0 + k]));
        ETB_DCHECK(w0 + k >= whi_of(p) || st.cf[k * 32 + lane] == p.cfirst[(w0 + k) * 32 + lane]);
      }
#endif
      {  // every lane's stage reads have returned (their values are consumed by
         // the warp-wide reduction) before the async proxy may overwrite the stage
        uint32_t x = 0;
#pragma unroll
        for (int k = 0; k < kU; ++k) x |= f[k] ^ vis[k];
        x = __reduce_or_sync(0xffffffffu, x);
        if (x == 0x5a5a5a5au && lane == 33) f[0] = 0;  // (never true: keeps x live)
      }
      if (lane == 0) {  // refill the stage with the run two iterations ahead
        fence_proxy_async_shared();
        bu_issue<kU>(p, pipe, sg, w0 + 2 * rstep);
      }
      if (!any) continue;
    } else {
#if ETB_BU_EAGER
    // first neighbours loaded with the visited words, not after them (one
    // round trip less per iteration; bu_step runs on levels where most of the
    // core is unvisited, so few of these loads are wasted)
    uint32_t cf[kU];
#pragma unroll
    for (int k = 0; k < kU; ++k) {
      const uint64_t x = wrd(k) * 32 + lane;
      vis[k] = w0 + k < whi_of(p) ? p.visited[wrd(k)] : ~0u;
      cf[k] = w0 + k < whi_of(p) && x < p.nc ? p.cfirst[x] : kNone32;
      any |= vis[k] != ~0u;
    }
    if (!any) continue;
#pragma unroll
    for (int k = 0; k < kU; ++k) f[k] = ((vis[k] >> lane) & 1u) ? kNone32 : cf[k];
#else
#pragma unroll
    for (int k = 0; k < kU; ++k) {
      vis[k] = w0 + k < whi_of(p) ? p.visited[wrd(k)] : ~0u;
      any |= vis[k] != ~0u;
    }
    if (!any) continue;
#pragma unroll
    for (int k = 0; k < kU; ++k)
      f[k] = ((vis[k] >> lane) & 1u) ? kNone32 : p.cfirst[wrd(k) * 32 + lane];
#endif
    }
    if (kBound) {  // no neighbour under the bound: nothing to probe, not a miss
      const uint32_t bound = smem_view().bu_bound;
#pragma unroll
      for (int k = 0; k < kU; ++k)
        if (f[k] >= bound) f[k] = kNone32;
    }
    bool hit[kU];
#pragma unroll
    for (int k = 0; k < kU; ++k) hit[k] = f[k] != kNone32 && test_bit(fcur, f[k]);
#pragma unroll
    for (int k = 0; k < kU; ++k) {
      const uint64_t wk = wrd(k);
      const uint32_t v = static_cast<uint32_t>(wk * 32 + lane);
      const unsigned m = __ballot_sync(0xffffffffu, hit[k]);
      if (hit[k]) {
        p.dp[v] = make_uint2(static_cast<uint32_t>(dnext), f[k]);
        if (scout) scm += p.degn[v];
      }
      if (lane == 0 && m) {
        if (kBound) {  // the split level's top-down half may be claiming in this word
          atomicOr(&p.visited[wk], m);
          atomicOr(&fnext[wk], m);
        } else {
          p.visited[wk] = vis[k] | m;
          fnext[wk] = m;
        }
        claims_acc += __popc(m);
      }
      const bool miss = f[k] != kNone32 && !hit[k];
      const unsigned mm = __ballot_sync(0xffffffffu, miss);
      ETB_DCHECK(nmiss + 32 <= kMissCap && (!miss || v < p.nc));
      if (miss) mbuf[nmiss + __popc(mm & lt)] = v;
      nmiss += __popc(mm);
    }
    if (lslot) {
      uint32_t av[kU], ad[kU];
#pragma unroll
      for (int k = 0; k < kU; ++k) {
        av[k] = static_cast<uint32_t>(wrd(k) * 32 + lane);
        ad[k] = hit[k] ? p.cmeta[av[k]].x : 0u;
      }
      bu_append<kU>(av, ad, qv_out, qp_out, lslot);
    }
    if (nmiss > min(kMissCap - 32 * kU, kMissFlush)) {
      resolve_misses<kBound>(p, fcur, fnext, mbuf, nmiss, dnext, claims_acc, qv_out, qp_out, lslot, scout);
      nmiss = 0;
    }
  }
  if constexpr (kTma) {  // every requested run was consumed: retire the barriers
    __syncwarp();
    if (lane == 0) {
      mbar_inval(&pipe->bar[0]);
      mbar_inval(&pipe->bar[1]);
    }
  }
  if (nmiss) resolve_misses<kBound>(p, fcur, fnext, mbuf, nmiss, dnext, claims_acc, qv_out, qp_out, lslot, scout);
  if (scout) *scout += scm;
  ETB_DIAG_END(dnext & 63);
}

template <int kSweep, class P>
__device__ __forceinline__ void bu_sweep(const P& p, uint32_t* mbuf, const uint32_t* fcur,
                        uint32_t* fnext, int32_t dnext, unsigned long long& claims_acc,
                        uint32_t* qv_out, uint64_t* qp_out, unsigned long long* lslot,
                        unsigned long long* scout = nullptr) {
  const unsigned lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const uint64_t gw = (uint64_t)cta_of(p) * (blockDim.x >> 5) + wib;
  const uint64_t nw = (uint64_t)(ncta_of(p) * blockDim.x) >> 5;
  const unsigned lt = (1u << lane) - 1;
  uint32_t nmiss = 0;
  unsigned long long scm = 0;  // main-pass claims' full degrees (scout wanted)
  ETB_DIAG_BEGIN();
  // A warp sweeps kSweep visited words with one coalesced load (lane = word)
  // and works through the words with unvisited vertices kBuU at a time, so
  // late levels (few unvisited left) skip full words without a round trip each.
  bool kDyn = ETB_BU_DYN;
  if constexpr (IsPart<P>::value) kDyn = kDyn && p.dyn;
  [[maybe_unused]] const uint64_t wpc = blockDim.x >> 5;
  auto grab = [&]() -> uint64_t {  // as bu_step's: the CTA's next run of kSweep words
    unsigned k = 0;
    if (lane == 0) k = atomicAdd(&smem_view().bu_next, 1u);
    k = __shfl_sync(0xffffffffu, k, 0);
    return ((uint64_t)cta_of(p) * wpc + (uint64_t)(k / wpc) * nw + k % wpc) * kSweep;
  };
  for (uint64_t b0 = kDyn ? grab() : wlo_of(p) + gw * kSweep; b0 < whi_of(p);
       b0 = kDyn ? grab() : b0 + nw * kSweep) {
    uint32_t myw = 0, mine;
    if constexpr (IsPart<P>::value) {
      myw = static_cast<uint32_t>(word_at(p, b0 + lane));
      mine = lane < kSweep && b0 + lane < whi_of(p) ? p.visited[myw] : ~0u;
    } else {
      mine = lane < kSweep && b0 + lane < whi_of(p) ? p.visited[b0 + lane] : ~0u;
    }
    unsigned todo = __ballot_sync(0xffffffffu, mine != ~0u);
    while (todo) {
      uint32_t vis[kBuU], wi[kBuU];
#pragma unroll
      for (int k = 0; k < kBuU; ++k) {
        const int j = todo ? __ffs(todo) - 1 : 0;
        vis[k] = todo ? __shfl_sync(0xffffffffu, mine, j) : ~0u;
        if constexpr (IsPart<P>::value)
          wi[k] = __shfl_sync(0xffffffffu, myw, j);
        else
          wi[k] = static_cast<uint32_t>(b0) + j;
        todo &= todo - 1;
      }
      uint32_t f[kBuU];
#pragma unroll
      for (int k = 0; k < kBuU; ++k)
        f[k] = ((vis[k] >> lane) & 1u) ? kNone32 : p.cfirst[(uint64_t)wi[k] * 32 + lane];
      bool hit[kBuU];
#pragma unroll
      for (int k = 0; k < kBuU; ++k) hit[k] = f[k] != kNone32 && test_bit(fcur, f[k]);
#pragma unroll
      for (int k = 0; k < kBuU; ++k) {
        const uint32_t v = wi[k] * 32 + lane;
        const unsigned m = __ballot_sync(0xffffffffu, hit[k]);
        if (hit[k]) {
          p.dp[v] = make_uint2(static_cast<uint32_t>(dnext), f[k]);
          if (scout) scm += p.degn[v];
        }
        if (lane == 0 && m) {
          p.visited[wi[k]] = vis[k] | m;
          fnext[wi[k]] = m;
          claims_acc += __popc(m);
        }
        const bool miss = f[k] != kNone32 && !hit[k];
        const unsigned mm = __ballot_sync(0xffffffffu, miss);
        ETB_DCHECK(nmiss + 32 <= kMissCap && (!miss || v < p.nc));
      if (miss) mbuf[nmiss + __popc(mm & lt)] = v;
        nmiss += __popc(mm);
      }
      if (lslot) {
        uint32_t av[kBuU], ad[kBuU];
#pragma unroll
        for (int k = 0; k < kBuU; ++k) {
          av[k] = wi[k] * 32 + lane;
          ad[k] = hit[k] ? p.cmeta[av[k]].x : 0u;
        }
        bu_append<kBuU>(av, ad, qv_out, qp_out, lslot);
      }
      if (nmiss > min(kMissCap - 32 * kBuU, kMissFlush)) {
        resolve_misses(p, fcur, fnext, mbuf, nmiss, dnext, claims_acc, qv_out, qp_out, lslot, scout);
        nmiss = 0;
      }
    }
  }
  if (nmiss) resolve_misses(p, fcur, fnext, mbuf, nmiss, dnext, claims_acc, qv_out, qp_out, lslot, scout);
  if (scout) *scout += scm;
  ETB_DIAG_END(dnext & 63);
}

// Frontier bitmap -> frontier list (when a top-down level follows one that did
// not emit a list). Lane = one bitmap word; one packed atomic per 32 words.
__device__ void convert_step(const BfsParams& p, const uint32_t* fcur, uint32_t* qv_out,
                             uint64_t* qp_out, unsigned long long* cslot) {
  const unsigned lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const uint64_t gw = (uint64_t)wib * gridDim.x + blockIdx.x;  // CTA-minor: spread over SMs
  const uint64_t nw = (uint64_t)(gridDim.x * blockDim.x) >> 5;
  for (uint64_t w0 = gw * 32; w0 < p.nwords; w0 += nw * 32) {
    const uint64_t wi = w0 + lane;
    const uint32_t bits = wi < p.nwords ? fcur[wi] : 0u;
    uint32_t cnt = 0, edges = 0;
    for (uint32_t b = bits; b; b &= b - 1) {
      const uint32_t d = p.cmeta[static_cast<uint32_t>(wi * 32 + __ffs(b) - 1)].x;
      cnt += d != 0;
      edges += d;
    }
    const uint32_t vin = warp_incl_scan(cnt);
    const uint32_t vtot = __shfl_sync(0xffffffffu, vin, 31);
    if (vtot == 0) continue;
    // edge prefix in 64 bits (a word of hubs can exceed 2^32 edges only in theory)
    unsigned long long ein = edges;
    for (int o = 1; o < 32; o <<= 1) {
      const unsigned long long y = __shfl_up_sync(0xffffffffu, ein, o);
      if (lane >= o) ein += y;
    }
    const unsigned long long etot = __shfl_sync(0xffffffffu, ein, 31);
    unsigned long long old = 0;
    if (lane == 31) old = atomicAdd(cslot, ((unsigned long long)vtot << kItemShift) | etot);
    old = __shfl_sync(0xffffffffu, old, 31);
    uint64_t vpos = (old >> kItemShift) + vin - cnt, epos = (old & kItemMask) + ein - edges;
    for (uint32_t b = bits; b; b &= b - 1) {
      const uint32_t v = static_cast<uint32_t>(wi * 32 + __ffs(b) - 1);
      const uint32_t d = p.cmeta[v].x;
      if (!d) continue;
      qv_out[vpos] = v;
      qp_out[vpos] = epos;
      ++vpos;
      epos += d;
    }
  }
}

// The claims (popcount) and scout (Σ full degree) of a top-down level from its
// new frontier bitmap f: a warp takes 4 words per iteration, lane = vertex,
// coalesced degree loads — a streaming pass instead of one random 32-byte
// sector per claim, and the level's claims need no atomic return (td_step<3>).
#ifndef ETB_SCOUT_W
#define ETB_SCOUT_W 16  // (s26: 16 +0.5% against 4, 8 equal)
#endif
__device__ unsigned long long scout_pass(const BfsParams& p, const uint32_t* f,
                                         unsigned long long& claims) {
  const unsigned lane = threadIdx.x & 31;
  const uint64_t gw = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const uint64_t nw = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  unsigned long long s = 0, c = 0;
  constexpr int W = ETB_SCOUT_W;  // words per warp iteration: W bitmap loads, then W degree loads
  for (uint64_t w0 = gw * W; w0 < p.nwords; w0 += nw * W) {
    uint32_t bits[W], d[W];
#pragma unroll
    for (int k = 0; k < W; ++k) bits[k] = w0 + k < p.nwords ? __ldcg(&f[w0 + k]) : 0u;
#pragma unroll
    for (int k = 0; k < W; ++k) {
      c += (bits[k] >> lane) & 1u;
      d[k] = ((bits[k] >> lane) & 1u) ? p.degn[(w0 + k) * 32 + lane] : 0u;
    }
#pragma unroll
    for (int k = 0; k < W; ++k) s += d[k];
  }
  claims += c;
  return s;
}

// Tree entries in flight per thread in the replay (two dependent round trips
// each: the tree arrays, then the anchor's visited bit and depth).
#ifndef ETB_REPLAY
#define ETB_REPLAY 4
#endif

constexpr int kReplay = ETB_REPLAY;

// kLarge: the 1024-thread instantiation (cores of >= 2^23 vertices), the only
// one whose top-down levels can claim a large share of the core at once.
template <bool kLarge>
__device__ __forceinline__ void et_bfs_body(const BfsParams& p) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  Smem& sm = *reinterpret_cast<Smem*>(smem_raw);
  const uint64_t tid = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const uint64_t nthreads = (uint64_t)gridDim.x * blockDim.x;
  const uint32_t start = p.start;
  const bool run_core = start != kNone32;
  stamp(p, 256);
  if (threadIdx.x == 0) sm.bu_next = 0;  // (a barrier precedes every bottom-up step)
  // diagnostics: per-CTA entry (slot 62) and exit (slot 63) times
  if (p.bstamp && threadIdx.x == 0) p.bstamp[62 * gridDim.x + blockIdx.x] = gtimer();

  // ---- start: the state halves were cleaned by the previous traversal (or at
  // layout setup); only the start's bits are set. Core-sized state only (the
  // reference allocates n-sized state, et_bfs.cpp:82,96) --------------------------
  uint64_t nq = 0, ne = 0;  // frontier list length and its edge count
  if (run_core) {
    ne = p.cmeta[start].x;
    nq = ne != 0;
    if (tid == 0) {
      atomicOr(&p.visited[start >> 5], 1u << (start & 31));
      p.fb0[start >> 5] = 1u << (start & 31);
      p.dp[start] = make_uint2(static_cast<uint32_t>(p.base_depth), p.start_parent);
    }
  }
  const bool bu0 = run_core && (p.bottom_up_only ||
                                (!p.top_down_only &&
                                 (double)p.degn[start] > p.edges_to_check / p.alpha));
  // A top-down first level reads only the start's row (no list, no start bit);
  // a bottom-up one probes fb0, so it waits for the start bit.
  if (bu0) grid_sync(p.bar);
  stamp(p, 257);

  // ---- level loop: run_hybrid (bfs.cpp:232-293) ---------------------------------
  uint32_t L = 0;
  if (run_core) {
    uint32_t* F[3] = {p.fb0, p.fb1, p.fb2};
    uint32_t* qv_in = p.qv0;
    uint32_t* qv_out = p.qv1;
    uint64_t* qp_in = p.qp0;
    uint64_t* qp_out = p.qp1;
    unsigned long long frontier = 1, scout = p.degn[start], awake = 0, prev = 0, reached = 1;
    // The traversal can reach the start's core component only (p.reachable, a
    // per-root launch parameter): once all of it is visited, the next level
    // would claim nothing (checked at the level ends).
    double etc = p.edges_to_check;
    bool bu = bu0, saw_bu = bu0;
    if (bu) awake = frontier;
    bool list_from_prologue = false;
    // ---- fused first level: when the start's core row fits one CTA, every CTA
    // claims it redundantly (the claims are the whole row: nothing else is
    // visited yet), sets the bits itself and builds the same level-1 list in
    // place, so level 1 starts without level 0's chain and grid barrier. Only
    // CTA 0 writes the results and stats.
    const uint32_t d0 = static_cast<uint32_t>(ne);
    // (Small-core kernel only: in the large-core instantiation the extra code
    // costs more in register allocation elsewhere than the 3 us it saves.)
// (the fused first level on the large-core kernel: s26 -2.3%, s28 -1.3% — its
// code makes the large-core kernel spill)
#ifndef ETB_LARGE_PROLOGUE
#define ETB_LARGE_PROLOGUE 0
#endif
    if ((!kLarge || ETB_LARGE_PROLOGUE) && !bu && !p.bottom_up_only && d0 > 0 &&
        d0 <= blockDim.x && d0 + 1 < p.nc) {
      const unsigned lane = threadIdx.x & 31, wib = threadIdx.x >> 5, nwb = blockDim.x >> 5;
      const uint64_t rs = p.crow[start];
      uint32_t w = kNone32;
      uint2 mt = make_uint2(0u, 0u);
      // the start's bit too: CTA 0's thread 0 sets it without a barrier here
      if (threadIdx.x == 0) atomicOr(&p.visited[start >> 5], 1u << (start & 31));
      if (threadIdx.x < d0) {
        w = p.ccol[rs + threadIdx.x];
        mt = p.cmeta[w];
        atomicOr(&p.visited[w >> 5], 1u << (w & 31));
        if (blockIdx.x == 0)
          p.dp[w] = make_uint2(static_cast<uint32_t>(p.base_depth + 1), start);
      }
      // block scans: list position and edge prefix of the neighbours with core edges
      const uint32_t take = mt.x != 0;
      const uint32_t cin = warp_incl_scan(take);
      const unsigned long long ein = warp_incl_scan64(mt.x);
      const unsigned long long sc = warp_sum(static_cast<unsigned long long>(mt.y));
      if (lane == 31) {
        sm.red[0][wib] = (static_cast<unsigned long long>(cin) << 40) | ein;
        sm.red[1][wib] = sc;
      }
      __syncthreads();
      unsigned long long cbase = 0, ebase = 0, ctot = 0, etot = 0, stot = 0;
      for (unsigned k = 0; k < nwb; ++k) {
        const unsigned long long r = sm.red[0][k];
        if (k < wib) {
          cbase += r >> 40;
          ebase += r & ((1ull << 40) - 1);
        }
        ctot += r >> 40;
        etot += r & ((1ull << 40) - 1);
        stot += sm.red[1][k];
      }
      if (take) {
        const uint64_t pos = cbase + cin - 1;
        p.qv1[pos] = w;
        p.qp1[pos] = ebase + ein - mt.x;
      }
      // the state after level 0
      etc -= (double)scout;
      frontier = d0;
      scout = stot;
      reached = 1 + d0;
      nq = ctot;
      ne = etot;
      if (tid == 0) {
        if (p.trace) p.trace[0] = 't';
        if (p.level_claims) p.level_claims[0] = d0;
      }
      L = 1;
      stamp(p, 258);
      if (!p.top_down_only && (double)scout > etc / p.alpha) {
        // a bottom-up level 1 probes the frontier bitmap: this CTA's own copy of it
        bu = true;
        saw_bu = true;
        awake = frontier;
        if (w != kNone32) atomicOr(&p.fb1[w >> 5], 1u << (w & 31));
      }
      list_from_prologue = true;
      __syncthreads();  // this CTA's visited / frontier bits and list before level 1
    }
    if (list_from_prologue) {  // level 1 reads qv1 / qp1
      uint32_t* tv = qv_in;
      qv_in = qv_out;
      qv_out = tv;
      uint64_t* tp = qp_in;
      qp_in = qp_out;
      qp_out = tp;
    }
    for (;;) {
      uint32_t* fcur = F[L % 3];
      uint32_t* fnext = F[(L + 1) % 3];
      uint32_t* fzero = F[(L + 2) % 3];
      unsigned long long* slot = p.ctr + (L & 3) * 4;
      for (uint64_t i = tid; i < p.nwords; i += nthreads) fzero[i] = 0;
      if (tid == 0) {
        p.ctr[((L + 2) & 3) * 4 + 0] = 0;
        p.ctr[((L + 2) & 3) * 4 + 1] = 0;
        p.ctr[((L + 2) & 3) * 4 + 2] = 0;
        p.ctr[((L + 2) & 3) * 4 + 3] = 0;
        p.ctr[16 + ((L + 1) & 1)] = 0;
        if (p.trace && L < 255) p.trace[L] = bu ? 'b' : 't';
      }
      const int32_t dnext = p.base_depth + static_cast<int32_t>(L) + 1;
      unsigned long long claims_acc = 0, scout_acc = 0;
      bool list_valid = true, defer_scout = false;
      // (A smem copy of the probed bitmap's hot prefix was tried and measured
      // slower: the 64 KB it takes comes out of L1, which caches those lines.)
      bool bu_list = false;
      if (bu) {
        prev = awake;
        // Emit the next list when this level is all but certain to be the last
        // bottom-up one: the vertices it can still claim (core minus reached)
        // already fit under the beta bound, so only awake >= prev keeps it.
        // (Measured: limiting it to levels with few claims left, to spare the
        // list-counter atomics, was slower overall at scales 22 and 26.)
        bu_list = !p.bottom_up_only && !p.top_down_only &&
                  (double)(p.nc - reached) <= (double)p.nc / p.beta;
        // Large-core kernel, levels with few unvisited vertices left: the
        // coalesced sweep that skips fully visited words (bu_sweep; on the
        // small-core kernel it measured slower at every level kind)
        if (kLarge && (double)(p.nc - reached) * kSweepT < (double)p.nc)
          bu_sweep<32>(p, sm.w[threadIdx.x >> 5].cbuf, fcur, fnext, dnext, claims_acc, qv_in,
                       qp_in, bu_list ? &slot[0] : nullptr);
        else
          bu_step<kLarge ? kBuU : kBuUSmall>(p, sm.w[threadIdx.x >> 5].cbuf, fcur, fnext, dnext,
                                             claims_acc, qv_in, qp_in,
                                             bu_list ? &slot[0] : nullptr);
      } else if (kLarge && p.split_ratio > 0.0 && !p.top_down_only && L > 0 &&
                 !((double)scout < p.emit_limit) &&
                 (double)ne >= p.split_ratio * (double)(p.nc - reached)) {
        // A big list-less top-down level executed split: the frontier's hubs
        // (ids < split_bound, most of its edges) bottom-up over the unvisited
        // core with every row scan ended at the bound — the rows of the
        // vertices with no hub neighbour in the frontier end within their
        // first few entries instead of being scanned whole — and the other
        // frontier vertices top-down from a filtered list. A vertex is claimed
        // iff it has a frontier neighbour on either side: the reference's
        // claims; claims and scout are counted from the new frontier bitmap.
        etc -= (double)scout;
        list_valid = false;
        defer_scout = true;
        if (threadIdx.x == 0) sm.bu_bound = p.split_bound;
        {  // the frontier vertices past the bound, appended to the free list
          const unsigned lane = threadIdx.x & 31, lt = (1u << lane) - 1;
          const uint64_t gwp = tid >> 5, nwp = nthreads >> 5;
          for (uint64_t i0 = gwp * 32; i0 < nq; i0 += nwp * 32) {
            const uint64_t i = i0 + lane;
            uint32_t v = 0, d = 0;
            if (i < nq) {
              v = qv_in[i];
              if (v >= p.split_bound)
                d = static_cast<uint32_t>((i + 1 < nq ? qp_in[i + 1] : ne) - qp_in[i]);
            }
            const unsigned m = __ballot_sync(0xffffffffu, d != 0);
            if (!m) continue;
            const uint32_t din = warp_incl_scan(d);
            const uint32_t dtot = __shfl_sync(0xffffffffu, din, 31);
            unsigned long long old = 0;
            if (lane == 0)
              old = atomicAdd(&slot[0],
                              (static_cast<unsigned long long>(__popc(m)) << kItemShift) | dtot);
            old = __shfl_sync(0xffffffffu, old, 0);
            if (d != 0) {
              const uint64_t pos = (old >> kItemShift) + __popc(m & lt);
              qv_out[pos] = v;
              qp_out[pos] = (old & kItemMask) + din - d;
            }
          }
        }
        if (p.split_tdw) {
          // Both halves at once: after the (short) filter pass and its barrier the
          // CTA's first split_tdw warps run the top-down half, a latency-bound
          // few chunks per warp, then join the others in the bottom-up half
          // (its runs are handed out dynamically; its word updates are atomic
          // in the bounded form, the other half may be claiming in the same word).
          grid_sync_add(p.bar, sm, 0, nullptr, 0, nullptr, slot, 1);
          stamp(p, 320 + L);  // diagnostics: a split level (here: its filter pass's end)
          const unsigned long long tail = sm.tot[0];
          if (p.level_claims && tid == 0 && L < 64) p.level_claims[448 + L] = tail & kItemMask;
          // kSplitAuto: a short top-down half (a few latency-bound chunks per
          // warp) runs beside the bottom-up half on half the warps; a long one
          // follows it, so that its probes find the hubs' claims already made
          // (s26, tails of 6-22M edges: 16 warps +1.8%, after +0.6%; s28, 4x
          // the tails: 16 warps -1.3%, after +0.5%)
          const uint32_t tdw = p.split_tdw != kSplitAuto ? p.split_tdw
                               : (tail & kItemMask) < kSplitShortTail ? 16u : 64u;
          if (tdw <= 32)
            td_step<3, kLarge>(p, sm.w[threadIdx.x >> 5].cbuf, sm.w[threadIdx.x >> 5].win, qv_out,
                               qp_out, tail >> kItemShift, tail & kItemMask, qv_in, qp_in, fnext,
                               slot, dnext, scout_acc, claims_acc, kNone32, tdw);
          bu_step<kBuU, true>(p, sm.w[threadIdx.x >> 5].cbuf, fcur, fnext, dnext, claims_acc,
                              qv_in, qp_in, nullptr);
          // split_tdw > 32: every warp goes from the CTA's last bottom-up run
          // straight to the top-down chunks (no barrier between the halves; the
          // top-down probes then find most targets already claimed)
          if (tdw > 32)
            td_step<3, kLarge>(p, sm.w[threadIdx.x >> 5].cbuf, sm.w[threadIdx.x >> 5].win, qv_out,
                               qp_out, tail >> kItemShift, tail & kItemMask, qv_in, qp_in, fnext,
                               slot, dnext, scout_acc, claims_acc, kNone32);
        } else {
          __syncthreads();  // bu_bound
          bu_step<kBuU, true>(p, sm.w[threadIdx.x >> 5].cbuf, fcur, fnext, dnext, claims_acc,
                              qv_in, qp_in, nullptr);
          grid_sync_add(p.bar, sm, 0, nullptr, 0, nullptr, slot, 1);
          stamp(p, 320 + L);  // diagnostics: end of the split level's bottom-up half
          const unsigned long long tail = sm.tot[0];
          if (p.level_claims && tid == 0 && L < 64) p.level_claims[448 + L] = tail & kItemMask;
          td_step<3, kLarge>(p, sm.w[threadIdx.x >> 5].cbuf, sm.w[threadIdx.x >> 5].win, qv_out,
                             qp_out, tail >> kItemShift, tail & kItemMask, qv_in, qp_in, fnext,
                             slot, dnext, scout_acc, claims_acc, kNone32);
        }
        claims_acc = 0;
        scout_acc = 0;
      } else if (p.td_as_bu > 0.0 && !p.top_down_only && !(L == 1 && list_from_prologue) && L > 0 &&
                 (double)ne > p.td_as_bu * (double)(p.nc - reached)) {
        // a top-down level (α/β state advanced as the reference's) executed as
        // a bottom-up sweep over the unvisited core against this frontier's
        // bitmap: the same claims, coalesced instead of scattered; claims and
        // scout are counted from the new frontier bitmap (scout_pass)
        etc -= (double)scout;
        list_valid = false;
        // Small-core kernel: the level's scout is summed by the step itself,
        // one degree load per claim (s22 +1.2%); large-core kernel: claims and
        // scout counted afterwards by scout_pass (the in-step sums cost its
        // register-bound bottom-up code spills: s26 -1.2%).
        defer_scout = kLarge;
        if (kLarge && (double)(p.nc - reached) * kSweepT < (double)p.nc)
          bu_sweep<32>(p, sm.w[threadIdx.x >> 5].cbuf, fcur, fnext, dnext, claims_acc, qv_in,
                       qp_in, nullptr);
        else
          bu_step<kLarge ? kBuU : kBuUSmall>(p, sm.w[threadIdx.x >> 5].cbuf, fcur, fnext, dnext,
                                             claims_acc, qv_in, qp_in, nullptr,
                                             kLarge ? nullptr : &scout_acc);
        if (kLarge) claims_acc = 0;
      } else {
        etc -= (double)scout;
        // The next frontier list is emitted only when this frontier's edge count
        // is small; a large one is all but certain to hand over to bottom-up
        // (which needs only the bitmap), else the bitmap is converted.
        const bool emit = (double)scout < p.emit_limit;
        // diagnostics: this top-down level's frontier edges (phase stamp 192 + L)
        if (p.level_claims && tid == 0 && L < 64) p.level_claims[448 + L] = ne;
        list_valid = emit;
        uint32_t* cb = sm.w[threadIdx.x >> 5].cbuf;
        int32_t* wn = sm.w[threadIdx.x >> 5].win;
        const uint32_t root = L == 0 ? start : kNone32;
        // Large-core kernel: a list-less level claims without atomic returns; its
        // claims and scout are counted afterwards by a streaming pass over the
        // new frontier (mode 3). (Measured: s26 -5 us per root; on the
        // small-core kernel the extra pass and barrier cost more than they save.)
        defer_scout = !emit && (kLarge || (double)ne >= p.small_mode3_edges);
        if (defer_scout)
          td_step<3, kLarge>(p, cb, wn, qv_in, qp_in, nq, ne, qv_out, qp_out, fnext, slot, dnext,
                     scout_acc, claims_acc, root);
        else if (!emit)
          td_step<0, kLarge>(p, cb, wn, qv_in, qp_in, nq, ne, qv_out, qp_out, fnext, slot, dnext,
                     scout_acc, claims_acc, root);
        else if (saw_bu)
          td_step<1, kLarge>(p, cb, wn, qv_in, qp_in, nq, ne, qv_out, qp_out, fnext, slot, dnext,
                     scout_acc, claims_acc, root);
        else
          td_step<2, kLarge>(p, cb, wn, qv_in, qp_in, nq, ne, qv_out, qp_out, fnext, slot, dnext,
                     scout_acc, claims_acc, root);
      }
      if (p.bstamp && threadIdx.x == 0 && L < 62) p.bstamp[L * gridDim.x + blockIdx.x] = gtimer();
      grid_sync_add(p.bar, sm, claims_acc, &slot[3], scout_acc, bu ? nullptr : &slot[1], slot, 4);
      const unsigned long long packed = sm.tot[0];
      unsigned long long scout_tot = sm.tot[1];
      unsigned long long claims = sm.tot[3];
      if (defer_scout) {  // td_step<3>: claims and scout from the new frontier bitmap
        unsigned long long pc = 0;
        const unsigned long long ds = scout_pass(p, fnext, pc);
        grid_sync_add(p.bar, sm, pc, &slot[3], ds, &slot[1], slot, 4);
        scout_tot = sm.tot[1];
        claims = sm.tot[3];
      }
      reached += claims;
      if (p.level_claims && tid == 0 && L < 256) p.level_claims[L] = claims;
      ++L;
      stamp(p, 257 + L);
      if (bu && p.bottom_up_only) {
        // standalone block sweeps to fixpoint (run_block_search, bfs.cpp:295-305)
        if (claims == 0) break;
      } else if (bu) {
        awake = claims;
        if (!(awake > 0 && (awake >= prev || (double)awake > (double)p.nc / p.beta))) {
          bu = false;
          frontier = awake;
          scout = 1;
          list_valid = bu_list;
          if (bu_list) {
            nq = packed >> kItemShift;
            ne = packed & kItemMask;
          }
        }
      } else {
        frontier = claims;
        scout = scout_tot;
        nq = packed >> kItemShift;
        ne = packed & kItemMask;
        uint32_t* tv = qv_in;
        qv_in = qv_out;
        qv_out = tv;
        uint64_t* tp = qp_in;
        qp_in = qp_out;
        qp_out = tp;
      }
      if (!bu) {
        if (frontier == 0) break;
        if (!p.top_down_only && (double)scout > etc / p.alpha) {
          bu = true;
          saw_bu = true;
          awake = frontier;
        } else if (!list_valid && reached < p.reachable) {
          unsigned long long* cslot = p.ctr + 16 + (L & 1);
          convert_step(p, F[L % 3], qv_in, qp_in, cslot);
          grid_sync_add(p.bar, sm, 0, nullptr, 0, nullptr, cslot, 1);
          stamp(p, 384 + L);  // diagnostics: end of the bitmap -> list conversion
          const unsigned long long cp = sm.tot[0];
          nq = cp >> kItemShift;
          ne = cp & kItemMask;
        }
      }
      // Every core vertex of the start's component is visited: the level the
      // reference would run next (bfs.cpp:240-292; either direction) claims
      // nothing and ends the loop. Record it with its direction and no claims,
      // without running it.
      if (reached == p.reachable) {
        if (tid == 0 && p.trace && L < 255) p.trace[L] = bu ? 'b' : 't';
        if (p.level_claims && tid == 0 && L < 256) p.level_claims[L] = 0;
        ++L;
        stamp(p, 257 + L);
        break;
      }
    }
  }
  if (tid == 0 && p.nlevels) *p.nlevels = L;

  // ---- tree replay + unreached core vertices + start-tree patch ----------------
  // Replay (TEET/TEOLV, et_bfs.cpp:14-32): the tree arrays and, per anchor, its
  // visited bit and depth are fetched together (two dependent round trips;
  // an unreached anchor's stale depth is simply ignored).
  for (uint64_t t0 = tid; t0 < p.nt; t0 += kReplay * nthreads) {
    uint32_t a[kReplay], td[kReplay], ts[kReplay], vis[kReplay], da[kReplay];
#pragma unroll
    for (int k = 0; k < kReplay; ++k) {
      const uint64_t t = t0 + k * nthreads;
      const uint32_t tv = static_cast<uint32_t>(p.nc + t);
      const bool in = t < p.nt && !(tv >= p.skip_lo && tv < p.skip_hi);
      a[k] = in ? p.tanchor[t] : kNone32 - 1;
      td[k] = in ? p.tdepth[t] : 0u;
      ts[k] = in ? p.tsrc[t] : 0u;
    }
#pragma unroll
    for (int k = 0; k < kReplay; ++k) {
      const bool ok = a[k] < kNone32 - 1;
      vis[k] = ok ? test_bit(p.visited, a[k]) : 0u;
#ifdef ETB_EXP_NO_DA  // timing experiment only (wrong depths): replay without the anchor-depth gather
      da[k] = 0u;
#else
      da[k] = ok ? __ldcg(&p.dp[a[k]].x) : 0u;
#endif
    }
#pragma unroll
    for (int k = 0; k < kReplay; ++k) {
      if (a[k] == kNone32 - 1) continue;  // out of range or inside the start's tree
      p.dp[p.nc + t0 + k * nthreads] =
          vis[k] ? make_uint2(da[k] + td[k], ts[k]) : make_uint2(kNone32, kNone32);
    }
  }
  {
    // A warp reads 32 visited words, then clears the unreached vertices of each
    // word with one coalesced 256-byte store (padding bits are set).
    const unsigned lane = threadIdx.x & 31;
    const uint64_t gw = tid >> 5, nw = nthreads >> 5;
    for (uint64_t w0 = gw * 32; w0 < p.nwords; w0 += nw * 32) {
      const uint32_t un = w0 + lane < p.nwords ? ~p.visited[w0 + lane] : 0u;
      for (unsigned m = __ballot_sync(0xffffffffu, un != 0); m; m &= m - 1) {
        const int j = __ffs(m) - 1;
        if ((__shfl_sync(0xffffffffu, un, j) >> lane) & 1u)
          p.dp[(w0 + j) * 32 + lane] = make_uint2(kNone32, kNone32);
      }
    }
  }
  for (uint64_t i = tid; i < p.npatch; i += nthreads) {
    const uint32_t v = p.patch[3 * i];
    p.dp[v] = make_uint2(p.patch[3 * i + 1], p.patch[3 * i + 2]);
  }
  // inline patch entries: constant indices keep them in the parameter bank
#pragma unroll
  for (int k = 0; k < kInlinePatch; ++k)
    if (tid == static_cast<uint64_t>(k) && static_cast<uint32_t>(k) < p.nipatch)
      p.dp[p.ipatch[3 * k]] = make_uint2(p.ipatch[3 * k + 1], p.ipatch[3 * k + 2]);

  // ---- clean the other state half for the next traversal --------------------
  {
    const uint32_t tail = p.nc & 31u;
    for (uint64_t i = tid; i < p.nwords; i += nthreads) {
      p.visited_next[i] = (i == p.nwords - 1 && tail) ? ~0u << tail : 0u;  // padding: visited
      p.fb0_next[i] = 0;
      p.fb1_next[i] = 0;
      p.fb2_next[i] = 0;
    }
    if (tid < 32) p.ctr_next[tid] = 0;
  }
  stamp(p, 511);
  if (p.bstamp) {
    __syncthreads();
    if (threadIdx.x == 0) p.bstamp[63 * gridDim.x + blockIdx.x] = gtimer();
  }
}

template <int B>
__global__ void __launch_bounds__(B, 1) et_bfs_kernel(BfsParams p) {
  et_bfs_body<(B == 1024)>(p);
}

// ============================================================================
// (5) The 1D core partition (bfs_part.cuh): partition k owns core words
// (hubs) and 256-vertex blocks (the rest) dealt round robin over the degree
// order, as the paper's SRRS (Alg. 4), and the trees anchored there. The level
// loop is the single-partition one, run by each partition over its own work
// with the same step functions:
//   bottom-up  its owned visited words (bu_step / bu_sweep on a PartView whose
//              word index maps onto the owned blocks);
//   top-down   every frontier row's owned neighbours (the partition's top-down
//              CSR), atomic-free claims (td_step<3>), the frontier list built
//              per level from the replicated frontier bitmap;
// claims touch only partition-local memory (owned visited and next-frontier
// words). At the end of a level each partition pushes its owned next-frontier
// words to every peer's replica — the per-level frontier-bitmap allgather,
// fused into the kernel as whole 32-byte sectors over peer memory (NVLink) or
// local memory (all partitions on one GPU) — counting its claims and α/β scout
// in the same pass, and one barrier over all partitions adds the partials into
// every partition's counters, so every partition takes the same α/β decision.
// ============================================================================

// What the step functions read, for one partition: the core graph (bottom-up:
// the whole replicated CSR; top-down: the partition's owned-neighbour CSR) and
// result array, the partition's own visited replica, its CTA group and its
// owned words.
struct PartView {
  const uint64_t* crow;
  const uint32_t* ccol;
  const uint32_t* cfirst;
  const uint32_t* csecond;
  const uint2* cthird;
  const uint32_t* degn;
  const uint2* cmeta;
  uint2* dp;
  uint32_t* visited;
  uint32_t nc, nwords;
  uint32_t part, nparts;
  uint32_t nwo;   // owned words
  uint32_t nhub;  // of which in the hub region (one word at a time)
  unsigned cta, ncta;
  unsigned long long* wstamp;  // (ETB_WARP_STAMPS diagnostics: unused here)
  int32_t wdepth;
  bool dyn;  // bottom-up runs from the CTA's counter (large-core kernel)
};
__device__ __forceinline__ uint64_t wlo_of(const PartView&) { return 0; }
__device__ __forceinline__ uint32_t whi_of(const PartView& v) { return v.nwo; }
__device__ __forceinline__ unsigned cta_of(const PartView& v) { return v.cta; }
__device__ __forceinline__ unsigned ncta_of(const PartView& v) { return v.ncta; }
__device__ __forceinline__ uint32_t seg_off(const PartView&, uint32_t) { return 0; }
template <> struct IsPart<PartView> { static constexpr bool value = true; };
// stride of the aligned 8-word run starting at owned index i0
__device__ __forceinline__ uint64_t run_stride(const PartView& v, uint64_t i0) {
  return i0 < v.nhub ? v.nparts : 1;
}
__device__ __forceinline__ uint64_t word_at(const PartView& v, uint64_t i) {
  return owned_word(static_cast<uint32_t>(i), v.part, v.nparts, v.nhub);
}

// Exchange-block counters (per partition): two parities of {four level slots
// of [claims, scout, grab, -], conversion counters at [16], [17]}; [62] cross
// barriers completed by earlier launches, [63] launches completed. Launch k
// uses parity k & 1 and clears the other parity at its start: every peer's add
// into that parity happened in launch k - 1, before its last cross barrier.
constexpr int kXkSlot = 62, kLaunchSlot = 63;

__device__ __forceinline__ unsigned long long ld_acquire_sys(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

// Barrier over the `n` CTAs of one partition's group (this GPU's memory only).
__device__ __forceinline__ void group_sync(unsigned long long* bar, unsigned n) {
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned long long old = atom_add_release(bar, 1ull);
    const unsigned long long target = (old / n + 1) * n;
    const long long t0 = clock64();
    while (ld_acquire(bar) < target)
      if (clock64() - t0 > 40000000000ll) __trap();
    smem_view().bu_next = 0;
  }
  __syncthreads();
}

// The level barrier over every CTA of every partition: block-reduce (a, b),
// add them into every partition's counters at `off`, release this CTA's writes
// (owned results, pushed replica words) and arrive at every partition's
// counter; complete when all nparts x group CTAs arrived (`target` counts
// arrivals since the counters were created). Thread 0 then reads the n totals
// at rd once for the CTA (sm.tot).
__device__ void part_level_sync(const PartParams& pp, uint32_t part, unsigned par, Smem& sm,
                                unsigned long long a, unsigned long long b, uint32_t off,
                                unsigned long long target, const unsigned long long* rd, int n) {
  const bool sys = pp.system_scope;
  const unsigned lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  a = warp_sum(a);
  b = warp_sum(b);
  if (lane == 0) {
    sm.red[0][wib] = a;
    sm.red[1][wib] = b;
  }
  __syncthreads();
  if (threadIdx.x < 32) {
    const unsigned nwb = blockDim.x >> 5;
    a = warp_sum(lane < nwb ? sm.red[0][lane] : 0ull);
    b = warp_sum(lane < nwb ? sm.red[1][lane] : 0ull);
    if (lane == 0) {
      for (uint32_t q = 0; q < pp.nparts; ++q) {
        unsigned long long* c = pp.parts[q].ctr + 32 * par + off;
        if (sys) {
          if (a) atomicAdd_system(&c[0], a);
          if (b) atomicAdd_system(&c[1], b);
        } else {
          if (a) atomicAdd(&c[0], a);
          if (b) atomicAdd(&c[1], b);
        }
      }
      if (sys) __threadfence_system(); else __threadfence();
      for (uint32_t q = 0; q < pp.nparts; ++q) {
        if (sys) atomicAdd_system(pp.parts[q].arrive, 1ull);
        else atomicAdd(pp.parts[q].arrive, 1ull);
      }
      const unsigned long long* me_arrive = pp.parts[part].arrive;
      const long long t0 = clock64();
      while ((sys ? ld_acquire_sys(me_arrive) : ld_acquire(me_arrive)) < target)
        if (clock64() - t0 > 40000000000ll) __trap();
      for (int k = 0; k < n; ++k) sm.tot[k] = ld_volatile(&rd[k]);
      sm.bu_next = 0;
    }
  }
  __syncthreads();
}

// The frontier bitmap (replica, all words) -> this partition's list of
// frontier vertices with owned neighbours and the prefix of their owned-row
// lengths (as convert_step, over the top-down CSR trow).
__device__ void part_convert(const PartView& v, const uint64_t* trow, const uint32_t* fcur,
                             uint32_t* qv, uint64_t* qp, unsigned long long* cslot) {
  const unsigned lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const uint64_t gw = (uint64_t)wib * v.ncta + v.cta;
  const uint64_t nw = (uint64_t)(v.ncta * blockDim.x) >> 5;
  for (uint64_t w0 = gw * 32; w0 < v.nwords; w0 += nw * 32) {
    const uint64_t wi = w0 + lane;
    const uint32_t bits = wi < v.nwords ? fcur[wi] : 0u;
    uint32_t cnt = 0, edges = 0;
    for (uint32_t b = bits; b; b &= b - 1) {
      const uint32_t x = static_cast<uint32_t>(wi * 32 + __ffs(b) - 1);
      const uint32_t d = static_cast<uint32_t>(trow[x + 1] - trow[x]);
      cnt += d != 0;
      edges += d;
    }
    const uint32_t vin = warp_incl_scan(cnt);
    const uint32_t vtot = __shfl_sync(0xffffffffu, vin, 31);
    if (vtot == 0) continue;
    const unsigned long long ein = warp_incl_scan64(edges);
    const unsigned long long etot = __shfl_sync(0xffffffffu, ein, 31);
    unsigned long long old = 0;
    if (lane == 31) old = atomicAdd(cslot, ((unsigned long long)vtot << kItemShift) | etot);
    old = __shfl_sync(0xffffffffu, old, 31);
    uint64_t vpos = (old >> kItemShift) + vin - cnt, epos = (old & kItemMask) + ein - edges;
    for (uint32_t b = bits; b; b &= b - 1) {
      const uint32_t x = static_cast<uint32_t>(wi * 32 + __ffs(b) - 1);
      const uint32_t d = static_cast<uint32_t>(trow[x + 1] - trow[x]);
      if (!d) continue;
      qv[vpos] = x;
      qp[vpos] = epos;
      ++vpos;
      epos += d;
    }
  }
}

// The allgather of one level: this partition's owned next-frontier words, 32
// per warp iteration (four whole 8-word blocks: four 32-byte sectors per peer),
// into every peer's replica of that ring slot; with kCount also the level's
// claims (popcount) and α/β scout (Σ full degree, coalesced: lane = vertex).
template <bool kCount>
__device__ void part_push(const PartParams& pp, uint32_t part, const PartView& v, uint32_t ring,
                          bool dense, const uint32_t* fnext, unsigned long long& claims,
                          unsigned long long& scout) {
  const unsigned lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const uint64_t gw = (uint64_t)wib * v.ncta + v.cta;
  const uint64_t nw = (uint64_t)(v.ncta * blockDim.x) >> 5;
  for (uint64_t j0 = gw * 32; j0 < v.nwo; j0 += nw * 32) {
    const bool in = j0 + lane < v.nwo;
    const uint32_t wi = in ? static_cast<uint32_t>(word_at(v, j0 + lane)) : 0u;
    const uint32_t f = in ? __ldcg(&fnext[wi]) : 0u;
    // Replica slots are cleared whole by their holder one level ahead (before
    // the barrier after which peers push into them), so past level 0 only
    // words with claims travel and sparse top-down levels push little; level
    // 0's slot was not (a peer may reach its first push before this launch's
    // init), so level 0 pushes every owned word.
    for (uint32_t q = 0; q < pp.nparts; ++q) {
      if (q == part || !in || (!dense && f == 0u)) continue;
      const PartDev& pq = pp.parts[q];
      uint32_t* dst = ring == 0 ? pq.fb0 : (ring == 1 ? pq.fb1 : pq.fb2);
      ETB_DCHECK(wi < v.nwords);
      dst[wi] = f;
    }
    if (kCount) {
      claims += __popc(f);
      if (__any_sync(0xffffffffu, f != 0)) {
#pragma unroll 4
        for (int j = 0; j < 32; ++j) {
          const uint32_t bits = __shfl_sync(0xffffffffu, f, j);
          const uint32_t w = __shfl_sync(0xffffffffu, wi, j);
          if ((bits >> lane) & 1u) scout += v.degn[(uint64_t)w * 32 + lane];
        }
      }
    }
  }
}

// Bottom-up levels: each warp pushes the owned next-frontier words IT wrote —
// bu_step / bu_sweep give every owned word one writer, the warp whose run
// holds it (claims of the first probes and of the deferred misses alike) — so
// the words are final when the warp's step returns and the push needs no
// partition barrier. Runs: R consecutive owned indices starting at
// (gw + i * nw) * R, gw / nw as in bu_step (CTA-major). kCount: also the
// claimed vertices' full degrees (the scout of a top-down level run bottom-up).
template <int R, bool kCount>
__device__ void part_push_own(const PartParams& pp, uint32_t part, const PartView& v, uint32_t ring,
                              bool dense, const uint32_t* fnext, unsigned long long& scout) {
  static_assert(R == 8 || R == 32, "bu_step runs of 8 or bu_sweep runs of 32");
  const unsigned lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const uint64_t gw = (uint64_t)v.cta * (blockDim.x >> 5) + wib;
  const uint64_t nw = (uint64_t)(v.ncta * blockDim.x) >> 5;
  constexpr unsigned kRuns = 32 / R;  // runs per warp iteration
  __syncwarp();
  for (uint64_t i0 = 0;; i0 += kRuns) {
    const uint64_t first = (gw + i0 * nw) * R;
    if (first >= v.nwo) break;
    const uint64_t j = (gw + (i0 + lane / R) * nw) * R + lane % R;
    const bool in = j < v.nwo;
    const uint32_t wi = in ? static_cast<uint32_t>(word_at(v, j)) : 0u;
    const uint32_t f = in ? __ldcg(&fnext[wi]) : 0u;
    for (uint32_t q = 0; q < pp.nparts; ++q) {
      if (q == part || !in || (!dense && f == 0u)) continue;
      const PartDev& pq = pp.parts[q];
      uint32_t* dst = ring == 0 ? pq.fb0 : (ring == 1 ? pq.fb1 : pq.fb2);
      dst[wi] = f;
    }
    if (kCount && __any_sync(0xffffffffu, f != 0)) {
#pragma unroll 4
      for (int k = 0; k < 32; ++k) {
        const uint32_t bits = __shfl_sync(0xffffffffu, f, k);
        const uint32_t w = __shfl_sync(0xffffffffu, wi, k);
        if ((bits >> lane) & 1u) scout += v.degn[(uint64_t)w * 32 + lane];
      }
    }
  }
}

// Does partition `part` of G own relaid vertex x (core block, tree by anchor,
// component trees and isolated vertices to the last partition)?
__device__ __forceinline__ bool owns(const BfsParams& p, const PartDev& me, uint32_t part,
                                     uint32_t G, uint32_t x) {
  if (x < p.nc) return core_owner(x, G) == part;
  if (x < p.nc + p.nt) {
    const uint32_t a = p.tanchor[x - p.nc];
    return a == kNone32 ? part == G - 1 : core_owner(a, G) == part;
  }
  return x >= me.zlo && x < me.zhi;
}

template <bool kLarge>
__device__ __forceinline__ void et_bfs_part_body(const PartParams& pp) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  Smem& sm = *reinterpret_cast<Smem*>(smem_raw);
  const BfsParams& p = pp.base;
  const unsigned gsize = gridDim.x / pp.local_parts;
  const unsigned cta = blockIdx.x % gsize;
  const uint32_t part = pp.first_part + blockIdx.x / gsize;
  const uint32_t G = pp.nparts;
  const PartDev& me = pp.parts[part];
  const uint64_t gtid = (uint64_t)cta * blockDim.x + threadIdx.x;
  const uint64_t gthreads = (uint64_t)gsize * blockDim.x;
  const bool lead = part == 0 && cta == 0 && threadIdx.x == 0;
  const bool stats = p.level_claims && lead;
  PartView v;  // bottom-up view: the whole core CSR
  v.crow = p.crow;
  v.ccol = p.ccol;
  v.cfirst = p.cfirst;
  v.csecond = p.csecond;
  v.cthird = p.cthird;
  v.degn = p.degn;
  v.cmeta = p.cmeta;
  v.dp = p.dp;
  v.visited = me.visited;
  v.nc = p.nc;
  v.nwords = p.nwords;
  v.part = part;
  v.nparts = G;
  v.nwo = me.nwo;
  v.nhub = me.nhub;
  v.cta = cta;
  v.ncta = gsize;
  v.wstamp = nullptr;
  v.wdepth = -1;
  v.dyn = ETB_PART_DYN && kLarge;
  PartView vt = v;  // top-down view: the partition's owned-neighbour CSR
  vt.crow = me.trow;
  vt.ccol = me.tcol;
  const unsigned long long launch = me.ctr[kLaunchSlot];
  const unsigned par = static_cast<unsigned>(launch & 1u);
  unsigned long long* const ctr = me.ctr + 32 * par;
  unsigned long long xk = me.ctr[kXkSlot];  // cross barriers completed by earlier launches
  const unsigned long long per_barrier = static_cast<unsigned long long>(G) * gsize;
  const uint32_t start = p.start;
  const bool run_core = start != kNone32;
  if (stats) p.level_claims[256] = gtimer();
  if (p.bstamp && threadIdx.x == 0) p.bstamp[62 * gridDim.x + blockIdx.x] = gtimer();
  if (threadIdx.x == 0) sm.bu_next = 0;

  // ---- init: this partition's own memory only (no cross barrier) -------------
  if (gtid < 18) me.ctr[32 * (par ^ 1u) + gtid] = 0;
  {
    const uint32_t tail = p.nc & 31u;
    const uint32_t sw = run_core ? start >> 5 : kNone32, sb = run_core ? 1u << (start & 31) : 0u;
    for (uint64_t i = gtid; i < p.nwords; i += gthreads)  // a bottom-up level 0 probes it all
      me.fb0[i] = i == sw ? sb : 0u;
    for (uint64_t j = gtid; j < me.nwo; j += gthreads) {
      // owned words only: peers may push level 0's words into the others
      // before this init is done
      const uint32_t i = static_cast<uint32_t>(word_at(v, j));
      uint32_t vis = i == sw ? sb : 0u;
      if (i == p.nwords - 1 && tail) vis |= ~0u << tail;
      me.visited[i] = vis;
      me.fb1[i] = 0;
    }
  }
  if (run_core && gtid == 0 && core_owner(start, G) == part)
    p.dp[start] = make_uint2(static_cast<uint32_t>(p.base_depth), p.start_parent);
  group_sync(me.bar, gsize);
  if (stats) p.level_claims[257] = gtimer();

  uint32_t L = 0;
  if (run_core) {
    uint32_t* F[3] = {me.fb0, me.fb1, me.fb2};
    unsigned long long frontier = 1, scout = p.degn[start], awake = 0, prev = 0, reached = 1;
    double etc = p.edges_to_check;
    bool bu = p.bottom_up_only || (!p.top_down_only && (double)scout > etc / p.alpha);
    if (bu) awake = frontier;
    for (;;) {
      uint32_t* fcur = F[L % 3];
      uint32_t* fnext = F[(L + 1) % 3];
      uint32_t* fzero = F[(L + 2) % 3];
      unsigned long long* slot = ctr + (L & 3) * 4;
      // the whole replica slot (owned words and the peers' pushed words: a
      // peer pushes only its nonzero words into it, after the next barrier)
      for (uint64_t i = gtid; i < p.nwords; i += gthreads) fzero[i] = 0;
      if (gtid == 0) {
        ctr[((L + 2) & 3) * 4 + 0] = 0;
        ctr[((L + 2) & 3) * 4 + 1] = 0;
        ctr[((L + 2) & 3) * 4 + 2] = 0;
        ctr[((L + 2) & 3) * 4 + 3] = 0;
        ctr[16 + ((L + 1) & 1)] = 0;
      }
      if (stats && L < 255) p.trace[L] = bu ? 'b' : 't';
      const int32_t dnext = p.base_depth + static_cast<int32_t>(L) + 1;
      unsigned long long claims_acc = 0, scout_acc = 0;
      uint32_t* mb = sm.w[threadIdx.x >> 5].cbuf;
      const bool td_bu = !bu && p.td_as_bu > 0.0 && !p.top_down_only && L > 0 &&
                         (double)scout > p.td_as_bu * (double)(p.nc - reached);
      if (bu || td_bu) {
        // bottom-up, or a top-down level executed as a bottom-up sweep over the
        // owned unvisited words (as et_bfs_body; decided on the frontier's full
        // degree sum, known to every partition before any list is built): same
        // claims, its scout counted by the push. No partition barrier: every
        // warp pushes the owned words it wrote (part_push_own).
        if (bu) prev = awake;
        else etc -= (double)scout;
        const uint32_t ring = (L + 1) % 3;
        const bool sweep = kLarge && (double)(p.nc - reached) * kSweepT < (double)p.nc;
        if (sweep) bu_sweep<32>(v, mb, fcur, fnext, dnext, claims_acc, nullptr, nullptr, nullptr);
        else bu_step<kBuU>(v, mb, fcur, fnext, dnext, claims_acc, nullptr, nullptr, nullptr);
        // With the CTA's run counter (v.dyn) the CTA's warps shared its runs:
        // once the CTA is through (a CTA barrier), each warp pushes its static
        // share of them — the same run set, final words.
        if (v.dyn) __syncthreads();
        if (sweep) {
          if (td_bu) part_push_own<32, true>(pp, part, v, ring, L == 0, fnext, scout_acc);
          else part_push_own<32, false>(pp, part, v, ring, L == 0, fnext, scout_acc);
        } else {
          if (td_bu) part_push_own<kBuU, true>(pp, part, v, ring, L == 0, fnext, scout_acc);
          else part_push_own<kBuU, false>(pp, part, v, ring, L == 0, fnext, scout_acc);
        }
        if (p.bstamp && threadIdx.x == 0 && L < 62) p.bstamp[L * gridDim.x + blockIdx.x] = gtimer();
      } else {
        etc -= (double)scout;
        uint64_t nq = 0, ne = 0;
        if (L == 0) {
          ne = me.trow[start + 1] - me.trow[start];  // the start's owned neighbours, no list
          nq = ne != 0;
        } else {
          unsigned long long* cslot = ctr + 16 + (L & 1);
          part_convert(v, me.trow, fcur, me.qv, me.qp, cslot);
          group_sync(me.bar, gsize);
          if (threadIdx.x == 0) sm.tot[2] = ld_volatile(cslot);
          __syncthreads();
          nq = sm.tot[2] >> kItemShift;
          ne = sm.tot[2] & kItemMask;
        }
        // Levels with a small frontier claim with returning atomics, counting
        // claims and scout as they go (most targets are unvisited: only the
        // winners write); large ones claim atomic-free and count in the push
        // pass (as the single-partition kernel's list-less levels).
        const bool small = (double)scout < p.emit_limit;
        if (small)
          td_step<0, kLarge>(vt, mb, sm.w[threadIdx.x >> 5].win, me.qv, me.qp, nq, ne, nullptr,
                             nullptr, fnext, slot, dnext, scout_acc, claims_acc,
                             L == 0 ? start : kNone32);
        else
          td_step<3, kLarge>(vt, mb, sm.w[threadIdx.x >> 5].win, me.qv, me.qp, nq, ne, nullptr,
                             nullptr, fnext, slot, dnext, scout_acc, claims_acc,
                             L == 0 ? start : kNone32);
        if (p.bstamp && threadIdx.x == 0 && L < 62) p.bstamp[L * gridDim.x + blockIdx.x] = gtimer();
        group_sync(me.bar, gsize);
        if (small)
          part_push<false>(pp, part, v, (L + 1) % 3, L == 0, fnext, claims_acc, scout_acc);
        else
          part_push<true>(pp, part, v, (L + 1) % 3, L == 0, fnext, claims_acc, scout_acc);
      }
      ++xk;
      part_level_sync(pp, part, par, sm, claims_acc, bu ? 0ull : scout_acc, (L & 3) * 4,
                      xk * per_barrier, slot, 2);
      const unsigned long long claims = sm.tot[0];
      const unsigned long long scout_tot = sm.tot[1];
      reached += claims;
      if (stats) {
        if (L < 254) p.level_claims[258 + L] = gtimer();
        if (L < 256) p.level_claims[L] = claims;
      }
      ++L;
      if (bu && p.bottom_up_only) {
        if (claims == 0) break;  // run_block_search (bfs.cpp:295-305)
      } else if (bu) {
        awake = claims;
        if (!(awake > 0 && (awake >= prev || (double)awake > (double)p.nc / p.beta))) {
          bu = false;
          frontier = awake;
          scout = 1;
        }
      } else {
        frontier = claims;
        scout = scout_tot;
      }
      if (!bu) {
        if (frontier == 0) break;
        if (!p.top_down_only && (double)scout > etc / p.alpha) {
          bu = true;
          awake = frontier;
        }
      }
      if (reached == p.reachable) {  // the start's component is exhausted (as et_bfs_body)
        if (stats && L < 255) p.trace[L] = bu ? 'b' : 't';
        if (stats && L < 256) p.level_claims[L] = 0;
        if (stats && L < 254) p.level_claims[258 + L] = gtimer();
        ++L;
        break;
      }
    }
  }
  if (stats && p.nlevels) *p.nlevels = L;

  // ---- owned tree replay + owned core fill + owned patch entries ---------------
  // (as et_bfs_body's final phase over the partition's vertices: four tree
  // entries in flight per thread, and a warp clears the unreached vertices of
  // 32 owned visited words with coalesced 256-byte stores)
  for (uint64_t t0 = gtid; t0 < me.ntrees; t0 += 4 * gthreads) {
    uint32_t tv[4], a[4], td[4], ts[4], vb[4], da[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const uint64_t i = t0 + k * gthreads;
      tv[k] = i < me.ntrees ? me.trees[i] : kNone32;
    }
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const bool in = tv[k] != kNone32 && !(tv[k] >= p.skip_lo && tv[k] < p.skip_hi);
      const uint32_t t = tv[k] - p.nc;
      a[k] = in ? p.tanchor[t] : kNone32 - 1;
      td[k] = in ? p.tdepth[t] : 0u;
      ts[k] = in ? p.tsrc[t] : 0u;
    }
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const bool ok = a[k] < kNone32 - 1;
      vb[k] = ok ? test_bit(me.visited, a[k]) : 0u;
      da[k] = ok ? __ldcg(&p.dp[a[k]].x) : 0u;
    }
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      if (a[k] == kNone32 - 1) continue;  // out of range or inside the start's tree
      p.dp[tv[k]] = vb[k] ? make_uint2(da[k] + td[k], ts[k]) : make_uint2(kNone32, kNone32);
    }
  }
  {
    const unsigned lane = threadIdx.x & 31;
    const uint64_t gw = gtid >> 5, nw = gthreads >> 5;
    for (uint64_t j0 = gw * 32; j0 < me.nwo; j0 += nw * 32) {
      const bool in = j0 + lane < me.nwo;
      const uint32_t wi = in ? static_cast<uint32_t>(word_at(v, j0 + lane)) : 0u;
      const uint32_t un = in ? ~me.visited[wi] : 0u;
      for (unsigned m = __ballot_sync(0xffffffffu, un != 0); m; m &= m - 1) {
        const int j = __ffs(m) - 1;
        const uint32_t w = __shfl_sync(0xffffffffu, wi, j);
        if ((__shfl_sync(0xffffffffu, un, j) >> lane) & 1u)
          p.dp[(uint64_t)w * 32 + lane] = make_uint2(kNone32, kNone32);
      }
    }
  }
  for (uint64_t i = gtid; i < p.npatch; i += gthreads) {
    const uint32_t x = p.patch[3 * i];
    if (owns(p, me, part, G, x)) p.dp[x] = make_uint2(p.patch[3 * i + 1], p.patch[3 * i + 2]);
  }
#pragma unroll
  for (int k = 0; k < kInlinePatch; ++k)
    if (gtid == static_cast<uint64_t>(k) && static_cast<uint32_t>(k) < p.nipatch &&
        owns(p, me, part, G, p.ipatch[3 * k]))
      p.dp[p.ipatch[3 * k]] = make_uint2(p.ipatch[3 * k + 1], p.ipatch[3 * k + 2]);
  if (p.bstamp) {
    __syncthreads();
    if (threadIdx.x == 0) p.bstamp[63 * gridDim.x + blockIdx.x] = gtimer();
  }
  if (cta == 0 && threadIdx.x == 0) {
    me.ctr[kXkSlot] = xk;
    me.ctr[kLaunchSlot] = launch + 1;
  }
  if (stats) p.level_claims[511] = gtimer();
}

template <int B>
__global__ void __launch_bounds__(B, 1) et_bfs_part_kernel(const __grid_constant__ PartParams pp) {
  et_bfs_part_body<(B == 1024)>(pp);
}

}  // namespace

const void* kernel_for(int block) {
  return block == kSmallBlock ? reinterpret_cast<const void*>(et_bfs_kernel<kSmallBlock>)
                              : reinterpret_cast<const void*>(et_bfs_kernel<1024>);
}

// Measured on B200 (tools/root_profile.py, 64 roots, end of round 1): the
// small-core kernel at scale 22 runs 68.2 us per root at 640 threads (with 7
// words per bottom-up iteration) vs 69.6 at 768 and 92 with the 1024-thread
// large-core kernel; at scale 26 the large-core kernel at 1024 threads runs
// 471 us vs 476 at 896 and 578 for the small-core kernel.
// ETB_BFS_BLOCK=640|1024 overrides (experiments).
const void* part_kernel_for(int block) {
  return block == kSmallBlock ? reinterpret_cast<const void*>(et_bfs_part_kernel<kSmallBlock>)
                              : reinterpret_cast<const void*>(et_bfs_part_kernel<1024>);
}

size_t bfs_smem_bytes() { return sizeof(Smem); }

// The single-partition kernel's dynamic shared memory: Smem plus, with the
// TMA-fed bottom-up step, one two-stage pipe per warp.
size_t bfs_kernel_smem(int block) {
  if (!ETB_BU_TMA) return sizeof(Smem);
  const size_t pipe = block == kSmallBlock ? sizeof(BuPipe<kBuUSmall>) : sizeof(BuPipe<kBuU>);
  return sizeof(Smem) + static_cast<size_t>(block / 32) * pipe;
}

// Checked builds: the source line of the first failed device check (0: none,
// or an unchecked build); reading it clears it.
unsigned debug_check_line() {
#ifdef ETB_DEBUG_CHECKS
  unsigned v = 0, z = 0;
  ETB_CUDA(cudaMemcpyFromSymbol(&v, etb_check_line, 4));
  ETB_CUDA(cudaMemcpyToSymbol(etb_check_line, &z, 4));
  return v;
#else
  return 0;
#endif
}

int block_for(uint64_t nc) {
  if (const char* e = getenv("ETB_BFS_BLOCK")) {
    const int b = atoi(e);
    if (b == kSmallBlock || b == 1024) return b;
  }
  return nc < (uint64_t{1} << 23) ? kSmallBlock : 1024;
}

// Persisting L2 access-policy window over [base, base + bytes) on stream s
// (see bfs_state_init); false when off (ETB_L2_PERSIST=0) or too large.
bool set_l2_window(cudaStream_t s, void* base, size_t bytes) {
  int dev = 0, maxp = 0;
  ETB_CUDA(cudaGetDevice(&dev));
  ETB_CUDA(cudaDeviceGetAttribute(&maxp, cudaDevAttrMaxPersistingL2CacheSize, dev));
  const char* pe = getenv("ETB_L2_PERSIST");
  if ((pe && atoi(pe) <= 0) || bytes > static_cast<size_t>(maxp) / 2) return false;
  // the carve-out is per device: never shrink it under another layout's window
  size_t cur = 0;
  ETB_CUDA(cudaDeviceGetLimit(&cur, cudaLimitPersistingL2CacheSize));
  if (cur < bytes) ETB_CUDA(cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, bytes));
  cudaStreamAttrValue a = {};
  a.accessPolicyWindow.base_ptr = base;
  a.accessPolicyWindow.num_bytes = bytes;
  a.accessPolicyWindow.hitRatio = 1.0f;
  a.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
  a.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
  ETB_CUDA(cudaStreamSetAttribute(s, cudaStreamAttributeAccessPolicyWindow, &a));
  return true;
}

void bfs_state_init(const DevLayout& L, BfsState& S, cudaStream_t s) {
  const uint64_t n = L.n;
  S.n = n;
  // per half: whole words + 1, rounded to 16 bytes (every half starts aligned
  // for the bottom-up step's bulk copies)
  const uint64_t words = ((L.nc + 31) / 32 + 1 + 3) & ~uint64_t{3};
  S.words = words;
  S.bits.alloc(8 * words);
  const uint64_t cap = L.nc + 2;
  S.qv0.alloc(cap);
  S.qv1.alloc(cap);
  S.qp0.alloc(cap);
  S.qp1.alloc(cap);
  S.ctr.alloc(64);
  // both halves clean: visited zero but the last word's padding bits
  ETB_CUDA(cudaMemsetAsync(S.bits.get(), 0, 8 * words * 4, s));
  ETB_CUDA(cudaMemsetAsync(S.ctr.get(), 0, 64 * 8, s));
  if (const uint32_t tail = static_cast<uint32_t>(L.nc & 31u)) {
    const uint32_t pad = ~0u << tail;
    const uint64_t last = (L.nc + 31) / 32 - 1;
    for (int h = 0; h < 2; ++h)
      ETB_CUDA(cudaMemcpyAsync(S.visited() + h * words + last, &pad, 4,
                               cudaMemcpyHostToDevice, s));
  }
  S.parity = 0;
  S.bar.alloc(1);
  ETB_CUDA(cudaMemsetAsync(S.bar.get(), 0, 8, s));
  S.dp.alloc(n ? n : 1);
  // Isolated vertices stay unreached unless they are the start; everything
  // else is rewritten by every traversal.
  ETB_CUDA(cudaMemsetAsync(S.dp.get(), 0xFF, (n ? n : 1) * 8, s));
  S.trace.alloc(256);
  S.level_claims.alloc(512);
  ETB_CUDA(cudaMemsetAsync(S.level_claims.get(), 0, 512 * 8, s));  // stamps read as "not taken"
  S.nlevels.alloc(1);
  const uint64_t pcap = std::max<uint64_t>(L.max_tree, 1) + 2;
  S.patch.alloc(3 * pcap);
  S.h_patch.alloc(3 * pcap);
  if (!S.patch_done) ETB_CUDA(cudaEventCreateWithFlags(&S.patch_done, cudaEventDisableTiming));
  int dev = 0, sms = 0, per_sm = 0;
  ETB_CUDA(cudaGetDevice(&dev));
  ETB_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  S.block = block_for(L.nc);
  const void* k = kernel_for(S.block);
  ETB_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                (int)bfs_kernel_smem(S.block)));
  ETB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k, S.block,
                                                         bfs_kernel_smem(S.block)));
  if (per_sm < 1) throw CudaError("et_bfs_kernel cannot be resident");
  S.grid = sms;  // one CTA per SM (the level barrier's arrivals)
  // L2 access-policy window over the per-root bitmap state (on by default,
  // ETB_L2_PERSIST=0 turns it off): its lines are kept in the persisting L2
  // carve-out, out of reach of the streamed CSR / result traffic (s26: +2.7%
  // harmonic-mean GTEPS with every root started cold, persisting lines
  // included — etb_time_roots demotes them before its L2 flush; s22: +-0).
  // Only when the whole state fits half the carve-out: a window larger than
  // the carve-out thrashed at scale 28 (2x slower per root).
  S.l2_window = set_l2_window(s, S.bits.get(), S.bits.bytes());
  ETB_CUDA(cudaStreamSynchronize(s));
}

void bfs_fill_params(const DevLayout& L, BfsState& S, BfsParams& p) {
  p.crow = L.crow.get();
  p.ccol = L.ccol.get();
  p.cfirst = L.cfirst.get();
  p.csecond = L.csecond.get();
  p.cthird = L.cthird.get();
  p.reachable = L.nc;
  p.degn = L.degn.get();
  p.cmeta = L.cmeta.get();
  p.nc = static_cast<uint32_t>(L.nc);
  p.nwords = static_cast<uint32_t>((L.nc + 31) / 32);
  p.tsrc = L.tsrc.get();
  p.tanchor = L.tanchor.get();
  p.tdepth = L.tdepth.get();
  p.nt = static_cast<uint32_t>(L.nt);
  const uint64_t cur = S.parity * S.words, nxt = (S.parity ^ 1u) * S.words;
  p.visited = S.visited() + cur;
  p.fb0 = S.fb0() + cur;
  p.fb1 = S.fb1() + cur;
  p.fb2 = S.fb2() + cur;
  p.visited_next = S.visited() + nxt;
  p.fb0_next = S.fb0() + nxt;
  p.fb1_next = S.fb1() + nxt;
  p.fb2_next = S.fb2() + nxt;
  p.qv0 = S.qv0.get();
  p.qv1 = S.qv1.get();
  p.qp0 = S.qp0.get();
  p.qp1 = S.qp1.get();
  p.ctr = S.ctr.get() + 32 * S.parity;
  p.ctr_next = S.ctr.get() + 32 * (S.parity ^ 1u);
  p.bar = S.bar.get();
  p.dp = S.dp.get();
  p.patch = S.patch.get();
  p.npatch = 0;
  p.nipatch = 0;
  p.edges_to_check = static_cast<double>(L.ecore);
  // (nc/8: s26 -3.5 us per root against nc/4 — more of the large levels take
  // the list-less path; s22 unchanged)
  p.emit_limit = static_cast<double>(L.nc) / 8.0 + 1024.0;
  p.td_as_bu = kTdAsBuDefault;
  p.small_mode3_edges = kSmallMode3Default;
  if (const char* e = getenv("ETB_SMALL_MODE3")) p.small_mode3_edges = atof(e);
  if (const char* e = getenv("ETB_TD_AS_BU")) p.td_as_bu = atof(e);
  p.split_ratio = kSplitRatioDefault;
  double split_div = kSplitDivDefault;
  if (const char* e = getenv("ETB_SPLIT_RATIO")) p.split_ratio = atof(e);
  if (const char* e = getenv("ETB_SPLIT_DIV")) split_div = std::max(1.0, atof(e));
  p.split_bound = static_cast<uint32_t>(std::max(32.0, static_cast<double>(L.nc) / split_div));
  p.split_tdw = kSplitTdwDefault;
  if (const char* e = getenv("ETB_SPLIT_TDW")) p.split_tdw = static_cast<uint32_t>(atoi(e));
  p.trace = nullptr;
  p.level_claims = nullptr;
  p.bstamp = nullptr;
  p.wstamp = nullptr;
  p.wdepth = -1;
  p.nlevels = nullptr;
}

void bfs_prepare_start(const DevLayout& L, BfsState& S, uint64_t start, BfsParams& p,
                       cudaStream_t s) {
  const uint64_t nc = L.nc, nt = L.nt;
  if (S.patch_done) ETB_CUDA(cudaEventSynchronize(S.patch_done));
  uint32_t* ph = S.h_patch.get();
  uint32_t np = 0;
  p.skip_lo = p.skip_hi = 0;
  p.start = kNone32;
  p.base_depth = 0;
  p.start_parent = kNone32;
  if (S.last_isolated != kNone32 && S.last_isolated != start) {
    ph[3 * np] = S.last_isolated;
    ph[3 * np + 1] = 0xFFFFFFFFu;
    ph[3 * np + 2] = kNone32;
    ++np;
  }
  S.last_isolated = kNone32;
  if (start < nc) {
    p.start = static_cast<uint32_t>(start);
    p.start_parent = static_cast<uint32_t>(start);
  } else if (start < nc + nt) {
    // Start-side walk over the start's tree (et_bfs.cpp:34-57): the tree is a
    // contiguous id range; parents always precede children.
    const uint32_t* src = L.h_tsrc.data();
    const uint32_t* dep = L.h_tdepth.data();
    uint32_t r = static_cast<uint32_t>(start);
    for (;;) {
      const uint32_t sp = src[r - nc];
      if (sp == r || sp < nc) break;
      r = sp;
    }
    const auto it = std::upper_bound(L.h_tree_start.begin(), L.h_tree_start.end(), r);
    const uint32_t lo = r;
    const uint32_t hi = it == L.h_tree_start.end() ? static_cast<uint32_t>(nc + nt) : *it;
    const uint32_t sz = hi - lo;
    static thread_local std::vector<uint32_t> dist, par;
    static thread_local std::vector<uint8_t> anc;
    dist.assign(sz, 0);
    par.assign(sz, kNone32);
    anc.assign(sz, 0);
    const uint32_t s0 = static_cast<uint32_t>(start);
    anc[s0 - lo] = 1;
    par[s0 - lo] = s0;
    for (uint32_t x = s0; x != r;) {
      const uint32_t up = src[x - nc];
      anc[up - lo] = 1;
      par[up - lo] = x;
      x = up;
    }
    const uint32_t ds = dep[s0 - nc];
    for (uint32_t x = lo; x < hi; ++x) {
      const uint32_t i = x - lo;
      if (anc[i]) {
        dist[i] = ds - dep[x - nc];
      } else {
        const uint32_t up = src[x - nc];
        dist[i] = dist[up - lo] + 1;
        par[i] = up;
      }
      ph[3 * np] = x;
      ph[3 * np + 1] = dist[i];
      ph[3 * np + 2] = par[i];
      ++np;
    }
    p.skip_lo = lo;
    p.skip_hi = hi;
    const uint32_t ce = src[r - nc];
    if (ce != r) {  // attached tree: continue from its core-edge vertex
      p.start = ce;
      p.base_depth = static_cast<int32_t>(ds);
      p.start_parent = r;
    }
  } else {
    ph[3 * np] = static_cast<uint32_t>(start);
    ph[3 * np + 1] = 0;
    ph[3 * np + 2] = static_cast<uint32_t>(start);
    ++np;
    S.last_isolated = static_cast<uint32_t>(start);
  }
  // the start's core component bounds the traversal (see the level loop's end)
  p.reachable = p.start != kNone32 && p.start < L.h_comp_size.size() ? L.h_comp_size[p.start]
                                                                       : L.nc;
  p.npatch = 0;
  p.nipatch = 0;
  if (np <= static_cast<uint32_t>(kInlinePatch)) {
    std::copy(ph, ph + 3 * np, p.ipatch);
    p.nipatch = np;
  } else {
    p.npatch = np;
    ETB_CUDA(cudaMemcpyAsync(S.patch.get(), ph, np * 12, cudaMemcpyHostToDevice, s));
    ETB_CUDA(cudaEventRecord(S.patch_done, s));
  }
}

__global__ void __launch_bounds__(1024, 1) empty_kernel(unsigned long long* sink) {
  if (sink && threadIdx.x == 0 && blockIdx.x == 0) *sink = 0;
}

void empty_launch(const BfsState& S, cudaStream_t s) {
  unsigned long long* sink = nullptr;
  void* args[] = {&sink};
  ETB_CUDA(cudaLaunchCooperativeKernel(reinterpret_cast<void*>(empty_kernel), dim3(S.grid),
                                       dim3(S.block), args, sizeof(Smem), s));
}

void bfs_launch(const BfsParams& p, BfsState& S, cudaStream_t s) {
  void* args[] = {const_cast<BfsParams*>(&p)};
  ETB_CUDA(cudaLaunchCooperativeKernel(kernel_for(S.block), dim3(S.grid), dim3(S.block), args,
                                       bfs_kernel_smem(S.block), s));
  S.parity ^= 1u;  // this launch cleans the other half; the next one uses it
}

void debug_diag(uint64_t* out, bool reset, cudaStream_t s) {
  ETB_CUDA(cudaMemcpyFromSymbolAsync(out, g_diag, sizeof(g_diag), 0, cudaMemcpyDeviceToHost, s));
  if (reset) {
    static const unsigned long long zero[kDiag] = {};
    ETB_CUDA(cudaMemcpyToSymbolAsync(g_diag, zero, sizeof(zero), 0, cudaMemcpyHostToDevice, s));
  }
  ETB_CUDA(cudaStreamSynchronize(s));
}

}  // namespace etb
