// (5) Partitioned ET-BFS kernel — see bfs_part.cuh for the scheme.
#include <algorithm>

#include "bfs_dev.cuh"
#include "bfs_part.cuh"

namespace etb {
namespace {

using namespace dev;

constexpr int kPBlock = 512;
constexpr int kPWarps = kPBlock / 32;
constexpr int kPEpl = kTdChunk / 32;
constexpr int kPMiss = 256;
constexpr int kPBuU = 4;
constexpr unsigned long long kPGrab = 4;

struct PSmem {
  uint32_t mbuf[kPWarps][kPMiss];
  unsigned long long red[2][kPWarps];
  unsigned long long tot[4];  // values read once per CTA after a barrier
};

// The next-frontier replicas of every partition (index ni of the ring), so a
// claim is published to all partitions as it happens: no exchange phase.
struct Peers {
  uint32_t* f[kMaxParts];
  uint32_t n;
  uint32_t self;
  bool sys;
  __device__ __forceinline__ void or_bit(uint32_t v) const {
    for (uint32_t q = 0; q < n; ++q) {
      if (sys && q != self) atomicOr_system(&f[q][v >> 5], 1u << (v & 31));
      else atomicOr(&f[q][v >> 5], 1u << (v & 31));
    }
  }
  __device__ __forceinline__ void store_word(uint64_t w, uint32_t m) const {
    for (uint32_t q = 0; q < n; ++q) f[q][w] = m;  // owned words: one writer
  }
};

// ctr layout (per partition, exchange block): [0..15] four level slots of
// {claims, scout, top-down grab counter, unused}; [16], [17] conversion
// counters (packed list length << 36 | owned edges); [30] cross barriers completed by
// earlier launches.
constexpr int kShift = 36;
constexpr unsigned long long kMask = (1ull << kShift) - 1;

__device__ __forceinline__ unsigned long long ld_acquire_sys(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ void fence(bool sys) {
  if (sys) __threadfence_system(); else __threadfence();
}

// Barrier over the nb CTAs of one partition's block group.
__device__ void group_sync(unsigned long long* bar, unsigned nb, bool sys) {
  __syncthreads();
  if (threadIdx.x == 0) {
    fence(sys);
    const unsigned long long old = atomicAdd(bar, 1ull);
    const unsigned long long target = (old / nb + 1) * nb;
    const long long t0 = clock64();
    while (ld_acquire(bar) < target)
      if (clock64() - t0 > 40000000000ll) __trap();
    fence(sys);
  }
  __syncthreads();
}

// The level barrier over every CTA of every partition. Each CTA reduces its
// (a, b) partials, adds them into every partition's counters `off`, publishes
// its writes (replica words, results) and arrives at every partition's
// counter; the barrier completes when all nparts x gsize CTAs have arrived
// (`target` counts arrivals since the counters were created). Thread 0 then
// reads the n counters at `rd` once for the CTA (sm.tot).
__device__ void part_sync(const PartParams& pp, const PartDev& me, PSmem& sm,
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
    a = warp_sum(lane < kPWarps ? sm.red[0][lane] : 0ull);
    b = warp_sum(lane < kPWarps ? sm.red[1][lane] : 0ull);
    if (lane == 0) {
      for (uint32_t q = 0; q < pp.nparts; ++q) {
        unsigned long long* c = pp.parts[q].ctr + off;
        if (sys) {
          if (a) atomicAdd_system(&c[0], a);
          if (b) atomicAdd_system(&c[1], b);
        } else {
          if (a) atomicAdd(&c[0], a);
          if (b) atomicAdd(&c[1], b);
        }
      }
      fence(sys);  // release: the CTA's writes (ordered by bar.sync) before the arrival
      for (uint32_t q = 0; q < pp.nparts; ++q) {
        if (sys) atomicAdd_system(pp.parts[q].arrive, 1ull);
        else atomicAdd(pp.parts[q].arrive, 1ull);
      }
      const long long t0 = clock64();
      while ((sys ? ld_acquire_sys(me.arrive) : ld_acquire(me.arrive)) < target)
        if (clock64() - t0 > 40000000000ll) __trap();
      for (int k = 0; k < n; ++k) sm.tot[k] = ld_volatile(&rd[k]);
    }
  }
  __syncthreads();
}

// Replicated frontier bitmap -> this partition's list of frontier vertices
// with a non-empty owned segment.
__device__ void part_convert(const BfsParams& p, const PartDev& me, const uint32_t* fcur,
                             unsigned long long* cslot, uint64_t gw, uint64_t nw) {
  const unsigned lane = threadIdx.x & 31;
  for (uint64_t w0 = gw * 32; w0 < p.nwords; w0 += nw * 32) {
    const uint64_t wi = w0 + lane;
    const uint32_t bits = wi < p.nwords ? fcur[wi] : 0u;
    uint32_t cnt = 0, nch = 0;  // vertices with an owned segment, their owned edges
    for (uint32_t b = bits; b; b &= b - 1) {
      const uint32_t c = me.seg[static_cast<uint32_t>(wi * 32 + __ffs(b) - 1)].y;
      cnt += c != 0;
      nch += c;
    }
    const uint32_t vin = warp_incl_scan(cnt), cin = warp_incl_scan(nch);
    const uint32_t vtot = __shfl_sync(0xffffffffu, vin, 31);
    if (vtot == 0) continue;
    const uint32_t ctot = __shfl_sync(0xffffffffu, cin, 31);
    unsigned long long old = 0;
    if (lane == 31) old = atomicAdd(cslot, ((unsigned long long)vtot << kShift) | ctot);
    old = __shfl_sync(0xffffffffu, old, 31);
    uint64_t vpos = (old >> kShift) + vin - cnt, cpos = (old & kMask) + cin - nch;
    for (uint32_t b = bits; b; b &= b - 1) {
      const uint32_t v = static_cast<uint32_t>(wi * 32 + __ffs(b) - 1);
      const uint32_t c = me.seg[v].y;
      if (!c) continue;
      me.qv[vpos] = v;
      me.qp[vpos] = cpos;
      ++vpos;
      cpos += c;
    }
  }
}

// Top-down over the owned segments of the frontier rows, merge path: the list
// holds the frontier vertices with a non-empty owned segment and the exclusive
// prefix of the segment lengths; the concatenated segments are cut into
// kTdChunk-edge chunks (long segments span many, short ones share one), a
// warp's chunk window of list entries staged in shared memory (as td_step in
// bfs.cu, without the list emission: partitions rebuild their lists from the
// replicated bitmap).
__device__ __forceinline__ uint32_t pwin_search(const int32_t* win, int32_t rel) {
  uint32_t lo = 0, hi = kTdChunk;
  while (hi - lo > 1) {
    const uint32_t m = (lo + hi) >> 1;
    if (win[m] <= rel) lo = m; else hi = m;
  }
  return lo;
}

__device__ void part_td(const BfsParams& p, const PartDev& me, uint64_t nq, uint64_t ne,
                        const Peers& fnext, unsigned long long* grab, int32_t dnext, uint64_t gw,
                        uint64_t nw, int32_t* win, unsigned long long& scout_acc,
                        unsigned long long& claims_acc) {
  const unsigned lane = threadIdx.x & 31;
  const uint64_t nu = (ne + kTdChunk - 1) / kTdChunk;
  const uint32_t* qv = me.qv;
  const uint64_t* qp = me.qp;
  for (uint64_t g0 = gw, gn = 1; g0 < nu;) {
    const uint64_t g1 = min(nu, g0 + gn);
    uint64_t i = find_vertex(qp, nq, g0 * kTdChunk);
    for (uint64_t c = g0; c < g1; ++c) {
      const uint64_t e0 = c * kTdChunk, e1 = min(ne, e0 + kTdChunk);
      const uint64_t qi = qp[i];
      const uint64_t iend = i + 1 < nq ? qp[i + 1] : ne;
      const bool single = iend >= e1;
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
        inext = i + pwin_search(win, kTdChunk);
      } else {
        inext = iend == e1 ? i + 1 : i;
      }
      uint32_t u[kPEpl], w[kPEpl], vw[kPEpl];
      bool cl[kPEpl];
      if (single) {  // one segment: its vertex and start once for the chunk
        const uint32_t uu = qv[i];
        const uint64_t base = p.crow[uu] + me.seg[uu].x + (e0 - qi);
#pragma unroll
        for (int j = 0; j < kPEpl; ++j) {
          const uint32_t rel = lane + 32 * j;
          u[j] = rel < e1 - e0 ? uu : kNone32;
          w[j] = u[j] != kNone32 ? p.ccol[base + rel] : kNone32;
        }
      } else {
        uint32_t k = pwin_search(win, static_cast<int32_t>(lane));
#pragma unroll
        for (int j = 0; j < kPEpl; ++j) {
          const uint32_t rel = lane + 32 * j;
          while (k + 1 < kTdChunk && win[k + 1] <= static_cast<int32_t>(rel)) ++k;
          u[j] = rel < e1 - e0 ? qv[i + k] : kNone32;
          w[j] = static_cast<uint32_t>(k);
        }
#pragma unroll
        for (int j = 0; j < kPEpl; ++j) {
          const uint32_t rel = lane + 32 * j;
          uint32_t col = kNone32;
          if (u[j] != kNone32) {
            const uint64_t vs = w[j] == 0 ? qi : e0 + static_cast<uint64_t>(max(win[w[j]], 0));
            col = p.ccol[p.crow[u[j]] + me.seg[u[j]].x + (e0 + rel - vs)];
          }
          w[j] = col;
        }
      }
#pragma unroll
      for (int j = 0; j < kPEpl; ++j) vw[j] = w[j] != kNone32 ? me.visited[w[j] >> 5] : ~0u;
#pragma unroll
      for (int j = 0; j < kPEpl; ++j) {
        const uint32_t bit = 1u << (w[j] & 31);
        cl[j] = false;
        if (!(vw[j] & bit)) cl[j] = !(atomicOr(&me.visited[w[j] >> 5], bit) & bit);
      }
      uint32_t dg[kPEpl];
#pragma unroll
      for (int j = 0; j < kPEpl; ++j) {
        dg[j] = 0;
        if (cl[j]) {
          p.dp[w[j]] = make_uint2(static_cast<uint32_t>(dnext), u[j]);
          fnext.or_bit(w[j]);
          dg[j] = p.degn[w[j]];
        }
      }
#pragma unroll
      for (int j = 0; j < kPEpl; ++j) {
        scout_acc += dg[j];
        claims_acc += cl[j];
      }
      __syncwarp();
      i = inext;
    }
    if (nu <= nw) break;
    unsigned long long next = 0;
    // guided grabs (as the large-core single-GPU kernel): 4..16 chunks,
    // shrinking with the chunks left, so the per-partition counter is not
    // saturated on levels with ~10^6 chunks
    const uint64_t rem = nu - min(nu, g1);
    const uint64_t want = nu <= 8 * nw ? 1 : max((uint64_t)kPGrab, min(uint64_t{16}, rem / (4 * nw)));
    if (lane == 0) next = nw + atomicAdd(grab, (unsigned long long)want);
    g0 = __shfl_sync(0xffffffffu, next, 0);
    gn = want;
  }
}

// Deferred bottom-up misses (as the single-GPU kernel's resolve_misses): each
// lane scans two rows together over their next kPLaneFirst neighbours (two
// probes per row in flight, per-row early exit); rows without a hit there are
// finished by the whole warp, 32 probes per round trip.
constexpr uint32_t kPLaneFirst = 64;

__device__ __forceinline__ void part_claim(const BfsParams& p, const PartDev& me,
                                           const Peers& fnext, uint32_t v, uint32_t par,
                                           int32_t dnext, unsigned long long& claims_acc) {
  p.dp[v] = make_uint2(static_cast<uint32_t>(dnext), par);
  atomicOr(&me.visited[v >> 5], 1u << (v & 31));
  fnext.or_bit(v);
  ++claims_acc;
}

__device__ void part_misses(const BfsParams& p, const PartDev& me, const uint32_t* fcur,
                            const Peers& fnext, uint32_t* mbuf, uint32_t nmiss, int32_t dnext,
                            unsigned long long& claims_acc) {
  const unsigned lane = threadIdx.x & 31;
  __syncwarp();
  uint32_t nlong = 0;
  for (uint32_t i0 = 0; i0 < nmiss; i0 += 64) {
    const uint32_t va = i0 + lane < nmiss ? mbuf[i0 + lane] : kNone32;
    const uint32_t vb = i0 + 32 + lane < nmiss ? mbuf[i0 + 32 + lane] : kNone32;
    uint64_t rba = 0, rea = 0, rbb = 0, reb = 0;
    if (va != kNone32) rba = p.crow[va], rea = p.crow[va + 1];
    if (vb != kNone32) rbb = p.crow[vb], reb = p.crow[vb + 1];
    const uint64_t la = min(rea, rba + 1 + kPLaneFirst), lb = min(reb, rbb + 1 + kPLaneFirst);
    uint64_t ea = rba + 1, eb = rbb + 1, enda = va != kNone32 ? la : 0,
             endb = vb != kNone32 ? lb : 0;
    uint32_t pa = 0, pb = 0;
    bool ha = false, hb = false;
    while (ea < enda || eb < endb) {
      const uint32_t x0 = ea < enda ? p.ccol[ea] : kNone32;
      const uint32_t x1 = ea + 1 < enda ? p.ccol[ea + 1] : kNone32;
      const uint32_t y0 = eb < endb ? p.ccol[eb] : kNone32;
      const uint32_t y1 = eb + 1 < endb ? p.ccol[eb + 1] : kNone32;
      const bool bx0 = x0 != kNone32 && test_bit(fcur, x0);
      const bool bx1 = x1 != kNone32 && test_bit(fcur, x1);
      const bool by0 = y0 != kNone32 && test_bit(fcur, y0);
      const bool by1 = y1 != kNone32 && test_bit(fcur, y1);
      if (bx0 || bx1) pa = bx0 ? x0 : x1, ha = true, enda = ea;
      else ea += 2;
      if (by0 || by1) pb = by0 ? y0 : y1, hb = true, endb = eb;
      else eb += 2;
    }
    if (ha) part_claim(p, me, fnext, va, pa, dnext, claims_acc);
    if (hb) part_claim(p, me, fnext, vb, pb, dnext, claims_acc);
    const bool lnga = va != kNone32 && !ha && la < rea;
    const bool lngb = vb != kNone32 && !hb && lb < reb;
    __syncwarp();
    const unsigned lma = __ballot_sync(0xffffffffu, lnga);
    if (lnga) mbuf[nlong + __popc(lma & ((1u << lane) - 1))] = va;
    nlong += __popc(lma);
    const unsigned lmb = __ballot_sync(0xffffffffu, lngb);
    if (lngb) mbuf[nlong + __popc(lmb & ((1u << lane) - 1))] = vb;
    nlong += __popc(lmb);
    __syncwarp();
  }
  for (uint32_t i = 0; i < nlong; ++i) {
    const uint32_t v = mbuf[i];
    const uint64_t rb = p.crow[v] + 1 + kPLaneFirst, re = p.crow[v + 1];
    uint32_t par = kNone32;
    for (uint64_t e0 = rb; e0 < re; e0 += 32) {
      const uint64_t e = e0 + lane;
      const uint32_t x = e < re ? p.ccol[e] : kNone32;
      const unsigned m = __ballot_sync(0xffffffffu, x != kNone32 && test_bit(fcur, x));
      if (m) {
        par = __shfl_sync(0xffffffffu, x, __ffs(m) - 1);
        break;
      }
    }
    if (lane == 0 && par != kNone32) part_claim(p, me, fnext, v, par, dnext, claims_acc);
  }
  __syncwarp();
}

// Bottom-up over the owned visited words.
__device__ void part_bu(const BfsParams& p, const PartDev& me, uint32_t* mbuf,
                        const uint32_t* fcur, const Peers& fnext, int32_t dnext, uint64_t gw,
                        uint64_t nw, unsigned long long& claims_acc) {
  const unsigned lane = threadIdx.x & 31;
  const unsigned lt = (1u << lane) - 1;
  const uint64_t wlo = me.lo >> 5, whi = (static_cast<uint64_t>(me.hi) + 31) >> 5;
  uint32_t nmiss = 0;
  for (uint64_t w0 = wlo + gw * kPBuU; w0 < whi; w0 += nw * kPBuU) {
    uint32_t vis[kPBuU];
    bool any = false;
#pragma unroll
    for (int k = 0; k < kPBuU; ++k) {
      vis[k] = w0 + k < whi ? me.visited[w0 + k] : ~0u;
      any |= vis[k] != ~0u;
    }
    if (!any) continue;
    uint32_t f[kPBuU];
#pragma unroll
    for (int k = 0; k < kPBuU; ++k)
      f[k] = ((vis[k] >> lane) & 1u) ? kNone32 : p.cfirst[(w0 + k) * 32 + lane];
    bool hit[kPBuU];
#pragma unroll
    for (int k = 0; k < kPBuU; ++k) hit[k] = f[k] != kNone32 && test_bit(fcur, f[k]);
#pragma unroll
    for (int k = 0; k < kPBuU; ++k) {
      const uint32_t v = static_cast<uint32_t>((w0 + k) * 32 + lane);
      const unsigned m = __ballot_sync(0xffffffffu, hit[k]);
      if (hit[k]) p.dp[v] = make_uint2(static_cast<uint32_t>(dnext), f[k]);
      if (lane == 0 && m) {
        me.visited[w0 + k] = vis[k] | m;
        fnext.store_word(w0 + k, m);
        claims_acc += __popc(m);
      }
      const bool miss = f[k] != kNone32 && !hit[k];
      const unsigned mm = __ballot_sync(0xffffffffu, miss);
      if (miss) mbuf[nmiss + __popc(mm & lt)] = v;
      nmiss += __popc(mm);
    }
    if (nmiss > kPMiss - 32 * kPBuU) {
      part_misses(p, me, fcur, fnext, mbuf, nmiss, dnext, claims_acc);
      nmiss = 0;
    }
  }
  if (nmiss) part_misses(p, me, fcur, fnext, mbuf, nmiss, dnext, claims_acc);
}

__device__ __forceinline__ bool owns(const PartDev& me, uint32_t v) {
  return (v >= me.lo && v < me.hi) || (v >= me.tlo && v < me.thi) || (v >= me.zlo && v < me.zhi);
}

__global__ void __launch_bounds__(kPBlock, 2) et_bfs_part_kernel(PartParams pp) {
  __shared__ PSmem sm;
  const BfsParams& p = pp.base;
  const uint32_t gsize = gridDim.x / pp.local_parts;
  const uint32_t group = blockIdx.x / gsize;
  const uint32_t part = pp.first_part + group;
  const PartDev& me = pp.parts[part];
  const bool sys = pp.system_scope;
  const bool leader_block = (blockIdx.x % gsize) == 0;
  const uint64_t gtid = (uint64_t)(blockIdx.x % gsize) * blockDim.x + threadIdx.x;
  const uint64_t gthreads = (uint64_t)gsize * blockDim.x;
  const uint64_t gw = gtid >> 5, nw = gthreads >> 5;
  const bool stats = p.level_claims && part == 0 && leader_block && threadIdx.x == 0;
  const uint32_t start = p.start;
  const bool run_core = start != kNone32;
  unsigned long long xk = me.ctr[30];  // cross barriers completed by earlier launches
  // phase timestamps as the single-partition kernel's (partition 0, block 0)
  auto pstamp = [&](uint32_t slot) {
    if (stats && slot < 512) p.level_claims[slot] = gtimer();
  };
  pstamp(256);

  // ---- init (own replicas) ----------------------------------------------------
  const uint32_t tail = p.nc & 31u;
  for (uint64_t i = gtid; i < p.nwords; i += gthreads) {
    uint32_t vis = 0, f0 = 0;
    if (i == p.nwords - 1 && tail) vis = ~0u << tail;
    if (run_core && i == (start >> 5)) {
      vis |= 1u << (start & 31);
      f0 = 1u << (start & 31);
    }
    me.visited[i] = vis;
    me.fb0[i] = f0;
    me.fb1[i] = 0;
    me.fb2[i] = 0;
  }
  if (gtid < 20) me.ctr[gtid] = 0;
  if (run_core && gtid == 0 && start >= me.lo && start < me.hi)
    p.dp[start] = make_uint2(static_cast<uint32_t>(p.base_depth), p.start_parent);
  const unsigned long long per_barrier = static_cast<unsigned long long>(pp.nparts) * gsize;
  ++xk;  // every partition initialised its replicas before any peer writes into them
  part_sync(pp, me, sm, 0, 0, 0, xk * per_barrier, nullptr, 0);
  pstamp(257);

  uint32_t L = 0;
  if (run_core) {
    uint32_t* F[3] = {me.fb0, me.fb1, me.fb2};
    unsigned long long frontier = 1, scout = p.degn[start], awake = 0, prev = 0, reached = 1;
    double etc = p.edges_to_check;
    bool bu = p.bottom_up_only || (!p.top_down_only && (double)scout > etc / p.alpha);
    if (bu) awake = frontier;
    for (;;) {
      const uint32_t fi = L % 3, ni = (L + 1) % 3, zi = (L + 2) % 3;
      uint32_t* fcur = F[fi];
      uint32_t* fnext = F[ni];
      uint32_t* fzero = F[zi];
      unsigned long long* slot = me.ctr + (L & 3) * 4;
      for (uint64_t i = gtid; i < p.nwords; i += gthreads) fzero[i] = 0;
      if (gtid == 0) {
        me.ctr[((L + 2) & 3) * 4 + 0] = 0;
        me.ctr[((L + 2) & 3) * 4 + 1] = 0;
        me.ctr[((L + 2) & 3) * 4 + 2] = 0;
        me.ctr[16 + ((L + 1) & 1)] = 0;
      }
      if (stats && L < 255) p.trace[L] = bu ? 'b' : 't';
      const int32_t dnext = p.base_depth + static_cast<int32_t>(L) + 1;
      unsigned long long claims_acc = 0, scout_acc = 0;
      Peers fn;  // this level's next-frontier replicas, ours and the peers'
      fn.n = pp.nparts;
      fn.self = part;
      fn.sys = sys;
      for (uint32_t q = 0; q < pp.nparts; ++q) {
        const PartDev& pq = pp.parts[q];
        fn.f[q] = q == part ? fnext : (ni == 0 ? pq.fb0 : (ni == 1 ? pq.fb1 : pq.fb2));
      }
      if (bu) {
        prev = awake;
        part_bu(p, me, sm.mbuf[threadIdx.x >> 5], fcur, fn, dnext, gw, nw, claims_acc);
      } else {
        etc -= (double)scout;
        unsigned long long* cslot = me.ctr + 16 + (L & 1);
        part_convert(p, me, fcur, cslot, gw, nw);
        group_sync(me.bar, gsize, sys);
        if (threadIdx.x == 0) sm.tot[2] = ld_volatile(cslot);  // once per CTA
        __syncthreads();
        const unsigned long long cp = sm.tot[2];
        part_td(p, me, cp >> kShift, cp & kMask, fn, &slot[2], dnext, gw, nw,
                reinterpret_cast<int32_t*>(sm.mbuf[threadIdx.x >> 5]), scout_acc, claims_acc);
      }
      // one barrier over all partitions: partials added everywhere, claims already
      // published into every replica
      ++xk;
      part_sync(pp, me, sm, claims_acc, scout_acc, (L & 3) * 4, xk * per_barrier, slot, 2);
      const unsigned long long claims = sm.tot[0];
      const unsigned long long scout_tot = sm.tot[1];
      reached += claims;
      pstamp(258 + L);
      if (stats && L < 256) p.level_claims[L] = claims;
      ++L;
      if (bu && p.bottom_up_only) {
        // standalone block sweeps to fixpoint (run_block_search, bfs.cpp:295-305)
        if (claims == 0) break;
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
      // every core vertex of the start's component visited: the next level
      // claims nothing (see bfs.cu)
      if (reached == p.reachable) {
        if (stats && L < 255) p.trace[L] = bu ? 'b' : 't';
        if (stats && L < 256) p.level_claims[L] = 0;
        ++L;
        pstamp(258 + L - 1);
        break;
      }
    }
  }
  if (stats && p.nlevels) *p.nlevels = L;
  if (leader_block && threadIdx.x == 0) me.ctr[30] = xk;

  // ---- owned core fill + owned tree replay + owned patch entries -----------------
  const uint64_t wlo = me.lo >> 5, whi = (static_cast<uint64_t>(me.hi) + 31) >> 5;
  for (uint64_t wi = wlo + gtid; wi < whi; wi += gthreads)
    for (uint32_t un = ~me.visited[wi]; un; un &= un - 1) {
      const uint64_t v = wi * 32 + __ffs(un) - 1;
      p.dp[v] = make_uint2(kNone32, kNone32);
    }
  for (uint64_t tv = me.tlo + gtid; tv < me.thi; tv += gthreads) {
    if (tv >= p.skip_lo && tv < p.skip_hi) continue;
    const uint64_t t = tv - p.nc;
    const uint32_t a = p.tanchor[t];
    uint2 out = make_uint2(kNone32, kNone32);
    if (a != kNone32 && test_bit(me.visited, a))
      out = make_uint2(__ldcg(&p.dp[a].x) + p.tdepth[t], p.tsrc[t]);
    p.dp[tv] = out;
  }
  for (uint64_t i = gtid; i < p.npatch; i += gthreads) {
    const uint32_t v = p.patch[3 * i];
    if (owns(me, v)) p.dp[v] = make_uint2(p.patch[3 * i + 1], p.patch[3 * i + 2]);
  }
#pragma unroll
  for (int k = 0; k < kInlinePatch; ++k)
    if (gtid == static_cast<uint64_t>(k) && static_cast<uint32_t>(k) < p.nipatch &&
        owns(me, p.ipatch[3 * k]))
      p.dp[p.ipatch[3 * k]] = make_uint2(p.ipatch[3 * k + 1], p.ipatch[3 * k + 2]);
  pstamp(511);
}

// seg[u] = {offset, length} of u's neighbours inside [lo, hi) (rows ascend).
__global__ void seg_kernel(const uint64_t* crow, const uint32_t* ccol, uint64_t nc, uint32_t lo,
                           uint32_t hi, uint2* seg) {
  for (uint64_t u = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; u < nc;
       u += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t rb = crow[u], re = crow[u + 1];
    uint64_t a = rb, b = re;
    while (a < b) {
      const uint64_t m = (a + b) >> 1;
      if (ccol[m] < lo) a = m + 1; else b = m;
    }
    uint64_t c = a, d = re;
    while (c < d) {
      const uint64_t m = (c + d) >> 1;
      if (ccol[m] < hi) c = m + 1; else d = m;
    }
    seg[u] = make_uint2(static_cast<uint32_t>(a - rb), static_cast<uint32_t>(c - a));
  }
}

}  // namespace

PartState::~PartState() {
  for (void* m : peer_maps)
    if (m) cudaIpcCloseMemHandle(m);
}

void part_bounds(const DevLayout& L, uint32_t nparts, std::vector<PartDev>& out) {
  if (nparts < 1 || nparts > kMaxParts)
    throw std::invalid_argument("etb_layout_partition: partitions must be in [1, 16]");
  out.assign(nparts, PartDev{});
  const uint64_t nc = L.nc, nt = L.nt;
  // Core: V_k = [k nc / G, (k+1) nc / G) rounded down to whole 32-vertex words.
  for (uint32_t k = 0; k < nparts; ++k) {
    const uint64_t lo = k == 0 ? 0 : ((k * nc / nparts) & ~uint64_t{31});
    const uint64_t hi = k + 1 == nparts ? nc : (((k + 1) * nc / nparts) & ~uint64_t{31});
    out[k].lo = static_cast<uint32_t>(lo);
    out[k].hi = static_cast<uint32_t>(std::max(lo, hi));
  }
  // Trees follow their anchor (trees are laid out in anchor order); component
  // trees and isolated vertices go to the last partition.
  const auto& anc = L.h_tanchor;
  uint64_t first_component = nt;
  for (uint64_t i = 0; i < nt; ++i)
    if (anc[i] == kNone32) {
      first_component = i;
      break;
    }
  for (uint32_t k = 0; k < nparts; ++k) {
    auto lb = [&](uint32_t bound) {
      return static_cast<uint64_t>(std::lower_bound(anc.begin(), anc.begin() + first_component,
                                                    bound) - anc.begin());
    };
    const uint64_t t0 = k == 0 ? 0 : lb(out[k].lo);
    const uint64_t t1 = k + 1 == nparts ? nt : lb(out[k + 1].lo);
    out[k].tlo = static_cast<uint32_t>(nc + t0);
    out[k].thi = static_cast<uint32_t>(nc + t1);
    out[k].zlo = out[k].zhi = static_cast<uint32_t>(L.n);
  }
  out[nparts - 1].zlo = static_cast<uint32_t>(nc + nt);
}

void part_build(const DevLayout& L, PartState& P, uint32_t nparts, uint32_t first, uint32_t local,
                cudaStream_t s) {
  P.nparts = nparts;
  P.first = first;
  P.local = local;
  part_bounds(L, nparts, P.h_parts);
  const uint64_t nc = L.nc;
  const uint64_t words = (nc + 31) / 32 + 1;
  P.seg.alloc(local * (nc ? nc : 1));
  P.visited.alloc(local * words);
  P.qv.alloc(local * (nc + 1));
  P.qp.alloc(local * (nc + 1));
  P.xbytes = ((3 * words * 4 + 255) / 256) * 256 + 32 * 8 + 256;
  P.xblock.alloc(local * P.xbytes);
  ETB_CUDA(cudaMemsetAsync(P.xblock.get(), 0, local * P.xbytes, s));
  P.bar.alloc(local);
  ETB_CUDA(cudaMemsetAsync(P.bar.get(), 0, local * 8, s));
  for (uint32_t j = 0; j < local; ++j) {
    PartDev& d = P.h_parts[first + j];
    unsigned char* xb = P.xblock.get() + j * P.xbytes;
    d.fb0 = reinterpret_cast<uint32_t*>(xb);
    d.fb1 = d.fb0 + words;
    d.fb2 = d.fb1 + words;
    d.ctr = reinterpret_cast<unsigned long long*>(xb + ((3 * words * 4 + 255) / 256) * 256);
    d.arrive = d.ctr + 32;
    d.bar = P.bar.get() + j;
    d.visited = P.visited.get() + j * words;
    d.qv = P.qv.get() + j * (nc + 1);
    d.qp = P.qp.get() + j * (nc + 1);
    uint2* sg = P.seg.get() + j * (nc ? nc : 1);
    d.seg = sg;
    if (nc) {
      seg_kernel<<<grid_for(nc, 256), 256, 0, s>>>(L.crow.get(), L.ccol.get(), nc, d.lo, d.hi, sg);
      ETB_LAUNCH_CHECK();
    }
  }
  P.d_parts.alloc(nparts);
  ETB_CUDA(cudaMemcpyAsync(P.d_parts.get(), P.h_parts.data(), nparts * sizeof(PartDev),
                           cudaMemcpyHostToDevice, s));
  int dev = 0, sms = 0, per_sm = 0;
  ETB_CUDA(cudaGetDevice(&dev));
  ETB_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  ETB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, et_bfs_part_kernel, kPBlock, 0));
  if (per_sm < 1) throw CudaError("et_bfs_part_kernel cannot be resident");
  int grid = sms * std::min(per_sm, 2);
  grid -= grid % static_cast<int>(local);  // equal block groups
  P.grid = grid;
  ETB_CUDA(cudaStreamSynchronize(s));
}

void part_launch(const PartParams& p, const PartState& P, cudaStream_t s) {
  void* args[] = {const_cast<PartParams*>(&p)};
  ETB_CUDA(cudaLaunchCooperativeKernel(reinterpret_cast<void*>(et_bfs_part_kernel), dim3(P.grid),
                                       dim3(kPBlock), args, 0, s));
}

}  // namespace etb
