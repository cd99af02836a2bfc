// Device primitives of the (untimed) preprocessing, hand-written for sm_100a:
// LSD radix sort of u64 keys (optionally carrying u32 values), stable unique /
// flagged selection, exclusive / inclusive scans and a sum reduction.
//
// Used by the CSR build (build.cpp:21-87 restated: key sort + dedupe, graph_build.cu),
// the relayout's order sorts (relayout.cpp:37-180, layout.cu) and the degree
// split (preprocess.cpp:16-67, graph_tools.cu). All of them are HBM-streaming
// passes; nothing here is on the timed BFS path.
//
// Scans and selections: three-phase tile passes (tile totals -> scan of the
// totals, recursively -> tile scan with its offset), 512 threads x 8 items per
// tile, loads and stores coalesced through a shared-memory transpose.
// Radix sort: 8-bit digits, one pass per digit below end_bit; each pass is an
// upsweep (per-CTA digit histograms over a contiguous key range, per-warp
// shared-memory counters), one scan of the digit-major [256 x CTAs] counts,
// and a downsweep that re-reads the range in rounds of 512 keys and scatters
// each key to its stable position: warp-level peers by __match_any_sync, then
// a per-digit prefix over the warps of the round, then the CTA's running
// per-digit offset. Ties keep input order, so the LSD passes compose to a
// stable sort of the keys' low end_bit bits (what the callers' packed keys need).
#include <algorithm>

#include "internal.cuh"

namespace etb {
namespace {

constexpr int kT = 512;           // threads per tile / per sort CTA
constexpr int kIpt = 8;           // items per thread per scan tile
constexpr int kTile = kT * kIpt;  // 4096 items per scan tile
constexpr int kWarps = kT / 32;
constexpr int kRadix = 256;

// ---- block scan of one value per thread (exclusive, returns the block total) ----
template <class T, class Op>
__device__ __forceinline__ T block_excl_scan(T v, T identity, Op op, T* warp_tot, T& total) {
  const unsigned lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  T x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const T y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= static_cast<unsigned>(o)) x = op(y, x);
  }
  if (lane == 31) warp_tot[w] = x;
  __syncthreads();
  if (w == 0) {
    T t = lane < static_cast<unsigned>(kWarps) ? warp_tot[lane] : identity;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const T y = __shfl_up_sync(0xffffffffu, t, o);
      if (lane >= static_cast<unsigned>(o)) t = op(y, t);
    }
    if (lane < static_cast<unsigned>(kWarps)) warp_tot[lane] = t;  // inclusive over warps
  }
  __syncthreads();
  const T before = w ? warp_tot[w - 1] : identity;
  total = warp_tot[kWarps - 1];
  const T excl = __shfl_up_sync(0xffffffffu, x, 1);
  const T r = lane ? op(before, excl) : before;
  __syncthreads();  // warp_tot reusable
  return r;
}

struct SumOp {
  template <class T>
  __device__ __forceinline__ T operator()(T a, T b) const { return a + b; }
};
struct MaxOp {
  template <class T>
  __device__ __forceinline__ T operator()(T a, T b) const { return a > b ? a : b; }
};

// Phase 1: per-tile totals.
template <class In, class T, class Op>
__global__ void __launch_bounds__(kT) tile_reduce_kernel(const In* in, uint64_t count, T identity,
                                                         Op op, T* tile_tot) {
  __shared__ T warp_tot[kWarps];
  const uint64_t base = (uint64_t)blockIdx.x * kTile;
  T acc = identity;
#pragma unroll
  for (int k = 0; k < kIpt; ++k) {
    const uint64_t i = base + (uint64_t)k * kT + threadIdx.x;
    if (i < count) acc = op(acc, static_cast<T>(in[i]));
  }
  T total;
  block_excl_scan<T>(acc, identity, op, warp_tot, total);
  if (threadIdx.x == 0) tile_tot[blockIdx.x] = total;
}

// Phase 3: each tile scanned with its offset (offsets == nullptr: single tile).
template <class In, class T, class Op, bool kInclusive>
__global__ void __launch_bounds__(kT) tile_scan_kernel(const In* in, T* out, uint64_t count,
                                                       T identity, Op op, const T* offsets) {
  __shared__ T s[kTile];
  __shared__ T warp_tot[kWarps];
  const uint64_t base = (uint64_t)blockIdx.x * kTile;
#pragma unroll
  for (int k = 0; k < kIpt; ++k) {  // striped, coalesced
    const uint64_t i = base + (uint64_t)k * kT + threadIdx.x;
    s[k * kT + threadIdx.x] = i < count ? static_cast<T>(in[i]) : identity;
  }
  __syncthreads();
  T v[kIpt];
  T acc = identity;
#pragma unroll
  for (int k = 0; k < kIpt; ++k) {  // blocked: thread t owns items t*8 .. t*8+7
    v[k] = s[threadIdx.x * kIpt + k];
    acc = op(acc, v[k]);
  }
  T total;
  T run = block_excl_scan<T>(acc, identity, op, warp_tot, total);
  if (offsets) run = op(offsets[blockIdx.x], run);
#pragma unroll
  for (int k = 0; k < kIpt; ++k) {
    const T x = v[k];
    if (kInclusive) {
      run = op(run, x);
      s[threadIdx.x * kIpt + k] = run;
    } else {
      s[threadIdx.x * kIpt + k] = run;
      run = op(run, x);
    }
  }
  __syncthreads();
#pragma unroll
  for (int k = 0; k < kIpt; ++k) {
    const uint64_t i = base + (uint64_t)k * kT + threadIdx.x;
    if (i < count) out[i] = s[k * kT + threadIdx.x];
  }
}

// Exclusive (or inclusive) scan of count items into out (out may alias in).
template <class In, class T, class Op, bool kInclusive>
void scan_any(const In* in, T* out, uint64_t count, T identity, Op op, cudaStream_t s) {
  if (count == 0) return;
  const uint64_t tiles = (count + kTile - 1) / kTile;
  if (tiles == 1) {
    tile_scan_kernel<In, T, Op, kInclusive><<<1, kT, 0, s>>>(in, out, count, identity, op, nullptr);
    ETB_CUDA(cudaGetLastError());
    return;
  }
  DevBuf<T> tot(tiles);
  tile_reduce_kernel<In, T, Op><<<tiles, kT, 0, s>>>(in, count, identity, op, tot.get());
  ETB_CUDA(cudaGetLastError());
  scan_any<T, T, Op, false>(tot.get(), tot.get(), tiles, identity, op, s);  // tile offsets
  tile_scan_kernel<In, T, Op, kInclusive><<<tiles, kT, 0, s>>>(in, out, count, identity, op,
                                                               tot.get());
  ETB_CUDA(cudaGetLastError());
}

// ---- stable selection: keep item i where pred(i) ------------------------------
struct UniquePred {
  const uint64_t* in;
  __device__ __forceinline__ bool operator()(uint64_t i) const {
    return i == 0 || in[i] != in[i - 1];
  }
};
struct FlagPred {
  const uint8_t* flags;
  __device__ __forceinline__ bool operator()(uint64_t i) const { return flags[i] != 0; }
};

template <class Pred>
__global__ void __launch_bounds__(kT) select_count_kernel(Pred pred, uint64_t count,
                                                          uint64_t* tile_cnt) {
  __shared__ uint64_t warp_tot[kWarps];
  const uint64_t base = (uint64_t)blockIdx.x * kTile;
  uint64_t c = 0;
#pragma unroll
  for (int k = 0; k < kIpt; ++k) {
    const uint64_t i = base + (uint64_t)k * kT + threadIdx.x;
    c += i < count && pred(i);
  }
  uint64_t total;
  block_excl_scan<uint64_t>(c, 0ull, SumOp{}, warp_tot, total);
  if (threadIdx.x == 0) tile_cnt[blockIdx.x] = total;
}

// Items are taken in blocked order per thread (t*8 .. t*8+7), so the block scan
// of per-thread counts gives every kept item its output slot in input order.
template <class Pred, class V>
__global__ void __launch_bounds__(kT) select_write_kernel(Pred pred, const V* in, uint64_t count,
                                                          const uint64_t* tile_off, V* out,
                                                          uint64_t* n_out) {
  __shared__ uint64_t warp_tot[kWarps];
  const uint64_t base = (uint64_t)blockIdx.x * kTile + (uint64_t)threadIdx.x * kIpt;
  bool keep[kIpt];
  uint64_t c = 0;
#pragma unroll
  for (int k = 0; k < kIpt; ++k) {
    const uint64_t i = base + k;
    keep[k] = i < count && pred(i);
    c += keep[k];
  }
  uint64_t total;
  uint64_t pos = block_excl_scan<uint64_t>(c, 0ull, SumOp{}, warp_tot, total) + tile_off[blockIdx.x];
#pragma unroll
  for (int k = 0; k < kIpt; ++k)
    if (keep[k]) out[pos++] = in[base + k];
  if (n_out && blockIdx.x == gridDim.x - 1 && threadIdx.x == 0)
    *n_out = tile_off[blockIdx.x] + total;
}

template <class Pred, class V>
uint64_t select_any(Pred pred, const V* in, V* out, uint64_t count, cudaStream_t s) {
  if (count == 0) return 0;
  const uint64_t tiles = (count + kTile - 1) / kTile;
  DevBuf<uint64_t> off(tiles + 1);
  select_count_kernel<Pred><<<tiles, kT, 0, s>>>(pred, count, off.get());
  ETB_CUDA(cudaGetLastError());
  scan_any<uint64_t, uint64_t, SumOp, false>(off.get(), off.get(), tiles, 0ull, SumOp{}, s);
  select_write_kernel<Pred, V><<<tiles, kT, 0, s>>>(pred, in, count, off.get(), out,
                                                    off.get() + tiles);
  ETB_CUDA(cudaGetLastError());
  return read_u64(off.get() + tiles, s);
}

// ---- LSD radix sort --------------------------------------------------------
__device__ __forceinline__ uint32_t digit_of(uint64_t k, int shift, uint32_t mask) {
  return static_cast<uint32_t>(k >> shift) & mask;
}

// Upsweep: CTA b histograms keys [b*per, (b+1)*per) into cnt[d * nb + b].
__global__ void __launch_bounds__(kT) radix_upsweep_kernel(const uint64_t* keys, uint64_t count,
                                                           uint64_t per, int shift, uint32_t mask,
                                                           uint32_t* cnt) {
  __shared__ uint32_t h[kWarps / 4][kRadix];  // one histogram per 4 warps
  for (int i = threadIdx.x; i < (kWarps / 4) * kRadix; i += kT) (&h[0][0])[i] = 0;
  __syncthreads();
  const uint64_t lo = (uint64_t)blockIdx.x * per, hi = min(count, lo + per);
  uint32_t* my = h[(threadIdx.x >> 5) >> 2];
  for (uint64_t i = lo + threadIdx.x; i < hi; i += kT) atomicAdd(&my[digit_of(keys[i], shift, mask)], 1u);
  __syncthreads();
  for (int d = threadIdx.x; d < kRadix; d += kT) {
    uint32_t c = 0;
#pragma unroll
    for (int j = 0; j < kWarps / 4; ++j) c += h[j][d];
    cnt[(uint64_t)d * gridDim.x + blockIdx.x] = c;
  }
}

// Downsweep: CTA b re-reads its range in rounds of kT keys (round-major input
// order) and writes each key (and value) to off[d * nb + b] + the number of
// keys of digit d before it in the range. Per-warp digit counts are double
// buffered by round parity, so a round needs two barriers.
template <bool kPairs>
__global__ void __launch_bounds__(kT) radix_downsweep_kernel(
    const uint64_t* keys, uint64_t* keys_out, const uint32_t* vals, uint32_t* vals_out,
    uint64_t count, uint64_t per, int shift, uint32_t mask, const uint64_t* off) {
  __shared__ uint32_t wc[2][kWarps][kRadix];  // per-warp digit counts -> warp offsets
  __shared__ uint64_t rbase[kRadix];          // this round's first position of digit d
  const unsigned lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < 2 * kWarps * kRadix; i += kT) (&wc[0][0][0])[i] = 0;
  uint64_t run = 0;  // thread d < kRadix: next output position of digit d
  if (threadIdx.x < kRadix) run = off[(uint64_t)threadIdx.x * gridDim.x + blockIdx.x];
  __syncthreads();
  const uint64_t lo = (uint64_t)blockIdx.x * per, hi = min(count, lo + per);
  const unsigned lt = (1u << lane) - 1;
  unsigned par = 0;
  for (uint64_t r0 = lo; r0 < hi; r0 += kT, par ^= 1u) {
    const uint64_t i = r0 + threadIdx.x;
    const bool in = i < hi;
    const uint64_t k = in ? keys[i] : 0;
    uint32_t v = 0;
    if (kPairs && in) v = vals[i];
    const uint32_t d = in ? digit_of(k, shift, mask) : kRadix;  // kRadix: padding lane
    const unsigned peers = __match_any_sync(0xffffffffu, d);
    const unsigned rank = __popc(peers & lt);
    if (in && rank == 0) wc[par][w][d] = __popc(peers);
    __syncthreads();
    if (threadIdx.x < kRadix) {  // digit column: exclusive prefix over the warps
      const unsigned dd = threadIdx.x;
      uint32_t sum = 0;
#pragma unroll
      for (int j = 0; j < kWarps; ++j) {
        const uint32_t c = wc[par][j][dd];
        wc[par][j][dd] = sum;
        sum += c;
        wc[par ^ 1u][j][dd] = 0;  // the next round's counters
      }
      rbase[dd] = run;
      run += sum;
    }
    __syncthreads();
    if (in) {
      const uint64_t pos = rbase[d] + wc[par][w][d] + rank;
      keys_out[pos] = k;
      if (kPairs) vals_out[pos] = v;
    }
  }
}

// One LSD pass per 8-bit digit of [0, end_bit); ping-pongs between the buffers
// and leaves the result in `keys` (and `vals`).
template <bool kPairs>
void radix_sort(DevBuf<uint64_t>& keys, DevBuf<uint64_t>& kalt, DevBuf<uint32_t>* vals,
                DevBuf<uint32_t>* valt, uint64_t count, int end_bit, cudaStream_t s) {
  if (count < 2 || end_bit <= 0) return;
  if (kalt.size() < count) kalt.alloc(count);
  if (kPairs && valt->size() < count) valt->alloc(count);
  int dev = 0, sms = 0;
  ETB_CUDA(cudaGetDevice(&dev));
  ETB_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  // CTA ranges: whole rounds, at most 3 CTAs per SM (shared memory of the downsweep)
  const uint64_t rounds = (count + kT - 1) / kT;
  const uint64_t nb = std::max<uint64_t>(1, std::min<uint64_t>(rounds, 3ull * sms));
  const uint64_t per = ((rounds + nb - 1) / nb) * kT;
  const uint64_t nbu = (count + per - 1) / per;
  static thread_local DevBuf<uint32_t> cnt;
  static thread_local DevBuf<uint64_t> off;
  if (cnt.size() < kRadix * nbu) cnt.alloc(kRadix * nbu);
  if (off.size() < kRadix * nbu) off.alloc(kRadix * nbu);
  uint64_t* ka = keys.get();
  uint64_t* kb = kalt.get();
  uint32_t* va = kPairs ? vals->get() : nullptr;
  uint32_t* vb = kPairs ? valt->get() : nullptr;
  int passes = 0;
  for (int shift = 0; shift < end_bit; shift += 8, ++passes) {
    const int bits = std::min(8, end_bit - shift);
    const uint32_t mask = (1u << bits) - 1u;
    radix_upsweep_kernel<<<nbu, kT, 0, s>>>(ka, count, per, shift, mask, cnt.get());
    ETB_CUDA(cudaGetLastError());
    scan_any<uint32_t, uint64_t, SumOp, false>(cnt.get(), off.get(), kRadix * nbu, 0ull, SumOp{},
                                               s);
    radix_downsweep_kernel<kPairs><<<nbu, kT, 0, s>>>(ka, kb, va, vb, count, per, shift, mask,
                                                      off.get());
    ETB_CUDA(cudaGetLastError());
    std::swap(ka, kb);
    std::swap(va, vb);
  }
  if (passes & 1) {
    std::swap(keys, kalt);
    if (kPairs) std::swap(*vals, *valt);
  }
}

}  // namespace

void sort_keys_u64(DevBuf<uint64_t>& keys, DevBuf<uint64_t>& alt, uint64_t count, int end_bit,
                   cudaStream_t s) {
  radix_sort<false>(keys, alt, nullptr, nullptr, count, end_bit, s);
}

void sort_pairs_u64_u32(DevBuf<uint64_t>& keys, DevBuf<uint64_t>& kalt, DevBuf<uint32_t>& vals,
                        DevBuf<uint32_t>& valt, uint64_t count, int end_bit, cudaStream_t s) {
  radix_sort<true>(keys, kalt, &vals, &valt, count, end_bit, s);
}

uint64_t read_u64(const uint64_t* dev, cudaStream_t s) {
  uint64_t h = 0;
  ETB_CUDA(cudaMemcpyAsync(&h, dev, 8, cudaMemcpyDeviceToHost, s));
  ETB_CUDA(cudaStreamSynchronize(s));
  return h;
}

uint64_t unique_u64(const uint64_t* in, uint64_t* out, uint64_t count, cudaStream_t s) {
  return select_any(UniquePred{in}, in, out, count, s);
}

uint64_t select_flagged_u32(const uint32_t* in, const uint8_t* flags, uint32_t* out,
                            uint64_t count, cudaStream_t s) {
  return select_any(FlagPred{flags}, in, out, count, s);
}

void exclusive_scan_u64(const uint64_t* in, uint64_t* out, uint64_t count, cudaStream_t s) {
  scan_any<uint64_t, uint64_t, SumOp, false>(in, out, count, 0ull, SumOp{}, s);
}

void exclusive_scan_u32_to_u64(const uint32_t* in, uint64_t* out, uint64_t count, cudaStream_t s) {
  scan_any<uint32_t, uint64_t, SumOp, false>(in, out, count, 0ull, SumOp{}, s);
}

void inclusive_max_scan_u32(const uint32_t* in, uint32_t* out, uint64_t count, cudaStream_t s) {
  scan_any<uint32_t, uint32_t, MaxOp, true>(in, out, count, 0u, MaxOp{}, s);
}

uint64_t reduce_sum_u64(const uint64_t* in, uint64_t count, cudaStream_t s) {
  if (count == 0) return 0;
  // tile totals, then totals of totals until one remains
  const uint64_t tiles = (count + kTile - 1) / kTile;
  DevBuf<uint64_t> tot(tiles);
  tile_reduce_kernel<uint64_t, uint64_t, SumOp><<<tiles, kT, 0, s>>>(in, count, 0ull, SumOp{},
                                                                     tot.get());
  ETB_CUDA(cudaGetLastError());
  if (tiles == 1) return read_u64(tot.get(), s);
  return reduce_sum_u64(tot.get(), tiles, s);
}

}  // namespace etb
