// (1) Graph construction on sm_100a.
//
// Kronecker generator: src/kronecker.cpp:23-69 — tuple i seeds SplitMix64
// with seed ^ i*0x2545f4914f6cdd1d and descends `scale` levels, picking a
// quadrant by u < a, u < a+b, u < a+b+c. The double compare u < x with
// u = (z>>11)*2^-53 is done exactly in integers as (z>>11) < ceil(x*2^53)
// (SURVEY.md Appendix C.1), thresholds computed on the host from the same
// doubles the reference uses (kronecker.cpp:40-41).
//
// CSR build: src/build.cpp:21-87 — symmetrise, drop self loops, sort+unique
// each row, count duplicates per direction then halve. Here every directed
// slot becomes one 64-bit key (src << b | dst); one radix sort + one unique
// produce all rows at once, canonical and identical to the reference.
#include <cmath>
#include <cstdlib>
#include <vector>

#include "internal.cuh"

namespace etb {
namespace {

struct KronDev {
  uint32_t scale;
  uint64_t seed;
  uint64_t ta, tab, tabc;  // ceil(x * 2^53) for x = a, a+b, a+b+c
};

uint64_t threshold(double x) {
  const double t = std::ceil(x * 9007199254740992.0);  // 2^53, exact scaling
  if (!(t > 0.0)) return 0;
  if (t >= 18446744073709551615.0) return ~uint64_t{0};
  return static_cast<uint64_t>(t);
}

KronDev to_dev(const etb_kron_params& p) {
  KronDev k;
  k.scale = p.scale;
  k.seed = p.seed;
  const double ab = p.a + p.b;
  const double abc = ab + p.c;
  k.ta = threshold(p.a);
  k.tab = threshold(ab);
  k.tabc = threshold(abc);
  return k;
}

__device__ __forceinline__ uint64_t splitmix64(uint64_t& state) {
  uint64_t z = (state += 0x9e3779b97f4a7c15ull);
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}

__device__ __forceinline__ void kron_tuple(const KronDev& k, uint64_t i, uint64_t& s,
                                           uint64_t& d) {
  uint64_t state = k.seed ^ (i * 0x2545f4914f6cdd1dull);
  s = 0;
  d = 0;
  for (uint32_t l = 0; l < k.scale; ++l) {
    const uint64_t u = splitmix64(state) >> 11;
    s = (s << 1) | (u >= k.tab);
    d = (d << 1) | ((u >= k.ta) & ((u < k.tab) | (u >= k.tabc)));
  }
}

__global__ void kron_tuples_kernel(KronDev k, uint64_t first, uint64_t count, uint32_t* src,
                                   uint32_t* dst) {
  for (uint64_t j = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; j < count;
       j += (uint64_t)gridDim.x * blockDim.x) {
    uint64_t s, d;
    kron_tuple(k, first + j, s, d);
    src[j] = static_cast<uint32_t>(s);
    dst[j] = static_cast<uint32_t>(d);
  }
}

__global__ void kron_pairs64_kernel(KronDev k, uint64_t first, uint64_t count, uint64_t* pairs) {
  for (uint64_t j = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; j < count;
       j += (uint64_t)gridDim.x * blockDim.x) {
    uint64_t s, d;
    kron_tuple(k, first + j, s, d);
    reinterpret_cast<ulonglong2*>(pairs)[j] = make_ulonglong2(s, d);
  }
}

__device__ __forceinline__ void count_loop(bool loop, unsigned long long* loops) {
  const unsigned m = __ballot_sync(__activemask(), loop);
  if (m && (threadIdx.x & 31) == __ffs(m) - 1) atomicAdd(loops, (unsigned long long)__popc(m));
}

// Two directed keys per tuple; self loops become two sentinel keys (src = n)
// that sort past every real key and are trimmed.
__device__ __forceinline__ void emit_keys(uint64_t s, uint64_t d, uint64_t j, int b, uint64_t n,
                                          uint64_t* keys, unsigned long long* loops) {
  const bool loop = (s == d);
  ulonglong2 kv;
  if (loop) {
    kv.x = kv.y = n << b;
  } else {
    kv.x = (s << b) | d;
    kv.y = (d << b) | s;
  }
  reinterpret_cast<ulonglong2*>(keys)[j] = kv;
  count_loop(loop, loops);
}

__global__ void kron_keys_kernel(KronDev k, uint64_t first, uint64_t count, int b, uint64_t n,
                                 uint64_t* keys, unsigned long long* loops) {
  for (uint64_t j = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; j < count;
       j += (uint64_t)gridDim.x * blockDim.x) {
    uint64_t s, d;
    kron_tuple(k, first + j, s, d);
    emit_keys(s, d, j, b, n, keys, loops);
  }
}

__global__ void tuples_keys_kernel(const uint32_t* src, const uint32_t* dst, uint64_t count, int b,
                                   uint64_t n, uint64_t* keys, unsigned long long* loops) {
  for (uint64_t j = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; j < count;
       j += (uint64_t)gridDim.x * blockDim.x)
    emit_keys(src[j], dst[j], j, b, n, keys, loops);
}

__global__ void pairs_keys_kernel(const uint64_t* pairs, uint64_t count, int b, uint64_t n,
                                  uint64_t* keys, unsigned long long* loops) {
  for (uint64_t j = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; j < count;
       j += (uint64_t)gridDim.x * blockDim.x) {
    const ulonglong2 p = reinterpret_cast<const ulonglong2*>(pairs)[j];
    emit_keys(p.x, p.y, j, b, n, keys, loops);
  }
}

// row[v] = first index whose key's source field is >= v (lower bound).
__global__ void row_offsets_kernel(const uint64_t* keys, uint64_t nkeys, int b, uint64_t n,
                                   uint64_t* row) {
  for (uint64_t v = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; v <= n;
       v += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t target = v << b;
    uint64_t lo = 0, hi = nkeys;
    while (lo < hi) {
      const uint64_t mid = (lo + hi) >> 1;
      if (keys[mid] < target) lo = mid + 1; else hi = mid;
    }
    row[v] = lo;
  }
}

__global__ void cols_kernel(const uint64_t* keys, uint64_t nkeys, uint64_t mask, uint32_t* col) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < nkeys;
       i += (uint64_t)gridDim.x * blockDim.x)
    col[i] = static_cast<uint32_t>(keys[i] & mask);
}

__global__ void degree_kernel(const uint64_t* row, uint64_t n, uint32_t* deg) {
  for (uint64_t v = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; v < n;
       v += (uint64_t)gridDim.x * blockDim.x)
    deg[v] = static_cast<uint32_t>(row[v + 1] - row[v]);
}

// Sorted keys (with 2*loops trailing sentinels) -> canonical CSR.
void finish_csr(DevBuf<uint64_t>& keys, uint64_t nkeys, uint64_t loops, uint64_t n, int b,
                DevGraph& out, uint64_t* dups, cudaStream_t s) {
  DevBuf<uint64_t> alt;
  sort_keys_u64(keys, alt, nkeys, 2 * b, s);
  const uint64_t valid = nkeys - 2 * loops;
  if (alt.size() < valid) alt.alloc(valid);
  const uint64_t uniq = unique_u64(keys.get(), alt.get(), valid, s);
  keys.release();
  if (dups) *dups = (valid - uniq) / 2;
  out.n = n;
  out.nnz = uniq;
  out.row.alloc(n + 1);
  out.col.alloc(uniq ? uniq : 1);
  out.deg.alloc(n ? n : 1);
  row_offsets_kernel<<<grid_for(n + 1, 256), 256, 0, s>>>(alt.get(), uniq, b, n, out.row.get());
  ETB_LAUNCH_CHECK();
  if (uniq) {
    cols_kernel<<<grid_for(uniq, 256), 256, 0, s>>>(alt.get(), uniq, (uint64_t{1} << b) - 1,
                                                     out.col.get());
    ETB_LAUNCH_CHECK();
  }
  if (n) {
    degree_kernel<<<grid_for(n, 256), 256, 0, s>>>(out.row.get(), n, out.deg.get());
    ETB_LAUNCH_CHECK();
  }
  ETB_CUDA(cudaStreamSynchronize(s));
}

// ---- bucketed build (large scales) --------------------------------------------
// The key array of a whole graph is 16 B per tuple; at scale 28 that is 69 GB,
// twice with the sort's double buffer. The generator is counter based, so the
// tuples are cheap to regenerate: one pass histograms the directed slots by
// source, then every bucket of source ids regenerates the tuples, keeps only its
// slots, sorts and dedups them and appends its rows to the CSR.
constexpr int kHistBins = 1024;

__global__ void kron_hist_kernel(KronDev k, uint64_t t, int shift, unsigned long long* hist,
                                 unsigned long long* loops) {
  __shared__ unsigned int sh[kHistBins];
  for (int i = threadIdx.x; i < kHistBins; i += blockDim.x) sh[i] = 0;
  __syncthreads();
  unsigned long long myloops = 0;
  for (uint64_t j = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; j < t;
       j += (uint64_t)gridDim.x * blockDim.x) {
    uint64_t s, d;
    kron_tuple(k, j, s, d);
    if (s == d) {
      ++myloops;
    } else {
      atomicAdd(&sh[s >> shift], 1u);
      atomicAdd(&sh[d >> shift], 1u);
    }
  }
  __syncthreads();
  for (int i = threadIdx.x; i < kHistBins; i += blockDim.x)
    if (sh[i]) atomicAdd(&hist[i], (unsigned long long)sh[i]);
  for (int o = 16; o; o >>= 1) myloops += __shfl_xor_sync(0xffffffffu, myloops, o);
  if ((threadIdx.x & 31) == 0 && myloops) atomicAdd(loops, myloops);
}

// Keys of the directed slots whose source lies in [lo, hi), appended with one
// atomic per CTA iteration (block-level scan).
__global__ void __launch_bounds__(1024) kron_bucket_kernel(KronDev k, uint64_t t, uint64_t lo,
                                                            uint64_t hi, int b, uint64_t* keys,
                                                            unsigned long long* cnt) {
  __shared__ unsigned int wsum[32];
  __shared__ unsigned long long base_sh;
  const unsigned lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  for (uint64_t base = blockIdx.x * (uint64_t)blockDim.x; base < t;
       base += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t j = base + threadIdx.x;
    uint64_t k0 = 0, k1 = 0;
    unsigned c = 0;
    if (j < t) {
      uint64_t s, d;
      kron_tuple(k, j, s, d);
      if (s != d) {
        if (s >= lo && s < hi) k0 = (s << b) | d, ++c;
        if (d >= lo && d < hi) (c ? k1 : k0) = (d << b) | s, ++c;
      }
    }
    unsigned incl = c;
    for (int o = 1; o < 32; o <<= 1) {
      const unsigned y = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += y;
    }
    if (lane == 31) wsum[wib] = incl;
    __syncthreads();
    if (wib == 0) {
      unsigned x = lane < (blockDim.x >> 5) ? wsum[lane] : 0u, xi = x;
      for (int o = 1; o < 32; o <<= 1) {
        const unsigned y = __shfl_up_sync(0xffffffffu, xi, o);
        if (lane >= o) xi += y;
      }
      wsum[lane] = xi - x;  // exclusive warp offsets
      if (lane == 31) base_sh = xi ? atomicAdd(cnt, (unsigned long long)xi) : 0ull;
    }
    __syncthreads();
    const uint64_t pos = base_sh + wsum[wib] + incl - c;
    if (c > 0) keys[pos] = k0;
    if (c > 1) keys[pos + 1] = k1;
    __syncthreads();
  }
}

// row[v] for v in [lo, hi] from a sorted unique bucket, offset by `base`.
__global__ void bucket_rows_kernel(const uint64_t* keys, uint64_t nkeys, int b, uint64_t lo,
                                   uint64_t hi, uint64_t base, uint64_t* row) {
  for (uint64_t v = lo + blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; v <= hi;
       v += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t target = v << b;
    uint64_t a = 0, e = nkeys;
    while (a < e) {
      const uint64_t m = (a + e) >> 1;
      if (keys[m] < target) a = m + 1; else e = m;
    }
    row[v] = base + a;
  }
}

void build_csr_bucketed(const etb_kron_params& p, uint64_t cap_keys, DevGraph& out,
                        uint64_t* self_loops, uint64_t* dups, cudaStream_t s) {
  const uint64_t n = uint64_t{1} << p.scale;
  const uint64_t t = n * p.edgefactor;
  const int b = bits_for(n);
  const int shift = p.scale > 10 ? static_cast<int>(p.scale) - 10 : 0;
  const KronDev k = to_dev(p);
  DevBuf<unsigned long long> hist(kHistBins + 2);
  ETB_CUDA(cudaMemsetAsync(hist.get(), 0, (kHistBins + 2) * 8, s));
  kron_hist_kernel<<<grid_for(t, 256), 256, 0, s>>>(k, t, shift, hist.get(), hist.get() + kHistBins);
  ETB_LAUNCH_CHECK();
  std::vector<unsigned long long> h(kHistBins + 1);
  ETB_CUDA(cudaMemcpyAsync(h.data(), hist.get(), (kHistBins + 1) * 8, cudaMemcpyDeviceToHost, s));
  ETB_CUDA(cudaStreamSynchronize(s));
  const uint64_t loops = h[kHistBins];
  if (self_loops) *self_loops = loops;
  const uint64_t slots = 2 * (t - loops);
  out.n = n;
  out.row.alloc(n + 1);
  out.col.alloc(slots ? slots : 1);
  out.deg.alloc(n ? n : 1);
  // buckets of whole histogram bins, each within cap_keys (a single bin may exceed it)
  std::vector<std::pair<uint64_t, uint64_t>> buckets;  // bin ranges
  uint64_t acc = 0, first = 0;
  const uint64_t nbins = std::min<uint64_t>(kHistBins, (n + (uint64_t{1} << shift) - 1) >> shift);
  for (uint64_t i = 0; i < nbins; ++i) {
    if (acc && acc + h[i] > cap_keys) {
      buckets.emplace_back(first, i);
      first = i;
      acc = 0;
    }
    acc += h[i];
  }
  buckets.emplace_back(first, nbins);
  uint64_t maxb = 0;
  for (auto& bk : buckets) {
    uint64_t c = 0;
    for (uint64_t i = bk.first; i < bk.second; ++i) c += h[i];
    maxb = std::max(maxb, c);
  }
  DevBuf<uint64_t> keys(maxb ? maxb : 1), alt(maxb ? maxb : 1);
  DevBuf<unsigned long long> cnt(1);
  uint64_t base = 0, dropped = 0;
  for (auto& bk : buckets) {
    const uint64_t lo = bk.first << shift, hi = std::min(n, bk.second << shift);
    ETB_CUDA(cudaMemsetAsync(cnt.get(), 0, 8, s));
    kron_bucket_kernel<<<grid_for(t, 1024, 148u * 8u), 1024, 0, s>>>(k, t, lo, hi, b, keys.get(),
                                                                    cnt.get());
    ETB_LAUNCH_CHECK();
    const uint64_t nk = read_u64(reinterpret_cast<uint64_t*>(cnt.get()), s);
    sort_keys_u64(keys, alt, nk, 2 * b, s);
    const uint64_t uniq = unique_u64(keys.get(), alt.get(), nk, s);
    dropped += nk - uniq;
    if (hi > lo) {
      bucket_rows_kernel<<<grid_for(hi - lo + 1, 256), 256, 0, s>>>(alt.get(), uniq, b, lo, hi, base,
                                                                    out.row.get());
      ETB_LAUNCH_CHECK();
    }
    if (uniq) {
      cols_kernel<<<grid_for(uniq, 256), 256, 0, s>>>(alt.get(), uniq, (uint64_t{1} << b) - 1,
                                                       out.col.get() + base);
      ETB_LAUNCH_CHECK();
    }
    base += uniq;
  }
  out.nnz = base;
  if (dups) *dups = dropped / 2;
  if (n) {
    degree_kernel<<<grid_for(n, 256), 256, 0, s>>>(out.row.get(), n, out.deg.get());
    ETB_LAUNCH_CHECK();
  }
  ETB_CUDA(cudaStreamSynchronize(s));
}

void check_n(uint64_t n) {
  if (n > kMaxDeviceVertices)
    throw std::invalid_argument("build_csr: vertex count exceeds the 32-bit device id range");
}

}  // namespace

void kron_validate(const etb_kron_params& p) {
  // kronecker.cpp:24-27, same messages.
  if (p.scale > 48) throw std::invalid_argument("generate_kronecker: scale > 48");
  if (p.edgefactor < 1) throw std::invalid_argument("generate_kronecker: edgefactor < 1");
  if (std::fabs(p.a + p.b + p.c + p.d - 1.0) > 1e-12)
    throw std::invalid_argument("generate_kronecker: probabilities must sum to 1");
  const uint64_t n = uint64_t{1} << p.scale;
  const uint64_t t = n * p.edgefactor;
  if (t / p.edgefactor != n) throw std::runtime_error("generate_kronecker: tuple count overflows");
}

void kron_generate_tuples(const etb_kron_params& p, uint64_t first, uint64_t count, uint32_t* src,
                          uint32_t* dst, cudaStream_t s) {
  if (!count) return;
  kron_tuples_kernel<<<grid_for(count, 256), 256, 0, s>>>(to_dev(p), first, count, src, dst);
  ETB_LAUNCH_CHECK();
}

void kron_generate_pairs64(const etb_kron_params& p, uint64_t first, uint64_t count,
                           uint64_t* pairs, cudaStream_t s) {
  if (!count) return;
  kron_pairs64_kernel<<<grid_for(count, 256), 256, 0, s>>>(to_dev(p), first, count, pairs);
  ETB_LAUNCH_CHECK();
}

void build_csr_from_generator(const etb_kron_params& p, DevGraph& out, uint64_t* self_loops,
                              uint64_t* dups, cudaStream_t s) {
  kron_validate(p);
  const uint64_t n = uint64_t{1} << p.scale;
  check_n(n);
  const uint64_t t = n * p.edgefactor;
  // Whole-graph key sort needs ~32 B per tuple (keys + sort buffer); bucket when
  // that does not fit comfortably (ETB_CSR_BUCKET_KEYS forces a bucket size).
  size_t free_b = 0, total_b = 0;
  ETB_CUDA(cudaMemGetInfo(&free_b, &total_b));
  uint64_t cap = 0;
  if (const char* e = std::getenv("ETB_CSR_BUCKET_KEYS")) cap = std::strtoull(e, nullptr, 10);
  if (!cap && 2 * t * 16 + 2 * t * 4 > static_cast<uint64_t>(free_b * 0.7))
    cap = static_cast<uint64_t>((free_b - 2 * t * 4) * 0.7) / 16;
  if (cap) {
    build_csr_bucketed(p, cap, out, self_loops, dups, s);
    return;
  }
  const int b = bits_for(n);
  DevBuf<uint64_t> keys(2 * t);
  DevBuf<unsigned long long> loops(1);
  ETB_CUDA(cudaMemsetAsync(loops.get(), 0, 8, s));
  kron_keys_kernel<<<grid_for(t, 256), 256, 0, s>>>(to_dev(p), 0, t, b, n, keys.get(),
                                                     loops.get());
  ETB_LAUNCH_CHECK();
  const uint64_t nl = read_u64(reinterpret_cast<uint64_t*>(loops.get()), s);
  if (self_loops) *self_loops = nl;
  finish_csr(keys, 2 * t, nl, n, b, out, dups, s);
}

void build_csr_from_device_tuples(uint64_t n, const uint32_t* src, const uint32_t* dst,
                                  uint64_t count, DevGraph& out, uint64_t* self_loops,
                                  uint64_t* dups, cudaStream_t s) {
  check_n(n);
  const int b = bits_for(n);
  DevBuf<uint64_t> keys(2 * count ? 2 * count : 1);
  DevBuf<unsigned long long> loops(1);
  ETB_CUDA(cudaMemsetAsync(loops.get(), 0, 8, s));
  if (count) {
    tuples_keys_kernel<<<grid_for(count, 256), 256, 0, s>>>(src, dst, count, b, n, keys.get(),
                                                             loops.get());
    ETB_LAUNCH_CHECK();
  }
  const uint64_t nl = read_u64(reinterpret_cast<uint64_t*>(loops.get()), s);
  if (self_loops) *self_loops = nl;
  finish_csr(keys, 2 * count, nl, n, b, out, dups, s);
}

void build_csr_from_host_pairs(uint64_t n, const uint64_t* pairs, uint64_t count, DevGraph& out,
                               uint64_t* self_loops, uint64_t* dups, cudaStream_t s) {
  check_n(n);
  const int b = bits_for(n);
  DevBuf<uint64_t> keys(2 * count ? 2 * count : 1);
  DevBuf<unsigned long long> loops(1);
  ETB_CUDA(cudaMemsetAsync(loops.get(), 0, 8, s));
  // Stage the host tuples through HBM in chunks; each chunk lands directly in
  // the key buffer's own slots (2 u64 per tuple) and is rewritten in place.
  const uint64_t chunk = uint64_t{1} << 26;
  for (uint64_t first = 0; first < count; first += chunk) {
    const uint64_t c = std::min(chunk, count - first);
    uint64_t* slot = keys.get() + 2 * first;
    ETB_CUDA(cudaMemcpyAsync(slot, pairs + 2 * first, c * 16, cudaMemcpyHostToDevice, s));
    pairs_keys_kernel<<<grid_for(c, 256), 256, 0, s>>>(slot, c, b, n, slot, loops.get());
    ETB_LAUNCH_CHECK();
  }
  const uint64_t nl = read_u64(reinterpret_cast<uint64_t*>(loops.get()), s);
  if (self_loops) *self_loops = nl;
  finish_csr(keys, 2 * count, nl, n, b, out, dups, s);
}

}  // namespace etb
