// Device helpers shared by the single- and multi-partition BFS kernels.
#pragma once

#include "bfs.cuh"

// Checked builds (-DETB_DEBUG_CHECKS, tools/build_variant.py): bounds and
// capacity asserts on the traversal's index arithmetic; the first violation's
// source line is recorded in etb_check_line (read by etb_debug_check_line) —
// compute-sanitizer is closed on this pool, so the checked library is run over
// the GPU parity suites instead.
#ifdef ETB_DEBUG_CHECKS
static __device__ unsigned int etb_check_line = 0;  // per translation unit
#define ETB_DCHECK(c)                                     \
  do {                                                    \
    if (!(c)) atomicCAS(&::etb_check_line, 0u, __LINE__); \
  } while (0)
#else
#define ETB_DCHECK(c) \
  do {                \
  } while (0)
#endif

namespace etb {
namespace dev {

__device__ __forceinline__ unsigned long long ld_acquire(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ unsigned long long ld_volatile(const unsigned long long* p) {
  return *reinterpret_cast<const volatile unsigned long long*>(p);
}

__device__ __forceinline__ unsigned long long atom_add_release(unsigned long long* p,
                                                              unsigned long long x) {
  unsigned long long v;
  asm volatile("atom.add.release.gpu.global.u64 %0, [%1], %2;" : "=l"(v) : "l"(p), "l"(x) : "memory");
  return v;
}

// Monotonic-counter grid barrier: every CTA adds 1; the barrier of a CTA that
// saw value `old` completes at the next multiple of gridDim.x. The CTA's writes
// are ordered by bar.sync + the release add (cumulative), the reads after it by
// the acquire poll + bar.sync: no full fences (tools/barrier_bench.cu measured
// 1.6 vs 2.0 us per barrier against __threadfence + atomicAdd).
__device__ __forceinline__ void grid_arrive_wait(unsigned long long* bar) {
  const unsigned long long nb = gridDim.x;
  const unsigned long long old = atom_add_release(bar, 1ull);
  const unsigned long long target = (old / nb + 1) * nb;
  const long long t0 = clock64();
  while (ld_acquire(bar) < target) {
    if (clock64() - t0 > 40000000000ll) __trap();  // ~20 s: never hang the GPU
  }
}

inline __device__ void grid_sync(unsigned long long* bar) {
  __syncthreads();
  if (threadIdx.x == 0) grid_arrive_wait(bar);
  __syncthreads();
}

// clock64 read that waits for x (diagnostics: phase boundaries after a load)
__device__ __forceinline__ long long clock_after(uint32_t x) {
  long long t;
  asm volatile("mov.u64 %0, %%clock64;" : "=l"(t) : "r"(x));
  return t;
}

__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// ---- bulk async copies (TMA engine, cp.async.bulk) into shared memory, with
// mbarrier transaction counts (sm_90+; SASS UBLKCP / SYNCS) -------------------
__device__ __forceinline__ uint32_t smem_addr(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* b, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(b)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_inval(uint64_t* b) {
  asm volatile("mbarrier.inval.shared::cta.b64 [%0];" ::"r"(smem_addr(b)) : "memory");
}
__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
// generic-proxy global writes (earlier levels, other SMs) before async-proxy reads
__device__ __forceinline__ void fence_proxy_async_global() {
  asm volatile("fence.proxy.async.global;" ::: "memory");
}
// generic-proxy shared-memory accesses before async-proxy writes (stage reuse)
__device__ __forceinline__ void fence_proxy_async_shared() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(b)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* b) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_addr(dst)),
      "l"(src), "r"(bytes), "r"(smem_addr(b))
      : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t phase) {
  asm volatile(
      "{\n .reg .pred p;\n WAIT_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra WAIT_%=;\n}" ::"r"(smem_addr(b)),
      "r"(phase)
      : "memory");
}

__device__ __forceinline__ unsigned long long warp_sum(unsigned long long v) {
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

__device__ __forceinline__ bool test_bit(const uint32_t* bm, uint32_t v) {
  return (bm[v >> 5] >> (v & 31)) & 1u;
}

__device__ __forceinline__ uint32_t warp_incl_scan(uint32_t x) {
  const unsigned lane = threadIdx.x & 31;
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  return x;
}

__device__ __forceinline__ unsigned long long warp_incl_scan64(unsigned long long x) {
  const unsigned lane = threadIdx.x & 31;
  for (int o = 1; o < 32; o <<= 1) {
    const unsigned long long y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  return x;
}

// Index of the last list entry whose chunk prefix is <= unit (32-ary search).
inline __device__ uint64_t find_vertex(const uint64_t* qp, uint64_t nq, uint64_t unit) {
  const unsigned lane = threadIdx.x & 31;
  uint64_t lo = 0, hi = nq;  // invariant: qp[lo] <= unit < qp[hi] (qp[nq] = +inf)
  while (hi - lo > 32) {
    const uint64_t stride = (hi - lo + 31) / 32;
    const uint64_t idx = lo + lane * stride;
    const bool le = idx < hi && qp[idx] <= unit;
    const unsigned m = __ballot_sync(0xffffffffu, le);
    const uint64_t j = 31 - __clz(m);
    const uint64_t nlo = lo + j * stride;
    hi = min(hi, nlo + stride);
    lo = nlo;
  }
  const uint64_t idx = lo + lane;
  const unsigned m = __ballot_sync(0xffffffffu, idx < hi && qp[idx] <= unit);
  return lo + (31 - __clz(m));
}

}  // namespace dev
}  // namespace etb
