// Diagnostics: device-wide rate of random 4-byte bitmap probes by where the
// bitmap lives — global memory (L2-resident, the traversal's probes today),
// the CTA's own shared memory, or distributed shared memory spread over a
// thread-block cluster of C CTAs (each CTA holds 1/C of the words; a probe
// reads the owner CTA's slice through ld.shared::cluster). Also prints how
// many clusters of each size fit at once (SMs a persistent kernel would keep).
// 1024 threads per CTA, one CTA per SM, K independent probes per thread.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 tools/dsmem_probe_bench.cu -o tools/dsmem_probe_bench.bin
#include <cooperative_groups.h>
#include <cuda_runtime.h>
#include <cstdio>

namespace cg = cooperative_groups;

constexpr int kThreads = 1024;
constexpr unsigned kSliceWords = 48 * 1024;  // 192 KB of bitmap per CTA

__device__ __forceinline__ unsigned hash(unsigned x) {
  x ^= x >> 16; x *= 0x7feb352du; x ^= x >> 15; x *= 0x846ca68bu; x ^= x >> 16;
  return x;
}

template <int K>
__global__ void __launch_bounds__(kThreads, 1) probe_global(const unsigned* bm, unsigned mask,
                                                             int iters, unsigned* sink) {
  const unsigned t = blockIdx.x * blockDim.x + threadIdx.x;
  unsigned acc = 0;
  for (int i = 0; i < iters; ++i) {
    unsigned v[K];
#pragma unroll
    for (int k = 0; k < K; ++k) v[k] = bm[hash(t * 7919u + i * 104729u + k) & mask];
#pragma unroll
    for (int k = 0; k < K; ++k) acc += v[k];
  }
  if (acc == 0x12345u) sink[0] = acc;
}

// kC == 1: the CTA's own shared memory; kC > 1: the cluster's.
template <int kC, int K>
__global__ void __launch_bounds__(kThreads, 1) probe_shared(int iters, unsigned* sink) {
  extern __shared__ unsigned slice[];
  for (unsigned i = threadIdx.x; i < kSliceWords; i += blockDim.x) slice[i] = hash(i + blockIdx.x);
  cg::cluster_group cl = cg::this_cluster();
  if constexpr (kC > 1) cl.sync();
  else __syncthreads();
  const unsigned t = blockIdx.x * blockDim.x + threadIdx.x;
  unsigned acc = 0;
  for (int i = 0; i < iters; ++i) {
    unsigned v[K];
#pragma unroll
    for (int k = 0; k < K; ++k) {
      const unsigned h = hash(t * 7919u + i * 104729u + k);
      const unsigned w = h % (kSliceWords * kC);
      if constexpr (kC > 1) v[k] = *cl.map_shared_rank(slice + w % kSliceWords, w / kSliceWords);
      else v[k] = slice[w];
    }
#pragma unroll
    for (int k = 0; k < K; ++k) acc += v[k];
  }
  if constexpr (kC > 1) cl.sync();  // slices stay alive until every reader is done
  if (acc == 0x12345u) sink[0] = acc;
}

template <class F>
float time_it(F launch) {
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  launch();
  cudaEventRecord(a);
  launch();
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms = 0;
  cudaEventElapsedTime(&ms, a, b);
  return ms;
}

template <int kC, int K>
void run_shared(int sms, unsigned* sink) {
  auto k = probe_shared<kC, K>;
  const int smem = kSliceWords * 4;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (kC > 8) cudaFuncSetAttribute(k, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  cudaLaunchConfig_t cfg = {};
  cudaLaunchAttribute at[1];
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = smem;
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = kC;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  int clusters = sms / kC;
  if (kC > 1) {
    cfg.gridDim = dim3(kC);
    if (cudaOccupancyMaxActiveClusters(&clusters, (void*)k, &cfg) != cudaSuccess || clusters < 1) {
      printf("smem C=%2d: cannot be resident (%s)\n", kC, cudaGetErrorString(cudaGetLastError()));
      return;
    }
  }
  cfg.gridDim = dim3(clusters * kC);
  const int iters = 256;
  const float ms = time_it([&] { cudaLaunchKernelEx(&cfg, k, iters, sink); });
  const cudaError_t e = cudaGetLastError();
  const double n = double(clusters) * kC * kThreads * iters * K;
  printf("%s C=%2d K=%d: %3d CTAs resident, bitmap %5.2f MB per cluster: %7.1f G probes/s "
         "(%.1f per SM-cycle at 1.965 GHz) %s\n",
         kC == 1 ? "smem " : "dsmem", kC, K, clusters * kC, kSliceWords * 4.0 * kC / 1e6,
         n / (ms * 1e-3) / 1e9, n / (ms * 1e-3) / (clusters * kC) / 1.965e9,
         e == cudaSuccess ? "" : cudaGetErrorString(e));
}

template <int K>
void run_global(int sms, const unsigned* bm, unsigned words, unsigned* sink) {
  const int iters = 256;
  const float ms = time_it([&] { probe_global<K><<<sms, kThreads>>>(bm, words - 1, iters, sink); });
  const double n = double(sms) * kThreads * iters * K;
  printf("global     K=%d: %3d CTAs, bitmap %5.2f MB (L2):    %7.1f G probes/s (%.1f per SM-cycle)\n", K,
         sms, words * 4.0 / 1e6, n / (ms * 1e-3) / 1e9, n / (ms * 1e-3) / sms / 1.965e9);
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  unsigned* sink;
  cudaMalloc(&sink, 4);
  const unsigned words = 1u << 20;  // 4 MB: the order of a scale-26 core bitmap (3 MB)
  unsigned* bm;
  cudaMalloc(&bm, words * 4);
  cudaMemset(bm, 0x5a, words * 4);
  run_global<4>(sms, bm, words, sink);
  run_global<8>(sms, bm, words, sink);
  run_global<4>(sms, bm, 1u << 14, sink);  // 64 KB: an L1-resident hub region
  run_shared<1, 4>(sms, sink);
  run_shared<1, 8>(sms, sink);
  run_shared<2, 4>(sms, sink);
  run_shared<2, 8>(sms, sink);
  run_shared<4, 8>(sms, sink);
  run_shared<8, 4>(sms, sink);
  run_shared<8, 8>(sms, sink);
  run_shared<16, 8>(sms, sink);
  return 0;
}
