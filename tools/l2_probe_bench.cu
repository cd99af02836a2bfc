// Diagnostics: the device-wide rate of random 4-byte probes (loads, ldcg loads,
// reductions, returning atomics) into an L2-resident bitmap, the operation
// that bounds the large top-down levels. One CTA of 1024 threads per SM, K
// independent probes in flight per thread.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 tools/l2_probe_bench.cu -o tools/l2_probe_bench.bin
#include <cuda_runtime.h>
#include <cstdio>

__device__ __forceinline__ unsigned hash(unsigned x) {
  x ^= x >> 16; x *= 0x7feb352du; x ^= x >> 15; x *= 0x846ca68bu; x ^= x >> 16;
  return x;
}

// kSkew: half of the probes go to the first 1024 words (the hub words of a
// degree-sorted layout); kSkew == 2 also transposes words within 1024-word
// blocks (w -> (w & 31) << 5 | (w >> 5) & 31), spreading them over 32 lines.
template <int kOp, int K, int kSkew = 0>
__global__ void __launch_bounds__(1024, 1) probe(unsigned* bm, unsigned mask, int iters,
                                                 unsigned* sink) {
  const unsigned t = blockIdx.x * blockDim.x + threadIdx.x;
  unsigned acc = 0;
  for (int i = 0; i < iters; ++i) {
    unsigned idx[K];
#pragma unroll
    for (int k = 0; k < K; ++k) {
      const unsigned h = hash(t * 7919u + (unsigned)i * 104729u + k);
      idx[k] = kSkew && (h & 1u) ? (h >> 1) & 1023u : h & mask;
      if (kSkew == 2) idx[k] = (idx[k] & ~1023u) | ((idx[k] & 31u) << 5) | ((idx[k] >> 5) & 31u);
    }
    unsigned v[K];
#pragma unroll
    for (int k = 0; k < K; ++k) {
      if (kOp == 0) v[k] = bm[idx[k]];
      else if (kOp == 1) v[k] = __ldcg(&bm[idx[k]]);
      else if (kOp == 2) { atomicOr(&bm[idx[k]], 1u << (k & 31)); v[k] = 0; }
      else v[k] = atomicOr(&bm[idx[k]], 1u << (k & 31));
    }
#pragma unroll
    for (int k = 0; k < K; ++k) acc += v[k];
  }
  if (acc == 0x12345u) sink[0] = acc;
}

template <int kOp, int K, int kSkew = 0>
void run(const char* name, unsigned* bm, unsigned words, unsigned* sink, int sms) {
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const int iters = 64;
  probe<kOp, K, kSkew><<<sms, 1024>>>(bm, words - 1, iters, sink);
  cudaEventRecord(a);
  probe<kOp, K, kSkew><<<sms, 1024>>>(bm, words - 1, iters, sink);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  const double n = double(sms) * 1024 * iters * K;
  printf("%-8s skew=%d K=%d bitmap %6.1f MB: %7.1f G probes/s (%.1f us)\n", name, kSkew, K, words * 4.0 / 1e6,
         n / (ms * 1e-3) / 1e9, ms * 1e3);
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  unsigned* bm = nullptr;
  unsigned* sink = nullptr;
  cudaMalloc(&bm, 64u << 20);
  cudaMalloc(&sink, 4);
  cudaMemset(bm, 0, 64u << 20);
  for (int sk = 1; sk <= 2; ++sk) {
    const unsigned words = 1u << 20;
    if (sk == 1) {
      run<0, 8, 1>("ld", bm, words, sink, sms);
      run<3, 8, 1>("atom.or", bm, words, sink, sms);
      run<2, 8, 1>("red.or", bm, words, sink, sms);
    } else {
      run<0, 8, 2>("ld", bm, words, sink, sms);
      run<3, 8, 2>("atom.or", bm, words, sink, sms);
      run<2, 8, 2>("red.or", bm, words, sink, sms);
    }
  }
  for (unsigned words : {1u << 18, 1u << 20, 1u << 24}) {  // 1 MB, 4 MB, 64 MB
    run<0, 4>("ld", bm, words, sink, sms);
    run<0, 8>("ld", bm, words, sink, sms);
    run<1, 8>("ldcg", bm, words, sink, sms);
    run<2, 8>("red.or", bm, words, sink, sms);
    run<3, 8>("atom.or", bm, words, sink, sms);
  }
  printf("err=%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
