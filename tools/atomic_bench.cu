// Diagnostics: cost of one returning 64-bit atomicAdd per warp on ONE address
// vs spread over S addresses (the list-append counters of the BFS levels).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 tools/atomic_bench.cu -o tools/ab.bin
#include <cuda_runtime.h>
#include <cstdio>

__global__ void __launch_bounds__(1024, 1) k(unsigned long long* ctr, int spread, int reps,
                                             unsigned long long* sink) {
  const unsigned lane = threadIdx.x & 31;
  const unsigned gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  unsigned long long acc = 0;
  for (int r = 0; r < reps; ++r) {
    if (lane == 0 && spread > 0) acc += atomicAdd(&ctr[(gw % spread) * 16], 1ull + acc);
    acc = __shfl_sync(0xffffffffu, acc, 0);
  }
  if (acc == 12345) *sink = acc;
}

int main() {
  unsigned long long *ctr, *sink;
  cudaMalloc(&ctr, 1 << 20);
  cudaMalloc(&sink, 8);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const int spreads[] = {0, 1, 2, 4, 8, 16, 148};
  for (int reps : {1, 4}) {
    for (int sp : spreads) {
      float best = 1e9;
      for (int it = 0; it < 10; ++it) {
        cudaMemset(ctr, 0, 1 << 20);
        cudaEventRecord(a);
        k<<<148, 1024>>>(ctr, sp, reps, sink);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        if (ms < best) best = ms;
      }
      printf("reps=%d spread=%3d (4736 warps): %.2f us\n", reps, sp, best * 1e3f);
    }
  }
  printf("err=%s\n", cudaGetErrorString(cudaGetLastError()));
}
