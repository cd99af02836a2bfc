// Diagnostics: event-timed cost of an empty kernel launch for several grid /
// block / shared-memory / launch-mode shapes (the traversal's fixed floor).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 tools/launch_floor.cu -o /tmp/lf
#include <cuda_runtime.h>
#include <algorithm>
#include <cstdio>
#include <vector>

__global__ void empty_k(int* sink) {
  extern __shared__ int sm[];
  if (sink && threadIdx.x == 0) sm[0] = 1;
}

int main() {
  cudaStream_t s;
  cudaStreamCreate(&s);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaFuncSetAttribute(empty_k, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int blocks[] = {256, 512, 1024};
  const int mult[] = {1, 2, 4};
  const int smems[] = {0, 33 * 1024};
  for (int coop = 0; coop < 2; ++coop)
    for (int bs : blocks)
      for (int m : mult)
        for (int sm : smems) {
          if (bs * m > 2048) continue;
          std::vector<float> t;
          for (int i = 0; i < 40; ++i) {
            cudaEventRecord(a, s);
            int* sink = nullptr;
            void* args[] = {&sink};
            if (coop)
              cudaLaunchCooperativeKernel((void*)empty_k, dim3(sms * m), dim3(bs), args, sm, s);
            else
              empty_k<<<sms * m, bs, sm, s>>>(sink);
            cudaEventRecord(b, s);
            cudaEventSynchronize(b);
            float ms;
            cudaEventElapsedTime(&ms, a, b);
            if (i >= 8) t.push_back(ms * 1e3f);
          }
          std::sort(t.begin(), t.end());
          printf("coop=%d block=%4d grid=%3dx%d smem=%5d  median=%.2f us  min=%.2f\n", coop, bs, sms,
                 m, sm, t[t.size() / 2], t[0]);
        }
  // back-to-back: 20 launches between one pair of events
  for (int coop = 0; coop < 2; ++coop) {
    cudaEventRecord(a, s);
    for (int i = 0; i < 20; ++i) {
      int* sink = nullptr;
      void* args[] = {&sink};
      if (coop)
        cudaLaunchCooperativeKernel((void*)empty_k, dim3(sms), dim3(1024), args, 33 * 1024, s);
      else
        empty_k<<<sms, 1024, 33 * 1024, s>>>(sink);
    }
    cudaEventRecord(b, s);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    printf("back-to-back coop=%d: %.2f us per launch\n", coop, ms * 1e3f / 20);
  }
  // after a 2xL2 memset (the bench's flush), as in the per-root sequence
  void* flush = nullptr;
  const size_t fb = 256ull << 20;
  cudaMalloc(&flush, fb);
  for (int coop = 0; coop < 2; ++coop)
    for (int sm : {0, 48 * 1024, 100 * 1024}) {
      std::vector<float> t;
      for (int i = 0; i < 40; ++i) {
        cudaMemsetAsync(flush, i & 0xff, fb, s);
        cudaEventRecord(a, s);
        int* sink = nullptr;
        void* args[] = {&sink};
        if (coop)
          cudaLaunchCooperativeKernel((void*)empty_k, dim3(sms), dim3(768), args, sm, s);
        else
          empty_k<<<sms, 768, sm, s>>>(sink);
        cudaEventRecord(b, s);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        if (i >= 8) t.push_back(ms * 1e3f);
      }
      std::sort(t.begin(), t.end());
      printf("after memset coop=%d block=768 smem=%6d median=%.2f us min=%.2f\n", coop, sm,
             t[t.size() / 2], t[0]);
    }
  printf("err=%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
