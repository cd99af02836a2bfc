// Diagnostics: event-timed cost of an empty cooperative launch (148 x 768,
// 33 KB smem) as a function of the kernel parameter size.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 tools/param_floor.cu -o tools/pf.bin
#include <cuda_runtime.h>
#include <algorithm>
#include <cstdio>
#include <vector>

template <int N>
struct P {
  unsigned long long v[N / 8];
};

template <int N>
__global__ void __launch_bounds__(768, 1) k(P<N> p) {
  extern __shared__ int sm[];
  if (p.v[0] == 12345 && threadIdx.x == 0) sm[0] = 1;
}

template <int N>
void run(cudaStream_t s, cudaEvent_t a, cudaEvent_t b, int coop) {
  P<N> p{};
  void* args[] = {&p};
  cudaFuncSetAttribute(k<N>, cudaFuncAttributeMaxDynamicSharedMemorySize, 48 * 1024);
  std::vector<float> t;
  for (int i = 0; i < 60; ++i) {
    cudaEventRecord(a, s);
    if (coop)
      cudaLaunchCooperativeKernel((void*)k<N>, dim3(148), dim3(768), args, 33 * 1024, s);
    else
      k<N><<<148, 768, 33 * 1024, s>>>(p);
    cudaEventRecord(b, s);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    if (i >= 10) t.push_back(ms * 1e3f);
  }
  std::sort(t.begin(), t.end());
  std::printf("coop=%d param=%5d B  median %.2f us  p10 %.2f\n", coop, N, t[t.size() / 2],
              t[t.size() / 10]);
}

int main() {
  cudaStream_t s;
  cudaStreamCreate(&s);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (int coop = 0; coop < 2; ++coop) {
    run<64>(s, a, b, coop);
    run<256>(s, a, b, coop);
    run<512>(s, a, b, coop);
    run<1024>(s, a, b, coop);
    run<2048>(s, a, b, coop);
    run<4000>(s, a, b, coop);
  }
  std::printf("err=%s\n", cudaGetErrorString(cudaGetLastError()));
}
