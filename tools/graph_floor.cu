// Diagnostics: event-timed cost of an empty 148 x 768 (33 KB smem) kernel,
// direct cooperative launch vs. a one-node CUDA graph (kernel node set to
// cooperative) whose parameters are updated before every launch.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 tools/graph_floor.cu -o tools/gf.bin
#include <cuda_runtime.h>
#include <algorithm>
#include <cstdio>
#include <vector>

struct P {
  unsigned long long v[48];
};

__global__ void __launch_bounds__(768, 1) k(P p) {
  extern __shared__ int sm[];
  if (p.v[0] == 12345 && threadIdx.x == 0) sm[0] = 1;
}

int main() {
  cudaStream_t s;
  cudaStreamCreate(&s);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  P p{};
  void* args[] = {&p};
  std::vector<float> t;
  for (int i = 0; i < 80; ++i) {
    cudaEventRecord(a, s);
    cudaLaunchCooperativeKernel((void*)k, dim3(148), dim3(768), args, 33 * 1024, s);
    cudaEventRecord(b, s);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    if (i >= 10) t.push_back(ms * 1e3f);
  }
  std::sort(t.begin(), t.end());
  std::printf("direct coop: median %.2f us p10 %.2f\n", t[t.size() / 2], t[t.size() / 10]);

  cudaGraph_t g;
  cudaGraphCreate(&g, 0);
  cudaKernelNodeParams kp{};
  kp.func = (void*)k;
  kp.gridDim = dim3(148);
  kp.blockDim = dim3(768);
  kp.sharedMemBytes = 33 * 1024;
  kp.kernelParams = args;
  cudaGraphNode_t n;
  cudaGraphAddKernelNode(&n, g, nullptr, 0, &kp);
  cudaLaunchAttributeValue v{};
  v.cooperative = 1;
  cudaGraphKernelNodeSetAttribute(n, cudaLaunchAttributeCooperative, &v);
  cudaGraphExec_t ge;
  cudaGraphInstantiate(&ge, g, 0);
  t.clear();
  for (int i = 0; i < 80; ++i) {
    p.v[0] = i;
    cudaGraphExecKernelNodeSetParams(ge, n, &kp);
    cudaEventRecord(a, s);
    cudaGraphLaunch(ge, s);
    cudaEventRecord(b, s);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    if (i >= 10) t.push_back(ms * 1e3f);
  }
  std::sort(t.begin(), t.end());
  std::printf("graph coop:  median %.2f us p10 %.2f\n", t[t.size() / 2], t[t.size() / 10]);
  std::printf("err=%s\n", cudaGetErrorString(cudaGetLastError()));
}
