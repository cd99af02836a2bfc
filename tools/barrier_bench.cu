// Diagnostics: per-barrier cost of grid-barrier variants for the traversal's
// launch shape (one 1024-thread CTA per SM).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 tools/barrier_bench.cu -o tools/bb.bin
#include <cuda_runtime.h>
#include <cstdio>

__device__ __forceinline__ unsigned long long ld_acq(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ unsigned long long ld_rlx(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ unsigned long long atom_add_rel(unsigned long long* p, unsigned long long x) {
  unsigned long long v;
  asm volatile("atom.add.release.gpu.global.u64 %0, [%1], %2;" : "=l"(v) : "l"(p), "l"(x) : "memory");
  return v;
}
__device__ __forceinline__ void red_add_rel(unsigned long long* p, unsigned long long x) {
  asm volatile("red.release.gpu.global.add.u64 [%0], %1;" ::"l"(p), "l"(x) : "memory");
}

template <int V>
__global__ void __launch_bounds__(1024, 1) bar_k(unsigned long long* bar, int iters, int* work) {
  unsigned long long epoch = 0;
  const unsigned long long nb = gridDim.x;
  for (int it = 0; it < iters; ++it) {
    // a little memory traffic so fences have something to order
    if (work) work[(blockIdx.x * 1024 + threadIdx.x + it) & ((1 << 20) - 1)] += 1;
    __syncthreads();
    if (threadIdx.x == 0) {
      if (V == 0) {
        __threadfence();
        const unsigned long long old = atomicAdd(bar, 1ull);
        const unsigned long long target = (old / nb + 1) * nb;
        while (ld_acq(bar) < target) {
        }
        __threadfence();
      } else if (V == 1) {
        const unsigned long long old = atom_add_rel(bar, 1ull);
        const unsigned long long target = (old / nb + 1) * nb;
        while (ld_acq(bar) < target) {
        }
      } else if (V == 2) {
        red_add_rel(bar, 1ull);
        epoch += nb;
        while (ld_acq(bar) < epoch) {
        }
      } else if (V == 3) {  // relaxed polling, one acquire fence at the end
        red_add_rel(bar, 1ull);
        epoch += nb;
        while (ld_rlx(bar) < epoch) {
        }
        asm volatile("fence.acq_rel.gpu;" ::: "memory");
      }
    }
    __syncthreads();
  }
}

template <int V>
float run(unsigned long long* bar, int* work, int sms, int iters) {
  cudaMemset(bar, 0, 8);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  void* args[] = {&bar, &iters, &work};
  cudaLaunchCooperativeKernel((void*)bar_k<V>, dim3(sms), dim3(1024), args, 0, 0);
  cudaMemset(bar, 0, 8);
  cudaEventRecord(a);
  cudaLaunchCooperativeKernel((void*)bar_k<V>, dim3(sms), dim3(1024), args, 0, 0);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  return ms * 1e3f / iters;
}

int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  unsigned long long* bar;
  int* work;
  cudaMalloc(&bar, 8);
  cudaMalloc(&work, 4 << 20);
  cudaMemset(work, 0, 4 << 20);
  for (int w = 0; w < 2; ++w) {
    int* wk = w ? work : nullptr;
    printf("work=%d fence+atomicAdd+acq: %.3f us\n", w, run<0>(bar, wk, sms, 4000));
    printf("work=%d atom.release+acq:     %.3f us\n", w, run<1>(bar, wk, sms, 4000));
    printf("work=%d red.release+acq:      %.3f us\n", w, run<2>(bar, wk, sms, 4000));
    printf("work=%d red.release+rlx+fence:%.3f us\n", w, run<3>(bar, wk, sms, 4000));
  }
  printf("err=%s\n", cudaGetErrorString(cudaGetLastError()));
}
