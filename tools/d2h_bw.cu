// Diagnostics: device -> pinned host bandwidth for a 16 MB result, one copy vs.
// split over 2 / 4 streams.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 tools/d2h_bw.cu -o tools/d2h.bin
#include <cuda_runtime.h>
#include <chrono>
#include <cstdio>

int main() {
  const size_t bytes = 16u << 20;
  void *d, *h;
  cudaMalloc(&d, bytes);
  cudaMallocHost(&h, bytes);
  cudaStream_t s[4];
  for (auto& x : s) cudaStreamCreateWithFlags(&x, cudaStreamNonBlocking);
  for (int parts : {1, 2, 4}) {
    double best = 1e9;
    for (int it = 0; it < 20; ++it) {
      auto t0 = std::chrono::steady_clock::now();
      const size_t chunk = bytes / parts;
      for (int p = 0; p < parts; ++p)
        cudaMemcpyAsync(static_cast<char*>(h) + p * chunk, static_cast<char*>(d) + p * chunk,
                        chunk, cudaMemcpyDeviceToHost, s[p]);
      for (int p = 0; p < parts; ++p) cudaStreamSynchronize(s[p]);
      const double us =
          std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - t0).count();
      if (us < best) best = us;
    }
    std::printf("parts=%d  %.1f us  %.1f GB/s\n", parts, best, bytes / best / 1e3);
  }
  return 0;
}
