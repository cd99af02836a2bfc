// Shared plumbing for the sm_100a ET-BFS kernels: error handling that maps to
// the reference's exception classes, RAII device buffers, small device helpers.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <stdexcept>
#include <string>
#include <utility>

namespace etb {

constexpr uint32_t kNone32 = 0xFFFFFFFFu;
// Device vertex ids are 32-bit and the CSR sort key packs (src << b | dst) with
// b = bits_for(n) into 64 bits, so n <= 2^31 (scale 31; BASELINE tops out at 28).
constexpr uint64_t kMaxDeviceVertices = uint64_t{1} << 31;

// Caller errors (reference: std::invalid_argument) and data errors
// (reference: std::runtime_error) keep the reference's C++ types so the C-ABI
// can map them to ETB_EINVAL / ETB_ERUNTIME; CUDA failures get their own type.
struct CudaError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

[[noreturn]] inline void cuda_fail(cudaError_t e, const char* what, const char* file, int line) {
  throw CudaError(std::string("CUDA error ") + cudaGetErrorString(e) + " in " + what + " at " +
                  file + ":" + std::to_string(line));
}

#define ETB_CUDA(call)                                                 \
  do {                                                                 \
    cudaError_t etb_e_ = (call);                                       \
    if (etb_e_ != cudaSuccess) ::etb::cuda_fail(etb_e_, #call, __FILE__, __LINE__); \
  } while (0)

#define ETB_LAUNCH_CHECK() ETB_CUDA(cudaGetLastError())

// Owning device allocation (cudaMalloc; no async pool so sizes are explicit).
template <typename T>
class DevBuf {
 public:
  DevBuf() = default;
  explicit DevBuf(size_t n) { alloc(n); }
  ~DevBuf() { release(); }
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  DevBuf(DevBuf&& o) noexcept : p_(o.p_), n_(o.n_) { o.p_ = nullptr, o.n_ = 0; }
  DevBuf& operator=(DevBuf&& o) noexcept {
    if (this != &o) {
      release();
      p_ = o.p_, n_ = o.n_;
      o.p_ = nullptr, o.n_ = 0;
    }
    return *this;
  }
  void alloc(size_t n) {
    release();
    n_ = n;
    if (n) ETB_CUDA(cudaMalloc(&p_, n * sizeof(T)));
  }
  void release() {
    if (p_) cudaFree(p_);
    p_ = nullptr;
    n_ = 0;
  }
  T* get() const { return p_; }
  size_t size() const { return n_; }
  size_t bytes() const { return n_ * sizeof(T); }
  explicit operator bool() const { return p_ != nullptr; }

 private:
  T* p_ = nullptr;
  size_t n_ = 0;
};

// Pinned host staging buffer.
template <typename T>
class HostBuf {
 public:
  HostBuf() = default;
  ~HostBuf() { release(); }
  HostBuf(const HostBuf&) = delete;
  HostBuf& operator=(const HostBuf&) = delete;
  void alloc(size_t n) {
    release();
    n_ = n;
    if (n) ETB_CUDA(cudaMallocHost(&p_, n * sizeof(T)));
  }
  void release() {
    if (p_) cudaFreeHost(p_);
    p_ = nullptr;
    n_ = 0;
  }
  T* get() const { return p_; }
  size_t size() const { return n_; }

 private:
  T* p_ = nullptr;
  size_t n_ = 0;
};

inline unsigned grid_for(uint64_t n, unsigned block, unsigned cap = 148u * 32u) {
  uint64_t g = (n + block - 1) / block;
  if (g < 1) g = 1;
  if (g > cap) g = cap;
  return static_cast<unsigned>(g);
}

// Bits needed so that every value in [0, n] fits (n itself is used as a sentinel).
inline int bits_for(uint64_t n) {
  int b = 1;
  while ((uint64_t{1} << b) <= n) ++b;
  return b;
}

struct Ctx;  // per-device stream + scratch (defined in capi.cu)

}  // namespace etb
