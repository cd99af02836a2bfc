// Content hash for the drop-in's device caches (host only, internal): a cache
// keyed on storage addresses reuses a stale device copy when a new graph lands
// at freed addresses or an array is edited in place, so the caches key on the
// CONTENT of the caller's arrays instead.
#pragma once

#include <cstdint>
#include <cstring>
#include <vector>

namespace etbfs {
namespace detail {

// Content hash of a host array: 64-bit words folded through four independent
// multiply-rotate lanes (several GB/s; a cache key, not a checksum).
inline uint64_t hash_bytes(const void* data, size_t bytes, uint64_t seed) {
  const unsigned char* p = static_cast<const unsigned char*>(data);
  uint64_t h[4] = {seed ^ 0x9E3779B97F4A7C15ull, seed + 0xBF58476D1CE4E5B9ull,
                   ~seed, seed * 0x94D049BB133111EBull + 1};
  size_t i = 0;
  auto step = [](uint64_t a, uint64_t x) {
    a ^= x * 0x9E3779B97F4A7C15ull;
    a = (a << 31) | (a >> 33);
    return a * 0xBF58476D1CE4E5B9ull;
  };
  for (; i + 32 <= bytes; i += 32) {
    uint64_t w[4];
    std::memcpy(w, p + i, 32);
    for (int k = 0; k < 4; ++k) h[k] = step(h[k], w[k]);
  }
  uint64_t tail = bytes;
  for (; i < bytes; ++i) tail = step(tail, p[i]);
  uint64_t r = step(step(step(step(tail, h[0]), h[1]), h[2]), h[3]);
  r ^= r >> 29;
  return r;
}

template <typename T>
inline uint64_t hash_vec(const std::vector<T>& v, uint64_t seed) {
  return hash_bytes(v.data(), v.size() * sizeof(T), seed ^ v.size());
}


}  // namespace detail
}  // namespace etbfs
