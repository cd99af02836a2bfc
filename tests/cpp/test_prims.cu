// Checks the hand-written preprocessing primitives (csrc/prims.cu) against
// host std:: algorithms on seeded random inputs: radix sort of keys and of
// (key, value) pairs (stability: values are input positions), unique, flagged
// selection, exclusive / inclusive scans and the sum reduction. Prints one line
// per case and "prims ok" at the end; exits non-zero on the first mismatch.
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <numeric>
#include <random>
#include <vector>

#include "../../paper_2009_07463_b200/csrc/internal.cuh"

using namespace etb;

static int fails = 0;
#define CHECK(c, ...)                           \
  do {                                          \
    if (!(c)) {                                 \
      std::printf("FAIL: " __VA_ARGS__);        \
      std::printf("\n");                        \
      ++fails;                                  \
      return;                                   \
    }                                           \
  } while (0)

template <class T>
static void up(DevBuf<T>& d, const std::vector<T>& h) {
  d.alloc(std::max<size_t>(h.size(), 1));
  if (!h.empty()) ETB_CUDA(cudaMemcpy(d.get(), h.data(), h.size() * sizeof(T), cudaMemcpyHostToDevice));
}
template <class T>
static std::vector<T> down(const T* d, size_t n) {
  std::vector<T> h(n);
  if (n) ETB_CUDA(cudaMemcpy(h.data(), d, n * sizeof(T), cudaMemcpyDeviceToHost));
  return h;
}

static std::vector<uint64_t> keys_for(std::mt19937_64& rng, uint64_t n, int end_bit, bool dups) {
  std::vector<uint64_t> k(n);
  const uint64_t mask = end_bit >= 64 ? ~0ull : ((1ull << end_bit) - 1);
  const uint64_t narrow = dups ? std::max<uint64_t>(1, n / 8) : ~0ull;
  for (auto& x : k) {
    uint64_t r = rng() & mask;
    if (dups) r = (r % narrow) & mask;
    x = r;
  }
  return k;
}

static void case_sort(uint64_t n, int end_bit, bool dups, uint64_t seed) {
  std::mt19937_64 rng(seed);
  auto k = keys_for(rng, n, end_bit, dups);
  // keys only
  {
    DevBuf<uint64_t> dk, alt;
    up(dk, k);
    sort_keys_u64(dk, alt, n, end_bit, nullptr);
    ETB_CUDA(cudaDeviceSynchronize());
    auto got = down(dk.get(), n);
    auto want = k;
    std::sort(want.begin(), want.end());
    CHECK(got == want, "sort_keys n=%llu end_bit=%d", (unsigned long long)n, end_bit);
  }
  // pairs: value = input position; equal keys must keep input order
  {
    std::vector<uint32_t> v(n);
    std::iota(v.begin(), v.end(), 0u);
    DevBuf<uint64_t> dk, kalt;
    DevBuf<uint32_t> dv, valt;
    up(dk, k);
    up(dv, v);
    sort_pairs_u64_u32(dk, kalt, dv, valt, n, end_bit, nullptr);
    ETB_CUDA(cudaDeviceSynchronize());
    auto gk = down(dk.get(), n);
    auto gv = down(dv.get(), n);
    std::vector<uint32_t> wv(n);
    std::iota(wv.begin(), wv.end(), 0u);
    std::stable_sort(wv.begin(), wv.end(), [&](uint32_t a, uint32_t b) { return k[a] < k[b]; });
    std::vector<uint64_t> wk(n);
    for (uint64_t i = 0; i < n; ++i) wk[i] = k[wv[i]];
    CHECK(gk == wk && gv == wv, "sort_pairs n=%llu end_bit=%d", (unsigned long long)n, end_bit);
  }
  std::printf("sort n=%llu end_bit=%d dups=%d ok\n", (unsigned long long)n, end_bit, (int)dups);
}

static void case_select_scan(uint64_t n, uint64_t seed) {
  std::mt19937_64 rng(seed);
  auto k = keys_for(rng, n, 20, true);
  std::sort(k.begin(), k.end());
  {
    DevBuf<uint64_t> dk, out;
    up(dk, k);
    out.alloc(std::max<uint64_t>(n, 1));
    const uint64_t m = unique_u64(dk.get(), out.get(), n, nullptr);
    auto want = k;
    want.erase(std::unique(want.begin(), want.end()), want.end());
    CHECK(m == want.size() && down(out.get(), m) == want, "unique n=%llu", (unsigned long long)n);
  }
  {
    std::vector<uint32_t> v(n);
    std::vector<uint8_t> f(n);
    for (uint64_t i = 0; i < n; ++i) v[i] = static_cast<uint32_t>(rng()), f[i] = (rng() % 3) == 0;
    DevBuf<uint32_t> dv, out;
    DevBuf<uint8_t> df;
    up(dv, v);
    up(df, f);
    out.alloc(std::max<uint64_t>(n, 1));
    const uint64_t m = select_flagged_u32(dv.get(), df.get(), out.get(), n, nullptr);
    std::vector<uint32_t> want;
    for (uint64_t i = 0; i < n; ++i)
      if (f[i]) want.push_back(v[i]);
    CHECK(m == want.size() && down(out.get(), m) == want, "select_flagged n=%llu",
          (unsigned long long)n);
    // exclusive u32 -> u64 and inclusive max
    DevBuf<uint64_t> o64;
    o64.alloc(std::max<uint64_t>(n, 1));
    exclusive_scan_u32_to_u64(dv.get(), o64.get(), n, nullptr);
    std::vector<uint64_t> w64(n);
    uint64_t run = 0;
    for (uint64_t i = 0; i < n; ++i) w64[i] = run, run += v[i];
    CHECK(down(o64.get(), n) == w64, "exclusive_scan_u32_to_u64 n=%llu", (unsigned long long)n);
    DevBuf<uint32_t> omax;
    omax.alloc(std::max<uint64_t>(n, 1));
    inclusive_max_scan_u32(dv.get(), omax.get(), n, nullptr);
    std::vector<uint32_t> wm(n);
    uint32_t mx = 0;
    for (uint64_t i = 0; i < n; ++i) wm[i] = mx = std::max(mx, v[i]);
    CHECK(down(omax.get(), n) == wm, "inclusive_max_scan_u32 n=%llu", (unsigned long long)n);
  }
  {
    std::vector<uint64_t> a(n);
    for (auto& x : a) x = rng() >> 20;
    DevBuf<uint64_t> da, o;
    up(da, a);
    o.alloc(std::max<uint64_t>(n, 1));
    exclusive_scan_u64(da.get(), o.get(), n, nullptr);
    std::vector<uint64_t> w(n);
    uint64_t run = 0;
    for (uint64_t i = 0; i < n; ++i) w[i] = run, run += a[i];
    CHECK(down(o.get(), n) == w, "exclusive_scan_u64 n=%llu", (unsigned long long)n);
    // in place
    exclusive_scan_u64(da.get(), da.get(), n, nullptr);
    CHECK(down(da.get(), n) == w, "exclusive_scan_u64 in place n=%llu", (unsigned long long)n);
    up(da, a);
    CHECK(reduce_sum_u64(da.get(), n, nullptr) == run, "reduce_sum_u64 n=%llu",
          (unsigned long long)n);
  }
  std::printf("select/scan n=%llu ok\n", (unsigned long long)n);
}

int main() {
  const uint64_t sizes[] = {0, 1, 2, 3, 511, 512, 513, 4095, 4096, 4097, 100000, 1u << 20,
                            (1u << 22) + 12345};
  uint64_t seed = 1;
  for (uint64_t n : sizes) {
    for (int eb : {1, 7, 8, 9, 16, 23, 40, 64}) case_sort(n, eb, (seed & 1) != 0, seed++);
    case_select_scan(n, seed++);
  }
  case_sort(25u << 20, 52, true, seed++);    // several CTA ranges x 7 passes
  case_select_scan(17'000'001, seed++);     // three scan levels
  if (fails) {
    std::printf("%d failures\n", fails);
    return 1;
  }
  std::printf("prims ok\n");
  return 0;
}
