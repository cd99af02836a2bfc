// Thin wrappers over CUB device primitives (radix sort / unique / scan /
// select). Used only by the untimed preprocessing; the BFS hot path is all
// hand-written kernels (bfs.cu).
#include <cub/cub.cuh>

#include "internal.cuh"

namespace etb {
namespace {

struct Temp {
  DevBuf<uint8_t> buf;
  void* get(size_t bytes) {
    if (buf.size() < bytes) buf.alloc(bytes + (bytes >> 3) + 256);
    return buf.get();
  }
};
thread_local Temp g_temp;

}  // namespace

void sort_keys_u64(DevBuf<uint64_t>& keys, DevBuf<uint64_t>& alt, uint64_t count, int end_bit,
                   cudaStream_t s) {
  if (count < 2) return;
  if (alt.size() < count) alt.alloc(count);
  cub::DoubleBuffer<uint64_t> db(keys.get(), alt.get());
  size_t bytes = 0;
  ETB_CUDA(cub::DeviceRadixSort::SortKeys(nullptr, bytes, db, (int64_t)count, 0, end_bit, s));
  ETB_CUDA(cub::DeviceRadixSort::SortKeys(g_temp.get(bytes), bytes, db, (int64_t)count, 0, end_bit,
                                          s));
  if (db.Current() != keys.get()) std::swap(keys, alt);
}

void sort_pairs_u64_u32(DevBuf<uint64_t>& keys, DevBuf<uint64_t>& kalt, DevBuf<uint32_t>& vals,
                        DevBuf<uint32_t>& valt, uint64_t count, int end_bit, cudaStream_t s) {
  if (count < 2) return;
  if (kalt.size() < count) kalt.alloc(count);
  if (valt.size() < count) valt.alloc(count);
  cub::DoubleBuffer<uint64_t> dk(keys.get(), kalt.get());
  cub::DoubleBuffer<uint32_t> dv(vals.get(), valt.get());
  size_t bytes = 0;
  ETB_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, bytes, dk, dv, (int64_t)count, 0, end_bit, s));
  ETB_CUDA(cub::DeviceRadixSort::SortPairs(g_temp.get(bytes), bytes, dk, dv, (int64_t)count, 0,
                                           end_bit, s));
  if (dk.Current() != keys.get()) std::swap(keys, kalt);
  if (dv.Current() != vals.get()) std::swap(vals, valt);
}

uint64_t read_u64(const uint64_t* dev, cudaStream_t s) {
  uint64_t h = 0;
  ETB_CUDA(cudaMemcpyAsync(&h, dev, 8, cudaMemcpyDeviceToHost, s));
  ETB_CUDA(cudaStreamSynchronize(s));
  return h;
}

uint64_t unique_u64(const uint64_t* in, uint64_t* out, uint64_t count, cudaStream_t s) {
  if (count == 0) return 0;
  DevBuf<uint64_t> n_sel(1);
  size_t bytes = 0;
  ETB_CUDA(cub::DeviceSelect::Unique(nullptr, bytes, in, out, n_sel.get(), (int64_t)count, s));
  ETB_CUDA(cub::DeviceSelect::Unique(g_temp.get(bytes), bytes, in, out, n_sel.get(),
                                     (int64_t)count, s));
  return read_u64(n_sel.get(), s);
}

void exclusive_scan_u64(const uint64_t* in, uint64_t* out, uint64_t count, cudaStream_t s) {
  if (count == 0) return;
  size_t bytes = 0;
  ETB_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, bytes, in, out, (int64_t)count, s));
  ETB_CUDA(cub::DeviceScan::ExclusiveSum(g_temp.get(bytes), bytes, in, out, (int64_t)count, s));
}

void exclusive_scan_u32_to_u64(const uint32_t* in, uint64_t* out, uint64_t count, cudaStream_t s) {
  if (count == 0) return;
  cub::TransformInputIterator<uint64_t, cub::CastOp<uint64_t>, const uint32_t*> it(
      in, cub::CastOp<uint64_t>());
  size_t bytes = 0;
  ETB_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, bytes, it, out, (int64_t)count, s));
  ETB_CUDA(cub::DeviceScan::ExclusiveSum(g_temp.get(bytes), bytes, it, out, (int64_t)count, s));
}

uint64_t select_flagged_u32(const uint32_t* in, const uint8_t* flags, uint32_t* out,
                            uint64_t count, cudaStream_t s) {
  if (count == 0) return 0;
  DevBuf<uint64_t> n_sel(1);
  size_t bytes = 0;
  ETB_CUDA(cub::DeviceSelect::Flagged(nullptr, bytes, in, flags, out, n_sel.get(), (int64_t)count,
                                      s));
  ETB_CUDA(cub::DeviceSelect::Flagged(g_temp.get(bytes), bytes, in, flags, out, n_sel.get(),
                                      (int64_t)count, s));
  return read_u64(n_sel.get(), s);
}

uint64_t reduce_sum_u64(const uint64_t* in, uint64_t count, cudaStream_t s) {
  if (count == 0) return 0;
  DevBuf<uint64_t> r(1);
  size_t bytes = 0;
  ETB_CUDA(cub::DeviceReduce::Sum(nullptr, bytes, in, r.get(), (int64_t)count, s));
  ETB_CUDA(cub::DeviceReduce::Sum(g_temp.get(bytes), bytes, in, r.get(), (int64_t)count, s));
  return read_u64(r.get(), s);
}

void inclusive_max_scan_u32(const uint32_t* in, uint32_t* out, uint64_t count, cudaStream_t s) {
  if (count == 0) return;
  size_t bytes = 0;
  ETB_CUDA(cub::DeviceScan::InclusiveScan(nullptr, bytes, in, out, cub::Max(), (int64_t)count, s));
  ETB_CUDA(cub::DeviceScan::InclusiveScan(g_temp.get(bytes), bytes, in, out, cub::Max(),
                                          (int64_t)count, s));
}

}  // namespace etb
