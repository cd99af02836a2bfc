// (5) Host side of the 1D core partition — partition bounds, per-partition
// buffers, the launch. The kernel (et_bfs_part_kernel) lives in bfs.cu next to
// the single-partition kernel whose step functions it runs; bfs_part.cuh has
// the scheme.
#include <algorithm>

#include "bfs_dev.cuh"
#include "bfs_part.cuh"

namespace etb {
namespace {

// Top-down CSR of partition k: per core row, the neighbours it owns (rows stay
// sorted). count pass, then (after a scan) fill pass.
__global__ void owned_count_kernel(const uint64_t* crow, const uint32_t* ccol, uint64_t nc,
                                   uint32_t k, uint32_t G, uint32_t* cnt) {
  for (uint64_t u = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; u < nc;
       u += (uint64_t)gridDim.x * blockDim.x) {
    uint32_t c = 0;
    for (uint64_t e = crow[u]; e < crow[u + 1]; ++e) c += core_owner(ccol[e], G) == k;
    cnt[u] = c;
  }
}

__global__ void owned_fill_kernel(const uint64_t* crow, const uint32_t* ccol, uint64_t nc,
                                  uint32_t k, uint32_t G, const uint64_t* trow, uint32_t* tcol) {
  for (uint64_t u = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; u < nc;
       u += (uint64_t)gridDim.x * blockDim.x) {
    uint64_t o = trow[u];
    for (uint64_t e = crow[u]; e < crow[u + 1]; ++e)
      if (core_owner(ccol[e], G) == k) tcol[o++] = ccol[e];
  }
}

}  // namespace

PartState::~PartState() {
  for (void* m : peer_maps)
    if (m) cudaIpcCloseMemHandle(m);
}

void part_owners(const DevLayout& L, uint32_t nparts, uint32_t* owner) {
  if (nparts < 1 || nparts > kMaxParts)
    throw std::invalid_argument("etb_layout_partition: partitions must be in [1, 16]");
  const uint64_t nc = L.nc, nt = L.nt;
  for (uint64_t v = 0; v < nc; ++v) owner[v] = core_owner(static_cast<uint32_t>(v), nparts);
  for (uint64_t t = 0; t < nt; ++t) {
    const uint32_t a = L.h_tanchor[t];
    owner[nc + t] = a == kNone32 ? nparts - 1 : core_owner(a, nparts);
  }
  for (uint64_t v = nc + nt; v < L.n; ++v) owner[v] = nparts - 1;
}

void part_build(const DevLayout& L, PartState& P, uint32_t nparts, uint32_t first, uint32_t local,
                cudaStream_t s) {
  if (nparts < 1 || nparts > kMaxParts)
    throw std::invalid_argument("etb_layout_partition: partitions must be in [1, 16]");
  P.nparts = nparts;
  P.first = first;
  P.local = local;
  const uint64_t nc = L.nc, nt = L.nt;
  const uint32_t nw = static_cast<uint32_t>((nc + 31) / 32);
  const uint64_t words = nw + 1;
  P.h_parts.assign(nparts, PartDev{});
  std::vector<std::vector<uint32_t>> trees(nparts);
  for (uint64_t t = 0; t < nt; ++t) {
    const uint32_t a = L.h_tanchor[t];
    trees[a == kNone32 ? nparts - 1 : core_owner(a, nparts)].push_back(
        static_cast<uint32_t>(nc + t));
  }
  for (uint32_t k = 0; k < nparts; ++k) {
    PartDev& d = P.h_parts[k];
    d.part = k;
    d.nwo = owned_words(nw, k, nparts);
    d.nhub = owned_hub_words(nw, k, nparts);
    d.ntrees = static_cast<uint32_t>(trees[k].size());
    d.zlo = d.zhi = static_cast<uint32_t>(L.n);
  }
  P.h_parts[nparts - 1].zlo = static_cast<uint32_t>(nc + nt);
  P.qv.alloc(local * (nc + 1));
  P.qp.alloc(local * (nc + 1));
  // per local partition: fb0 | fb1 | fb2 | visited replica | counters — the
  // frontier replicas and counters are what peers write (the IPC export); the
  // whole state sits under the stream's persisting L2 window
  P.xbytes = ((4 * words * 4 + 255) / 256) * 256 + (kCtrWords + 32) * 8;
  P.xblock.alloc(local * P.xbytes);
  ETB_CUDA(cudaMemsetAsync(P.xblock.get(), 0, local * P.xbytes, s));
  P.bar.alloc(local);
  ETB_CUDA(cudaMemsetAsync(P.bar.get(), 0, local * 8, s));
  P.trow.resize(local);
  P.tcol.resize(local);
  P.trees.resize(local);
  DevBuf<uint32_t> cnt(nc ? nc : 1);
  for (uint32_t j = 0; j < local; ++j) {
    const uint32_t k = first + j;
    PartDev& d = P.h_parts[k];
    unsigned char* xb = P.xblock.get() + j * P.xbytes;
    d.fb0 = reinterpret_cast<uint32_t*>(xb);
    d.fb1 = d.fb0 + words;
    d.fb2 = d.fb1 + words;
    d.ctr = reinterpret_cast<unsigned long long*>(xb + ((4 * words * 4 + 255) / 256) * 256);
    d.arrive = d.ctr + kCtrWords;
    d.bar = P.bar.get() + j;
    d.visited = d.fb2 + words;
    d.qv = P.qv.get() + j * (nc + 1);
    d.qp = P.qp.get() + j * (nc + 1);
    // the top-down CSR of this partition's owned neighbours
    P.trow[j].alloc(nc + 1);
    uint64_t ne = 0;
    if (nc) {
      owned_count_kernel<<<grid_for(nc, 256), 256, 0, s>>>(L.crow.get(), L.ccol.get(), nc, k,
                                                           nparts, cnt.get());
      ETB_LAUNCH_CHECK();
      exclusive_scan_u32_to_u64(cnt.get(), P.trow[j].get(), nc, s);
      uint64_t last = 0;
      uint32_t lastc = 0;
      ETB_CUDA(cudaMemcpyAsync(&last, P.trow[j].get() + nc - 1, 8, cudaMemcpyDeviceToHost, s));
      ETB_CUDA(cudaMemcpyAsync(&lastc, cnt.get() + nc - 1, 4, cudaMemcpyDeviceToHost, s));
      ETB_CUDA(cudaStreamSynchronize(s));
      ne = last + lastc;
    }
    ETB_CUDA(cudaMemcpyAsync(P.trow[j].get() + nc, &ne, 8, cudaMemcpyHostToDevice, s));
    P.tcol[j].alloc(ne ? ne : 1);
    if (nc) {
      owned_fill_kernel<<<grid_for(nc, 256), 256, 0, s>>>(L.crow.get(), L.ccol.get(), nc, k,
                                                          nparts, P.trow[j].get(),
                                                          P.tcol[j].get());
      ETB_LAUNCH_CHECK();
    }
    d.trow = P.trow[j].get();
    d.tcol = P.tcol[j].get();
    P.trees[j].alloc(trees[k].empty() ? 1 : trees[k].size());
    if (!trees[k].empty())
      ETB_CUDA(cudaMemcpyAsync(P.trees[j].get(), trees[k].data(), trees[k].size() * 4,
                               cudaMemcpyHostToDevice, s));
    d.trees = P.trees[j].get();
    ETB_CUDA(cudaStreamSynchronize(s));  // the host vectors above
  }
  P.d_parts.alloc(nparts);
  ETB_CUDA(cudaMemcpyAsync(P.d_parts.get(), P.h_parts.data(), nparts * sizeof(PartDev),
                           cudaMemcpyHostToDevice, s));
  int dev = 0, sms = 0, per_sm = 0;
  ETB_CUDA(cudaGetDevice(&dev));
  ETB_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  P.block = block_for(nc);
  const void* kf = part_kernel_for(P.block);
  ETB_CUDA(cudaFuncSetAttribute(kf, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                static_cast<int>(bfs_smem_bytes())));
  ETB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kf, P.block, bfs_smem_bytes()));
  if (per_sm < 1) throw CudaError("et_bfs_part_kernel cannot be resident");
  int grid = sms;  // one CTA per SM, as the single-partition kernel
  grid -= grid % static_cast<int>(local);  // equal block groups
  P.grid = grid;
  set_l2_window(s, P.xblock.get(), local * P.xbytes);
  ETB_CUDA(cudaStreamSynchronize(s));
}

void part_launch(const PartParams& p, const PartState& P, cudaStream_t s) {
  void* args[] = {const_cast<PartParams*>(&p)};
  ETB_CUDA(cudaLaunchCooperativeKernel(const_cast<void*>(part_kernel_for(P.block)), dim3(P.grid),
                                       dim3(P.block), args, bfs_smem_bytes(), s));
}

}  // namespace etb
