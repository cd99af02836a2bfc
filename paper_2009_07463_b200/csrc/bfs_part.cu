// (5) Host side of the 1D core partition — partition bounds, per-partition
// buffers, the launch. The kernel (et_bfs_part_kernel) lives in bfs.cu next to
// the single-partition kernel whose step functions it runs; bfs_part.cuh has
// the scheme.
#include <algorithm>

#include "bfs_dev.cuh"
#include "bfs_part.cuh"

namespace etb {
namespace {

// seg[u] = {offset, length} of u's neighbours inside [lo, hi) (rows ascend).
__global__ void seg_kernel(const uint64_t* crow, const uint32_t* ccol, uint64_t nc, uint32_t lo,
                           uint32_t hi, uint2* seg) {
  for (uint64_t u = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; u < nc;
       u += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t rb = crow[u], re = crow[u + 1];
    uint64_t a = rb, b = re;
    while (a < b) {
      const uint64_t m = (a + b) >> 1;
      if (ccol[m] < lo) a = m + 1; else b = m;
    }
    uint64_t c = a, d = re;
    while (c < d) {
      const uint64_t m = (c + d) >> 1;
      if (ccol[m] < hi) c = m + 1; else d = m;
    }
    seg[u] = make_uint2(static_cast<uint32_t>(a - rb), static_cast<uint32_t>(c - a));
  }
}

}  // namespace

PartState::~PartState() {
  for (void* m : peer_maps)
    if (m) cudaIpcCloseMemHandle(m);
}

void part_bounds(const DevLayout& L, uint32_t nparts, std::vector<PartDev>& out) {
  if (nparts < 1 || nparts > kMaxParts)
    throw std::invalid_argument("etb_layout_partition: partitions must be in [1, 16]");
  out.assign(nparts, PartDev{});
  const uint64_t nc = L.nc, nt = L.nt;
  // Core: V_k = [k nc / G, (k+1) nc / G) rounded down to whole 32-vertex words.
  for (uint32_t k = 0; k < nparts; ++k) {
    const uint64_t lo = k == 0 ? 0 : ((k * nc / nparts) & ~uint64_t{31});
    const uint64_t hi = k + 1 == nparts ? nc : (((k + 1) * nc / nparts) & ~uint64_t{31});
    out[k].lo = static_cast<uint32_t>(lo);
    out[k].hi = static_cast<uint32_t>(std::max(lo, hi));
  }
  // Trees follow their anchor (trees are laid out in anchor order); component
  // trees and isolated vertices go to the last partition.
  const auto& anc = L.h_tanchor;
  uint64_t first_component = nt;
  for (uint64_t i = 0; i < nt; ++i)
    if (anc[i] == kNone32) {
      first_component = i;
      break;
    }
  for (uint32_t k = 0; k < nparts; ++k) {
    auto lb = [&](uint32_t bound) {
      return static_cast<uint64_t>(std::lower_bound(anc.begin(), anc.begin() + first_component,
                                                    bound) - anc.begin());
    };
    const uint64_t t0 = k == 0 ? 0 : lb(out[k].lo);
    const uint64_t t1 = k + 1 == nparts ? nt : lb(out[k + 1].lo);
    out[k].tlo = static_cast<uint32_t>(nc + t0);
    out[k].thi = static_cast<uint32_t>(nc + t1);
    out[k].zlo = out[k].zhi = static_cast<uint32_t>(L.n);
  }
  out[nparts - 1].zlo = static_cast<uint32_t>(nc + nt);
}

void part_build(const DevLayout& L, PartState& P, uint32_t nparts, uint32_t first, uint32_t local,
                cudaStream_t s) {
  P.nparts = nparts;
  P.first = first;
  P.local = local;
  part_bounds(L, nparts, P.h_parts);
  const uint64_t nc = L.nc;
  const uint64_t words = (nc + 31) / 32 + 1;
  P.seg.alloc(local * (nc ? nc : 1));
  P.visited.alloc(local * words);
  P.qv.alloc(local * (nc + 1));
  P.qp.alloc(local * (nc + 1));
  P.xbytes = ((3 * words * 4 + 255) / 256) * 256 + (kCtrWords + 32) * 8;
  P.xblock.alloc(local * P.xbytes);
  ETB_CUDA(cudaMemsetAsync(P.xblock.get(), 0, local * P.xbytes, s));
  P.bar.alloc(local);
  ETB_CUDA(cudaMemsetAsync(P.bar.get(), 0, local * 8, s));
  for (uint32_t j = 0; j < local; ++j) {
    PartDev& d = P.h_parts[first + j];
    unsigned char* xb = P.xblock.get() + j * P.xbytes;
    d.fb0 = reinterpret_cast<uint32_t*>(xb);
    d.fb1 = d.fb0 + words;
    d.fb2 = d.fb1 + words;
    d.ctr = reinterpret_cast<unsigned long long*>(xb + ((3 * words * 4 + 255) / 256) * 256);
    d.arrive = d.ctr + kCtrWords;
    d.bar = P.bar.get() + j;
    d.visited = P.visited.get() + j * words;
    d.qv = P.qv.get() + j * (nc + 1);
    d.qp = P.qp.get() + j * (nc + 1);
    uint2* sg = P.seg.get() + j * (nc ? nc : 1);
    d.seg = sg;
    if (nc) {
      seg_kernel<<<grid_for(nc, 256), 256, 0, s>>>(L.crow.get(), L.ccol.get(), nc, d.lo, d.hi, sg);
      ETB_LAUNCH_CHECK();
    }
  }
  P.d_parts.alloc(nparts);
  ETB_CUDA(cudaMemcpyAsync(P.d_parts.get(), P.h_parts.data(), nparts * sizeof(PartDev),
                           cudaMemcpyHostToDevice, s));
  int dev = 0, sms = 0, per_sm = 0;
  ETB_CUDA(cudaGetDevice(&dev));
  ETB_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  P.block = block_for(nc);
  const void* k = part_kernel_for(P.block);
  ETB_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                static_cast<int>(bfs_smem_bytes())));
  ETB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k, P.block, bfs_smem_bytes()));
  if (per_sm < 1) throw CudaError("et_bfs_part_kernel cannot be resident");
  int grid = sms;  // one CTA per SM, as the single-partition kernel
  grid -= grid % static_cast<int>(local);  // equal block groups
  P.grid = grid;
  ETB_CUDA(cudaStreamSynchronize(s));
}

void part_launch(const PartParams& p, const PartState& P, cudaStream_t s) {
  void* args[] = {const_cast<PartParams*>(&p)};
  ETB_CUDA(cudaLaunchCooperativeKernel(const_cast<void*>(part_kernel_for(P.block)), dim3(P.grid),
                                       dim3(P.block), args, bfs_smem_bytes(), s));
}

}  // namespace etb
