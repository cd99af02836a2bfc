// (5) 1D core partition of the ET-BFS across G partitions.
//
// Partition k owns the core ids [lo_k, hi_k) (Eq. 1 of the paper,
// V_k = [k n/G, (k+1) n/G), the rule of proj/src/preprocess.cpp:77, rounded
// to 32-vertex bitmap words) and the edge trees anchored there. The core CSR
// is replicated (s28's u32 core CSR is ~34 GB of a 180 GB B200); work is
// partitioned, so every claim is local:
//   * bottom-up: partition k sweeps only its owned vertices;
//   * top-down:  partition k expands every frontier row restricted to the
//                neighbours it owns (rows are sorted, so that is one
//                contiguous segment per row: seg[u] = {offset, length});
//   * after each level each partition writes its owned slice of the next
//     frontier bitmap into every peer's replica and adds its claim / scout
//     partials into every peer's counters (peer memory over NVLink, or plain
//     device memory when the partitions share one GPU), then a cross-partition
//     barrier; every partition then takes the same α/β decision.
// One kernel serves both deployments: G partitions in one cooperative launch on
// one GPU (block group g = partition g; this is also how the multi-GPU code is
// exercised on a single device), or one partition per GPU with peer pointers
// opened through CUDA IPC (one process per GPU).
#pragma once

#include "bfs.cuh"

namespace etb {

constexpr int kMaxParts = 16;
// u64 counters at the start of a partition's exchange block (bfs.cu: two
// parities of level slots, launch bookkeeping); the arrival counter follows.
constexpr uint64_t kCtrWords = 64;

// Device-visible descriptor of one partition. Pointers must be valid on the
// device running the kernel (own buffers, or IPC-mapped peer buffers; for a
// peer only the exchange block fb/ctr/arrive is used).
struct PartDev {
  uint32_t lo, hi;        // owned core ids, lo % 32 == 0
  uint32_t tlo, thi;      // owned edge-tree ids
  uint32_t zlo, zhi;      // owned isolated ids (last partition only)
  const uint2* seg;       // [nc] {offset in row, length} of neighbours in [lo, hi)
  uint32_t* visited;      // replica, owned words used
  uint32_t* fb0;          // frontier replicas (all words) — exchange block
  uint32_t* fb1;
  uint32_t* fb2;
  unsigned long long* ctr;     // kCtrWords level / launch counters — exchange block
  unsigned long long* arrive;  // cross-partition barrier counter — exchange block
  unsigned long long* bar;     // group barrier counter (local)
  uint32_t* qv;                // top-down frontier list (this partition's chunking)
  uint64_t* qp;
};

struct PartParams {
  BfsParams base;         // shared graph, result array `dp`, per-call fields, stats
  const PartDev* parts;   // [nparts]
  uint32_t nparts;
  uint32_t first_part;    // partitions run by this launch: [first, first + local)
  uint32_t local_parts;
  int system_scope;       // 1 when peers are other GPUs (fences at system scope)
};

// Host-side owner of the partition buffers on one device.
struct PartState {
  uint32_t nparts = 0, first = 0, local = 0;
  std::vector<PartDev> h_parts;     // descriptors as seen from this device
  DevBuf<PartDev> d_parts;
  DevBuf<uint2> seg;                // local partitions' segments, [local][nc]
  DevBuf<uint32_t> visited, qv;     // [local][words] / [local][nc]
  DevBuf<uint64_t> qp;
  DevBuf<unsigned char> xblock;     // exchange blocks, one per local partition
  uint64_t xbytes = 0;              // bytes per exchange block
  DevBuf<unsigned long long> bar;
  int grid = 0, block = 0;
  std::vector<void*> peer_maps;     // IPC-opened peer exchange blocks
  ~PartState();
};

// Partition boundaries (host): core ranges word aligned, trees by anchor.
void part_bounds(const DevLayout& L, uint32_t nparts, std::vector<PartDev>& out);
// Build `local` partitions [first, first + local) of `nparts` on this device.
void part_build(const DevLayout& L, PartState& P, uint32_t nparts, uint32_t first, uint32_t local,
                cudaStream_t s);
void part_launch(const PartParams& p, const PartState& P, cudaStream_t s);

// bfs.cu: the partitioned kernel for a block size, the shared-memory size of
// both kernels, and the block size for a core size.
const void* part_kernel_for(int block);
size_t bfs_smem_bytes();
int block_for(uint64_t nc);

}  // namespace etb
