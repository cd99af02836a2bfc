// (5) 1D core partition of the ET-BFS across G partitions.
//
// Ownership. The core ids are degree sorted (relayout_csr), so equal vertex
// ranges (the paper's Eq. 1, proj/src/preprocess.cpp:77) would give partition 0
// the hubs — most top-down edges — and the last partition the low-degree
// vertices, most bottom-up misses. As the paper's static round-robin shuffle
// (SRRS, Alg. 4) does for its NUMA segments, ownership is distributed round
// robin over the degree order — the top 8K·G hubs one 32-vertex word at a
// time, the rest in 256-vertex blocks (8 bitmap words = one 32-byte sector, so the
// exchanged bitmap words stay whole sectors) — and the edge trees anchored in
// them; component trees and isolated vertices go to the last partition.
//
// Work. The core CSR is replicated (bottom-up scans whole rows); each partition
// also holds a top-down CSR of every core row restricted to its owned
// neighbours, so every claim is local:
//   * bottom-up: partition k sweeps its owned visited words against the
//     replicated frontier bitmap;
//   * top-down:  partition k expands every frontier row's owned neighbours;
//   * after each level each partition pushes its owned next-frontier words to
//     every peer's replica (the per-level bitmap allgather, fused in the kernel)
//     and adds its claim / scout partials into every peer's counters (peer
//     memory over NVLink, or device memory when the partitions share one GPU);
//     one barrier over all partitions; every partition then takes the same α/β
//     decision.
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
// Ownership granularity: the first kPartHubWordsPer·G bitmap words (the
// highest-degree core vertices: 16K at G = 2, 64K at G = 8) are dealt one word
// (32 vertices) at a time, the rest in blocks of kPartBlockWords words (256
// vertices, one 32-byte sector of bitmap): at s22 the top 256-vertex block
// alone holds 6% of the degree mass (G = 8: 1.33x the mean share) against 1.5%
// for the top word. Every partition then owns a multiple of 8 hub words, so
// an aligned run of 8 owned words is either 8 hub words G apart or one block.
constexpr uint32_t kPartHubWordsPer = 256;
constexpr uint32_t kPartBlockWords = 8;

__host__ __device__ __forceinline__ uint32_t hub_words(uint32_t G) { return kPartHubWordsPer * G; }

// Owner of core vertex v among G partitions.
__host__ __device__ __forceinline__ uint32_t core_owner(uint32_t v, uint32_t G) {
  const uint32_t w = v >> 5;
  return w < hub_words(G) ? w % G : ((w - hub_words(G)) / kPartBlockWords) % G;
}
// Hub words (the one-word-at-a-time region) owned by partition k of G.
__host__ __device__ __forceinline__ uint32_t owned_hub_words(uint32_t nwords, uint32_t k,
                                                             uint32_t G) {
  const uint32_t hn = nwords < hub_words(G) ? nwords : hub_words(G);
  return hn > k ? (hn - 1 - k) / G + 1 : 0;
}
// Bitmap words owned by partition k of G (nwords words in all).
__host__ __device__ __forceinline__ uint32_t owned_words(uint32_t nwords, uint32_t k, uint32_t G) {
  const uint32_t hub = owned_hub_words(nwords, k, G);
  if (nwords <= hub_words(G)) return hub;
  const uint32_t tn = nwords - hub_words(G);
  const uint32_t nb = (tn + kPartBlockWords - 1) / kPartBlockWords;
  if (k >= nb) return hub;
  const uint32_t blocks = (nb - 1 - k) / G + 1;  // k, k + G, ... < nb
  const uint32_t last = k + (blocks - 1) * G;    // possibly partial
  const uint32_t in_last = tn - last * kPartBlockWords;
  return hub + (blocks - 1) * kPartBlockWords + (in_last < kPartBlockWords ? in_last : kPartBlockWords);
}
// The j-th owned word of partition k of G, which owns nhub hub words.
__host__ __device__ __forceinline__ uint32_t owned_word(uint32_t j, uint32_t k, uint32_t G,
                                                       uint32_t nhub) {
  if (j < nhub) return j * G + k;
  j -= nhub;
  return hub_words(G) + ((j / kPartBlockWords) * G + k) * kPartBlockWords + j % kPartBlockWords;
}

// Device-visible descriptor of one partition. Pointers must be valid on the
// device running the kernel (own buffers, or IPC-mapped peer buffers; for a
// peer only the exchange block fb/ctr/arrive is used).
struct PartDev {
  uint32_t part;          // k
  uint32_t nwo;           // owned bitmap words
  uint32_t nhub;          // of which in the hub region
  const uint64_t* trow;   // [nc + 1] top-down CSR: each core row's owned neighbours
  const uint32_t* tcol;
  const uint32_t* trees;  // owned edge-tree vertex ids (relaid), ascending
  uint32_t ntrees;
  uint32_t zlo, zhi;      // owned isolated ids (last partition only)
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
  std::vector<DevBuf<uint64_t>> trow;  // local partitions' top-down CSRs
  std::vector<DevBuf<uint32_t>> tcol, trees;
  DevBuf<uint32_t> visited, qv;     // [local][words] / [local][nc]
  DevBuf<uint64_t> qp;
  DevBuf<unsigned char> xblock;     // exchange blocks, one per local partition
  uint64_t xbytes = 0;              // bytes per exchange block
  DevBuf<unsigned long long> bar;
  int grid = 0, block = 0;
  std::vector<void*> peer_maps;     // IPC-opened peer exchange blocks
  ~PartState();
};

// The owning partition of every relaid vertex (host; owner[n]).
void part_owners(const DevLayout& L, uint32_t nparts, uint32_t* owner);
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
