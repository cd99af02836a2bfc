// (2a) Vertex classification on sm_100a — classify_vertices / compute_peak_height
// (src/classify.cpp:10-66, Alg. 8).
//
// mh == 0  : purely local — VZ/TL by degree, CE = CI that lost a TL neighbour.
// mh == -1 : the reference's Gauss-Seidel fixpoint equals "not in the 2-core"
//            (order independent), so a frontier k-core
//            peel reproduces it with linear work.
// mh >= 1 and the peak height are index-order dependent. Each Gauss-Seidel
//            round is emulated exactly: within round h, v is peeled iff it is
//            CI and (num_pre[v] == 0 || num_pre[v] - #{u < v peeled in round h}
//            == 1). That is a recursion over lower indices only (a DAG), solved
//            by in-place relaxation sweeps until no flag changes; the unique
//            fixed point is the sequential sweep's result.
#include "internal.cuh"

namespace etb {
namespace {

constexpr uint8_t CI = ETB_CI, CE = ETB_CE, TI = ETB_TI, TL = ETB_TL, VZ = ETB_VZ;

__global__ void leaf_pass_kernel(const uint32_t* deg, uint64_t n, uint8_t* type, uint32_t* live,
                                 uint32_t* queue, unsigned long long* qlen) {
  for (uint64_t v = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; v < n;
       v += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t d = deg[v];
    live[v] = d;
    const uint8_t t = d == 0 ? VZ : (d == 1 ? TL : CI);
    type[v] = t;
    if (t == TL && queue) {
      const unsigned long long pos = atomicAdd(qlen, 1ull);
      queue[pos] = static_cast<uint32_t>(v);
    }
  }
}

// One peel round: every queued vertex decrements its neighbours' live counts;
// a CI vertex whose count falls 2 -> 1 (a unique transition) leaves the 2-core.
__global__ void peel_round_kernel(const uint64_t* row, const uint32_t* col, const uint32_t* q,
                                  uint64_t qn, uint8_t* type, uint32_t* live, uint32_t* nq,
                                  unsigned long long* nqlen) {
  const unsigned lane = threadIdx.x & 31;
  const uint64_t warp = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
  const uint64_t nwarps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  for (uint64_t i = warp; i < qn; i += nwarps) {
    const uint32_t v = q[i];
    for (uint64_t k = row[v] + lane; k < row[v + 1]; k += 32) {
      const uint32_t w = col[k];
      const uint32_t old = atomicSub(&live[w], 1u);
      if (old == 2 && type[w] == CI) {
        type[w] = TI;
        const unsigned long long pos = atomicAdd(nqlen, 1ull);
        nq[pos] = w;
      }
    }
  }
}

__global__ void leaf_decrement_kernel(const uint64_t* row, const uint32_t* col, const uint8_t* type,
                                      uint64_t n, uint32_t* live) {
  for (uint64_t v = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; v < n;
       v += (uint64_t)gridDim.x * blockDim.x)
    if (type[v] == TL) atomicSub(&live[col[row[v]]], 1u);
}

__global__ void core_edge_kernel(const uint32_t* deg, const uint32_t* live, uint64_t n,
                                 uint8_t* type, unsigned long long* counts) {
  __shared__ unsigned long long sc[5];
  if (threadIdx.x < 5) sc[threadIdx.x] = 0;
  __syncthreads();
  for (uint64_t v = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; v < n;
       v += (uint64_t)gridDim.x * blockDim.x) {
    uint8_t t = type[v];
    if (t == CI && live[v] != deg[v]) {
      t = CE;
      type[v] = CE;
    }
    atomicAdd(&sc[t], 1ull);
  }
  __syncthreads();
  if (threadIdx.x < 5 && sc[threadIdx.x]) atomicAdd(&counts[threadIdx.x], sc[threadIdx.x]);
}

// ---- exact Gauss-Seidel rounds (mh >= 1, peak height) -------------------------
// cand: CI vertex that could be peeled this round (num_pre == 0, or num_pre - 1
// <= number of lower CI neighbours). x: current guess of "peeled this round".
__global__ void gs_candidates_kernel(const uint64_t* row, const uint32_t* col, const uint8_t* type,
                                     const uint32_t* pre, uint64_t n, uint8_t* cand, uint8_t* x,
                                     unsigned long long* ncand) {
  for (uint64_t v = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; v < n;
       v += (uint64_t)gridDim.x * blockDim.x) {
    uint8_t c = 0, xv = 0;
    if (type[v] == CI) {
      const uint32_t p = pre[v];
      if (p <= 1) {
        c = 1;
      } else {
        uint32_t low = 0;
        for (uint64_t k = row[v]; k < row[v + 1] && low + 1 < p; ++k) {
          const uint32_t u = col[k];
          if (u >= v) break;  // rows ascend
          low += type[u] == CI;
        }
        c = (low + 1 >= p);
      }
      xv = c && p <= 1;
    }
    cand[v] = c;
    x[v] = xv;
    if (c) atomicAdd(ncand, 1ull);
  }
}

__global__ void gs_sweep_kernel(const uint64_t* row, const uint32_t* col, const uint32_t* pre,
                                const uint8_t* cand, uint64_t n, uint8_t* x, int* changed) {
  for (uint64_t v = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; v < n;
       v += (uint64_t)gridDim.x * blockDim.x) {
    if (!cand[v]) continue;
    const uint32_t p = pre[v];
    uint32_t cnt = 0;
    for (uint64_t k = row[v]; k < row[v + 1]; ++k) {
      const uint32_t u = col[k];
      if (u >= v) break;
      cnt += cand[u] && *(volatile uint8_t*)&x[u];
    }
    const uint8_t nx = (p == 0) || (p >= cnt && p - cnt == 1);
    if (nx != x[v]) {
      x[v] = nx;
      *changed = 1;
    }
  }
}

__global__ void gs_apply_kernel(const uint64_t* row, const uint32_t* col, const uint8_t* cand,
                                const uint8_t* x, uint64_t n, uint8_t* type, uint32_t* live,
                                int* found) {
  for (uint64_t v = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; v < n;
       v += (uint64_t)gridDim.x * blockDim.x) {
    if (!cand[v] || !x[v]) continue;
    type[v] = TI;
    *found = 1;
    for (uint64_t k = row[v]; k < row[v + 1]; ++k) atomicSub(&live[col[k]], 1u);
  }
}

__global__ void count_type_kernel(const uint8_t* type, uint64_t n, uint8_t t,
                                  unsigned long long* out) {
  unsigned long long c = 0;
  for (uint64_t v = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; v < n;
       v += (uint64_t)gridDim.x * blockDim.x)
    c += type[v] == t;
  for (int o = 16; o; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
  if ((threadIdx.x & 31) == 0 && c) atomicAdd(out, c);
}

int read_int(const int* d, cudaStream_t s) {
  int h = 0;
  ETB_CUDA(cudaMemcpyAsync(&h, d, 4, cudaMemcpyDeviceToHost, s));
  ETB_CUDA(cudaStreamSynchronize(s));
  return h;
}

}  // namespace

void classify_device(const DevGraph& g, int64_t mh, DevBuf<uint8_t>& type, uint64_t counts[5],
                     uint64_t* productive_rounds, cudaStream_t s) {
  if (mh < -1) throw std::invalid_argument("classify_vertices: mh must be -1 or >= 0");
  const uint64_t n = g.n;
  type.alloc(n ? n : 1);
  DevBuf<uint32_t> live(n ? n : 1);
  DevBuf<unsigned long long> ctr(8);
  ETB_CUDA(cudaMemsetAsync(ctr.get(), 0, 64, s));
  const unsigned gb = grid_for(n, 256);
  uint64_t rounds = 0;
  const bool gs = productive_rounds != nullptr || mh >= 1;

  if (!gs && mh == -1) {
    // Frontier peel to the fixpoint (order independent).
    DevBuf<uint32_t> qa(n ? n : 1), qb(n ? n : 1);
    leaf_pass_kernel<<<gb, 256, 0, s>>>(g.deg.get(), n, type.get(), live.get(), qa.get(),
                                        ctr.get());
    ETB_LAUNCH_CHECK();
    uint64_t qn = read_u64(reinterpret_cast<uint64_t*>(ctr.get()), s);
    int cur = 0;
    while (qn > 0) {
      unsigned long long* nl = ctr.get() + 1 + (cur & 1);
      ETB_CUDA(cudaMemsetAsync(nl, 0, 8, s));
      peel_round_kernel<<<grid_for(qn * 32, 256), 256, 0, s>>>(
          g.row.get(), g.col.get(), cur ? qb.get() : qa.get(), qn, type.get(), live.get(),
          cur ? qa.get() : qb.get(), nl);
      ETB_LAUNCH_CHECK();
      qn = read_u64(reinterpret_cast<uint64_t*>(nl), s);
      cur ^= 1;
    }
  } else {
    leaf_pass_kernel<<<gb, 256, 0, s>>>(g.deg.get(), n, type.get(), live.get(), nullptr, nullptr);
    ETB_LAUNCH_CHECK();
    leaf_decrement_kernel<<<gb, 256, 0, s>>>(g.row.get(), g.col.get(), type.get(), n, live.get());
    ETB_LAUNCH_CHECK();
    if (mh != 0) {
      // The reference enters round 1 only if the leaf pass found a leaf.
      DevBuf<uint32_t> pre(n ? n : 1);
      DevBuf<uint8_t> cand(n ? n : 1), x(n ? n : 1);
      DevBuf<int> flags(2);
      // The reference enters round 1 only if the leaf pass marked a leaf.
      ETB_CUDA(cudaMemsetAsync(ctr.get(), 0, 8, s));
      count_type_kernel<<<gb, 256, 0, s>>>(type.get(), n, TL, ctr.get());
      ETB_LAUNCH_CHECK();
      bool found = read_u64(reinterpret_cast<uint64_t*>(ctr.get()), s) > 0;
      for (int64_t h = 1; found && (mh == -1 || h <= mh); ++h) {
        ETB_CUDA(cudaMemcpyAsync(pre.get(), live.get(), n * 4, cudaMemcpyDeviceToDevice, s));
        ETB_CUDA(cudaMemsetAsync(ctr.get(), 0, 8, s));
        gs_candidates_kernel<<<gb, 256, 0, s>>>(g.row.get(), g.col.get(), type.get(), pre.get(), n,
                                                cand.get(), x.get(), ctr.get());
        ETB_LAUNCH_CHECK();
        if (read_u64(reinterpret_cast<uint64_t*>(ctr.get()), s) == 0) break;
        for (;;) {
          ETB_CUDA(cudaMemsetAsync(flags.get(), 0, 4, s));
          gs_sweep_kernel<<<gb, 256, 0, s>>>(g.row.get(), g.col.get(), pre.get(), cand.get(), n,
                                             x.get(), flags.get());
          ETB_LAUNCH_CHECK();
          if (!read_int(flags.get(), s)) break;
        }
        ETB_CUDA(cudaMemsetAsync(flags.get() + 1, 0, 4, s));
        gs_apply_kernel<<<gb, 256, 0, s>>>(g.row.get(), g.col.get(), cand.get(), x.get(), n,
                                           type.get(), live.get(), flags.get() + 1);
        ETB_LAUNCH_CHECK();
        found = read_int(flags.get() + 1, s) != 0;
        if (found) ++rounds;
      }
    }
  }
  ETB_CUDA(cudaMemsetAsync(ctr.get(), 0, 64, s));
  core_edge_kernel<<<gb, 256, 0, s>>>(g.deg.get(), live.get(), n, type.get(), ctr.get());
  ETB_LAUNCH_CHECK();
  unsigned long long h[5];
  ETB_CUDA(cudaMemcpyAsync(h, ctr.get(), 40, cudaMemcpyDeviceToHost, s));
  ETB_CUDA(cudaStreamSynchronize(s));
  for (int i = 0; i < 5; ++i) counts[i] = h[i];
  if (productive_rounds) *productive_rounds = rounds;
}

}  // namespace etb
