// The extern "C" boundary (include/etbfs_cuda.h). Every entry point converts
// exceptions into status codes: std::invalid_argument -> ETB_EINVAL (the
// reference's caller errors, same messages), std::runtime_error ->
// ETB_ERUNTIME, CUDA failures -> ETB_ECUDA.
#include <algorithm>
#include <chrono>
#include <cstring>
#include <memory>
#include <string>
#include <thread>
#include <vector>

#include <unistd.h>

#include "bfs.cuh"
#include "bfs_part.cuh"

struct etb_graph {
  // shared with the layouts built from it (they keep it alive past etb_graph_free)
  std::shared_ptr<etb::DevGraph> sp = std::make_shared<etb::DevGraph>();
  etb::DevGraph& g = *sp;
  int device = 0;
  cudaStream_t stream = nullptr;
  ~etb_graph() {
    if (stream) cudaStreamDestroy(stream);
  }
};

struct etb_layout {
  etb::DevLayout L;
  etb::BfsState S;
  int device = 0;
  cudaStream_t stream = nullptr;
  cudaEvent_t ev[4] = {nullptr, nullptr, nullptr, nullptr};
  etb::DevBuf<uint8_t> flush;
  std::unique_ptr<etb::PartState> P;  // 1D core partition (null = single-partition kernel)
  int system_scope = 0;               // peers are other GPUs
  ~etb_layout() {
    for (auto& e : ev)
      if (e) cudaEventDestroy(e);
    if (stream) cudaStreamDestroy(stream);
  }
};

namespace {

thread_local std::string g_err;

template <typename F>
int guarded(F&& f) {
  try {
    f();
    return ETB_OK;
  } catch (const std::invalid_argument& e) {
    g_err = e.what();
    return ETB_EINVAL;
  } catch (const etb::CudaError& e) {
    g_err = e.what();
    return ETB_ECUDA;
  } catch (const std::bad_alloc&) {
    g_err = "out of host memory";
    return ETB_ERUNTIME;
  } catch (const std::runtime_error& e) {
    g_err = e.what();
    return ETB_ERUNTIME;
  } catch (const std::exception& e) {
    g_err = e.what();
    return ETB_ERUNTIME;
  } catch (...) {
    g_err = "unknown error";
    return ETB_ERUNTIME;
  }
}

void need(const void* p, const char* what) {
  if (!p) throw std::invalid_argument(std::string(what) + ": null argument");
}

}  // namespace

namespace etb {
void set_last_error(const char* msg) { g_err = msg; }  // for the host-only entry points
}  // namespace etb

namespace {

cudaStream_t new_stream() {
  cudaStream_t s;
  ETB_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
  return s;
}

int current_device() {
  int d = 0;
  ETB_CUDA(cudaGetDevice(&d));
  return d;
}

uint64_t physical_memory_bytes() {
  const long pages = sysconf(_SC_PHYS_PAGES), page = sysconf(_SC_PAGE_SIZE);
  if (pages <= 0 || page <= 0) return ~uint64_t{0};
  return uint64_t(pages) * uint64_t(page);
}

void widen(const uint32_t* in, uint64_t n, uint64_t* out) {
  for (uint64_t i = 0; i < n; ++i) out[i] = in[i] == etb::kNone32 ? ETB_NO_VERTEX : in[i];
}

template <typename T>
std::vector<T> download(const T* d, uint64_t n, cudaStream_t s) {
  std::vector<T> h(n);
  if (n) ETB_CUDA(cudaMemcpyAsync(h.data(), d, n * sizeof(T), cudaMemcpyDeviceToHost, s));
  ETB_CUDA(cudaStreamSynchronize(s));
  return h;
}

void finish_layout(etb_layout* h) {
  etb::bfs_state_init(h->L, h->S, h->stream);
  for (auto& e : h->ev) ETB_CUDA(cudaEventCreate(&e));
}

etb::BfsParams run_bfs(etb_layout* h, uint64_t start, const etb_bfs_options* o,
                       bool want_stats, cudaEvent_t pre_launch = nullptr,
                       unsigned long long* bstamp = nullptr,
                       unsigned long long* wstamp = nullptr, int32_t wdepth = -1) {
  const etb::DevLayout& L = h->L;
  if (start >= L.n) throw std::invalid_argument("et_bfs: start out of range");
  etb_bfs_options opt{ETB_KERNEL_HYBRID, ETB_REPLAY_TEET, 14.0, 24.0};
  if (o) opt = *o;
  if (opt.replay == ETB_REPLAY_TEOLV && L.mh != 0)
    throw std::invalid_argument("et_bfs: leaves-only replay needs a height-0 classification");
  if (opt.replay != ETB_REPLAY_TEET && opt.replay != ETB_REPLAY_TEOLV)
    throw std::invalid_argument("et_bfs: unknown tree replay");
  if (opt.kernel < ETB_KERNEL_TOP_DOWN || opt.kernel > ETB_KERNEL_HYBRID_BLOCK_SEARCH)
    throw std::invalid_argument("et_bfs: unknown core kernel");
  etb::BfsParams p{};
  etb::bfs_fill_params(L, h->S, p);
  etb::bfs_prepare_start(L, h->S, start, p, h->stream);
  const bool hybrid = opt.kernel == ETB_KERNEL_HYBRID || opt.kernel == ETB_KERNEL_DEGREE_AWARE ||
                      opt.kernel == ETB_KERNEL_HYBRID_BLOCK_SEARCH;
  if (p.start != etb::kNone32 && hybrid && (!(opt.alpha > 0.0) || !(opt.beta > 0.0)))
    throw std::invalid_argument("run_hybrid: alpha and beta must be positive");
  p.alpha = opt.alpha;
  p.beta = opt.beta;
  p.top_down_only = opt.kernel == ETB_KERNEL_TOP_DOWN;
  p.bottom_up_only = opt.kernel == ETB_KERNEL_BLOCK_SEARCH;
  if (want_stats) {
    p.trace = h->S.trace.get();
    p.level_claims = h->S.level_claims.get();
    p.nlevels = h->S.nlevels.get();
    ETB_CUDA(cudaMemsetAsync(p.trace, 0, 256, h->stream));
  }
  p.bstamp = bstamp;
  p.wstamp = wstamp;
  p.wdepth = wdepth;
  if (pre_launch) ETB_CUDA(cudaEventRecord(pre_launch, h->stream));
  if (h->P) {
    etb::PartParams pp{};
    pp.base = p;
    pp.parts = h->P->d_parts.get();
    pp.nparts = h->P->nparts;
    pp.first_part = h->P->first;
    pp.local_parts = h->P->local;
    pp.system_scope = h->system_scope;
    etb::part_launch(pp, *h->P, h->stream);
  } else {
    etb::bfs_launch(p, h->S, h->stream);
  }
  h->S.has_result = true;
  h->S.assembled = false;
  h->S.last_start = start;
  return p;
}

void collect_stats(etb_layout* h, etb_bfs_stats* st) {
  uint32_t nl = 0;
  std::memset(st, 0, sizeof(*st));
  ETB_CUDA(cudaMemcpyAsync(&nl, h->S.nlevels.get(), 4, cudaMemcpyDeviceToHost, h->stream));
  ETB_CUDA(cudaMemcpyAsync(st->direction_trace, h->S.trace.get(), 255, cudaMemcpyDeviceToHost,
                           h->stream));
  ETB_CUDA(cudaMemcpyAsync(st->level_claims, h->S.level_claims.get(), 256 * 8,
                           cudaMemcpyDeviceToHost, h->stream));
  uint64_t ts[256];
  ETB_CUDA(cudaMemcpyAsync(ts, h->S.level_claims.get() + 256, 256 * 8, cudaMemcpyDeviceToHost,
                           h->stream));
  ETB_CUDA(cudaStreamSynchronize(h->stream));
  // both kernels stamp (partition 0's first block when partitioned); a rank
  // that does not run partition 0 has no stamps
  if (ts[0] && ts[255] >= ts[0]) {
    for (uint32_t i = 0; i <= nl && i + 1 < 255; ++i)
      st->level_ns[i] = ts[1 + i] >= ts[0] ? ts[1 + i] - ts[0] : 0;
    st->total_ns = ts[255] - ts[0];
  }
  st->levels = nl;
  st->direction_trace[std::min<uint32_t>(nl, 255)] = 0;
  for (uint32_t i = 0; i < nl && i < 255; ++i) st->bottom_up_levels += st->direction_trace[i] == 'b';
}

__global__ void te_kernel(const uint2* dp, const uint32_t* degn, uint64_t n,
                          unsigned long long* out) {
  unsigned long long acc = 0;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x)
    if (static_cast<int32_t>(dp[i].x) >= 0) acc += degn[i];
  for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if ((threadIdx.x & 31) == 0 && acc) atomicAdd(out, acc);
}

// te_kernel over the vertices partition `part` of G owns (bfs_part.cuh).
__global__ void te_owned_kernel(const uint2* dp, const uint32_t* degn, uint64_t n, uint64_t nc,
                                uint64_t nt, const uint32_t* tanchor, uint32_t part, uint32_t G,
                                unsigned long long* out) {
  unsigned long long acc = 0;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x) {
    uint32_t o;
    if (i < nc) o = etb::core_owner(static_cast<uint32_t>(i), G);
    else if (i < nc + nt) o = tanchor[i - nc] == etb::kNone32 ? G - 1 : etb::core_owner(tanchor[i - nc], G);
    else o = G - 1;
    if (o == part && static_cast<int32_t>(dp[i].x) >= 0) acc += degn[i];
  }
  for (int s = 16; s; s >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, s);
  if ((threadIdx.x & 31) == 0 && acc) atomicAdd(out, acc);
}

// Interleaved {depth, parent} -> separate arrays (either may be null).
__global__ void split_kernel(const uint2* dp, uint64_t n, int32_t* depth, uint32_t* parent,
                             uint64_t* parent64) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x) {
    const uint2 e = dp[i];
    if (depth) depth[i] = static_cast<int32_t>(e.x);
    if (parent) parent[i] = e.y;
    if (parent64) parent64[i] = e.y == etb::kNone32 ? ~0ull : e.y;
  }
}

// 0xFF fill of a host range by up to 8 threads (the calling one included): the
// unreached marker of every output type is all ones (-1 / UINT32_MAX /
// ETB_NO_VERTEX). One thread fills ~10-15 GB/s, a device->host DMA moves 55.
void host_fill_ones(void* dst, size_t bytes) {
  constexpr size_t kPerThread = size_t{4} << 20;
  unsigned hw = std::thread::hardware_concurrency();
  size_t want = std::min<size_t>({size_t{8}, hw ? hw : 1, bytes / kPerThread});
  if (want <= 1) {
    std::memset(dst, 0xFF, bytes);
    return;
  }
  const size_t part = ((bytes / want) + 63) & ~size_t{63};
  std::vector<std::thread> th;
  th.reserve(want - 1);
  char* p = static_cast<char*>(dst);
  for (size_t t = 1; t < want; ++t) {
    const size_t lo = std::min(bytes, t * part), hi = std::min(bytes, (t + 1) * part);
    if (hi > lo) th.emplace_back([p, lo, hi] { std::memset(p + lo, 0xFF, hi - lo); });
  }
  std::memset(p, 0xFF, std::min(bytes, part));
  for (auto& t : th) t.join();
}

// Split the last result on the device and copy the requested parts to host.
// Only the live prefix [0, nc + nt) of the relaid id space crosses PCIe: the
// isolated vertices that close it (layout.cu) are unreached in every result
// unless one of them is the start, so the host fills their range itself while
// the DMA of the prefix runs (half of n at Graph500 scales 26-28).
void download_result(etb_layout* h, int32_t* depth, uint32_t* parent, uint64_t* parent64) {
  const uint64_t n = h->L.n;
  if (!n || (!depth && !parent && !parent64)) return;
  auto& S = h->S;
  cudaStream_t s = h->stream;
  // a partitioned layout's result may have been assembled by the caller
  // through etb_result_device_ptr: copy it whole
  const uint64_t live = h->P ? n : std::min<uint64_t>(n, h->L.nc + h->L.nt);
  if (live) {
    // staging buffers persist with the layout: no allocation (and no
    // synchronising free) inside the reference-facing call
    if (depth && S.tmp_depth.size() < live) S.tmp_depth.alloc(live);
    if (parent && S.tmp_parent.size() < live) S.tmp_parent.alloc(live);
    if (parent64 && S.tmp_parent64.size() < live) S.tmp_parent64.alloc(live);
    split_kernel<<<etb::grid_for(live, 256), 256, 0, s>>>(
        S.dp.get(), live, depth ? S.tmp_depth.get() : nullptr,
        parent ? S.tmp_parent.get() : nullptr, parent64 ? S.tmp_parent64.get() : nullptr);
    ETB_LAUNCH_CHECK();
    if (depth)
      ETB_CUDA(cudaMemcpyAsync(depth, S.tmp_depth.get(), live * 4, cudaMemcpyDeviceToHost, s));
    if (parent)
      ETB_CUDA(cudaMemcpyAsync(parent, S.tmp_parent.get(), live * 4, cudaMemcpyDeviceToHost, s));
    if (parent64)
      ETB_CUDA(cudaMemcpyAsync(parent64, S.tmp_parent64.get(), live * 8, cudaMemcpyDeviceToHost, s));
  }
  if (live < n) {
    const uint64_t tail = n - live;
    if (depth) host_fill_ones(depth + live, tail * 4);
    if (parent) host_fill_ones(parent + live, tail * 4);
    if (parent64) host_fill_ones(parent64 + live, tail * 8);
    const uint64_t st = S.last_start;  // an isolated start is its own depth-0 root
    if (st >= live && st < n) {
      if (depth) depth[st] = 0;
      if (parent) parent[st] = static_cast<uint32_t>(st);
      if (parent64) parent64[st] = st;
    }
  }
  ETB_CUDA(cudaStreamSynchronize(s));
}

// Relaid {depth, parent} -> original ids (translate_tree + tree_levels,
// validate.hpp:48-50): levels u64 (kUnreached = ~0), parent u64 (kNoVertex).
__global__ void lift_kernel(const uint2* dp, const uint32_t* new2old, uint64_t n, uint64_t* lv,
                            uint64_t* par) {
  for (uint64_t v = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; v < n;
       v += (uint64_t)gridDim.x * blockDim.x) {
    const uint2 e = dp[v];
    const uint32_t o = new2old[v];
    if (lv) lv[o] = static_cast<int32_t>(e.x) >= 0 ? e.x : ~0ull;
    if (par) par[o] = e.y == etb::kNone32 ? ~0ull : new2old[e.y];
  }
}

__global__ void widen_kernel(const uint32_t* in, uint64_t n, uint64_t* out) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x)
    out[i] = in[i] == etb::kNone32 ? ~0ull : in[i];
}

void download_widened(const uint32_t* d, uint64_t n, uint64_t* host, cudaStream_t s) {
  if (!n) return;
  etb::DevBuf<uint64_t> tmp(n);
  widen_kernel<<<etb::grid_for(n, 256), 256, 0, s>>>(d, n, tmp.get());
  ETB_LAUNCH_CHECK();
  ETB_CUDA(cudaMemcpyAsync(host, tmp.get(), n * 8, cudaMemcpyDeviceToHost, s));
  ETB_CUDA(cudaStreamSynchronize(s));
}

}  // namespace

extern "C" {

const char* etb_last_error(void) { return g_err.c_str(); }

int etb_version(void) { return 1; }

int etb_device_count(int* count) {
  return guarded([&] {
    need(count, "etb_device_count");
    ETB_CUDA(cudaGetDeviceCount(count));
  });
}

int etb_set_device(int device) { return guarded([&] { ETB_CUDA(cudaSetDevice(device)); }); }

int etb_generate_kronecker(const etb_kron_params* p, uint64_t* out_pairs) {
  return guarded([&] {
    need(p, "generate_kronecker");
    etb::kron_validate(*p);
    const uint64_t n = uint64_t{1} << p->scale;
    const uint64_t t = n * p->edgefactor;
    if (t > physical_memory_bytes() / 16)
      throw std::runtime_error("generate_kronecker: edge list would exceed physical memory");
    need(out_pairs, "generate_kronecker");
    cudaStream_t s = new_stream();
    std::unique_ptr<CUstream_st, decltype(&cudaStreamDestroy)> guard(s, cudaStreamDestroy);
    const uint64_t chunk = std::min<uint64_t>(t, uint64_t{1} << 25);
    etb::DevBuf<uint64_t> buf(2 * (chunk ? chunk : 1));
    for (uint64_t first = 0; first < t; first += chunk) {
      const uint64_t c = std::min(chunk, t - first);
      etb::kron_generate_pairs64(*p, first, c, buf.get(), s);
      ETB_CUDA(cudaMemcpyAsync(out_pairs + 2 * first, buf.get(), c * 16, cudaMemcpyDeviceToHost,
                               s));
      ETB_CUDA(cudaStreamSynchronize(s));
    }
  });
}

int etb_graph_from_edges(uint64_t n, const uint64_t* pairs, uint64_t count, etb_graph** out,
                         uint64_t* self_loops, uint64_t* dups) {
  return guarded([&] {
    need(out, "build_csr");
    *out = nullptr;
    if (n > (uint64_t{1} << 48))
      throw std::invalid_argument("build_csr: vertex count exceeds 2^48");
    if (count) need(pairs, "build_csr");
    for (uint64_t i = 0; i < count; ++i)  // build.cpp:26-31, same message
      if (pairs[2 * i] >= n || pairs[2 * i + 1] >= n)
        throw std::invalid_argument("build_csr: endpoint out of range at edge index " +
                                    std::to_string(i));
    auto h = std::make_unique<etb_graph>();
    h->device = current_device();
    h->stream = new_stream();
    etb::build_csr_from_host_pairs(n, pairs, count, h->g, self_loops, dups, h->stream);
    *out = h.release();
  });
}

int etb_graph_generate(const etb_kron_params* p, etb_graph** out, uint64_t* self_loops,
                       uint64_t* dups) {
  return guarded([&] {
    need(p, "generate_kronecker");
    need(out, "generate_kronecker");
    *out = nullptr;
    auto h = std::make_unique<etb_graph>();
    h->device = current_device();
    h->stream = new_stream();
    etb::build_csr_from_generator(*p, h->g, self_loops, dups, h->stream);
    *out = h.release();
  });
}

int etb_graph_from_csr(uint64_t n, const uint64_t* row, const uint64_t* cols, etb_graph** out) {
  return guarded([&] {
    need(out, "etb_graph_from_csr");
    need(row, "etb_graph_from_csr");
    *out = nullptr;
    if (n > etb::kMaxDeviceVertices)
      throw std::invalid_argument("etb_graph_from_csr: vertex count exceeds the device id range");
    const uint64_t nnz = row[n];
    if (nnz) need(cols, "etb_graph_from_csr");
    std::vector<uint32_t> c32(nnz);
    for (uint64_t i = 0; i < nnz; ++i) {
      if (cols[i] >= n) throw std::invalid_argument("etb_graph_from_csr: column out of range");
      c32[i] = static_cast<uint32_t>(cols[i]);
    }
    std::vector<uint32_t> deg(n);
    for (uint64_t v = 0; v < n; ++v) {
      if (row[v + 1] < row[v]) throw std::invalid_argument("etb_graph_from_csr: bad row offsets");
      deg[v] = static_cast<uint32_t>(row[v + 1] - row[v]);
    }
    auto h = std::make_unique<etb_graph>();
    h->device = current_device();
    h->stream = new_stream();
    auto& G = h->g;
    G.n = n;
    G.nnz = nnz;
    G.row.alloc(n + 1);
    G.col.alloc(nnz ? nnz : 1);
    G.deg.alloc(n ? n : 1);
    ETB_CUDA(cudaMemcpyAsync(G.row.get(), row, (n + 1) * 8, cudaMemcpyHostToDevice, h->stream));
    if (nnz)
      ETB_CUDA(cudaMemcpyAsync(G.col.get(), c32.data(), nnz * 4, cudaMemcpyHostToDevice, h->stream));
    if (n)
      ETB_CUDA(cudaMemcpyAsync(G.deg.get(), deg.data(), n * 4, cudaMemcpyHostToDevice, h->stream));
    ETB_CUDA(cudaStreamSynchronize(h->stream));
    *out = h.release();
  });
}

int etb_graph_info(const etb_graph* g, uint64_t* n, uint64_t* nnz) {
  return guarded([&] {
    need(g, "etb_graph_info");
    if (n) *n = g->g.n;
    if (nnz) *nnz = g->g.nnz;
  });
}

int etb_graph_degree_split(const etb_graph* g, uint64_t limit, uint64_t* in_plus,
                           uint64_t* minus_offsets, uint64_t* minus_cols) {
  return guarded([&] {
    need(g, "etb_graph_degree_split");
    need(minus_offsets, "etb_graph_degree_split");
    ETB_CUDA(cudaSetDevice(g->device));
    etb::graph_degree_split(g->g, limit, in_plus, minus_offsets, minus_cols, g->stream);
  });
}

int etb_graph_levels(const etb_graph* g, uint64_t root, uint64_t* levels) {
  return guarded([&] {
    need(g, "etb_graph_levels");
    need(levels, "etb_graph_levels");
    if (root >= g->g.n) throw std::invalid_argument("oracle_bfs: root out of range");
    ETB_CUDA(cudaSetDevice(g->device));
    etb::DevBuf<uint32_t> lvl;
    etb::graph_levels(g->g, root, lvl, g->stream);
    std::vector<uint32_t> h(g->g.n);
    if (g->g.n)
      ETB_CUDA(cudaMemcpyAsync(h.data(), lvl.get(), g->g.n * 4, cudaMemcpyDeviceToHost,
                               g->stream));
    ETB_CUDA(cudaStreamSynchronize(g->stream));
    for (uint64_t i = 0; i < g->g.n; ++i) levels[i] = h[i] == etb::kNone32 ? ~uint64_t{0} : h[i];
  });
}

int etb_graph_validate_tree(const etb_graph* g, uint64_t root, const uint64_t* parent,
                            uint64_t* counts, uint64_t* where, uint32_t* first_count) {
  return guarded([&] {
    need(g, "etb_graph_validate_tree");
    need(parent, "etb_graph_validate_tree");
    need(counts, "etb_graph_validate_tree");
    if (root >= g->g.n) throw std::invalid_argument("validate_bfs_tree: root out of range");
    ETB_CUDA(cudaSetDevice(g->device));
    uint64_t out[8] = {};
    std::vector<uint64_t> first[6];
    etb::graph_validate_tree(g->g, root, parent, out, first, g->stream);
    bool ok = true;
    for (int r = 1; r <= 5; ++r) ok = ok && out[r] == 0;
    counts[0] = ok;
    for (int r = 1; r <= 7; ++r) counts[r] = out[r];
    for (int r = 1; r <= 5; ++r) {
      const size_t m = std::min<size_t>(first[r].size(), 25);
      if (first_count) first_count[r - 1] = static_cast<uint32_t>(m);
      if (where)
        for (size_t i = 0; i < m; ++i)
          where[(r - 1) * 25 + i] = r == 4 ? (first[r][i] >> 32) : first[r][i];
    }
  });
}

int etb_steps_run(const etb_graph* g, int op, uint64_t limit, uint64_t* visited,
                  uint64_t* current, uint64_t* next, uint64_t* parent, const uint64_t* in_plus,
                  const uint64_t* minus_offsets, const uint64_t* minus_cols, double alpha,
                  double beta, uint64_t* stats, char* trace, uint64_t trace_cap) {
  return guarded([&] {
    need(g, "etb_steps_run");
    if (op < 0 || op > 8) throw std::invalid_argument("etb_steps_run: unknown op");
    const bool split = op == 2 || op == 3 || op == 6 || op == 7 || op == 8;
    if (split && (!in_plus || !minus_offsets || (minus_offsets[g->g.n] && !minus_cols)))
      throw std::invalid_argument("run_hybrid: bottom-up kind needs a degree split");
    if (op >= 5 && op <= 7 && (!(alpha > 0.0) || !(beta > 0.0)))
      throw std::invalid_argument("run_hybrid: alpha and beta must be positive");
    if (g->g.n) {
      need(visited, "etb_steps_run");
      need(current, "etb_steps_run");
      need(next, "etb_steps_run");
      need(parent, "etb_steps_run");
    }
    ETB_CUDA(cudaSetDevice(g->device));
    uint64_t out[6] = {};
    std::string tr;
    etb::step_run(g->g, op, limit, visited, current, next, parent, in_plus, minus_offsets,
                  minus_cols, alpha, beta, out, trace ? &tr : nullptr, g->stream);
    if (stats)
      for (int i = 0; i < 6; ++i) stats[i] += out[i];
    if (trace && trace_cap) {
      const size_t m = std::min<size_t>(tr.size(), trace_cap - 1);
      std::memcpy(trace, tr.data(), m);
      trace[m] = 0;
    }
  });
}

int etb_tree_replay(int leaves_only, const uint64_t* src, const uint64_t* dst,
                    const uint64_t* core_edge, uint64_t count, const uint64_t* visited_words,
                    uint64_t words, uint64_t* parent, uint64_t n) {
  return guarded([&] {
    if (count) {
      need(src, "etb_tree_replay");
      need(dst, "etb_tree_replay");
      need(core_edge, "etb_tree_replay");
    }
    if (n) need(parent, "etb_tree_replay");
    if (words) need(visited_words, "etb_tree_replay");
    for (uint64_t i = 0; i < count; ++i) {  // the host side validates the indices
      const uint64_t guard = leaves_only ? src[i] : core_edge[i];
      if (dst[i] >= n || (guard != ~uint64_t{0} && guard >= words * 64))
        throw std::invalid_argument("teet: entry index out of range");
    }
    cudaStream_t s = nullptr;
    ETB_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
    struct StreamDel {
      cudaStream_t s;
      ~StreamDel() { cudaStreamDestroy(s); }
    } del{s};
    etb::tree_replay_run(leaves_only, src, dst, core_edge, count, visited_words, words, parent, n,
                         s);
  });
}

int etb_graph_download(const etb_graph* g, uint64_t* row, uint64_t* cols, uint64_t* degrees) {
  return guarded([&] {
    need(g, "etb_graph_download");
    ETB_CUDA(cudaSetDevice(g->device));
    const auto& G = g->g;
    if (row && G.n + 1)
      ETB_CUDA(cudaMemcpyAsync(row, G.row.get(), (G.n + 1) * 8, cudaMemcpyDeviceToHost, g->stream));
    if (cols) download_widened(G.col.get(), G.nnz, cols, g->stream);
    if (degrees && G.n) {
      auto d = download(G.deg.get(), G.n, g->stream);
      for (uint64_t i = 0; i < G.n; ++i) degrees[i] = d[i];
    }
    ETB_CUDA(cudaStreamSynchronize(g->stream));
  });
}

void etb_graph_free(etb_graph* g) { delete g; }

int etb_classify(const etb_graph* g, int64_t mh, uint8_t* types_out, uint64_t* counts_out) {
  return guarded([&] {
    need(g, "classify_vertices");
    ETB_CUDA(cudaSetDevice(g->device));
    etb::DevBuf<uint8_t> type;
    uint64_t counts[5];
    etb::classify_device(g->g, mh, type, counts, nullptr, g->stream);
    if (types_out && g->g.n)
      ETB_CUDA(cudaMemcpyAsync(types_out, type.get(), g->g.n, cudaMemcpyDeviceToHost, g->stream));
    ETB_CUDA(cudaStreamSynchronize(g->stream));
    if (counts_out) std::memcpy(counts_out, counts, sizeof counts);
  });
}

int etb_peak_height(const etb_graph* g, uint64_t* ph) {
  return guarded([&] {
    need(g, "compute_peak_height");
    need(ph, "compute_peak_height");
    ETB_CUDA(cudaSetDevice(g->device));
    etb::DevBuf<uint8_t> type;
    uint64_t counts[5];
    etb::classify_device(g->g, -1, type, counts, ph, g->stream);
  });
}

int etb_layout_build(const etb_graph* g, int64_t mh, etb_layout** out) {
  return guarded([&] {
    need(g, "relayout_csr");
    need(out, "relayout_csr");
    *out = nullptr;
    ETB_CUDA(cudaSetDevice(g->device));
    auto h = std::make_unique<etb_layout>();
    h->device = g->device;
    h->stream = new_stream();
    {
      etb::DevBuf<uint8_t> type;
      uint64_t counts[5];
      etb::classify_device(g->g, mh, type, counts, nullptr, h->stream);
      etb::build_layout(g->g, type.get(), mh, h->L, h->stream);
    }
    h->L.src_graph = g->sp;
    finish_layout(h.get());
    *out = h.release();
  });
}

int etb_layout_build_types(const etb_graph* g, const uint8_t* types, int64_t mh,
                           etb_layout** out) {
  return guarded([&] {
    need(g, "relayout_csr");
    need(out, "relayout_csr");
    *out = nullptr;
    if (g->g.n) need(types, "relayout_csr");
    for (uint64_t i = 0; i < g->g.n; ++i)
      if (types[i] > ETB_VZ) throw std::invalid_argument("relayout_csr: bad vertex type");
    ETB_CUDA(cudaSetDevice(g->device));
    auto h = std::make_unique<etb_layout>();
    h->device = g->device;
    h->stream = new_stream();
    {
      etb::DevBuf<uint8_t> type(g->g.n ? g->g.n : 1);
      if (g->g.n)
        ETB_CUDA(cudaMemcpyAsync(type.get(), types, g->g.n, cudaMemcpyHostToDevice, h->stream));
      etb::build_layout(g->g, type.get(), mh, h->L, h->stream);
    }
    h->L.src_graph = g->sp;
    finish_layout(h.get());
    *out = h.release();
  });
}

int etb_layout_info_get(const etb_layout* h, etb_layout_info* info) {
  return guarded([&] {
    need(h, "etb_layout_info");
    need(info, "etb_layout_info");
    const auto& L = h->L;
    info->vertex_count = L.n;
    info->core_vertex_count = L.nc;
    info->tree_vertex_count = L.nt;
    info->isolated_count = L.nz;
    info->core_directed_edges = L.ecore;
    info->directed_edges = L.nnz_full;
    info->tree_count = L.tree_count;
    info->max_tree_size = L.max_tree;
    info->mh = L.mh;
  });
}

int etb_layout_download_maps(const etb_layout* h, uint64_t* new2old, uint64_t* old2new,
                             uint8_t* types) {
  return guarded([&] {
    need(h, "etb_layout_download_maps");
    ETB_CUDA(cudaSetDevice(h->device));
    const auto& L = h->L;
    if (new2old) widen(download(L.new2old.get(), L.n, h->stream).data(), L.n, new2old);
    if (old2new) widen(download(L.old2new.get(), L.n, h->stream).data(), L.n, old2new);
    if (types && L.n) {
      ETB_CUDA(cudaMemcpyAsync(types, L.type.get(), L.n, cudaMemcpyDeviceToHost, h->stream));
      ETB_CUDA(cudaStreamSynchronize(h->stream));
    }
  });
}

int etb_layout_download_graph(const etb_layout* h, uint64_t* row, uint64_t* cols) {
  return guarded([&] {
    need(h, "etb_layout_download_graph");
    ETB_CUDA(cudaSetDevice(h->device));
    etb::DevBuf<uint64_t> r;
    etb::DevBuf<uint32_t> c;
    etb::build_full_relabelled(h->L, r, c, h->stream);
    if (row)
      ETB_CUDA(cudaMemcpyAsync(row, r.get(), (h->L.n + 1) * 8, cudaMemcpyDeviceToHost, h->stream));
    if (cols) download_widened(c.get(), h->L.nnz_full, cols, h->stream);
    ETB_CUDA(cudaStreamSynchronize(h->stream));
  });
}

int etb_layout_download_etl(const etb_layout* h, uint64_t* src, uint64_t* dst, uint64_t* ce) {
  return guarded([&] {
    need(h, "extract_edge_tree_list");
    const auto& L = h->L;
    for (uint64_t i = 0; i < L.nt; ++i) {
      if (src) src[i] = L.h_tsrc[i];
      if (dst) dst[i] = L.nc + i;
      if (ce) ce[i] = L.h_tanchor[i] == etb::kNone32 ? ETB_NO_VERTEX : L.h_tanchor[i];
    }
  });
}

int etb_layout_restricted_edges(const etb_layout* h, uint64_t* count) {
  return guarded([&] {
    need(h, "restricted_edge_count");
    need(count, "restricted_edge_count");
    *count = h->L.ecore;
  });
}

void etb_layout_free(etb_layout* h) { delete h; }

int etb_bfs_device(etb_layout* h, uint64_t start, const etb_bfs_options* opts,
                   etb_bfs_stats* stats) {
  return guarded([&] {
    need(h, "et_bfs");
    ETB_CUDA(cudaSetDevice(h->device));
    run_bfs(h, start, opts, stats != nullptr);
    if (stats) collect_stats(h, stats);
  });
}

int etb_bfs(etb_layout* h, uint64_t start, const etb_bfs_options* opts, int32_t* depth_out,
            uint64_t* parent_out, etb_bfs_stats* stats) {
  return guarded([&] {
    need(h, "et_bfs");
    ETB_CUDA(cudaSetDevice(h->device));
    run_bfs(h, start, opts, stats != nullptr);
    download_result(h, depth_out, nullptr, parent_out);
    if (stats) collect_stats(h, stats);
  });
}

int etb_bfs_compact(etb_layout* h, uint64_t start, const etb_bfs_options* opts, int32_t* depth,
                    uint32_t* parent) {
  return guarded([&] {
    need(h, "et_bfs");
    ETB_CUDA(cudaSetDevice(h->device));
    run_bfs(h, start, opts, false);
    download_result(h, depth, parent, nullptr);
  });
}

int etb_result_device_ptr(etb_layout* h, uint32_t** dp) {
  return guarded([&] {
    need(h, "etb_result_device_ptr");
    need(dp, "etb_result_device_ptr");
    *dp = reinterpret_cast<uint32_t*>(h->S.dp.get());
  });
}

int etb_result_download_original(etb_layout* h, uint64_t* levels, uint64_t* parent) {
  return guarded([&] {
    need(h, "etb_result_download_original");
    if (!h->S.has_result) throw std::invalid_argument("etb_result_download_original: no result");
    if (h->P && h->P->local < h->P->nparts && !h->S.assembled)
      throw std::invalid_argument("etb_result_download_original: result is spread over several "
                                  "GPUs");
    ETB_CUDA(cudaSetDevice(h->device));
    const uint64_t n = h->L.n;
    if (!n || (!levels && !parent)) return;
    cudaStream_t s = h->stream;
    etb::DevBuf<uint64_t> lv, pa;
    if (levels) lv.alloc(n);
    if (parent) pa.alloc(n);
    lift_kernel<<<etb::grid_for(n, 256), 256, 0, s>>>(h->S.dp.get(), h->L.new2old.get(), n,
                                                       lv.get(), pa.get());
    ETB_LAUNCH_CHECK();
    if (levels) ETB_CUDA(cudaMemcpyAsync(levels, lv.get(), n * 8, cudaMemcpyDeviceToHost, s));
    if (parent) ETB_CUDA(cudaMemcpyAsync(parent, pa.get(), n * 8, cudaMemcpyDeviceToHost, s));
    ETB_CUDA(cudaStreamSynchronize(s));
  });
}

int etb_result_mark_assembled(etb_layout* h) {
  return guarded([&] {
    need(h, "etb_result_mark_assembled");
    if (!h->S.has_result) throw std::invalid_argument("etb_result_mark_assembled: no result");
    h->S.assembled = true;
  });
}

int etb_result_download(etb_layout* h, int32_t* depth, uint32_t* parent) {
  return guarded([&] {
    need(h, "etb_result_download");
    ETB_CUDA(cudaSetDevice(h->device));
    download_result(h, depth, parent, nullptr);
  });
}

int etb_result_traversed_edges(etb_layout* h, uint64_t* te) {
  return guarded([&] {
    need(h, "etb_result_traversed_edges");
    need(te, "etb_result_traversed_edges");
    ETB_CUDA(cudaSetDevice(h->device));
    etb::DevBuf<unsigned long long> acc(1);
    ETB_CUDA(cudaMemsetAsync(acc.get(), 0, 8, h->stream));
    if (h->P && h->P->local < h->P->nparts && !h->S.assembled) {
      // Multi-GPU: this device holds only its partitions' results; the caller
      // sums the partial counts over ranks.
      for (uint32_t j = 0; j < h->P->local; ++j)
        te_owned_kernel<<<etb::grid_for(h->L.n, 256), 256, 0, h->stream>>>(
            h->S.dp.get(), h->L.degn.get(), h->L.n, h->L.nc, h->L.nt, h->L.tanchor.get(),
            h->P->first + j, h->P->nparts, acc.get());
    } else {
      te_kernel<<<etb::grid_for(h->L.n, 256), 256, 0, h->stream>>>(h->S.dp.get(), h->L.degn.get(),
                                                                    h->L.n, acc.get());
    }
    ETB_LAUNCH_CHECK();
    *te = etb::read_u64(reinterpret_cast<uint64_t*>(acc.get()), h->stream) / 2;
  });
}

int etb_result_validate(etb_layout* h, uint64_t start, uint64_t* counts) {
  return guarded([&] {
    need(h, "etb_result_validate");
    need(counts, "etb_result_validate");
    if (start >= h->L.n) throw std::invalid_argument("validate_bfs_tree: root out of range");
    if (h->P && h->P->local < h->P->nparts && !h->S.assembled)
      throw std::invalid_argument("etb_result_validate: result is spread over several GPUs "
                                  "(merge the ranks' owned slices, then etb_result_mark_assembled)");
    ETB_CUDA(cudaSetDevice(h->device));
    etb::validate_result(h->L, h->S.dp.get(), start, counts, h->stream);
  });
}

int etb_result_work(etb_layout* h, uint64_t start, const etb_bfs_options* opts,
                    uint64_t* levels, uint64_t* bytes, uint32_t* nlevels, char* trace,
                    uint64_t* total_bytes) {
  return guarded([&] {
    need(h, "etb_result_work");
    need(total_bytes, "etb_result_work");
    if (h->P) throw std::invalid_argument("etb_result_work: single-partition layouts only");
    ETB_CUDA(cudaSetDevice(h->device));
    run_bfs(h, start, opts, true);
    etb_bfs_stats st;
    collect_stats(h, &st);
    // levels recorded but not run (the start's component was exhausted) end the
    // trace with zero claims: no work
    int nl = static_cast<int>(st.levels);
    while (nl > 0 && st.level_claims[nl - 1] == 0) --nl;
    *total_bytes = etb::result_work(h->L, h->S.dp.get(), st.direction_trace, nl, levels, bytes,
                                    h->stream);
    if (nlevels) *nlevels = static_cast<uint32_t>(nl);
    if (trace) {
      std::memcpy(trace, st.direction_trace, nl);
      trace[nl] = 0;
    }
  });
}

int etb_time_roots_wall(etb_layout* h, const uint64_t* starts, uint64_t count, int warmup,
                        const etb_bfs_options* opts, double* ms_out) {
  return guarded([&] {
    need(h, "etb_time_roots_wall");
    if (count) need(starts, "etb_time_roots_wall");
    ETB_CUDA(cudaSetDevice(h->device));
    for (int w = 0; w < warmup && count; ++w) run_bfs(h, starts[w % count], opts, false);
    ETB_CUDA(cudaStreamSynchronize(h->stream));
    for (uint64_t i = 0; i < count; ++i) {
      const auto t0 = std::chrono::steady_clock::now();
      run_bfs(h, starts[i], opts, false);
      ETB_CUDA(cudaStreamSynchronize(h->stream));
      const auto t1 = std::chrono::steady_clock::now();
      if (ms_out) ms_out[i] = std::chrono::duration<double, std::milli>(t1 - t0).count();
    }
  });
}

int etb_debug_check_line(uint32_t* line) {
  return guarded([&] {
    need(line, "etb_debug_check_line");
    *line = etb::debug_check_line();
  });
}

int etb_debug_diag(etb_layout* h, uint64_t* out320, int reset) {
  return guarded([&] {
    need(h, "etb_debug_diag");
    need(out320, "etb_debug_diag");
    ETB_CUDA(cudaSetDevice(h->device));
    etb::debug_diag(out320, reset != 0, h->stream);
  });
}

int etb_debug_phase_stamps(etb_layout* h, uint64_t* out256) {
  return guarded([&] {
    need(h, "etb_debug_phase_stamps");
    need(out256, "etb_debug_phase_stamps");
    ETB_CUDA(cudaMemcpyAsync(out256, h->S.level_claims.get() + 256, 256 * 8,
                             cudaMemcpyDeviceToHost, h->stream));
    ETB_CUDA(cudaStreamSynchronize(h->stream));
  });
}

int etb_debug_block_stamps(etb_layout* h, uint64_t start, uint64_t* out, uint64_t cap,
                           uint32_t* grid, uint32_t* levels) {
  return guarded([&] {
    need(h, "etb_debug_block_stamps");
    ETB_CUDA(cudaSetDevice(h->device));
    // partitioned layouts: CTA c belongs to partition c / (grid / partitions)
    const uint64_t g = static_cast<uint64_t>(h->P ? h->P->grid : h->S.grid);
    etb::DevBuf<unsigned long long> st(64 * g);
    ETB_CUDA(cudaMemsetAsync(st.get(), 0, 64 * g * 8, h->stream));
    run_bfs(h, start, nullptr, true, nullptr, st.get());
    uint64_t t0 = 0;
    uint32_t nl = 0;
    ETB_CUDA(cudaMemcpyAsync(&t0, h->S.level_claims.get() + 256, 8, cudaMemcpyDeviceToHost,
                             h->stream));
    ETB_CUDA(cudaMemcpyAsync(&nl, h->S.nlevels.get(), 4, cudaMemcpyDeviceToHost, h->stream));
    std::vector<uint64_t> hs(64 * g);
    ETB_CUDA(cudaMemcpyAsync(hs.data(), st.get(), 64 * g * 8, cudaMemcpyDeviceToHost, h->stream));
    ETB_CUDA(cudaStreamSynchronize(h->stream));
    for (uint64_t i = 0; i < std::min<uint64_t>(cap, 64 * g); ++i) out[i] = hs[i] ? hs[i] - t0 : 0;
    if (grid) *grid = static_cast<uint32_t>(g);
    if (levels) *levels = nl;
  });
}

int etb_debug_warp_stamps(etb_layout* h, uint64_t start, int32_t depth, uint64_t* out,
                          uint64_t cap, uint32_t* nwarps) {
  return guarded([&] {
    need(h, "etb_debug_warp_stamps");
    if (h->P) throw std::invalid_argument("etb_debug_warp_stamps: single-partition kernel only");
    ETB_CUDA(cudaSetDevice(h->device));
    const uint64_t nw = static_cast<uint64_t>(h->S.grid) * (h->S.block / 32);
    etb::DevBuf<unsigned long long> st(8 * nw);
    ETB_CUDA(cudaMemsetAsync(st.get(), 0, 8 * nw * 8, h->stream));
    run_bfs(h, start, nullptr, true, nullptr, nullptr, st.get(), depth);
    uint64_t t0 = 0;
    ETB_CUDA(cudaMemcpyAsync(&t0, h->S.level_claims.get() + 256, 8, cudaMemcpyDeviceToHost,
                             h->stream));
    std::vector<uint64_t> hs(8 * nw);
    ETB_CUDA(cudaMemcpyAsync(hs.data(), st.get(), 8 * nw * 8, cudaMemcpyDeviceToHost, h->stream));
    ETB_CUDA(cudaStreamSynchronize(h->stream));
    for (uint64_t w = 0; w < nw; ++w)
      if (hs[8 * w]) hs[8 * w] -= t0;
    std::copy(hs.begin(), hs.begin() + std::min<uint64_t>(cap, 8 * nw), out);
    if (nwarps) *nwarps = static_cast<uint32_t>(nw);
  });
}

int etb_debug_launch_floor(etb_layout* h, int iters, double* empty_us) {
  return guarded([&] {
    need(h, "etb_debug_launch_floor");
    need(empty_us, "etb_debug_launch_floor");
    ETB_CUDA(cudaSetDevice(h->device));
    std::vector<float> t;
    for (int i = 0; i < std::max(iters, 1) + 3; ++i) {
      ETB_CUDA(cudaEventRecord(h->ev[2], h->stream));
      etb::empty_launch(h->S, h->stream);
      ETB_CUDA(cudaEventRecord(h->ev[1], h->stream));
      ETB_CUDA(cudaEventSynchronize(h->ev[1]));
      float ms = 0.f;
      ETB_CUDA(cudaEventElapsedTime(&ms, h->ev[2], h->ev[1]));
      if (i >= 3) t.push_back(ms);
    }
    std::sort(t.begin(), t.end());
    *empty_us = t[t.size() / 2] * 1e3;
  });
}

int etb_layout_partition(etb_layout* h, uint32_t parts) {
  return guarded([&] {
    need(h, "etb_layout_partition");
    ETB_CUDA(cudaSetDevice(h->device));
    if (parts <= 1) {
      h->P.reset();
      return;
    }
    auto P = std::make_unique<etb::PartState>();
    etb::part_build(h->L, *P, parts, 0, parts, h->stream);
    h->P = std::move(P);
    h->system_scope = 0;
  });
}

int etb_layout_partition_scope(etb_layout* h, int system_scope) {
  return guarded([&] {
    need(h, "etb_layout_partition_scope");
    if (!h->P) throw std::invalid_argument("etb_layout_partition_scope: layout is not partitioned");
    h->system_scope = system_scope ? 1 : 0;
  });
}

int etb_layout_partition_owner(const etb_layout* h, uint32_t parts, uint32_t* owner) {
  return guarded([&] {
    need(h, "etb_layout_partition_owner");
    if (h->L.n) need(owner, "etb_layout_partition_owner");
    etb::part_owners(h->L, parts, owner);
  });
}

// Multi-process, one GPU per process. The blob a rank exports describes its
// partition's exchange block (frontier replicas + counters) by CUDA IPC handle.
struct MpBlob {
  cudaIpcMemHandle_t handle;
  uint64_t xbytes;
  uint64_t words;
  uint32_t rank, world;
};

int etb_mp_blob_size(void) { return static_cast<int>(sizeof(MpBlob)); }

int etb_mp_export(etb_layout* h, uint32_t world, uint32_t rank, void* blob_out) {
  return guarded([&] {
    need(h, "etb_mp_export");
    need(blob_out, "etb_mp_export");
    if (world < 2 || rank >= world) throw std::invalid_argument("etb_mp_export: bad rank/world");
    ETB_CUDA(cudaSetDevice(h->device));
    auto P = std::make_unique<etb::PartState>();
    etb::part_build(h->L, *P, world, rank, 1, h->stream);
    MpBlob b{};
    ETB_CUDA(cudaIpcGetMemHandle(&b.handle, P->xblock.get()));
    b.xbytes = P->xbytes;
    b.words = (h->L.nc + 31) / 32 + 1;
    b.rank = rank;
    b.world = world;
    std::memcpy(blob_out, &b, sizeof b);
    h->P = std::move(P);
    h->system_scope = 1;
  });
}

int etb_mp_connect(etb_layout* h, const void* blobs) {
  return guarded([&] {
    need(h, "etb_mp_connect");
    need(blobs, "etb_mp_connect");
    if (!h->P || h->P->local != 1) throw std::invalid_argument("etb_mp_connect: call etb_mp_export first");
    ETB_CUDA(cudaSetDevice(h->device));
    etb::PartState& P = *h->P;
    const MpBlob* all = static_cast<const MpBlob*>(blobs);
    for (uint32_t q = 0; q < P.nparts; ++q) {
      if (all[q].rank != q || all[q].world != P.nparts)
        throw std::invalid_argument("etb_mp_connect: blobs must be ordered by rank");
      if (q == P.first) continue;
      void* base = nullptr;
      ETB_CUDA(cudaIpcOpenMemHandle(&base, all[q].handle, cudaIpcMemLazyEnablePeerAccess));
      P.peer_maps.push_back(base);
      etb::PartDev& d = P.h_parts[q];
      const uint64_t words = all[q].words;
      d.fb0 = static_cast<uint32_t*>(base);
      d.fb1 = d.fb0 + words;
      d.fb2 = d.fb1 + words;
      d.ctr = reinterpret_cast<unsigned long long*>(static_cast<unsigned char*>(base) +
                                                    ((3 * words * 4 + 255) / 256) * 256);
      d.arrive = d.ctr + etb::kCtrWords;
    }
    ETB_CUDA(cudaMemcpyAsync(P.d_parts.get(), P.h_parts.data(), P.nparts * sizeof(etb::PartDev),
                             cudaMemcpyHostToDevice, h->stream));
    ETB_CUDA(cudaStreamSynchronize(h->stream));
  });
}

int etb_host_register(void* ptr, uint64_t bytes) {
  return guarded([&] {
    need(ptr, "etb_host_register");
    ETB_CUDA(cudaHostRegister(ptr, bytes, cudaHostRegisterDefault));
  });
}

int etb_host_unregister(void* ptr) {
  return guarded([&] {
    need(ptr, "etb_host_unregister");
    ETB_CUDA(cudaHostUnregister(ptr));
  });
}

int etb_time_roots(etb_layout* h, const uint64_t* starts, uint64_t count, int warmup,
                   int flush_l2, const etb_bfs_options* opts, double* ms_out,
                   double* kernel_ms_out) {
  return guarded([&] {
    need(h, "etb_time_roots");
    if (count) need(starts, "etb_time_roots");
    ETB_CUDA(cudaSetDevice(h->device));
    cudaStream_t s = h->stream;
    if (flush_l2 && !h->flush) {
      int l2 = 0;
      ETB_CUDA(cudaDeviceGetAttribute(&l2, cudaDevAttrL2CacheSize, h->device));
      h->flush.alloc(std::max<uint64_t>(uint64_t(l2) * 2, uint64_t{1} << 26));
    }
    for (int w = 0; w < warmup && count; ++w) run_bfs(h, starts[w % count], opts, false);
    ETB_CUDA(cudaStreamSynchronize(s));
    for (uint64_t i = 0; i < count; ++i) {
      // The flush (a 2x-L2 memset) runs while the host walks the start and
      // enqueues the traversal, so the events time the device work of the
      // per-root sequence (patch copy + kernel) on a stream that is fed ahead,
      // not the host's launch latency (the synchronous, wall-clock path is
      // what bench.py's e2e number measures).
      // With the persisting L2 window on, its lines are first demoted to
      // normal so that the flush evicts them too: every root starts cold.
      if (flush_l2 && h->S.l2_window && !getenv("ETB_KEEP_PERSIST"))
        ETB_CUDA(cudaCtxResetPersistingL2Cache());
      if (flush_l2) ETB_CUDA(cudaMemsetAsync(h->flush.get(), i & 0xFF, h->flush.size(), s));
      ETB_CUDA(cudaEventRecord(h->ev[0], s));
      // the pre-launch event only when kernel times are asked for: a third
      // event in the sequence adds its own ~2 us to the whole-call time
      run_bfs(h, starts[i], opts, false, kernel_ms_out ? h->ev[2] : nullptr);
      ETB_CUDA(cudaEventRecord(h->ev[1], s));
      ETB_CUDA(cudaEventSynchronize(h->ev[1]));
      float ms = 0.f, kms = 0.f;
      ETB_CUDA(cudaEventElapsedTime(&ms, h->ev[0], h->ev[1]));
      if (kernel_ms_out) ETB_CUDA(cudaEventElapsedTime(&kms, h->ev[2], h->ev[1]));
      if (ms_out) ms_out[i] = ms;
      if (kernel_ms_out) kernel_ms_out[i] = kms;
    }
  });
}

}  // extern "C"
