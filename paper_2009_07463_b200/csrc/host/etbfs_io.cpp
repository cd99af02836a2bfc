// Graph and parent-tree files behind the C-ABI (include/etbfs_cuda.h) and the
// C++ drop-in (include/etbfs/io.hpp). Formats, validation order and error
// messages follow the reference (proj/src/io.cpp:47-181, documented in
// proj/include/etbfs/io.hpp:9-45); the implementation is bulk I/O: whole-file
// reads and one buffered write, little-endian words moved with memcpy (the
// reference streams 8 bytes per call), so a scale-28 edge list (69 GB) is
// bounded by the disk, not by per-element stream calls.
#include <algorithm>
#include <charconv>
#include <cstdio>
#include <cstring>
#include <memory>
#include <new>
#include <stdexcept>
#include <string>
#include <string_view>
#include <vector>

#include "etbfs/io.hpp"
#include "etbfs_cuda.h"

namespace etb {
void set_last_error(const char* msg);  // capi.cu
}

namespace {

constexpr uint64_t kMaxVertices = uint64_t{1} << 48;  // types.hpp kMaxVertexCount
constexpr char kGraphMagic[4] = {'E', 'T', 'G', '1'};
constexpr char kTreeMagic[4] = {'E', 'T', 'T', '1'};
static_assert(__BYTE_ORDER__ == __ORDER_LITTLE_ENDIAN__, "files are little endian");

[[noreturn]] void at_offset(const std::string& path, uint64_t off, const std::string& what) {
  throw std::runtime_error(path + ": " + what + " (byte offset " + std::to_string(off) + ")");
}
[[noreturn]] void at_line(const std::string& path, uint64_t line, const std::string& what) {
  throw std::runtime_error(path + ": " + what + " (line " + std::to_string(line) + ")");
}

struct File {
  std::FILE* f = nullptr;
  ~File() {
    if (f) std::fclose(f);
  }
};

std::vector<char> slurp(const std::string& path) {
  File in{std::fopen(path.c_str(), "rb")};
  if (!in.f) throw std::runtime_error(path + ": cannot open for reading");
  std::vector<char> buf;
  std::fseek(in.f, 0, SEEK_END);
  const long sz = std::ftell(in.f);
  std::fseek(in.f, 0, SEEK_SET);
  buf.resize(sz > 0 ? static_cast<size_t>(sz) : 0);
  if (!buf.empty() && std::fread(buf.data(), 1, buf.size(), in.f) != buf.size())
    throw std::runtime_error(path + ": read failed");
  return buf;
}

// Sequential writer with one large buffer.
struct Out {
  std::string path;
  File out;
  std::vector<char> buf;
  explicit Out(const std::string& p, bool binary) : path(p) {
    out.f = std::fopen(p.c_str(), binary ? "wb" : "w");
    if (!out.f) throw std::runtime_error(p + ": cannot open for writing");
    buf.reserve(size_t{1} << 22);
  }
  void flush() {
    if (!buf.empty() && std::fwrite(buf.data(), 1, buf.size(), out.f) != buf.size())
      throw std::runtime_error(path + ": write failed");
    buf.clear();
  }
  void put(const void* p, size_t n) {
    if (buf.size() + n > buf.capacity()) flush();
    if (n > buf.capacity()) {
      if (std::fwrite(p, 1, n, out.f) != n) throw std::runtime_error(path + ": write failed");
      return;
    }
    buf.insert(buf.end(), static_cast<const char*>(p), static_cast<const char*>(p) + n);
  }
  void u64(uint64_t v) { put(&v, 8); }
  void close() {
    flush();
    if (std::fflush(out.f) != 0 || std::ferror(out.f)) throw std::runtime_error(path + ": write failed");
  }
};

uint64_t get_u64(const std::vector<char>& b, uint64_t& off, const std::string& path) {
  if (b.size() < off + 8) at_offset(path, off, "unexpected end of file");
  uint64_t v;
  std::memcpy(&v, b.data() + off, 8);
  off += 8;
  return v;
}

uint64_t parse_u64(std::string_view tok, const std::string& path, uint64_t line) {
  uint64_t v = 0;
  const auto [ptr, ec] = std::from_chars(tok.data(), tok.data() + tok.size(), v);
  if (ec != std::errc{} || ptr != tok.data() + tok.size())
    at_line(path, line, "expected an unsigned integer, got \"" + std::string(tok) + "\"");
  return v;
}

}  // namespace

// A loaded edge list: vertex count + interleaved (src, dst) pairs.
struct etb_edgefile {
  uint64_t vertex_count = 0;
  std::vector<uint64_t> pairs;
};

namespace etb::io {

void read_graph(const std::string& path, int format, etb_edgefile& out) {
  if (format == ETB_FORMAT_BINARY) {
    const std::vector<char> b = slurp(path);
    if (b.size() < 4 || std::memcmp(b.data(), kGraphMagic, 4) != 0)
      at_offset(path, 0, "bad magic, expected ETG1");
    uint64_t off = 4;
    out.vertex_count = get_u64(b, off, path);
    if (out.vertex_count > kMaxVertices)
      at_offset(path, off - 8, "vertex count exceeds the supported maximum");
    const uint64_t m = get_u64(b, off, path);
    if (b.size() < off || (b.size() - off) / 16 < m)
      at_offset(path, off, "file too short for declared edge count");
    out.pairs.resize(2 * m);
    if (m) std::memcpy(out.pairs.data(), b.data() + off, 16 * m);
    const uint64_t n = out.vertex_count;
    for (uint64_t i = 0; i < m; ++i)  // first offending record, as the reference reports it
      if (out.pairs[2 * i] >= n || out.pairs[2 * i + 1] >= n)
        at_offset(path, off + 16 * i, "edge endpoint out of range");
    return;
  }
  if (format != ETB_FORMAT_TEXT) throw std::invalid_argument("unknown graph format");
  const std::vector<char> b = slurp(path);
  bool declared = false;
  uint64_t inferred = 0, line_no = 0;
  out.vertex_count = 0;
  out.pairs.clear();
  std::string_view all(b.data(), b.size());
  while (!all.empty()) {
    const size_t nl = all.find('\n');
    std::string_view view = all.substr(0, nl);
    all = nl == std::string_view::npos ? std::string_view{} : all.substr(nl + 1);
    ++line_no;
    while (!view.empty() && (view.back() == '\r' || view.back() == ' ')) view.remove_suffix(1);
    while (!view.empty() && view.front() == ' ') view.remove_prefix(1);
    if (view.empty()) continue;
    if (view.front() == '#') {
      constexpr std::string_view kHeader = "# vertices ";
      if (view.substr(0, kHeader.size()) == kHeader) {
        out.vertex_count = parse_u64(view.substr(kHeader.size()), path, line_no);
        declared = true;
      }
      continue;
    }
    const size_t sp = view.find(' ');
    if (sp == std::string_view::npos) at_line(path, line_no, "expected \"src dst\"");
    const uint64_t src = parse_u64(view.substr(0, sp), path, line_no);
    std::string_view rest = view.substr(sp + 1);
    while (!rest.empty() && rest.front() == ' ') rest.remove_prefix(1);
    const uint64_t dst = parse_u64(rest, path, line_no);
    if (declared && (src >= out.vertex_count || dst >= out.vertex_count))
      at_line(path, line_no, "edge endpoint out of range");
    inferred = std::max({inferred, src + 1, dst + 1});
    out.pairs.push_back(src);
    out.pairs.push_back(dst);
  }
  if (!declared) out.vertex_count = inferred;
  if (out.vertex_count > kMaxVertices)
    at_line(path, line_no, "vertex count exceeds the supported maximum");
}

void write_graph(const std::string& path, int format, uint64_t n, const uint64_t* pairs,
                 uint64_t m) {
  if (format == ETB_FORMAT_BINARY) {
    Out o(path, true);
    o.put(kGraphMagic, 4);
    o.u64(n);
    o.u64(m);
    if (m) o.put(pairs, 16 * m);
    o.close();
    return;
  }
  if (format != ETB_FORMAT_TEXT) throw std::invalid_argument("unknown graph format");
  Out o(path, false);
  char line[64];
  const int h = std::snprintf(line, sizeof line, "# vertices %llu\n",
                              static_cast<unsigned long long>(n));
  o.put(line, static_cast<size_t>(h));
  for (uint64_t i = 0; i < m; ++i) {
    char* p = line;
    p = std::to_chars(p, line + 30, pairs[2 * i]).ptr;
    *p++ = ' ';
    p = std::to_chars(p, line + 62, pairs[2 * i + 1]).ptr;
    *p++ = '\n';
    o.put(line, static_cast<size_t>(p - line));
  }
  o.close();
}

void write_tree(const std::string& path, uint64_t n, uint64_t root, const uint64_t* parent) {
  Out o(path, true);
  o.put(kTreeMagic, 4);
  o.u64(n);
  o.u64(root);
  if (n) o.put(parent, 8 * n);
  o.close();
}

// parent == nullptr: sizes only.
void read_tree(const std::string& path, uint64_t* n_out, uint64_t* root_out, uint64_t* parent,
               uint64_t cap) {
  const std::vector<char> b = slurp(path);
  if (b.size() < 4 || std::memcmp(b.data(), kTreeMagic, 4) != 0)
    at_offset(path, 0, "bad magic, expected ETT1");
  uint64_t off = 4;
  const uint64_t n = get_u64(b, off, path);
  if (n > kMaxVertices) at_offset(path, off - 8, "vertex count exceeds the supported maximum");
  const uint64_t root = get_u64(b, off, path);
  if (n > 0 && root >= n) at_offset(path, off - 8, "root out of range");
  if (b.size() - off < 8 * n) {  // the reference fails on the first missing slot
    const uint64_t whole = (b.size() - off) / 8;
    at_offset(path, off + 8 * whole, "unexpected end of file");
  }
  if (n_out) *n_out = n;
  if (root_out) *root_out = root;
  if (!parent) return;
  if (cap < n) throw std::invalid_argument("etb_tree_file_read: parent buffer too small");
  if (n) std::memcpy(parent, b.data() + off, 8 * n);
}

}  // namespace etb::io

namespace {

template <typename F>
int io_guarded(F&& f) {
  try {
    f();
    return ETB_OK;
  } catch (const std::invalid_argument& e) {
    etb::set_last_error(e.what());
    return ETB_EINVAL;
  } catch (const std::bad_alloc&) {
    etb::set_last_error("out of host memory");
    return ETB_ERUNTIME;
  } catch (const std::exception& e) {
    etb::set_last_error(e.what());
    return ETB_ERUNTIME;
  }
}

void need(const void* p, const char* what) {
  if (!p) throw std::invalid_argument(std::string(what) + ": null argument");
}

}  // namespace

extern "C" {

int etb_graph_file_read(const char* path, int format, etb_edgefile** out) {
  return io_guarded([&] {
    need(path, "etb_graph_file_read");
    need(out, "etb_graph_file_read");
    auto f = std::make_unique<etb_edgefile>();
    etb::io::read_graph(path, format, *f);
    *out = f.release();
  });
}

int etb_graph_file_info(const etb_edgefile* f, uint64_t* vertex_count, uint64_t* edge_count,
                        const uint64_t** pairs) {
  return io_guarded([&] {
    need(f, "etb_graph_file_info");
    if (vertex_count) *vertex_count = f->vertex_count;
    if (edge_count) *edge_count = f->pairs.size() / 2;
    if (pairs) *pairs = f->pairs.data();
  });
}

void etb_graph_file_free(etb_edgefile* f) { delete f; }

int etb_graph_file_write(const char* path, int format, uint64_t vertex_count,
                         const uint64_t* pairs, uint64_t edge_count) {
  return io_guarded([&] {
    need(path, "etb_graph_file_write");
    if (edge_count) need(pairs, "etb_graph_file_write");
    etb::io::write_graph(path, format, vertex_count, pairs, edge_count);
  });
}

int etb_tree_file_write(const char* path, uint64_t vertex_count, uint64_t root,
                        const uint64_t* parent) {
  return io_guarded([&] {
    need(path, "etb_tree_file_write");
    if (vertex_count) need(parent, "etb_tree_file_write");
    etb::io::write_tree(path, vertex_count, root, parent);
  });
}

int etb_tree_file_read(const char* path, uint64_t* vertex_count, uint64_t* root,
                       uint64_t* parent, uint64_t cap) {
  return io_guarded([&] {
    need(path, "etb_tree_file_read");
    etb::io::read_tree(path, vertex_count, root, parent, cap);
  });
}

int etb_graph_from_file(const char* path, int format, etb_graph** out) {
  etb_edgefile* f = nullptr;
  int rc = etb_graph_file_read(path, format, &f);
  if (rc != ETB_OK) return rc;
  rc = etb_graph_from_edges(f->vertex_count, f->pairs.data(), f->pairs.size() / 2, out, nullptr,
                            nullptr);
  etb_graph_file_free(f);
  return rc;
}

}  // extern "C"

// ---- C++ drop-in (include/etbfs/io.hpp) ---------------------------------------
namespace etbfs {

namespace {
int fmt(GraphFormat f) { return f == GraphFormat::kBinary ? ETB_FORMAT_BINARY : ETB_FORMAT_TEXT; }
}  // namespace

void write_graph(const std::string& path, const EdgeList& edges, GraphFormat format) {
  static_assert(sizeof(Edge) == 16, "Edge is two u64");
  etb::io::write_graph(path, fmt(format), edges.vertex_count,
                       reinterpret_cast<const uint64_t*>(edges.edges.data()), edges.edges.size());
}

EdgeList read_graph(const std::string& path, GraphFormat format) {
  etb_edgefile f;
  etb::io::read_graph(path, fmt(format), f);
  EdgeList out;
  out.vertex_count = f.vertex_count;
  out.edges.resize(f.pairs.size() / 2);
  for (size_t i = 0; i < out.edges.size(); ++i)
    out.edges[i] = Edge{f.pairs[2 * i], f.pairs[2 * i + 1]};
  return out;
}

void write_tree(const std::string& path, const BfsTree& tree) {
  etb::io::write_tree(path, tree.parent.size(), tree.root, tree.parent.data());
}

BfsTree read_tree(const std::string& path) {
  BfsTree t;
  uint64_t n = 0, root = 0;
  etb::io::read_tree(path, &n, &root, nullptr, 0);
  t.parent.resize(n);
  etb::io::read_tree(path, &n, &root, t.parent.data(), n);
  t.root = root;
  return t;
}

GraphFormat parse_graph_format(const std::string& name) {
  if (name == "binary") return GraphFormat::kBinary;
  if (name == "text") return GraphFormat::kText;
  throw std::invalid_argument("unknown graph format \"" + name + "\" (binary or text)");
}

}  // namespace etbfs
