"""ctypes mirror of the reference ``etbfs`` API over the C-ABI (include/etbfs_cuda.h).

Reference interfaces mirrored (paths under /root/reference/proj/include/etbfs):
  generate_kronecker      kronecker.hpp:34        -> generate_kronecker()
  build_csr               build.hpp:19            -> build_csr()
  classify_vertices       classify.hpp:33         -> classify_vertices()
  compute_peak_height     classify.hpp:38         -> compute_peak_height()
  count_types             classify.hpp:40         -> count_types()
  relayout_csr            relayout.hpp:40         -> relayout_csr()
  extract_edge_tree_list  relayout.hpp:52         -> extract_edge_tree_list()
  et_bfs                  et_bfs.hpp:53           -> et_bfs()
  restricted_edge_count   bfs.hpp:123             -> EtLayout.restricted_edge_count
"""
from __future__ import annotations

import ctypes as C
import enum
import os
from dataclasses import dataclass, field

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
# ETB_LIB points at another build of the same library (A/B kernel experiments).
_LIB_PATH = os.environ.get("ETB_LIB") or os.path.join(HERE, "lib", "libetbfs_b200.so")

NO_VERTEX = np.uint64(0xFFFFFFFFFFFFFFFF)  # types.hpp:13 kNoVertex

ETB_OK, ETB_EINVAL, ETB_ERUNTIME, ETB_ECUDA, ETB_ENOTSUP = 0, -1, -2, -3, -4


class VertexType(enum.IntEnum):  # types.hpp:55-61
    CORE_INTERNAL = 0
    CORE_EDGE = 1
    TREE_INTERNAL = 2
    TREE_LEAF = 3
    VERTEX_ZERO = 4


class CoreKernel(enum.IntEnum):  # et_bfs.hpp:10-16
    TOP_DOWN = 0
    HYBRID = 1
    DEGREE_AWARE = 2
    BLOCK_SEARCH = 3
    HYBRID_BLOCK_SEARCH = 4


class TreeReplay(enum.IntEnum):  # et_bfs.hpp:19-22
    TEET = 0
    TEOLV = 1


@dataclass
class HybridPolicy:  # bfs.hpp:19-22
    alpha: float = 14.0
    beta: float = 24.0


@dataclass
class KroneckerParams:  # kronecker.hpp:12-20
    scale: int = 0
    edgefactor: int = 16
    a: float = 0.57
    b: float = 0.19
    c: float = 0.19
    d: float = 0.05
    seed: int = 0


@dataclass
class TypeCounts:  # classify.hpp:12-27
    core_internal: int = 0
    core_edge: int = 0
    tree_internal: int = 0
    tree_leaf: int = 0
    vertex_zero: int = 0

    def total(self):
        return self.core_internal + self.core_edge + self.tree_internal + self.tree_leaf + \
            self.vertex_zero

    def core(self):
        return self.core_internal + self.core_edge

    def tree(self):
        return self.tree_internal + self.tree_leaf


# ------------------------------------------------------------------ ctypes --
class _Kron(C.Structure):
    _fields_ = [("scale", C.c_uint32), ("edgefactor", C.c_uint64), ("a", C.c_double),
                ("b", C.c_double), ("c", C.c_double), ("d", C.c_double), ("seed", C.c_uint64)]


class _LayoutInfo(C.Structure):
    _fields_ = [("vertex_count", C.c_uint64), ("core_vertex_count", C.c_uint64),
                ("tree_vertex_count", C.c_uint64), ("isolated_count", C.c_uint64),
                ("core_directed_edges", C.c_uint64), ("directed_edges", C.c_uint64),
                ("tree_count", C.c_uint64), ("max_tree_size", C.c_uint64), ("mh", C.c_int64)]


class _BfsOptions(C.Structure):
    _fields_ = [("kernel", C.c_int), ("replay", C.c_int), ("alpha", C.c_double),
                ("beta", C.c_double)]


class _BfsStats(C.Structure):
    _fields_ = [("levels", C.c_uint32), ("bottom_up_levels", C.c_uint32),
                ("direction_trace", C.c_char * 256), ("level_claims", C.c_uint64 * 256),
                ("level_ns", C.c_uint64 * 256), ("total_ns", C.c_uint64)]


_lib = None


def lib_path() -> str:
    return _LIB_PATH


def lib() -> C.CDLL:
    """Load the sm_100a library; fails loudly (no fallback) when it is missing."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(_LIB_PATH):
        raise RuntimeError(f"{_LIB_PATH} is not built; run __graft_entry__.build() "
                           "(python paper_2009_07463_b200/build_lib.py)")
    L = C.CDLL(_LIB_PATH)
    vp, u64, i64, i32 = C.c_void_p, C.c_uint64, C.c_int64, C.c_int
    P64 = C.POINTER(C.c_uint64)

    def sig(name, *args):
        f = getattr(L, name)
        f.restype = i32
        f.argtypes = list(args)

    L.etb_last_error.restype = C.c_char_p
    L.etb_last_error.argtypes = []
    sig("etb_version")
    sig("etb_device_count", C.POINTER(C.c_int))
    sig("etb_set_device", C.c_int)
    sig("etb_generate_kronecker", C.POINTER(_Kron), vp)
    sig("etb_graph_from_edges", u64, vp, u64, C.POINTER(vp), P64, P64)
    sig("etb_graph_generate", C.POINTER(_Kron), C.POINTER(vp), P64, P64)
    sig("etb_graph_info", vp, P64, P64)
    sig("etb_graph_download", vp, vp, vp, vp)
    L.etb_graph_free.restype = None
    L.etb_graph_free.argtypes = [vp]
    sig("etb_classify", vp, i64, vp, vp)
    sig("etb_peak_height", vp, P64)
    sig("etb_layout_build", vp, i64, C.POINTER(vp))
    sig("etb_layout_build_types", vp, vp, i64, C.POINTER(vp))
    sig("etb_layout_info_get", vp, C.POINTER(_LayoutInfo))
    sig("etb_layout_download_maps", vp, vp, vp, vp)
    sig("etb_layout_download_graph", vp, vp, vp)
    sig("etb_layout_download_etl", vp, vp, vp, vp)
    sig("etb_layout_restricted_edges", vp, P64)
    L.etb_layout_free.restype = None
    L.etb_layout_free.argtypes = [vp]
    sig("etb_bfs_device", vp, u64, C.POINTER(_BfsOptions), C.POINTER(_BfsStats))
    sig("etb_bfs", vp, u64, C.POINTER(_BfsOptions), vp, vp, C.POINTER(_BfsStats))
    sig("etb_bfs_compact", vp, u64, C.POINTER(_BfsOptions), vp, vp)
    sig("etb_result_device_ptr", vp, C.POINTER(vp))
    sig("etb_result_download", vp, vp, vp)
    sig("etb_result_mark_assembled", vp)
    sig("etb_result_download_original", vp, vp, vp)
    sig("etb_result_traversed_edges", vp, P64)
    sig("etb_result_validate", vp, u64, vp)
    sig("etb_debug_phase_stamps", vp, vp)
    sig("etb_debug_diag", vp, vp, i32)
    sig("etb_debug_launch_floor", vp, i32, C.POINTER(C.c_double))
    sig("etb_debug_check_line", C.POINTER(C.c_uint32))
    sig("etb_debug_block_stamps", vp, u64, vp, u64, C.POINTER(C.c_uint32), C.POINTER(C.c_uint32))
    sig("etb_debug_warp_stamps", vp, u64, C.c_int32, vp, u64, C.POINTER(C.c_uint32))
    sig("etb_layout_partition", vp, C.c_uint32)
    sig("etb_layout_partition_owner", vp, C.c_uint32, vp)
    sig("etb_layout_partition_scope", vp, C.c_int)
    sig("etb_mp_blob_size")
    sig("etb_mp_export", vp, C.c_uint32, C.c_uint32, vp)
    sig("etb_mp_connect", vp, vp)
    sig("etb_host_register", vp, u64)
    sig("etb_host_unregister", vp)
    sig("etb_time_roots", vp, vp, u64, C.c_int, C.c_int, C.POINTER(_BfsOptions), vp, vp)
    sig("etb_time_roots_wall", vp, vp, u64, C.c_int, C.POINTER(_BfsOptions), vp)
    sig("etb_result_work", vp, u64, C.POINTER(_BfsOptions), vp, vp, C.POINTER(C.c_uint32),
        C.c_char_p, P64)
    sig("etb_graph_degree_split", vp, u64, vp, vp, vp)
    sig("etb_graph_levels", vp, u64, vp)
    sig("etb_graph_validate_tree", vp, u64, vp, vp, vp, vp)
    cp = C.c_char_p
    sig("etb_graph_file_read", cp, i32, C.POINTER(vp))
    sig("etb_graph_file_info", vp, P64, P64, C.POINTER(C.POINTER(C.c_uint64)))
    L.etb_graph_file_free.restype = None
    L.etb_graph_file_free.argtypes = [vp]
    sig("etb_graph_file_write", cp, i32, u64, vp, u64)
    sig("etb_graph_from_file", cp, i32, C.POINTER(vp))
    sig("etb_tree_file_write", cp, u64, u64, vp)
    sig("etb_tree_file_read", cp, P64, P64, vp, u64)
    _lib = L
    return L


def _check(rc: int):
    if rc == ETB_OK:
        return
    msg = lib().etb_last_error().decode()
    if rc == ETB_EINVAL:
        raise ValueError(msg)
    if rc == ETB_ENOTSUP:
        raise NotImplementedError(msg)
    raise RuntimeError(msg)


def _ptr(a):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


def _kron(p: KroneckerParams) -> _Kron:
    return _Kron(p.scale, p.edgefactor, p.a, p.b, p.c, p.d, p.seed)


def _opts(kernel, replay, policy) -> _BfsOptions:
    pol = policy or HybridPolicy()
    return _BfsOptions(int(kernel), int(replay), float(pol.alpha), float(pol.beta))


# ------------------------------------------------------------------- graph --
def generate_kronecker(params: KroneckerParams | None = None, **kw) -> np.ndarray:
    """generate_kronecker (kronecker.hpp:34) on the GPU: (T, 2) u64 (src, dst)."""
    p = params or KroneckerParams(**kw)
    t = (1 << p.scale) * p.edgefactor if p.scale <= 48 else 0
    out = np.empty((max(t, 1), 2), np.uint64)
    _check(lib().etb_generate_kronecker(C.byref(_kron(p)), _ptr(out)))
    return out[:t]


class Csr:
    """A CsrGraph (types.hpp:38-50) resident in HBM (original ids)."""

    def __init__(self, handle, n, nnz, self_loops=0, duplicates=0):
        self._h = handle
        self.vertex_count = n
        self.directed_edge_count = nnz
        self.dropped_self_loops = self_loops
        self.dropped_duplicates = duplicates

    def __del__(self):
        h = getattr(self, "_h", None)
        if h and _lib is not None:
            _lib.etb_graph_free(h)
            self._h = None

    @property
    def handle(self):
        return self._h

    def undirected_edge_count(self):
        return self.directed_edge_count // 2

    def degrees(self):
        """degrees u64[n] (types.hpp:43) without downloading the adjacency."""
        deg = np.empty(max(self.vertex_count, 1), np.uint64)
        _check(lib().etb_graph_download(self._h, None, None, _ptr(deg)))
        return deg[: self.vertex_count]

    def download(self):
        """(row_offsets u64[n+1], col_indices u64[nnz], degrees u64[n])."""
        n, m = self.vertex_count, self.directed_edge_count
        row = np.empty(n + 1, np.uint64)
        col = np.empty(max(m, 1), np.uint64)
        deg = np.empty(max(n, 1), np.uint64)
        _check(lib().etb_graph_download(self._h, _ptr(row), _ptr(col), _ptr(deg)))
        return row, col[:m], deg[:n]


def _finish_csr(h, sl, du) -> Csr:
    n, m = C.c_uint64(), C.c_uint64()
    _check(lib().etb_graph_info(h, C.byref(n), C.byref(m)))
    return Csr(h, n.value, m.value, sl.value, du.value)


def build_csr(vertex_count: int, pairs: np.ndarray) -> Csr:
    """build_csr (build.hpp:19): symmetric, deduplicated, self-loop free, on the GPU."""
    pairs = np.ascontiguousarray(pairs, dtype=np.uint64).reshape(-1, 2)
    h = C.c_void_p()
    sl, du = C.c_uint64(), C.c_uint64()
    _check(lib().etb_graph_from_edges(int(vertex_count), _ptr(pairs), pairs.shape[0],
                                      C.byref(h), C.byref(sl), C.byref(du)))
    return _finish_csr(h, sl, du)


def generate_graph(params: KroneckerParams | None = None, **kw) -> Csr:
    """generate_kronecker + build_csr fused on the device (tuples never leave HBM)."""
    p = params or KroneckerParams(**kw)
    h = C.c_void_p()
    sl, du = C.c_uint64(), C.c_uint64()
    _check(lib().etb_graph_generate(C.byref(_kron(p)), C.byref(h), C.byref(sl), C.byref(du)))
    return _finish_csr(h, sl, du)


# ------------------------------------------------------------ preprocessing --
def classify_vertices(g: Csr, mh: int) -> np.ndarray:
    """classify_vertices (classify.hpp:33): u8 VertexType per original id."""
    t = np.empty(max(g.vertex_count, 1), np.uint8)
    _check(lib().etb_classify(g.handle, int(mh), _ptr(t), None))
    return t[: g.vertex_count]


def compute_peak_height(g: Csr) -> int:
    """compute_peak_height (classify.hpp:38), exact Gauss-Seidel emulation."""
    ph = C.c_uint64()
    _check(lib().etb_peak_height(g.handle, C.byref(ph)))
    return ph.value


def count_types(types) -> TypeCounts:
    """count_types (classify.hpp:40)."""
    c = np.bincount(np.asarray(types, np.uint8), minlength=5)
    return TypeCounts(*[int(x) for x in c[:5]])


class EtLayout:
    """A ClassifiedGraph (types.hpp:69-76) + its EdgeTreeList, BFS-ready in HBM."""

    def __init__(self, handle, graph=None):
        self._h = handle
        self._graph = graph  # the device CSR must outlive the layout (graph(), validate)
        info = _LayoutInfo()
        _check(lib().etb_layout_info_get(handle, C.byref(info)))
        self.vertex_count = info.vertex_count
        self.core_vertex_count = info.core_vertex_count
        self.tree_vertex_count = info.tree_vertex_count
        self.isolated_count = info.isolated_count
        self.restricted_edge_count = info.core_directed_edges
        self.directed_edge_count = info.directed_edges
        self.tree_count = info.tree_count
        self.max_tree_size = info.max_tree_size
        self.mh = info.mh
        self._maps = None

    def __del__(self):
        h = getattr(self, "_h", None)
        if h and _lib is not None:
            _lib.etb_layout_free(h)
            self._h = None

    @property
    def handle(self):
        return self._h

    def _load_maps(self):
        if self._maps is None:
            n = self.vertex_count
            a = np.empty(max(n, 1), np.uint64)
            b = np.empty(max(n, 1), np.uint64)
            t = np.empty(max(n, 1), np.uint8)
            _check(lib().etb_layout_download_maps(self._h, _ptr(a), _ptr(b), _ptr(t)))
            self._maps = (a[:n], b[:n], t[:n])
        return self._maps

    @property
    def new2old(self):
        return self._load_maps()[0]

    @property
    def old2new(self):
        return self._load_maps()[1]

    @property
    def vertex_type(self):
        return self._load_maps()[2]

    def graph(self):
        """The relabelled CsrGraph: (row_offsets, col_indices) u64."""
        n, m = self.vertex_count, self.directed_edge_count
        row = np.empty(n + 1, np.uint64)
        col = np.empty(max(m, 1), np.uint64)
        _check(lib().etb_layout_download_graph(self._h, _ptr(row), _ptr(col)))
        return row, col[:m]


def partition(cg: "EtLayout", parts: int, system_scope: bool = False) -> None:
    """Run subsequent traversals of cg with the 1D core partition (parts >= 2) on
    this device, or back on the single-partition kernel (parts <= 1).
    system_scope runs the exchange with the multi-GPU (system-scope) fences,
    atomics and polls."""
    _check(lib().etb_layout_partition(cg.handle, int(parts)))
    if parts > 1 and system_scope:
        _check(lib().etb_layout_partition_scope(cg.handle, 1))


def partition_owner(cg: "EtLayout", parts: int) -> np.ndarray:
    """u32[n]: the partition owning each relaid vertex (bfs_part.cuh rule)."""
    o = np.empty(max(cg.vertex_count, 1), np.uint32)
    _check(lib().etb_layout_partition_owner(cg.handle, int(parts), _ptr(o)))
    return o[: cg.vertex_count]


def relayout_csr(g: Csr, types=None, mh: int = -1) -> EtLayout:
    """relayout_csr (relayout.hpp:40). types=None classifies on the device first."""
    h = C.c_void_p()
    if types is None:
        _check(lib().etb_layout_build(g.handle, int(mh), C.byref(h)))
    else:
        t = np.ascontiguousarray(types, np.uint8)
        if t.size != g.vertex_count:
            raise ValueError("relayout_csr: types length does not match vertex count")
        _check(lib().etb_layout_build_types(g.handle, _ptr(t), int(mh), C.byref(h)))
    return EtLayout(h, g)


def extract_edge_tree_list(cg: EtLayout):
    """extract_edge_tree_list (relayout.hpp:52): (src, dst, core_edge) u64 arrays."""
    m = cg.tree_vertex_count
    s, d, c = (np.empty(max(m, 1), np.uint64) for _ in range(3))
    _check(lib().etb_layout_download_etl(cg.handle, _ptr(s), _ptr(d), _ptr(c)))
    return s[:m], d[:m], c[:m]


# ---------------------------------------------------------------- traversal --
@dataclass
class BfsStats:  # bfs.hpp:27-33 KernelStats
    levels: int = 0
    bottom_up_levels: int = 0
    direction_trace: str = ""
    level_claims: list = field(default_factory=list)
    level_ns: list = field(default_factory=list)  # [init end, level 0 end, ...] from entry
    total_ns: int = 0


@dataclass
class BfsResult:  # types.hpp:96-99 BfsTree (+ the device's exact depth array)
    root: int
    parent: np.ndarray   # u64, relaid ids, NO_VERTEX unreached
    depth: np.ndarray    # i32, -1 unreached
    stats: BfsStats | None = None


def et_bfs(cg: EtLayout, start: int, kernel=CoreKernel.HYBRID, replay=TreeReplay.TEET,
           policy: HybridPolicy | None = None, stats: bool = False,
           want_parent: bool = True, want_depth: bool = True) -> BfsResult:
    """et_bfs (et_bfs.hpp:53) on the GPU; results in relaid ids."""
    n = cg.vertex_count
    depth = np.empty(max(n, 1), np.int32) if want_depth else None
    parent = np.empty(max(n, 1), np.uint64) if want_parent else None
    st = _BfsStats() if stats else None
    o = _opts(kernel, replay, policy)
    _check(lib().etb_bfs(cg.handle, int(start), C.byref(o), _ptr(depth), _ptr(parent),
                         C.byref(st) if st is not None else None))
    bs = None
    if st is not None:
        bs = BfsStats(st.levels, st.bottom_up_levels, st.direction_trace.decode(),
                      list(st.level_claims[: st.levels]), list(st.level_ns[: st.levels + 1]),
                      st.total_ns)
    return BfsResult(int(start), parent[:n] if parent is not None else None,
                     depth[:n] if depth is not None else None, bs)


def bfs_device(cg: EtLayout, start: int, kernel=CoreKernel.HYBRID, replay=TreeReplay.TEET,
               policy: HybridPolicy | None = None) -> None:
    """et_bfs leaving depth/parent in HBM (the timed hot path)."""
    o = _opts(kernel, replay, policy)
    _check(lib().etb_bfs_device(cg.handle, int(start), C.byref(o), None))


def result_download(cg: EtLayout, depth: np.ndarray | None = None,
                    parent: np.ndarray | None = None):
    """Last result as compact i32 depth / u32 parent (UINT32_MAX unreached)."""
    n = cg.vertex_count
    if depth is None:
        depth = np.empty(max(n, 1), np.int32)
    if parent is None:
        parent = np.empty(max(n, 1), np.uint32)
    _check(lib().etb_result_download(cg.handle, _ptr(depth), _ptr(parent)))
    return depth[:n], parent[:n]


def result_original(cg: EtLayout, levels: bool = True, parent: bool = True):
    """Last result in original ids (translate_tree + tree_levels): (levels u64,
    parent u64), NO_VERTEX for unreached; either None when not asked for."""
    n = cg.vertex_count
    lv = np.empty(max(n, 1), np.uint64) if levels else None
    pa = np.empty(max(n, 1), np.uint64) if parent else None
    _check(lib().etb_result_download_original(cg.handle, _ptr(lv), _ptr(pa)))
    return (lv[:n] if lv is not None else None), (pa[:n] if pa is not None else None)


def result_validate(cg: EtLayout, start: int) -> dict:
    """validate_bfs_tree rules 1-5 on the device for the last result."""
    c = np.zeros(6, np.uint64)
    _check(lib().etb_result_validate(cg.handle, int(start), _ptr(c)))
    return {"rule1": int(c[0]), "rule2": int(c[1]), "rule3": int(c[2]), "rule4": int(c[3]),
            "rule5": int(c[4]), "reached": int(c[5]),
            "passed": bool((c[:5] == 0).all())}


def result_traversed_edges(cg: EtLayout) -> int:
    te = C.c_uint64()
    _check(lib().etb_result_traversed_edges(cg.handle, C.byref(te)))
    return te.value


def time_roots(cg: EtLayout, starts, warmup=3, flush_l2=True, kernel=CoreKernel.HYBRID,
               replay=TreeReplay.TEET, policy: HybridPolicy | None = None,
               kernel_times: bool = True):
    """Per-root CUDA-event times (ms): (whole call incl. start-side walk, kernel only).
    kernel_times=False leaves out the pre-launch event (kernel times None): the
    whole-call times then carry no third event."""
    s = np.ascontiguousarray(starts, np.uint64)
    ms = np.empty(max(s.size, 1), np.float64)
    kms = np.empty(max(s.size, 1), np.float64) if kernel_times else None
    o = _opts(kernel, replay, policy)
    _check(lib().etb_time_roots(cg.handle, _ptr(s), s.size, int(warmup), int(bool(flush_l2)),
                                C.byref(o), _ptr(ms), _ptr(kms)))
    return ms[: s.size], (kms[: s.size] if kms is not None else None)


def time_roots_wall(cg: EtLayout, starts, warmup=3, kernel=CoreKernel.HYBRID,
                    replay=TreeReplay.TEET, policy: HybridPolicy | None = None):
    """Per-root wall-clock ms of etb_bfs_device + stream synchronise (launch latency
    and the start-side walk included; no L2 flush, no host copy)."""
    s = np.ascontiguousarray(starts, np.uint64)
    ms = np.empty(max(s.size, 1), np.float64)
    o = _opts(kernel, replay, policy)
    _check(lib().etb_time_roots_wall(cg.handle, _ptr(s), s.size, int(warmup), C.byref(o), _ptr(ms)))
    return ms[: s.size]


@dataclass
class Work:
    """Algorithmic work of one traversal (etb_result_work, csrc/work.cu)."""
    trace: str
    levels: np.ndarray   # (nl, 4): frontier-or-unvisited, columns read, claims, BU misses
    bytes: np.ndarray    # (nl + 1,): per level, then replay / fill / reset
    total_bytes: int


def result_work(cg: EtLayout, start: int, kernel=CoreKernel.HYBRID, replay=TreeReplay.TEET,
                policy: HybridPolicy | None = None) -> Work:
    lv = np.zeros(4 * 64, np.uint64)
    by = np.zeros(65, np.uint64)
    nl = C.c_uint32()
    tr = C.create_string_buffer(66)
    tot = C.c_uint64()
    o = _opts(kernel, replay, policy)
    _check(lib().etb_result_work(cg.handle, int(start), C.byref(o), _ptr(lv), _ptr(by),
                                 C.byref(nl), tr, C.byref(tot)))
    k = nl.value
    return Work(tr.value.decode(), lv[: 4 * k].reshape(k, 4), by[: k + 1], tot.value)


def device_count() -> int:
    c = C.c_int()
    _check(lib().etb_device_count(C.byref(c)))
    return c.value


# ---- graph and parent-tree files (io.hpp:9-45) ---------------------------------
GRAPH_FORMATS = {"binary": 0, "text": 1}  # GraphFormat (io.hpp:11)


def parse_graph_format(name: str) -> str:
    """parse_graph_format (io.hpp:44): "binary" / "text", else ValueError."""
    if name not in GRAPH_FORMATS:
        raise ValueError(f'unknown graph format "{name}" (binary or text)')
    return name


def write_graph(path: str, vertex_count: int, pairs: np.ndarray, fmt: str = "binary") -> None:
    """write_graph (io.hpp:23): ETG1 or text, byte-identical to the reference."""
    pairs = np.ascontiguousarray(pairs, dtype=np.uint64).reshape(-1, 2)
    _check(lib().etb_graph_file_write(os.fsencode(path), GRAPH_FORMATS[parse_graph_format(fmt)],
                                      int(vertex_count), _ptr(pairs), pairs.shape[0]))


def read_graph(path: str, fmt: str = "binary"):
    """read_graph (io.hpp:24) -> (vertex_count, pairs u64[m, 2]); RuntimeError names
    the path and the byte offset or line, as the reference's."""
    h = C.c_void_p()
    _check(lib().etb_graph_file_read(os.fsencode(path), GRAPH_FORMATS[parse_graph_format(fmt)],
                                     C.byref(h)))
    try:
        n, m = C.c_uint64(), C.c_uint64()
        p = C.POINTER(C.c_uint64)()
        _check(lib().etb_graph_file_info(h, C.byref(n), C.byref(m), C.byref(p)))
        pairs = (np.ctypeslib.as_array(p, shape=(2 * m.value,)).copy() if m.value
                 else np.empty(0, np.uint64))
        return n.value, pairs.reshape(-1, 2)
    finally:
        lib().etb_graph_file_free(h)


def build_csr_from_file(path: str, fmt: str = "binary") -> Csr:
    """read_graph + build_csr with the tuples going straight to the device."""
    h = C.c_void_p()
    _check(lib().etb_graph_from_file(os.fsencode(path), GRAPH_FORMATS[parse_graph_format(fmt)],
                                     C.byref(h)))
    return _finish_csr(h, C.c_uint64(0), C.c_uint64(0))


def write_tree(path: str, root: int, parent: np.ndarray) -> None:
    """write_tree (io.hpp:30): ETT1 {n, root, parent u64[n]} (kNoVertex unreached)."""
    parent = np.ascontiguousarray(parent, dtype=np.uint64)
    _check(lib().etb_tree_file_write(os.fsencode(path), parent.size, int(root), _ptr(parent)))


def read_tree(path: str):
    """read_tree (io.hpp:31) -> (root, parent u64[n])."""
    n, root = C.c_uint64(), C.c_uint64()
    _check(lib().etb_tree_file_read(os.fsencode(path), C.byref(n), C.byref(root), None, 0))
    parent = np.empty(n.value, np.uint64)
    _check(lib().etb_tree_file_read(os.fsencode(path), C.byref(n), C.byref(root), _ptr(parent),
                                    n.value))
    return root.value, parent


# ---- checker-side helpers on a device graph (preprocess.hpp / validate.hpp) ----
def split_degree_aware(g: Csr, neighbor_limit: int | None = None):
    """split_degree_aware (preprocess.hpp:69) on the GPU -> (in_plus u64[n],
    minus_offsets u64[n+1], minus_cols u64[...]); None keeps every neighbour."""
    lim = 0xFFFFFFFFFFFFFFFF if neighbor_limit is None else int(neighbor_limit)
    n = g.vertex_count
    moff = np.empty(n + 1, np.uint64)
    _check(lib().etb_graph_degree_split(g.handle, lim, None, _ptr(moff), None))
    in_plus = np.empty(max(n, 1), np.uint64)
    minus = np.empty(max(int(moff[n]), 1), np.uint64)
    _check(lib().etb_graph_degree_split(g.handle, lim, _ptr(in_plus), _ptr(moff), _ptr(minus)))
    return in_plus[:n], moff, minus[: int(moff[n])]


def oracle_bfs(g: Csr, root: int) -> np.ndarray:
    """oracle_bfs (validate.hpp:37): BFS levels (u64, NO_VERTEX unreached) from an
    independent level-synchronous device BFS."""
    lv = np.empty(max(g.vertex_count, 1), np.uint64)
    _check(lib().etb_graph_levels(g.handle, int(root), _ptr(lv)))
    return lv[: g.vertex_count]


RULE_MESSAGES = {1: "root is not its own parent", 4: "edge spans more than one level"}


def validate_bfs_tree(g: Csr, root: int, parent: np.ndarray) -> dict:
    """validate_bfs_tree (validate.hpp:46) of a parent array in g's ids, on the GPU:
    {passed, rule_counts[1..5], reached_count, traversed_edge_count, failures}."""
    parent = np.ascontiguousarray(parent, np.uint64)
    if parent.size != g.vertex_count:
        raise ValueError("validate_bfs_tree: tree does not match graph vertex count")
    counts = np.zeros(8, np.uint64)
    where = np.zeros(125, np.uint64)
    first = np.zeros(5, np.uint32)
    _check(lib().etb_graph_validate_tree(g.handle, int(root), _ptr(parent), _ptr(counts),
                                         _ptr(where), _ptr(first)))
    failures = []
    for r in range(1, 6):
        for i in range(int(first[r - 1])):
            failures.append((r, int(where[(r - 1) * 25 + i])))
    return {"passed": bool(counts[0]), "rule_counts": [int(x) for x in counts[1:6]],
            "reached_count": int(counts[6]), "traversed_edge_count": int(counts[7]),
            "failures": failures}
