"""TEST INFRASTRUCTURE ONLY — the CPU checker, never the product.

ctypes wrappers over
  * ``liboracle.so``        — our plain-C restatement (oracle/etbfs_oracle.c), and
  * ``_ref/libetbfs_ref.so``— the unmodified reference sources compiled from
                              /root/reference/proj (oracle/Makefile, ``make ref``)
                              plus the marshalling shim oracle/ref_shim.cpp.

Only tests/, ``__graft_entry__.smoke()`` and bench.py's cpu-baseline / reference
arm may import this package.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libetbfs_ref.so")
REF_SRC = "/root/reference/proj"

NO_VERTEX = np.uint64(0xFFFFFFFFFFFFFFFF)
U64P = np.ctypeslib.ndpointer(np.uint64, flags="C_CONTIGUOUS")
U8P = np.ctypeslib.ndpointer(np.uint8, flags="C_CONTIGUOUS")
F64P = np.ctypeslib.ndpointer(np.float64, flags="C_CONTIGUOUS")
I32P = np.ctypeslib.ndpointer(np.int32, flags="C_CONTIGUOUS")

CORE_INTERNAL, CORE_EDGE, TREE_INTERNAL, TREE_LEAF, VERTEX_ZERO = range(5)


def build(ref: bool | None = None) -> None:
    """Compile liboracle.so (always) and, when the reference tree is present,
    oracle/_ref/libetbfs_ref.so. Building the checker is not using it."""
    subprocess.run(["make", "-s", "-C", HERE, "all"], check=True)
    if ref is None:
        ref = os.path.isdir(REF_SRC)
    if ref:
        subprocess.run(["make", "-s", "-j8", "-C", HERE, "ref"], check=True)


_orc = None
_ref = None


def _sig(f, res, *args):
    f.restype = res
    f.argtypes = list(args)


def orc() -> C.CDLL:
    global _orc
    if _orc is None:
        if not os.path.exists(ORACLE_SO):
            build(ref=False)
        L = C.CDLL(ORACLE_SO)
        vp, u64, i64, u32, d = C.c_void_p, C.c_uint64, C.c_int64, C.c_uint32, C.c_double
        _sig(L.orc_last_error, C.c_char_p)
        _sig(L.orc_generate_kronecker, C.c_int, u32, u64, d, d, d, d, u64, U64P)
        _sig(L.orc_build_csr, vp, u64, U64P, u64, C.POINTER(u64), C.POINTER(u64))
        _sig(L.orc_csr_free, None, vp)
        _sig(L.orc_csr_n, u64, vp)
        _sig(L.orc_csr_nnz, u64, vp)
        _sig(L.orc_csr_copy, None, vp, U64P, U64P)
        _sig(L.orc_classify, i64, vp, i64, U8P)
        _sig(L.orc_relayout, vp, vp, U8P, i64)
        _sig(L.orc_cg_free, None, vp)
        _sig(L.orc_cg_core, u64, vp)
        _sig(L.orc_cg_nnz, u64, vp)
        _sig(L.orc_cg_graph, vp, vp)
        _sig(L.orc_cg_copy, None, vp, U64P, U8P, U64P, U64P)
        _sig(L.orc_extract_etl, i64, vp, vp, vp, vp)
        _sig(L.orc_restricted_edge_count, u64, vp, u64)
        _sig(L.orc_bfs_levels, C.c_int, vp, u64, U64P)
        _sig(L.orc_select_roots, C.c_int, vp, u64, u64, U64P)
        _sig(L.orc_traversed_edges, u64, vp, U64P)
        _sig(L.orc_check_tree, u64, vp, u64, U64P, U64P)
        _sig(L.orc_fnv1a64, u64, vp, u64)
        _sig(L.orc_hybrid_trace, i64, vp, u64, u64, d, d, C.c_char_p, u64)
        _orc = L
    return _orc


def ref_available() -> bool:
    return os.path.exists(REF_SO)


def ref() -> C.CDLL:
    global _ref
    if _ref is None:
        if not os.path.exists(REF_SO):
            raise RuntimeError(f"{REF_SO} not built (needs /root/reference; run `make -C oracle ref`)")
        L = C.CDLL(REF_SO)
        vp, u64, i64, u32, d = C.c_void_p, C.c_uint64, C.c_int64, C.c_uint32, C.c_double
        _sig(L.ref_last_error, C.c_char_p)
        cp = C.c_char_p
        _sig(L.ref_write_graph, C.c_int, cp, C.c_int, u64, vp, u64)
        _sig(L.ref_split_degree_aware, C.c_int, vp, u64, vp, vp, vp)
        _sig(L.ref_validate_report, C.c_int, vp, u64, vp, vp, vp)
        _sig(L.ref_read_graph, C.c_int, cp, C.c_int, C.POINTER(u64), C.POINTER(u64), vp)
        _sig(L.ref_write_tree, C.c_int, cp, u64, u64, vp)
        _sig(L.ref_read_tree, C.c_int, cp, C.POINTER(u64), C.POINTER(u64), vp)
        _sig(L.ref_set_threads, None, C.c_int)
        _sig(L.ref_generate_kronecker, C.c_int, u32, u64, d, d, d, d, u64, U64P)
        _sig(L.ref_build_csr, vp, u64, U64P, u64, C.POINTER(u64), C.POINTER(u64))
        _sig(L.ref_csr_nnz, u64, vp)
        _sig(L.ref_csr_n, u64, vp)
        _sig(L.ref_csr_copy, None, vp, vp, vp)
        _sig(L.ref_csr_free, None, vp)
        _sig(L.ref_csr_alloc, vp, u64, u64, C.POINTER(vp), C.POINTER(vp), C.POINTER(vp))
        _sig(L.ref_classify, C.c_int, vp, i64, U8P)
        _sig(L.ref_peak_height, i64, vp)
        _sig(L.ref_prepare, vp, vp, i64)
        _sig(L.ref_prep_core, u64, vp)
        _sig(L.ref_prep_etl_size, u64, vp)
        _sig(L.ref_prep_nnz, u64, vp)
        _sig(L.ref_prep_restricted_edges, u64, vp)
        _sig(L.ref_prep_copy, None, vp, vp, vp, vp, vp, vp, vp, vp)
        _sig(L.ref_prep_free, None, vp)
        _sig(L.ref_et_bfs, d, vp, u64, C.c_int, C.c_int, d, d, vp, C.c_char_p, u64)
        _sig(L.ref_bfs_hybrid, C.c_int, vp, u64, d, d, vp, C.c_char_p, u64)
        _sig(L.ref_oracle_bfs, C.c_int, vp, u64, U64P)
        _sig(L.ref_validate, C.c_int, vp, u64, U64P, C.POINTER(u64), C.POINTER(C.c_int))
        _sig(L.ref_select_roots, C.c_int, vp, u64, u64, U64P)
        _sig(L.ref_fnv1a64, u64, vp, u64)
        _sig(L.ref_kron_csr, vp, u32, u64, u64, C.POINTER(u64), C.POINTER(u64), C.POINTER(u64))
        _sig(L.ref_csr_fnv, None, vp, U64P)
        _sig(L.ref_prep_fnv, None, vp, U64P)
        _sig(L.ref_prep_from_arrays, vp, u64, u64, i64, vp, vp, vp, vp, u64, vp, vp, vp)
        _sig(L.ref_run_benchmark, C.c_int, u32, u64, u64, C.c_int, i64, C.c_int, u64, u64, u64,
             U64P, F64P, U64P, I32P, C.POINTER(d), C.POINTER(d))
        _ref = L
    return _ref


def _ptr(a):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


# --------------------------------------------------------------- restatement
def fnv1a64(arr: np.ndarray) -> str:
    """FNV-1a-64 over the array's little-endian bytes."""
    a = np.ascontiguousarray(arr)
    return format(orc().orc_fnv1a64(a.ctypes.data_as(C.c_void_p), a.nbytes), "016x")


class OracleCsr:
    """A CSR built by the C restatement (build.cpp:21-87)."""

    def __init__(self, n: int, pairs: np.ndarray):
        L = orc()
        pairs = np.ascontiguousarray(pairs, dtype=np.uint64).reshape(-1)
        sl, du = C.c_uint64(), C.c_uint64()
        self.h = L.orc_build_csr(n, pairs, pairs.size // 2, C.byref(sl), C.byref(du))
        if not self.h:
            raise ValueError(L.orc_last_error().decode())
        self.n = n
        self.self_loops, self.duplicates = sl.value, du.value
        self._owned = True

    @classmethod
    def _wrap(cls, h, n):
        o = cls.__new__(cls)
        o.h, o.n, o._owned = h, n, False
        o.self_loops = o.duplicates = 0
        return o

    def __del__(self):
        if getattr(self, "_owned", False) and self.h:
            orc().orc_csr_free(self.h)
            self.h = None

    @property
    def nnz(self) -> int:
        return orc().orc_csr_nnz(self.h)

    def arrays(self):
        row = np.empty(self.n + 1, np.uint64)
        col = np.empty(max(self.nnz, 1), np.uint64)
        orc().orc_csr_copy(self.h, row, col)
        return row, col[: self.nnz]

    def degrees(self):
        row, _ = self.arrays()
        return np.diff(row)

    def classify(self, mh: int):
        t = np.empty(max(self.n, 1), np.uint8)
        rounds = orc().orc_classify(self.h, mh, t)
        if rounds < 0:
            raise ValueError(orc().orc_last_error().decode())
        return t[: self.n], rounds

    def levels(self, root: int):
        lv = np.empty(self.n, np.uint64)
        if orc().orc_bfs_levels(self.h, root, lv) != 0:
            raise ValueError(orc().orc_last_error().decode())
        return lv

    def select_roots(self, count: int, seed: int):
        out = np.empty(count, np.uint64)
        if orc().orc_select_roots(self.h, count, seed, out) != 0:
            raise RuntimeError(orc().orc_last_error().decode())
        return out

    def traversed_edges(self, levels):
        return orc().orc_traversed_edges(self.h, np.ascontiguousarray(levels, np.uint64))

    def check_tree(self, root, parent, levels) -> int:
        return orc().orc_check_tree(self.h, root, np.ascontiguousarray(parent, np.uint64),
                                    np.ascontiguousarray(levels, np.uint64))

    def restricted_edge_count(self, limit):
        return orc().orc_restricted_edge_count(self.h, limit)

    def hybrid_trace(self, limit, start, alpha=14.0, beta=24.0) -> str:
        buf = C.create_string_buffer(4096)
        r = orc().orc_hybrid_trace(self.h, limit, start, alpha, beta, buf, 4096)
        if r < 0:
            raise ValueError(orc().orc_last_error().decode())
        return buf.value.decode()


class OracleLayout:
    """relayout_csr + extract_edge_tree_list by the C restatement."""

    def __init__(self, csr: OracleCsr, mh: int, types=None):
        L = orc()
        if types is None:
            types, _ = csr.classify(mh)
        self.h = L.orc_relayout(csr.h, np.ascontiguousarray(types, np.uint8), mh)
        self.n = csr.n
        self.core = L.orc_cg_core(self.h)
        self.graph = OracleCsr._wrap(L.orc_cg_graph(self.h), self.n)

    def __del__(self):
        if getattr(self, "h", None):
            orc().orc_cg_free(self.h)
            self.h = None

    def arrays(self):
        n = self.n
        new2old = np.empty(max(n, 1), np.uint64)
        types = np.empty(max(n, 1), np.uint8)
        nnz = orc().orc_cg_nnz(self.h)
        row = np.empty(n + 1, np.uint64)
        col = np.empty(max(nnz, 1), np.uint64)
        orc().orc_cg_copy(self.h, new2old, types, row, col)
        return new2old[:n], types[:n], row, col[:nnz]

    def etl(self):
        L = orc()
        cnt = L.orc_extract_etl(self.h, None, None, None)
        if cnt < 0:
            raise RuntimeError(L.orc_last_error().decode())
        s = np.empty(max(cnt, 1), np.uint64)
        d = np.empty(max(cnt, 1), np.uint64)
        c = np.empty(max(cnt, 1), np.uint64)
        L.orc_extract_etl(self.h, _ptr(s), _ptr(d), _ptr(c))
        return s[:cnt], d[:cnt], c[:cnt]


def oracle_generate(scale, ef=16, seed=1, a=0.57, b=0.19, c=0.19, d=0.05) -> np.ndarray:
    t = (1 << scale) * ef
    out = np.empty(2 * t, np.uint64)
    if orc().orc_generate_kronecker(scale, ef, a, b, c, d, seed, out) != 0:
        raise ValueError(orc().orc_last_error().decode())
    return out.reshape(-1, 2)


# ------------------------------------------------------------------ reference
class RefCsr:
    """A CSR built by the compiled reference (etbfs_ref::build_csr)."""

    def __init__(self, n: int, pairs: np.ndarray):
        L = ref()
        pairs = np.ascontiguousarray(pairs, dtype=np.uint64).reshape(-1)
        sl, du = C.c_uint64(), C.c_uint64()
        self.h = L.ref_build_csr(n, pairs, pairs.size // 2, C.byref(sl), C.byref(du))
        if not self.h:
            raise ValueError(L.ref_last_error().decode())
        self.n = n
        self.self_loops, self.duplicates = sl.value, du.value

    @classmethod
    def kronecker(cls, scale, ef=16, seed=1):
        """generate_kronecker -> build_csr inside the reference library, tuples freed
        before returning (the lean path: scale 26 fits a 62 GB host)."""
        L = ref()
        fnv, sl, du = C.c_uint64(), C.c_uint64(), C.c_uint64()
        h = L.ref_kron_csr(scale, ef, seed, C.byref(fnv), C.byref(sl), C.byref(du))
        if not h:
            raise ValueError(L.ref_last_error().decode())
        o = cls.__new__(cls)
        o.h, o.n = h, 1 << scale
        o.self_loops, o.duplicates, o.tuples_fnv = sl.value, du.value, format(fnv.value, "016x")
        return o

    def fnv(self):
        out = np.zeros(2, np.uint64)
        ref().ref_csr_fnv(self.h, out)
        return [format(int(x), "016x") for x in out]

    def degrees(self):
        row = np.empty(self.n + 1, np.uint64)
        ref().ref_csr_copy(self.h, _ptr(row), None)
        return np.diff(row)

    def __del__(self):
        if getattr(self, "h", None):
            ref().ref_csr_free(self.h)
            self.h = None

    @property
    def nnz(self):
        return ref().ref_csr_nnz(self.h)

    def arrays(self):
        row = np.empty(self.n + 1, np.uint64)
        col = np.empty(max(self.nnz, 1), np.uint64)
        ref().ref_csr_copy(self.h, _ptr(row), _ptr(col))
        return row, col[: self.nnz]

    def classify(self, mh):
        t = np.empty(max(self.n, 1), np.uint8)
        if ref().ref_classify(self.h, mh, t) != 0:
            raise ValueError(ref().ref_last_error().decode())
        return t[: self.n]

    def peak_height(self):
        return ref().ref_peak_height(self.h)

    def levels(self, root):
        lv = np.empty(self.n, np.uint64)
        if ref().ref_oracle_bfs(self.h, root, lv) != 0:
            raise ValueError(ref().ref_last_error().decode())
        return lv

    def select_roots(self, count, seed):
        out = np.empty(count, np.uint64)
        if ref().ref_select_roots(self.h, count, seed, out) != 0:
            raise RuntimeError(ref().ref_last_error().decode())
        return out

    def validate(self, root, parent):
        te, rule = C.c_uint64(), C.c_int()
        r = ref().ref_validate(self.h, root, np.ascontiguousarray(parent, np.uint64),
                               C.byref(te), C.byref(rule))
        if r < 0:
            raise ValueError(ref().ref_last_error().decode())
        return bool(r), te.value, rule.value

    def bfs_hybrid(self, root, alpha=14.0, beta=24.0):
        par = np.empty(self.n, np.uint64)
        buf = C.create_string_buffer(4096)
        if ref().ref_bfs_hybrid(self.h, root, alpha, beta, _ptr(par), buf, 4096) != 0:
            raise ValueError(ref().ref_last_error().decode())
        return par, buf.value.decode()


class RefPrepared:
    """relayout_csr(classify_vertices(g, mh)) + extract_edge_tree_list by the reference."""

    def __init__(self, csr: RefCsr, mh: int):
        L = ref()
        self.h = L.ref_prepare(csr.h, mh)
        if not self.h:
            raise RuntimeError(L.ref_last_error().decode())
        self.n = csr.n
        self.core = L.ref_prep_core(self.h)
        self.etl_size = L.ref_prep_etl_size(self.h)
        self.restricted_edges = L.ref_prep_restricted_edges(self.h)

    @classmethod
    def from_arrays(cls, n, core, mh, new2old, types, row, col, etl_src, etl_dst, etl_ce):
        """Wrap a layout produced elsewhere (byte-identical to the reference's, as the
        parity tests pin) as the reference's ClassifiedGraph + EdgeTreeList."""
        L = ref()
        keep = [np.ascontiguousarray(a, dt) for a, dt in
                ((new2old, np.uint64), (types, np.uint8), (row, np.uint64), (col, np.uint64),
                 (etl_src, np.uint64), (etl_dst, np.uint64), (etl_ce, np.uint64))]
        h = L.ref_prep_from_arrays(n, core, mh, *[_ptr(a) for a in keep[:4]], len(keep[4]),
                                   *[_ptr(a) for a in keep[4:]])
        if not h:
            raise RuntimeError(L.ref_last_error().decode())
        o = cls.__new__(cls)
        o.h, o.n, o.core, o.etl_size = h, n, core, len(keep[4])
        o.restricted_edges = L.ref_prep_restricted_edges(h)
        return o

    def fnv(self):
        out = np.zeros(4, np.uint64)
        ref().ref_prep_fnv(self.h, out)
        return [format(int(x), "016x") for x in out]

    def __del__(self):
        if getattr(self, "h", None):
            ref().ref_prep_free(self.h)
            self.h = None

    def arrays(self):
        n, m = self.n, self.etl_size
        nnz = ref().ref_prep_nnz(self.h)
        new2old = np.empty(max(n, 1), np.uint64)
        types = np.empty(max(n, 1), np.uint8)
        row = np.empty(n + 1, np.uint64)
        col = np.empty(max(nnz, 1), np.uint64)
        s = np.empty(max(m, 1), np.uint64)
        d = np.empty(max(m, 1), np.uint64)
        c = np.empty(max(m, 1), np.uint64)
        ref().ref_prep_copy(self.h, _ptr(new2old), _ptr(types), _ptr(row), _ptr(col),
                            _ptr(s), _ptr(d), _ptr(c))
        return dict(new2old=new2old[:n], types=types[:n], row=row, col=col[:nnz],
                    etl_src=s[:m], etl_dst=d[:m], etl_ce=c[:m])

    def et_bfs(self, start, kernel=1, replay=0, alpha=14.0, beta=24.0, want_parent=True):
        par = np.empty(self.n, np.uint64) if want_parent else None
        buf = C.create_string_buffer(4096)
        s = ref().ref_et_bfs(self.h, start, kernel, replay, alpha, beta, _ptr(par), buf, 4096)
        if s < 0:
            raise ValueError(ref().ref_last_error().decode())
        return par, buf.value.decode(), s


def ref_generate(scale, ef=16, seed=1, a=0.57, b=0.19, c=0.19, d=0.05) -> np.ndarray:
    t = (1 << scale) * ef
    out = np.empty(2 * t, np.uint64)
    if ref().ref_generate_kronecker(scale, ef, a, b, c, d, seed, out) != 0:
        raise ValueError(ref().ref_last_error().decode())
    return out.reshape(-1, 2)
