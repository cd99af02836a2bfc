"""B200-native edge-tree BFS (arXiv 2009.07463) — Python host mirror.

The product is the sm_100a shared library ``lib/libetbfs_b200.so`` behind the
C-ABI in ``include/etbfs_cuda.h``; this package is a thin ctypes mirror of the
reference's public C++ API (``/root/reference/proj/include/etbfs/*.hpp``) with
the same function names, argument meaning and error behaviour
(``std::invalid_argument`` -> ``ValueError``, ``std::runtime_error`` ->
``RuntimeError``). There is no CPU fallback: if the library is missing or no
GPU is present, every compute call raises.
"""
from .etbfs import (  # noqa: F401
    BfsResult,
    BfsStats,
    CoreKernel,
    Csr,
    EtLayout,
    HybridPolicy,
    KroneckerParams,
    TreeReplay,
    TypeCounts,
    VertexType,
    build_csr,
    build_csr_from_file,
    classify_vertices,
    compute_peak_height,
    count_types,
    et_bfs,
    extract_edge_tree_list,
    generate_graph,
    generate_kronecker,
    lib,
    parse_graph_format,
    read_graph,
    read_tree,
    write_graph,
    write_tree,
    lib_path,
    relayout_csr,
)

__all__ = [n for n in dir() if not n.startswith("_")]
