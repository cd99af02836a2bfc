"""Host-output calls (etb_bfs, etb_bfs_compact, etb_result_download): only the
live prefix [0, core + tree) of the relaid id space is copied device->host, the
isolated range is filled by the host. Every output array is checked against the
interleaved device result fetched whole (etb_result_device_ptr), from
garbage-filled host buffers, for core, tree and isolated starts."""
import ctypes as C

import numpy as np
import pytest
import torch

import paper_2009_07463_b200 as eb
from paper_2009_07463_b200 import etbfs as E

pytestmark = pytest.mark.gpu


class _DevArray:
    """An (n, 2) i32 view of the device result through __cuda_array_interface__."""

    def __init__(self, ptr, n):
        self.__cuda_array_interface__ = {"shape": (n, 2), "typestr": "<i4", "data": (ptr, False),
                                         "version": 3}


def device_result(cg):
    """The whole {depth, parent} result as the kernels left it in HBM."""
    p = C.c_void_p()
    E._check(E.lib().etb_result_device_ptr(cg.handle, C.byref(p)))
    t = torch.as_tensor(_DevArray(p.value, cg.vertex_count), device="cuda").cpu().numpy()
    return t[:, 0].copy(), t[:, 1].copy().view(np.uint32)


@pytest.mark.parametrize("scale,ef,mh", [(10, 2, -1), (14, 16, -1), (14, 4, 0)])
def test_host_outputs_equal_device_result(scale, ef, mh):
    g = eb.generate_graph(scale=scale, edgefactor=ef, seed=3)
    cg = eb.relayout_csr(g, mh=mh)
    n, nc, nt = cg.vertex_count, cg.core_vertex_count, cg.tree_vertex_count
    assert nc + nt < n, "the case needs isolated vertices"
    starts = [0, nc - 1, nc, nc + nt - 1, nc + nt, n - 1, nc // 2, nc + nt // 2, nc + nt + 1, 1]
    opt = E._opts(E.CoreKernel.HYBRID, E.TreeReplay.TEET, None)
    for s in starts:
        depth = np.full(n, 0x5A5A5A5A, np.int32)
        par64 = np.full(n, 0xABABABABABABABAB, np.uint64)
        E._check(E.lib().etb_bfs(cg.handle, int(s), C.byref(opt), depth.ctypes.data,
                                 par64.ctypes.data, None))
        want_d, want_p = device_result(cg)
        assert want_d[s] == 0 and want_p[s] == s
        assert (depth == want_d).all(), s
        assert (par64 == np.where(want_p == 0xFFFFFFFF, np.uint64(E.NO_VERTEX),
                                  want_p.astype(np.uint64))).all(), s
        d2 = np.full(n, 0x11111111, np.int32)
        p2 = np.full(n, 0x22222222, np.uint32)
        E._check(E.lib().etb_bfs_compact(cg.handle, int(s), C.byref(opt), d2.ctypes.data,
                                         p2.ctypes.data))
        want_d, want_p = device_result(cg)  # a rerun may pick other (equally valid) parents
        assert (d2 == want_d).all() and (p2 == want_p).all(), s
        d3 = np.full(n, 0x33333333, np.int32)
        p3 = np.full(n, 0x44444444, np.uint32)
        d3, p3 = E.result_download(cg, d3, p3)
        assert (d3 == want_d).all() and (p3 == want_p).all(), s
        # parent only, as the e2e bench line calls it
        p4 = np.full(n, 0x55555555, np.uint32)
        E._check(E.lib().etb_bfs_compact(cg.handle, int(s), C.byref(opt), None, p4.ctypes.data))
        assert (p4 == device_result(cg)[1]).all(), s


def test_large_isolated_range_is_filled_by_every_thread():
    """A tail long enough (> 4 MB per thread) to take the threaded fill."""
    g = eb.generate_graph(scale=22, edgefactor=2, seed=1)
    cg = eb.relayout_csr(g, mh=-1)
    n, live = cg.vertex_count, cg.core_vertex_count + cg.tree_vertex_count
    assert (n - live) * 4 > 8 << 20
    opt = E._opts(E.CoreKernel.HYBRID, E.TreeReplay.TEET, None)
    for s in (0, live, n - 1):
        p = np.full(n, 0x66666666, np.uint32)
        d = np.full(n, 0x77777777, np.int32)
        E._check(E.lib().etb_bfs_compact(cg.handle, int(s), C.byref(opt), d.ctypes.data,
                                         p.ctypes.data))
        want_d, want_p = device_result(cg)
        assert (d == want_d).all() and (p == want_p).all(), s
