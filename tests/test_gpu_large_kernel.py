"""The large-core instantiation (1024 threads: list-less top-down levels claim
with reductions and count claims/scout afterwards, deferred-scout pass) forced
on graphs the oracle finishes in seconds (ETB_BFS_BLOCK=1024 at layout
creation; normally only cores of >= 2^23 vertices use it): depths bit-exact
against the oracle, parents valid, direction traces equal to the reference's
golden traces (the α/β decisions depend on the deferred claims and scout)."""
import ctypes as C

import numpy as np
import pytest

import oracle as O
import paper_2009_07463_b200 as eb
from paper_2009_07463_b200 import etbfs as E
from test_gpu_parity import check_root
from test_gpu_stress import CASES

pytestmark = pytest.mark.gpu


@pytest.fixture
def large_kernel(monkeypatch):
    monkeypatch.setenv("ETB_BFS_BLOCK", "1024")


def block_of(cg, start):
    nw = C.c_uint32()
    out = np.zeros(8 * 148 * 32, np.uint64)
    E._check(E.lib().etb_debug_warp_stamps(cg.handle, start, -1, out.ctypes.data, out.size,
                                            C.byref(nw)))
    return 32 * nw.value // 148 if nw.value % 148 == 0 else None


def test_s16_roots_and_traces(large_kernel, kron16):
    k = kron16
    csr = eb.generate_graph(scale=16, edgefactor=16, seed=1)
    ocsr = O.OracleCsr(1 << 16, O.oracle_generate(16, 16, 1))
    for mh in (-1, 0):
        cg = eb.relayout_csr(csr, mh=mh)
        assert block_of(cg, int(cg.old2new[k["roots"][0]])) == 1024
        traces = k["layout"][str(mh)]["traces"]
        for i, root in enumerate(k["roots"][:64]):
            r = check_root(cg, ocsr, int(root))
            assert r.stats.direction_trace == traces[i], (mh, root)
        # top-down only: every level list-less or listed, all through the 1024 kernel
        for root in k["roots"][:8]:
            check_root(cg, ocsr, int(root), kernel=eb.CoreKernel.TOP_DOWN)


@pytest.mark.parametrize("name,n,pairs", CASES, ids=[c[0] for c in CASES])
def test_extreme_shapes(large_kernel, name, n, pairs):
    g = eb.build_csr(n, pairs)
    oc = O.OracleCsr(n, pairs)
    cg = eb.relayout_csr(g, mh=-1)
    rng = np.random.default_rng(5)
    for root in [0, n - 1] + [int(x) for x in rng.integers(0, n, 2)]:
        check_root(cg, oc, root)
        E.bfs_device(cg, int(cg.old2new[root]))
        assert E.result_validate(cg, int(cg.old2new[root]))["passed"], (name, root)


@pytest.mark.parametrize("ratio,div", [("0.05", "4"), ("0.05", "64"), ("0.5", "1000000"), ("2", "1024"),
                                       ("0", "1024")])
def test_split_levels_s16(large_kernel, monkeypatch, kron16, ratio, div):
    """Split top-down levels (frontier hubs bottom-up with rows ended at an id
    bound, the other frontier vertices top-down from a filtered list) forced onto
    nearly every list-less level (a tiny ratio) with bounds from a quarter of the
    core down to the 32-vertex floor, at the default and switched off: depths
    against the oracle, parents valid, the reference's direction traces and
    traversed-edge counts."""
    monkeypatch.setenv("ETB_SPLIT_RATIO", ratio)
    monkeypatch.setenv("ETB_SPLIT_DIV", div)
    k = kron16
    csr = eb.generate_graph(scale=16, edgefactor=16, seed=1)
    ocsr = O.OracleCsr(1 << 16, O.oracle_generate(16, 16, 1))
    for mh in (-1, 0):
        cg = eb.relayout_csr(csr, mh=mh)
        traces = k["layout"][str(mh)]["traces"]
        for i, root in enumerate(k["roots"][:32]):
            r = check_root(cg, ocsr, int(root))
            assert r.stats.direction_trace == traces[i], (mh, root, ratio, div)
            s = int(cg.old2new[int(root)])
            E.bfs_device(cg, s)
            assert E.result_validate(cg, s)["passed"], (mh, root)
            assert E.result_traversed_edges(cg) == k["traversed_edges"][i]
        # the split path was taken: its bottom-up half leaves a phase stamp
        ph = np.zeros(256, np.uint64)
        E._check(E.lib().etb_debug_phase_stamps(cg.handle, ph.ctypes.data))
        if float(ratio) == 0.05:
            assert ph[64:128].any(), "no level ran split"
        if float(ratio) == 0:
            assert not ph[64:128].any()
