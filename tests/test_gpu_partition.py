"""GPU parity of the 1D core partition: the partitioned kernel
run with G partitions on one device (the multi-GPU algorithm, peer exchange in
local memory) must give the oracle's depths and valid parents, the reference's
α/β traces, and the same traversed-edge counts as the single-partition kernel."""
import numpy as np
import pytest

import oracle as O
import paper_2009_07463_b200 as eb
from conftest import edges_of
from paper_2009_07463_b200 import etbfs as E
from paper_2009_07463_b200.multi import partition_owner
from test_gpu_parity import check_root

pytestmark = pytest.mark.gpu


def test_owner_matches_host_rule(kron16):
    cg = eb.relayout_csr(eb.generate_graph(scale=16, edgefactor=16, seed=1), mh=-1)
    _, _, ce = eb.extract_edge_tree_list(cg)
    anchor = np.where(ce == O.NO_VERTEX, np.uint64(0xFFFFFFFF), ce)
    for parts in (1, 2, 3, 8, 16):
        want = partition_owner(cg.core_vertex_count, cg.tree_vertex_count, cg.vertex_count,
                               anchor, parts)
        assert (E.partition_owner(cg, parts) == want).all(), parts


def test_partitioned_corpus_all_starts(corpus):
    for g in corpus:
        csr = eb.build_csr(g["n"], edges_of(g))
        ocsr = O.OracleCsr(g["n"], edges_of(g))
        for mh in (-1, 0):
            cg = eb.relayout_csr(csr, mh=mh)
            for parts in (2, 3, 5):
                E.partition(cg, parts, system_scope=parts == 3)
                for st in range(g["n"]):
                    root = int(cg.new2old[st])
                    check_root(cg, ocsr, root)
                    check_root(cg, ocsr, root, kernel=eb.CoreKernel.TOP_DOWN)
            E.partition(cg, 1)


@pytest.mark.parametrize("parts,sys_scope", [(2, False), (4, False), (8, False), (2, True),
                                            (8, True)])
def test_partitioned_s16_64_roots(kron16, parts, sys_scope):
    """sys_scope: the multi-GPU code path (system-scope fences, counter atomics
    and barrier polls, as between GPUs over NVLink) run by the one-launch
    emulation, so it executes without kernels waiting on other launches."""
    k = kron16
    csr = eb.generate_graph(scale=16, edgefactor=16, seed=1)
    ocsr = O.OracleCsr(1 << 16, O.oracle_generate(16, 16, 1))
    cg = eb.relayout_csr(csr, mh=-1)
    E.partition(cg, parts, system_scope=sys_scope)
    for i, root in enumerate(k["roots"]):
        r = check_root(cg, ocsr, int(root))
        assert r.stats.direction_trace == k["layout"]["-1"]["traces"][i]
    E.bfs_device(cg, int(cg.old2new[k["roots"][0]]))
    assert E.result_traversed_edges(cg) == k["traversed_edges"][0]


@pytest.mark.slow
def test_partitioned_s22(kron_big):
    k = [x for x in kron_big if x["scale"] == 22][0]
    csr = eb.generate_graph(scale=22, edgefactor=16, seed=1)
    ocsr = O.OracleCsr(1 << 22, O.oracle_generate(22, 16, 1))
    cg = eb.relayout_csr(csr, mh=-1)
    E.partition(cg, 8)
    for root, te in zip(k["roots"][:4], k["traversed_edges"]):
        check_root(cg, ocsr, int(root))
        E.bfs_device(cg, int(cg.old2new[root]))
        assert E.result_traversed_edges(cg) == te
    starts = cg.old2new[np.array(k["roots"][:8], np.int64)]
    ms, kms = E.time_roots(cg, starts, warmup=2, flush_l2=True)
    assert (kms > 0).all()
