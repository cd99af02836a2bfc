"""GPU tree validation (validate_bfs_tree rules 1-5 on the device) — the
size-independent property used for parity at BASELINE's full sizes: a tree that
passes rules 1-5 has exact BFS depths. Checked against the oracle at s16, run on
every root at s22 and s26, and shown to reject each class of corrupted tree
(restating the reference's mutation corpus idea, proj/tests/acceptance.cpp:557-670)."""
import numpy as np
import pytest
import torch

import oracle as O
import paper_2009_07463_b200 as eb
from paper_2009_07463_b200 import etbfs as E
from bench import select_roots_from_degrees

pytestmark = pytest.mark.gpu


class _DevArray:
    """Zero-copy view of the layout's result array {depth, parent} via
    __cuda_array_interface__ (test-only fault injection)."""

    def __init__(self, ptr, n):
        self.__cuda_array_interface__ = {"shape": (n, 2), "typestr": "<i4", "data": (ptr, False),
                                         "version": 3}


def result_tensor(cg):
    import ctypes as C
    p = C.c_void_p()
    E._check(E.lib().etb_result_device_ptr(cg.handle, C.byref(p)))
    return torch.as_tensor(_DevArray(p.value, cg.vertex_count), device="cuda")


def test_validator_accepts_exact_trees_s16(kron16):
    g = eb.generate_graph(scale=16, edgefactor=16, seed=1)
    cg = eb.relayout_csr(g, mh=-1)
    for root, te in zip(kron16["roots"], kron16["traversed_edges"]):
        s = int(cg.old2new[root])
        E.bfs_device(cg, s)
        v = E.result_validate(cg, s)
        assert v["passed"], (root, v)
        assert E.result_traversed_edges(cg) == te


def test_validator_rejects_each_fault_class(kron16):
    g = eb.generate_graph(scale=16, edgefactor=16, seed=1)
    cg = eb.relayout_csr(g, mh=-1)
    s = int(cg.old2new[kron16["roots"][0]])
    rng = np.random.default_rng(3)

    def fresh():
        E.bfs_device(cg, s)
        torch.cuda.synchronize()
        return result_tensor(cg)

    dp = fresh()
    reached = torch.nonzero((dp[:, 0] >= 0)
                            & (torch.arange(dp.shape[0], device="cuda") != s)).flatten()
    v = int(reached[rng.integers(0, reached.numel())])
    # rule 1: root not its own parent
    dp = fresh()
    dp[s, 1] = v
    assert E.result_validate(cg, s)["rule1"] > 0
    # rule 3: a parent that is not a neighbour (the root itself is far from most vertices)
    dp = fresh()
    far = int(torch.nonzero(dp[:, 0] == dp[:, 0].max()).flatten()[0])
    dp[far, 1] = s
    out = E.result_validate(cg, s)
    assert out["rule3"] > 0 or out["rule2"] > 0
    # rule 2/4: a depth off by one
    dp = fresh()
    dp[v, 0] += 2
    out = E.result_validate(cg, s)
    assert out["rule2"] > 0 and out["rule4"] > 0
    # rule 5: a reached vertex dropped from the tree
    dp = fresh()
    dp[v, 0] = -1
    dp[v, 1] = -1
    assert E.result_validate(cg, s)["rule5"] > 0
    assert E.result_validate(cg, s)["passed"] is False
    assert E.result_validate(cg, s)["reached"] >= 1


@pytest.mark.slow
@pytest.mark.parametrize("scale,nroots", [(22, 64), (26, 64)])
def test_all_roots_valid_at_full_size(scale, nroots):
    g = eb.generate_graph(scale=scale, edgefactor=16, seed=1)
    cg = eb.relayout_csr(g, mh=-1)
    roots = select_roots_from_degrees(g.degrees(), 64, 1)[:nroots]
    for r in roots:
        s = int(cg.old2new[int(r)])
        E.bfs_device(cg, s)
        v = E.result_validate(cg, s)
        assert v["passed"], (int(r), v)
