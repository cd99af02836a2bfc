"""Checker-side and preprocessing helpers on the GPU (csrc/graph_tools.cu) against
the compiled reference: split_degree_aware (proj/src/preprocess.cpp:16-60),
oracle_bfs (validate.cpp:77-91) and validate_bfs_tree (validate.cpp:95-158) on
correct and corrupted trees (the mutation classes of proj/tests/acceptance.cpp:
557-670, restated)."""
import numpy as np
import pytest

import oracle as O
import paper_2009_07463_b200 as eb
from conftest import edges_of
from paper_2009_07463_b200 import etbfs as E

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built")]
NO = np.uint64(0xFFFFFFFFFFFFFFFF)


def ref_split(rc, n, limit):
    R = O.ref()
    moff = np.empty(n + 1, np.uint64)
    assert R.ref_split_degree_aware(rc.h, limit, None, moff.ctypes.data, None) == 0
    in_plus = np.empty(max(n, 1), np.uint64)
    minus = np.empty(max(int(moff[n]), 1), np.uint64)
    assert R.ref_split_degree_aware(rc.h, limit, in_plus.ctypes.data, moff.ctypes.data,
                                    minus.ctypes.data) == 0
    return in_plus[:n], moff, minus[: int(moff[n])]


def ref_report(rc, root, parent):
    out = np.zeros(8, np.uint64)
    where = np.zeros(125, np.uint64)
    par = np.ascontiguousarray(parent, np.uint64)
    assert O.ref().ref_validate_report(rc.h, root, par.ctypes.data, out.ctypes.data,
                                       where.ctypes.data) == 0
    return out, where


def graphs(corpus):
    for g in corpus:
        yield g["name"], g["n"], edges_of(g)
    yield "kron-s12", 1 << 12, O.oracle_generate(12, 16, 3)


def test_degree_split_matches_reference(corpus):
    for name, n, pairs in graphs(corpus):
        g = eb.build_csr(n, pairs)
        rc = O.RefCsr(n, pairs)
        for limit in (None, n // 2, 0):
            lim = 0xFFFFFFFFFFFFFFFF if limit is None else limit
            got = E.split_degree_aware(g, limit)
            want = ref_split(rc, n, lim)
            for a, b in zip(got, want):
                assert np.array_equal(a, b), (name, limit)


def test_oracle_levels_match_reference(corpus):
    for name, n, pairs in graphs(corpus):
        g = eb.build_csr(n, pairs)
        rc = O.RefCsr(n, pairs)
        for root in range(0, n, max(1, n // 7)):
            assert np.array_equal(E.oracle_bfs(g, root), rc.levels(root)), (name, root)


def mutations(parent, root, rng, n):
    """Corrupted copies of a valid tree: one per rule class."""
    reached = np.nonzero((parent != NO) & (np.arange(n) != root))[0]
    out = []
    if reached.size:
        v = int(rng.choice(reached))
        p = parent.copy(); p[root] = v; out.append(("root", p))                 # rule 1
        p = parent.copy(); p[v] = np.uint64(n + 5); out.append(("badptr", p))    # 2 + 3
        p = parent.copy(); p[v] = NO; out.append(("drop", p))                     # 5 (+2)
        w = int(rng.choice(reached))
        p = parent.copy(); p[v] = w; p[w] = v; out.append(("cycle", p))          # 2 + 3
        far = int(rng.integers(0, n))
        p = parent.copy(); p[v] = far; out.append(("reparent", p))               # 3 / 4
    unreached = np.nonzero(parent == NO)[0]
    if unreached.size and reached.size:
        u = int(rng.choice(unreached))
        p = parent.copy(); p[u] = int(rng.choice(reached)); out.append(("adopt", p))  # 5
    return out


def test_validator_matches_reference(corpus):
    rng = np.random.default_rng(7)
    for name, n, pairs in graphs(corpus):
        g = eb.build_csr(n, pairs)
        rc = O.RefCsr(n, pairs)
        for root in range(0, n, max(1, n // 5)):
            parent, _ = rc.bfs_hybrid(root)
            parent = np.asarray(parent, np.uint64)
            cases = [("valid", parent)] + mutations(parent, root, rng, n)
            for label, p in cases:
                got = E.validate_bfs_tree(g, root, p)
                want, where = ref_report(rc, root, p)
                assert got["passed"] == bool(want[0]), (name, root, label)
                assert got["reached_count"] == int(want[6]), (name, root, label)
                assert got["traversed_edge_count"] == int(want[7]), (name, root, label)
                for r in (1, 3, 4, 5):  # same failures, same order, same cap
                    mine = [w for rr, w in got["failures"] if rr == r]
                    ref = [int(x) for x in where[(r - 1) * 25:(r - 1) * 25 + int(want[r])]]
                    assert mine == ref, (name, root, label, r)
                assert (got["rule_counts"][1] > 0) == (int(want[2]) > 0), (name, root, label)
