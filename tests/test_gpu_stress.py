"""Shapes far from Kronecker, on the product kernel: a long cycle (tens of
thousands of levels), a long path (all edge tree), a big star (one hub, every
other vertex a leaf), a dense clique, a grid, and a mixture of components —
depths checked against the CPU oracle, parents by the device validator."""
import numpy as np
import pytest

import oracle as O
import paper_2009_07463_b200 as eb
from paper_2009_07463_b200 import etbfs as E

pytestmark = pytest.mark.gpu
NO = np.uint64(0xFFFFFFFFFFFFFFFF)


def cycle(n):
    v = np.arange(n, dtype=np.uint64)
    return np.stack([v, (v + 1) % n], 1)


def path(n):
    v = np.arange(n - 1, dtype=np.uint64)
    return np.stack([v, v + 1], 1)


def star(n):
    v = np.arange(1, n, dtype=np.uint64)
    return np.stack([np.zeros_like(v), v], 1)


def clique(k):
    a, b = np.triu_indices(k, 1)
    return np.stack([a, b], 1).astype(np.uint64)


def grid(w, h):
    idx = np.arange(w * h, dtype=np.uint64).reshape(h, w)
    right = np.stack([idx[:, :-1].ravel(), idx[:, 1:].ravel()], 1)
    down = np.stack([idx[:-1, :].ravel(), idx[1:, :].ravel()], 1)
    return np.vstack([right, down])


def mixture():
    parts, off = [], 0
    for e, n in ((cycle(500), 500), (path(300), 300), (star(200), 200), (clique(40), 40),
                 (grid(30, 20), 600), (np.empty((0, 2), np.uint64), 50)):
        parts.append(e + np.uint64(off))
        off += n
    return off, np.vstack(parts)


def long_miss():
    """A bottom-up level where a vertex with > 1024 core neighbours misses on its
    first (highest-degree) neighbour and scans its row with the whole warp:
    R - N_i (1500, in a ring), H - every N_i, H - Z, Z - Y_0..Y_9 (a ring)."""
    k, y = 1500, 10
    R, H, Z = 0, 1, 2
    N = np.arange(3, 3 + k, dtype=np.uint64)
    Y = np.arange(3 + k, 3 + k + y, dtype=np.uint64)
    e = [np.stack([np.full(k, R, np.uint64), N], 1), np.stack([N, np.roll(N, 1)], 1),
         np.stack([np.full(k, H, np.uint64), N], 1), np.array([[H, Z]], np.uint64),
         np.stack([np.full(y, Z, np.uint64), Y], 1), np.stack([Y, np.roll(Y, 1)], 1)]
    return 3 + k + y, np.vstack(e)


CASES = [("longmiss",) + long_miss(), ("cycle", 1 << 15, cycle(1 << 15)), ("path", 1 << 15, path(1 << 15)),
         ("star", 1 << 18, star(1 << 18)), ("clique", 1500, clique(1500)),
         ("grid", 300 * 200, grid(300, 200)), ("mixture",) + mixture()]


@pytest.mark.parametrize("name,n,pairs", CASES, ids=[c[0] for c in CASES])
def test_extreme_shapes(name, n, pairs):
    g = eb.build_csr(n, pairs)
    oc = O.OracleCsr(n, pairs)
    rng = np.random.default_rng(11)
    for mh in (-1, 0):
        cg = eb.relayout_csr(g, mh=mh)
        for root in [0, n - 1] + [int(x) for x in rng.integers(0, n, 3)]:
            s = int(cg.old2new[root])
            r = eb.et_bfs(cg, s, stats=True)
            want = oc.levels(root)
            got = np.full(n, NO, np.uint64)
            ok = r.depth >= 0
            got[np.asarray(cg.new2old, np.int64)[ok]] = r.depth[ok].astype(np.uint64)
            assert np.array_equal(got, want), (name, mh, root)
            E.bfs_device(cg, s)
            assert E.result_validate(cg, s)["passed"], (name, mh, root)


def warp_scan_graph():
    """H's core row holds 100 higher-degree neighbours (a clique D) before its
    only frontier neighbour F, so a bottom-up level scans past the lane-scan
    prefix into the warp scan: R - F - G triangle, H - F, H - D_i, D a clique."""
    R, F, G, H = 0, 1, 2, 3
    D = np.arange(4, 104, dtype=np.uint64)
    a, b = np.triu_indices(len(D), 1)
    e = [np.array([[R, F], [F, G], [G, R], [H, F]], np.uint64),
         np.stack([np.full(len(D), H, np.uint64), D], 1), np.stack([D[a], D[b]], 1)]
    return 104, np.vstack(e)


def test_bottom_up_warp_scan():
    n, pairs = warp_scan_graph()
    g = eb.build_csr(n, pairs)
    oc = O.OracleCsr(n, pairs)
    cg = eb.relayout_csr(g, mh=-1)
    for root in (0, 1, 3, 50):
        s = int(cg.old2new[root])
        for kw in ({"policy": eb.HybridPolicy(alpha=1e18)},
                   {"kernel": eb.CoreKernel.BLOCK_SEARCH}):
            r = eb.et_bfs(cg, s, stats=True, **kw)
            got = np.full(n, NO, np.uint64)
            ok = r.depth >= 0
            got[np.asarray(cg.new2old, np.int64)[ok]] = r.depth[ok].astype(np.uint64)
            assert np.array_equal(got, oc.levels(root)), (root, kw)
            assert "b" in r.stats.direction_trace

