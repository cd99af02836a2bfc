"""The measurement entry points behind bench.py's roofline and timing lines:
etb_result_work's per-level counters against a host recount from the result
depths and the relabelled CSR (the reference's step semantics, bfs.cpp:61-111),
the wall-clock timer, and the original-id result download against the oracle."""
import numpy as np
import pytest

import oracle as O
import paper_2009_07463_b200 as eb
from paper_2009_07463_b200 import etbfs as E

pytestmark = pytest.mark.gpu


def host_work(row, col, nc, depth, trace):
    """Per level (frontier-or-unvisited, columns read, claims, first-probe misses)."""
    dcore = depth[:nc].astype(np.int64)
    base = int(dcore[dcore >= 0].min())
    out = []
    for L, d in enumerate(trace):
        lvl = base + L
        claims = int(np.count_nonzero(dcore == lvl + 1))
        if d == "t":
            fr = np.nonzero(dcore == lvl)[0]
            cols = 0
            for u in fr:
                nb = col[row[u]:row[u + 1]]
                cols += int(np.count_nonzero(nb < nc))
            out.append((len(fr), cols, claims, 0))
        else:
            un = np.nonzero((dcore < 0) | (dcore > lvl))[0]
            extra = misses = 0
            for v in un:
                nb = col[row[v]:row[v + 1]]
                nb = nb[nb < nc]
                hit = np.nonzero(dcore[nb.astype(np.int64)] == lvl)[0]
                probes = int(hit[0]) + 1 if hit.size else len(nb)
                if probes > 1:
                    extra += probes - 1
                    misses += 1
            out.append((len(un), extra, claims, misses))
    return out


@pytest.mark.parametrize("mh", [-1, 0])
def test_result_work_matches_host_recount(mh):
    g = eb.generate_graph(scale=12, edgefactor=16, seed=1)
    cg = eb.relayout_csr(g, mh=mh)
    row, col = cg.graph()
    nc = cg.core_vertex_count
    from bench import select_roots_from_degrees
    roots = select_roots_from_degrees(g.degrees(), 6, 1)
    for r in roots:
        s = int(cg.old2new[int(r)])
        rep = E.TreeReplay.TEOLV if mh == 0 else E.TreeReplay.TEET
        w = E.result_work(cg, s, replay=rep)
        res = eb.et_bfs(cg, s, replay=rep, want_parent=False)
        want = host_work(row, col, nc, res.depth, w.trace)
        assert [tuple(int(x) for x in lv) for lv in w.levels] == want, (r, w.trace)
        assert w.total_bytes == int(w.bytes.sum()) and w.total_bytes > 0
        # the work model never exceeds SURVEY's B_alg normalisation by the edges
        assert w.bytes[:-1].sum() < 8 * cg.restricted_edge_count + 64 * nc


def test_wall_timer_and_original_download():
    g = eb.generate_graph(scale=12, edgefactor=16, seed=1)
    cg = eb.relayout_csr(g, mh=-1)
    ocsr = O.OracleCsr(1 << 12, O.oracle_generate(12, 16, 1))
    roots = ocsr.select_roots(4, 1)
    starts = cg.old2new[roots.astype(np.int64)]
    ms = E.time_roots_wall(cg, starts, warmup=3)
    assert ms.shape == (4,) and (ms > 0).all()
    for r, s in zip(roots, starts):
        E.bfs_device(cg, int(s))
        lv, par = E.result_original(cg)
        assert (lv == ocsr.levels(int(r))).all()
        assert ocsr.check_tree(int(r), par, lv) == 0
        assert par[int(r)] == int(r)
