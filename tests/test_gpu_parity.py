"""GPU parity: the sm_100a path through the C-ABI vs the CPU oracle and the
golden fixtures produced by running the reference. Integer work, so every
comparison is bit-exact; parents (race-dependent by design) are
checked for validity: a true neighbour exactly one level up, root self-parented,
unreached <-> no parent."""
import numpy as np
import pytest

import oracle as O
import paper_2009_07463_b200 as eb
from conftest import edges_of, levels_list
from paper_2009_07463_b200 import etbfs as E
from paper_2009_07463_b200.etbfs import (bfs_device, result_download, result_traversed_edges,
                                         time_roots)

pytestmark = pytest.mark.gpu

NO32 = 0xFFFFFFFF


def lift(cg: eb.EtLayout, depth, parent):
    """Relaid (depth i32, parent u64) -> original-space (levels u64, parent u64)."""
    n = cg.vertex_count
    new2old = cg.new2old
    lv = np.full(n, O.NO_VERTEX, np.uint64)
    par = np.full(n, O.NO_VERTEX, np.uint64)
    reached = depth >= 0
    lv[new2old[reached]] = depth[reached].astype(np.uint64)
    ok = parent != O.NO_VERTEX
    par[new2old[ok]] = new2old[parent[ok].astype(np.int64)]
    return lv, par


def check_root(cg, ocsr, root_orig, kernel=eb.CoreKernel.HYBRID, replay=eb.TreeReplay.TEET,
               policy=None):
    start = int(cg.old2new[root_orig])
    r = eb.et_bfs(cg, start, kernel=kernel, replay=replay, policy=policy, stats=True)
    lv, par = lift(cg, r.depth, r.parent)
    want = ocsr.levels(int(root_orig))
    assert (lv == want).all(), f"depth mismatch from root {root_orig}"
    bad = ocsr.check_tree(int(root_orig), par, want)
    assert bad == 0, f"invalid parent at vertex {bad - 1} (root {root_orig})"
    return r


# ------------------------------------------------------------------ graph ---
def test_generator_bit_exact_small_scales():
    for scale, ef, seed in [(0, 16, 1), (1, 3, 5), (5, 16, 1), (10, 16, 2), (12, 4, 9), (16, 16, 1)]:
        got = eb.generate_kronecker(scale=scale, edgefactor=ef, seed=seed)
        want = O.oracle_generate(scale, ef, seed)
        assert got.shape == want.shape and (got == want).all(), (scale, ef, seed)


def test_generator_nondefault_initiator():
    got = eb.generate_kronecker(scale=11, edgefactor=8, a=0.45, b=0.25, c=0.15, d=0.15, seed=3)
    want = O.oracle_generate(11, 8, 3, 0.45, 0.25, 0.15, 0.15)
    assert (got == want).all()


def test_generator_s16_anchor(kron16):
    assert O.fnv1a64(eb.generate_kronecker(scale=16, edgefactor=16, seed=1)) == kron16["tuples_fnv"]


def test_build_csr_corpus(corpus):
    for g in corpus:
        csr = eb.build_csr(g["n"], edges_of(g))
        row, col, deg = csr.download()
        assert row.tolist() == g["row"], g["name"]
        assert col.tolist() == g["col"], g["name"]
        assert (np.diff(row) == deg).all()
        assert (csr.dropped_self_loops, csr.dropped_duplicates) == (g["self_loops"],
                                                                    g["duplicates"]), g["name"]


def test_build_csr_s16_fused_and_uploaded(kron16):
    k = kron16
    for csr in (eb.generate_graph(scale=16, edgefactor=16, seed=1),
                eb.build_csr(1 << 16, O.oracle_generate(16, 16, 1))):
        row, col, _ = csr.download()
        assert O.fnv1a64(row) == k["row_fnv"] and O.fnv1a64(col) == k["col_fnv"]
        assert (csr.dropped_self_loops, csr.dropped_duplicates) == (k["self_loops"],
                                                                    k["duplicates"])


def test_build_csr_edge_cases():
    csr = eb.build_csr(5, np.zeros((0, 2), np.uint64))  # edgeless
    row, col, deg = csr.download()
    assert row.tolist() == [0] * 6 and col.size == 0
    csr = eb.build_csr(3, np.array([[1, 1], [2, 2]], np.uint64))  # only self loops
    assert csr.directed_edge_count == 0 and csr.dropped_self_loops == 2
    csr = eb.build_csr(2, np.array([[0, 1]] * 7 + [[1, 0]] * 3, np.uint64))  # duplicates
    assert csr.directed_edge_count == 2 and csr.dropped_duplicates == 9


# --------------------------------------------------------------- classify ---
def test_classify_corpus(corpus):
    for g in corpus:
        csr = eb.build_csr(g["n"], edges_of(g))
        for mh, want in g["classify"].items():
            assert eb.classify_vertices(csr, int(mh)).tolist() == want, (g["name"], mh)
        assert eb.compute_peak_height(csr) == g["peak_height"], g["name"]


def test_classify_kats():
    # proj/tests/test_classify.cpp:80-138 (values restated from the reference's KATs)
    CI, CE, TI, TL, VZ = range(5)
    path = lambda n: eb.build_csr(n, np.array([[v, v + 1] for v in range(n - 1)], np.uint64))
    g = path(5)
    assert eb.classify_vertices(g, -1).tolist() == [TL, TI, TI, TI, TL]
    assert eb.classify_vertices(g, 1).tolist() == [TL, TI, TI, CE, TL]
    assert eb.classify_vertices(g, 0).tolist() == [TL, CE, CI, CE, TL]
    assert eb.compute_peak_height(g) == 2
    g = path(7)
    assert eb.compute_peak_height(g) == 2
    assert eb.classify_vertices(g, 1).tolist() == [TL, TI, TI, TI, TI, CE, TL]
    with pytest.raises(ValueError, match="mh must be -1 or >= 0"):
        eb.classify_vertices(g, -2)


def test_classify_s16(kron16):
    csr = eb.generate_graph(scale=16, edgefactor=16, seed=1)
    for mh, counts in kron16["classes"].items():
        t = eb.classify_vertices(csr, int(mh))
        assert np.bincount(t, minlength=5).tolist() == counts
    assert eb.compute_peak_height(csr) == kron16["peak_height"]


# ----------------------------------------------------------------- layout ---
def test_layout_corpus(corpus):
    for g in corpus:
        csr = eb.build_csr(g["n"], edges_of(g))
        for mh, lay in g["layout"].items():
            cg = eb.relayout_csr(csr, mh=int(mh))
            assert cg.core_vertex_count == lay["core"], (g["name"], mh)
            assert cg.new2old.tolist() == lay["new2old"], (g["name"], mh)
            s, d, c = eb.extract_edge_tree_list(cg)
            got = [[int(a), int(b), -1 if z == O.NO_VERTEX else int(z)] for a, b, z in zip(s, d, c)]
            assert got == lay["etl"], (g["name"], mh)
            assert cg.restricted_edge_count == lay["restricted_edges"], (g["name"], mh)
            row, col = cg.graph()
            rg = O.OracleLayout(O.OracleCsr(g["n"], edges_of(g)), int(mh))
            _, _, rrow, rcol = rg.arrays()
            assert (row == rrow).all() and (col == rcol).all(), (g["name"], mh)


def test_layout_frozen_kats():
    # proj/tests/test_relayout.cpp:110-158
    tri = np.array([[0, 1], [1, 2], [0, 2], [2, 3], [3, 4], [3, 5]], np.uint64)
    cg = eb.relayout_csr(eb.build_csr(6, tri), mh=-1)
    assert cg.core_vertex_count == 3
    assert cg.new2old.tolist() == [2, 0, 1, 3, 4, 5]
    s, d, c = eb.extract_edge_tree_list(cg)
    assert [(int(a), int(b), int(z)) for a, b, z in zip(s, d, c)] == [(0, 3, 0), (3, 4, 0),
                                                                      (3, 5, 0)]
    star = np.array([[0, v] for v in range(1, 5)], np.uint64)
    cg = eb.relayout_csr(eb.build_csr(5, star), mh=-1)
    assert cg.core_vertex_count == 0 and cg.new2old.tolist() == [0, 1, 2, 3, 4]
    s, d, c = eb.extract_edge_tree_list(cg)
    assert (int(s[0]), int(d[0]), c[0]) == (0, 0, O.NO_VERTEX)


def test_extract_errors_match_reference_messages():
    # proj/tests/test_relayout.cpp:194-220 (manual type vectors)
    CI, CE, TI, TL, VZ = range(5)
    g = eb.build_csr(3, np.array([[0, 1], [0, 2], [1, 2]], np.uint64))
    with pytest.raises(RuntimeError, match="touches the core more than once"):
        eb.relayout_csr(g, types=np.array([CE, CE, TI], np.uint8), mh=2)
    g = eb.build_csr(4, np.array([[0, 1], [1, 2], [2, 3], [1, 3]], np.uint64))
    with pytest.raises(RuntimeError, match="cycle through tree vertices"):
        eb.relayout_csr(g, types=np.array([CE, TI, TI, TI], np.uint8), mh=1)
    g = eb.build_csr(2, np.array([[0, 1]], np.uint64))
    with pytest.raises(RuntimeError, match="isolated-typed vertex has incident edges"):
        eb.relayout_csr(g, types=np.array([TL, VZ], np.uint8), mh=0)


def test_layout_s16_hashes(kron16):
    csr = eb.generate_graph(scale=16, edgefactor=16, seed=1)
    for mh, lay in kron16["layout"].items():
        cg = eb.relayout_csr(csr, mh=int(mh))
        assert cg.core_vertex_count == lay["core"]
        assert cg.tree_vertex_count == lay["etl_size"]
        assert cg.restricted_edge_count == lay["restricted_edges"]
        assert O.fnv1a64(cg.new2old) == lay["new2old_fnv"]
        row, col = cg.graph()
        assert O.fnv1a64(row) == lay["relaid_row_fnv"] and O.fnv1a64(col) == lay["relaid_col_fnv"]
        s, d, c = eb.extract_edge_tree_list(cg)
        assert O.fnv1a64(np.stack([s, d, c], 1)) == lay["etl_fnv"]


# -------------------------------------------------------------------- BFS ---
def test_bfs_corpus_all_starts(corpus):
    """Every start of every corpus graph, mh -1/0/1, hybrid + top-down (+TEOLV at mh 0):
    depths bit-exact vs the golden oracle levels (relaid space)."""
    for g in corpus:
        csr = eb.build_csr(g["n"], edges_of(g))
        ocsr = O.OracleCsr(g["n"], edges_of(g))
        for mh, lay in g["layout"].items():
            cg = eb.relayout_csr(csr, mh=int(mh))
            for st in range(g["n"]):
                root = int(cg.new2old[st])
                for kernel in (eb.CoreKernel.HYBRID, eb.CoreKernel.TOP_DOWN):
                    check_root(cg, ocsr, root, kernel=kernel)
                if int(mh) == 0:
                    check_root(cg, ocsr, root, replay=eb.TreeReplay.TEOLV)
            for st, r in lay["roots"].items():
                res = eb.et_bfs(cg, int(st), stats=True)
                assert levels_list(np.where(res.depth < 0, O.NO_VERTEX,
                                            res.depth.astype(np.uint64))) == r["levels"]
                assert res.stats.direction_trace == r["trace"], (g["name"], mh, st)


def test_bfs_policy_kats():
    # proj/tests/test_bfs_kernels.cpp:185-218 restated on the composite: path-4 with
    # α→0 stays top-down; α huge goes bottom-up from the first level; star switches.
    path = np.array([[v, v + 1] for v in range(5)], np.uint64)
    cycle = np.vstack([path, [[5, 0]]]).astype(np.uint64)
    cg = eb.relayout_csr(eb.build_csr(6, cycle), mh=-1)
    oc = O.OracleCsr(6, cycle)
    r = check_root(cg, oc, 0, policy=eb.HybridPolicy(alpha=1e-9))
    assert set(r.stats.direction_trace) == {"t"}
    r = check_root(cg, oc, 0, policy=eb.HybridPolicy(alpha=1e18))
    assert set(r.stats.direction_trace) == {"b"}
    with pytest.raises(ValueError, match="alpha and beta must be positive"):
        eb.et_bfs(cg, 0, policy=eb.HybridPolicy(alpha=0.0))


def test_bfs_errors_and_isolated():
    cg = eb.relayout_csr(eb.build_csr(5, np.array([[0, 1], [1, 2]], np.uint64)), mh=-1)
    with pytest.raises(ValueError, match="start out of range"):
        eb.et_bfs(cg, 99)
    with pytest.raises(ValueError, match="leaves-only replay needs a height-0"):
        eb.et_bfs(cg, 0, replay=eb.TreeReplay.TEOLV)
    iso = 4  # isolated vertices close the index space (test_et_bfs.cpp:171-179)
    assert cg.vertex_type[iso] == eb.VertexType.VERTEX_ZERO
    r = eb.et_bfs(cg, iso)
    assert r.parent[iso] == iso and r.depth[iso] == 0
    assert all(r.parent[v] == O.NO_VERTEX for v in range(5) if v != iso)
    r = eb.et_bfs(cg, 0)  # the previous isolated start must be reset
    assert r.parent[iso] == O.NO_VERTEX and r.depth[iso] == -1


def kron_check(scale, ef, roots_orig, mh, nroots, traces=None, replay=eb.TreeReplay.TEET):
    csr = eb.generate_graph(scale=scale, edgefactor=ef, seed=1)
    ocsr = O.OracleCsr(1 << scale, O.oracle_generate(scale, ef, 1))
    cg = eb.relayout_csr(csr, mh=mh)
    for i, root in enumerate(roots_orig[:nroots]):
        r = check_root(cg, ocsr, int(root), replay=replay)
        if traces is not None:
            assert r.stats.direction_trace == traces[i], (scale, root)
    return cg, ocsr


def test_bfs_s16_64_roots(kron16):
    k = kron16
    for mh in (-1, 0):
        cg, ocsr = kron_check(16, 16, k["roots"], mh, 64, traces=k["layout"][str(mh)]["traces"])
        # device traversed-edge count (validate.cpp:151-156) == reference TE
        start = int(cg.old2new[k["roots"][0]])
        bfs_device(cg, start)
        assert result_traversed_edges(cg) == k["traversed_edges"][0]
    kron_check(16, 16, k["roots"], 0, 8, replay=eb.TreeReplay.TEOLV)


@pytest.mark.slow
def test_bfs_s24ef4_tiny_component_roots(kron_big):
    """C3's roots 2590069 and 5097554 sit in TL-pair components (TE = 1)."""
    k = [x for x in kron_big if x["scale"] == 24][0]
    csr = eb.generate_graph(scale=24, edgefactor=4, seed=1)
    ocsr = O.OracleCsr(1 << 24, O.oracle_generate(24, 4, 1))
    cg = eb.relayout_csr(csr, mh=-1)
    for root in (2590069, 5097554):
        assert root in k["roots"]
        check_root(cg, ocsr, root)
        bfs_device(cg, int(cg.old2new[root]))
        assert result_traversed_edges(cg) == 1


def test_timing_api_and_result_download(kron16):
    cg = eb.relayout_csr(eb.generate_graph(scale=16, edgefactor=16, seed=1), mh=-1)
    starts = cg.old2new[np.array(kron16["roots"][:8], np.int64)]
    ms, kms = time_roots(cg, starts, warmup=3, flush_l2=True)
    assert (ms > 0).all() and (kms > 0).all() and (kms <= ms + 1e-6).all()
    depth, parent = result_download(cg)
    assert depth.dtype == np.int32 and parent.dtype == np.uint32
    assert depth[int(starts[-1])] == 0 or cg.vertex_type[int(starts[-1])] >= 2


def test_bucketed_builds_match(kron16, monkeypatch):
    """The large-scale path (CSR and core CSR built in source buckets, as used at
    scale 28) forced on s16 with small buckets: identical graph and layout."""
    monkeypatch.setenv("ETB_CSR_BUCKET_KEYS", "150000")
    csr = eb.generate_graph(scale=16, edgefactor=16, seed=1)
    row, col, _ = csr.download()
    assert O.fnv1a64(row) == kron16["row_fnv"] and O.fnv1a64(col) == kron16["col_fnv"]
    assert (csr.dropped_self_loops, csr.dropped_duplicates) == (kron16["self_loops"],
                                                                kron16["duplicates"])
    cg = eb.relayout_csr(csr, mh=-1)
    lay = kron16["layout"]["-1"]
    assert O.fnv1a64(cg.new2old) == lay["new2old_fnv"]
    ocsr = O.OracleCsr(1 << 16, O.oracle_generate(16, 16, 1))
    for root in kron16["roots"][:8]:
        check_root(cg, ocsr, int(root))


def test_split_kernels_corpus(corpus):
    """CoreKernel::kDegreeAware / kBlockSearch / kHybridBlockSearch (et_bfs.hpp:10-16):
    level-exact like every kernel (test_et_bfs.cpp:158-169); block search runs
    bottom-up sweeps only, one 'b' per step until a step claims nothing."""
    for g in corpus:
        csr = eb.build_csr(g["n"], edges_of(g))
        ocsr = O.OracleCsr(g["n"], edges_of(g))
        cg = eb.relayout_csr(csr, mh=-1)
        for st in range(g["n"]):
            root = int(cg.new2old[st])
            for k in (eb.CoreKernel.DEGREE_AWARE, eb.CoreKernel.HYBRID_BLOCK_SEARCH):
                check_root(cg, ocsr, root, kernel=k)
            r = check_root(cg, ocsr, root, kernel=eb.CoreKernel.BLOCK_SEARCH)
            tr = r.stats.direction_trace
            assert set(tr) <= {"b"}, tr
            if st < cg.core_vertex_count:
                lv = ocsr.levels(root)
                core_depth = max(int(x) for x, v in zip(lv, range(g["n"]))
                                 if x != O.NO_VERTEX and int(cg.old2new[v]) < cg.core_vertex_count)
                assert len(tr) == core_depth + 1, (g["name"], st, tr)


def test_bfs_compact_outputs(kron16):
    """etb_bfs_compact (the e2e API) into pageable and pinned (registered) host
    buffers equals that traversal's device result (parents can differ between
    runs: top-down claims race)."""
    from paper_2009_07463_b200 import etbfs as E
    g = eb.generate_graph(scale=16, edgefactor=16, seed=1)
    cg = eb.relayout_csr(g, mh=-1)
    n = cg.vertex_count
    L = E.lib()
    for root in kron16["roots"][:4]:
        s = int(cg.old2new[root])
        for pinned in (False, True):
            par = np.full(n, 7, np.uint32)
            dep = np.full(n, 7, np.int32)
            if pinned:
                E._check(L.etb_host_register(par.ctypes.data, par.nbytes))
                E._check(L.etb_host_register(dep.ctypes.data, dep.nbytes))
            try:
                E._check(L.etb_bfs_compact(cg.handle, s, None, dep.ctypes.data, par.ctypes.data))
            finally:
                if pinned:
                    E._check(L.etb_host_unregister(par.ctypes.data))
                    E._check(L.etb_host_unregister(dep.ctypes.data))
            d2, p2 = result_download(cg)  # u32 parents, UINT32_MAX unreached
            assert np.array_equal(par, p2), (root, pinned)
            assert np.array_equal(dep, d2), (root, pinned)
            assert E.result_validate(cg, s)["passed"], (root, pinned)


@pytest.mark.slow
def test_whole_graph_top_down_s20():
    """Top-down only on the whole graph (every vertex in the traversed block, as
    bfs_top_down / run_benchmark(kTopDown) use it): frontier lists full of
    one-edge rows, so 128-edge chunks made of 128 rows occur — the next chunk
    then starts exactly one row past the merge-path window."""
    csr = eb.generate_graph(scale=20, edgefactor=16, seed=1)
    n = csr.vertex_count
    ocsr = O.OracleCsr(n, O.oracle_generate(20, 16, 1))
    cg = eb.relayout_csr(csr, types=np.zeros(n, np.uint8), mh=-1)
    for parts in (1, 4):
        E.partition(cg, parts)
        for root in ocsr.select_roots(16, 2):
            check_root(cg, ocsr, int(root), kernel=eb.CoreKernel.TOP_DOWN)
    E.partition(cg, 1)
