"""Pin the CPU oracle (oracle/etbfs_oracle.c) against the golden fixtures made
by running the compiled reference (tests/golden/make_golden.py), and — when
oracle/_ref is built here — against the live reference. CPU only."""
import numpy as np
import pytest

import oracle as O
from conftest import edges_of, levels_list


def test_corpus_csr_classify_layout(corpus):
    for g in corpus:
        n = g["n"]
        csr = O.OracleCsr(n, edges_of(g))
        row, col = csr.arrays()
        assert row.tolist() == g["row"], g["name"]
        assert col.tolist() == g["col"], g["name"]
        assert (csr.self_loops, csr.duplicates) == (g["self_loops"], g["duplicates"]), g["name"]
        for mh, want in g["classify"].items():
            t, rounds = csr.classify(int(mh))
            assert t.tolist() == want, (g["name"], mh)
        _, ph = csr.classify(-1)
        assert ph == g["peak_height"], g["name"]
        for mh, lay in g["layout"].items():
            L = O.OracleLayout(csr, int(mh))
            new2old, types, rrow, rcol = L.arrays()
            assert L.core == lay["core"], (g["name"], mh)
            assert new2old.tolist() == lay["new2old"], (g["name"], mh)
            s, d, c = L.etl()
            got = [[int(a), int(b), -1 if z == O.NO_VERTEX else int(z)] for a, b, z in zip(s, d, c)]
            assert got == lay["etl"], (g["name"], mh)
            assert L.graph.restricted_edge_count(L.core) == lay["restricted_edges"]
            for st, r in lay["roots"].items():
                assert levels_list(L.graph.levels(int(st))) == r["levels"], (g["name"], mh, st)
                if int(st) < L.core:
                    assert L.graph.hybrid_trace(L.core, int(st)) == r["trace"], (g["name"], mh, st)


def test_kronecker_s16_anchors(kron16):
    k = kron16
    pairs = O.oracle_generate(16, 16, 1)
    assert O.fnv1a64(pairs) == k["tuples_fnv"]
    n = 1 << 16
    csr = O.OracleCsr(n, pairs)
    row, col = csr.arrays()
    assert (csr.self_loops, csr.duplicates, csr.nnz) == (k["self_loops"], k["duplicates"], k["nnz"])
    assert O.fnv1a64(row) == k["row_fnv"] and O.fnv1a64(col) == k["col_fnv"]
    roots = csr.select_roots(64, 1)
    assert roots.tolist() == k["roots"]
    assert roots[:8].tolist() == [23745, 51467, 640, 15525, 34165, 15784, 20321, 24000]
    for mh, counts in k["classes"].items():
        t, rounds = csr.classify(int(mh))
        assert np.bincount(t, minlength=5).tolist() == counts
    assert csr.classify(-1)[1] == k["peak_height"]
    for mh, lay in k["layout"].items():
        L = O.OracleLayout(csr, int(mh))
        new2old, _, rrow, rcol = L.arrays()
        s, d, c = L.etl()
        assert L.core == lay["core"]
        assert len(s) == lay["etl_size"]
        assert O.fnv1a64(new2old) == lay["new2old_fnv"]
        assert O.fnv1a64(rrow) == lay["relaid_row_fnv"]
        assert O.fnv1a64(rcol) == lay["relaid_col_fnv"]
        assert O.fnv1a64(np.stack([s, d, c], 1)) == lay["etl_fnv"]
        assert L.graph.restricted_edge_count(L.core) == lay["restricted_edges"]
        old2new = np.empty(n, np.uint64)
        old2new[new2old] = np.arange(n, dtype=np.uint64)
        # traces for core starts (tree starts walk to their CE first; covered on GPU)
        for r, tr in zip(roots[:16], lay["traces"][:16]):
            st = int(old2new[int(r)])
            if st < L.core:
                assert L.graph.hybrid_trace(L.core, st) == tr
    for r, f, te in zip(roots, k["levels_fnv"], k["traversed_edges"]):
        lv = csr.levels(int(r))
        assert O.fnv1a64(lv) == f
        assert csr.traversed_edges(lv) == te


@pytest.mark.slow
def test_kronecker_big_counts(kron_big):
    """C2 (s22/ef16) and C3 (s24/ef4): generator/CSR hashes and ET class counts."""
    for k in kron_big:
        n = 1 << k["scale"]
        pairs = O.oracle_generate(k["scale"], k["edgefactor"], k["seed"])
        assert O.fnv1a64(pairs) == k["tuples_fnv"]
        csr = O.OracleCsr(n, pairs)
        del pairs
        assert (csr.self_loops, csr.duplicates, csr.nnz) == (k["self_loops"], k["duplicates"],
                                                             k["nnz"])
        row, col = csr.arrays()
        assert O.fnv1a64(row) == k["row_fnv"] and O.fnv1a64(col) == k["col_fnv"]
        del col
        assert csr.select_roots(64, 1).tolist() == k["roots"]
        t, _ = csr.classify(0)
        assert np.bincount(t, minlength=5).tolist() == k["classes"]["0"]
        lv = csr.levels(k["roots"][0])
        assert O.fnv1a64(lv) == k["levels_fnv"][0]


@pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built (needs /root/reference)")
def test_restatement_matches_live_reference():
    """Random graphs with self loops/dups/isolated vertices: C restatement == reference."""
    rng = np.random.default_rng(7)
    for trial in range(30):
        n = int(rng.integers(2, 400))
        m = int(rng.integers(0, 3 * n))
        pairs = rng.integers(0, n, size=(m, 2)).astype(np.uint64)
        a, b = O.OracleCsr(n, pairs), O.RefCsr(n, pairs)
        ra, ca = a.arrays()
        rb, cb = b.arrays()
        assert (ra == rb).all() and (ca == cb).all()
        for mh in (-1, 0, 1, 2):
            assert (a.classify(mh)[0] == b.classify(mh)).all()
        assert a.classify(-1)[1] == b.peak_height()
        for mh in (-1, 0, 1):
            L, R = O.OracleLayout(a, mh), O.RefPrepared(b, mh)
            x, y = L.arrays(), R.arrays()
            assert (x[0] == y["new2old"]).all()
            s, d, c = L.etl()
            assert (s == y["etl_src"]).all() and (d == y["etl_dst"]).all() and \
                (c == y["etl_ce"]).all()
        r = int(rng.integers(0, n))
        assert (a.levels(r) == b.levels(r)).all()


def test_oracle_errors():
    with pytest.raises(ValueError, match="endpoint out of range at edge index 1"):
        O.OracleCsr(3, np.array([[0, 1], [1, 3]], np.uint64))
    csr = O.OracleCsr(3, np.array([[0, 1], [1, 2]], np.uint64))
    with pytest.raises(ValueError, match="mh must be -1 or >= 0"):
        csr.classify(-2)
