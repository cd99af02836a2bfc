"""GPU runs exchange files with the CPU reference tools:
an ETG1 file goes straight to a device CSR with the reference's hashes, and a
device BFS tree written as ETT1 is read back and validated by the compiled
reference (read_tree + validate_bfs_tree, proj/src/validate.cpp:95-158)."""
import numpy as np
import pytest

import oracle as O
import paper_2009_07463_b200 as eb

pytestmark = pytest.mark.gpu


def test_etg1_to_device_csr(tmp_path, kron16):
    p = str(tmp_path / "c1.etg")
    eb.write_graph(p, 1 << 16, O.oracle_generate(16, 16, 1))
    g = eb.build_csr_from_file(p)
    row, col, _ = g.download()
    assert O.fnv1a64(row) == kron16["row_fnv"] and O.fnv1a64(col) == kron16["col_fnv"]
    tp = str(tmp_path / "c1.txt")
    n, pairs = eb.read_graph(p)
    eb.write_graph(tp, n, pairs[:5000], "text")
    gt = eb.build_csr_from_file(tp, "text")
    assert gt.vertex_count == 1 << 16


@pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built")
def test_device_tree_file_validates_in_reference(tmp_path, kron16):
    pairs = O.oracle_generate(16, 16, 1)
    g = eb.build_csr(1 << 16, pairs)
    cg = eb.relayout_csr(g, mh=-1)
    ref = O.RefCsr(1 << 16, pairs)
    for root, te in list(zip(kron16["roots"], kron16["traversed_edges"]))[:6]:
        r = eb.et_bfs(cg, int(cg.old2new[root]), want_depth=False)
        # BfsTree in original ids (translate_tree, validate.cpp:160-175)
        new2old = np.asarray(cg.new2old, np.uint64)
        par = np.full(cg.vertex_count, np.uint64(0xFFFFFFFFFFFFFFFF), np.uint64)
        ok = r.parent != np.uint64(0xFFFFFFFFFFFFFFFF)
        par[new2old[ok]] = new2old[r.parent[ok].astype(np.int64)]
        path = str(tmp_path / f"t{root}.ett")
        eb.write_tree(path, root, par)
        got_root, got = eb.read_tree(path)
        assert got_root == root and np.array_equal(got, par)
        valid, ref_te, rule = ref.validate(root, got)
        assert valid and ref_te == te, (root, rule)


@pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built")
def test_bench_report_v1_and_tree_out(tmp_path, kron16):
    """bench.py --report-json writes the reference's schema-v1 report; --tree-out the
    first root's tree, which the reference validates."""
    import json
    import os
    import subprocess
    import sys
    root_dir = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    rj, tt = str(tmp_path / "r.json"), str(tmp_path / "t.ett")
    subprocess.run([sys.executable, os.path.join(root_dir, "bench.py"), "--scale", "16",
                    "--steps", "1", "--warmup", "3", "--secondary", "0", "--no-paper-mode",
                    "--emulate-partitions", "", "--no-cpu-baseline",
                    "--report-json", rj, "--tree-out", tt], check=True, capture_output=True,
                   cwd=root_dir, timeout=600)
    rep = json.load(open(rj))
    assert rep["schema_version"] == 1
    assert set(rep) == {"schema_version", "config", "graph", "aggregate", "per_root"}
    assert set(rep["aggregate"]) == {"mean_gteps", "min_gteps", "max_gteps",
                                     "harmonic_mean_seconds", "preprocessing_seconds", "all_valid"}
    assert rep["aggregate"]["all_valid"] and len(rep["per_root"]) == 64
    assert [r["root"] for r in rep["per_root"]] == kron16["roots"]
    assert [r["traversed_edges"] for r in rep["per_root"]] == kron16["traversed_edges"]
    root, parent = eb.read_tree(tt)
    assert root == kron16["roots"][0]
    valid, te, rule = O.RefCsr(1 << 16, O.oracle_generate(16, 16, 1)).validate(root, parent)
    assert valid and te == kron16["traversed_edges"][0], rule
