"""Graph / parent-tree files (include/etbfs/io.hpp, csrc/host/etbfs_io.cpp) against
the reference's formats (proj/include/etbfs/io.hpp:9-45, proj/src/io.cpp:47-181).

Restates the reference's own io tests (proj/tests/test_io.cpp: documented byte
layout, write-read-write fixpoint, edgeless graphs, text header, headerless
inference, CRLF/padding/comments, error locations), pins the ETG1 file of the
C1 tuples to SURVEY.md Appendix A's SHA-256, and — with oracle/_ref built — checks
byte identity and identical error messages against the compiled reference.
Host-only code: runs without a GPU."""
import ctypes as C
import hashlib
import os

import numpy as np
import pytest

import oracle as O
import paper_2009_07463_b200 as eb

NO = np.uint64(0xFFFFFFFFFFFFFFFF)


def u64le(*vals):
    return b"".join(int(v).to_bytes(8, "little") for v in vals)


def rand_pairs(n, m, seed):
    rng = np.random.default_rng(seed)
    return rng.integers(0, n, size=(m, 2), dtype=np.uint64)


def err(fn):
    with pytest.raises((RuntimeError, ValueError)) as e:
        fn()
    return str(e.value)


# ---- the reference's byte layouts (test_io.cpp cases, restated) ---------------
def test_binary_layout_exact(tmp_path):
    p = str(tmp_path / "layout.etg")
    eb.write_graph(p, 3, np.array([[0, 2], [2, 1]], np.uint64))
    assert open(p, "rb").read() == b"ETG1" + u64le(3, 2, 0, 2, 2, 1)


def test_write_read_write_fixpoint(tmp_path):
    a, b = str(tmp_path / "a.etg"), str(tmp_path / "b.etg")
    pairs = rand_pairs(90, 400, 11)
    eb.write_graph(a, 90, pairs)
    n, got = eb.read_graph(a)
    eb.write_graph(b, n, got)
    assert open(a, "rb").read() == open(b, "rb").read()
    assert n == 90 and np.array_equal(got, pairs)


@pytest.mark.parametrize("fmt", ["binary", "text"])
def test_edgeless_keeps_vertex_count(tmp_path, fmt):
    p = str(tmp_path / "empty")
    eb.write_graph(p, 5, np.empty((0, 2), np.uint64), fmt)
    n, got = eb.read_graph(p, fmt)
    assert n == 5 and got.shape == (0, 2)


def test_text_header_and_inference(tmp_path):
    p = str(tmp_path / "h.txt")
    eb.write_graph(p, 3, np.array([[0, 2], [2, 1]], np.uint64), "text")
    assert open(p).read() == "# vertices 3\n0 2\n2 1\n"
    assert eb.read_graph(p, "text")[0] == 3
    open(p, "w").write("4 9\n1 0\n")
    n, got = eb.read_graph(p, "text")
    assert n == 10 and got.tolist() == [[4, 9], [1, 0]]
    open(p, "wb").write(b"# vertices 6\r\n\r\n# a comment\n  2   5 \r\n\n0 1\r\n")
    n, got = eb.read_graph(p, "text")
    assert n == 6 and got.tolist() == [[2, 5], [0, 1]]


def test_error_locations(tmp_path):
    p = str(tmp_path / "bad")
    open(p, "w").write("0 1\nlonely\n")
    m = err(lambda: eb.read_graph(p, "text"))
    assert 'expected "src dst"' in m and "line 2" in m and p in m
    open(p, "w").write("0 x\n")
    assert 'expected an unsigned integer, got "x"' in err(lambda: eb.read_graph(p, "text"))
    open(p, "w").write("# vertices 2\n0 5\n")
    assert "edge endpoint out of range (line 2)" in err(lambda: eb.read_graph(p, "text"))
    open(p, "wb").write(b"ETG2" + u64le(1, 0))
    assert "bad magic, expected ETG1 (byte offset 0)" in err(lambda: eb.read_graph(p))
    open(p, "wb").write(b"ETG1" + u64le(4, 3) + u64le(0, 1))
    assert "file too short for declared edge count (byte offset 20)" in err(lambda: eb.read_graph(p))
    open(p, "wb").write(b"ETG1" + u64le(4, 2) + u64le(0, 1, 3, 4))
    assert "edge endpoint out of range (byte offset 36)" in err(lambda: eb.read_graph(p))
    open(p, "wb").write(b"ETG1" + u64le(1 << 49, 0))
    assert "vertex count exceeds the supported maximum (byte offset 4)" in err(
        lambda: eb.read_graph(p))
    assert "cannot open for reading" in err(lambda: eb.read_graph(str(tmp_path / "missing")))
    assert 'unknown graph format "csv" (binary or text)' in err(lambda: eb.parse_graph_format("csv"))


def test_tree_files(tmp_path):
    p = str(tmp_path / "t.ett")
    parent = np.array([1, 1, NO, 1], np.uint64)
    eb.write_tree(p, 1, parent)
    assert open(p, "rb").read() == b"ETT1" + u64le(4, 1, 1, 1, int(NO), 1)
    root, got = eb.read_tree(p)
    assert root == 1 and np.array_equal(got, parent)
    open(p, "wb").write(b"ETT1" + u64le(2, 5))
    assert "root out of range (byte offset 12)" in err(lambda: eb.read_tree(p))
    open(p, "wb").write(b"ETT1" + u64le(3, 0, 0))
    assert "unexpected end of file (byte offset 28)" in err(lambda: eb.read_tree(p))
    open(p, "wb").write(b"ETG1" + u64le(0, 0))
    assert "bad magic, expected ETT1" in err(lambda: eb.read_tree(p))


# ---- golden anchor: SURVEY.md Appendix A ----------------------------------------
def test_c1_etg1_sha256(tmp_path, kron16):
    """The ETG1 file of the C1 tuples (s16/ef16, seed 1) hashes to the anchor measured
    from the compiled reference's write_graph."""
    pairs = O.oracle_generate(16, 16, 1)
    p = str(tmp_path / "c1.etg")
    eb.write_graph(p, 1 << 16, pairs)
    data = open(p, "rb").read()
    assert len(data) == 16_777_236
    assert hashlib.sha256(data).hexdigest() == (
        "6ed6678270d5057938b8700e2e901660d4f87819469f52375842402544745b39")
    n, back = eb.read_graph(p)
    assert n == 1 << 16 and O.fnv1a64(back) == kron16["tuples_fnv"]


# ---- the compiled reference, live ----------------------------------------------
needs_ref = pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built")


def ref_err(rc):
    assert rc != 0
    return O.ref().ref_last_error().decode()


@needs_ref
@pytest.mark.parametrize("fmt", ["binary", "text"])
def test_byte_identical_to_reference(tmp_path, fmt):
    R = O.ref()
    text = int(fmt == "text")
    for n, m, seed in [(90, 400, 11), (1, 0, 0), (1000, 5000, 3)]:
        pairs = rand_pairs(n, m, seed) if m else np.empty((0, 2), np.uint64)
        ours, theirs = str(tmp_path / "ours"), str(tmp_path / "theirs")
        eb.write_graph(ours, n, pairs, fmt)
        flat = np.ascontiguousarray(pairs).reshape(-1)
        assert R.ref_write_graph(os.fsencode(theirs), text, n, flat.ctypes.data, m) == 0
        assert open(ours, "rb").read() == open(theirs, "rb").read()
        rn, rm = C.c_uint64(), C.c_uint64()
        assert R.ref_read_graph(os.fsencode(ours), text, C.byref(rn), C.byref(rm), None) == 0
        back = np.empty(2 * rm.value, np.uint64)
        assert R.ref_read_graph(os.fsencode(ours), text, C.byref(rn), C.byref(rm),
                                back.ctypes.data) == 0
        assert rn.value == n and np.array_equal(back.reshape(-1, 2), pairs)


@needs_ref
def test_error_messages_match_reference(tmp_path):
    R = O.ref()
    p = str(tmp_path / "bad")
    cases = [
        ("text", b"0 1\nlonely\n"), ("text", b"0 x\n"), ("text", b"# vertices 2\n0 5\n"),
        ("text", b"5 y 7\n"), ("text", b"# vertices q\n"), ("text", b"-1 2\n"),
        ("binary", b"ETG2" + u64le(1, 0)), ("binary", b"ET"), ("binary", b"ETG1" + u64le(4)),
        ("binary", b"ETG1" + u64le(4, 3) + u64le(0, 1)),
        ("binary", b"ETG1" + u64le(4, 2) + u64le(0, 1, 3, 4)),
        ("binary", b"ETG1" + u64le(1 << 49, 0)),
    ]
    for fmt, data in cases:
        open(p, "wb").write(data)
        n, m = C.c_uint64(), C.c_uint64()
        theirs = ref_err(R.ref_read_graph(os.fsencode(p), int(fmt == "text"), C.byref(n),
                                          C.byref(m), None))
        assert err(lambda: eb.read_graph(p, fmt)) == theirs, (fmt, data)
    for data in [b"ETT1" + u64le(2, 5), b"ETT1" + u64le(3, 0, 0), b"ETG1" + u64le(0, 0),
                 b"ETT1" + u64le(1 << 50, 0), b"ETT1" + u64le(2)]:
        open(p, "wb").write(data)
        n, root = C.c_uint64(), C.c_uint64()
        theirs = ref_err(R.ref_read_tree(os.fsencode(p), C.byref(n), C.byref(root), None))
        assert err(lambda: eb.read_tree(p)) == theirs, data


@needs_ref
def test_tree_files_cross_read(tmp_path):
    R = O.ref()
    rng = np.random.default_rng(5)
    parent = rng.integers(0, 500, size=500, dtype=np.uint64)
    parent[rng.integers(0, 500, size=40)] = NO
    ours, theirs = str(tmp_path / "o.ett"), str(tmp_path / "t.ett")
    eb.write_tree(ours, 7, parent)
    assert R.ref_write_tree(os.fsencode(theirs), parent.size, 7, parent.ctypes.data) == 0
    assert open(ours, "rb").read() == open(theirs, "rb").read()
    n, root = C.c_uint64(), C.c_uint64()
    back = np.empty(500, np.uint64)
    assert R.ref_read_tree(os.fsencode(ours), C.byref(n), C.byref(root), back.ctypes.data) == 0
    assert (n.value, root.value) == (500, 7) and np.array_equal(back, parent)
