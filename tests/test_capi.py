"""CPU-side checks of the C-ABI boundary: the sm_100a library is built for
sm_100a, loads, exports every symbol include/etbfs_cuda.h declares, and fails
loudly (never falls back to a CPU path) when no GPU is present."""
import os
import re
import subprocess

import numpy as np
import pytest

import paper_2009_07463_b200 as eb
from conftest import ROOT

HEADER = os.path.join(ROOT, "include", "etbfs_cuda.h")


def declared_symbols():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(etb_[a-z0-9_]+)\s*\(", text)))


def test_header_declares_the_boundary():
    syms = declared_symbols()
    for s in ("etb_generate_kronecker", "etb_graph_from_edges", "etb_classify",
              "etb_peak_height", "etb_layout_build", "etb_layout_download_etl", "etb_bfs",
              "etb_bfs_device", "etb_time_roots"):
        assert s in syms


def test_library_exports_every_declared_symbol():
    L = eb.lib()
    for s in declared_symbols():
        assert hasattr(L, s), s
    out = subprocess.run(["nm", "-D", "--defined-only", eb.lib_path()], capture_output=True,
                         text=True).stdout
    for s in declared_symbols():
        assert re.search(rf"\bT {s}\b", out), s


def test_library_is_sm100a():
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", eb.lib_path()],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_no_cpu_fallback_without_gpu():
    if os.path.exists("/dev/nvidia0"):
        pytest.skip("GPU present")
    with pytest.raises(RuntimeError, match="CUDA"):
        eb.generate_graph(scale=8)
    with pytest.raises(RuntimeError, match="CUDA"):
        eb.build_csr(4, np.array([[0, 1]], np.uint64))


def test_caller_errors_use_reference_messages_before_touching_the_gpu():
    # build_csr validates endpoints first (build.cpp:26-31), exactly like the reference.
    with pytest.raises(ValueError, match="endpoint out of range at edge index 2"):
        eb.build_csr(3, np.array([[0, 1], [1, 2], [2, 3]], np.uint64))
    with pytest.raises(ValueError, match="scale > 48"):
        eb.generate_kronecker(scale=49)
    with pytest.raises(ValueError, match="probabilities must sum to 1"):
        eb.generate_kronecker(scale=4, a=0.5)
