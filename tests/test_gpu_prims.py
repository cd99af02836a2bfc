"""Runs tests/cpp/test_prims.cu on the GPU: the hand-written preprocessing
primitives (radix sort of keys and stable pairs, unique, flagged selection,
scans, reduction; csrc/prims.cu) against host std:: algorithms on seeded inputs
from 0 to 25M items and every digit width. The end-to-end CSR / relayout hashes
(test_gpu_parity*.py) check the same code through the reference's builds."""
import subprocess

import pytest

from conftest import ROOT

pytestmark = pytest.mark.gpu


def test_prims_vs_host():
    import sys
    sys.path.insert(0, ROOT)
    from paper_2009_07463_b200 import build_lib
    exe = build_lib.build_prims_test()
    r = subprocess.run([exe], capture_output=True, text=True, timeout=900)
    print(r.stdout[-4000:])
    assert r.returncode == 0, (r.stdout[-2000:], r.stderr[-2000:])
    assert "prims ok" in r.stdout
