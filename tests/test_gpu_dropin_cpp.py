"""Runs the C++ drop-in test binary (tests/cpp/test_dropin.cpp): the reference's
public C++ API, driven like the reference's own unit tests, on the GPU."""
import os
import subprocess

import pytest

from conftest import ROOT

pytestmark = pytest.mark.gpu


def test_cpp_dropin_api():
    import sys
    sys.path.insert(0, ROOT)
    from paper_2009_07463_b200 import build_lib
    exe = build_lib.build_cpp_tests()
    r = subprocess.run([exe], capture_output=True, text=True, timeout=900)
    print(r.stdout)
    print(r.stderr[-4000:])
    assert r.returncode == 0, r.stderr[-4000:]
    assert "0 failures" in r.stdout
