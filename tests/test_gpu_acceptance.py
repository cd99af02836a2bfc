"""The reference's own acceptance gate (proj/tests/acceptance.cpp, criteria 1-8,
SPEC.md:636-654), compiled UNMODIFIED against the drop-in headers include/etbfs
and linked with libetbfs_b200.so (build_lib.build_acceptance, in the container
that has /root/reference; the binary travels to the GPU box). Every call it
makes — generator, CSR, classification, relayout, ETL, the whole-graph and
composite kernels, the oracle, the validator and run_benchmark — runs on the
B200 through the C-ABI."""
import os
import subprocess

import pytest

from conftest import ROOT

pytestmark = [pytest.mark.gpu, pytest.mark.slow]

BIN = os.path.join(ROOT, "tests", "cpp", "bin", "acceptance_ref")


@pytest.mark.skipif(not os.path.exists(BIN), reason="acceptance_ref not built (needs /root/reference)")
def test_reference_acceptance_gate_on_gpu():
    r = subprocess.run([BIN], capture_output=True, text=True, timeout=2400)
    print(r.stdout)
    print(r.stderr[-4000:])
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith(("PASS", "FAIL"))]
    assert len(lines) == 8, r.stdout[-4000:]
    assert all(ln.startswith("PASS") for ln in lines), "\n".join(lines)
    assert r.returncode == 0
