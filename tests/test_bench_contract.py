"""bench.py's JSON contract: the reference arm on CPU (small scale, runs here
when oracle/_ref is built) and our arm on the GPU — one JSON line on stdout
with the keys the driver reads, numbers of the right kind."""
import json
import os
import subprocess
import sys

import pytest

import oracle as O

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BASE_KEYS = {"metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
             "higher_is_better", "scaling", "vs_baseline", "dtype", "data", "config", "e2e"}


def run_bench(*args, timeout=900):
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], cwd=ROOT,
                       capture_output=True, text=True, timeout=timeout)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout[-2000:]
    return json.loads(lines[0])


def check_common(d, steps, warmup):
    assert BASE_KEYS <= set(d), BASE_KEYS - set(d)
    assert d["n_gpus"] == 1 and d["steps"] == steps and d["warmup"] == warmup
    assert d["value"] > 0 and d["ms_per_step"] > 0 and d["higher_is_better"] is True
    assert d["unit"] == "GTEPS" and d["data"] == "synthetic"
    assert d["config"]["workload"].startswith("kronecker-s")
    e = d["e2e"]
    assert {"value", "unit", "h2d_bytes_per_step", "d2h_bytes_per_step"} <= set(e)


@pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built")
def test_reference_arm_line():
    d = run_bench("--impl", "reference", "--scale", "12", "--steps", "1", "--warmup", "3")
    check_common(d, 1, 3)
    assert d["impl"] == "reference"
    cb = d["cpu_baseline"]
    assert cb["kind"] == "reference" and cb["cores"] >= 1 and cb["value"] == d["value"]
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["d2h_bytes_per_step"] == 0


@pytest.mark.gpu
def test_gpu_arm_line():
    d = run_bench("--scale", "16", "--steps", "1", "--warmup", "3", "--no-cpu-baseline",
                  "--secondary", "0", "--no-paper-mode")
    check_common(d, 1, 3)
    r = d["roofline"]
    assert r["bound"] == "hbm" and r["unit"] == "GB/s" and r["peak"] > 0
    assert abs(r["frac"] - r["achieved"] / r["peak"]) < 1e-3
    # the work model: every traversal moves at least its bitmaps and results
    assert 0 < r["algorithmic_bytes_per_launch"] < r["b_alg"]["bytes_per_bfs"]
    assert r["frac"] <= 1.2
    assert d["gpu_launches"] == 64  # one traversal kernel per root of the step
    assert d["e2e"]["d2h_bytes_per_step"] > 0 and d["e2e"]["h2d_bytes_per_step"] > 0
    c = d["clocks"]
    assert {"sm_mhz", "sm_max_mhz", "reasons"} <= set(c)
    assert d["detail"]["all_valid"] is True


def test_gpus_flag_spawns_ranks():
    """--gpus N outside torchrun re-launches bench.py as N ranks (the driver's
    SCALE runs); every rank sees WORLD_SIZE = N (plumbing only, no GPU work)."""
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2",
                        "--dry-ranks"], cwd=ROOT, capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [json.loads(ln) for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert sorted(d["rank"] for d in lines) == [0, 1]
    assert all(d["n_gpus"] == 2 for d in lines)
