"""Build the in-tree sm_100a shared library libetbfs_b200.so with nvcc.

Every .cu under csrc/ is compiled for `-gencode arch=compute_100a,code=sm_100a`
with -lineinfo (ncu source view) and linked into one .so exporting the C-ABI of
include/etbfs_cuda.h. Objects are cached by mtime under build/.
"""
from __future__ import annotations

import concurrent.futures as cf
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
OBJ = os.path.join(ROOT, "build", "obj")
LIB = os.path.join(HERE, "lib", "libetbfs_b200.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
CXX = "/usr/bin/g++"
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC,-O3", "--expt-relaxed-constexpr",
         "-I" + os.path.join(ROOT, "include")]


def sources():
    cu = sorted(os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith(".cu"))
    host = os.path.join(CSRC, "host")
    cpp = sorted(os.path.join(host, f) for f in os.listdir(host) if f.endswith(".cpp"))
    return cu + cpp


def headers():
    out = [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".cuh", ".h"))]
    host = os.path.join(CSRC, "host")
    out += [os.path.join(host, f) for f in os.listdir(host) if f.endswith(".hpp")]
    out.append(os.path.join(ROOT, "include", "etbfs_cuda.h"))
    return out


def _compile(src: str, verbose: bool) -> str:
    obj = os.path.join(OBJ, os.path.basename(src) + ".o")
    dep_mtime = max([os.path.getmtime(src)] + [os.path.getmtime(h) for h in headers()])
    if os.path.exists(obj) and os.path.getmtime(obj) >= dep_mtime:
        return obj
    if src.endswith(".cpp"):
        # The C++ drop-in (reference signatures, C++20 std::span) is host-only code.
        cmd = [CXX, "-std=c++20", "-O2", "-fPIC", "-Wall", "-Wextra",
               "-I" + os.path.join(ROOT, "include"), "-c", src, "-o", obj]
    else:
        cmd = [NVCC, *ARCH, *FLAGS, "-c", src, "-o", obj]
    if verbose and not src.endswith(".cpp"):
        cmd.insert(1, "-Xptxas=-v")
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed for {src}:\n{r.stderr}")
    if verbose and r.stderr:
        sys.stderr.write(r.stderr)
    return obj


def build(verbose: bool = False) -> str:
    os.makedirs(OBJ, exist_ok=True)
    os.makedirs(os.path.dirname(LIB), exist_ok=True)
    srcs = sources()
    with cf.ThreadPoolExecutor(max_workers=min(8, len(srcs))) as ex:
        objs = list(ex.map(lambda s: _compile(s, verbose), srcs))
    newest = max(os.path.getmtime(o) for o in objs)
    if not os.path.exists(LIB) or os.path.getmtime(LIB) < newest:
        cmd = [NVCC, *ARCH, "-shared", "-o", LIB, *objs, "-lcudart"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"link failed:\n{r.stderr}")
    return LIB


if __name__ == "__main__":
    print(build(verbose="-v" in sys.argv))


def build_cpp_tests() -> str:
    """tests/cpp/test_dropin: the C++ drop-in API test binary (links the library)."""
    src = os.path.join(ROOT, "tests", "cpp", "test_dropin.cpp")
    out = os.path.join(ROOT, "tests", "cpp", "bin", "test_dropin")
    os.makedirs(os.path.dirname(out), exist_ok=True)
    deps = [src, LIB] + [os.path.join(ROOT, "include", "etbfs", f)
                         for f in os.listdir(os.path.join(ROOT, "include", "etbfs"))]
    if os.path.exists(out) and os.path.getmtime(out) >= max(os.path.getmtime(d) for d in deps):
        return out
    cmd = [CXX, "-std=c++20", "-O2", "-Wall", "-I" + os.path.join(ROOT, "include"), src, "-o", out,
           "-L" + os.path.dirname(LIB), "-letbfs_b200",
           "-Wl,-rpath,$ORIGIN/../../../paper_2009_07463_b200/lib"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"test_dropin build failed:\n{r.stderr}")
    return out


def build_prims_test() -> str:
    """tests/cpp/test_prims: the preprocessing primitives (csrc/prims.cu) against
    host std:: algorithms (links the library; internal C++ symbols)."""
    src = os.path.join(ROOT, "tests", "cpp", "test_prims.cu")
    out = os.path.join(ROOT, "tests", "cpp", "bin", "test_prims")
    os.makedirs(os.path.dirname(out), exist_ok=True)
    deps = [src, LIB] + headers()
    if os.path.exists(out) and os.path.getmtime(out) >= max(os.path.getmtime(d) for d in deps):
        return out
    cmd = [NVCC, *ARCH, *FLAGS, src, "-o", out, "-L" + os.path.dirname(LIB), "-letbfs_b200",
           "-Xlinker", "-rpath,$ORIGIN/../../../paper_2009_07463_b200/lib"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"test_prims build failed:\n{r.stderr}")
    return out


REF_ACCEPTANCE = "/root/reference/proj/tests/acceptance.cpp"
ACCEPTANCE_BIN = os.path.join(ROOT, "tests", "cpp", "bin", "acceptance_ref")


def build_acceptance() -> str | None:
    """The reference's UNMODIFIED acceptance gate (proj/tests/acceptance.cpp,
    compiled where it lies) against include/ + libetbfs_b200.so: the drop-in
    headers must accept the reference's own caller, and the gate then runs on
    the GPU (tests/test_gpu_acceptance.py). Needs /root/reference (this
    container); the built binary travels to the GPU box with the snapshot."""
    if not os.path.exists(REF_ACCEPTANCE):
        return ACCEPTANCE_BIN if os.path.exists(ACCEPTANCE_BIN) else None
    os.makedirs(os.path.dirname(ACCEPTANCE_BIN), exist_ok=True)
    deps = [REF_ACCEPTANCE, LIB] + [os.path.join(ROOT, "include", "etbfs", f)
                                    for f in os.listdir(os.path.join(ROOT, "include", "etbfs"))]
    if os.path.exists(ACCEPTANCE_BIN) and \
            os.path.getmtime(ACCEPTANCE_BIN) >= max(os.path.getmtime(d) for d in deps):
        return ACCEPTANCE_BIN
    cmd = [CXX, "-std=c++20", "-O2", "-fopenmp", "-I" + os.path.join(ROOT, "include"),
           REF_ACCEPTANCE, "-o", ACCEPTANCE_BIN, "-L" + os.path.dirname(LIB), "-letbfs_b200",
           "-Wl,-rpath,$ORIGIN/../../../paper_2009_07463_b200/lib"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"acceptance build failed:\n{r.stderr[-4000:]}")
    return ACCEPTANCE_BIN
