"""Build an A/B variant of the library: the normal objects, with the listed
sources recompiled under extra nvcc flags, linked into
tools/variants/<name>/libetbfs_b200.so (run it with ETB_LIB=<that path>).

  python tools/build_variant.py r8 -DETB_REPLAY=8 -- bfs.cu
"""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2009_07463_b200 import build_lib as B  # noqa: E402


def main():
    name = sys.argv[1]
    rest = sys.argv[2:]
    cut = rest.index("--")
    flags, files = rest[:cut], rest[cut + 1:]
    B.build()
    out_dir = os.path.join(ROOT, "tools", "variants", name)
    os.makedirs(out_dir, exist_ok=True)
    objs = []
    for src in B.sources():
        obj = os.path.join(B.OBJ, os.path.basename(src) + ".o")
        if os.path.basename(src) in files:
            vobj = os.path.join(out_dir, os.path.basename(src) + ".o")
            subprocess.run([B.NVCC, *B.ARCH, *B.FLAGS, *flags, "-c", src, "-o", vobj], check=True)
            obj = vobj
        objs.append(obj)
    lib = os.path.join(out_dir, "libetbfs_b200.so")
    subprocess.run([B.NVCC, *B.ARCH, "-shared", "-o", lib, *objs, "-lcudart"], check=True)
    print(lib)


if __name__ == "__main__":
    main()
