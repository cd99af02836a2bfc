"""Run the ET-BFS kernel for ONE of the 64 seed-1 roots a few times (profiling aid).

  python tools/one_root.py --scale 26 --index 0 --reps 3
Under ncu: ncu -k regex:et_bfs -s <reps-1> -c 1 ... python tools/one_root.py ...
"""
import argparse
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2009_07463_b200 as eb  # noqa: E402
from paper_2009_07463_b200 import etbfs as E  # noqa: E402
from bench import select_roots_from_degrees  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--scale", type=int, default=26)
    ap.add_argument("--edgefactor", type=int, default=16)
    ap.add_argument("--mh", type=int, default=-1)
    ap.add_argument("--index", type=int, default=0)
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--parts", type=int, default=1, help="1D core partitions on this device")
    args = ap.parse_args()
    g = eb.generate_graph(scale=args.scale, edgefactor=args.edgefactor, seed=1)
    cg = eb.relayout_csr(g, mh=args.mh)
    if args.parts > 1:
        E.partition(cg, args.parts)
    roots = select_roots_from_degrees(g.degrees(), 64, 1)
    s = int(cg.old2new[int(roots[args.index])])
    ms, kms = E.time_roots(cg, np.full(args.reps, s, np.uint64), warmup=0, flush_l2=True)
    print("root", int(roots[args.index]), "start", s, "kernel_ms", [round(x, 4) for x in kms])


if __name__ == "__main__":
    main()
