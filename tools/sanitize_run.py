"""Small driver for compute-sanitizer (racecheck / synccheck / memcheck): a few
roots of an s12 graph through the single-partition kernel (both ET modes, the
hybrid, top-down and block-search drivers) and the partitioned kernel (G = 2,
device and system scope), every result checked by the device validator.

  compute-sanitizer --tool racecheck python tools/sanitize_run.py
"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import paper_2009_07463_b200 as eb
    from paper_2009_07463_b200 import etbfs as E
    from bench import select_roots_from_degrees
    g = eb.generate_graph(scale=12, edgefactor=16, seed=1)
    roots = select_roots_from_degrees(g.degrees(), 6, 1)
    bad = 0
    for mh, rep in ((-1, E.TreeReplay.TEET), (0, E.TreeReplay.TEOLV)):
        cg = eb.relayout_csr(g, mh=mh)
        starts = cg.old2new[roots.astype(np.int64)]
        runs = [(1, False), (2, False), (2, True)]
        for parts, sys_scope in runs:
            E.partition(cg, parts, system_scope=sys_scope)
            for k in (E.CoreKernel.HYBRID, E.CoreKernel.TOP_DOWN, E.CoreKernel.BLOCK_SEARCH):
                for s in starts:
                    E.bfs_device(cg, int(s), kernel=k, replay=rep)
                    bad += not E.result_validate(cg, int(s))["passed"]
        E.partition(cg, 1)
    print("sanitize_run: invalid results", bad, flush=True)
    sys.exit(1 if bad else 0)


if __name__ == "__main__":
    main()
