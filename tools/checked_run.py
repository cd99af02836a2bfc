"""Run the corpus, s16 and small stress graphs through a checked build
(-DETB_DEBUG_CHECKS, ETB_LIB=tools/variants/checked/libetbfs_b200.so): after
every traversal read the first failed device check's source line; report the
graph, start, kernel and line of every failure and validate every result."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))


def main():
    import ctypes as C

    import paper_2009_07463_b200 as eb
    from conftest import edges_of, load_golden
    from paper_2009_07463_b200 import etbfs as E
    line = C.c_uint32()
    fails = 0
    graphs = [(g["name"], eb.build_csr(g["n"], edges_of(g))) for g in load_golden("corpus.json")["graphs"]]
    graphs.append(("kron14", eb.generate_graph(scale=14, edgefactor=16, seed=1)))
    graphs.append(("kron12ef4", eb.generate_graph(scale=12, edgefactor=4, seed=3)))
    n_whole = []
    for name, csr in graphs:
        layouts = [("mh-1", eb.relayout_csr(csr, mh=-1)), ("mh0", eb.relayout_csr(csr, mh=0)),
                   ("whole", eb.relayout_csr(csr, types=np.zeros(csr.vertex_count, np.uint8), mh=-1))]
        for lname, cg in layouts:
            n = cg.vertex_count
            starts = range(n) if n <= 400 else np.linspace(0, n - 1, 24).astype(int)
            for parts in (1, 2, 3):
                E.partition(cg, parts)
                for k in (E.CoreKernel.HYBRID, E.CoreKernel.TOP_DOWN, E.CoreKernel.BLOCK_SEARCH):
                    for s in starts:
                        rep = E.TreeReplay.TEOLV if lname == "mh0" else E.TreeReplay.TEET
                        E.bfs_device(cg, int(s), kernel=k, replay=rep)
                        ok = E.result_validate(cg, int(s))["passed"]
                        E._check(E.lib().etb_debug_check_line(C.byref(line)))
                        if line.value or not ok:
                            fails += 1
                            if fails <= 30:
                                print(f"FAIL {name} {lname} parts={parts} {k.name} start={s} "
                                      f"line={line.value} valid={ok}", flush=True)
            E.partition(cg, 1)
    print("checked_run: failures", fails, flush=True)
    sys.exit(1 if fails else 0)


if __name__ == "__main__":
    main()
