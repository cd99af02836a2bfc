import sys, os, ctypes as C
import numpy as np
sys.path.insert(0, os.getcwd())
import paper_2009_07463_b200 as eb
from paper_2009_07463_b200 import etbfs as E
from bench import select_roots_from_degrees
scale = int(sys.argv[1]) if len(sys.argv) > 1 else 26
g = eb.generate_graph(scale=scale, edgefactor=16, seed=1)
cg = eb.relayout_csr(g, mh=-1)
roots = select_roots_from_degrees(g.degrees(), 64, 1)
starts = cg.old2new[roots.astype(np.int64)]
line = C.c_uint32()
bad = 0
for i, s in enumerate(starts[:16]):
    E.bfs_device(cg, int(s))
    v = E.result_validate(cg, int(s))
    E._check(E.lib().etb_debug_check_line(C.byref(line)))
    print(i, int(roots[i]), v["passed"], "check_line", line.value, flush=True)
    bad += not v["passed"]
print("bad", bad)
