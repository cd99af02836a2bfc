"""Diagnose top-down-only traversals at scale 20 (acceptance criterion 7's
run_benchmark(kTopDown)): validate every root, whole-graph and ET layouts."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np
import paper_2009_07463_b200 as eb
from paper_2009_07463_b200 import etbfs as E
import oracle as O

scale = int(sys.argv[1]) if len(sys.argv) > 1 else 20
g = eb.generate_graph(scale=scale, edgefactor=16, seed=1)
n = g.vertex_count
ocsr = O.OracleCsr(n, O.oracle_generate(scale, 16, 1))
roots = ocsr.select_roots(64, 2)
for name, cg in [("whole", eb.relayout_csr(g, types=np.zeros(n, np.uint8), mh=-1)),
                 ("et", eb.relayout_csr(g, mh=-1))]:
    for kern in (E.CoreKernel.TOP_DOWN, E.CoreKernel.HYBRID, E.CoreKernel.BLOCK_SEARCH):
        bad = 0
        for r in roots:
            s = int(cg.old2new[int(r)])
            res = eb.et_bfs(cg, s, kernel=kern, stats=True, want_parent=False, want_depth=False)
            v = E.result_validate(cg, s)
            lv, _ = E.result_original(cg, parent=False)
            ok = (lv == ocsr.levels(int(r))).all()
            if not v["passed"] or not ok:
                bad += 1
                if bad <= 3:
                    print(name, kern.name, "root", int(r), "levels_ok", ok, v, res.stats.direction_trace,
                          res.stats.level_claims, flush=True)
        print(name, kern.name, "bad roots", bad, "of", len(roots), "nc", cg.core_vertex_count, flush=True)
