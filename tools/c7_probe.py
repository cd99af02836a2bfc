"""Per-root cost of the drop-in's timed call (etb_bfs with a host u64 parent
array, as run_benchmark times it) at scale 20: ET layout vs whole graph, with
and without top-down levels executed bottom-up."""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import paper_2009_07463_b200 as eb
    from paper_2009_07463_b200 import etbfs as E
    from bench import select_roots_from_degrees
    g = eb.generate_graph(scale=20, edgefactor=16, seed=1)
    n = g.vertex_count
    roots = select_roots_from_degrees(g.degrees(), 64, 2)
    for name, cg in (("et", eb.relayout_csr(g, mh=-1)),
                     ("whole", eb.relayout_csr(g, types=np.zeros(n, np.uint8), mh=-1))):
        starts = cg.old2new[roots.astype(np.int64)]
        par = np.empty(n, np.uint64)
        E._check(E.lib().etb_host_register(par.ctypes.data, par.nbytes))
        ts = []
        for s in starts:
            t0 = time.perf_counter()
            E._check(E.lib().etb_bfs(cg.handle, int(s), None, None, par.ctypes.data, None))
            ts.append(time.perf_counter() - t0)
        E._check(E.lib().etb_host_unregister(par.ctypes.data))
        ms, kms = E.time_roots(cg, starts, warmup=8, flush_l2=False)
        r = eb.et_bfs(cg, int(starts[0]), stats=True, want_parent=False, want_depth=False)
        print(name, os.environ.get("ETB_TD_AS_BU"), "call ms mean %.3f median %.3f max %.3f" %
              (1e3 * np.mean(ts), 1e3 * np.median(ts), 1e3 * np.max(ts)),
              "kernel ms mean %.4f max %.4f" % (np.mean(kms), np.max(kms)),
              r.stats.direction_trace, flush=True)


if __name__ == "__main__":
    main()
