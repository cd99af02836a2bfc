"""Per-partition level timing of the 1D core partition emulated on one GPU.

For each partition count G and the first --roots seed-1 roots, one traversal
with per-CTA step-end stamps (etb_debug_block_stamps); prints per level the
step-end time (us since kernel entry) of each partition's slowest CTA, so the
load balance between partitions (vertex-range ownership of a degree-sorted
core) is visible, and the per-level work counters of the single-partition run.

  python tools/part_balance.py --scale 26 --parts 1,2,4,8 --roots 4
"""
import argparse
import ctypes as C
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import paper_2009_07463_b200 as eb
    from paper_2009_07463_b200 import etbfs as E
    from bench import select_roots_from_degrees
    ap = argparse.ArgumentParser()
    ap.add_argument("--scale", type=int, default=26)
    ap.add_argument("--parts", default="1,2,4,8")
    ap.add_argument("--roots", type=int, default=4)
    a = ap.parse_args()
    g = eb.generate_graph(scale=a.scale, edgefactor=16, seed=1)
    cg = eb.relayout_csr(g, mh=-1)
    roots = select_roots_from_degrees(g.degrees(), 64, 1)[: a.roots]
    starts = cg.old2new[roots.astype(np.int64)]
    for G in [int(x) for x in a.parts.split(",")]:
        E.partition(cg, G)
        for s in starts:
            for _ in range(2):  # warm
                E.bfs_device(cg, int(s))
            cap = 64 * 160
            out = np.zeros(cap, np.uint64)
            grid, nl = C.c_uint32(), C.c_uint32()
            E._check(E.lib().etb_debug_block_stamps(cg.handle, int(s), out.ctypes.data, cap,
                                                    C.byref(grid), C.byref(nl)))
            gr = grid.value
            st = out[: 64 * gr].reshape(64, gr).astype(np.float64) / 1e3
            gs = gr // G
            r = eb.et_bfs(cg, int(s), stats=True, want_parent=False, want_depth=False)
            lines = []
            for L in range(min(nl.value, 62)):
                row = st[L]
                if not row.any():
                    continue
                per = [float(row[k * gs:(k + 1) * gs].max()) for k in range(G)]
                lines.append(f"L{L}{r.stats.direction_trace[L:L+1]}:" +
                             "/".join(f"{x:.1f}" for x in per))
            end = float(st[63].max())
            print(f"G={G} root={int(s)} total={r.stats.total_ns/1e3:.1f}us exit={end:.1f} "
                  + " ".join(lines), flush=True)
        E.partition(cg, 1)


if __name__ == "__main__":
    main()
