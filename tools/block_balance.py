"""Per-level CTA balance of the persistent BFS kernel (diagnostics).

For a root: per level, the spread of the times at which CTAs finished their
step (min / median / max, µs since kernel entry) — the gap max - median is time
the grid waits at the level barrier for stragglers.
  python tools/block_balance.py --scale 22 --index 26
"""
import argparse
import ctypes as C
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2009_07463_b200 as eb  # noqa: E402
from paper_2009_07463_b200 import etbfs as E  # noqa: E402
from bench import select_roots_from_degrees  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--scale", type=int, default=22)
    ap.add_argument("--edgefactor", type=int, default=16)
    ap.add_argument("--index", type=int, nargs="+", default=[0])
    args = ap.parse_args()
    g = eb.generate_graph(scale=args.scale, edgefactor=args.edgefactor, seed=1)
    cg = eb.relayout_csr(g, mh=-1)
    roots = select_roots_from_degrees(g.degrees(), 64, 1)
    for idx in args.index:
        s = int(cg.old2new[int(roots[idx])])
        for _ in range(3):  # warm
            E.bfs_device(cg, s)
        E.time_roots(cg, np.array([s], np.uint64), warmup=0, flush_l2=True)
        cap = 64 * 4096
        out = np.zeros(cap, np.uint64)
        grid, levels = C.c_uint32(), C.c_uint32()
        E._check(E.lib().etb_debug_block_stamps(cg.handle, s, out.ctypes.data, cap, C.byref(grid),
                                                 C.byref(levels)))
        r = eb.et_bfs(cg, s, stats=True, want_parent=False, want_depth=False)
        G = grid.value
        ph = np.zeros(256, np.uint64)
        E._check(E.lib().etb_debug_phase_stamps(cg.handle, ph.ctypes.data))
        conv = {L: (int(ph[128 + L]) - int(ph[0])) / 1e3 for L in range(1, 64) if ph[128 + L]}
        print(f"root index {idx} trace {r.stats.direction_trace} claims {r.stats.level_claims}")
        ent = out[62 * G:63 * G].view(np.int64).astype(np.float64) / 1e3
        ext = out[63 * G:64 * G].view(np.int64).astype(np.float64) / 1e3
        print(f"  CTA entry us: min {ent.min():6.1f} max {ent.max():6.1f}   exit: min {ext.min():6.1f} "
              f"med {np.median(ext):6.1f} max {ext.max():6.1f}   (device total {r.stats.total_ns / 1e3:.1f})")
        for L in range(levels.value):
            t_all = out[L * G:(L + 1) * G].astype(np.float64) / 1e3
            t = t_all[t_all > 0]
            if t.size:
                slow = np.argsort(-t_all)[:3]
                print(f"  L{L} {r.stats.direction_trace[L]} step-end us: min {t.min():8.1f} "
                      f"med {np.median(t):8.1f} p90 {np.percentile(t, 90):8.1f} max {t.max():8.1f}"
                      f"   level_end {r.stats.level_ns[L + 1] / 1e3:8.1f}"
                      + (f"   (list ready at {conv[L]:8.1f})" if L in conv else "")
                      + f"   slowest CTAs {slow.tolist()}")


if __name__ == "__main__":
    main()
