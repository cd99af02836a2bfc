"""Per-warp phase times of the top-down levels (diagnostics; needs a library
built with -DETB_WARP_STAMPS, selected with ETB_LIB).

For every top-down level of a root after level 0: per warp, its first chunk's
start (µs since kernel entry) and the time to each phase boundary — list
position known, columns loaded, visited words loaded, claim atomics returned,
chunk done (flush included) — as percentiles over the warps, plus the slowest
warps.
  ETB_LIB=.../ab_ws.so python tools/warp_stamps.py --scale 22 --index 0 4
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

GHZ = 1.965
PH = ["qp", "cols", "visited", "claims", "done"]


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
        r = eb.et_bfs(cg, s, stats=True, want_parent=False, want_depth=False)
        trace, claims = r.stats.direction_trace, r.stats.level_claims
        print(f"root index {idx} trace {trace} claims {claims}")
        for L in range(1, len(trace)):
            if trace[L] != "t" or claims[L] == 0:
                continue
            for _ in range(2):
                E.bfs_device(cg, s)
            E.time_roots(cg, np.array([s], np.uint64), warmup=0, flush_l2=True)
            cap = 8 * 148 * 32
            out = np.zeros(cap, np.uint64)
            nw = C.c_uint32()
            E._check(E.lib().etb_debug_warp_stamps(cg.handle, s, L + 1, out.ctypes.data, cap,
                                                    C.byref(nw)))
            w = out[: 8 * nw.value].reshape(-1, 8).astype(np.float64)
            w = w[w[:, 5] > 0]
            if not len(w):
                print(f"  L{L}: no stamps (start not in the core, or a non-stamp build)")
                continue
            st = w[:, 0] / 1e3
            ph = w[:, 1:6] / (GHZ * 1e3)
            print(f"  L{L} t claims {claims[L]}: {len(w)} warps, first chunk start us "
                  f"min {st.min():.1f} med {np.median(st):.1f} max {st.max():.1f}; "
                  f"single-row chunks {int(w[:, 7].sum())}")
            for k, name in enumerate(PH):
                x = ph[:, k]
                print(f"    -> {name:8s} us  p10 {np.percentile(x, 10):6.2f}  med {np.median(x):6.2f}"
                      f"  p90 {np.percentile(x, 90):6.2f}  max {x.max():6.2f}")
            slow = np.argsort(-(st + ph[:, 4]))[:8]
            for j in slow:
                print("    slow warp: start {:6.1f}  ".format(st[j])
                      + "  ".join(f"{n} {ph[j, k]:6.2f}" for k, n in enumerate(PH))
                      + f"  chunk {int(w[j, 6])} single {int(w[j, 7])}")


if __name__ == "__main__":
    main()
