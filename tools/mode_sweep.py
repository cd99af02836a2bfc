"""The bench protocol over the other ET modes and the core kernels (diagnostics):
for each (mh, replay, kernel) combination, the 64 seed-1 roots timed as in
bench.py (L2 flushed between roots, events around the launch), every root
validated on the device (validate_bfs_tree rules 1-5), harmonic-mean GTEPS
with the reference's TE.
  python tools/mode_sweep.py --scale 26
"""
import argparse
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2009_07463_b200 as eb  # noqa: E402
from paper_2009_07463_b200 import etbfs as E  # noqa: E402
from bench import harmonic_gteps, select_roots_from_degrees  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--scale", type=int, default=22)
    ap.add_argument("--edgefactor", type=int, default=16)
    args = ap.parse_args()
    g = eb.generate_graph(scale=args.scale, edgefactor=args.edgefactor, seed=1)
    roots = select_roots_from_degrees(g.degrees(), 64, 1)
    combos = [(-1, E.TreeReplay.TEET, E.CoreKernel.HYBRID),
              (0, E.TreeReplay.TEOLV, E.CoreKernel.HYBRID),
              (0, E.TreeReplay.TEET, E.CoreKernel.HYBRID),
              (-1, E.TreeReplay.TEET, E.CoreKernel.TOP_DOWN)]
    for mh, replay, kernel in combos:
        cg = eb.relayout_csr(g, mh=mh)
        starts = cg.old2new[roots.astype(np.int64)]
        ms, _ = E.time_roots(cg, starts, warmup=8, flush_l2=True, replay=replay, kernel=kernel,
                             kernel_times=False)
        te = np.empty(len(starts), np.float64)
        ok = 0
        for i, s in enumerate(starts):
            E.bfs_device(cg, int(s), replay=replay, kernel=kernel)
            ok += E.result_validate(cg, int(s))["passed"]
            te[i] = E.result_traversed_edges(cg)
        hm, _ = harmonic_gteps(te, np.asarray(ms) / 1e3)
        print(json.dumps({"scale": args.scale, "mh": mh, "replay": replay.name,
                          "kernel": kernel.name, "hm_gteps": round(hm, 1),
                          "mean_us": round(float(np.mean(ms)) * 1e3, 1),
                          "valid": f"{ok}/{len(starts)}", "core": int(cg.core_vertex_count)}),
              flush=True)


if __name__ == "__main__":
    main()
