"""A/B of environment-controlled kernel variants on the bench protocol.

Each variant is run in its own process (layouts read the env at creation):
64 seed-1 roots x --steps, L2 flushed between roots, CUDA events; prints the
harmonic-mean GTEPS and mean ms per root, and validates every root once.

  python tools/ab_env.py --scale 26 --variants "ETB_HOT_WORDS=0" "ETB_HOT_WORDS=32768"
"""
import argparse
import json
import os
import subprocess
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def child(args):
    import paper_2009_07463_b200 as eb
    from paper_2009_07463_b200 import etbfs as E
    from bench import harmonic_gteps, select_roots_from_degrees
    g = eb.generate_graph(scale=args.scale, edgefactor=args.edgefactor, seed=1)
    cg = eb.relayout_csr(g, mh=args.mh)
    if args.parts > 1:  # the 1D core partition, G partitions emulated on this GPU
        E.partition(cg, args.parts)
    roots = select_roots_from_degrees(g.degrees(), 64, 1)
    starts = cg.old2new[roots.astype(np.int64)]
    te = np.empty(64)
    ok = 0
    for i, s in enumerate(starts):
        E.bfs_device(cg, int(s))
        te[i] = E.result_traversed_edges(cg)
        ok += bool(E.result_validate(cg, int(s))["passed"])
    ms, _ = E.time_roots(cg, np.tile(starts, args.steps), warmup=64, flush_l2=True,
                         kernel_times=False)
    hm, _ = harmonic_gteps(np.tile(te, args.steps), ms / 1e3)
    per = ms.reshape(args.steps, 64).mean(axis=0)
    print(json.dumps({"hm": round(hm, 2), "ms": round(float(ms.mean()), 4), "valid": ok,
                      "slowest": [round(float(x), 3) for x in np.sort(per)[-4:]]}))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--scale", type=int, default=26)
    ap.add_argument("--edgefactor", type=int, default=16)
    ap.add_argument("--mh", type=int, default=-1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--parts", type=int, default=1)
    ap.add_argument("--repeat", type=int, default=1)
    ap.add_argument("--variants", nargs="*", default=[])
    ap.add_argument("--child", action="store_true")
    args = ap.parse_args()
    if args.child:
        return child(args)
    for rep in range(args.repeat):
        for v in args.variants:
            env = dict(os.environ)
            for kv in v.split():
                k, val = kv.split("=", 1)
                env[k] = val
            r = subprocess.run([sys.executable, os.path.abspath(__file__), "--child",
                                "--scale", str(args.scale), "--edgefactor", str(args.edgefactor),
                                "--mh", str(args.mh), "--steps", str(args.steps),
                                "--parts", str(args.parts)],
                               env=env, capture_output=True, text=True)
            line = [x for x in r.stdout.splitlines() if x.startswith("{")]
            print(f"[{rep}] {v:40s} {line[0] if line else r.stderr[-500:]}", flush=True)


if __name__ == "__main__":
    main()
