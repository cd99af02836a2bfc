"""Per-root device timeline of the persistent ET-BFS kernel (diagnostics only).

For each of the 64 seed-1 roots: direction trace, claims per level and the
per-level device durations (block 0's globaltimer stamps), plus the CUDA-event
kernel time. Usage: python tools/root_profile.py [--scale S] [--edgefactor E] [--mh M]
"""
import argparse
import json
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
    ap.add_argument("--mh", type=int, default=-1)
    ap.add_argument("--roots", type=int, default=64)
    ap.add_argument("--parts", type=int, default=1, help="1D core partitions on this device")
    ap.add_argument("--cold", action="store_true", help="per-level stats on a flushed L2")
    ap.add_argument("--diag", action="store_true",
                    help="-DETB_MISS_CYCLES build: bottom-up step / miss-resolution warp time per level")
    ap.add_argument("--clock-ghz", type=float, default=1.965)
    args = ap.parse_args()
    g = eb.generate_graph(scale=args.scale, edgefactor=args.edgefactor, seed=1)
    cg = eb.relayout_csr(g, mh=args.mh)
    if args.parts > 1:
        E.partition(cg, args.parts)
    roots = select_roots_from_degrees(g.degrees(), 64, 1)[: args.roots]
    starts = cg.old2new[roots.astype(np.int64)]
    ms, kms = E.time_roots(cg, starts, warmup=8, flush_l2=True)
    out = []
    import torch
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    for i, s in enumerate(starts):
        if args.cold:  # the stats run on a flushed L2, like the timed runs
            flush.zero_()
            torch.cuda.synchronize()
        else:
            E.time_roots(cg, starts[i:i + 1], warmup=0, flush_l2=True)  # warms this root
        diag = np.zeros(320, np.uint64)
        if args.diag:
            E._check(E.lib().etb_debug_diag(cg.handle, diag.ctypes.data, 1))
        r = eb.et_bfs(cg, int(s), stats=True, want_parent=False, want_depth=False)
        ns = r.stats.level_ns
        if args.diag:
            E._check(E.lib().etb_debug_diag(cg.handle, diag.ctypes.data, 1))
        import ctypes as C
        ph = np.zeros(256, np.uint64)
        E._check(E.lib().etb_debug_phase_stamps(cg.handle, ph.ctypes.data))
        td_edges = [int(ph[192 + L]) if r.stats.direction_trace[L:L + 1] == "t" else None
                    for L in range(len(r.stats.direction_trace))]
        dur = [round((ns[j + 1] - ns[j]) / 1e3, 1) for j in range(len(ns) - 1)]
        # split levels: time of the bottom-up half (stamp 320 + L) since the level's start
        split_bu = {L: round((int(ph[64 + L]) - int(ph[0]) - ns[L]) / 1e3, 1)
                    for L in range(min(len(ns) - 1, 60))
                    if ph[64 + L] and ns[L] < int(ph[64 + L]) - int(ph[0]) <= ns[L + 1]}  # (not a stale stamp)
        rec = {"root": int(roots[i]), "start": int(s), "type": int(cg.vertex_type[int(s)]),
               "kernel_us": round(float(kms[i]) * 1e3, 1), "call_us": round(float(ms[i]) * 1e3, 1), "device_us": round(r.stats.total_ns / 1e3, 1),
               "init_us": round(ns[0] / 1e3, 1) if ns else None, "trace": r.stats.direction_trace,
               "claims": r.stats.level_claims, "level_us": dur, "td_edges": td_edges,
               "split_bu_us": split_bu}
        if args.diag:  # mean per warp, us at the SM clock (--clock-ghz)
            nw = 148 * (1024 if cg.core_vertex_count >= (1 << 23) else 640) // 32
            cyc = lambda c: round(float(c) / nw / (args.clock_ghz * 1e3), 1)
            rec["bu_step_us"] = [cyc(diag[(L + 1) & 63]) for L in range(len(dur))]
            rec["bu_miss_us"] = [cyc(diag[64 + ((L + 1) & 63)]) for L in range(len(dur))]
            rec["bu_miss_max_us"] = [round(float(diag[256 + ((L + 1) & 63)]) / (args.clock_ghz * 1e3), 1)
                                     for L in range(len(dur))]
            d1 = lambda b: [int(diag[b + ((L + 1) & 31)]) for L in range(len(dur))]
            rec["deferred"], rec["past_second"] = d1(128), d1(160)
            rec["warp_rows"], rec["warp_rounds"] = d1(192), d1(224)
        out.append(rec)
        print(json.dumps(rec), flush=True)
    # Fixed cost: a start on an isolated vertex runs init + tree replay only.
    vz = np.nonzero(np.asarray(cg.vertex_type) == 4)[0]
    if vz.size:
        s = int(vz[0])
        _, fk = E.time_roots(cg, np.full(32, s, dtype=np.uint64), warmup=4, flush_l2=True)
        r = eb.et_bfs(cg, s, stats=True, want_parent=False, want_depth=False)
        print(json.dumps({"floor_kernel_us": round(float(np.median(fk)) * 1e3, 1),
                          "floor_device_us": round(r.stats.total_ns / 1e3, 1)}))
    import ctypes as C
    eu = C.c_double()
    E._check(E.lib().etb_debug_launch_floor(cg.handle, 32, C.byref(eu)))
    print(json.dumps({"empty_kernel_us": round(eu.value, 1)}))
    k = np.array([o["kernel_us"] for o in out])
    print(json.dumps({"kernel_us_mean": float(k.mean()), "kernel_us_max": float(k.max()),
                      "kernel_us_min": float(k.min())}))


if __name__ == "__main__":
    main()
