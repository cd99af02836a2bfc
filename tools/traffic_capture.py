"""DRAM traffic per BFS launch (diagnostics feeding bench.py's roofline.traffic).

Runs the first --roots seed-1 roots of the bench workload once each (after the
graph is built and warmed). Meant to run under
  ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
      --clock-control none -k regex:et_bfs_kernel --csv --log-file gpurun_out/traffic_sXX.csv \
      python tools/traffic_capture.py --scale XX
then `python tools/traffic_capture.py --parse gpurun_out/traffic_sXX.csv --scale XX` folds the
per-launch bytes into profiles/traffic.json (ncu replays flush the caches, matching the
bench's L2 flush between roots).
"""
import argparse
import csv
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def run(args):
    import paper_2009_07463_b200 as eb
    from paper_2009_07463_b200 import etbfs as E
    from bench import select_roots_from_degrees
    g = eb.generate_graph(scale=args.scale, edgefactor=16, seed=1)
    cg = eb.relayout_csr(g, mh=-1)
    roots = select_roots_from_degrees(g.degrees(), 64, 1)[: args.roots]
    starts = cg.old2new[roots.astype(np.int64)]
    E.time_roots(cg, starts, warmup=0, flush_l2=True)
    print("ran", len(starts), "roots")


def parse(args):
    per = {}
    with open(args.parse) as f:
        rows = [r for r in csv.reader(l for l in f if l.startswith('"'))]
    hdr = rows[0]
    ki, mi, vi = hdr.index("ID"), hdr.index("Metric Name"), hdr.index("Metric Value")
    for r in rows[1:]:
        if len(r) <= vi:
            continue
        val = float(r[vi].replace(",", ""))
        unit = r[hdr.index("Metric Unit")] if "Metric Unit" in hdr else ""
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1, "us": 1e3,
                 "ms": 1e6, "usecond": 1e3, "nsecond": 1, "msecond": 1e6}.get(unit, 1)
        per.setdefault(r[ki], {})[r[mi]] = val * scale
    launches = [v for v in per.values() if "dram__bytes_read.sum" in v]
    byts = [v["dram__bytes_read.sum"] + v["dram__bytes_write.sum"] for v in launches]
    ns = [v.get("gpu__time_duration.sum", 0.0) for v in launches]
    wl = f"kronecker-s{args.scale}-ef16-seed1"
    path = os.path.join(ROOT, "profiles", "traffic.json")
    data = json.load(open(path)) if os.path.exists(path) else {}
    data[wl] = {"dram_bytes_per_launch": [int(b) for b in byts], "mean": int(np.mean(byts)),
                "ncu_ns_per_launch": [round(x) for x in ns],
                "source": f"{os.path.relpath(args.parse, ROOT)} (ncu --metrics dram__bytes_*, "
                          f"{len(byts)} launches, cache flushed per replay)"}
    json.dump(data, open(path, "w"), indent=1)
    print(wl, "launches", len(byts), "mean MB", np.mean(byts) / 1e6)


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--scale", type=int, default=22)
    ap.add_argument("--roots", type=int, default=16)
    ap.add_argument("--parse", default=None)
    a = ap.parse_args()
    parse(a) if a.parse else run(a)
