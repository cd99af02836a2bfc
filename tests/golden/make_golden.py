"""Generate the golden fixtures in tests/golden/ by RUNNING the compiled,
unmodified reference (oracle/_ref/libetbfs_ref.so, built by `make -C oracle ref`
from /root/reference/proj/src). Run here, in the container that has
/root/reference:  python tests/golden/make_golden.py [--big]

Outputs (committed):
  corpus.json   — the reference test corpus (proj/tests/helpers.hpp:141-155
                  small_corpus + the KAT graphs of test_classify.cpp /
                  test_relayout.cpp / test_et_bfs.cpp) with the reference's
                  CSR, classification (mh -1/0/1/3), peak height, relayout
                  (new2old, ETL) for mh -1/0/1, BFS levels and α/β traces.
  kronecker_s16.json — C1 anchors (scale 16, ef 16, seed 1): hashes of the
                  tuples / CSR / relayout / ETL, BuildStats, the 64 roots,
                  per-root levels hashes, TE, direction traces.
  kronecker_big.json (--big) — C2 (s22/ef16) and C3 (s24/ef4) counts + hashes,
                  reference α/β traces for both ET modes and oracle_bfs level hashes
                  for all 64 roots.
  kronecker_huge.json (--huge) — the same record for C4 (s26/ef16), built by the
                  lean path (generate_kronecker -> build_csr with the tuples freed,
                  hashes computed inside the reference library): ~52 GB host RAM,
                  ~35 min on 8 cores.
"""
from __future__ import annotations

import argparse
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import oracle as O  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))


# std::mt19937_64 (Matsumoto & Nishimura 2004 parameters, as std::mt19937_64
# specifies them) — restated so the random corpus of helpers.hpp:73-80 can be
# reproduced; only used here, the fixture stores the resulting tuples.
class MT19937_64:
    def __init__(self, seed):
        self.mt = [0] * 312
        self.mt[0] = seed & 0xFFFFFFFFFFFFFFFF
        for i in range(1, 312):
            self.mt[i] = (6364136223846793005 * (self.mt[i - 1] ^ (self.mt[i - 1] >> 62)) + i) \
                & 0xFFFFFFFFFFFFFFFF
        self.i = 312

    def __call__(self):
        M = 0xFFFFFFFFFFFFFFFF
        if self.i >= 312:
            for k in range(312):
                y = (self.mt[k] & 0xFFFFFFFF80000000) | (self.mt[(k + 1) % 312] & 0x7FFFFFFF)
                v = self.mt[(k + 156) % 312] ^ (y >> 1)
                if y & 1:
                    v ^= 0xB5026F5AA96619E9
                self.mt[k] = v
            self.i = 0
        y = self.mt[self.i]
        self.i += 1
        y ^= (y >> 29) & 0x5555555555555555
        y ^= (y << 17) & 0x71D67FFFEDA60000
        y ^= (y << 37) & 0xFFF7EEE000000000
        y ^= y >> 43
        return y & M


def path(n):
    return n, [(v, v + 1) for v in range(n - 1)]


def cycle(n):
    _, e = path(n)
    if n >= 3:
        e.append((n - 1, 0))
    return n, e


def star(n):
    return n, [(0, v) for v in range(1, n)]


def complete(n):
    return n, [(u, v) for u in range(n) for v in range(u + 1, n)]


def binary_tree(n):
    return n, [((v - 1) // 2, v) for v in range(1, n)]


def random_list(n, tuples, seed):
    r = MT19937_64(seed)
    out = []
    for _ in range(tuples):
        a = r() % n
        b = r() % n
        out.append((a, b))
    return n, out


def small_corpus():
    """helpers.hpp:141-155"""
    c = [("path1", path(1)), ("path2", path(2)), ("path9", path(9)), ("cycle8", cycle(8)),
         ("star17", star(17)), ("complete6", complete(6)), ("binary31", binary_tree(31)),
         ("isolated6", (6, [])), ("disconnected7", (7, [(0, 1), (2, 3), (3, 4)]))]
    for seed in range(1, 11):
        c.append((f"random{seed}", random_list(20 + seed * 13, 30 + seed * 40, seed)))
    return c


def kat_graphs():
    """Graphs the reference's unit KATs pin (test_classify.cpp:80-138,
    test_relayout.cpp:110-158, test_et_bfs.cpp:54-179, test_bfs_kernels.cpp:185-256)."""
    return [("path3", path(3)), ("path4", path(4)), ("path5", path(5)), ("path6", path(6)),
            ("path7", path(7)), ("path8", path(8)), ("star5", star(5)), ("star300", star(300)),
            ("tri_subtree", (6, [(0, 1), (1, 2), (0, 2), (2, 3), (3, 4), (3, 5)])),
            ("cycle6", cycle(6)), ("clique5", complete(5)), ("pair4", (4, [(0, 1)])),
            ("pair2", (2, [(0, 1)])), ("chain5", (5, [(0, 1), (1, 2)])),
            ("restricted5", (5, [(0, 1), (0, 2), (1, 2), (2, 3), (3, 4), (0, 4)])),
            ("random400", random_list(400, 1500, 13)), ("random300", random_list(300, 1200, 77))]


def pick_roots(n, k):
    """helpers.hpp:133-138"""
    s = set()
    for i in range(k):
        if n > 0:
            s.add(i * (n - 1) // (k - 1 if k > 1 else 1))
    return sorted(s)


def lv_list(levels):
    return [-1 if x == O.NO_VERTEX else int(x) for x in levels]


def describe(name, n, edges):
    pairs = np.array(edges, dtype=np.uint64).reshape(-1, 2)
    g = O.RefCsr(n, pairs)
    row, col = g.arrays()
    rec = dict(name=name, n=n, edges=[list(map(int, e)) for e in edges],
               row=row.tolist(), col=col.tolist(), self_loops=g.self_loops,
               duplicates=g.duplicates, peak_height=int(g.peak_height()), classify={},
               layout={})
    for mh in (-1, 0, 1, 3):
        rec["classify"][str(mh)] = g.classify(mh).tolist()
    for mh in (-1, 0, 1):
        p = O.RefPrepared(g, mh)
        a = p.arrays()
        lay = dict(core=int(p.core), new2old=a["new2old"].tolist(),
                   etl=[[int(s) if s != O.NO_VERTEX else -1 for s in (x, y, z)]
                        for x, y, z in zip(a["etl_src"], a["etl_dst"], a["etl_ce"])],
                   restricted_edges=int(p.restricted_edges), roots={})
        # Relaid-space BFS levels + the reference's α/β trace per picked start.
        rg = O.RefCsr(n, np.stack([np.repeat(np.arange(n, dtype=np.uint64), np.diff(a["row"]).astype(np.int64)),
                                   a["col"]], 1) if a["col"].size else np.zeros((0, 2), np.uint64))
        for st in pick_roots(n, 5):
            par, trace, _ = p.et_bfs(st)
            lay["roots"][str(st)] = dict(levels=lv_list(rg.levels(st)), trace=trace)
        rec["layout"][str(mh)] = lay
    return rec


def corpus():
    recs = [describe(nm, n, e) for nm, (n, e) in small_corpus() + kat_graphs()]
    with open(os.path.join(OUT, "corpus.json"), "w") as f:
        json.dump(dict(generator="tests/golden/make_golden.py (compiled reference)",
                       graphs=recs), f, separators=(",", ":"))
    print("corpus.json:", len(recs), "graphs")


def kron_record(scale, ef, seed=1, nroots=64, level_roots=None, traces=True):
    n = 1 << scale
    pairs = O.ref_generate(scale, ef, seed)
    rec = dict(scale=scale, edgefactor=ef, seed=seed, tuples_fnv=O.fnv1a64(pairs))
    g = O.RefCsr(n, pairs)
    del pairs
    row, col = g.arrays()
    rec.update(self_loops=g.self_loops, duplicates=g.duplicates, nnz=int(g.nnz),
               row_fnv=O.fnv1a64(row), col_fnv=O.fnv1a64(col), max_degree=int(np.diff(row).max()))
    del col
    roots = g.select_roots(nroots, 1)
    rec["roots"] = roots.tolist()
    rec["peak_height"] = int(g.peak_height())
    rec["classes"] = {}
    rec["layout"] = {}
    for mh in (-1, 0, 1):
        t = g.classify(mh)
        rec["classes"][str(mh)] = np.bincount(t, minlength=5).tolist()
    for mh in (-1, 0):
        p = O.RefPrepared(g, mh)
        a = p.arrays()
        etl = np.stack([a["etl_src"], a["etl_dst"], a["etl_ce"]], 1)
        lay = dict(core=int(p.core), etl_size=int(p.etl_size),
                   restricted_edges=int(p.restricted_edges), new2old_fnv=O.fnv1a64(a["new2old"]),
                   relaid_row_fnv=O.fnv1a64(a["row"]), relaid_col_fnv=O.fnv1a64(a["col"]),
                   etl_fnv=O.fnv1a64(etl))
        if traces:
            old2new = np.empty(n, np.uint64)
            old2new[a["new2old"]] = np.arange(n, dtype=np.uint64)
            lay["traces"] = [p.et_bfs(int(old2new[r]), want_parent=False)[1] for r in roots]
        rec["layout"][str(mh)] = lay
        del a, p
    lr = roots if level_roots is None else roots[:level_roots]
    te, fnvs = [], []
    for r in lr:
        lv = g.levels(int(r))
        fnvs.append(O.fnv1a64(lv))
        reached = lv != O.NO_VERTEX
        te.append(int(np.diff(row)[reached].sum() // 2))
    rec["levels_fnv"] = fnvs
    rec["traversed_edges"] = te
    return rec


def kron_record_lean(scale, ef, seed=1, nroots=64, log=print):
    """One Kronecker config through the reference's lean path, every root's levels
    (oracle_bfs, validate.cpp:77-91) hashed, the α/β traces of et_bfs for mh=-1
    (TEET) and mh=0 (TEOLV) — the direction sequence a GPU run must reproduce."""
    import time
    t0 = time.time()
    n = 1 << scale
    g = O.RefCsr.kronecker(scale, ef, seed)
    row_fnv, col_fnv = g.fnv()
    deg = g.degrees().astype(np.int64)
    rec = dict(scale=scale, edgefactor=ef, seed=seed, tuples_fnv=g.tuples_fnv,
               self_loops=g.self_loops, duplicates=g.duplicates, nnz=int(g.nnz),
               row_fnv=row_fnv, col_fnv=col_fnv, max_degree=int(deg.max()))
    log(f"s{scale}: csr {time.time() - t0:.0f}s")
    roots = g.select_roots(nroots, 1)
    rec["roots"] = roots.tolist()
    rec["peak_height"] = int(g.peak_height())
    rec["classes"] = {str(mh): np.bincount(g.classify(mh), minlength=5).tolist()
                      for mh in (-1, 0, 1)}
    rec["layout"] = {}
    for mh in (-1, 0):
        p = O.RefPrepared(g, mh)
        n2o, row, col, etl = p.fnv()
        lay = dict(core=int(p.core), etl_size=int(p.etl_size),
                   restricted_edges=int(p.restricted_edges), new2old_fnv=n2o,
                   relaid_row_fnv=row, relaid_col_fnv=col, etl_fnv=etl)
        a_n2o = np.empty(n, np.uint64)
        O.ref().ref_prep_copy(p.h, O._ptr(a_n2o), None, None, None, None, None, None)
        old2new = np.empty(n, np.uint64)
        old2new[a_n2o] = np.arange(n, dtype=np.uint64)
        del a_n2o
        lay["traces"] = [p.et_bfs(int(old2new[r]), replay=0 if mh else 1,
                                  want_parent=False)[1] for r in roots]
        rec["layout"][str(mh)] = lay
        del p, old2new
        log(f"s{scale}: layout mh={mh} {time.time() - t0:.0f}s")
    te, fnvs, hist = [], [], []
    for r in roots:
        lv = g.levels(int(r))
        fnvs.append(format(int(O.ref().ref_fnv1a64(lv.ctypes.data, lv.nbytes)), "016x"))
        reached = lv != O.NO_VERTEX
        te.append(int(deg[reached].sum() // 2))
        hist.append(np.bincount(lv[reached].astype(np.int64)).tolist())
    rec["levels_fnv"] = fnvs
    rec["traversed_edges"] = te
    rec["level_histograms"] = hist
    log(f"s{scale}: levels {time.time() - t0:.0f}s")
    return rec


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--big", action="store_true")
    ap.add_argument("--huge", action="store_true")
    ap.add_argument("--only", action="store_true", help="skip corpus and s16")
    args = ap.parse_args()
    O.ref().ref_set_threads(os.cpu_count() or 1)
    if args.huge:
        rec = kron_record_lean(26, 16, log=lambda m: print(m, flush=True))
        with open(os.path.join(OUT, "kronecker_huge.json"), "w") as f:
            json.dump([rec], f, separators=(",", ":"))
        print("kronecker_huge.json")
        return
    if args.big and args.only:
        recs = [kron_record_lean(22, 16), kron_record_lean(24, 4)]
        with open(os.path.join(OUT, "kronecker_big.json"), "w") as f:
            json.dump(recs, f, separators=(",", ":"))
        print("kronecker_big.json")
        return
    corpus()
    with open(os.path.join(OUT, "kronecker_s16.json"), "w") as f:
        json.dump(kron_record(16, 16), f, indent=1)
    print("kronecker_s16.json")
    if args.big:
        recs = [kron_record_lean(22, 16), kron_record_lean(24, 4)]
        with open(os.path.join(OUT, "kronecker_big.json"), "w") as f:
            json.dump(recs, f, separators=(",", ":"))
        print("kronecker_big.json")


if __name__ == "__main__":
    main()
