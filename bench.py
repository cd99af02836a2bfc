"""ET-BFS benchmark on B200 — prints ONE JSON line (the driver's contract).

Metric (BASELINE.json): harmonic-mean GTEPS over 64 roots, plus the fraction of
the HBM TEPS roofline. Workload: Kronecker R-MAT scale 22 / edgefactor 16
(BASELINE configs[1], the largest config quoted on one GPU that the same run can
also time the reference on), generator seed 1, 64 roots from select_roots(seed
1), ET mode mh=-1 with TEET (the reference's BenchConfig defaults,
proj/include/etbfs/bench.hpp:30-45). Synthetic inputs produced by the
reference's own generator algorithm stand in for the paper's Graph500 inputs.

A "step" is one pass of the hot path over the 64 roots: per root, the
start-side walk + one persistent kernel that runs the whole core DO-BFS and the
edge-tree replay, results left in HBM. Per-root times come from CUDA events on
the launching stream; L2 is flushed (a 2x-L2 memset) between roots outside the
timed events.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--scale S] [--edgefactor E]
                  [--mh M] [--impl ours|reference] [--no-cpu-baseline]
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "harmonic-mean GTEPS over 64 roots at 1/2/4/8 B200; % of HBM TEPS roofline"
NROOTS = 64


def env_rank():
    return (int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)),
            int(os.environ.get("LOCAL_RANK", 0)))


def harmonic_gteps(te, seconds):
    te = np.asarray(te, np.float64)
    s = np.asarray(seconds, np.float64)
    g = te / s / 1e9
    return float(len(g) / np.sum(1.0 / g)), g


def measured_peak_hbm():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as f:
            return float(json.load(f)["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled every 200 ms during timing."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device):
        self.device = device
        self.proc = None
        self.path = None

    def __enter__(self):
        fd, self.path = tempfile.mkstemp(suffix=".csv")
        os.close(fd)
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None
        time.sleep(0.3)
        return self

    def __exit__(self, *a):
        if self.proc:
            time.sleep(0.25)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        rows = []
        try:
            for line in open(self.path):
                f = [x.strip() for x in line.split(",")]
                if len(f) >= 9:
                    rows.append(f)
        except Exception:
            pass
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        sm = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in rows if r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[5 + i] == "Active"})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(rows)}


def captured_traffic(workload):
    """DRAM bytes per launch of the BFS kernel from the committed ncu --set full
    capture (profiles/traffic.json), or None when this workload was not captured."""
    try:
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as f:
            return json.load(f)[workload]["mean"]
    except Exception:
        return None


def dram_block(workload, kernel_s, peak):
    """Measured DRAM efficiency beside the B_alg normalisation (SURVEY.md §8(d):
    B_alg counts every core edge once, a direction-optimizing BFS reads ~2% of
    them, so the B_alg fraction may exceed 1 and is not a DRAM figure)."""
    t = captured_traffic(workload)
    if not t:
        return None
    gbs = t / kernel_s / 1e9
    return {"bytes_per_launch": int(t), "achieved_gbs": round(gbs, 1), "frac": round(gbs / peak, 4),
            "source": "profiles/traffic.json (ncu dram__bytes_read+write per launch, caches "
                      "flushed per replay) / the mean CUDA-event kernel time of this run"}


def b_alg(nc, ecore, ntree):
    """algorithmic bytes per BFS (relaid space, u32 core ids)."""
    return 4 * ecore + 8 * (nc + 1) + 8 * nc + 16 * ntree


# --------------------------------------------------------------------- ours --
def run_ours(args):
    import paper_2009_07463_b200 as eb
    from paper_2009_07463_b200 import etbfs as E

    rank, world, local = env_rank()
    dist = None
    if world > 1:
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(local)
        dist.init_process_group("nccl")
    E.lib().etb_set_device(local)

    t0 = time.perf_counter()
    g = eb.generate_graph(scale=args.scale, edgefactor=args.edgefactor, seed=1)
    t_csr = time.perf_counter() - t0
    t1 = time.perf_counter()
    cg = eb.relayout_csr(g, mh=args.mh)
    t_layout = time.perf_counter() - t1
    preprocessing_s = time.perf_counter() - t0

    # Roots: select_roots(original, 64, seed 1) (bench.cpp:217-242) in original ids.
    roots = select_roots_from_degrees(g.degrees(), NROOTS, 1)
    starts = cg.old2new[roots.astype(np.int64)]
    if world > 1:
        # 1D core partition, one GPU per rank, exchange over NVLink peer memory
        # (bfs_part.cu). Every rank runs every root; the kernels synchronise.
        from paper_2009_07463_b200 import multi
        multi.connect(cg, rank, world)
        dist.barrier()

    te = np.empty(len(starts), np.uint64)
    valid = []
    for i, s in enumerate(starts):
        E.bfs_device(cg, int(s))
        te[i] = E.result_traversed_edges(cg)  # this rank's owned part when world > 1
        if world == 1:  # validate_bfs_tree rules 1-5 on the device, every root (untimed)
            valid.append(E.result_validate(cg, int(s))["passed"])
    if world > 1:
        t = torch.tensor(te.astype(np.int64), device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.SUM)
        te = t.cpu().numpy().astype(np.uint64)

    pol = eb.HybridPolicy()
    reps = np.tile(starts, args.steps)
    if world > 1:
        dist.barrier()
    with ClockSampler(local) as clk:
        ms, _ = E.time_roots(cg, reps, warmup=args.warmup * len(starts), flush_l2=True,
                             policy=pol, kernel_times=False)
    if world > 1:
        dist.barrier()
    clocks = clk.summary()
    # kernel-only times (roofline, diagnostics): one more pass with the pre-launch
    # event, outside the timed value
    _, kms = E.time_roots(cg, starts, warmup=len(starts), flush_l2=True, policy=pol)
    if world > 1:  # per-root device time = max over ranks
        for arr in (ms, kms):
            t = torch.tensor(arr, dtype=torch.float64, device="cuda")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            arr[:] = t.cpu().numpy()
    sec = ms / 1e3
    te_rep = np.tile(te, args.steps).astype(np.float64)
    hm, per = harmonic_gteps(te_rep, sec)
    giant = te_rep == te_rep.max()
    hm_giant, _ = harmonic_gteps(te_rep[giant], sec[giant])
    step_ms = float(ms.sum() / args.steps)
    value = hm

    # Roofline of the dominant (only) kernel: algorithmic bytes / kernel time.
    peak, peak_src = measured_peak_hbm()
    peak *= world
    balg = b_alg(cg.core_vertex_count, cg.restricted_edge_count, cg.tree_vertex_count)
    kern_s = float(np.mean(kms)) / 1e3
    achieved = balg / kern_s / 1e9
    roof_gteps = peak * 1e9 / (balg / float(te.max())) / 1e9

    # e2e: the C-ABI call with a HOST output buffer — the BfsTree content (parent of
    # every vertex, relaid ids, u32) copied device->host inside the wall-clock timing.
    n = cg.vertex_count
    parent_h = np.empty(n, np.uint32)
    eb.etbfs._check(E.lib().etb_host_register(parent_h.ctypes.data, parent_h.nbytes))
    e2e_t = []
    for s in np.concatenate([starts[:3], starts]):
        c0 = time.perf_counter()
        eb.etbfs._check(E.lib().etb_bfs_compact(cg.handle, int(s), None, None,
                                                parent_h.ctypes.data))
        e2e_t.append(time.perf_counter() - c0)
    e2e_t = np.array(e2e_t[3:])
    eb.etbfs._check(E.lib().etb_host_unregister(parent_h.ctypes.data))
    if world > 1:
        t = torch.tensor(e2e_t, dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_t = t.cpu().numpy()
    e2e_hm, _ = harmonic_gteps(te.astype(np.float64), e2e_t)

    # Per-level device timeline of the first root (stats run, untimed).
    r0 = eb.et_bfs(cg, int(starts[0]), stats=True, want_parent=False, want_depth=False)
    timeline = {"trace": r0.stats.direction_trace, "claims": r0.stats.level_claims,
                "level_end_us": [round(x / 1e3, 2) for x in r0.stats.level_ns],
                "total_us": round(r0.stats.total_ns / 1e3, 2)}

    out = {
        "metric": METRIC, "value": round(value, 3), "unit": "GTEPS", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(step_ms, 4),
        "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "u32", "data": "synthetic",
        "config": {"workload": f"kronecker-s{args.scale}-ef{args.edgefactor}-seed1",
                   "scale": args.scale, "edgefactor": args.edgefactor, "roots": NROOTS,
                   "root_seed": 1, "mh": args.mh, "replay": "teet", "alpha": 14.0, "beta": 24.0,
                   "parallelism": f"1d-core-partition-{world}gpu" if world > 1 else "1gpu",
                   "l2": "flushed between roots (2x L2 memset outside the timed events)"},
        "roofline": {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak,
                     "unit": "GB/s", "frac": round(achieved / peak, 4),
                     "traffic": captured_traffic(f"kronecker-s{args.scale}-ef{args.edgefactor}-seed1"),
                     "peak_source": peak_src, "algorithmic_bytes_per_bfs": int(balg),
                     "bytes_per_te": round(balg / float(te.max()), 3),
                     "roofline_gteps": round(roof_gteps, 1),
                     "frac_of_roofline_gteps": round(hm_giant / roof_gteps, 4),
                     "dram": dram_block(f"kronecker-s{args.scale}-ef{args.edgefactor}-seed1",
                                        kern_s, peak)},
        "e2e": {"value": round(e2e_hm, 3), "unit": "GTEPS",
                "h2d_bytes_per_step": 8 * len(starts),
                "d2h_bytes_per_step": 4 * n * len(starts),
                "api": "etb_bfs_compact (C-ABI, host parent u32[n] output, pinned, wall clock)"},
        "gpu_launches": int(len(reps)),
        "clocks": clocks,
        "detail": {"mean_gteps": round(float(per.mean()), 3), "min_gteps": round(float(per.min()), 3),
                   "max_gteps": round(float(per.max()), 3),
                   "hm_gteps_giant_component": round(hm_giant, 3),
                   "validated_roots": len(valid), "all_valid": all(valid) if valid else None,
                   "kernel_ms_mean": round(float(np.mean(kms)), 4),
                   "call_ms_mean": round(float(np.mean(ms)), 4),
                   "traversed_edges": int(te.max()),
                   "core_vertices": int(cg.core_vertex_count),
                   "tree_vertices": int(cg.tree_vertex_count),
                   "core_directed_edges": int(cg.restricted_edge_count),
                   "preprocessing_s": round(preprocessing_s, 3),
                   "generate_build_csr_s": round(t_csr, 3), "classify_relayout_s": round(t_layout, 3),
                   "timeline_root0": timeline},
    }
    if rank == 0 and args.report_json:
        write_report_v1(args, roots, te, sec[: len(starts)], valid, preprocessing_s,
                        g.vertex_count, g.undirected_edge_count())
    if rank == 0 and world == 1 and args.tree_out:
        # BenchConfig::tree_out (bench.hpp:45): the first root's tree, original ids, ETT1
        r0t = eb.et_bfs(cg, int(starts[0]), want_depth=False)
        new2old = np.asarray(cg.new2old, np.uint64)
        par = np.full(cg.vertex_count, np.uint64(0xFFFFFFFFFFFFFFFF), np.uint64)
        ok = r0t.parent != np.uint64(0xFFFFFFFFFFFFFFFF)
        par[new2old[ok]] = new2old[r0t.parent[ok].astype(np.int64)]
        eb.write_tree(args.tree_out, int(roots[0]), par)
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        out["cpu_baseline"] = cpu_baseline(args, roots[: args.cpu_roots])
    if rank == 0 and world == 1 and args.mh == -1 and not args.no_paper_mode:
        out["paper_mode"] = measure_paper_mode(g, roots, args.steps, args.warmup)
    scales = [int(x) for x in str(args.secondary_scale).split(",") if x.strip() and int(x)]
    scales = [x for x in scales if x != args.scale]
    if world == 1 and scales:
        del cg, g
        out["secondary"] = [measure_secondary(sc, args.edgefactor, args.mh, args.steps,
                                              args.warmup) for sc in scales]
    if world > 1:
        dist.destroy_process_group()
    if rank == 0:
        print(json.dumps(out), flush=True)


def write_report_v1(args, roots, te, seconds, valid, prep_s, n, m):
    """The reference's JSON report, schema v1 (report_to_json, bench.cpp:301-343),
    for the first timed pass over the roots, so GPU runs drop into the same
    tooling as `etbfs_bench --json` output."""
    gteps = [float(t) / s / 1e9 for t, s in zip(te, seconds)]
    rep = {
        "schema_version": 1,
        "config": {"kernel": "et-bfs", "mh": args.mh, "roots": len(roots), "seed": 1,
                   "threads": 0, "alpha": 14.0, "beta": 24.0, "replay": "teet",
                   "rm_zero": False, "round_robin": False, "degree_aware": False,
                   "block_search": False, "et": True, "segments": 0},
        "graph": {"vertex_count": int(n), "undirected_edge_count": int(m)},
        "aggregate": {"mean_gteps": float(np.mean(gteps)), "min_gteps": float(np.min(gteps)),
                      "max_gteps": float(np.max(gteps)),
                      "harmonic_mean_seconds": float(len(seconds) / np.sum(1.0 / seconds)),
                      "preprocessing_seconds": float(prep_s),
                      "all_valid": bool(all(valid)) if valid else False},
        "per_root": [{"root": int(r), "seconds": float(s), "traversed_edges": int(t),
                      "gteps": g, "valid": bool(valid[i]) if valid else False}
                     for i, (r, s, t, g) in enumerate(zip(roots, seconds, te, gteps))],
    }
    with open(args.report_json, "w") as f:
        json.dump(rep, f, indent=2)


def measure_paper_mode(g, roots, steps, warmup):
    """The paper's own configuration at the primary scale (mh=0 with TEOLV,
    PAPER.md:623): same protocol (L2 flushed between roots, events around the
    launch), every root validated on the device."""
    import paper_2009_07463_b200 as eb
    from paper_2009_07463_b200 import etbfs as E
    cg = eb.relayout_csr(g, mh=0)
    starts = cg.old2new[roots.astype(np.int64)]
    reps = np.tile(starts, steps)
    ms, _ = E.time_roots(cg, reps, warmup=warmup * len(starts), flush_l2=True,
                         replay=E.TreeReplay.TEOLV, kernel_times=False)
    sec = np.asarray(ms, np.float64).reshape(steps, len(starts)).mean(axis=0) / 1e3
    te = np.empty(len(starts), np.float64)
    ok = 0
    for i, s in enumerate(starts):
        E.bfs_device(cg, int(s), replay=E.TreeReplay.TEOLV)
        ok += E.result_validate(cg, int(s))["passed"]
        te[i] = E.result_traversed_edges(cg)
    hm, _ = harmonic_gteps(te, sec)
    return {"mh": 0, "replay": "teolv", "value": round(hm, 3), "unit": "GTEPS",
            "ms_per_bfs_mean": round(float(sec.mean()) * 1e3, 4),
            "validated_roots": int(ok), "all_valid": ok == len(starts),
            "core_vertices": int(cg.core_vertex_count)}


def measure_secondary(scale, ef, mh, steps, warmup):
    """The same timed protocol at BASELINE configs[3]'s scale (s26): HM GTEPS and
    the HBM-roofline fraction the north_star target is quoted on."""
    import paper_2009_07463_b200 as eb
    from paper_2009_07463_b200 import etbfs as E
    t0 = time.perf_counter()
    g = eb.generate_graph(scale=scale, edgefactor=ef, seed=1)
    cg = eb.relayout_csr(g, mh=mh)
    prep = time.perf_counter() - t0
    roots = select_roots_from_degrees(g.degrees(), NROOTS, 1)
    starts = cg.old2new[roots.astype(np.int64)]
    te = np.empty(len(starts), np.uint64)
    valid = []
    for i, s in enumerate(starts):
        E.bfs_device(cg, int(s))
        te[i] = E.result_traversed_edges(cg)
        valid.append(E.result_validate(cg, int(s))["passed"])
    ms, _ = E.time_roots(cg, np.tile(starts, steps), warmup=warmup * len(starts), flush_l2=True,
                         kernel_times=False)
    _, kms = E.time_roots(cg, starts, warmup=len(starts), flush_l2=True)
    te_rep = np.tile(te, steps).astype(np.float64)
    hm, per = harmonic_gteps(te_rep, ms / 1e3)
    peak, _ = measured_peak_hbm()
    balg = b_alg(cg.core_vertex_count, cg.restricted_edge_count, cg.tree_vertex_count)
    achieved = balg / (float(np.mean(kms)) / 1e3) / 1e9
    roof = peak / (balg / float(te.max()))
    return {"workload": f"kronecker-s{scale}-ef{ef}-seed1", "value": round(hm, 3), "unit": "GTEPS",
            "ms_per_bfs_mean": round(float(np.mean(ms)), 4),
            "min_gteps": round(float(per.min()), 3), "max_gteps": round(float(per.max()), 3),
            "traversed_edges": int(te.max()), "core_vertices": int(cg.core_vertex_count),
            "core_directed_edges": int(cg.restricted_edge_count),
            "tree_vertices": int(cg.tree_vertex_count),
            "roofline": {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak,
                         "unit": "GB/s", "frac": round(achieved / peak, 4),
                         "algorithmic_bytes_per_bfs": int(balg),
                         "bytes_per_te": round(balg / float(te.max()), 3),
                         "roofline_gteps": round(roof, 1),
                         "frac_of_roofline_gteps": round(hm / roof, 4),
                         "traffic": captured_traffic(f"kronecker-s{scale}-ef{ef}-seed1"),
                         "dram": dram_block(f"kronecker-s{scale}-ef{ef}-seed1",
                                            float(np.mean(kms)) / 1e3, peak)},
            "preprocessing_s": round(prep, 3), "gpu_launches": int(len(ms)),
            "validated_roots": len(valid), "all_valid": all(valid)}


def select_roots_from_degrees(deg, count, seed):
    """select_roots (bench.cpp:217-242) from a degree array (original ids)."""
    n = len(deg)
    eligible = int(np.count_nonzero(deg))
    taken = np.zeros(n, bool)
    out, distinct = [], 0
    state = seed
    M = 0xFFFFFFFFFFFFFFFF
    while len(out) < count:
        state = (state + 0x9E3779B97F4A7C15) & M
        z = state
        z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & M
        z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & M
        z ^= z >> 31
        v = z % n
        if deg[v] == 0:
            continue
        if taken[v] and distinct < eligible:
            continue
        if not taken[v]:
            taken[v] = True
            distinct += 1
        out.append(v)
    return np.array(out, np.uint64)


# ---------------------------------------------------------------- reference --
def ref_pipeline(scale, ef, mh, threads):
    """The reference's own untimed preprocessing (bench.cpp:253-256) via oracle/_ref."""
    import oracle as O
    O.ref().ref_set_threads(threads)
    t0 = time.perf_counter()
    pairs = O.ref_generate(scale, ef, 1)
    csr = O.RefCsr(1 << scale, pairs)
    del pairs
    prep = O.RefPrepared(csr, mh)
    a = prep.arrays()
    deg = np.diff(a["row"]).astype(np.int64)
    old2new = np.empty(1 << scale, np.int64)
    old2new[a["new2old"].astype(np.int64)] = np.arange(1 << scale)
    return csr, prep, deg, old2new, time.perf_counter() - t0


def ref_time_roots(prep, deg, starts):
    """Time the reference's et_bfs (the timed `traverse`, bench.cpp:269-271) per root."""
    secs, tes = [], []
    for s in starts:
        par, _, sec = prep.et_bfs(int(s), kernel=1, replay=0)
        tes.append(int(deg[par != 0xFFFFFFFFFFFFFFFF].sum() // 2))
        secs.append(sec)
    return np.array(secs), np.array(tes, np.float64)


def cpu_baseline(args, roots_orig):
    import oracle as O
    if not O.ref_available():
        return {"value": None, "unit": "GTEPS", "cores": 0, "kind": "reference",
                "sample": "oracle/_ref not built"}
    threads = os.cpu_count() or 1
    csr, prep, deg, old2new, prep_s = ref_pipeline(args.scale, args.edgefactor, args.mh, threads)
    starts = old2new[roots_orig.astype(np.int64)]
    secs, tes = ref_time_roots(prep, deg, starts)
    hm, _ = harmonic_gteps(tes, secs)
    return {"value": round(hm, 4), "unit": "GTEPS", "cores": threads, "kind": "reference",
            "sample": f"reference et_bfs (kHybrid, TEET, mh={args.mh}) on the first "
                      f"{len(starts)} of the 64 seed-1 roots, s{args.scale}/ef{args.edgefactor}, "
                      f"{threads} OpenMP threads; reference preprocessing {prep_s:.1f}s untimed",
            "cpu_model": cpu_model()}


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return None


def run_reference(args):
    rank, world, _ = env_rank()
    if rank != 0:
        return
    import oracle as O
    if not O.ref_available():
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref not built"}))
        return
    threads = os.cpu_count() or 1
    csr, prep, deg, old2new, prep_s = ref_pipeline(args.scale, args.edgefactor, args.mh, threads)
    roots = csr.select_roots(NROOTS, 1)
    starts = old2new[roots.astype(np.int64)]
    per_step = args.ref_roots_per_step
    for w in range(args.warmup):
        ref_time_roots(prep, deg, starts[(w * per_step) % NROOTS:][:per_step])
    secs, tes = [], []
    for k in range(args.steps):
        sl = [(k * per_step + j) % NROOTS for j in range(per_step)]
        s, t = ref_time_roots(prep, deg, starts[sl])
        secs.append(s)
        tes.append(t)
    secs = np.concatenate(secs)
    tes = np.concatenate(tes)
    hm, per = harmonic_gteps(tes, secs)
    out = {
        "impl": "reference", "metric": METRIC, "value": round(hm, 4), "unit": "GTEPS",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(float(secs.sum() / args.steps * 1e3), 3), "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "u64", "data": "synthetic",
        "config": {"workload": f"kronecker-s{args.scale}-ef{args.edgefactor}-seed1",
                   "scale": args.scale, "edgefactor": args.edgefactor, "roots": NROOTS,
                   "root_seed": 1, "mh": args.mh, "replay": "teet", "alpha": 14.0, "beta": 24.0,
                   "parallelism": f"openmp{threads}"},
        "cpu_baseline": {"value": round(hm, 4), "unit": "GTEPS", "cores": threads,
                         "kind": "reference",
                         "sample": f"{per_step} roots per step (round robin over the 64 seed-1 "
                                   f"roots), unmodified reference et_bfs via oracle/_ref",
                         "cpu_model": cpu_model()},
        "e2e": {"value": round(hm, 4), "unit": "GTEPS", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
        "detail": {"mean_gteps": round(float(per.mean()), 4), "preprocessing_s": round(prep_s, 2)},
    }
    print(json.dumps(out), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--scale", type=int, default=22)
    ap.add_argument("--edgefactor", type=int, default=16)
    ap.add_argument("--mh", type=int, default=-1)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-roots", type=int, default=16)
    ap.add_argument("--ref-roots-per-step", type=int, default=4)
    ap.add_argument("--report-json", default=None,
                    help="also write the reference's JSON report (schema v1, bench.cpp:301-343)")
    ap.add_argument("--tree-out", default=None,
                    help="write the first root's BFS tree (original ids) as an ETT1 file")
    ap.add_argument("--no-paper-mode", action="store_true",
                    help="skip the mh=0/TEOLV line at the primary scale")
    ap.add_argument("--secondary-scale", default="26,28",
                    help="comma list of further scales to time (0 = none); under 'secondary'")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
