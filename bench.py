"""ET-BFS benchmark on B200 — prints ONE JSON line (the driver's contract).

Metric (BASELINE.json): harmonic-mean GTEPS over 64 roots, plus the fraction of
the HBM TEPS roofline. Headline workload: Kronecker R-MAT scale 26 /
edgefactor 16 (BASELINE configs[3], the config the north_star target and the
metric are quoted on; it fits one B200), generator seed 1, 64 roots from
select_roots(seed 1), ET mode mh=-1 with TEET (the reference's BenchConfig
defaults, proj/include/etbfs/bench.hpp:30-45). Synthetic inputs produced by the
reference's own generator algorithm stand in for the paper's Graph500 inputs.
Secondary lines: s22/ef16 (configs[1]), s24/ef4 (configs[2], literal and
giant-component harmonic means), s28/ef16 (configs[4]) and the paper's own
mode (mh=0 with TEOLV) at the headline scale.

A "step" is one pass of the hot path over the 64 roots: per root, the
start-side walk + one persistent kernel that runs the whole core DO-BFS and the
edge-tree replay, results left in HBM. Per-root times come from CUDA events on
the launching stream; L2 is flushed (a 2x-L2 memset) between roots outside the
timed events.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--scale S] [--edgefactor E]
                  [--mh M] [--impl ours|reference] [--no-cpu-baseline]

--gpus N > 1 without a torchrun environment re-launches itself under
torch.distributed.run with N ranks (one per GPU, 1D core partition).
"""
from __future__ import annotations

import argparse
import gc
import json
import os
import socket
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
L2_NOTE = "flushed between roots (2x L2 memset outside the timed events)"


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


def captured_traffic(workload, per_launch=False):
    """DRAM bytes per launch of the BFS kernel from the committed ncu capture
    (profiles/traffic.json: the first roots of the workload, in order), or None
    when this workload was not captured."""
    try:
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as f:
            d = json.load(f)[workload]
        return [int(x) for x in d["dram_bytes_per_launch"]] if per_launch else int(d["mean"])
    except Exception:
        return None


def b_alg(nc, ecore, ntree):
    """Graph500-style normalisation (every core edge read once)."""
    return 4 * ecore + 8 * (nc + 1) + 8 * nc + 16 * ntree


def workload_name(scale, ef):
    return f"kronecker-s{scale}-ef{ef}-seed1"


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


# --------------------------------------------------------------------- ours --
class Dist:
    """torch.distributed plumbing for N > 1 (one rank per GPU); no-ops at N = 1."""

    def __init__(self):
        self.rank, self.world, self.local = env_rank()
        self.d = None
        if self.world > 1:
            import torch
            import torch.distributed as dist
            torch.cuda.set_device(self.local)
            dist.init_process_group("nccl")
            self.d = dist

    def barrier(self):
        if self.d:
            self.d.barrier()

    def reduce(self, arr, op):
        """All-reduce a host array (SUM or MAX) over ranks."""
        if not self.d:
            return arr
        import torch
        t = torch.tensor(np.asarray(arr, np.float64), device="cuda")
        self.d.all_reduce(t, op=getattr(self.d.ReduceOp, op))
        return t.cpu().numpy()

    def close(self):
        if self.d:
            self.d.destroy_process_group()


def prepare(scale, ef, mh):
    import paper_2009_07463_b200 as eb
    t0 = time.perf_counter()
    g = eb.generate_graph(scale=scale, edgefactor=ef, seed=1)
    t_csr = time.perf_counter() - t0
    cg = eb.relayout_csr(g, mh=mh)
    prep = time.perf_counter() - t0
    roots = select_roots_from_degrees(g.degrees(), NROOTS, 1)
    starts = cg.old2new[roots.astype(np.int64)]
    return g, cg, roots, starts, {"preprocessing_s": round(prep, 3),
                                  "generate_build_csr_s": round(t_csr, 3)}


def validate_all(cg, starts, replay, D):
    """TE per root + validate_bfs_tree rules 1-5 on the device, every root."""
    from paper_2009_07463_b200 import etbfs as E
    te = np.empty(len(starts), np.float64)
    valid = []
    for i, s in enumerate(starts):
        E.bfs_device(cg, int(s), replay=replay)
        if D.world > 1:
            from paper_2009_07463_b200 import multi
            multi.assemble_result(cg, D)
        te[i] = E.result_traversed_edges(cg)
        if D.rank == 0 or D.world == 1:
            valid.append(E.result_validate(cg, int(s))["passed"])
    return te, valid


def work_roofline(cg, starts, kms, replay, peak, workload, te):
    """The roofline of the timed kernel: per root, the bytes a direction-optimizing
    BFS with this root's level sequence must move (etb_result_work, csrc/work.cu)
    over its event-timed kernel duration; beside it the DRAM bytes ncu measured
    per launch (profiles/traffic.json) and SURVEY §8(d)'s B_alg normalisation."""
    from paper_2009_07463_b200 import etbfs as E
    works = [E.result_work(cg, int(s), replay=replay) for s in starts]
    wb = np.array([w.total_bytes for w in works], np.float64)
    kern_s = float(np.mean(kms)) / 1e3
    achieved = float(wb.mean()) / kern_s / 1e9
    traffic = captured_traffic(workload)
    balg = b_alg(cg.core_vertex_count, cg.restricted_edge_count, cg.tree_vertex_count)
    out = {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
           "frac": round(achieved / peak, 4), "traffic": traffic,
           "algorithmic_bytes_per_launch": int(wb.mean()),
           "algorithmic_bytes_model": "etb_result_work (csrc/work.cu): frontier rows of top-down "
                                      "levels, first-neighbour entry + probes to the first "
                                      "frontier neighbour of every unvisited core vertex on "
                                      "bottom-up levels, one result write per claim, core-sized "
                                      "bitmaps once per level, tree replay, unreached fill, "
                                      "state reset; mean over the 64 roots",
           "kernel_ms_mean": round(kern_s * 1e3, 4),
           "bytes_per_te": round(float(wb.mean()) / float(np.max(te)), 3)}
    if traffic:
        gbs = traffic / kern_s / 1e9
        per = captured_traffic(workload, per_launch=True) or []
        k = min(len(per), len(wb))
        ratio = float(np.sum(per[:k])) / float(np.sum(wb[:k])) if k else traffic / float(wb.mean())
        out["dram"] = {"bytes_per_launch": traffic, "achieved_gbs": round(gbs, 1),
                       "frac": round(gbs / peak, 4),
                       "traffic_over_algorithmic": round(ratio, 3),
                       "traffic_over_algorithmic_roots": k,
                       "source": "profiles/traffic.json (ncu dram__bytes_read+write per "
                                 "launch, caches flushed per replay)"}
    out["b_alg"] = {"bytes_per_bfs": int(balg), "bytes_per_te": round(balg / float(np.max(te)), 3),
                    "frac": round(balg / kern_s / 1e9 / peak, 4),
                    "note": "SURVEY §8(d) normalisation: every core edge read once; a "
                            "direction-optimizing BFS reads ~2% of them, so this can exceed 1"}
    w0 = works[0]
    out["root0_levels"] = {"trace": w0.trace,
                           "frontier_or_unvisited": [int(x) for x in w0.levels[:, 0]],
                           "columns_read": [int(x) for x in w0.levels[:, 1]],
                           "claims": [int(x) for x in w0.levels[:, 2]],
                           "bytes": [int(x) for x in w0.bytes]}
    return out


def measure(scale, ef, mh, replay, steps, warmup, D, full=True, ctx=None):
    """The timed protocol on one workload: 64 roots x steps, per-root CUDA events,
    L2 flushed between roots; max over ranks per root. full adds the kernel-only
    pass, the roofline, the wall-clock pass and the e2e C-ABI pass."""
    import paper_2009_07463_b200 as eb
    from paper_2009_07463_b200 import etbfs as E
    g, cg, roots, starts, prep = prepare(scale, ef, mh)
    if D.world > 1:
        from paper_2009_07463_b200 import multi
        multi.connect(cg, D.rank, D.world)
        D.barrier()
    te, valid = validate_all(cg, starts, replay, D)
    reps = np.tile(starts, steps)
    D.barrier()
    with ClockSampler(D.local) as clk:
        ms, _ = E.time_roots(cg, reps, warmup=warmup * len(starts), flush_l2=True, replay=replay,
                             kernel_times=False)
    D.barrier()
    ms = D.reduce(ms, "MAX")
    sec = ms / 1e3
    te_rep = np.tile(te, steps)
    hm, per = harmonic_gteps(te_rep, sec)
    giant = te_rep == te_rep.max()
    hm_giant, _ = harmonic_gteps(te_rep[giant], sec[giant])
    rec = {"workload": workload_name(scale, ef), "mh": mh,
           "replay": "teolv" if replay == E.TreeReplay.TEOLV else "teet",
           "value": round(hm, 3), "unit": "GTEPS",
           "ms_per_step": round(float(ms.sum() / steps), 4),
           "ms_per_bfs_mean": round(float(np.mean(ms)), 4),
           "mean_gteps": round(float(per.mean()), 3), "min_gteps": round(float(per.min()), 3),
           "max_gteps": round(float(per.max()), 3),
           "hm_gteps_giant_component": round(hm_giant, 3),
           "giant_roots": int(np.count_nonzero(te == te.max())),
           "traversed_edges": int(te.max()),
           "validated_roots": len(valid), "all_valid": bool(all(valid)) if valid else None,
           "core_vertices": int(cg.core_vertex_count),
           "core_directed_edges": int(cg.restricted_edge_count),
           "tree_vertices": int(cg.tree_vertex_count),
           "gpu_launches": int(len(reps)), "clocks": clk.summary(), **prep}
    small = te != te.max()
    if small.any():
        rec["non_giant_roots"] = [{"root": int(r), "te": int(t),
                                   "ms": round(float(np.mean(ms.reshape(steps, -1)[:, i])), 4)}
                                  for i, (r, t) in enumerate(zip(roots, te)) if small[i]]
    if full:
        peak, peak_src = measured_peak_hbm()
        peak *= D.world
        _, kms = E.time_roots(cg, starts, warmup=len(starts), flush_l2=True, replay=replay)
        kms = D.reduce(kms, "MAX")
        if D.world == 1:
            rec["roofline"] = work_roofline(cg, starts, kms, replay, peak, rec["workload"], te)
            rec["roofline"]["peak_source"] = peak_src
        # wall clock per call, launch latency included, no copy, no flush
        wall = D.reduce(E.time_roots_wall(cg, np.tile(starts, 2), warmup=3, replay=replay), "MAX")
        whm, _ = harmonic_gteps(np.tile(te, 2), wall / 1e3)
        rec["wall_no_copy"] = {"value": round(whm, 3), "unit": "GTEPS",
                               "ms_per_bfs_mean": round(float(np.mean(wall)), 4),
                               "api": "etb_bfs_device + stream synchronise, host timer"}
        rec["e2e"] = e2e(cg, starts, te, replay, D)
        r0 = eb.et_bfs(cg, int(starts[0]), replay=replay, stats=True, want_parent=False,
                       want_depth=False)
        rec["timeline_root0"] = {"trace": r0.stats.direction_trace,
                                 "claims": r0.stats.level_claims,
                                 "level_end_us": [round(x / 1e3, 2) for x in r0.stats.level_ns],
                                 "total_us": round(r0.stats.total_ns / 1e3, 2)}
    if ctx is not None:
        ctx.update(g=g, cg=cg, roots=roots, starts=starts, te=te, valid=valid, sec=sec)
    return rec


def measure_emulated(ctx, parts_list, steps, warmup):
    """The multi-GPU algorithm (1D core partition, per-level bitmap allgather
    fused in the kernel) with G partitions emulated in ONE cooperative launch on
    this GPU: each partition gets 1/G of the SMs and exchanges through local
    memory. Same protocol as the headline (64 roots x steps, L2 flushed, CUDA
    events); every root validated. A G-GPU run would give each partition a whole
    B200, so this measures the algorithm's overhead (exchange, extra barriers),
    not multi-GPU throughput."""
    from paper_2009_07463_b200 import etbfs as E
    import paper_2009_07463_b200 as eb
    cg, starts, te = ctx["cg"], ctx["starts"], ctx["te"]
    single = float(np.mean(ctx["sec"])) * 1e3
    out = []
    for G in parts_list:
        E.partition(cg, G)
        try:
            ok = 0
            for s, t in zip(starts, te):
                E.bfs_device(cg, int(s))
                ok += int(bool(E.result_validate(cg, int(s))["passed"]) and
                          E.result_traversed_edges(cg) == int(t))
            ms, _ = E.time_roots(cg, np.tile(starts, steps), warmup=warmup * len(starts),
                                 flush_l2=True, kernel_times=False)
            hm, _ = harmonic_gteps(np.tile(te, steps), ms / 1e3)
            r0 = eb.et_bfs(cg, int(starts[0]), stats=True, want_parent=False, want_depth=False)
            out.append({"partitions": G, "value": round(hm, 3), "unit": "GTEPS",
                        "ms_per_bfs_mean": round(float(np.mean(ms)), 4),
                        "vs_single_partition_time": round(float(np.mean(ms)) / single, 3),
                        "validated_roots": int(ok), "all_valid": bool(ok == len(starts)),
                        "timeline_root0": {"trace": r0.stats.direction_trace,
                                           "level_end_us": [round(x / 1e3, 2)
                                                            for x in r0.stats.level_ns],
                                           "total_us": round(r0.stats.total_ns / 1e3, 2)}})
        finally:
            E.partition(cg, 1)
    return {"note": "G partitions in one cooperative launch on ONE B200 (1/G of the SMs each, "
                    "exchange through local memory): the multi-GPU kernel's overhead, not a "
                    "multi-GPU number", "single_partition_ms_per_bfs": round(single, 4),
            "runs": out}


def e2e(cg, starts, te, replay, D):
    """The reference-facing C-ABI call with a HOST output buffer: et_bfs with the
    BfsTree content (parent of every vertex, relaid ids, u32) copied device->host
    inside the wall-clock timing (etb_bfs_compact). With N ranks each rank copies
    its own partition's slice."""
    from paper_2009_07463_b200 import etbfs as E
    n = cg.vertex_count
    parent_h = np.empty(n, np.uint32)
    E._check(E.lib().etb_host_register(parent_h.ctypes.data, parent_h.nbytes))
    opt = E._opts(E.CoreKernel.HYBRID, replay, None)
    t = []
    try:
        for s in np.concatenate([starts[:3], starts]):
            D.barrier()
            c0 = time.perf_counter()
            E._check(E.lib().etb_bfs_compact(cg.handle, int(s), E.C.byref(opt), None,
                                             parent_h.ctypes.data))
            t.append(time.perf_counter() - c0)
    finally:
        E._check(E.lib().etb_host_unregister(parent_h.ctypes.data))
    t = D.reduce(np.array(t[3:]), "MAX")
    hm, _ = harmonic_gteps(te, t)
    # the isolated vertices that close the relaid id space never cross PCIe: the
    # call fills their range of the host buffer itself while the DMA runs
    live = n if D.world > 1 else cg.core_vertex_count + cg.tree_vertex_count
    return {"value": round(hm, 3), "unit": "GTEPS", "h2d_bytes_per_step": 8 * len(starts),
            "d2h_bytes_per_step": 4 * live * len(starts),
            "host_filled_bytes_per_step": 4 * (n - live) * len(starts),
            "api": "etb_bfs_compact (C-ABI, host parent u32[n] output, pinned, wall clock)"}


def run_ours(args):
    from paper_2009_07463_b200 import etbfs as E
    D = Dist()
    E.lib().etb_set_device(D.local)
    ctx = {}
    p = measure(args.scale, args.edgefactor, args.mh, E.TreeReplay.TEET, args.steps, args.warmup,
                D, full=True, ctx=ctx)
    out = {
        "metric": METRIC, "value": p["value"], "unit": "GTEPS", "n_gpus": D.world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": p["ms_per_step"],
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "u32",
        "data": "synthetic",
        "config": {"workload": p["workload"], "scale": args.scale, "edgefactor": args.edgefactor,
                   "roots": NROOTS, "root_seed": 1, "mh": args.mh, "replay": "teet",
                   "alpha": 14.0, "beta": 24.0,
                   "parallelism": f"1d-core-partition-{D.world}gpu" if D.world > 1 else "1gpu",
                   "l2": L2_NOTE},
        "roofline": p.pop("roofline", None),
        "e2e": p.pop("e2e"),
        "gpu_launches": p["gpu_launches"],
        "clocks": p.pop("clocks"),
        "detail": p,
    }
    if D.rank == 0 and args.report_json:
        write_report_v1(args, ctx["roots"], ctx["te"], ctx["sec"][:NROOTS], ctx["valid"],
                        p["preprocessing_s"], ctx["g"].vertex_count,
                        ctx["g"].undirected_edge_count())
    if D.rank == 0 and D.world == 1 and args.tree_out:
        # BenchConfig::tree_out (bench.hpp:45): the first root's tree, original ids, ETT1
        import paper_2009_07463_b200 as eb
        from paper_2009_07463_b200 import etbfs as E
        E.bfs_device(ctx["cg"], int(ctx["starts"][0]))
        _, par = E.result_original(ctx["cg"], levels=False)
        eb.write_tree(args.tree_out, int(ctx["roots"][0]), par)
    if D.world == 1 and not args.no_cpu_baseline:
        out["cpu_baseline"] = cpu_baseline(args, ctx)
    if D.world == 1 and args.emulate_partitions:
        out["partitioned_emulation"] = measure_emulated(
            ctx, [int(x) for x in args.emulate_partitions.split(",") if x.strip()], args.steps,
            args.warmup)
    ctx.clear()
    gc.collect()
    if D.world == 1:
        sec = []
        if args.mh == -1 and not args.no_paper_mode:
            pm = measure(args.scale, args.edgefactor, 0, E.TreeReplay.TEOLV, args.steps,
                         args.warmup, D, full=False)
            pm["note"] = "the paper's configuration (mh=0, TEOLV; PAPER.md:623), same protocol"
            sec.append(pm)
            gc.collect()
        for spec in [x for x in str(args.secondary).split(",") if x.strip() and x.strip() != "0"]:
            sc, ef = (int(v) for v in spec.split("/"))
            if (sc, ef) == (args.scale, args.edgefactor):
                continue
            r = measure(sc, ef, args.mh, E.TreeReplay.TEET, args.steps, args.warmup, D, full=True)
            r.pop("timeline_root0", None)
            sec.append(r)
            gc.collect()
        out["secondary"] = sec
    D.close()
    if D.rank == 0:
        print(json.dumps(out, default=_json_default), flush=True)


def _json_default(o):
    if isinstance(o, np.generic):
        return o.item()
    raise TypeError(f"not JSON serializable: {type(o).__name__}")


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


# ---------------------------------------------------------------- reference --
def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return None


def ref_time_roots(prep, deg, starts, replay=0):
    """Time the reference's et_bfs (the timed `traverse`, bench.cpp:269-271) per root."""
    secs, tes = [], []
    for s in starts:
        par, _, sec = prep.et_bfs(int(s), kernel=1, replay=replay)
        tes.append(int(deg[par != 0xFFFFFFFFFFFFFFFF].sum() // 2))
        secs.append(sec)
    return np.array(secs), np.array(tes, np.float64)


def cpu_baseline(args, ctx):
    """The reference's own et_bfs (oracle/_ref, all host cores) timed on a bounded
    sample of the headline workload. Its input ClassifiedGraph + EdgeTreeList is
    the device layout downloaded and wrapped in the reference's types: it is
    byte-identical to the reference's relayout_csr + extract_edge_tree_list
    (tests/test_gpu_parity.py pins new2old / relaid CSR / ETL hashes against the
    reference at s16, s22, s24/ef4 and s26), which spares the reference's
    single-threaded preprocessing (~6 min at s26) — untimed in the reference's
    own harness too (bench.cpp:253-256)."""
    import oracle as O
    if not O.ref_available():
        return {"value": None, "unit": "GTEPS", "cores": 0, "kind": "reference",
                "sample": "oracle/_ref not built"}
    threads = os.cpu_count() or 1
    O.ref().ref_set_threads(threads)
    cg = ctx["cg"]
    t0 = time.perf_counter()
    n = cg.vertex_count
    new2old, _, types = cg.new2old, cg.old2new, cg.vertex_type
    row, col = cg.graph()
    from paper_2009_07463_b200 import etbfs as E
    src, dst, ce = E.extract_edge_tree_list(cg)
    prep = O.RefPrepared.from_arrays(n, cg.core_vertex_count, args.mh, new2old, types, row, col,
                                     src, dst, ce)
    del col, src, dst, ce
    gc.collect()
    load_s = time.perf_counter() - t0
    deg = np.diff(row).astype(np.int64)
    starts = ctx["starts"][: args.cpu_roots]
    secs, tes = ref_time_roots(prep, deg, starts)
    del prep
    hm, _ = harmonic_gteps(tes, secs)
    k = len(starts)
    gsec = np.asarray(ctx["sec"]).reshape(-1, NROOTS)[:, :k]
    ghm, _ = harmonic_gteps(np.tile(ctx["te"][:k], gsec.shape[0]), gsec.reshape(-1))
    return {"value": round(hm, 4), "unit": "GTEPS", "cores": threads, "kind": "reference",
            "gpu_same_roots_gteps": round(ghm, 3),
            "sample": f"unmodified reference et_bfs (kHybrid, TEET, mh={args.mh}) via oracle/_ref "
                      f"on the first {len(starts)} of the 64 seed-1 roots of "
                      f"{workload_name(args.scale, args.edgefactor)}, {threads} OpenMP threads, "
                      f"{float(secs.sum()):.1f}s of CPU work; its ClassifiedGraph is the device "
                      f"layout downloaded ({load_s:.1f}s, untimed; byte-identical to the "
                      f"reference's relayout, pinned by the parity tests)",
            "seconds_per_root": [round(float(x), 4) for x in secs],
            "cpu_model": cpu_model()}


def run_reference(args):
    """The unmodified reference's own pipeline (oracle/_ref, compiled from
    /root/reference/proj/src by oracle/Makefile): generate_kronecker -> build_csr
    (tuples freed, the lean path) -> classify_vertices -> relayout_csr ->
    extract_edge_tree_list untimed (bench.cpp:253-256), then its et_bfs timed per
    root (bench.cpp:269-271), ref_roots_per_step roots per step, all host cores."""
    rank, world, _ = env_rank()
    if rank != 0:
        return
    import oracle as O
    if not O.ref_available():
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref not built"}))
        return
    threads = os.cpu_count() or 1
    O.ref().ref_set_threads(threads)
    t0 = time.perf_counter()
    csr = O.RefCsr.kronecker(args.scale, args.edgefactor, 1)
    deg_orig = csr.degrees()
    prep = O.RefPrepared(csr, args.mh)
    roots = csr.select_roots(NROOTS, 1)
    n = 1 << args.scale
    new2old = np.empty(n, np.uint64)
    O.ref().ref_prep_copy(prep.h, O._ptr(new2old), None, None, None, None, None, None)
    old2new = np.empty(n, np.int64)
    old2new[new2old.astype(np.int64)] = np.arange(n)
    deg = deg_orig[new2old.astype(np.int64)].astype(np.int64)  # relaid-space degrees
    del csr
    gc.collect()
    prep_s = time.perf_counter() - t0
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
        "n_gpus": max(world, args.gpus), "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(float(secs.sum() / args.steps * 1e3), 3), "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "u64", "data": "synthetic",
        "config": {"workload": workload_name(args.scale, args.edgefactor),
                   "scale": args.scale, "edgefactor": args.edgefactor, "roots": NROOTS,
                   "root_seed": 1, "mh": args.mh, "replay": "teet", "alpha": 14.0, "beta": 24.0,
                   "parallelism": f"openmp{threads}", "l2": "not flushed (CPU)"},
        "cpu_baseline": {"value": round(hm, 4), "unit": "GTEPS", "cores": threads,
                         "kind": "reference",
                         "sample": f"{per_step} roots per step (round robin over the 64 seed-1 "
                                   f"roots), unmodified reference et_bfs via oracle/_ref after its "
                                   f"own untimed preprocessing ({prep_s:.0f}s)",
                         "cpu_model": cpu_model()},
        "e2e": {"value": round(hm, 4), "unit": "GTEPS", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
        "detail": {"mean_gteps": round(float(per.mean()), 4), "preprocessing_s": round(prep_s, 2),
                   "roots_timed": int(len(secs)), "traversed_edges": int(tes.max())},
    }
    print(json.dumps(out), flush=True)


# --------------------------------------------------------------------- main --
def spawn_ranks(n):
    """--gpus N > 1 outside torchrun: re-launch this command as N ranks."""
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={n}", "--master-addr", "127.0.0.1", "--master-port", str(port),
           os.path.abspath(__file__), *sys.argv[1:]]
    return subprocess.call(cmd)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--scale", type=int, default=26)
    ap.add_argument("--edgefactor", type=int, default=16)
    ap.add_argument("--mh", type=int, default=-1)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-roots", type=int, default=8)
    ap.add_argument("--ref-roots-per-step", type=int, default=2)
    ap.add_argument("--report-json", default=None,
                    help="also write the reference's JSON report (schema v1, bench.cpp:301-343)")
    ap.add_argument("--tree-out", default=None,
                    help="write the first root's BFS tree (original ids) as an ETT1 file")
    ap.add_argument("--no-paper-mode", action="store_true",
                    help="skip the mh=0/TEOLV line at the headline scale")
    ap.add_argument("--secondary", default="22/16,24/4,28/16",
                    help="comma list of scale/edgefactor workloads timed under 'secondary' "
                         "(0 = none)")
    ap.add_argument("--emulate-partitions", default="2,4,8",
                    help="partition counts emulated on one GPU at the headline scale ('' = none)")
    ap.add_argument("--dry-ranks", action="store_true", help=argparse.SUPPRESS)
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "ours" and args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(spawn_ranks(args.gpus))
    if args.dry_ranks:  # launch plumbing only (tests): each rank reports its place
        rank, world, local = env_rank()
        print(json.dumps({"dry_ranks": True, "rank": rank, "n_gpus": world, "local_rank": local}),
              flush=True)
        return
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
