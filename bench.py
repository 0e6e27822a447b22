#!/usr/bin/env python
"""Benchmark of the level-scheduled PageRank solve (one JSON line on rank 0).

A step = one full solve of the hot path (the level loop of R3 over the
component DAG, then R1) on one synthetic BASELINE.json config with the layout
resident in HBM.  `value` = GEdge-updates/s (SolveReport.total_edge_work per
second) with weights/ranks already on the device; `e2e` = the same metric
through the C-ABI call lr_solve with pinned host buffers (weights H2D and
R3+R1 D2H inside the timed region).

  python bench.py [--config 5] [--steps K] [--warmup W] [--gpus N] [--impl ours|reference]

Default workload: config 5 (R-MAT scale 26, the north-star graph).

N>1 runs under torchrun; see DESIGN.md "Multi-GPU" for what is sharded.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "PageRank GEdge-updates/s (level-scheduled R3 solve + R1, tol 1e-12)"
UNIT = "GEdge-updates/s"
C_DAMP = 0.85
TOL = 1e-12


def log(*a):
    print(*a, file=sys.stderr, flush=True)


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


class Clocks:
    """nvidia-smi sampling during the timed region (B200_PROFILING.md clocks line)."""

    def __init__(self, gpu=0):
        self.gpu = gpu
        self.samples = []
        self._stop = threading.Event()
        self._t = None

    def __enter__(self):
        q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap,utilization.gpu")

        def run():
            while not self._stop.is_set():
                try:
                    out = subprocess.run(["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={q}",
                                          "--format=csv,noheader,nounits"], capture_output=True, text=True,
                                         timeout=5).stdout.strip()
                    if out:
                        self.samples.append([x.strip() for x in out.split(",")])
                except Exception:
                    pass
                self._stop.wait(0.2)

        self._t = threading.Thread(target=run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        busy = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit() and s[6].isdigit()
                and int(s[6]) > 10] or sm
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4) if s[2 + i].lower() == "active"})
        return {"sm_mhz": float(np.median(busy)) if busy else None,
                "sm_max_mhz": float(self.samples[0][1]) if self.samples[0][1].replace(".", "").isdigit() else None,
                "reasons": reasons, "samples": len(self.samples)}


def build_graph(lr, cfg, shrink):
    t0 = time.perf_counter()
    g = lr.config_graph(cfg, shrink)
    return g, (time.perf_counter() - t0) * 1e3


# BASELINE.json configs (same recipes as paper_1609_09068_b200.config_graph and
# oracle/lr_gen.c; kept here so the reference arm never imports the product)
WORKLOADS = {
    1: "planted 100k: 200 SCCs U[16,1024] rescaled to 50k vertices, out-trees, 50k inter edges, 10% dangling",
    2: "R-MAT scale 20, edge factor 16, (0.57,0.19,0.19,0.05), loops+dups removed",
    3: "R-MAT scale 23, edge factor 8, then 30% of vertices lose their out-edges",
    4: "deep DAG: 1000 levels x 16k vertices, SCCs U[2,64] (deg 6) + trees (branch U[1,4]), reach 1..8",
    5: "R-MAT scale 26, edge factor 16, (0.57,0.19,0.19,0.05), dedup",
}


def workload_name(cfg, shrink):
    return f"config{cfg}" + (f"-shrink{shrink}" if shrink else "") + ": " + WORKLOADS[cfg]


def config_dict(cfg, shrink, n, m):
    """The workload, identical in both arms (the driver compares them)."""
    return {"workload": workload_name(cfg, shrink), "c": C_DAMP, "tol": TOL, "weights": "uniform 1/|V|",
            "vertices": int(n), "edges": int(m), "small_threshold": 100,
            "l2": "GPU arm: L2 flushed (512 MB write) before every timed step"}


# ------------------------------------------------------------------ CPU legs
def cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


class RefLeg:
    """The reference's CPU path on the same workload: the levelrank sources
    compiled unmodified (oracle/_ref) when present, else the plain-C port
    (oracle/).  The graph comes from oracle/lr_gen.c (same edges as the
    product generator) and is built by the reference's own Graph::from_edges;
    partition + schedule run once (timed: the drop-in comparison), then each
    timed step is the reference's level loop (engine.cpp:126-158, unit
    solvers + propagate_weights) over that schedule with a pool of all host
    threads.  Bounded sample: when the full solve would not fit the budget,
    the SccLarge power series stops after its first multiply (every other
    unit is solved in full)."""

    def __init__(self, cfg, shrink, threads=None, budget_s=20.0):
        self.cfg, self.shrink, self.budget_s = cfg, shrink, budget_s
        self.threads = int(threads or os.cpu_count() or 1)
        self.err = None

    def setup(self):
        try:
            sys.path.insert(0, os.path.join(ROOT, "oracle"))
            from oracle_py import Oracle, Ref
            t0 = time.perf_counter()
            n, src, dst = Oracle().gen_config(self.cfg, self.shrink, threads=self.threads)
            self.gen_ms = (time.perf_counter() - t0) * 1e3
            self.n = n
            self.w = np.full(n, 1.0 / n)
            self.kind = "reference" if Ref.available() else "port"
            t0 = time.perf_counter()
            if self.kind == "reference":
                self.g = Ref().graph(n, src, dst)
                del src, dst
                self.graph_ms = (time.perf_counter() - t0) * 1e3
                t0 = time.perf_counter()
                self.prep = self.g.prepare(100)  # find_components + build_schedule
                self.prep_ms = (time.perf_counter() - t0) * 1e3
                # the SccLarge series stopped after one multiply (do-while,
                # solvers.cpp:146-160): every other unit in full plus one multiply
                _, _, iters, ms = self.g.prep_solve(self.prep, self.w, C_DAMP, TOL, large_tol=1e300,
                                                    threads=self.threads)
                self.large_tol = 0.0 if (iters == 0 or ms * 130 <= self.budget_s * 1e3) else 1e300
            else:
                self.g = Oracle().graph(n, src, dst)
                del src, dst
                self.graph_ms = (time.perf_counter() - t0) * 1e3
                self.prep_ms = None
            self.m = self.g.m
        except Exception as e:  # reported, never required
            self.err = e

    def steps(self, reps):
        if self.err:
            raise self.err
        out = []
        for _ in range(reps):
            if self.kind == "reference":
                _, work, iters, ms = self.g.prep_solve(self.prep, self.w, C_DAMP, TOL, large_tol=self.large_tol,
                                                       threads=self.threads)
                full = self.large_tol <= TOL
                sample = (f"reference level loop (oracle/_ref, -O3 -DNDEBUG, Parallel pool of {self.threads} on "
                          f"{cpu_model()}) over its own schedule; SccLarge series "
                          f"{'in full' if full else 'stopped after its first multiply'} ({iters} multiplies, "
                          f"{work / 1e9:.2f} G edge updates); graph + partition + schedule built once, untimed")
                cores = self.threads
            else:
                work, ms = self.g.sample_large_scc(self.w, C_DAMP, 4)
                sample = "oracle port: 4 multiplies of the largest SccLarge unit (push COO)"
                cores = 1
            out.append({"value": work / (ms / 1e3) / 1e9 if ms > 0 else None, "unit": UNIT, "cores": cores,
                        "kind": self.kind, "sample": sample, "edge_updates": int(work), "ms": ms})
        return out

    def methods(self):
        """SURVEY 8(d) CPU side on the same graph and weights: the reference's
        Sequential and Parallel level loops and its whole-graph power series
        (compute_baseline, solvers.cpp:164-198).  Each runs in full when the
        full solve fits the budget, else as the same bounded sample (the
        baseline: one whole-graph multiply, tol = inf)."""
        if self.err or self.kind != "reference":
            return None
        full = self.large_tol <= TOL
        res = {"threads": self.threads, "cpu_model": cpu_model(), "full_solves": full}
        for name, th in (("sequential", 1), ("parallel", self.threads)):
            _, work, iters, ms = self.g.prep_solve(self.prep, self.w, C_DAMP, TOL, large_tol=self.large_tol,
                                                   threads=th)
            res[name] = {"ms": ms, "edge_updates": int(work), "ge_s": work / ms / 1e6}
        t0 = time.perf_counter()
        _, rep = self.g.compute_baseline(self.w, C_DAMP, TOL if full else 1e300)
        ms = (time.perf_counter() - t0) * 1e3
        work = int(rep["iterative_edge_work"])
        res["whole_graph_baseline"] = {"ms": ms, "iterations": int(rep["total_iterations"]), "edge_updates": work,
                                       "ge_s": work / ms / 1e6}
        return res

    def drop_in(self, rate):
        """The reference's compute_pagerank wall (engine.cpp:99-180) =
        partition + schedule (measured) + solve (measured in full when the
        sample is the full solve, else extrapolated from the sample's rate)."""
        if self.err or self.kind != "reference":
            return None
        return {"partition_schedule_ms": self.prep_ms, "from_edges_ms": self.graph_ms,
                "solve_measured": self.large_tol <= TOL, "edge_update_rate_ge_s": rate}


def run_reference(args):
    """--impl reference: the reference's own CPU implementation of the path."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    leg = RefLeg(args.config, args.shrink, budget_s=args.ref_budget)
    leg.setup()
    steps = leg.steps(args.warmup + args.steps)[args.warmup:]
    res = steps[-1]
    value = float(np.mean([s["value"] for s in steps]))
    ms = float(np.mean([s["ms"] for s in steps]))
    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic", "impl": "reference",
            "config": config_dict(args.config, args.shrink, leg.n, leg.m),
            "cpu_baseline": {k: res[k] for k in ("value", "unit", "cores", "kind", "sample")},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "setup_s": {"generate": leg.gen_ms / 1e3, "from_edges": leg.graph_ms / 1e3,
                        "partition_schedule": (leg.prep_ms or 0) / 1e3},
            "product_library_mapped": product_mapped()}
    print(json.dumps(line), flush=True)


def product_mapped():
    """True if this process mapped the product's liblevelrank_b200.so."""
    try:
        with open("/proc/self/maps") as f:
            return any("liblevelrank_b200" in ln for ln in f)
    except OSError:
        return None


# ------------------------------------------------------------------ GPU leg
def run_ours(args):
    import torch
    import paper_1609_09068_b200 as lr

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    dist = None
    if world > 1:
        import torch.distributed as dist
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = torch.device("cuda", local)
    torch.cuda.set_device(dev)

    g, gen_ms = build_graph(lr, args.config, args.shrink)
    log(f"[rank {rank}] graph n={g.n} m={g.m} built in {gen_ms / 1e3:.1f}s")
    if world > 1:
        # the giant SCC is row-sharded over the ranks; NCCL id from rank 0
        obj = [lr.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        eng = lr.Engine(g, 100, device=local, rank=rank, world=world, nccl_id=obj[0])
    else:
        eng = lr.Engine(g, 100, device=local)
    log(f"[rank {rank}] plan {eng.plan_ms / 1e3:.1f}s upload {eng.upload_ms / 1e3:.1f}s "
        f"device bytes {eng.device_bytes() / 1e9:.2f} GB")
    n = g.n
    leg = setup_thread = None
    stream = torch.cuda.ExternalStream(eng.stream, device=dev)
    w_dev = torch.full((n,), 1.0 / n, dtype=torch.float64, device=dev)
    r3_dev = torch.empty(n, dtype=torch.float64, device=dev)
    r1_dev = torch.empty(n, dtype=torch.float64, device=dev)
    flush = torch.empty(512 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)  # > 126 MB L2
    params = lr.SolverParams(C_DAMP, TOL)

    # one host-API solve for the report (edge work, iteration counts)
    r3h, r1h, info0, iters = eng.solve(np.full(n, 1.0 / n), params)
    res_report = lr.compute_pagerank  # noqa: F841 (API kept for parity tests)
    layout = eng.plan.layout()
    kinds = layout["unit_kind"]
    edges = layout["unit_edges"]
    large = kinds == 3
    work = int((iters[large] * edges[large]).sum() + edges[~large].sum() + len(layout["xsrc"]))
    # in-edges of the largest grid unit served by K4c's shared-memory head
    # (spmv.cu: 16k head rows while the unit's pushed vector is <= 48 MB, else 8k)
    head_share = None
    if large.any():
        u = int(np.argmax(np.where(large, edges, -1)))
        r0, r1 = int(layout["unit_row_begin"][u]), int(layout["unit_row_begin"][u + 1])
        nhead = min(16384 if (r1 - r0) * 8 <= (48 << 20) else 8192, r1 - r0)
        ip = layout["iptr"]
        cols = layout["isrc"][ip[r0]:ip[r1]]
        head_share = float(np.count_nonzero(cols < r0 + nhead)) / max(1, len(cols))
    n_levels, n_units = int(layout["n_levels"]), int(layout["n_units"])
    del layout

    def dev_step():
        return eng.solve_ptr(w_dev.data_ptr(), r3_dev.data_ptr(), r1_dev.data_ptr(), host=False, params=params)

    torch.cuda.synchronize()
    for _ in range(args.warmup):
        dev_step()
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    times = []
    infos = []
    with Clocks(local) as clk:
        for _ in range(args.steps):
            with torch.cuda.stream(stream):
                flush.zero_()
                a = torch.cuda.Event(enable_timing=True)
                b = torch.cuda.Event(enable_timing=True)
                a.record(stream)
                infos.append(dev_step())
                b.record(stream)
            b.synchronize()
            times.append(a.elapsed_time(b))
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    ms = float(np.mean(times))
    if dist:
        t = torch.tensor([ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    value = work / (ms / 1e3) / 1e9  # one job split over the ranks (strong scaling)

    # e2e through lr_solve with pinned host buffers
    w_h = torch.full((n,), 1.0 / n, dtype=torch.float64).pin_memory()
    r3_h = torch.empty(n, dtype=torch.float64).pin_memory()

    # the reference's compute_pagerank returns R3 (EngineResult.ranks); R1 is
    # still computed on the device every step, only its copy-back is left out
    def host_step():
        return eng.solve_ptr(w_h.data_ptr(), r3_h.data_ptr(), 0, host=True, params=params)

    for _ in range(max(1, args.warmup)):
        host_step()
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    e2e_times = []
    for _ in range(args.steps):
        with torch.cuda.stream(stream):
            flush.zero_()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        host_step()
        e2e_times.append((time.perf_counter() - t0) * 1e3)
    e2e_ms = float(np.mean(e2e_times))
    if dist:
        t = torch.tensor([e2e_ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_ms = float(t.item())
    e2e_value = work / (e2e_ms / 1e3) / 1e9
    # the reference CPU leg builds its graph and schedule on a host thread
    # (ctypes calls release the GIL) -- only after the timed device and e2e
    # loops, overlapping the GPU whole-graph ablation below
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        leg = RefLeg(args.config, args.shrink, budget_s=args.ref_budget)
        setup_thread = threading.Thread(target=leg.setup, daemon=True)
        setup_thread.start()
    # parity spot check of the timed path vs the host-API result
    # (K5 accumulates rows with shared-memory atomics, whose arrival order varies
    # from launch to launch: results agree to rounding, iteration counts exactly)
    ref_t = torch.from_numpy(r3h)
    rel = float(((r3_h - ref_t).abs() / ref_t.abs().clamp_min(1e-300)).max())
    assert rel <= 1e-12, f"device-resident and host-API solves differ: max relative {rel:.3e}"
    assert all(i["total_iterations"] == info0["total_iterations"] for i in infos), "iteration totals differ between solves"

    inf = infos[-1]
    peak, peak_kind = peaks()
    achieved = None
    if inf["spmv_active_ms"] > 0:
        achieved = inf["spmv_bytes"] / (inf["spmv_active_ms"] / 1e3) / 1e9
    traffic = None
    tpath = os.path.join(ROOT, "profiles", f"traffic_config{args.config}.json")
    if os.path.exists(tpath) and not args.shrink:
        with open(tpath) as f:
            traffic = json.load(f).get("dram_bytes_per_launch")
    roofline = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                "frac": (achieved / peak) if achieved else None, "traffic": traffic,
                "frac_vs_nominal_8000": (achieved / 8000.0) if achieved else None,
                "kernel": ("k_spmv_blk (K5: SccLarge power-series SpMV by dest-row blocks, source-sorted in-edges)"
                           if eng.blk_units() > 0 else "k_spmv_seg (K4c: SccLarge power-series SpMV)"),
                "peak_kind": peak_kind,
                "algorithmic_bytes_per_launch": (inf["spmv_bytes"] / inf["spmv_active_launches"])
                if inf["spmv_active_launches"] else None,
                "avg_launch_ms": (inf["spmv_active_ms"] / inf["spmv_active_launches"])
                if inf["spmv_active_launches"] else None,
                "spmv_share_of_step": inf["spmv_active_ms"] / ms if ms > 0 else None}
    # the bound that applies (profiles/r01_gather_ceiling.md): every in-edge not
    # served by the shared-memory head is one random 8-byte gather = one L2 sector
    if achieved and head_share is not None and inf["spmv_edges"] and eng.blk_units() == 0:
        g_per_s = inf["spmv_edges"] * (1.0 - head_share) / (inf["spmv_active_ms"] / 1e3)
        roofline["gathers"] = {"head_share_of_in_edges": head_share, "global_gathers_per_s": g_per_s,
                               "ceiling_l2_resident_per_s": 195e9, "ceiling_171MB_uniform_per_s": 86e9,
                               "frac_of_l2_resident_ceiling": g_per_s / 195e9,
                               "source": "tools/gather_bench.cu, profiles/r01_gather_ceiling.md"}

    # ablation on the same GPU: the reference's partition-free whole-graph power
    # series (compute_baseline, lr_plan_build_baseline) over the same graph
    gpu_base = None
    if world == 1 and not args.no_gpu_baseline:
        try:
            beng = lr.Engine(g, device=local, baseline=True)
            binfo0 = beng.solve_ptr(w_dev.data_ptr(), r3_dev.data_ptr(), r1_dev.data_ptr(), host=False, params=params)
            bt = []
            for _ in range(args.steps):
                with torch.cuda.stream(stream):
                    flush.zero_()
                torch.cuda.synchronize()
                bi = beng.solve_ptr(w_dev.data_ptr(), r3_dev.data_ptr(), r1_dev.data_ptr(), host=False,
                                    params=params)
                bt.append(bi["device_ms"])
            bms = float(np.mean(bt))
            bwork = int(binfo0["iterative_edge_work"])
            gpu_base = {"what": "whole-graph power series (compute_baseline) on this GPU, same graph and weights",
                        "value": bwork / (bms / 1e3) / 1e9, "unit": UNIT, "ms_per_step": bms,
                        "iterations": int(binfo0["total_iterations"]), "edge_updates_per_step": bwork,
                        "partitioned_speedup": bms / ms, "plan_s": beng.plan_ms / 1e3}
            del beng
        except Exception as e:  # reported, never required
            gpu_base = {"value": None, "error": str(e)}

    cpu = None
    methods = None
    ref_drop = None
    if leg is not None:
        setup_thread.join()
        try:
            cpu = leg.steps(1)[0]
            methods = leg.methods()
            cpu["reference_methods"] = methods
            ref_drop = leg.drop_in(cpu["value"])
        except Exception as e:  # the baseline is reported, never required
            cpu = {"value": None, "unit": UNIT, "cores": 0, "kind": "reference", "sample": f"failed: {e}"}

    # the drop-in call a user makes (lr_compute_pagerank: partition + layout on
    # the host, upload, one solve with host buffers) against the reference's
    # compute_pagerank wall (partition + schedule + solve)
    drop_in = {"ours_ms": {"plan": eng.plan_ms, "upload": eng.upload_ms, "solve_host_buffers": e2e_ms,
                           "total": eng.plan_ms + eng.upload_ms + e2e_ms}}
    if ref_drop:
        solve_ms = None
        if methods and methods.get("full_solves"):
            solve_ms = methods["parallel"]["ms"]
        elif ref_drop.get("edge_update_rate_ge_s"):
            solve_ms = work / ref_drop["edge_update_rate_ge_s"] / 1e6
        ref_drop["solve_ms"] = solve_ms
        ref_drop["solve_ms_kind"] = "measured (Parallel pool)" if ref_drop["solve_measured"] else \
            "extrapolated: this workload's edge updates at the sampled rate"
        ref_drop["total_ms"] = ref_drop["partition_schedule_ms"] + (solve_ms or 0.0)
        drop_in["reference_ms"] = ref_drop
        drop_in["speedup"] = ref_drop["total_ms"] / drop_in["ours_ms"]["total"]

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": config_dict(args.config, args.shrink, n, g.m),
            "parallelism": (f"giant-SCC rows sharded over {world} GPUs (chunked NCCL exchange per iteration), "
                            "large levels' other units split over the GPUs") if world > 1 else "1 GPU",
            "workload_stats": {"edge_updates_per_step": work, "iterative_edge_work": int(info0["iterative_edge_work"]),
                               "large_scc_iterations": int(iters[large].max()) if large.any() else 0,
                               "levels": n_levels, "units": n_units},
            "setup_s": {"generate": gen_ms / 1e3, "plan": eng.plan_ms / 1e3, "upload": eng.upload_ms / 1e3},
            "e2e": {"value": e2e_value, "unit": UNIT, "ms_per_step": e2e_ms, "h2d_bytes_per_step": 8 * n,
                    "d2h_bytes_per_step": 8 * n, "returns": "R3 (the reference's EngineResult.ranks); R1 computed on "
                    "the device, not copied back"},
            "gpu_launches": int(inf["kernel_launches"]) * args.steps,
            "roofline": roofline,
            "cpu_baseline": cpu,
            "drop_in": drop_in,
            "gpu_baseline": gpu_base,
            "clocks": clk.summary(),
        }
        print(json.dumps(line), flush=True)
    if dist:
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", type=int, default=int(os.environ.get("LR_BENCH_CONFIG", "5")))
    ap.add_argument("--shrink", type=int, default=0)
    ap.add_argument("--ref-budget", type=float, default=20.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-gpu-baseline", action="store_true")
    args = ap.parse_args()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
