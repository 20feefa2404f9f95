#!/usr/bin/env python
"""Benchmark of the B200 Vietoris-Rips filtration build (BASELINE.json metric:
ranked simplices/s (edges + triangles + tetrahedra) and HBM GB/s vs peak).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--workload C5B] [--impl ours|reference]

One step = one full vrb_build (S1-S8: distances, edge ranking, neighbourhood
lists, triangle count + fill with D_2 rows, tie-group sort) over the
workload's synthetic points, already resident in HBM.  Outputs (55 GB for
C5B) are far larger than L2 and L2 is additionally flushed between steps.
For N > 1 (torchrun) every rank runs vrb_build_dist; time = max over ranks.

--impl reference times the CPU oracle (oracle/, single thread) on a bounded
sample of the same workload (the base contract's reference arm; this tier has
no reference implementation).
"""
from __future__ import annotations

import argparse
import json
import math
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import workloads  # noqa: E402

METRIC = "ranked simplices/sec (edges+tri+tet)"
UNIT = "simplices/s"
# bytes each triangle's outputs take (vertices 12 + filt 4 + D_2 rows 12):
# the fill kernel's algorithmic bytes per unit
TRI_OUT_BYTES = 28
TET_OUT_BYTES = 36    # 4 vertices + filt + 4 D_3 rows, u32 each
# SURVEY 8(d) B_alg per unit for the whole path (sort-based accounting)
SURVEY_BALG = {"edge_k1": 44, "edge_k2": 56, "tri": 44, "tet": 52}
ORACLE_SAMPLE = {"C1": 50, "C2": 1000, "C3": 900, "C4": 2200, "C5A": 6000, "C5B": 4400, "HIV": 500}


def _host_cpu():
    """(logical cores of the host, CPU model) -- context for the oracle baseline."""
    model = None
    try:
        with open("/proc/cpuinfo") as f:
            for ln in f:
                if ln.startswith("model name"):
                    model = ln.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    return os.cpu_count(), model


def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "50"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.th = threading.Thread(target=self._read, daemon=True)
            self.th.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], [], set()
        names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 6:
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[2:6]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        if not sm:
            return None
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": float(max(mx)), "reasons": sorted(reasons),
                "samples": len(sm)}


def _ncu_traffic(workload: str, kernel: str):
    """dram read+write bytes per launch of the roofline kernel, from the
    committed ncu capture (profiles/fill_traffic.json)."""
    path = os.path.join(ROOT, "profiles", "fill_traffic.json")
    try:
        with open(path) as f:
            d = json.load(f)
        e = d.get(workload, {})
        return e.get("dram_bytes_per_launch") if e.get("kernel", "k_triangles<fill>") == kernel else None
    except Exception:
        return None


def oracle_sample(workload: workloads.Workload, m: int):
    """Time the oracle (as it stands) on the first m points of the workload:
    steps 1-7 (edges, ranks, simplices, order, boundary).  Returns
    (simplices, seconds)."""
    import oracle

    X = workload.points()[:m]
    if workload.kind == "matrix":
        X = np.ascontiguousarray(X[:, :m])
    t0 = time.perf_counter()
    o = oracle.Oracle(None, workload.radius, D=X) if workload.kind == "matrix" else oracle.Oracle(X, workload.radius)
    units = o.E
    if workload.maxdim >= 1:
        units += o.simplices(2)[0].shape[0]
    if workload.maxdim >= 2:
        units += o.simplices(3)[0].shape[0]
    dt = time.perf_counter() - t0
    del o
    return units, dt


def run_reference(args, rank, world):
    if rank != 0:
        return
    w = workloads.WORKLOADS[args.workload]
    m = min(ORACLE_SAMPLE.get(args.workload, 2000), w.points().shape[0])
    # ORACLE_SAMPLE is sized for ~10-30 s per step; many steps shrink the
    # sample so the whole run stays within a few minutes (the oracle's work
    # grows as m^3 with triangles, m^2 for edges only)
    nrun = max(1, args.steps + args.warmup)
    if nrun > 8:
        m = max(50, int(m * (8.0 / nrun) ** (1.0 / (3.0 if w.maxdim >= 1 else 2.0))))
    for _ in range(args.warmup):
        oracle_sample(w, m)
    tot_units, tot_s = 0, 0.0
    for _ in range(args.steps):
        u, s = oracle_sample(w, m)
        tot_units += u
        tot_s += s
    value = tot_units / tot_s
    sample = f"first {m} of {w.points().shape[0]} points of {args.workload}, full oracle steps 1-7"
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * tot_s / args.steps,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64/u32",
        "data": "synthetic", "config": {"workload": args.workload, "desc": w.config, "maxdim": w.maxdim,
                                        "radius": w.radius if math.isfinite(w.radius) else "inf",
                                        "sample_points": m},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": 1, "kind": "oracle", "sample": sample,
                         "host_cores": _host_cpu()[0], "host_cpu": _host_cpu()[1]},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--workload", default="C5B", choices=sorted(workloads.WORKLOADS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    if args.warmup < 3 and args.impl == "ours":
        args.warmup = 3

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        return run_reference(args, rank, world)

    import torch
    import torch.distributed as dist

    import paper_1809_04424_b200 as vrb

    # VRB_DIST_BACKEND=gloo: exercise the N > 1 path with several ranks on one
    # GPU (tests only: gloo stages the exchange through the host); default NCCL
    backend = os.environ.get("VRB_DIST_BACKEND", "nccl")
    dev_index = local % max(1, torch.cuda.device_count()) if backend != "nccl" else local
    torch.cuda.set_device(dev_index)
    if world > 1:
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", dev_index))
        else:
            dist.init_process_group(backend)
    w = workloads.WORKLOADS[args.workload]
    X = w.points()
    Xd = torch.from_numpy(X).cuda()
    vrb.use_torch_allocator(True)
    flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")   # 512 MB > 126 MB L2

    def one_build(points):
        if w.kind == "matrix":   # F3: a distance matrix (HIV), one GPU
            if world > 1:
                raise SystemExit("distance-matrix workloads run on one GPU")
            return vrb.build_dm(points, maxdim=w.maxdim, radius=w.radius)
        if world > 1:
            return vrb.build_dist(points, maxdim=w.maxdim, radius=w.radius)
        return vrb.build(points, maxdim=w.maxdim, radius=w.radius)

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    for _ in range(args.warmup):
        r = one_build(Xd)
        del r
    torch.cuda.synchronize()

    vrb.set_profiling(True)
    step_ms, fill_ms, tet_ms, stage_acc = [], [], [], {}
    edge_path = None
    counts = None
    launches = 0
    s = torch.cuda.current_stream()
    with ClockSampler(dev_index) as clocks:
        for _ in range(args.steps):
            flush.fill_(1)
            barrier()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            l0 = vrb.launch_count()
            e0.record(s)
            r = one_build(Xd)
            e1.record(s)
            torch.cuda.synchronize()
            launches += vrb.launch_count() - l0
            step_ms.append(e0.elapsed_time(e1))
            st = vrb.last_stage_ms()
            fill_ms.append(st["fill"])
            tet_ms.append(st["tet_fill"])
            for k, v in st.items():
                stage_acc[k] = stage_acc.get(k, 0.0) + v
            if counts is None:
                counts = [r.count(k) for k in range(w.maxdim + 2)]
                edge_path = vrb.last_edge_path()
            del r
    vrb.set_profiling(False)
    # F1 (outside the step): dimension-0 persistence of a build, device-timed;
    # one untimed call first (first launches of its kernels), then the median
    # of 3 calls on fresh handles (the call is short and has host syncs)
    h0 = None
    if world == 1:
        h0_ms = []
        for rep in range(4):
            r = one_build(Xd)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(s)
            _, _, ness = r.h0()
            e1.record(s)
            torch.cuda.synchronize()
            if rep:
                h0_ms.append(e0.elapsed_time(e1))
            del r
        h0 = {"ms": float(np.median(h0_ms)), "ms_all": h0_ms, "essential_bars": int(ness),
              "finite_bars": int(counts[0][0] - ness) if counts else None}
        # F1 "clear and compress": D_2 without the H0 forest's rows,
        # on a build whose H0 is already computed (device-timed, not part of the step)
        if w.maxdim >= 1:
            cc_ms = []
            for rep in range(2):   # the first call also grows the allocator's pool for its outputs
                r = one_build(Xd)
                r.h0()
                torch.cuda.synchronize()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(s)
                cp, rv, rm = r.compress_d2()
                e1.record(s)
                torch.cuda.synchronize()
                cc_ms.append(e0.elapsed_time(e1))
                if rep == 0:
                    del r, cp, rv, rm
            T_ = counts[2][0]
            h0["clear_compress"] = {"ms": cc_ms[-1], "ms_first_call": cc_ms[0], "d2_rows": int(counts[1][0]),
                                    "rows_kept": int(rm.numel()),
                                    "d2_nnz": int(3 * T_), "nnz_kept": int(rv.numel()),
                                    "nnz_removed_frac": (1.0 - rv.numel() / (3 * T_)) if T_ else 0.0}
            del r, cp, rv, rm
    total_ms = float(sum(step_ms))
    if world > 1:
        t = torch.tensor([total_ms], device="cuda", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_ms = float(t.item())
    units_global = sum(c[0] for c in counts[1:])            # E + T (+ Q), global
    value = units_global * args.steps / (total_ms / 1e3)
    ms_per_step = total_ms / args.steps

    # roofline of the dominant kernel: the triangle fill (k_triangles<true>),
    # or the tetrahedron fill when it takes longer (max dim 2)
    peak, peak_kind = _peaks()
    T_local = counts[2][2] if len(counts) > 2 else 0
    Q_local = counts[3][2] if len(counts) > 3 else 0
    fill_avg = float(np.mean(fill_ms)) if fill_ms else 0.0
    tet_avg = float(np.mean(tet_ms)) if tet_ms else 0.0
    roofline = None
    if Q_local and tet_avg > fill_avg:
        kname = "k_tets_dense<fill>" if X.shape[0] <= 16384 else "k_tets<fill>"
        bytes_per_launch, kern_ms = TET_OUT_BYTES * Q_local, tet_avg
    elif T_local and fill_avg > 0:
        kname, bytes_per_launch, kern_ms = "k_triangles<fill>", TRI_OUT_BYTES * T_local, fill_avg
    elif w.maxdim == 0 and stage_acc.get("edge_rank", 0.0) > 0:
        # edges only (C5A): S3 as a whole against SURVEY 8(d)'s 44 B per edge
        # (sort payload written and read once + the edge outputs)
        kname = "S3 edge rank (" + edge_path + " path)"
        bytes_per_launch, kern_ms = SURVEY_BALG["edge_k1"] * counts[1][2], stage_acc["edge_rank"] / args.steps
    else:
        kname = None
    if kname:
        achieved = bytes_per_launch / (kern_ms / 1e3) / 1e9
        traffic = _ncu_traffic(args.workload, kname) if world == 1 else None   # capture is of the 1-GPU launch
        roofline = {"bound": "hbm", "kernel": kname, "achieved": achieved, "peak": peak,
                    "peak_kind": peak_kind, "unit": "GB/s", "frac": achieved / peak,
                    "traffic": traffic, "algorithmic_bytes_per_launch": bytes_per_launch,
                    "kernel_ms": kern_ms, "share_of_step": kern_ms / (ms_per_step or 1.0)}
    # whole-path fraction against SURVEY 8(d) B_alg
    E = counts[1][0]
    T = counts[2][0] if len(counts) > 2 else 0
    Q = counts[3][0] if len(counts) > 3 else 0
    balg = (E * (SURVEY_BALG["edge_k2"] if w.maxdim >= 1 else SURVEY_BALG["edge_k1"]) + T * SURVEY_BALG["tri"]
            + Q * SURVEY_BALG["tet"])
    path_gbs = balg / (ms_per_step / 1e3) / 1e9

    # e2e: through the C-ABI host path: pinned host points -> H2D inside
    # vrb_build -> build -> D2H of the per-dimension counts and value_of_rank
    e2e = None
    if not args.no_e2e:
        Xh = torch.from_numpy(X).pin_memory()
        # pinned host buffer for the result read-back, allocated once (a
        # pinned allocation is host work outside the library call)
        host_vor = torch.empty(max(1, counts[1][0]), dtype=torch.float64, pin_memory=True)
        e2e_ms = []
        d2h = 0
        for _ in range(max(1, min(args.steps, 3))):
            flush.fill_(2)
            barrier()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(s)
            r = one_build(Xh)
            vor = r.rank_values()
            host_vor[:vor.numel()].copy_(vor, non_blocking=True)
            e1.record(s)
            torch.cuda.synchronize()
            cnts = [r.count(k)[0] for k in range(w.maxdim + 2)]
            e2e_ms.append(e0.elapsed_time(e1))
            d2h = vor.numel() * 8 + 8 * len(cnts)
            del r, vor
        em = float(sum(e2e_ms))
        if world > 1:
            t = torch.tensor([em], device="cuda", dtype=torch.float64)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            em = float(t.item())
        e2e = {"value": units_global * len(e2e_ms) / (em / 1e3), "unit": UNIT,
               "h2d_bytes_per_step": int(X.nbytes), "d2h_bytes_per_step": int(d2h),
               "ms_per_step": em / len(e2e_ms),
               "d2h": "per-dimension counts + value_of_rank; the simplex, filt and boundary arrays "
                      "stay device-resident for the persistence reduction (%.1f GB for this workload)"
                      % (4e-9 * (2 * counts[1][0] + sum((k + 2) * counts[k][0] + (k + 1) * counts[k][0]
                                                       for k in range(2, len(counts)))))}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        m = min(ORACLE_SAMPLE.get(args.workload, 2000), X.shape[0])
        u, sec = oracle_sample(w, m)
        cpu = {"value": u / sec, "unit": UNIT, "cores": 1, "kind": "oracle",
               "sample": f"first {m} of {X.shape[0]} points of {args.workload} ({u} simplices, "
                         f"{sec:.1f} s), oracle steps 1-7 single-threaded",
               "host_cores": _host_cpu()[0], "host_cpu": _host_cpu()[1]}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64/u32", "data": "synthetic",
            "config": {"workload": args.workload, "desc": w.config, "n": int(X.shape[0]), "d": int(X.shape[1]),
                       "maxdim": w.maxdim, "radius": w.radius if math.isfinite(w.radius) else "inf",
                       "E": int(E), "T": int(T), "l2": "flushed (512 MB write) between steps; outputs >> L2",
                       "parallelism": f"owner-edge ranges x{world}" if world > 1 else "single GPU"},
            "gpu_launches": int(launches),
            "gpu_launches_per_step": int(launches // max(1, args.steps)),
            "roofline": roofline,
            "path_roofline": {"survey_balg_bytes": int(balg), "achieved_gbs": path_gbs, "peak": peak,
                              "frac": path_gbs / peak},
            "stage_ms": {k: v / args.steps for k, v in stage_acc.items()},
            "edge_path": edge_path,
            "clocks": clocks.summary(),
            "h0_barcodes": h0,
            "e2e": e2e,
            "cpu_baseline": cpu,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
