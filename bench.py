#!/usr/bin/env python
"""Benchmark of the hot path (BASELINE.json metric): grid-node x control updates per
second of the semi-Lagrangian value-iteration sweeps, and time-to-solution of one
pass of the whole path (coarse pre-solve -> trajectory labels -> prolongation ->
partitioned fine solves -> min assembly), §4 ISA (line 389-408).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config 3] [--impl reference]

One process per GPU: with N > 1 and no torchrun environment, the script re-executes
itself under torch.distributed.run (N ranks, NCCL).  Prints ONE JSON line on rank 0.
Default workload: BASELINE configs[2] (4097^2 Zermelo, 16 sub-domains, fp32) — the
largest configuration that fits one GPU's time budget.  Inputs are
seeded and synthetic (hj_workloads).
"""
from __future__ import annotations

import argparse
import glob
import json
import os
import socket
import statistics
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import hj_workloads as W  # noqa: E402

METRIC = "grid-node x control updates/sec per sweep; time-to-solution at 1/2/4/8 B200"
UNIT = "node-control updates/s"
DEFAULT_CONFIG = 3
# Roofline of the fine sweep: the bracket of one node x control update is
# a bilinear form in the control's weights, so at least 3 fused multiply-adds; the FMA
# pipes retire 128 FMA lanes per SM clock.
FMA_PER_UPDATE = 3
FMA_LANES_PER_SM_CLK = 128
# algorithmic bytes per evaluated fine node and sweep: read V^n once
# (its neighbourhood is reused from shared memory), write V^{n+1}, read the class byte
BYTES_PER_NODE = {"f32": 4 + 4 + 1, "f64": 8 + 8 + 1}


def load_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f), "measured"
    except OSError:
        return {"hbm_gbs": 6650.0, "sm_max_mhz": 1965.0}, "fallback"


def ncu_evidence(workload):
    """The newest committed ncu summary of this workload's dominant kernel
    (profiles/<round>/ncu_roofline_<workload>.json, tools/ncu_roofline.py).  Newest = the
    last session directory in name order (r01 < ... < r13 < r2 < r2s < r2u): file mtimes
    are all equal in a fresh checkout."""
    paths = sorted(glob.glob(os.path.join(ROOT, "profiles", "*", f"ncu_roofline_{workload}.json")))
    if not paths:
        return None
    with open(paths[-1]) as f:
        d = json.load(f)
    d["file"] = os.path.relpath(paths[-1], ROOT)
    return d


class ClockSampler:
    """nvidia-smi style sampling of SM clocks and throttle reasons (NVML) during the
    timed region."""

    def __init__(self, index=0, period=0.1):
        self.index, self.period = index, period
        self.samples, self.reasons = [], set()
        self.max_mhz = None
        self._stop = threading.Event()
        self._t = None
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception:  # pragma: no cover
            self.nv = None

    def _run(self):
        nv = self.nv
        names = {"hw_slowdown": 0x8, "hw_thermal_slowdown": 0x40, "sw_thermal_slowdown": 0x20,
                 "sw_power_cap": 0x4, "hw_power_brake_slowdown": 0x80}
        while not self._stop.is_set():
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM))
                r = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for n, bit in names.items():
                    if r & bit:
                        self.reasons.add(n)
            except Exception:
                pass
            self._stop.wait(self.period)

    def __enter__(self):
        if self.nv:
            self._t = threading.Thread(target=self._run, daemon=True)
            self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self._t:
            self._t.join()

    def summary(self):
        return {"sm_mhz": statistics.median(self.samples) if self.samples else None,
                "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons),
                "samples": len(self.samples)}


# ----------------------------------------------------------------------------------
# the oracle on host cores (reference arm and cpu_baseline): Jacobi sweeps of its fp64
# operator over a bounded sample of the fine grid's rows
# ----------------------------------------------------------------------------------
def oracle_rows_rate(prob, rows):
    """One application of the oracle's T to `rows` consecutive node rows (axis 1) in the
    middle of the fine grid's first plane, on V = V^0.  Returns (updates/s, seconds,
    interior nodes of the sample, the row range)."""
    import oracle
    o = oracle.OracleProblem(prob)
    cls = o.classes()
    V = o.initial(cls)
    out = V.copy()
    n0, n1 = prob.grid.n[0], prob.grid.n[1]
    r0 = max(0, n1 // 2 - rows // 2)
    r1 = min(n1, r0 + rows)
    interior = int((cls[r0 * n0:r1 * n0] == oracle.INTERIOR).sum())
    t0 = time.perf_counter()
    o.apply_T_rows(V, cls, out, r0, r1)
    dt = time.perf_counter() - t0
    return interior * prob.n_controls / dt, dt, interior, (r0, r1)


def sample_rows(prob, target_updates):
    n0 = prob.grid.n[0]
    per_row = n0 * prob.n_controls
    return int(max(1, min(prob.grid.n[1], target_updates // per_row)))


def run_reference(args, cfg, rank, world):
    """--impl reference: the oracle (this tier's reference arm) on the host's cores."""
    if rank != 0:
        return
    import oracle
    prob = cfg.fine
    rows = sample_rows(prob, args.ref_updates)
    for _ in range(args.warmup):
        oracle_rows_rate(prob, rows)
    rates, times = [], []
    for _ in range(args.steps):
        r, dt, interior, rr = oracle_rows_rate(prob, rows)
        rates.append(r)
        times.append(dt)
    value = float(np.mean(rates))
    sample = (f"per step: 1 Jacobi application of the fp64 oracle operator to node rows "
              f"[{rr[0]}, {rr[1]}) of the {list(prob.grid.n)} fine grid ({interior} interior "
              f"nodes x {prob.n_controls} controls, {oracle.threads()} OpenMP threads)")
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT,
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": 1e3 * float(np.mean(times)), "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": cfg.name, "grid": list(prob.grid.n),
                       "controls": prob.n_controls, "sample_rows": list(rr),
                       "l2": "CPU run (no GPU L2)"},
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": oracle.threads(),
                             "kind": "oracle", "sample": sample},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def respawn_under_torchrun(n):
    """bench.py --gpus N outside torchrun: re-execute under torch.distributed.run."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()),
           os.path.abspath(__file__), *sys.argv[1:]]
    os.execv(sys.executable, cmd)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", type=int, default=DEFAULT_CONFIG)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--dtype", default=None)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--ref-updates", type=float, default=1.2e8,
                    help="node x control updates per reference-arm step (a row sample)")
    ap.add_argument("--labeller", default="trajectory", choices=["trajectory", "ra"],
                    help="sub-domain reconstruction: north_star trajectories or the paper's RA")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)

    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        respawn_under_torchrun(args.gpus)
    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    local = int(os.environ.get("LOCAL_RANK", 0))
    cfg = W.make(args.config)

    if args.impl == "reference":
        run_reference(args, cfg, rank, world)
        return

    import torch
    import torch.distributed as dist

    from paper_1405_3521_b200 import hj, pipeline

    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dtype = args.dtype or cfg.dtype
    fine = hj.DeviceProblem(cfg.fine, dtype, reuse_buffers=True)
    coarse = hj.DeviceProblem(cfg.coarse, dtype, reuse_buffers=True)
    l2_flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device="cuda")

    def barrier():
        if world > 1:
            dist.barrier()

    def step():
        return pipeline.run_isa(cfg, dtype, rank=rank, world=world, fine=fine, coarse=coarse,
                                labeller=args.labeller)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()

    st = torch.cuda.current_stream()
    step_ms, nominal, evaluated, fine_eval, fine_nodes = [], 0, 0, 0, 0
    sweep_ms, launches = 0.0, 0
    with ClockSampler(local) as clocks:
        for _ in range(args.steps):
            l2_flush.fill_(1)                       # L2 flush between timed steps
            barrier()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(st)
            res = step()
            e1.record(st)
            torch.cuda.synchronize()
            barrier()
            step_ms.append(e0.elapsed_time(e1))
            rc = res["coarse_report"]
            fr = [r for r in res["reports"] if r is not None]
            nominal += rc["node_updates"] + sum(r["node_updates"] for r in fr)
            fine_eval += sum(r["evaluated_updates"] for r in fr)
            evaluated += rc["evaluated_updates"] + sum(r["evaluated_updates"] for r in fr)
            if fr:
                sweep_ms += fr[0]["device_ms"]
            # coarse solve + label/prolong (2) + plan (2) + partitioned solve
            launches += rc["launches"] + 2 + 2 + sum(r["launches"] for r in fr)
    total_ms = float(np.sum(step_ms))
    mine = {"rank": rank, "subdomains": [k for k in range(cfg.m) if (res["solve_set"] >> k) & 1],
            "step_ms": [round(x, 3) for x in step_ms], "fine_ms": res["timings"]["fine_ms"],
            "evaluated_updates_per_step": evaluated / args.steps,
            "fine_sweeps": max((r["iterations"] for r in res["reports"] if r), default=0)}
    per_rank = [mine]
    if world > 1:
        t = torch.tensor([total_ms, nominal, evaluated, fine_eval, sweep_ms], dtype=torch.float64,
                         device="cuda")
        tmax = t.clone()
        dist.all_reduce(tmax, op=dist.ReduceOp.MAX)
        dist.all_reduce(t, op=dist.ReduceOp.SUM)
        total_ms, nominal, evaluated, fine_eval = (float(tmax[0]), float(t[1]), float(t[2]),
                                                   float(t[3]))
        sweep_ms = float(tmax[4])
        per_rank = [None] * world
        dist.all_gather_object(per_rank, mine)
    value = evaluated / (total_ms / 1e3)

    # ---- end to end through the public API with host buffers ------------------
    h_in = {"fine_piece": fine.piece.cpu().pin_memory(), "coarse_piece": coarse.piece.cpu().pin_memory()}
    if fine.speed is not None:
        h_in["fine_speed"] = fine.speed.cpu().pin_memory()
        h_in["coarse_speed"] = coarse.speed.cpu().pin_memory()
    # (the result's own dtype: a converting device->host copy is not asynchronous)
    h_out = torch.empty(fine.N, dtype=torch.float64 if dtype == "f64" else
                        torch.float32).pin_memory()
    h2d = sum(t.numel() * t.element_size() for t in h_in.values())
    d2h = h_out.numel() * h_out.element_size()
    e2e_ms, e2e_eval = [], 0
    for it in range(1 + max(1, min(args.steps, 2))):     # (pass 0: untimed warm-up)
        l2_flush.fill_(1)
        barrier()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        fine.piece.copy_(h_in["fine_piece"], non_blocking=True)
        coarse.piece.copy_(h_in["coarse_piece"], non_blocking=True)
        if fine.speed is not None:
            fine.speed.copy_(h_in["fine_speed"], non_blocking=True)
            coarse.speed.copy_(h_in["coarse_speed"], non_blocking=True)
        res = step()
        h_out.copy_(res["V"], non_blocking=True)
        e1.record(st)
        torch.cuda.synchronize()
        barrier()
        if it == 0:
            continue
        e2e_ms.append(e0.elapsed_time(e1))
        e2e_eval += res["coarse_report"]["evaluated_updates"] + sum(
            r["evaluated_updates"] for r in res["reports"] if r is not None)
    e2e_total = float(np.sum(e2e_ms))
    if world > 1:
        t = torch.tensor([e2e_total, e2e_eval], dtype=torch.float64, device="cuda")
        tmax = t.clone()
        dist.all_reduce(tmax, op=dist.ReduceOp.MAX)
        dist.all_reduce(t, op=dist.ReduceOp.SUM)
        e2e_total, e2e_eval = float(tmax[0]), float(t[1])
    e2e_value = e2e_eval / (e2e_total / 1e3)

    # label / sub-domain statistics of the last pass (GPU margins; R11)
    lab = res["labels"]
    labels = None
    if lab.get("label") is not None:
        mar = lab["margin"]
        bits = res["mask"]
        cover = int(sum(int(((bits >> k) & 1).sum()) for k in range(res["n_sets"])))
        labels = {"coarse_nodes": int(mar.numel()),
                  "margin_ties": int((mar <= 1e-9).sum()),
                  "unlabelled_all_sets": int((lab["label"] == -1).sum()),
                  "exit_set": int((lab["label"] == -2).sum()),
                  "sets": res["n_sets"],
                  "subdomain_nodes_over_N": round(cover / fine.N, 3)}

    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return

    peaks, peak_kind = load_peaks()
    sm_mhz = float(peaks.get("sm_max_mhz", 1965.0))
    peak_fma = 148 * FMA_LANES_PER_SM_CLK * sm_mhz * 1e6 / 1e12   # T FMA/s
    # per GPU and step: the fine solve's evaluated updates (all ranks / N) over the fine-solve
    # device time of the slowest rank
    fine_s = sweep_ms / args.steps / 1e3
    fine_upd = fine_eval / world / args.steps
    achieved = fine_upd * FMA_PER_UPDATE / fine_s / 1e12 if fine_s else 0.0
    ncu = ncu_evidence(cfg.name)
    fine_nodes_eval = fine_upd / cfg.fine.n_controls
    l2_alg = fine_nodes_eval * BYTES_PER_NODE[dtype] / fine_s / 1e9 if fine_s else 0.0
    roofline = {"bound": "alu", "achieved": achieved, "peak": peak_fma, "unit": "TFMA/s",
                "frac": achieved / peak_fma,
                "traffic": ncu.get("dram_bytes_per_launch") if ncu else None,
                "kernel": "fine sweep (the partitioned solve's cooperative k_sweep_* launch): "
                          "evaluated node x control updates x 3 FMA / fine-solve device time",
                "peak_source": f"FMA pipes 148 SM x {FMA_LANES_PER_SM_CLK} lanes x "
                               f"{sm_mhz:.0f} MHz ({peak_kind} sm_max_mhz; DESIGN.md §6)",
                "fma_per_update": FMA_PER_UPDATE,
                "l2_algorithmic_gbs": l2_alg,
                "l2_algorithmic_note": f"{BYTES_PER_NODE[dtype]} B per evaluated node "
                                       "(read V^n, write V^{n+1}, class) / fine-solve time",
                "hbm_frac_algorithmic": l2_alg / float(peaks.get("hbm_gbs", 6650.0)),
                "ncu": ncu}

    cpu = None
    if world == 1 and not args.no_cpu_baseline:
        import oracle
        rows = sample_rows(cfg.fine, 2.0e8)
        rate, dt, interior, rr = oracle_rows_rate(cfg.fine, rows)
        cpu = {"value": rate, "unit": UNIT, "cores": oracle.threads(), "kind": "oracle",
               "sample": f"1 Jacobi application of the fp64 oracle operator to node rows "
                         f"[{rr[0]}, {rr[1]}) of the {list(cfg.fine.grid.n)} fine grid "
                         f"({interior} interior nodes x {cfg.fine.n_controls} controls, "
                         f"{dt:.1f} s)"}

    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": total_ms / args.steps, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": dtype, "data": "synthetic",
            "config": {"workload": cfg.name, "grid": list(cfg.fine.grid.n),
                       "coarse": list(cfg.coarse.grid.n), "controls": cfg.fine.n_controls,
                       "subdomains": cfg.m, "band": cfg.band, "tol": cfg.fine.tol,
                       "parallelism": f"sub-domains over {world} GPU(s), one MIN all-reduce",
                       "labeller": args.labeller,
                       "l2": "flushed (256 MiB write) between timed steps"},
            "value_note": "evaluated node x control updates: the brackets the kernels "
                          "computed (exactly skipped nodes, and control segments the "
                          "cooperative field kernel prunes by their exact corner bound, are "
                          "not counted) / time-to-solution",
            "time_to_solution_ms": total_ms / args.steps,
            "step_ms": [round(x, 3) for x in step_ms],
            "nominal_updates_per_s": nominal / (total_ms / 1e3),
            "fine_sweeps": mine["fine_sweeps"],
            "labels": labels,
            "per_rank": per_rank,
            "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": h2d,
                    "d2h_bytes_per_step": d2h, "ms_per_step": e2e_total / len(e2e_ms)},
            "gpu_launches": launches,
            "roofline": roofline,
            "cpu_baseline": cpu,
            "clocks": clocks.summary(),
            "stages_ms": res["timings"]}
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
