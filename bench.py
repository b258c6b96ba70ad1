#!/usr/bin/env python
"""Benchmark of the hot path (BASELINE.json metric): grid-node x control updates per
second of the semi-Lagrangian value-iteration sweeps, and time-to-solution of one
pass of the whole path (coarse pre-solve -> trajectory labels -> prolongation ->
partitioned fine solves -> min assembly).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config 2] [--impl reference]

One process per GPU (torchrun for N > 1).  Prints ONE JSON line on rank 0.
Default workload: BASELINE configs[1] (1025^2 variable-speed eikonal, fp32).
Inputs are seeded and synthetic (hj_workloads); see DESIGN.md §6.
"""
from __future__ import annotations

import argparse
import json
import os
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
# Roofline of the fine sweep: the bracket of one node x control update is
# a bilinear form in the control's weights, so at least 3 fused multiply-adds (the
# difference form C0 + ax A1 + ay (A2 + ax A3)); the FMA pipes retire 128 FMA lanes per
# SM clock (FFMA2 packs two per issue slot but not per pipe cycle — measured).
FMA_PER_UPDATE = {2: 3, 3: 3}
FMA_LANES_PER_SM_CLK = 128


def load_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f), "measured"
    except OSError:
        return {"hbm_gbs": 6650.0, "sm_max_mhz": 1965.0}, "fallback"


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


def oracle_sweep_rate(prob, sweeps=1):
    """The oracle as it stands: Jacobi sweeps of its operator over the whole fine grid."""
    import oracle
    o = oracle.OracleProblem(prob)
    cls = o.classes()
    V = o.initial(cls)
    interior = int((cls == oracle.INTERIOR).sum())
    t0 = time.perf_counter()
    for _ in range(sweeps):
        V, _ = o.apply_T(V, cls)
    dt = time.perf_counter() - t0
    return interior * prob.n_controls * sweeps / dt, dt, interior


def run_reference(args, cfg, rank, world):
    """--impl reference: the oracle (this tier's reference arm) on host cores."""
    if rank != 0:
        return
    prob = cfg.fine
    for _ in range(args.warmup):
        oracle_sweep_rate(prob, 1)
    rates, times = [], []
    for _ in range(args.steps):
        r, dt, interior = oracle_sweep_rate(prob, 1)
        rates.append(r)
        times.append(dt)
    value = float(np.mean(rates))
    sample = (f"1 Jacobi sweep of the oracle operator over the full {prob.grid.n} fine grid "
              f"({interior} interior nodes x {prob.n_controls} controls) per step")
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT,
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": 1e3 * float(np.mean(times)), "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": cfg.name, "grid": list(prob.grid.n),
                       "controls": prob.n_controls, "l2": "inputs > L1; CPU run"},
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": 1, "kind": "oracle",
                             "sample": sample},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", type=int, default=2)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--dtype", default=None)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--labeller", default="trajectory", choices=["trajectory", "ra"],
                    help="sub-domain reconstruction: north_star trajectories or the paper's RA")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)

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
    step_ms, updates, fine_eval, sweep_ms, sweep_launches, launches = [], 0, 0, 0.0, 0, 0
    evaluated = 0
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
            u = rc["node_updates"] + sum(r["node_updates"] for r in fr)
            updates += u
            fine_eval += sum(r["evaluated_updates"] for r in fr)
            evaluated += rc["evaluated_updates"] + sum(r["evaluated_updates"] for r in fr)
            if fr:
                sweep_ms += fr[0]["device_ms"]
                sweep_launches += fr[0]["launches"] - len(fr) - 3
            # coarse solve + label/prolong (2) + plan (2) + partitioned solve
            launches += rc["launches"] + 2 + 2 + sum(r["launches"] for r in fr)
    total_ms = float(np.sum(step_ms))
    if world > 1:
        t = torch.tensor([total_ms, updates, evaluated], dtype=torch.float64, device="cuda")
        tmax = t.clone()
        dist.all_reduce(tmax, op=dist.ReduceOp.MAX)
        dist.all_reduce(t, op=dist.ReduceOp.SUM)
        total_ms, updates, evaluated = float(tmax[0]), float(t[1]), float(t[2])
    value = updates / (total_ms / 1e3)

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
    e2e_ms, e2e_updates = [], 0
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
        if it == 0:
            continue
        e2e_ms.append(e0.elapsed_time(e1))
        e2e_updates += res["coarse_report"]["node_updates"] + sum(
            r["node_updates"] for r in res["reports"] if r is not None)
    e2e_total = float(np.sum(e2e_ms))
    if world > 1:
        t = torch.tensor([e2e_total, e2e_updates], dtype=torch.float64, device="cuda")
        tmax = t.clone()
        dist.all_reduce(tmax, op=dist.ReduceOp.MAX)
        dist.all_reduce(t, op=dist.ReduceOp.SUM)
        e2e_total, e2e_updates = float(tmax[0]), float(t[1])
    e2e_value = e2e_updates / (e2e_total / 1e3)

    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return

    peaks, peak_kind = load_peaks()
    sm_mhz = float(peaks.get("sm_max_mhz", 1965.0))
    peak_fma = 148 * FMA_LANES_PER_SM_CLK * sm_mhz * 1e6 / 1e12   # T FMA/s
    dim = cfg.fine.grid.dim
    achieved = fine_eval * FMA_PER_UPDATE[dim] / (sweep_ms / 1e3) / 1e12 if sweep_ms else 0
    traffic = None
    tpath = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tpath):
        with open(tpath) as f:
            traffic = json.load(f).get(cfg.name)
    roofline = {"bound": "alu", "achieved": achieved, "peak": peak_fma, "unit": "TFMA/s",
                "frac": achieved / peak_fma, "traffic": traffic,
                "kernel": "fine sweep (k_sweep_*): evaluated node x control updates x 3 FMA "
                          "/ fine-solve device time",
                "avg_launch_us": 1e3 * sweep_ms / max(sweep_launches, 1),
                "peak_source": f"FMA pipes 148 SM x {FMA_LANES_PER_SM_CLK} lanes x "
                               f"{sm_mhz:.0f} MHz ({peak_kind} sm_max_mhz; DESIGN.md §6)",
                "fma_per_update": FMA_PER_UPDATE[dim]}

    cpu = None
    if world == 1 and not args.no_cpu_baseline:
        rate, dt, interior = oracle_sweep_rate(cfg.fine, 2)
        cpu = {"value": rate, "unit": UNIT, "cores": 1, "kind": "oracle",
               "sample": f"2 Jacobi sweeps of the fp64 oracle operator over the full "
                         f"{cfg.fine.grid.n} fine grid ({dt:.1f} s)"}

    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": total_ms / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": dtype, "data": "synthetic",
            "config": {"workload": cfg.name, "grid": list(cfg.fine.grid.n),
                       "coarse": list(cfg.coarse.grid.n), "controls": cfg.fine.n_controls,
                       "subdomains": cfg.m, "band": cfg.band, "tol": cfg.fine.tol,
                       "parallelism": f"subdomains over {world} GPU(s)",
                       "labeller": args.labeller,
                       "l2": "flushed (256 MiB write) between timed steps"},
            "time_to_solution_ms": total_ms / args.steps,
            "step_ms": [round(x, 3) for x in step_ms],
            "evaluated_updates_per_s": evaluated / (total_ms / 1e3),
            "fine_sweeps": max((r["iterations"] for r in res["reports"] if r), default=0),
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
