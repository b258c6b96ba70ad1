"""The whole hot path as one call: coarse pre-solve -> coarse feedback labels ->
prolongation -> partitioned fine solves -> min assembly (§4 ISA, with the
north_star's trajectory labelling), optionally sharded over ranks.

Every step is a libhj.so entry point; this module only sequences them and, for
N > 1 ranks, does the one collective the method has: the final element-wise MIN
of the ranks' assembled fields (NCCL through torch.distributed).
"""
from __future__ import annotations

import time

import torch

from . import hj


def solve_set_for_rank(owners, rank):
    bits = 0
    for k, r in enumerate(owners):
        if r == rank:
            bits |= 1 << k
    return bits


def gather_min(V, group=None):
    """The method's only collective: element-wise MIN of the ranks' assembled fields
    (each rank holds v_out where it owns no sub-domain, and every value is <= v_out)."""
    torch.distributed.all_reduce(V, op=torch.distributed.ReduceOp.MIN, group=group)
    return V


EXIT_TOL_FACTOR = 10.0   # exit test threshold = 10 x the coarse solve's tolerance (R9b)


def exit_problem(coarse):
    """The coarse problem with no target node (every piece -1): its solution Vexit is the
    value when the box exit (cost v_out) is the only way the cost ends (reading R9b).
    Cached on the DeviceProblem."""
    dp = getattr(coarse, "_exit_dp", None)
    if dp is None:
        piece = torch.full_like(coarse.piece, -1)
        dp = hj.DeviceProblem(coarse.prob, coarse.dtype, coarse.device, piece=piece,
                              speed=coarse.speed, g=coarse.g, reuse_buffers=coarse.reuse)
        coarse._exit_dp = dp
    return dp


def run_isa(cfg, dtype="f32", device="cuda", rank=0, world=1, group=None, fine=None, coarse=None,
            gather=True, labeller="trajectory", ra_params=(1.0, 1.0, 0.5), exit_set=True):
    """Returns dict(V=assembled fine field (on every rank after the MIN all-reduce when
    gather), labels, mask, n_sets, plan, owners, reports, timings).  exit_set: the box
    boundary is a piece of its own (R9b) — unlabelled coarse nodes whose value needs no
    target form the set n_sets - 1 instead of joining every piece's set."""
    t = {}
    fine = fine or hj.DeviceProblem(cfg.fine, dtype, device)
    coarse = coarse or hj.DeviceProblem(cfg.coarse, dtype, device)
    s = torch.cuda.current_stream()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(5)]
    ev[0].record(s)
    if labeller == "ra":   # the paper's RA: auxiliary solves + threshold
        C, M, q = ra_params
        ra = hj.hj_ra_subdomains(coarse, cfg.m, C, M, q, fine=fine, ratio=cfg.ratio,
                                 band=cfg.band)
        Vc, rep_c = ra["Vmin"], dict(ra["reports"][0])
        for key in ("node_updates", "evaluated_updates", "launches"):
            rep_c[key] = sum(r[key] for r in ra["reports"])
        ev[1].record(s)
        lab = dict(label=None, mask=ra["mask"], coarse_mask=ra["coarse_mask"], Vaux=ra["Vaux"],
                   n_sets=cfg.m)
    else:
        Vc, rep_c = hj.hj_solve(coarse)
        Vexit = None
        if exit_set:
            ex = exit_problem(coarse)
            Vexit, rep_e = hj.hj_solve(ex, V=hj._buf(coarse, "Vexit", coarse.N,
                                                     hj._torch_dtype(coarse.dtype)))
            rep_c = dict(rep_c)
            for key in ("node_updates", "evaluated_updates", "launches"):
                rep_c[key] += rep_e[key]
        ev[1].record(s)
        lab = hj.hj_label_subdomains(coarse, Vc, cfg.n_max_steps, fine, cfg.ratio, cfg.band,
                                     cfg.m, Vexit=Vexit,
                                     exit_tol=EXIT_TOL_FACTOR * cfg.coarse.tol)
    ev[2].record(s)
    n_sets = lab["n_sets"]
    plan, ws = hj.hj_partition_plan(fine, lab["mask"], n_sets)
    owners = hj.hj_assign_subdomains(plan, world)
    solve_set = solve_set_for_rank(owners, rank)
    Vbar, reps = hj.hj_solve_partitioned(fine, lab["mask"], n_sets, plan, ws, solve_set=solve_set)
    ev[3].record(s)
    if world > 1 and gather:
        gather_min(Vbar, group)
    ev[4].record(s)
    torch.cuda.synchronize()
    t["coarse_ms"] = ev[0].elapsed_time(ev[1])
    t["label_ms"] = ev[1].elapsed_time(ev[2])
    t["fine_ms"] = ev[2].elapsed_time(ev[3])
    t["gather_ms"] = ev[3].elapsed_time(ev[4])
    return dict(V=Vbar, Vc=Vc, coarse_report=rep_c, labels=lab, mask=lab["mask"], n_sets=n_sets,
                plan=plan,
                owners=owners, solve_set=solve_set, reports=reps, timings=t)
