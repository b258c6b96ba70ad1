"""Multi-rank host logic on CPU (gloo, world size 2): sub-domain assignment, per-rank
solve sets and the MIN gather reproduce the single-process ISA assembly.  The
per-sub-domain solves here are the oracle's (CPU); the GPU path runs the same
sequence through libhj.so (pipeline.run_isa)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import hj_workloads as W
import oracle


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _plan_like(mask, m):
    from paper_1405_3521_b200 import hj
    plan = (hj.hj_subdomain * m)()
    for k in range(m):
        nodes = int(((mask >> k) & 1).sum())
        plan[k].n_nodes = nodes
        plan[k].work = float(nodes) * (1.0 + k)   # uneven on purpose
    return plan


def _worker(rank, world, port, cfg_args, ret):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_1405_3521_b200 import hj, pipeline
    cfg = W.make(*cfg_args)
    oc = oracle.OracleProblem(cfg.coarse)
    Vc, _, _ = oc.solve()
    lab, _, _, _ = oc.label(Vc, np.arange(oc.N), cfg.n_max_steps)
    mask = oracle.prolong(cfg.coarse.grid, cfg.fine.grid, cfg.ratio, cfg.band, lab, cfg.m,
                          cfg.fine.piece)
    owners = hj.hj_assign_subdomains(_plan_like(mask, cfg.m), world)
    mine = pipeline.solve_set_for_rank(owners, rank)
    of = oracle.OracleProblem(cfg.fine)
    Vk = []
    for k in range(cfg.m):
        if (mine >> k) & 1:
            Vk.append(of.solve_subdomain(mask, k)[0])
        else:
            Vk.append(np.full(of.N, cfg.fine.v_out))
    owned_mask = np.where(((mask[:, None] >> np.arange(cfg.m, dtype=np.uint64)) & np.uint64(1)).astype(bool) &
                          np.array([(mine >> k) & 1 for k in range(cfg.m)], bool)[None, :],
                          1, 0)
    bits = (owned_mask * (1 << np.arange(cfg.m))).sum(axis=1).astype(np.uint64)
    local = oracle.assemble(bits, Vk, cfg.fine.v_out)
    t = torch.from_numpy(local.copy())
    pipeline.gather_min(t)
    ret[rank] = (t.numpy(), owners, mine)
    dist.destroy_process_group()


def test_two_ranks_min_gather_reproduces_single_process():
    cfg_args = (1,)
    port = _free_port()
    mgr = mp.Manager()
    ret = mgr.dict()
    mp.spawn(_worker, args=(2, port, cfg_args, ret), nprocs=2, join=True)
    V0, owners, mine0 = ret[0]
    V1, _, mine1 = ret[1]
    assert np.array_equal(V0, V1)
    assert mine0 & mine1 == 0 and (mine0 | mine1) == (1 << 4) - 1   # a partition of the set
    assert set(owners) == {0, 1}
    cfg = W.make(*cfg_args)
    full = oracle.isa(cfg.fine, cfg.coarse, cfg.ratio, cfg.band, cfg.m, cfg.n_max_steps,
                      exit_set=False)
    assert np.array_equal(V0, full["Vbar"])
