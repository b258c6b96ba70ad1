"""The N > 1 path of the partitioned solve on the GPU (one device here):
sub-domains assigned to ranks by hj_assign_subdomains, each rank solving only its own set
(solve_set) and holding v_out elsewhere, then the one collective, the element-wise MIN.
The result must reproduce the single-rank ISA pass bit for bit."""
import os
import socket

import numpy as np
import pytest

import hj_workloads as W

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover - CPU container
    pytest.skip("needs a CUDA device", allow_module_level=True)

import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402

from paper_1405_3521_b200 import pipeline  # noqa: E402

SMALL = {2: (128 / 1024, 2), 3: (96 / 4096, 2), 5: (128 / 16384, 4)}


def _cfg(idx):
    s, r = SMALL[idx]
    return W.make(idx, scale=s, ratio=r)


@pytest.mark.parametrize("idx", [2, 3, 5])
@pytest.mark.parametrize("world", [2, 3, 8])
def test_rank_shares_min_reproduce_single_rank(idx, world):
    """Every rank's share computed in turn on one device, combined by torch.minimum (the
    MIN all-reduce's arithmetic): bit-identical to world = 1; the shares partition the
    sub-domains."""
    cfg = _cfg(idx)
    r1 = pipeline.run_isa(cfg, cfg.dtype)
    ref, n_sets = r1["V"].clone(), r1["n_sets"]
    acc, sets = None, []
    for r in range(world):
        out = pipeline.run_isa(cfg, cfg.dtype, rank=r, world=world, gather=False)
        sets.append(out["solve_set"])
        acc = out["V"].clone() if acc is None else torch.minimum(acc, out["V"])
    assert torch.equal(acc, ref)
    u = 0
    for s in sets:
        assert s & u == 0
        u |= s
    assert u == (1 << n_sets) - 1


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, idx, ret):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    cfg = _cfg(idx)
    # the ranks share one device: they take turns for the solves (no two processes'
    # cooperative grids on one GPU at once), then meet in the real collective
    out = None
    for turn in range(world):
        if turn == rank:
            out = pipeline.run_isa(cfg, cfg.dtype, rank=rank, world=world, gather=False)
            torch.cuda.synchronize()
        dist.barrier()
    V = out["V"].clone()
    pipeline.gather_min(V)            # all_reduce(MIN) on the CUDA tensor (gloo)
    torch.cuda.synchronize()
    ret[rank] = (V.cpu().numpy(), out["solve_set"])
    dist.destroy_process_group()


@pytest.mark.timeout(600)
def test_two_processes_gloo_min_allreduce_on_cuda_tensors():
    idx = 2
    cfg = _cfg(idx)
    r1 = pipeline.run_isa(cfg, cfg.dtype)
    ref, n_sets = r1["V"].cpu().numpy(), r1["n_sets"]
    mgr = mp.Manager()
    ret = mgr.dict()
    mp.spawn(_worker, args=(2, _port(), idx, ret), nprocs=2, join=True)
    V0, s0 = ret[0]
    V1, s1 = ret[1]
    assert np.array_equal(V0, V1) and np.array_equal(V0, ref)
    assert s0 & s1 == 0 and (s0 | s1) == (1 << n_sets) - 1
