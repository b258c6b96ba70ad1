"""Whole-grid hj_solve of one config's fine (or coarse) problem, for ncu captures
and quick timings: python tools/prof_solve.py CONFIG [DTYPE] [KERNEL] [fine|coarse] [REPS] [MAX_ITER]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import hj_workloads as W  # noqa: E402
from paper_1405_3521_b200 import hj  # noqa: E402

a = sys.argv[1:] + [None] * 6
idx = int(a[0] or 2)
cfg = W.make(idx)
dtype = a[1] or cfg.dtype
kernel = a[2] or "auto"
which = a[3] or "fine"
reps = int(a[4] or 1)
prob = getattr(cfg, which)
max_iter = int(a[5]) if a[5] else prob.max_iter
dp = hj.DeviceProblem(prob, dtype, sweep_kernel=kernel)
for r in range(reps):
    t0 = time.perf_counter()
    V, rep = hj.hj_solve(dp, max_iter=max_iter, allow_not_converged=True)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    print(f"config {idx} {which} {dtype} {kernel}: iters={rep['iterations']} conv={rep['converged']} "
          f"device_ms={rep['device_ms']:.2f} wall_ms={1e3 * dt:.1f} launches={rep['launches']} "
          f"evaluated={rep['evaluated_updates']:.3e} nominal={rep['node_updates']:.3e} "
          f"eval_rate={rep['evaluated_updates'] / max(rep['device_ms'], 1e-9) * 1e3:.3e}/s",
          flush=True)
