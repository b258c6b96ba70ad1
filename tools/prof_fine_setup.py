"""Where the partitioned fine solve's time goes outside the cooperative kernel:
python tools/prof_fine_setup.py [CONFIG] — event-timed plan / solve of one ISA pass."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import hj_workloads as W  # noqa: E402
from paper_1405_3521_b200 import hj  # noqa: E402

idx = int(sys.argv[1]) if len(sys.argv) > 1 else 2
cfg = W.make(idx)
fine = hj.DeviceProblem(cfg.fine, cfg.dtype, reuse_buffers=True)
coarse = hj.DeviceProblem(cfg.coarse, cfg.dtype, reuse_buffers=True)
for rep in range(4):
    s = torch.cuda.current_stream()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
    Vc, _ = hj.hj_solve(coarse)
    lab = hj.hj_label_subdomains(coarse, Vc, cfg.n_max_steps, fine, cfg.ratio, cfg.band, cfg.m)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    ev[0].record(s)
    plan, ws = hj.hj_partition_plan(fine, lab["mask"], cfg.m)
    ev[1].record(s)
    t1 = time.perf_counter()
    Vbar, reps = hj.hj_solve_partitioned(fine, lab["mask"], cfg.m, plan, ws)
    ev[2].record(s)
    t2 = time.perf_counter()
    torch.cuda.synchronize()
    print(f"plan {ev[0].elapsed_time(ev[1]):.3f} ms (host {1e3 * (t1 - t0):.3f})  "
          f"solve {ev[1].elapsed_time(ev[2]):.3f} ms (host {1e3 * (t2 - t1):.3f})  "
          f"device_ms of the sweeps {max(r['device_ms'] for r in reps if r):.3f}")
