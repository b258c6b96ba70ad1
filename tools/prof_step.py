"""One bench step (config 2 by default) for ncu captures: warm-up pass, then the
profiled pass.  Usage: python tools/prof_step.py [config] [dtype]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import hj_workloads as W  # noqa: E402
from paper_1405_3521_b200 import hj, pipeline  # noqa: E402

idx = int(sys.argv[1]) if len(sys.argv) > 1 else 2
cfg = W.make(idx)
dtype = sys.argv[2] if len(sys.argv) > 2 else cfg.dtype
fine = hj.DeviceProblem(cfg.fine, dtype)
coarse = hj.DeviceProblem(cfg.coarse, dtype)
for _ in range(2):
    res = pipeline.run_isa(cfg, dtype, fine=fine, coarse=coarse)
torch.cuda.synchronize()
print({k: round(v, 3) for k, v in res["timings"].items()},
      "fine sweeps", max(r["iterations"] for r in res["reports"] if r))
