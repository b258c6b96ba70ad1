"""Repeat a partitioned ISA pass and report bitwise differences (debugging aid):
python tools/determinism.py CONFIG SCALE KERNEL [REPS]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import hj_workloads as W  # noqa: E402
from paper_1405_3521_b200 import hj, pipeline  # noqa: E402

idx, sc, kernel = int(sys.argv[1]), float(sys.argv[2]), sys.argv[3]
reps = int(sys.argv[4]) if len(sys.argv) > 4 else 3
cfg = W.make(idx, scale=sc)
fine = hj.DeviceProblem(cfg.fine, cfg.dtype, sweep_kernel=kernel)
ref = None
for r in range(reps):
    res = pipeline.run_isa(cfg, cfg.dtype, fine=fine)
    torch.cuda.synchronize()
    V, its = res["V"].double().clone(), [x["iterations"] for x in res["reports"] if x]
    if ref is None:
        ref = (V, its)
        print(f"config {idx} scale {sc} {kernel} list={os.environ.get('HJ_COOP_LIST', 'auto')}: sweeps {its}")
    else:
        d = (V - ref[0]).abs()
        print(f"  rep {r}: max diff {float(d.max()):.3e} n diff {int((d > 0).sum())} same sweeps {its == ref[1]}")
