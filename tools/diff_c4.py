"""Config 4 partitioned ISA: dubins vs dubins_coop (debugging aid): python tools/diff_c4.py SCALE"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import hj_workloads as W  # noqa: E402
from paper_1405_3521_b200 import hj, pipeline  # noqa: E402

sc = float(sys.argv[1]) if len(sys.argv) > 1 else 0.5
cfg = W.make(4, scale=sc)
out = {}
for kernel in ("dubins", "dubins_coop", "dubins_coop"):
    fine = hj.DeviceProblem(cfg.fine, cfg.dtype, sweep_kernel=kernel)
    res = pipeline.run_isa(cfg, cfg.dtype, fine=fine)
    torch.cuda.synchronize()
    its = [r["iterations"] for r in res["reports"] if r]
    V = res["V"].double()
    if kernel in out:
        d = (V - out[kernel][0]).abs()
        print("repeat", kernel, "max diff", float(d.max()), "n diff", int((d > 0).sum()), its == out[kernel][1])
    else:
        out[kernel] = (V, its)
    print(kernel, its)
d = (out["dubins"][0] - out["dubins_coop"][0]).abs()
print("dubins vs coop: max diff", float(d.max()), "n diff", int((d > 0).sum()), "of", d.numel())
