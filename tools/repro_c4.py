"""Config 4 ISA pass at a few scales (debugging aid): python tools/repro_c4.py [SCALES...]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import hj_workloads as W  # noqa: E402
from paper_1405_3521_b200 import pipeline  # noqa: E402

for sc in [float(a) for a in sys.argv[1:]] or [0.25, 0.5, 1.0]:
    cfg = W.make(4, scale=sc)
    try:
        res = pipeline.run_isa(cfg, cfg.dtype)
        torch.cuda.synchronize()
        print("scale", sc, cfg.fine.grid.n, "ok", {k: round(v, 2) for k, v in res["timings"].items()},
              flush=True)
    except Exception as e:      # noqa: BLE001
        print("scale", sc, cfg.fine.grid.n, "FAILED", str(e)[:200], flush=True)
        break
