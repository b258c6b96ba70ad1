"""Label statistics of a config's coarse trajectories and sub-domain coverage:
python tools/diag_labels.py CONFIG"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import hj_workloads as W  # noqa: E402
from paper_1405_3521_b200 import hj  # noqa: E402

idx = int(sys.argv[1]) if len(sys.argv) > 1 else 5
cfg = W.make(idx)
coarse = hj.DeviceProblem(cfg.coarse, cfg.dtype)
fine = hj.DeviceProblem(cfg.fine, cfg.dtype)
Vc, rep = hj.hj_solve(coarse)
out = hj.hj_label_subdomains(coarse, Vc, cfg.n_max_steps, fine, cfg.ratio, cfg.band, cfg.m)
lab = out["label"].cpu().numpy()
steps = out["steps"].cpu().numpy()
print(f"config {idx}: coarse {cfg.coarse.grid.n}, n_max {cfg.n_max_steps}, coarse iters {rep['iterations']}")
print("labels histogram (-1 first):", np.bincount(lab + 1, minlength=cfg.m + 1).tolist())
print("steps of -1 nodes: max", steps[lab < 0].max() if (lab < 0).any() else None,
      " ==n_max:", int((steps[lab < 0] >= cfg.n_max_steps).sum()))
mask = out["mask"].cpu().numpy().view(np.uint32)
cov = [(int(((mask >> k) & 1).sum())) for k in range(cfg.m)]
print("fine nodes per sub-domain / grid:", [round(c / mask.size, 3) for c in cov])
