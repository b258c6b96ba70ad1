"""How many nodes change per sweep (and how many a node-level dirty test would
evaluate) vs how many the tile-level skip evaluates.  Config 2 fine, fp32."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import torch.nn.functional as F  # noqa: E402

import hj_workloads as W  # noqa: E402
from paper_1405_3521_b200 import hj  # noqa: E402

idx = int(sys.argv[1]) if len(sys.argv) > 1 else 2
cfg = W.make(idx)
p = cfg.fine
n = p.grid.n
dp = hj.DeviceProblem(p, "f32", sweep_kernel="local_packed")
_, full = hj.hj_solve(dp)
N = full["iterations"]
interior = int((torch.as_tensor(p.piece) < 0).sum())
tot_changed = tot_dirty = tot_tile = 0
for k in list(range(1, N, max(1, N // 40))):
    Va, _ = hj.hj_solve(dp, max_iter=k, allow_not_converged=True)
    Vb, _ = hj.hj_solve(dp, max_iter=k + 1, allow_not_converged=True)
    Vc, _ = hj.hj_solve(dp, max_iter=k + 2, allow_not_converged=True)
    ch1 = (Va != Vb).view(n[1], n[0]).float()           # changed in sweep k+1
    ch2 = (Vb != Vc).view(n[1], n[0]).float()           # changed in sweep k+2
    dirty = F.max_pool2d(ch1[None, None], 3, 1, 1)[0, 0]   # candidates for sweep k+2
    t32 = F.max_pool2d(ch1[None, None], 32, 32, ceil_mode=True)[0, 0]
    tiles = F.max_pool2d(t32[None, None], 3, 1, 1)[0, 0]   # tile-level active set
    print(f"sweep {k + 2}: changed {int(ch2.sum())}  node-dirty {int(dirty.sum())}  "
          f"tile-active nodes {int(tiles.sum()) * 1024}", flush=True)
