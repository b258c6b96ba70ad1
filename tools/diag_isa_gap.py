#!/usr/bin/env python
"""Where does the ISA result exceed the whole-grid solution?  (usage:
python tools/diag_isa_gap.py IDX [SCALE] [exit|noexit] [BAND])

Runs the whole-grid GPU solve and the ISA pass of a config, and for the fine nodes with
Vbar - V > 1e-3 prints their number, position, set membership (which sets, exit bit),
the coarse labels around them, and the coarse values Vc / Vexit there."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import hj_workloads as W  # noqa: E402
from paper_1405_3521_b200 import hj, pipeline  # noqa: E402

idx = int(sys.argv[1])
scale = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
exit_set = (sys.argv[3] if len(sys.argv) > 3 else "exit") == "exit"
cfg = W.make(idx, scale=scale)
if len(sys.argv) > 4:
    cfg.band = int(sys.argv[4])
g = cfg.fine.grid
n0, n1 = g.n[0], g.n[1]
fine = hj.DeviceProblem(cfg.fine, cfg.dtype)
V, rep = hj.hj_solve(fine)
Vw = V.double().cpu().numpy()
del V
res = pipeline.run_isa(cfg, cfg.dtype, fine=fine, exit_set=exit_set)
Vbar = res["V"].double().cpu().numpy()
mask = res["mask"].cpu().numpy().view(np.uint64)
lab = res["labels"]["label"].cpu().numpy()
Vc = res["Vc"].double().cpu().numpy()
n_sets = res["n_sets"]
cover = 0
for c0 in range(0, len(mask), 1 << 24):
    cover += int(np.unpackbits(mask[c0:c0 + (1 << 24)].view(np.uint8)).sum())
print(f"band {cfg.band}: sum|S_k|/N = {cover / len(mask):.3f}; ISA stages (ms) "
      f"{ {k: round(v, 1) for k, v in res['timings'].items()} }")
print(f"config {idx} scale {scale} fine {g.n} exit_set {exit_set} sets {n_sets} whole sweeps "
      f"{rep['iterations']} set sweeps {[r['iterations'] for r in res['reports']]}")
diff = Vbar - Vw
bad = np.nonzero(diff > 1e-3)[0]
print(f"diff range [{diff.min():.3e}, {diff.max():.3e}]; nodes > 1e-3: {len(bad)} "
      f"({100 * len(bad) / len(diff):.3f} %); > 1e-5: {(np.abs(diff) > 1e-5).sum()}")
if len(bad):
    i, j = bad % n0, bad // n0
    x = g.lo[0] + i * g.spacing(0)
    y = g.lo[1] + j * g.spacing(1)
    print(f"bad x in [{x.min():.3f}, {x.max():.3f}], y in [{y.min():.3f}, {y.max():.3f}]")
    print("x histogram", np.histogram(x, bins=8, range=(g.lo[0], g.hi[0]))[0])
    print("y histogram", np.histogram(y, bins=8, range=(g.lo[1], g.hi[1]))[0])
    mb = mask[bad]
    pop = np.array([bin(int(m)).count("1") for m in mb[:20000]])
    print("sets per bad node (first 20000):", np.bincount(pop)[:40])
    if n_sets > cfg.m:
        ex = (mb >> np.uint64(cfg.m)) & np.uint64(1)
        print(f"exit bit set at {int(ex.sum())} of {len(bad)}; exit-only at "
              f"{int((mb == (np.uint64(1) << np.uint64(cfg.m))).sum())}")
    cg = cfg.coarse.grid
    r0, r1 = cfg.ratio
    ci, cj = np.rint(i / r0).astype(int), np.rint(j / r1).astype(int)
    cl = lab[ci + cg.n[0] * cj]
    u, c = np.unique(cl, return_counts=True)
    print("nearest coarse label of bad nodes:", dict(zip(u.tolist(), c.tolist())))
    print("coarse label histogram (all):", dict(zip(*[a.tolist() for a in np.unique(lab, return_counts=True)])))
    pick = bad[np.argsort(-diff[bad])[:12]]
    for p in pick:
        pi, pj = p % n0, p // n0
        cc = int(round(pi / r0)) + cg.n[0] * int(round(pj / r1))
        print(f"  node ({pi},{pj}) x=({g.lo[0] + pi * g.spacing(0):.4f},{g.lo[1] + pj * g.spacing(1):.4f}) "
              f"Vw {Vw[p]:.4f} Vbar {Vbar[p]:.4f} mask {int(mask[p]):#x} coarse label {lab[cc]} Vc {Vc[cc]:.4f}")
