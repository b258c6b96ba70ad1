"""One whole ISA pass (coarse solve, labels, partitioned fine solve) of a config, with
stage times and per-sub-domain iteration counts: python tools/prof_isa.py CONFIG [REPS]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import hj_workloads as W  # noqa: E402
from paper_1405_3521_b200 import hj, pipeline  # noqa: E402

args = [a for a in sys.argv[1:] if not a.startswith("--")]
idx = int(args[0]) if len(args) > 0 else 2
reps = int(args[1]) if len(args) > 1 else 1
exit_set = "--no-exit" not in sys.argv
cfg = W.make(idx)
fine = hj.DeviceProblem(cfg.fine, cfg.dtype)
coarse = hj.DeviceProblem(cfg.coarse, cfg.dtype)
for r in range(reps):
    t0 = time.perf_counter()
    res = pipeline.run_isa(cfg, cfg.dtype, fine=fine, coarse=coarse, exit_set=exit_set)
    torch.cuda.synchronize()
    reps_ = [x for x in res["reports"] if x]
    print(f"config {idx}: wall {1e3 * (time.perf_counter() - t0):.1f} ms  stages "
          f"{ {k: round(v, 2) for k, v in res['timings'].items()} }  sweeps per sub-domain "
          f"{[x['iterations'] for x in reps_]}  box nodes {[p.box_nodes for p in res['plan']][:8]}...  "
          f"evaluated {sum(x['evaluated_updates'] for x in reps_):.3e}", flush=True)
    lab = res["labels"]
    if lab.get("label") is not None:
        n = res["n_sets"]
        bits = res["mask"]
        cover = [int(((bits >> k) & 1).sum()) for k in range(n)]
        print(f"  sets {n}, labels -1: {int((lab['label'] == -1).sum())}, exit set (-2): "
              f"{int((lab['label'] == -2).sum())}, sum|S_k|/N = {sum(cover) / fine.N:.3f}, "
              f"sum box/N = {sum(p.box_nodes for p in res['plan']) / fine.N:.3f}", flush=True)
    if "--shares" in sys.argv:
        # per-set work actually done (evaluated updates) and the LPT split over 2/4/8 ranks
        # (hj_assign_subdomains' own assignment): the largest rank's share of the work bounds
        # the partitioned solve's parallel efficiency
        work = [x["evaluated_updates"] if x else 0 for x in res["reports"]]
        tot = float(sum(work))
        print("  per set: " + ", ".join(f"{k}:{x['iterations']}sw/{p.n_nodes / fine.N:.3f}N/"
                                         f"{w / tot:.3f}" for k, (x, p, w) in
                                         enumerate(zip(res["reports"], res["plan"], work)) if x))
        for world in (2, 4, 8):
            owners = hj.hj_assign_subdomains(res["plan"], world)
            per = [sum(w for w, o in zip(work, owners) if o == r) for r in range(world)]
            print(f"  world {world}: rank work shares {[round(p / tot, 3) for p in per]}; "
                  f"max-rank bound on efficiency {tot / (world * max(per)):.3f}", flush=True)
