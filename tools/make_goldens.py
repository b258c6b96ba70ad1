#!/usr/bin/env python
"""Write the full-size fp64 goldens the GPU parity tests compare against.

Calls ONLY oracle/ (and the seeded generators in hj_workloads): for each requested
BASELINE config, the whole ISA pass of the oracle from scratch — coarse value
iteration, trajectory labels, prolongation with the band, the masked sub-domain
solves and the min assembly (§4 ISA, line 389-408; north_star labelling) —
and stores the assembled fine field Vbar (all nodes, or a seeded sample of nodes for
grids too large to commit whole), the coarse labels with their margins, and the
iteration counts.

    OMP_NUM_THREADS=8 python tools/make_goldens.py 2 [4 ...]

Output: tests/golden/c{idx}_isa.npz  (+ a line per config in tests/golden/README.md)
"""
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import hj_workloads as W  # noqa: E402
import oracle  # noqa: E402

MAX_STORED = 1 << 20     # nodes of Vbar stored per golden (a seeded sample above this)


def sample_nodes(N, seed=1405):
    if N <= MAX_STORED:
        return None
    rng = np.random.default_rng(seed)
    return np.sort(rng.choice(N, MAX_STORED, replace=False))


def main(idxs):
    for idx in idxs:
        cfg = W.make(idx)
        t0 = time.time()
        res = oracle.isa(cfg.fine, cfg.coarse, cfg.ratio, cfg.band, cfg.m, cfg.n_max_steps)
        dt = time.time() - t0
        N = cfg.fine.grid.size
        pick = sample_nodes(N)
        Vbar = res["Vbar"] if pick is None else res["Vbar"][pick]
        out = os.path.join(ROOT, "tests", "golden", f"c{idx}_isa.npz")
        np.savez_compressed(out, Vbar=Vbar, nodes=np.array([] if pick is None else pick, np.int64),
                            sampled=np.array(pick is not None), labels=res["labels"],
                            label_margin=res["label_margin"], label_geo=res["label_geo"],
                            label_steps=res["label_steps"], Vc=res["Vc"],
                            iters=np.array(res["iters"]), coarse_iters=np.array(res["coarse_iters"]),
                            threads=np.array(oracle.threads()), seconds=np.array(dt))
        line = (f"- `c{idx}_isa.npz`: {cfg.name}, oracle.isa() from scratch in {dt:.0f} s on "
                f"{oracle.threads()} threads; Vbar at {'all' if pick is None else len(pick)} of "
                f"{N} nodes; sub-domain iterations {list(res['iters'])}\n")
        with open(os.path.join(ROOT, "tests", "golden", "README.md"), "a") as f:
            f.write(line)
        print(line, end="", flush=True)


if __name__ == "__main__":
    main([int(a) for a in sys.argv[1:]] or [2])
