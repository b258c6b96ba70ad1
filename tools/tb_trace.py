"""Per-CTA timeline of one temporally blocked sweep launch (hj_debug_set_trace):
python tools/tb_trace.py [CONFIG] [MAX_ITER] — the trace holds the last launch."""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import hj_workloads as W  # noqa: E402
from paper_1405_3521_b200 import hj  # noqa: E402

idx = int(sys.argv[1]) if len(sys.argv) > 1 else 2
max_iter = int(sys.argv[2]) if len(sys.argv) > 2 else 400
kernel = sys.argv[3] if len(sys.argv) > 3 else "local_tb"
cfg = W.make(idx)
dp = hj.DeviceProblem(cfg.fine, "f32", sweep_kernel=kernel)
cap = 1 << 16
buf = torch.zeros(8 * cap, dtype=torch.int64, device="cuda")
L = hj.lib()
L.hj_debug_set_trace.argtypes = [ctypes.c_void_p, ctypes.c_longlong, ctypes.c_longlong]
hj.hj_solve(dp, max_iter=max_iter, allow_not_converged=True)      # warm
L.hj_debug_set_trace(buf.data_ptr(), cap, ((max_iter - 1) // 8) * 8)
V, rep = hj.hj_solve(dp, max_iter=max_iter, allow_not_converged=True)
torch.cuda.synchronize()
L.hj_debug_set_trace(None, 0, 0)
t = buf.view(-1, 8).cpu().numpy()
t = t[t[:, 1] > 0]
t0 = t[:, 1].min()
start, end, work, sm = (t[:, 1] - t0) / 1e3, (t[:, 2] - t0) / 1e3, t[:, 3], t[:, 0]
act = t[:, 2] > 0
print(f"CTAs traced {len(t)}  active {act.sum()}  span {end.max():.1f} us")
d = end[act] - start[act]
print(f"active CTA duration us: min {d.min():.1f} med {np.median(d):.1f} max {d.max():.1f}")
print(f"active start us: min {start[act].min():.1f} med {np.median(start[act]):.1f} max {start[act].max():.1f}")
ph = t[:, 4:8].astype(float) / 1965.0   # cycles -> us at max clock
heavy = np.argsort(-(t[:, 2] - t[:, 1]))[:10]
print("phase us (stage, scan, pairs, tail) heaviest:", [tuple(np.round(ph[i], 1)) for i in heavy])
print("phase us mean:", np.round(ph[act].mean(0), 1))
print("listed nodes (sum over sub-sweeps) of active CTAs: min %d med %d max %d" % (
    work[act].min(), np.median(work[act]), work[act].max()))
order = np.argsort(-d)[:8]
print("longest CTAs (dur us, listed, start us, sm):",
      [(round(float(d[i]), 1), int(work[act][i]), round(float(start[act][i]), 1), int(sm[act][i])) for i in order])
per_sm = np.bincount(sm[act].astype(int), minlength=148)
print("active CTAs per SM histogram:", np.bincount(per_sm))
wsm = np.bincount(sm[act].astype(int), weights=work[act], minlength=148)
print(f"owned node-updates per SM: mean {wsm.mean():.0f} max {wsm.max():.0f}")
busy = np.zeros(148)
for s_, a, b_ in zip(sm[act].astype(int), start[act], end[act]):
    busy[s_] = max(busy[s_], b_)
print(f"per-SM last active end us: min {busy.min():.1f} med {np.median(busy):.1f} max {busy.max():.1f}")
