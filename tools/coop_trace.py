"""Per-sweep timeline of the cooperative local kernel (block 0's view) — needs a library
built with the trace compiled in: bash tools/build_variant.sh /tmp/libhj_tr.so -DHJ_COOP_TRACE=1,
then HJ_LIB_PATH=/tmp/libhj_tr.so;
python tools/coop_trace.py [CONFIG] — items, block-0 item phase, barrier wait, per sweep."""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import hj_workloads as W  # noqa: E402
from paper_1405_3521_b200 import hj  # noqa: E402

idx = int(sys.argv[1]) if len(sys.argv) > 1 else 2
isa = len(sys.argv) > 2 and sys.argv[2] == "isa"
coarse = len(sys.argv) > 2 and sys.argv[2] == "coarse"
cfg = W.make(idx)
dp = hj.DeviceProblem(cfg.coarse if coarse else cfg.fine, "f32",
                      sweep_kernel=os.environ.get("HJ_TRACE_KERNEL", "auto"))
cap = 1 << 12
buf = torch.zeros((8 + 256) * cap + 16, dtype=torch.int64, device="cuda")
L = hj.lib()
L.hj_debug_set_trace.argtypes = [ctypes.c_void_p, ctypes.c_longlong, ctypes.c_longlong]
if isa:      # trace the partitioned fine solve of one ISA pass (the last cooperative launch)
    from paper_1405_3521_b200 import pipeline
    fine = hj.DeviceProblem(cfg.fine, cfg.dtype, reuse_buffers=True)
    coarse = hj.DeviceProblem(cfg.coarse, cfg.dtype, reuse_buffers=True)
    pipeline.run_isa(cfg, cfg.dtype, fine=fine, coarse=coarse)
    L.hj_debug_set_trace(buf.data_ptr(), cap, -1)
    res = pipeline.run_isa(cfg, cfg.dtype, fine=fine, coarse=coarse)
    torch.cuda.synchronize()
    L.hj_debug_set_trace(None, 0, 0)
    rep = dict(iterations=max(r["iterations"] for r in res["reports"] if r),
               device_ms=res["reports"][0]["device_ms"])
else:
    hj.hj_solve(dp)
    L.hj_debug_set_trace(buf.data_ptr(), cap, -1)
    V, rep = hj.hj_solve(dp)
    torch.cuda.synchronize()
    L.hj_debug_set_trace(None, 0, 0)
hb = buf.cpu().numpy()
t = hb[: 8 * cap].reshape(-1, 8)[: rep["iterations"]].astype(np.float64)
raw = hb[: 8 * cap].reshape(-1, 8)[: rep["iterations"], 3]
arr = hb[8 * cap:(8 + 256) * cap].reshape(-1, 256)[: rep["iterations"]].astype(np.float64)
ncta = int((arr[0] > 0).sum())
arr = arr[:, :ncta]
last = arr.max(axis=1)
spread = (last - arr.min(axis=1)) / 1e3
b0late = (last - arr[:, 0]) / 1e3
bar = (t[:, 2] - last) / 1e3
items = (raw & 0xffff).astype(np.float64)
scan = (raw >> 16).astype(np.float64) / 1e3
work = (t[:, 1] - t[:, 0]) / 1e3
sync = (t[:, 2] - t[:, 1]) / 1e3
gap = (t[1:, 0] - t[:-1, 2]) / 1e3
ts = t[:, 0] + raw.astype(np.float64) // 65536
has = t[:, 4] > 0
ph = {"w0 load us": (t[:, 4] - ts), "w0 eval us": (t[:, 5] - t[:, 4]),
      "w0 mark us": (t[:, 6] - t[:, 5]), "cta wait us": (t[:, 7] - t[:, 6]),
      "reduce us": (t[:, 1] - t[:, 7])}
ph = {k: v[has] / 1e3 for k, v in ph.items()}
print(f"sweeps {len(t)}  total {(t[-1, 2] - t[0, 0]) / 1e6:.2f} ms  device {rep['device_ms']:.2f} ms")
for name, x in (("block0 items", items), ("block0 scan us", scan), ("block0 work us", work),
                ("sync us", sync), ("post-sync us", gap),
                ("arrival spread us", spread), ("last - block0 us", b0late),
                ("barrier after last us", bar), *ph.items()):
    print(f"{name:15s} mean {x.mean():8.2f}  med {np.median(x):8.2f}  max {x.max():8.2f}")
for k in (0, 100, 300, 500, 700):
    if k < len(t):
        print(f"  sweep {k}: items {int(items[k])} work {work[k]:.1f} us sync {sync[k]:.1f} us")
# which CTAs arrive last: per-CTA mean lateness (arrival - mean arrival of the sweep)
late = (arr - arr.mean(axis=1, keepdims=True)) / 1e3
ml = late.mean(axis=0)
order = np.argsort(ml)
print("CTA lateness us: earliest", [(int(i), round(float(ml[i]), 2)) for i in order[:4]],
      "latest", [(int(i), round(float(ml[i]), 2)) for i in order[-4:]],
      "std of per-CTA means", round(float(ml.std()), 2), "mean per-sweep std",
      round(float(late.std(axis=1).mean()), 2))
