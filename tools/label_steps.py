"""Feedback-trajectory statistics of one ISA pass (steps per coarse node), for sizing the
labelling kernel: python tools/label_steps.py [CONFIG]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import hj_workloads as W  # noqa: E402
from paper_1405_3521_b200 import pipeline  # noqa: E402

idx = int(sys.argv[1]) if len(sys.argv) > 1 else 2
cfg = W.make(idx)
res = pipeline.run_isa(cfg, cfg.dtype)
st = res["labels"]["steps"].float()
print(f"config {idx}: trajectory steps mean {st.mean().item():.1f} max {st.max().item():.0f} "
      f"over {st.numel()} coarse nodes (total {st.sum().item():.0f})")
