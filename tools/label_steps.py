import sys, os
sys.path.insert(0, os.getcwd())
import torch
import hj_workloads as W
from paper_1405_3521_b200 import hj, pipeline
cfg = W.make(2)
res = pipeline.run_isa(cfg, cfg.dtype)
st = res["labels"]["steps"].float()
print("steps mean", st.mean().item(), "max", st.max().item(), "nodes", st.numel(), "sum", st.sum().item())
