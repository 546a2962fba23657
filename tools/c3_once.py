"""Dev: one config-3 batch step on the split path (ncu target:
line_split_*_kernel).  usage: c3_once.py [exact|fma]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
from paper_2008_03276_b200.ehl import LineContactBatch
ps = [bench._line_params(m, l) for m, l in bench.config3_cases(0)]
b = LineContactBatch(ps, 1024, exact=(sys.argv[1:] or ["exact"])[0] == "exact", path="split")
b.step()
torch.cuda.synchronize()
print("ok")
