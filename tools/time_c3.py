"""Time config 3 (1024 line contacts, N = 1025) per outer iteration on both
line paths, exact and FMA (device events)."""
import sys
import os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
from paper_2008_03276_b200.ehl import LineContactBatch

cases = bench.config3_cases(0)
ps = [bench._line_params(m, l) for m, l in cases]
for path in (sys.argv[1:] or ["split", "fused"]):
    for exact in (True, False):
        b = LineContactBatch(ps, 1024, exact=exact, path=path)
        for _ in range(3):
            b.step()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(5):
            b.step()
        e1.record()
        e1.synchronize()
        print(f"{path:6s} exact={exact}: {e0.elapsed_time(e1) / 5:.3f} ms/iter", flush=True)
