"""Dev: CUPTI trace of config-3 line steps (kernel durations and gaps)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from torch.profiler import profile, ProfilerActivity
from paper_2008_03276_b200.ehl import EhlParams, LineContactBatch, moes_convert
def params(m, l):
    u, w = moes_convert(m=m, l=l, g=5000.0)
    return EhlParams.line_from_loads(5000.0, u, w, domain=(-4.5, 1.5))
rng = np.random.default_rng(3)
ps = [params(m, l) for m, l in zip(np.exp(rng.uniform(np.log(5), np.log(200), 1024)), rng.uniform(5, 15, 1024))]
b = LineContactBatch(ps, 1024)
for _ in range(3): b.step()
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    for _ in range(5): b.step()
    torch.cuda.synchronize()
ev = sorted([e for e in prof.events() if e.device_type.name == "CUDA"], key=lambda e: e.time_range.start)
for e in ev: print(f"{e.time_range.start/1e3:10.3f} ms  {e.device_time/1e3:8.3f} ms  {e.name[:60]}")
