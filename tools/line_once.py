"""Dev: config-3 line batch steps (ncu target: ehl_line_kernel)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2008_03276_b200.ehl import EhlParams, LineContactBatch, moes_convert
def params(m, l):
    u, w = moes_convert(m=m, l=l, g=5000.0)
    return EhlParams.line_from_loads(5000.0, u, w, domain=(-4.5, 1.5))
rng = np.random.default_rng(3)
ps = [params(m, l) for m, l in zip(np.exp(rng.uniform(np.log(5), np.log(200), 1024)), rng.uniform(5, 15, 1024))]
b = LineContactBatch(ps, 1024)
for _ in range(3): b.step()
torch.cuda.synchronize()
print("ok")
