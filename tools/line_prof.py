"""Dev: phase cycles of the fused line step (build with
PAQIF_NVCC_EXTRA=-DPAQIF_LINE_PROF; case 0 prints per launch)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2008_03276_b200.ehl import EhlParams, LineContactBatch, moes_convert
def params(m, l):
    u, w = moes_convert(m=m, l=l, g=5000.0)
    return EhlParams.line_from_loads(5000.0, u, w, domain=(-4.5, 1.5))
b = LineContactBatch([params(20.0, 10.0)], 512)
for _ in range(3): b.step()
torch.cuda.synchronize()
rng = np.random.default_rng(3)
ps = [params(m, l) for m, l in zip(np.exp(rng.uniform(np.log(5), np.log(200), 148)), rng.uniform(5, 15, 148))]
b = LineContactBatch(ps, 1024)
for _ in range(3): b.step()
torch.cuda.synchronize()
