"""Dev: per-case cycles / SM schedule of one config-3 launch (PAQIF_LINE_PROF build)."""
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
for _ in range(4): b.step()
torch.cuda.synchronize()
