"""Dev timing of the fused line-contact step (configs 1 and 3)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2008_03276_b200.ehl import EhlParams, LineContactBatch, moes_convert

def params(m, l):
    u, w = moes_convert(m=m, l=l, g=5000.0)
    return EhlParams.line_from_loads(5000.0, u, w, domain=(-4.5, 1.5))

for exact in (True, False):
    b = LineContactBatch([params(20.0, 10.0)], 512, exact=exact)
    for _ in range(5): b.step()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(200): b.step()
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 200
    print(f"config1 exact={exact}: {ms*1e3:.1f} us/iter, {1e3/ms:.0f} iters/s", flush=True)

rng = np.random.default_rng(3)
Ms = np.exp(rng.uniform(np.log(5), np.log(200), 1024)); Ls = rng.uniform(5, 15, 1024)
ps = [params(m, l) for m, l in zip(Ms, Ls)]
for exact in (True, False):
    b = LineContactBatch(ps, 1024, exact=exact)
    for _ in range(3): b.step()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5): b.step()
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 5
    info = b.info.cpu().numpy()
    print(f"config3 exact={exact}: {ms:.3f} ms/iter, {1024*1e3/ms:.3e} case-iters/s, ladder cases {(info & 3 > 0).sum()}", flush=True)
