"""A/B check of the LCP kernel on the config-2 workload (dev tool): exact vs
FMA arithmetic -- agreement (passes, active sets, values) and timing."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2008_03276_b200.batch import LcpSolver
from paper_2008_03276_b200.workloads import lcp_batch as gen

B = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
bands, f = gen(2024, B)
tb = torch.from_numpy(bands).cuda(); tf = torch.from_numpy(f).cuda()
res = {}
for name, exact in (("exact", True), ("fma", False)):
    s = LcpSolver(B, 1026, 8, exact)
    for _ in range(2): s.launch(tb, tf)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5): s.launch(tb, tf)
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 5
    res[name] = [t.cpu().numpy().copy() for t in (s.u, s.active, s.passes, s.status, s.res)]
    print(f"{name}: {ms:.3f} ms  rows/s={B*1025/(ms*1e-3):.3e}  passes mean {res[name][2].mean():.3f} "
          f"max {res[name][2].max()}  status max {res[name][3].max()}", flush=True)
u0, a0, p0, s0, r0 = res["exact"]
u, a, p, s, r = res["fma"]
rel = np.abs(u - u0).max() / max(np.abs(u0).max(), 1e-300)
print(f"fma vs exact: max rel {rel:.3e} same passes {np.array_equal(p, p0)} "
      f"same active {np.array_equal(a, a0)} same status {np.array_equal(s, s0)}")
