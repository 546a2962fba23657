"""Dev: solve_ehl with device-side stop tests vs the per-iteration host loop."""
import time, sys
sys.path.insert(0, "/root/repo")
from paper_2008_03276_b200.ehl import solve_ehl, EhlParams, moes_convert
from paper_2008_03276_b200.errors import NonConvergenceError
u_, w_ = moes_convert(m=20.0, l=10.0, g=5000.0)
p = EhlParams.line_from_loads(5000.0, u_, w_, domain=(-4.5, 1.5))
for collect in (None, lambda *a: None, None):
    t0 = time.perf_counter()
    try: solve_ehl(p, 512, tol=0.0, tol_fb=0.0, max_outer=400, collect=collect)
    except NonConvergenceError: pass
    print("collect" if collect else "device", (time.perf_counter()-t0)/400*1e6, "us/iter")
