"""Dev timing of the point-contact outer iteration (configs 4 and 5)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2008_03276_b200.ehl import EhlParams, PointContact

sizes = [int(a) for a in sys.argv[1:]] or [512, 2048]
for n, m, iters in ((512, 100.0, 5), (2048, 1000.0, 2)):
    if n not in sizes:
        continue
    p = EhlParams.point_from_moes(m, 10.0, domain=(-4.5, 1.5), lo_y=-3.0)
    for exact in (True, False):
        pc = PointContact(p, n, exact=exact)
        pc.step(); pc.sync()
        t0 = time.perf_counter()
        for _ in range(iters):
            pc.step()
        t_enq = time.perf_counter() - t0
        pc.sync()
        dt = (time.perf_counter() - t0) / iters
        s = pc.snapshot()
        print(f"n={n} exact={exact}: {dt*1e3:.1f} ms/iter (enqueue {t_enq/iters*1e3:.1f} ms), "
              f"res {s['res']:.4g}, newton lines {int(s['newton'].sum())}/{n-1}, "
              f"x rungs>0 {(s['x_rungs'] > 0).sum()}, y rungs>0 {(s['y_rungs'] > 0).sum()}",
              flush=True)
        pc.close()
if "--cpu" in sys.argv or os.environ.get("TIME_CPU"):
    import oracle.ehl_point_oracle as P
    c = P.point_case(100.0, 10.0)
    f = P.PointFilm(512, c)
    u = P.hertz_start(c, f)
    t0 = time.perf_counter()
    P.point_step(u, c.h0, 0, c, f)
    print(f"oracle n=512: {time.perf_counter() - t0:.2f} s/iter", flush=True)
