"""Dev: CUPTI trace of one point sweep -- per-kernel totals and idle gaps."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from torch.profiler import profile, ProfilerActivity
from paper_2008_03276_b200.ehl import EhlParams, PointContact
n = int(sys.argv[1]) if len(sys.argv) > 1 else 512
p = EhlParams.point_from_moes(100.0 if n <= 512 else 1000.0, 10.0, domain=(-4.5, 1.5), lo_y=-3.0)
pc = PointContact(p, n)
pc.step(); pc.sync()
for name, fn in (("x", lambda: pc.sweep(0)), ("y", lambda: pc.sweep(3, 0, 0))):
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        fn(); pc.sync()
    ev = sorted([e for e in prof.events() if e.device_type.name == "CUDA"], key=lambda e: e.time_range.start)
    agg = {}
    for e in ev:
        k = e.name.split("<")[0].split("(")[0]
        a = agg.setdefault(k, [0, 0.0])
        a[0] += 1; a[1] += e.device_time
    span = ev[-1].time_range.end - ev[0].time_range.start
    busy = sum(e.device_time for e in ev)
    print(f"{name}-sweep n={n}: span {span/1e3:.1f} ms, kernels {busy/1e3:.1f} ms, gaps {(span-busy)/1e3:.1f} ms")
    for k, (c, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
        print(f"   {c:6d} {t/1e3:9.2f} ms  {t/c:8.1f} us/launch  {k}")
