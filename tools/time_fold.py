"""Dev timing of one full 2-D deformation fold per grid size: kernel time
from the CUPTI trace (torch.profiler), set_state wall time beside it."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from torch.profiler import profile, ProfilerActivity
from paper_2008_03276_b200.ehl import EhlParams, PointContact
for n in (512, 2048):
    p = EhlParams.point_from_moes(100.0, 10.0, domain=(-4.5, 1.5), lo_y=-3.0)
    pc = PointContact(p, n)
    u = pc.snapshot()["u"]
    pc.set_state(u, -0.5)
    t0 = time.perf_counter()
    for _ in range(5):
        pc.set_state(u, -0.5)
    dt = (time.perf_counter() - t0) / 5
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        for _ in range(5):
            pc.set_state(u, -0.5)
        torch.cuda.synchronize()
    ks = [e for e in prof.events() if "fft_conv" in e.name]
    kt = sum(e.device_time for e in ks) / max(1, len(ks))
    print(f"n={n}: set_state (H2D + one fold) {dt*1e3:.2f} ms; fold kernel {kt/1e3:.3f} ms"
          f" ({len(ks)} launches)", flush=True)
