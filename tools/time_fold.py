"""Dev timing of one full 2-D deformation fold (set_state) per grid size."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2008_03276_b200.ehl import EhlParams, PointContact
for n in (512, 2048):
    p = EhlParams.point_from_moes(100.0, 10.0, domain=(-4.5, 1.5), lo_y=-3.0)
    pc = PointContact(p, n)
    u = pc.snapshot()["u"]
    st = torch.cuda.ExternalStream(pc.stream_handle())
    pc.set_state(u, -0.5)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    for _ in range(5):
        pc.set_state(u, -0.5)
    dt = (time.perf_counter() - t0) / 5
    print(f"n={n}: set_state (H2D + one fold) {dt*1e3:.2f} ms", flush=True)
