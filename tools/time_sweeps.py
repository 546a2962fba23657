"""Dev timing: x-sweep vs y-sweep vs residual of the point contact."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2008_03276_b200.ehl import EhlParams, PointContact
n = int(sys.argv[1]) if len(sys.argv) > 1 else 512
p = EhlParams.point_from_moes(100.0 if n <= 512 else 1000.0, 10.0, domain=(-4.5, 1.5), lo_y=-3.0)
pc = PointContact(p, n)
pc.step(); pc.sync()
st = torch.cuda.ExternalStream(pc.stream_handle())
for name, fn in (("x-sweep (hybrid)", lambda: pc.sweep(0)), ("y-sweep", lambda: pc.sweep(3, 0, 0)),
                 ("residual", lambda: pc.L.paqif_ehl_point_residual(pc._h.ptr))):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st); fn(); e1.record(st); e1.synchronize()
    print(f"{name}: {e0.elapsed_time(e1):.1f} ms", flush=True)
