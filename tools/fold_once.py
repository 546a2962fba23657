"""Dev: folds at 2049^2 (ncu target: fft_conv_kernel)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2008_03276_b200.ehl import EhlParams, PointContact
n = int(sys.argv[1]) if len(sys.argv) > 1 else 2048
pc = PointContact(EhlParams.point_from_moes(1000.0, 10.0, domain=(-4.5, 1.5), lo_y=-3.0), n)
u = pc.snapshot()["u"]
for _ in range(3):
    pc.set_state(u, -0.5)
print("ok")
