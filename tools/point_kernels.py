"""Dev: one config-4 / config-5 outer iteration (ncu launch-list target for
the per-kernel split of the point contact: films, x/y line kernels, folds).
usage: point_kernels.py [n]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2008_03276_b200.ehl import EhlParams, PointContact
n = int(sys.argv[1]) if len(sys.argv) > 1 else 512
m = 100.0 if n <= 512 else 1000.0
pc = PointContact(EhlParams.point_from_moes(m, 10.0, domain=(-4.5, 1.5), lo_y=-3.0), n)
pc.step()
pc.sync()
print("ok", pc.status())
